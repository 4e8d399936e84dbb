timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2j_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r2j_pytest.log
timeout 600 python tools/gemv_lib_bench.py 40 deepseek,qwen2,mixtral 1,2,4,6,8 > gpurun_out/r2j_gemv.log 2>&1; echo gemv rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ffn[12] --csv python tools/gemv_lib_bench.py 3 deepseek,mixtral 1,4,6 > gpurun_out/r2j_ncu.csv 2>&1; echo ncu rc=$?
timeout 300 python tools/tail_bench.py > gpurun_out/r2j_tail.json 2>&1; echo tail rc=$?
