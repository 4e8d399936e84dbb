set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_ep_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2b_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/r2b_pytest.log
timeout 600 python tools/gemv_lib_bench.py 40 deepseek,qwen2,mixtral 1,2,4,6,8 > gpurun_out/r2b_gemv.log 2>&1; echo gemv rc=$?
cat gpurun_out/r2b_gemv.log | tail -20
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ffn --csv python tools/gemv_lib_bench.py 3 deepseek 4,6 > gpurun_out/r2b_ncu_gemv.csv 2>&1; echo ncu rc=$?
tail -30 gpurun_out/r2b_ncu_gemv.csv
