timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -m gpu -p no:cacheprovider -x -k "q4" > gpurun_out/r2v_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2v_pytest.log
timeout 600 python tools/q4_bench.py 1,2,4,6,8 > gpurun_out/r2v_q4.log 2>&1; echo q4 rc=$?
cat gpurun_out/r2v_q4.log
