set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x -k "fused or gemv or deepseek or mixtral" > gpurun_out/r2d_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2d_pytest.log
HM_GEMV_MINB=4 timeout 600 python tools/gemv_lib_bench.py 40 deepseek,qwen2,mixtral 1,2,4,6,8 > gpurun_out/r2d_gemv4.log 2>&1; echo gemv rc=$?
cat gpurun_out/r2d_gemv4.log | tail -20
HM_GEMV_MINB=3 timeout 600 python tools/gemv_lib_bench.py 40 deepseek,qwen2,mixtral 1,2,4,6,8 > gpurun_out/r2d_gemv3.log 2>&1; echo gemv rc=$?
cat gpurun_out/r2d_gemv3.log | tail -20
