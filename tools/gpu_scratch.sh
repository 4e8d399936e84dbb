timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_qwen2_shape_gpu.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r3_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r3_pytest.log
timeout 600 python tools/gemv_lib_bench.py 30 deepseek,qwen2 > gpurun_out/r3_gemv.log 2>&1; echo gemv rc=$?
cat gpurun_out/r3_gemv.log | tail -20
