timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x -k "splitk" > gpurun_out/r2ai_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/r2ai_pytest.log
GEMV_PATHS=split,splitk timeout 300 python tools/gemv_lib_bench.py 40 deepseek,qwen2,mixtral 1,2,4,6,8 2>&1 | tail -16
