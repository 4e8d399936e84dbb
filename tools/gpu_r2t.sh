# bulk-copy GEMV: bit-identity test + A/B against the register pair
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x -k "bulk or fused_gemv or deepseek or mixtral_shape" > gpurun_out/r2t_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2t_pytest.log
timeout 600 python tools/gemv_lib_bench.py 30 deepseek,qwen2,mixtral 1,2,4,6,8 2>&1 | tail -20; echo bench rc=$?
HM_BULK_SMEM_KB=100 timeout 600 python tools/gemv_lib_bench.py 30 deepseek,mixtral 2,6,8 2>&1 | tail -8
HM_BULK_SMEM_KB=128 timeout 600 python tools/gemv_lib_bench.py 30 deepseek,mixtral 2,6,8 2>&1 | tail -8
