# narrow GEMV variants (one DRAM round trip per warp) A/B
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x -k "bulk or fused_gemv or deepseek or mixtral_shape or ffn" > gpurun_out/r2u_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2u_pytest.log
for v in "HM_GEMV_NARROW=0" "HM_GEMV_NARROW=1 HM_GEMV_NARROW_RPW=1" "HM_GEMV_NARROW=1 HM_GEMV_NARROW_RPW=2" "HM_GEMV_NARROW=1 HM_GEMV_NARROW_RPW=3"; do
echo "== $v"; env $v timeout 300 python tools/gemv_lib_bench.py 40 deepseek,qwen2 1,2,4,6,8 2>&1 | tail -10
done
