# 4-bit GEMV: L2 chunk prefetch + PDL A/B
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -m gpu -p no:cacheprovider -x -k "q4" > gpurun_out/r2aa_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2aa_pytest.log
for v in 1 0 1; do echo "== HM_Q4_L2PF=$v"; HM_Q4_L2PF=$v timeout 300 python tools/q4_bench.py 1,2,4,6,8 2>&1 | tail -15; done
