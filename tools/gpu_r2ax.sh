timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -m gpu -p no:cacheprovider -x -k "q4" > gpurun_out/r2ax_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r2ax_pytest.log
for r in 1 2; do for v in 1 0; do echo "== PRESTAGE=$v"; HM_Q4_PRESTAGE=$v timeout 300 python tools/q4_bench.py 1,2,4,6 2>&1 | grep -E "^(mixtral|deepseek|qwen2)" | tr '\n' ' '; echo; done; done
