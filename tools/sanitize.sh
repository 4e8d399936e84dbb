#!/bin/bash
# compute-sanitizer passes over the GPU suite (one GPU; run under gpurun).
# Host-waiting kernels are ungated (HM_TIMING_GATE=0) so the tools' serialised
# execution cannot wait on the host.  Logs: gpurun_out/sanitizer_*.log
export HM_TIMING_GATE=0
compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py \
  -q -m gpu -p no:cacheprovider -x -k "not mixtral_shape and not deepseek_shape and not bulk" > gpurun_out/sanitizer_memcheck.log 2>&1
compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_runtime_gpu.py \
  tests/test_baselines_gpu.py tests/test_hf_pinned.py tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x \
  -k "not released_shapes and not mixtral_shape" > gpurun_out/sanitizer_memcheck_runtime.log 2>&1
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -p no:cacheprovider -x -k "router_parity or permute or expert_ffn_gemv or gemm_narrow or combine" \
  > gpurun_out/sanitizer_racecheck.log 2>&1
compute-sanitizer --tool synccheck python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -x \
  -k "router or permute or gemv or gemm or bulk" > gpurun_out/sanitizer_synccheck.log 2>&1
grep -h "SUMMARY" gpurun_out/sanitizer_*.log
