#!/bin/bash
# One-GPU ncu evidence for a round (run under gpurun): the whole-bench launch
# list and full captures of the dominant kernels.  Summarise here with
#   python tools/ncu_summary.py $out/*.ncu-rep --launches $out/launches.csv --out profiles/<round>_ncu_summary.md
out=${1:-gpurun_out/prof}
mkdir -p $out
P=profiles/b200_mixtral_profile.txt
# nothing may wait on the host under ncu's serialised kernel replay
export HM_TIMING_GATE=0 HM_ZERO_COPY=0
# launch list of a short bench run (fixed profile: no calibration under the profiler)
# (HM_NCU_TIMED=1 + --profile-from-start off: only the bench's timed decode steps are profiled)
HM_NCU_TIMED=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file $out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --extra-configs '' --no-refit --profile-file $P > $out/bench_under_ncu.log 2>&1
# decode GEMV (Mixtral, 2 experts: the 25 % budget's typical GPU batch), full set
for k in ffn1_gemv ffn2_gemv; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $out/$k \
    python tools/kernels_main.py gemv 3 > /dev/null 2>&1
done
# decode GEMV at the DeepSeek (6 experts) and Qwen2 (4 experts) shapes, full set (split pair, path 3)
for cfg in "deepseek 6" "qwen2 4"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffn[12]_gemv" -s 6 -c 2 -o $out/gemv_$1 \
    python tools/gemv_lib_bench.py 3 $1 $2 > /dev/null 2>&1
done
# prefill grouped GEMM (tcgen05): both modes of the 256-token Mixtral groups
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expert_gemm -s 2 -c 2 -o $out/expert_gemm \
  python tools/kernels_main.py gemm 2 > /dev/null 2>&1
# decode critical-path kernels (router mirror, combine tail)
TAIL_REPS=3 timeout 600 ncu --set full --clock-control none -k regex:"router_fused|combine_tail" -s 6 -c 2 -o $out/tail \
  python tools/tail_bench.py > /dev/null 2>&1
ls -la $out
