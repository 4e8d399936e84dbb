#!/bin/bash
# ncu durations of the decode GEMV kernels: two-launch (HM_GEMV_FUSED=0) vs fused (1).
out=${1:-gpurun_out/gemv_ab}
mkdir -p $out
for f in 0 1; do
  HM_GEMV_FUSED=$f timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
    -k regex:"gemv" --csv --log-file $out/f$f.csv python tools/kernels_main.py gemv 3 > $out/f$f.json 2>&1
done
