#!/bin/bash
# All BASELINE.json configs on one GPU (GPU box): Mixtral / DeepSeek / Qwen2 (10/25/50 %), plus the baselines.
out=${1:-gpurun_out/configs}
mkdir -p $out
timeout 900 python bench.py --shape mixtral --steps 8 > $out/mixtral_25.json 2> $out/mixtral_25.err
timeout 900 python bench.py --shape mixtral --steps 8 --prefetch --no-cpu-baseline > $out/mixtral_25_prefetch.json 2> $out/mixtral_25_prefetch.err
timeout 900 python bench.py --shape deepseek --steps 16 > $out/deepseek_25.json 2> $out/deepseek_25.err
timeout 900 python bench.py --shape deepseek --steps 16 --prefetch --no-cpu-baseline > $out/deepseek_25_prefetch.json 2> $out/deepseek_25_prefetch.err
for r in 0.1 0.25 0.5; do
  timeout 900 python bench.py --shape qwen2 --ratio $r --steps 8 --prefetch --no-cpu-baseline > $out/qwen2_$r.json 2> $out/qwen2_$r.err
done
for s in fixed_frequency_map gpu_ondemand static_layer_split; do
  timeout 900 python bench.py --shape mixtral --scheduling $s --steps 6 --no-cpu-baseline > $out/mixtral_$s.json 2> $out/mixtral_$s.err
done
timeout 600 python bench.py --impl reference --shape mixtral --steps 4 > $out/reference_mixtral.json 2> $out/reference_mixtral.err
