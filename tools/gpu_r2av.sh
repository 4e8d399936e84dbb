# batched prefill experts A/B (TTFT), same box, interleaved
for r in 1 2 3; do for v in 1 0; do for sh in mixtral deepseek qwen2; do
HM_PREFILL_BATCH=$v timeout 600 python bench.py --shape $sh --extra-configs "" --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/r2av.out 2>/dev/null
python - <<PY
import json
d=json.loads([x for x in open("gpurun_out/r2av.out") if x.startswith("{")][-1])
print("batch=$v $sh run=$r prefill_ms %.1f predicted %.1f" % (d["prefill"]["ms"], d["model_vs_measured"]["predicted_ttft_ms"]))
PY
done; done; done
