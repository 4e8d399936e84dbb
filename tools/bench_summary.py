"""One-screen summary of a bench.py JSON line: python tools/bench_summary.py FILE"""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(line)
print("value", round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "ms/step", round(d["ms_per_step"], 2),
      "prefill ms", round(d["prefill"]["ms"], 1))
print("roofline frac", round(d["roofline"]["frac"], 3), "step_roofline", json.dumps(d["step_roofline"])[:300])
print("per_step", json.dumps(d["per_step"]))
print("model_vs_measured", {k: round(v, 3) for k, v in d["model_vs_measured"].items() if isinstance(v, float)})
print("cpu_baseline", (d.get("cpu_baseline") or {}).get("value"), "clocks", d["clocks"])
for k, v in d.get("configs", {}).items():
    sr = v.get("step_roofline", {})
    print(f"{k:12s} decode {v.get('decode_tok_s', 0):7.2f} e2e {v.get('e2e_tok_s', 0):7.2f} prefill {v.get('prefill_ms', 0):7.1f}"
          f" step_frac {sr.get('frac', 0):.3f} host_worker_gbs {sr.get('host_worker_gbs', 0):.0f} probe {sr.get('host_read_probe_gbs', 0):.0f}"
          f" cpu/gpu {v.get('per_step', {}).get('cpu_experts')}/{v.get('per_step', {}).get('gpu_experts')}")
