"""Markdown table of a config sweep (tools/run_configs.sh output directory).

  python tools/configs_table.py gpurun_out/configs_r01b > profiles/r01b_configs/README.md
"""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
rows = []
for f in sorted(d.glob("*.json")):
    lines = [l for l in f.read_text().splitlines() if l.strip().startswith("{")]
    if not lines:
        rows.append(f"| {f.stem} | (no result) | | | | | | |")
        continue
    j = json.loads(lines[-1])
    if j.get("impl") == "reference":
        rows.append(f"| {f.stem} | {j['value']:.2f} tok/s (CPU oracle port, {j['cpu_baseline']['cores']} cores) "
                    f"| | | | | | |")
        continue
    ps = j.get("per_step", {})
    pf = j.get("prefill", {})
    rf = j.get("roofline", {})
    sr = j.get("step_roofline", {})
    cfg = j.get("config", {})
    rows.append(f"| {f.stem} | {j['value']:.2f} | {j['e2e']['value']:.2f} | {pf.get('ms', 0):.0f} | "
                f"{ps.get('gpu_experts', 0):.1f} / {ps.get('cpu_experts', 0):.1f} | "
                f"{sr.get('frac', 0):.2f} | {rf.get('frac', 0):.2f} | "
                f"{cfg.get('scheduling')}, prefetch={cfg.get('prefetch')}, ratio slots={cfg.get('cache_slots')} |")
print("| run | decode tok/s | e2e tok/s | prefill ms (1k tok) | GPU / CPU experts per token | step roofline frac | "
      "decode GEMV HBM frac | notes |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
