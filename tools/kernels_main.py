"""Standalone kernel runs for ncu captures and quick roofline checks (GPU box)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2504_05897_b200.microbench import gemm_bench, gemv_bench  # noqa: E402

shapes = {"mixtral": (4096, 14336), "deepseek": (2048, 1408), "qwen2": (3584, 2560)}
which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
res = {}
for name, (H, I) in shapes.items():
    if which in ("all", "gemv"):
        res[f"{name}-gemv-2"] = gemv_bench(H, I, n_experts=2, reps=reps)
        res[f"{name}-gemv-8"] = gemv_bench(H, I, n_experts=8, n_slots=16, reps=reps)
    if which in ("all", "gemm"):
        for m in (128, 256, 512):
            res[f"{name}-gemm-{m}"] = gemm_bench(H, I, rows_per_expert=m, n_experts=8, reps=max(2, reps // 4))
print(json.dumps(res, indent=1))
