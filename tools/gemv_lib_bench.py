"""Decode expert-FFN throughput from back-to-back launches issued inside the
library (hm_bench_expert_ffn: no Python between launches), weights rotating
over a slot set well above L2.

  python tools/gemv_lib_bench.py [reps] [shapes] [counts]
"""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
shapes = {"mixtral": (4096, 14336), "deepseek": (2048, 1408), "qwen2": (3584, 2560)}
if len(sys.argv) > 2:  # shape filter, e.g. `deepseek`
    shapes = {k: v for k, v in shapes.items() if k in sys.argv[2].split(",")}
counts = tuple(int(c) for c in sys.argv[3].split(",")) if len(sys.argv) > 3 else (1, 2, 4, 8, 16)
import os
paths = {k: v for k, v in {"split": 3, "bulk": 5, "fused": 4}.items()
         if k in os.environ.get("GEMV_PATHS", "split").split(",")}
res = {}
for name, (H, I) in shapes.items():
    eb = 3 * H * I * 2
    for n in counts:
        n_slots = min(max(2 * n, int(4 * 126e6 // eb) + n), max(2 * n, int(24e9 // eb)))
        pool = (torch.randn((n_slots, 3 * H * I), device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn((n, H), device="cuda").to(torch.bfloat16)
        h = torch.empty((n, I), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((n, H), device="cuda")
        row = {}
        for pname, path in paths.items():
            ms = C.c_float()
            _lib.check(_lib.lib.hm_bench_expert_ffn(pool.data_ptr(), n_slots, H, I, n, 1, x.data_ptr(), h.data_ptr(),
                                                    out.data_ptr(), path, reps,
                                                    torch.cuda.current_stream().cuda_stream, C.byref(ms)))
            row[pname] = {"us": round(1e3 * ms.value, 2), "gbs": round(n * eb / (ms.value * 1e-3) / 1e9, 1)}
        res[f"{name}-n{n}"] = row
        print(name, n, row, flush=True)
        del pool
        torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/gemv_paths.json").write_text(json.dumps(res))
