"""One decode-GEMV configuration, launched back to back from the library (for ncu).

  python tools/gemv_one.py <shape> <n_groups> <path: 3 pair | 4 dep> [reps]
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

shapes = {"mixtral": (4096, 14336), "deepseek": (2048, 1408), "qwen2": (3584, 2560)}
H, I = shapes[sys.argv[1]]
n, path = int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
eb = 3 * H * I * 2
n_slots = max(2 * n, int(4 * 126e6 // eb) + n)
pool = (torch.randn((n_slots, 3 * H * I), device="cuda") * 0.02).to(torch.bfloat16)
x = torch.randn((n, H), device="cuda").to(torch.bfloat16)
h = torch.empty((n, I), dtype=torch.bfloat16, device="cuda")
out = torch.empty((n, H), device="cuda")
ms = C.c_float()
_lib.check(_lib.lib.hm_bench_expert_ffn(pool.data_ptr(), n_slots, H, I, n, 1, x.data_ptr(), h.data_ptr(),
                                        out.data_ptr(), path, reps, torch.cuda.current_stream().cuda_stream,
                                        C.byref(ms)))
print(f"{sys.argv[1]} n={n} path={path}: {1e3 * ms.value:.2f} us, {n * eb / (ms.value * 1e-3) / 1e9:.0f} GB/s")
