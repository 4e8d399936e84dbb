"""Per-thread phase timeline of the host worker's AMX expert (hm_cpu_expert,
M >= 8, HM_AMX_ALGO=0 path): pack, phase 1 (W13 + SwiGLU), phase 2 (W2).

  python tools/amx_phase_prof.py [H I]
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
H, I = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 1408)))
NT = int(os.environ.get("NT", os.cpu_count()))
n_img = int(os.environ.get("N_IMG", "16"))
store = np.random.default_rng(0).integers(0x3000, 0x3c00, size=(n_img, 3 * H * I), dtype=np.uint16)
pool = C.c_void_p()
lib.hm_cpu_pool_create(NT, C.byref(pool))
prof = np.zeros((NT, 4), np.int64)
for M in (32, 64, 128, 256):
    x = np.full((M, H), 0x3F80, np.uint16)
    out = np.empty((M, H), np.float32)
    rec, walls = [], []
    lib.hm_cpu_decode_profile(1, None, 0)
    for r in range(12):
        t0 = time.perf_counter()
        _lib.check(lib.hm_cpu_expert(pool, store[r % n_img].ctypes.data, H, I, x.ctypes.data, M, out.ctypes.data))
        walls.append(time.perf_counter() - t0)
        lib.hm_cpu_decode_profile(1, prof.ctypes.data, NT)
        if r >= 2:
            rec.append(prof.copy())
    a = np.array(rec) / 1e3
    med = lambda v: float(np.median(v))  # noqa: E731
    fl = 2 * M * 3 * H * I
    print(f"M={M}: wall {1e6 * med(walls):.0f} us ({fl / med(walls) / 1e12:.2f} TF/s) | start max {med(a[:, :, 0].max(1)):.0f}"
          f" | packed {med(a[:, :, 1].max(1)):.0f} | ph1 min/med/max {med(a[:, :, 2].min(1)):.0f}/"
          f"{med(np.median(a[:, :, 2], 1)):.0f}/{med(a[:, :, 2].max(1)):.0f} | ph2 min/med/max "
          f"{med(a[:, :, 3].min(1)):.0f}/{med(np.median(a[:, :, 3], 1)):.0f}/{med(a[:, :, 3].max(1)):.0f}", flush=True)
lib.hm_cpu_decode_profile(0, None, 0)
