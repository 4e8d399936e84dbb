"""Interleaved A/B of the decode phase-barrier prefetch (hm_cpu_set_decode_bridge):
settings alternate every call on pinned images, so host-bandwidth drift on a
shared box hits both arms alike.

  python tools/host_bridge_ab.py [calls]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
calls = int(sys.argv[1]) if len(sys.argv) > 1 else 400
arms = (0, 256, 1024)
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))
for name, H, I, n_img, counts in (("deepseek", 2048, 1408, 96, (1, 2, 4)), ("mixtral", 4096, 14336, 8, (1, 2))):
    elems = 3 * H * I
    t = torch.empty((n_img, elems), dtype=torch.int16).pin_memory()
    t.random_(0, 1 << 14)
    for n in counts:
        x = np.full((n, H), 0x3F80, np.uint16)
        out = np.empty((n, H), np.float32)
        xs = (C.c_void_p * n)(*[x[i:i + 1].ctypes.data for i in range(n)])
        outs = (C.c_void_p * n)(*[out[i:i + 1].ctypes.data for i in range(n)])
        imgs = (C.c_void_p * n)()
        res = {a: [] for a in arms}
        reps = calls if name == "deepseek" else calls // 8
        k = 0
        for r in range(reps + len(arms)):
            a = arms[r % len(arms)]
            lib.hm_cpu_set_decode_bridge(a)
            for i in range(n):
                imgs[i] = t[k % n_img].data_ptr()
                k += 1
            t0 = time.perf_counter()
            lib.hm_cpu_experts_decode(pool, imgs, xs, n, H, I, outs)
            dt = time.perf_counter() - t0
            if r >= len(arms):
                res[a].append(dt)
            s0 = time.perf_counter() + 40e-6
            while time.perf_counter() < s0:
                pass
        line = " | ".join(f"bridge {a:4d}KB {n * elems * 2 / np.median(v) / 1e9:6.1f} GB/s" for a, v in res.items())
        print(f"{name:8s} n={n}: {line}", flush=True)
    t = None
lib.hm_cpu_pool_destroy(pool)
