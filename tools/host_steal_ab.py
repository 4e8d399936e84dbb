"""Interleaved A/B of decode work stealing (hm_cpu_set_decode_steal) on pinned
images: the arms alternate every call so host-bandwidth drift hits both alike;
plus the per-thread phase spread (hm_cpu_decode_profile) of each arm.

  python tools/host_steal_ab.py [calls]
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
NT = 16
calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
pool = C.c_void_p()
lib.hm_cpu_pool_create(NT, C.byref(pool))
prof = np.zeros((NT, 4), np.int64)
lib.hm_cpu_decode_profile(1, None, 0)
for name, H, I, n_img, counts, reps in (("mixtral", 4096, 14336, 8, (1, 2), calls // 8),
                                         ("deepseek", 2048, 1408, 96, (1, 2, 4), calls)):
    elems = 3 * H * I
    t = torch.empty((n_img, elems), dtype=torch.int16).pin_memory()
    t.random_(0, 1 << 14)
    for n in counts:
        x = np.full((n, H), 0x3F80, np.uint16)
        out = np.empty((n, H), np.float32)
        xs = (C.c_void_p * n)(*[x[i:i + 1].ctypes.data for i in range(n)])
        outs = (C.c_void_p * n)(*[out[i:i + 1].ctypes.data for i in range(n)])
        imgs = (C.c_void_p * n)()
        res = {0: [], 1: []}
        spread = {0: [], 1: []}
        k = 0
        for r in range(2 * reps + 4):
            arm = r % 2
            lib.hm_cpu_set_decode_steal(arm)
            for i in range(n):
                imgs[i] = t[k % n_img].data_ptr()
                k += 1
            t0 = time.perf_counter()
            lib.hm_cpu_experts_decode(pool, imgs, xs, n, H, I, outs)
            dt = time.perf_counter() - t0
            lib.hm_cpu_decode_profile(1, prof.ctypes.data, NT)
            if r >= 4:
                res[arm].append(n * elems * 2 / dt / 1e9)
                spread[arm].append((prof[:, 1].max() - np.median(prof[:, 1])) / 1e3)
            s0 = time.perf_counter() + 40e-6
            while time.perf_counter() < s0:
                pass
        print(f"{name:8s} n={n}: static {np.median(res[0]):6.1f} GB/s (phase-1 straggler +{np.median(spread[0]):6.1f} us)"
              f" | stealing {np.median(res[1]):6.1f} GB/s (+{np.median(spread[1]):6.1f} us)", flush=True)
    t = None
lib.hm_cpu_set_decode_steal(1)
lib.hm_cpu_decode_profile(0, None, 0)
