"""Why are one-expert decode calls slower per byte than two-expert calls?
Interleaved variants on pinned Mixtral/DeepSeek images: n=1, n=2, n=2 with the
same image twice, n=1 on a pool of 8 threads, grain 0 vs 16.

  python tools/host_n_ab.py [calls]
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
calls = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pools = {}
for nt in (16, 8):
    p = C.c_void_p()
    lib.hm_cpu_pool_create(nt, C.byref(p))
    pools[nt] = p
for name, H, I, n_img in (("mixtral", 4096, 14336, 8), ("deepseek", 2048, 1408, 96)):
    elems = 3 * H * I
    t = torch.empty((n_img, elems), dtype=torch.int16).pin_memory()
    t.random_(0, 1 << 14)
    x = np.full((2, H), 0x3F80, np.uint16)
    out = np.empty((2, H), np.float32)
    xs = (C.c_void_p * 2)(x[0:1].ctypes.data, x[1:2].ctypes.data)
    outs = (C.c_void_p * 2)(out[0:1].ctypes.data, out[1:2].ctypes.data)
    variants = [("n1", 1, False, 16, 16), ("n2", 2, False, 16, 16), ("n2same", 2, True, 16, 16),
                ("n1-pool8", 1, False, 8, 16), ("n1-grain0", 1, False, 16, 0), ("n2-grain0", 2, False, 16, 0)]
    res = {v[0]: [] for v in variants}
    k = 0
    reps = calls if name == "mixtral" else calls * 8
    for r in range(reps):
        for vname, n, same, nt, grain in variants:
            lib.hm_cpu_set_decode_grain(grain)
            imgs = (C.c_void_p * 2)()
            imgs[0] = t[k % n_img].data_ptr()
            imgs[1] = imgs[0] if same else t[(k + 1) % n_img].data_ptr()
            k += 2
            t0 = time.perf_counter()
            lib.hm_cpu_experts_decode(pools[nt], imgs, xs, n, H, I, outs)
            dt = time.perf_counter() - t0
            res[vname].append(n * elems * 2 / dt / 1e9)
    lib.hm_cpu_set_decode_grain(16)
    print(name, " | ".join(f"{v} {np.median(g):6.1f}" for v, g in res.items()), flush=True)
    t = None
