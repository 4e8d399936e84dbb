"""Per-thread phase timeline of hm_cpu_experts_decode (hm_cpu_decode_profile):
start skew, phase-1 spread, barrier wait and phase-2 spread for DeepSeek /
Mixtral single-token calls on pinned images, medians over many calls.

  python tools/host_phase_prof.py
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
import os
NT = int(os.environ.get("NT", os.cpu_count()))
pool = C.c_void_p()
lib.hm_cpu_pool_create(NT, C.byref(pool))
prof = np.zeros((NT, 4), np.int64)
CASES = (("deepseek", 2048, 1408, 96, (1, 2, 3, 4), 300), ("mixtral", 4096, 14336, 8, (1,), 30),
         ("qwen2", 3584, 2560, 48, (1, 2, 3, 4), 100))
ONLY = os.environ.get("ONLY")  # e.g. deepseek:1,2
if ONLY:
    nm, cs = ONLY.split(":")
    CASES = tuple((c[0], c[1], c[2], c[3], tuple(int(v) for v in cs.split(",")), c[5]) for c in CASES if c[0] == nm)
Q4 = os.environ.get("Q4") == "1"  # 4-bit images through hm_cpu_experts_decode_q4 (wall time only)
for name, H, I, n_img, counts, calls in CASES:
    elems = 3 * H * I
    if Q4:
        nb = C.c_size_t()
        lib.hm_q4_image_bytes(H, I, C.byref(nb))
        elems = nb.value // 2
        n_img *= 4
    t = torch.empty((n_img, elems), dtype=torch.int16)
    if torch.cuda.is_available():  # pinned like the runtime's master store
        t = t.pin_memory()
    t.random_(0, 1 << 14)
    if Q4:  # valid bf16 scales (0.01) after the nibbles
        t.view(torch.uint8)[:, H * I * 3 // 2:].view(torch.int16).fill_(0x3C23)
    for n in counts:
        x = np.full((n, H), 0x3F80, np.uint16)
        out = np.empty((n, H), np.float32)
        xs = (C.c_void_p * n)(*[x[i:i + 1].ctypes.data for i in range(n)])
        outs = (C.c_void_p * n)(*[out[i:i + 1].ctypes.data for i in range(n)])
        imgs = (C.c_void_p * n)()
        rec, walls = [], []
        lib.hm_cpu_decode_profile(1, None, 0)
        k = 0
        for r in range(calls):
            for i in range(n):
                imgs[i] = t[k % n_img].data_ptr()
                k += 1
            t0 = time.perf_counter()
            (lib.hm_cpu_experts_decode_q4 if Q4 else lib.hm_cpu_experts_decode)(pool, imgs, xs, n, H, I, outs)
            walls.append(time.perf_counter() - t0)
            lib.hm_cpu_decode_profile(1, prof.ctypes.data, NT)
            if r >= 3:
                rec.append(prof.copy())
            s0 = time.perf_counter() + 40e-6
            while time.perf_counter() < s0:
                pass
        a = np.array(rec) / 1e3  # us
        med = lambda v: float(np.median(v))  # noqa: E731
        print(f"{name} n={n}: wall {1e6 * med(walls):.1f} us | start max {med(a[:, :, 0].max(1)):.1f} | "
              f"phase1 min/med/max {med(a[:, :, 1].min(1)):.1f}/{med(np.median(a[:, :, 1], 1)):.1f}/"
              f"{med(a[:, :, 1].max(1)):.1f} | barrier passed {med(a[:, :, 2].max(1)):.1f} | "
              f"phase2 min/med/max {med(a[:, :, 3].min(1)):.1f}/{med(np.median(a[:, :, 3], 1)):.1f}/"
              f"{med(a[:, :, 3].max(1)):.1f} | GB/s {n * elems * 2 / med(walls) / 1e9:.1f}", flush=True)
    t = None
lib.hm_cpu_decode_profile(0, None, 0)
