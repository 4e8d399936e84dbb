"""Host stream-read GB/s per call size (hm_host_read_bw, one pass per call over
rotating, never-cached ranges of a 12 GB buffer): the fixed cost of one
all-threads read call, for the host worker's small-expert decode.

  python tools/host_read_sizes.py
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
NT = int(os.environ.get("NT", os.cpu_count()))
pool = C.c_void_p()
lib.hm_cpu_pool_create(NT, C.byref(pool))
total = int(os.environ.get("BUF_GB", "12")) << 30
t = torch.empty(total, dtype=torch.uint8)
if torch.cuda.is_available():
    t = t.pin_memory()
t.fill_(3)
base = t.data_ptr()
g = C.c_double()
for mb in (1, 2, 4, 8, 17, 35, 70, 140, 350):
    nbytes = mb << 20
    n_off = total // nbytes
    walls, k = [], 0
    for r in range(max(20, min(400, (4 << 30) // nbytes))):
        off = (k % n_off) * nbytes
        k += 7
        t0 = time.perf_counter()
        lib.hm_host_read_bw(pool, C.c_void_p(base + off), nbytes, 1, C.byref(g))
        walls.append(time.perf_counter() - t0)
    w = float(np.median(walls[3:]))
    print(f"{mb:4d} MB: {w * 1e6:8.1f} us/call  {nbytes / w / 1e9:6.1f} GB/s", flush=True)
