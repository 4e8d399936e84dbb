"""Host worker GB/s for Mixtral-shaped experts at decode (M=1): single expert and
a layer's batch of 2, per thread count (prefetch knobs via HM_PF_DIST / HM_PF_HINT)."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

H, I = 4096, 14336
n_img = 8
lib = _lib.lib
store = np.random.default_rng(0).integers(0, 1 << 14, size=(n_img, 3 * H * I), dtype=np.uint16)
x = np.full((4, H), 0x3F80, np.uint16)
out = np.empty((4, H), np.float32)
tag = f"dist={os.environ.get('HM_PF_DIST', 'def')} hint={os.environ.get('HM_PF_HINT', 'def')}"
for nt in [int(a) for a in (sys.argv[1:] or ["16"])]:
    pool = C.c_void_p()
    lib.hm_cpu_pool_create(nt, C.byref(pool))
    bw = C.c_double()
    lib.hm_host_read_bw(pool, store.ctypes.data, store.nbytes, 3, C.byref(bw))
    lib.hm_cpu_expert(pool, store[0].ctypes.data, H, I, x.ctypes.data, 1, out.ctypes.data)
    reps = 16
    t = time.perf_counter()
    for r in range(reps):
        lib.hm_cpu_expert(pool, store[r % n_img].ctypes.data, H, I, x.ctypes.data, 1, out.ctypes.data)
    dt = (time.perf_counter() - t) / reps
    imgs = (C.c_void_p * 2)()
    xs = (C.c_void_p * 2)(x[0:1].ctypes.data, x[1:2].ctypes.data)
    outs = (C.c_void_p * 2)(out[0:1].ctypes.data, out[1:2].ctypes.data)
    t = time.perf_counter()
    for r in range(reps // 2):
        imgs[0], imgs[1] = store[(2 * r) % n_img].ctypes.data, store[(2 * r + 1) % n_img].ctypes.data
        lib.hm_cpu_experts_decode(pool, imgs, xs, 2, H, I, outs)
    dt2 = (time.perf_counter() - t) / reps
    print(f"[{tag}] threads {nt}: single {dt * 1e3:.3f} ms/expert {store[0].nbytes / dt / 1e9:.1f} GB/s | "
          f"batch-2 {dt2 * 1e3:.3f} ms/expert {store[0].nbytes / dt2 / 1e9:.1f} GB/s | "
          f"stream-read {bw.value:.1f} GB/s", flush=True)
    lib.hm_cpu_pool_destroy(pool)
