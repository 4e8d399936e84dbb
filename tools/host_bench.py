"""Host worker GB/s for one Mixtral-shaped expert at decode (M=1), per thread count."""
import ctypes as C
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
for nt in [int(a) for a in (sys.argv[1:] or ["16", "12", "8"])]:
    pool = C.c_void_p()
    lib.hm_cpu_pool_create(nt, C.byref(pool))
    bw = C.c_double()
    lib.hm_host_read_bw(pool, store.ctypes.data, store.nbytes, 3, C.byref(bw))
    for m in (1, 2):
        lib.hm_cpu_expert(pool, store[0].ctypes.data, H, I, x.ctypes.data, m, out.ctypes.data)
        t = time.perf_counter()
        reps = 16
        for r in range(reps):
            lib.hm_cpu_expert(pool, store[r % n_img].ctypes.data, H, I, x.ctypes.data, m, out.ctypes.data)
        dt = (time.perf_counter() - t) / reps
        print(f"threads {nt} M={m}: {dt * 1e3:.3f} ms/expert, {store[0].nbytes / dt / 1e9:.1f} GB/s "
              f"(stream-read peak {bw.value:.1f} GB/s)", flush=True)
    lib.hm_cpu_pool_destroy(pool)
