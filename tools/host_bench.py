"""Host worker GB/s for Mixtral-shaped experts at decode (M=1): interleaved
variants (prefetch distance/hint x thread count) in one process, each next to
a fresh stream-read measurement, so host-memory noise hits all variants alike.

  python tools/host_bench.py [rounds]
"""
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
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
variants = [(16, 16384, 2), (16, 0, 0), (16, 8192, 2), (16, 32768, 2), (16, 16384, 1), (16, 65536, 2),
            (15, 16384, 2)]
pools = {}
for nt in sorted({v[0] for v in variants}):
    p = C.c_void_p()
    lib.hm_cpu_pool_create(nt, C.byref(p))
    pools[nt] = p
res = {v: [] for v in variants}
for rnd in range(rounds):
    for v in variants:
        nt, dist, hint = v
        lib.hm_cpu_set_prefetch(dist, hint)
        bw = C.c_double()
        lib.hm_host_read_bw(pools[nt], store.ctypes.data, store.nbytes, 2, C.byref(bw))
        imgs = (C.c_void_p * 2)()
        xs = (C.c_void_p * 2)(x[0:1].ctypes.data, x[1:2].ctypes.data)
        outs = (C.c_void_p * 2)(out[0:1].ctypes.data, out[1:2].ctypes.data)
        reps = 12
        t = time.perf_counter()
        for r in range(reps // 2):
            imgs[0], imgs[1] = store[(2 * r) % n_img].ctypes.data, store[(2 * r + 1) % n_img].ctypes.data
            lib.hm_cpu_experts_decode(pools[nt], imgs, xs, 2, H, I, outs)
        dt = (time.perf_counter() - t) / reps
        res[v].append((store[0].nbytes / dt / 1e9, bw.value))
for v, r in res.items():
    gb = [a for a, _ in r]
    sr = [b for _, b in r]
    print(f"threads {v[0]:2d} pf_dist {v[1]:5d} hint {v[2]}: expert {np.median(gb):6.1f} GB/s "
          f"(min {min(gb):6.1f}) | stream-read {np.median(sr):6.1f} GB/s | ratio {np.median(gb) / np.median(sr):.2f}")
for p in pools.values():
    lib.hm_cpu_pool_destroy(p)
