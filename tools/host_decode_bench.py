"""Host worker decode GB/s per model shape, A/B over the split granularity
(hm_cpu_set_decode_grain) with interleaved rounds and a stream-read reference.

  python tools/host_decode_bench.py [rounds]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
lib.hm_cpu_set_decode_grain.argtypes = [C.c_int]
# (name, H, I, experts per layer call, distinct images)
shapes = [("mixtral", 4096, 14336, 1, 6), ("mixtral", 4096, 14336, 2, 6), ("deepseek", 2048, 1408, 4, 64),
          ("qwen2", 3584, 2560, 4, 32)]
grains = [int(g) for g in __import__("os").environ.get("HM_BENCH_GRAINS", "0,16,64").split(",")]
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))
res = {}
for name, H, I, n, n_img in shapes:
    store = np.random.default_rng(0).integers(0, 1 << 14, size=(n_img, 3 * H * I), dtype=np.uint16)
    x = np.full((n, H), 0x3F80, np.uint16)
    out = np.empty((n, H), np.float32)
    xs = (C.c_void_p * n)(*[x[i:i + 1].ctypes.data for i in range(n)])
    outs = (C.c_void_p * n)(*[out[i:i + 1].ctypes.data for i in range(n)])
    imgs = (C.c_void_p * n)()
    for rnd in range(rounds):
        bw = C.c_double()
        lib.hm_host_read_bw(pool, store.ctypes.data, store.nbytes, 2, C.byref(bw))
        for g in (grains[rnd % len(grains):] + grains[:rnd % len(grains)]):  # rotate: no order bias
            lib.hm_cpu_set_decode_grain(g)
            reps = max(4, int(2e9 / (n * store[0].nbytes)))
            k = 0
            t = time.perf_counter()
            for r in range(reps):
                for i in range(n):
                    imgs[i] = store[k % n_img].ctypes.data
                    k += 1
                lib.hm_cpu_experts_decode(pool, imgs, xs, n, H, I, outs)
            dt = (time.perf_counter() - t) / reps
            res.setdefault((name, n, g), []).append((n * store[0].nbytes / dt / 1e9, bw.value, dt * 1e6))
    del store
for (name, n, g), r in res.items():
    gb = np.median([a for a, _, _ in r])
    sr = np.median([b for _, b, _ in r])
    us = np.median([c for _, _, c in r])
    print(f"{name:8s} n={n} grain {g:3d}: {gb:6.1f} GB/s ({us:8.1f} us/call) | stream-read {sr:6.1f} | ratio {gb / sr:.3f}")
lib.hm_cpu_pool_destroy(pool)
