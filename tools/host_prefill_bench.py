"""Host worker (AMX) time per expert vs token count M (prefill-sized groups)."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
H, I = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 14336)))
n_img = int(__import__("os").environ.get("N_IMG", "16"))
store = np.random.default_rng(0).integers(0x3000, 0x3c00, size=(n_img, 3 * H * I), dtype=np.uint16)
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))
res = {}
for M in (8, 16, 32, 64, 128, 256, 512):
    x = np.full((M, H), 0x3F80, np.uint16)
    out = np.empty((M, H), np.float32)
    ts = []
    for r in range(8):
        t = time.perf_counter()
        _lib.check(lib.hm_cpu_expert(pool, store[r % n_img].ctypes.data, H, I, x.ctypes.data, M, out.ctypes.data))
        ts.append(time.perf_counter() - t)
    t = min(ts[1:])
    res[M] = {"ms": round(1e3 * t, 3), "tflops": round(2 * M * 3 * H * I / t / 1e12, 2),
              "gbs": round(store[0].nbytes / t / 1e9, 1)}
print(json.dumps(res))
lib.hm_cpu_pool_destroy(pool)
