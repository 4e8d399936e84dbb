"""Host worker on 4-bit expert images: ms per expert at decode loads 1-4 (GB/s of
4-bit bytes), next to a stream-read of the same host memory."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))
res = {}
for name, H, I in (("mixtral", 4096, 14336), ("deepseek", 2048, 1408)):
    nb = C.c_size_t()
    lib.hm_q4_image_bytes(H, I, C.byref(nb))
    n_img = 8 if name == "mixtral" else 64
    store = np.random.default_rng(0).integers(0, 255, size=(n_img, nb.value), dtype=np.uint8)
    # valid bf16 scales (0.01) so the arithmetic is representative
    hi = H * I
    s_off = hi + hi // 2
    store[:, s_off:].view(np.uint16)[:] = 0x3C23
    bw = C.c_double()
    lib.hm_host_read_bw(pool, store.ctypes.data, store.nbytes, 2, C.byref(bw))
    for M in (1, 2, 4):
        x = np.full((M, H), 0x3F80, np.uint16)
        out = np.empty((M, H), np.float32)
        ts = []
        for r in range(12):
            t = time.perf_counter()
            _lib.check(lib.hm_cpu_expert_q4(pool, store[r % n_img].ctypes.data, H, I, x.ctypes.data, M,
                                            out.ctypes.data))
            ts.append(time.perf_counter() - t)
        t = float(np.median(ts[2:]))
        res[f"{name}-M{M}"] = {"ms": round(1e3 * t, 3), "gbs": round(nb.value / t / 1e9, 1),
                               "stream_read_gbs": round(bw.value, 1)}
print(json.dumps(res))
lib.hm_cpu_pool_destroy(pool)
