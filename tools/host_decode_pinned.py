"""Host worker decode GB/s on pageable (numpy) vs pinned (cudaHostAlloc, as the
runtime's master store) images, with and without a step-like idle gap between
calls -- DeepSeek / Mixtral shapes.

  python tools/host_decode_pinned.py
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
libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
cudart = torch.cuda.cudart()
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), flush=True)
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))


def spin(us):
    t = time.perf_counter() + us * 1e-6
    while time.perf_counter() < t:
        pass


for name, H, I, n_img in (("deepseek", 2048, 1408, 96), ("mixtral", 4096, 14336, 8)):
    elems = 3 * H * I
    for kind in __import__("os").environ.get("HM_KINDS", "numpy,pinned,thp_pinned").split(","):
        if kind == "numpy":
            store = np.random.default_rng(0).integers(0, 1 << 14, size=(n_img, elems), dtype=np.uint16)
            ptr = lambda i: store[i].ctypes.data  # noqa: E731
        elif kind == "thp_pinned":
            nbytes = n_img * elems * 2
            nb2 = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
            raw = libc.mmap(None, nb2 + (2 << 20), 3, 0x22, -1, 0)  # PROT_RW, MAP_PRIVATE|MAP_ANONYMOUS
            base = (raw + (2 << 20) - 1) // (2 << 20) * (2 << 20)
            libc.madvise(base, nb2, 14)  # MADV_HUGEPAGE
            arr = np.frombuffer((C.c_uint16 * (nb2 // 2)).from_address(base), dtype=np.uint16)
            arr[:] = 7
            assert cudart.cudaHostRegister(base, nb2, 0) == 0
            store = arr[: n_img * elems].reshape(n_img, elems)
            ptr = lambda i, st=store: st[i].ctypes.data  # noqa: E731
        else:
            t = torch.empty((n_img, elems), dtype=torch.int16).pin_memory()
            t.random_(0, 1 << 14)
            ptr = lambda i, t=t: t[i].data_ptr()  # noqa: E731
        for n in ((1, 2, 4) if name == "deepseek" else (1, 2)):
            x = np.full((n, H), 0x3F80, np.uint16)
            out = np.empty((n, H), np.float32)
            xs = (C.c_void_p * n)(*[x[i:i + 1].ctypes.data for i in range(n)])
            outs = (C.c_void_p * n)(*[out[i:i + 1].ctypes.data for i in range(n)])
            imgs = (C.c_void_p * n)()
            for gap in (0, 40):
                reps = max(8, int(1.5e9 / (n * elems * 2)))
                k, tot = 0, 0.0
                for r in range(reps + 3):
                    for i in range(n):
                        imgs[i] = ptr(k % n_img)
                        k += 1
                    if gap:
                        spin(gap)
                    t0 = time.perf_counter()
                    lib.hm_cpu_experts_decode(pool, imgs, xs, n, H, I, outs)
                    if r >= 3:
                        tot += time.perf_counter() - t0
                dt = tot / reps
                print(f"{name:8s} {kind:6s} n={n} gap={gap:2d}us: {n * elems * 2 / dt / 1e9:6.1f} GB/s "
                      f"({dt * 1e6:7.1f} us/call)", flush=True)
        if kind == "thp_pinned":
            cudart.cudaHostUnregister(base)
        store = t = None
lib.hm_cpu_pool_destroy(pool)
