"""Pinned host memory: cudaHostAlloc (4 KB pages) vs mmap + MADV_HUGEPAGE +
cudaHostRegister (2 MB transparent huge pages): host stream-read GB/s with the
worker pool and pinned H2D GB/s from each."""
import ctypes as C
import mmap
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
lib = _lib.lib
nbytes = 8 << 30
pool = C.c_void_p()
lib.hm_cpu_pool_create(0, C.byref(pool))
libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
cudart = torch.cuda.cudart()


def measure(ptr, label):
    bws = []
    for _ in range(4):
        bw = C.c_double()
        lib.hm_host_read_bw(pool, ptr, nbytes, 2, C.byref(bw))
        bws.append(bw.value)
    t = torch.empty(352 << 20, dtype=torch.uint8, device="cuda")
    host = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * (352 << 20)).from_address(ptr)))
    for _ in range(2):
        t.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        t.copy_(host, non_blocking=True)
    b.record()
    b.synchronize()
    print(label, "host read GB/s", [round(x, 1) for x in bws], "H2D GB/s", round(5 * (352 << 20) / (a.elapsed_time(b) / 1e3) / 1e9, 1))


for rnd in range(2):
    p = C.c_void_p()
    lib_rt = C.CDLL("libcudart.so.12") if False else None
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()  # cudaHostAlloc via torch's caching allocator
    h.fill_(1)
    measure(h.data_ptr(), "cudaHostAlloc ")
    del h
    addr = libc.mmap(None, nbytes, 3, 0x22, -1, 0)  # PROT_READ|WRITE, MAP_PRIVATE|ANONYMOUS
    libc.madvise(addr, nbytes, 14)  # MADV_HUGEPAGE
    arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(addr))
    arr[:] = 1
    r = cudart.cudaHostRegister(addr, nbytes, 0)
    measure(addr, f"THP+register({int(r)})")
    cudart.cudaHostUnregister(addr)
    ah = open("/proc/meminfo").read()
    print([l for l in ah.splitlines() if "AnonHuge" in l])
