"""Per-layer critical-path pieces of decode on the GPU box: the combine tail
(with 0..4 rows read zero-copy from mapped host memory), the fused router with
and without the host mirror, and the router -> host-flag round trip.

  python tools/tail_bench.py
"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

lib = _lib.lib
st = torch.cuda.current_stream()
sp = st.cuda_stream
res = {}


REPS = int(os.environ.get("TAIL_REPS", "200"))


def timed(fn, reps=None):
    reps = reps or REPS
    for _ in range(min(10, reps)):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


for name, H, N, K, S in (("mixtral", 4096, 8, 2, 0), ("deepseek", 2048, 64, 6, 2), ("qwen2", 3584, 64, 8, 8)):
    Kp = K + S
    out = torch.randn((Kp, H), device="cuda")
    host_out = torch.randn((Kp, H)).pin_memory()
    pos = torch.arange(Kp, dtype=torch.int32, device="cuda")
    w = torch.rand((Kp,), device="cuda")
    x = torch.randn((1, H), device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    Sd = torch.zeros((4, N), dtype=torch.float64, device="cuda")
    sc = torch.rand((N,), dtype=torch.float64, device="cuda")
    for nh in (0, 1, 2, 4):
        nh = min(nh, K)
        mask = (C.c_uint64 * 4)((1 << nh) - 1, 0, 0, 0)
        f = lambda: lib.hm_combine_tail(out.data_ptr(), host_out.data_ptr(), mask if nh else None, pos.data_ptr(),
                                        w.data_ptr(), 1, Kp, H, x.data_ptr(), y.data_ptr(), Sd.data_ptr(),
                                        sc.data_ptr(), 1, N, 2 * K, 0.5, sp)
        res[f"{name}-combine_tail-host{nh}-us"] = timed(f)
    ld = N + (1 if S else 0)
    logits = torch.randn((1, ld), device="cuda")
    E = N + S
    sel = torch.empty(64, dtype=torch.int32, device="cuda")
    wsel = torch.empty(64, device="cuda")
    posb = torch.empty(64, dtype=torch.int32, device="cuda")
    rsrc = torch.empty(64, dtype=torch.int32, device="cuda")
    xp = torch.empty((Kp, H), dtype=torch.bfloat16, device="cuda")
    meta = torch.empty(4096, dtype=torch.uint8, device="cuda")
    mi, md = meta.data_ptr(), meta.data_ptr() + 2048
    hmeta = torch.empty(4096, dtype=torch.uint8).pin_memory()
    hxp = torch.empty((Kp, H), dtype=torch.bfloat16).pin_memory()
    flag = torch.zeros(16, dtype=torch.int32).pin_memory()
    common = (logits.data_ptr(), 1, N, ld, K, 1, S, N if S else -1, x.data_ptr(), H, sel.data_ptr(), wsel.data_ptr(),
              posb.data_ptr(), rsrc.data_ptr(), xp.data_ptr(), mi, md)
    res[f"{name}-router_small-us"] = timed(lambda: lib.hm_router_fused_small(*common, sp))
    seq = [0]

    def mirror():
        seq[0] += 1
        lib.hm_router_fused_mirror(*common, hmeta.data_ptr(), hmeta.data_ptr() + 2048, hxp.data_ptr(),
                                   flag.data_ptr(), seq[0], sp)
    res[f"{name}-router_mirror-us"] = timed(mirror)
    # round trip: launch, spin on the flag (numpy view), n times
    fl = flag.numpy()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        t0 = time.perf_counter()
        mirror()
        while fl[0] != seq[0] % (1 << 31):
            pass
        ts.append(time.perf_counter() - t0)
    res[f"{name}-router_mirror-roundtrip-us-median"] = 1e6 * float(np.median(ts))
    # round trip via memcpy + event
    ev = torch.cuda.Event()
    ts = []
    for _ in range(REPS):
        t0 = time.perf_counter()
        lib.hm_router_fused_small(*common, sp)
        hmeta.copy_(meta, non_blocking=True)
        ev.record(st)
        ev.synchronize()
        ts.append(time.perf_counter() - t0)
    res[f"{name}-router_memcpy_event-roundtrip-us-median"] = 1e6 * float(np.median(ts))
print(json.dumps(res, indent=1))
