"""4-bit decode GEMV timing (hm_expert_ffn_q4, back-to-back from Python; the
kernels are long enough that launch overhead is hidden): GB/s of 4-bit image bytes."""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402
from paper_2504_05897_b200.kernels import groups_array  # noqa: E402

lib = _lib.lib
res = {}
for name, (H, I) in {"mixtral": (4096, 14336), "deepseek": (2048, 1408)}.items():
    nb = C.c_size_t()
    lib.hm_q4_image_bytes(H, I, C.byref(nb))
    sb = (nb.value + 255) // 256 * 256
    n_slots = 8
    pool = torch.randint(0, 255, (n_slots, sb), dtype=torch.uint8, device="cuda")
    for n in (1, 2, 4):
        x = torch.randn((n, H), device="cuda").to(torch.bfloat16)
        h = torch.empty((n, I), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((n, H), device="cuda")
        st = torch.cuda.current_stream()

        def run(i):
            arr = groups_array([((i * n + e) % n_slots, e, 1) for e in range(n)])
            _lib.check(lib.hm_expert_ffn_q4(pool.data_ptr(), sb, n_slots, H, I, arr, n, x.data_ptr(), n, h.data_ptr(),
                                            out.data_ptr(), None, 0, 1, st.cuda_stream))
        for i in range(3):
            run(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(20):
            run(i)
        b.record(st)
        b.synchronize()
        us = 1e3 * a.elapsed_time(b) / 20
        res[f"{name}-n{n}"] = {"us": round(us, 1), "gbs": round(n * nb.value / (us * 1e-6) / 1e9, 1)}
print(json.dumps(res))
