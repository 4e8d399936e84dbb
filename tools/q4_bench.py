"""4-bit decode GEMV timing (hm_expert_ffn_q4): 20 calls captured in one CUDA
graph and replayed (no Python between launches), weights rotating over a slot
set larger than L2: GB/s of 4-bit image bytes.

  python tools/q4_bench.py [counts]
"""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402
from paper_2504_05897_b200.kernels import groups_array  # noqa: E402

lib = _lib.lib
counts = tuple(int(c) for c in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1, 2, 4, 6, 8)
res = {}
for name, (H, I) in {"mixtral": (4096, 14336), "deepseek": (2048, 1408), "qwen2": (3584, 2560)}.items():
    nb = C.c_size_t()
    lib.hm_q4_image_bytes(H, I, C.byref(nb))
    sb = (nb.value + 255) // 256 * 256
    n_slots = max(16, -(-(600 << 20) // sb))
    pool = torch.randint(0, 255, (n_slots, sb), dtype=torch.uint8, device="cuda")
    for n in counts:
        x = torch.randn((n, H), device="cuda").to(torch.bfloat16)
        h = torch.empty((n, I), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((n, H), device="cuda")
        side = torch.cuda.Stream()
        arrs = [groups_array([((i * n + e) % n_slots, e, 1) for e in range(n)]) for i in range(20)]

        def run(i, st):
            _lib.check(lib.hm_expert_ffn_q4(pool.data_ptr(), sb, n_slots, H, I, arrs[i], n, x.data_ptr(), n,
                                            h.data_ptr(), out.data_ptr(), None, 0, 1, st.cuda_stream))
        with torch.cuda.stream(side):
            for i in range(3):
                run(i, side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(20):
                run(i, side)
        g.replay()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(3):
            g.replay()
        b.record(st)
        b.synchronize()
        us = 1e3 * a.elapsed_time(b) / 60
        res[f"{name}-n{n}"] = {"us": round(us, 2), "gbs": round(n * nb.value / (us * 1e-6) / 1e9, 1)}
        print(name, n, res[f"{name}-n{n}"], flush=True)
    del pool
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/q4_bench.json").write_text(json.dumps(res))
