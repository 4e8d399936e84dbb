"""Streaming-read floor per launch size (hm_bench_stream_read): what a pure
16-byte-load read of the decode GEMV's weight bytes takes back to back, as one
launch and as the dependent ffn1/ffn2-like pair, next to the GEMV itself.

  python tools/read_floor.py [reps]
"""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_05897_b200 import _lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
shapes = {"deepseek": (2048, 1408, (1, 2, 4, 6, 8)), "qwen2": (3584, 2560, (1, 2, 4, 8)),
          "mixtral": (4096, 14336, (1, 2))}
st = torch.cuda.current_stream().cuda_stream
res = {}
for name, (H, I, counts) in shapes.items():
    eb = 3 * H * I * 2
    for n in counts:
        nbytes = n * eb
        n_buf = max(2, int(600e6 // nbytes) + 1)
        buf = torch.empty(n_buf * nbytes, dtype=torch.uint8, device="cuda")
        buf.random_(0, 255)
        row = {}
        for pair in (0, 1):
            for bps in (2, 4, 8):
                ms = C.c_float()
                _lib.check(_lib.lib.hm_bench_stream_read(buf.data_ptr(), nbytes, n_buf, pair, bps, reps, st,
                                                         C.byref(ms)))
                row[f"{'pair' if pair else 'one'}_b{bps}"] = {"us": round(1e3 * ms.value, 2),
                                                              "gbs": round(nbytes / (ms.value * 1e-3) / 1e9, 1)}
        del buf
        torch.cuda.empty_cache()
        # the GEMV pair on the same size
        n_slots = min(max(2 * n, int(4 * 126e6 // eb) + n), max(2 * n, int(24e9 // eb)))
        pool = (torch.randn((n_slots, 3 * H * I), device="cuda") * 0.02).to(torch.bfloat16)
        x = torch.randn((n, H), device="cuda").to(torch.bfloat16)
        h = torch.empty((n, I), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((n, H), device="cuda")
        ms = C.c_float()
        _lib.check(_lib.lib.hm_bench_expert_ffn(pool.data_ptr(), n_slots, H, I, n, 1, x.data_ptr(), h.data_ptr(),
                                                out.data_ptr(), 3, reps, st, C.byref(ms)))
        row["gemv"] = {"us": round(1e3 * ms.value, 2), "gbs": round(nbytes / (ms.value * 1e-3) / 1e9, 1)}
        best_pair = min(v["us"] for k, v in row.items() if k.startswith("pair"))
        best_one = min(v["us"] for k, v in row.items() if k.startswith("one"))
        row["gemv_over_pair_floor"] = round(best_pair / row["gemv"]["us"], 3)
        row["gemv_over_one_floor"] = round(best_one / row["gemv"]["us"], 3)
        del pool
        torch.cuda.empty_cache()
        res[f"{name}-n{n}"] = row
        print(name, n, json.dumps(row), flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/read_floor.json").write_text(json.dumps(res, indent=1))
