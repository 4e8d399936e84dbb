"""Kernel micro-benchmarks for the roofline keys of bench.py and the ncu captures.

``gemm_bench``: the prefill grouped expert GEMM (tcgen05/TMA) over G resident
experts with M token rows each -- flops 2*M*3*H*I per expert.
``gemv_bench``: the decode weight-streaming expert GEMV -- bytes 3*H*I*2 per
expert.  Both time back-to-back launches issued inside the library
(hm_bench_expert_ffn, CUDA events on the launching stream, after warm-up),
rotating over enough slots that weights exceed L2.
"""
from __future__ import annotations

import torch

from . import _lib


def _pool(n_slots: int, H: int, I: int, seed: int = 0) -> torch.Tensor:
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn((n_slots, 3 * H * I), generator=g, device="cuda") * 0.02).to(torch.bfloat16).view(-1)


def _lib_bench(pool, n_slots, H, I, n_groups, rows, path, reps) -> float:
    """ms per hm_expert_ffn call, `reps` back-to-back calls issued inside the
    library (hm_bench_expert_ffn): no Python between launches."""
    import ctypes as C
    x = torch.randn((n_groups * rows, H), device="cuda").to(torch.bfloat16)
    h = torch.empty((n_groups * rows, I), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((n_groups * rows, H), device="cuda")
    ms = C.c_float()
    _lib.check(_lib.lib.hm_bench_expert_ffn(pool.data_ptr(), n_slots, H, I, n_groups, rows, x.data_ptr(),
                                            h.data_ptr(), out.data_ptr(), path, reps,
                                            torch.cuda.current_stream().cuda_stream, C.byref(ms)))
    return ms.value


def gemm_bench(H: int, I: int, rows_per_expert: int = 256, n_experts: int = 8, reps: int = 5, warmup: int = 2) -> dict:
    pool = _pool(n_experts, H, I)
    ms = _lib_bench(pool, n_experts, H, I, n_experts, rows_per_expert, _lib.FFN_GEMM, reps)
    rows = rows_per_expert * n_experts
    flops = 2.0 * rows * 3 * H * I
    wbytes = n_experts * 3 * H * I * 2
    del pool
    return {"ms": ms, "tflops": flops / (ms / 1e3) / 1e12, "flops": flops, "weight_bytes": wbytes,
            "hbm_gbs": wbytes / (ms / 1e3) / 1e9, "rows_per_expert": rows_per_expert, "experts": n_experts}


def gemv_bench(H: int, I: int, n_experts: int = 2, n_slots: int = 8, reps: int = 20, warmup: int = 3) -> dict:
    pool = _pool(n_slots, H, I)
    ms = _lib_bench(pool, n_slots, H, I, n_experts, 1, _lib.FFN_GEMV, reps)
    nbytes = n_experts * 3 * H * I * 2
    del pool
    return {"ms": ms, "gbs": nbytes / (ms / 1e3) / 1e9, "bytes": nbytes, "experts": n_experts}
