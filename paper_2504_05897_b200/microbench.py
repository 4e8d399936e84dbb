"""Kernel micro-benchmarks for the roofline keys of bench.py and the ncu captures.

``gemm_bench``: the prefill grouped expert GEMM (tcgen05/TMA) over G resident
experts with M token rows each -- flops 2*M*3*H*I per expert.
``gemv_bench``: the decode weight-streaming expert GEMV -- bytes 3*H*I*2 per
expert.  Both time back-to-back launches with CUDA events on the launching
stream, after warm-up, rotating over enough slots that weights exceed L2.
"""
from __future__ import annotations

import torch

from . import _lib
from .kernels import expert_ffn


def _pool(n_slots: int, H: int, I: int, seed: int = 0) -> torch.Tensor:
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn((n_slots, 3 * H * I), generator=g, device="cuda") * 0.02).to(torch.bfloat16).view(-1)


def gemm_bench(H: int, I: int, rows_per_expert: int = 256, n_experts: int = 8, reps: int = 5, warmup: int = 2) -> dict:
    pool = _pool(n_experts, H, I)
    rows = rows_per_expert * n_experts
    x = torch.randn((rows, H), device="cuda").to(torch.bfloat16)
    h = torch.empty((rows, I), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((rows, H), device="cuda")
    groups = [(e, e * rows_per_expert, rows_per_expert) for e in range(n_experts)]
    for _ in range(warmup):
        expert_ffn(pool, n_experts, H, I, groups, x, h, out, _lib.FFN_GEMM)
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        expert_ffn(pool, n_experts, H, I, groups, x, h, out, _lib.FFN_GEMM)
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    flops = 2.0 * rows * 3 * H * I
    wbytes = n_experts * 3 * H * I * 2
    del pool
    return {"ms": ms, "tflops": flops / (ms / 1e3) / 1e12, "flops": flops, "weight_bytes": wbytes,
            "hbm_gbs": wbytes / (ms / 1e3) / 1e9, "rows_per_expert": rows_per_expert, "experts": n_experts}


def gemv_bench(H: int, I: int, n_experts: int = 2, n_slots: int = 8, reps: int = 20, warmup: int = 3) -> dict:
    pool = _pool(n_slots, H, I)
    x = torch.randn((n_experts, H), device="cuda").to(torch.bfloat16)
    h = torch.empty((n_experts, I), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((n_experts, H), device="cuda")
    st = torch.cuda.current_stream()

    def launch(i: int) -> None:
        groups = [((i * n_experts + e) % n_slots, e, 1) for e in range(n_experts)]
        expert_ffn(pool, n_slots, H, I, groups, x, h, out, _lib.FFN_GEMV)

    for i in range(warmup):
        launch(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(reps):
        launch(i)
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    nbytes = n_experts * 3 * H * I * 2
    del pool
    return {"ms": ms, "gbs": nbytes / (ms / 1e3) / 1e9, "bytes": nbytes, "experts": n_experts}
