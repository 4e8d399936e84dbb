"""Warm-up calibration on the B200 box (§IV-A).

Measures the three resources the decision core plans with and fits a
``HardwareProfile`` with ``costs.calibrate`` (the reference's fits,
costs.py:134-219), all in seconds, for one expert of shape (H, I):

  gpu   one expert through ``hm_expert_ffn`` at loads 1..512 tokens (CUDA events)
  cpu   one expert on the AVX-512 host worker, in bursts of three after an idle
        gap: position 0 is the cold first expert of a burst (the reference's
        first-expert penalty, Fig. 3e).  At decode (every load 1) through the
        worker's decode entry (hm_cpu_experts_decode, the call the runtime
        makes per layer) after a gap like the step's router wait, so the
        fitted slope is the per-expert time the step actually pays.
  pcie  pinned H2D copies of 1/4, 1/2 and 1 expert image (CUDA events)
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch

from ._lib import check, lib
from .costs import CalibrationSample, calibrate


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def measure_samples(H: int, I: int, gpu_loads=(1, 2, 4, 8, 32, 128, 256, 384, 512), cpu_loads=(1, 2, 3, 4),
                    reps: int = 3, cpu_bursts: int = 2, n_images: int = 4, cpu_threads: int = 0,
                    seed: int = 0, weight_bits: int = 16) -> list[CalibrationSample]:
    """weight_bits 4: the same measurements on 4-bit expert images (hm_q4_*)."""
    from .kernels import expert_ffn, groups_array

    q4 = weight_bits == 4
    elems = 3 * H * I
    # host images well beyond the last-level cache (small experts would
    # otherwise be served from a 60-300 MB LLC and look faster than in the step)
    n_images = max(n_images, -(-(512 << 20) // (elems * (1 if q4 else 2))))
    slot_elems = elems
    if q4:
        nb = C.c_size_t()
        check(lib.hm_q4_image_bytes(H, I, C.byref(nb)))
        slot_elems = (nb.value + 255) // 256 * 256 // 2
    g = torch.Generator(device="cuda").manual_seed(seed)
    st0 = torch.cuda.current_stream().cuda_stream

    def image() -> torch.Tensor:  # one expert image in slot layout (bf16 view)
        w = (torch.randn(elems, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
        if not q4:
            return w
        q = torch.zeros(slot_elems * 2, dtype=torch.uint8, device="cuda")
        check(lib.hm_q4_quantize(w.data_ptr(), H, I, q.data_ptr(), st0))
        return q.view(torch.bfloat16)

    pool = image().view(1, slot_elems)
    host = torch.empty((n_images, slot_elems), dtype=torch.bfloat16).pin_memory()
    for i in range(n_images):
        host[i].copy_(image())
    scratch = torch.empty((1, elems), dtype=torch.bfloat16, device="cuda") if q4 else None

    def ffn(m: int) -> None:
        if q4:
            check(lib.hm_expert_ffn_q4(pool.data_ptr(), slot_elems * 2, 1, H, I, groups_array([(0, 0, m)]), 1,
                                       x.data_ptr(), maxm, h.data_ptr(), out.data_ptr(), scratch.data_ptr(), 1, 0,
                                       st0))
        else:
            expert_ffn(flat, 1, H, I, [(0, 0, m)], x, h, out)
    samples: list[CalibrationSample] = []
    st = torch.cuda.current_stream()
    maxm = max(gpu_loads)
    x = torch.randn((maxm, H), generator=g, device="cuda").to(torch.bfloat16)
    h = torch.empty((maxm, I), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((maxm, H), device="cuda")
    flat = pool.view(-1)
    for m in gpu_loads:
        ffn(m)
        a, b = _events()
        a.record(st)
        for _ in range(reps):
            ffn(m)
        b.record(st)
        b.synchronize()
        samples.append(CalibrationSample("gpu", float(m), 0, a.elapsed_time(b) / 1e3 / reps))

    cpool = C.c_void_p()
    check(lib.hm_cpu_pool_create(int(cpu_threads), C.byref(cpool)))
    try:
        xs = np.ascontiguousarray(x[: max(cpu_loads)].view(torch.int16).cpu().numpy().view(np.uint16))
        outs = np.empty((max(cpu_loads), H), dtype=np.float32)
        decode = all(m == 1 for m in cpu_loads)
        for m in cpu_loads:
            for burst in range(cpu_bursts):
                time.sleep(1e-4 if decode else 0.02)
                for pos in range(3):
                    img = host[(burst * 3 + pos) % n_images]
                    if decode:
                        ip, xp_, op = (C.c_void_p * 1)(img.data_ptr()), (C.c_void_p * 1)(xs.ctypes.data), \
                            (C.c_void_p * 1)(outs.ctypes.data)
                        fn = lib.hm_cpu_experts_decode_q4 if q4 else lib.hm_cpu_experts_decode
                        t0 = time.perf_counter()
                        check(fn(cpool, ip, xp_, 1, H, I, op))
                    else:
                        fn = lib.hm_cpu_expert_q4 if q4 else lib.hm_cpu_expert
                        t0 = time.perf_counter()
                        check(fn(cpool, img.data_ptr(), H, I, xs.ctypes.data, m, outs.ctypes.data))
                    samples.append(CalibrationSample("cpu", float(m), pos, time.perf_counter() - t0))
    finally:
        lib.hm_cpu_pool_destroy(cpool)

    for frac in (4, 2, 1):
        n = slot_elems // frac
        for i in range(n_images):  # warm every source range first: a cold first touch
            flat[:n].copy_(host[i, :n], non_blocking=True)  # reads ~25 % slower and skews the fit
        torch.cuda.synchronize()
        for r in range(reps + 1):  # the first copy after an idle gap is slow (link wake-up): not a sample
            a, b = _events()
            a.record(st)
            flat[:n].copy_(host[1 + r % (n_images - 1), :n], non_blocking=True)
            b.record(st)
            b.synchronize()
            if r > 0:
                samples.append(CalibrationSample("pcie", float(n * 2), 0, a.elapsed_time(b) / 1e3))
    torch.cuda.synchronize()
    return samples


def calibrate_shape(H: int, I: int, gpu_saturation_load: int = 256, **kw):
    """Measure and fit; returns (CalibrationResult, samples).  kw: measure_samples'
    options (e.g. weight_bits=4)."""
    samples = measure_samples(H, I, **kw)
    return calibrate(samples, gpu_saturation_load=gpu_saturation_load), samples


# Attention blocks of the named models (the non-expert part of one decoder
# layer): (hidden, query heads, kv heads, head dim) of the released configs;
# DeepSeek-V2-Lite's MLA (q 16 x 192, compressed kv 512 + 64 rope, kv_b up-
# projection) is costed by its projection shapes with 128-wide heads.
ATTENTION_SHAPES = {
    "tiny": dict(H=256, nh=4, nkv=4, hd=64, proj=None),
    "mixtral": dict(H=4096, nh=32, nkv=8, hd=128, proj=None),
    "qwen2": dict(H=3584, nh=28, nkv=4, hd=128, proj=None),
    "deepseek": dict(H=2048, nh=16, nkv=16, hd=128, proj=[(2048, 16 * 192), (2048, 576), (512, 16 * 256),
                                                         (16 * 128, 2048)]),
}


def measure_non_expert_time(family: str, tokens: int, context: int, reps: int = 20, seed: int = 0) -> float:
    """Seconds per layer of the non-expert work the reference folds into
    ``non_expert_time`` (costs.py:45, engine.py:307; SPEC.md: "attention etc.,
    default 0"): RMSNorm, the QKV / O projections and attention over a KV cache
    of ``context`` positions for ``tokens`` new tokens, at the family's shapes,
    bf16.  Calibration input only -- these are cuBLAS / SDPA library calls, not
    the MoE hot path; weights of several layers rotate so the projections stream
    from HBM as in a real step, captured in one CUDA graph and replayed."""
    import torch.nn.functional as F

    a = ATTENTION_SHAPES[family]
    H, nh, nkv, hd = a["H"], a["nh"], a["nkv"], a["hd"]
    proj = a["proj"] or [(H, (nh + 2 * nkv) * hd), (nh * hd, H)]
    g = torch.Generator(device="cuda").manual_seed(seed)
    per_layer = sum(i * o for i, o in proj) * 2
    n_layers = max(2, -(-(512 << 20) // per_layer))  # > 4x the 126 MB L2
    ws = [[(torch.randn((o, i), generator=g, device="cuda") * 0.02).to(torch.bfloat16) for i, o in proj]
          for _ in range(n_layers)]
    kc = torch.randn((1, nkv, context + tokens, hd), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn_like(kc)
    x = torch.randn((tokens, H), generator=g, device="cuda").to(torch.bfloat16)
    norm_w = torch.ones(H, device="cuda", dtype=torch.bfloat16)

    def layer(w) -> torch.Tensor:
        hn = F.rms_norm(x, (H,), norm_w)
        t = hn
        for m in w[:-1]:  # q/kv projections (DeepSeek: the chain of its MLA projections, shapes only)
            t = F.linear(hn if m.shape[1] == H else t[:, : m.shape[1]], m)
        qh = t[:, : nh * hd].reshape(tokens, nh, hd).transpose(0, 1).unsqueeze(0) if t.shape[1] >= nh * hd else \
            hn[:, : nh * hd].reshape(tokens, nh, hd).transpose(0, 1).unsqueeze(0)
        o = F.scaled_dot_product_attention(qh, kc, vc, is_causal=context == 0, enable_gqa=nh != nkv)
        o = o.squeeze(0).transpose(0, 1).reshape(tokens, nh * hd)
        return x + F.linear(o, w[-1])

    # one CUDA graph replays the layers back to back: the GPU time of the block,
    # not PyTorch's per-op launch overhead (~10 ops of a few us each at T = 1)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(n_layers):
            layer(ws[i])
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(n_layers):
            layer(ws[i])
    graph.replay()
    st = torch.cuda.current_stream()
    a0, b0 = _events()
    a0.record(st)
    for _ in range(reps):
        graph.replay()
    b0.record(st)
    b0.synchronize()
    return a0.elapsed_time(b0) / 1e3 / (reps * n_layers)
