"""ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

fp32 numpy restatement of the MoE layer numerics the B200 kernels compute.
The reference simulator never evaluates experts (core.py:3-7), so
expert-output parity is "unpinned by the reference": this file restates
Eq. 1 of the paper,

    y = sum_{i in TopK(softmax(x W_g))} w_i E_i(x),   E_i(x) = W2 (silu(Wg x) * (Wu x)),

with the routers of the model families the configs name (transformers 5.5):
  Mixtral   softmax -> top-K -> renormalise   (mixtral/modeling_mixtral.py:111-114)
  DeepSeek  softmax -> top-K, no renormalise  (deepseek_v2/modeling_deepseek_v2.py:103-120)
  Qwen2-MoE softmax -> top-K, shared expert * sigmoid(x . w_sg)  (qwen2_moe/modeling_qwen2_moe.py:346-370)
Top-K order follows the reference's tie rule: value descending, lower index
first (core.py:94-97, tracegen.py:139-141), applied to the fp32 logits.
Router indices and loads are therefore pinned to the reference's traces
(tests/test_router_real_shapes.py); the layer numerics are pinned to the
transformers 5.5 MoE blocks themselves (tests/test_hf_pinned.py, 1e-4 in fp32);
the B200 expert outputs are checked against both at bf16 tolerance (1e-2).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> fp32 (exact)."""
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round to nearest even."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rnd = ((b >> 16) & 1) + 0x7FFF
    return ((b + rnd) >> 16).astype(np.uint16)


def router(logits: np.ndarray, n_routed: int, k: int, renormalize: bool, n_shared: int = 0,
           shared_gate_col: int = -1):
    """logits [T, ld] fp32 -> sel [T, K+S], w [T, K+S], probs [T, N], counts [N+S], score_sum [N] (fp64)."""
    z = logits[:, :n_routed].astype(np.float32)
    T = z.shape[0]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m, dtype=np.float32)
    probs = (e / e.sum(axis=1, keepdims=True, dtype=np.float32)).astype(np.float32)
    idx = np.arange(n_routed)
    sel = np.empty((T, k + n_shared), dtype=np.int32)
    w = np.empty((T, k + n_shared), dtype=np.float32)
    for t in range(T):
        order = np.lexsort((idx, -z[t]))[:k]     # value desc, index asc
        p = probs[t, order]
        sel[t, :k] = order
        w[t, :k] = p / p.sum(dtype=np.float32) if renormalize else p
        g = 1.0 / (1.0 + np.exp(-logits[t, shared_gate_col])) if shared_gate_col >= 0 else 1.0
        sel[t, k:] = n_routed + np.arange(n_shared)
        w[t, k:] = g
    counts = np.bincount(sel.ravel(), minlength=n_routed + n_shared).astype(np.int32)
    score_sum = probs.astype(np.float64).sum(axis=0)
    return sel, w, probs, counts, score_sum


def expert(x: np.ndarray, gate: np.ndarray, up: np.ndarray, down: np.ndarray) -> np.ndarray:
    """SwiGLU expert in fp32: x [M, H], gate/up [I, H], down [H, I] (fp32 arrays)."""
    g = x @ gate.T
    u = x @ up.T
    with np.errstate(over="ignore"):  # exp(-g) -> inf for very negative g: silu -> -0, as intended
        h = g / (1.0 + np.exp(-g)) * u
    return h @ down.T


def moe_layer(x: np.ndarray, logits: np.ndarray, experts: list, n_routed: int, k: int, renormalize: bool,
              n_shared: int = 0, shared_gate_col: int = -1, residual: bool = False) -> np.ndarray:
    """Full layer: experts[e] = (gate, up, down) fp32 for e in [0, N+S)."""
    sel, w, *_ = router(logits, n_routed, k, renormalize, n_shared, shared_gate_col)
    y = np.zeros_like(x, dtype=np.float32)
    for e in range(n_routed + n_shared):
        rows = np.nonzero((sel == e).any(axis=1))[0]
        if len(rows) == 0:
            continue
        out = expert(x[rows], *experts[e])
        wt = np.array([w[t, list(sel[t]).index(e)] for t in rows], dtype=np.float32)
        y[rows] += wt[:, None] * out
    return y + x if residual else y


# ---------------------------------------------------------------- 4-bit experts
# Restatement of the 4-bit expert image (include/hybrimoe.h, hm_q4_*): weight-
# only int4, one bf16 scale per 128 weights of a row, w = (nibble - 8) * scale,
# rows in the bf16 image's order (W13 gate/up interleaved in 128-row blocks,
# then W2).  Layout: W13 nibbles [2I][H/2] | W2 nibbles [H][I/2] | W13 scales
# [2I][H/128] bf16 | W2 scales [H][I/128] bf16.
Q4G = 128


def q4_quantize_rows(w_bf16: np.ndarray):
    """uint16 bf16 rows [R, K] -> (nibble bytes [R, K/2] uint8, scales [R, K/128] uint16 bf16)."""
    w = bf16_to_f32(w_bf16)
    R, K = w.shape
    g = w.reshape(R, K // Q4G, Q4G)
    s_bits = f32_to_bf16(np.abs(g).max(axis=2) / np.float32(7.0))
    s = bf16_to_f32(s_bits)[:, :, None]
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(s > 0, np.rint(g / np.where(s > 0, s, 1)), 0)
    nib = (np.clip(q, -8, 7) + 8).astype(np.uint8).reshape(R, K)
    return (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8), s_bits


def q4_dequantize_rows(nib: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """(nibble bytes [R, K/2], bf16 scales [R, K/128]) -> fp32 rows [R, K]."""
    R = nib.shape[0]
    vals = np.empty((R, nib.shape[1] * 2), dtype=np.float32)
    vals[:, 0::2] = (nib & 15).astype(np.float32) - 8
    vals[:, 1::2] = (nib >> 4).astype(np.float32) - 8
    s = bf16_to_f32(scales)
    return (vals.reshape(R, -1, Q4G) * s[:, :, None]).reshape(R, -1)


def q4_image(w13_bf16: np.ndarray, w2_bf16: np.ndarray) -> np.ndarray:
    """bf16 rows of W13 [2I, H] (image order) and W2 [H, I] -> the 4-bit image bytes."""
    n13, s13 = q4_quantize_rows(w13_bf16)
    n2, s2 = q4_quantize_rows(w2_bf16)
    return np.concatenate([n13.reshape(-1), n2.reshape(-1), s13.reshape(-1).view(np.uint8),
                           s2.reshape(-1).view(np.uint8)])


def q4_expert(img: np.ndarray, H: int, I: int):
    """4-bit image bytes -> fp32 (gate [I, H], up [I, H], down [H, I])."""
    hi = H * I
    n13 = img[:hi].reshape(2 * I, H // 2)
    n2 = img[hi: hi + hi // 2].reshape(H, I // 2)
    o = hi + hi // 2
    s13 = img[o: o + 2 * I * (H // Q4G) * 2].view(np.uint16).reshape(2 * I, H // Q4G)
    o += 2 * I * (H // Q4G) * 2
    s2 = img[o: o + H * (I // Q4G) * 2].view(np.uint16).reshape(H, I // Q4G)
    w13 = q4_dequantize_rows(n13, s13).reshape(I // 128, 2, 128, H)
    return w13[:, 0].reshape(I, H), w13[:, 1].reshape(I, H), q4_dequantize_rows(n2, s2)
