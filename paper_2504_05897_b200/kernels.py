"""Thin torch-tensor front end for the sm_100a kernels of libhybrimoe.so.

PyTorch is plumbing here (device memory and streams); every computation is a
kernel in the native library.  Each wrapper validates devices/dtypes and
raises if CUDA is unavailable -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _p(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise RuntimeError("hybrimoe kernels need CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("hybrimoe kernels need contiguous tensors")
    return t.data_ptr()


def router_topk(logits: torch.Tensor, n_routed: int, k: int, renormalize: bool, n_shared: int = 0,
                shared_gate_col: int = -1, stream=None):
    """Returns (sel [T, K+S] int32, w [T, K+S] fp32, probs [T, N] fp32, counts [N+S] int32)."""
    T, ld = logits.shape
    dev = logits.device
    kp = k + n_shared
    sel = torch.empty((T, kp), dtype=torch.int32, device=dev)
    w = torch.empty((T, kp), dtype=torch.float32, device=dev)
    probs = torch.empty((T, n_routed), dtype=torch.float32, device=dev)
    counts = torch.empty((n_routed + n_shared,), dtype=torch.int32, device=dev)
    check(lib.hm_router_topk(_p(logits), T, n_routed, ld, k, int(renormalize), n_shared, shared_gate_col, _p(sel),
                             _p(w), _p(probs), _p(counts), _stream(stream)))
    return sel, w, probs, counts


def score_sums(probs: torch.Tensor, stream=None) -> torch.Tensor:
    T, N = probs.shape
    out = torch.empty((N,), dtype=torch.float64, device=probs.device)
    check(lib.hm_score_sums(_p(probs), T, N, _p(out), _stream(stream)))
    return out


def router_logits(x: torch.Tensor, wg: torch.Tensor, stream=None) -> torch.Tensor:
    T, H = x.shape
    N = wg.shape[0]
    out = torch.empty((T, N), dtype=torch.float32, device=x.device)
    check(lib.hm_router_logits(_p(x), _p(wg), T, H, N, _p(out), _stream(stream)))
    return out


def lookahead(x: torch.Tensor, gate_w: torch.Tensor, first_layer: int, horizon: int, n_routed: int, k: int,
              stream=None) -> torch.Tensor:
    """Predicted loads [horizon, N] int32 of layers first_layer.. for hidden state
    x: the gates gate_w [L, ld, H] through the router's top-K (hm_lookahead)."""
    T, H = x.shape
    counts = torch.empty((max(1, horizon), n_routed), dtype=torch.int32, device=x.device)
    check(lib.hm_lookahead(_p(x), _p(gate_w), first_layer, horizon, T, n_routed, gate_w.shape[1], k, H, _p(counts),
                           None, _stream(stream)))
    return counts[:horizon]


def offsets(counts: torch.Tensor, stream=None) -> torch.Tensor:
    E = counts.shape[0]
    out = torch.empty((E + 1,), dtype=torch.int32, device=counts.device)
    check(lib.hm_offsets(_p(counts), E, _p(out), _stream(stream)))
    return out


def permute(sel: torch.Tensor, offs: torch.Tensor, n_experts: int, stream=None):
    T, kp = sel.shape
    pos = torch.empty((T, kp), dtype=torch.int32, device=sel.device)
    row_src = torch.empty((T * kp,), dtype=torch.int32, device=sel.device)
    check(lib.hm_permute(_p(sel), T, kp, n_experts, _p(offs), _p(pos), _p(row_src), _stream(stream)))
    return pos, row_src


def gather_rows(x: torch.Tensor, row_src: torch.Tensor, kp: int, rows: int | None = None, out=None, stream=None):
    H = x.shape[1]
    rows = row_src.shape[0] if rows is None else rows
    xp = out if out is not None else torch.empty((rows, H), dtype=x.dtype, device=x.device)
    check(lib.hm_gather_rows(_p(x), _p(row_src), rows, kp, H, _p(xp), _stream(stream)))
    return xp


def groups_array(groups) -> C.Array:
    arr = (_lib.HmGroup * max(1, len(groups)))()
    for i, (slot, rb, rc) in enumerate(groups):
        arr[i].slot, arr[i].row_begin, arr[i].row_count = int(slot), int(rb), int(rc)
    return arr


def expert_ffn(pool: torch.Tensor, n_slots: int, H: int, I: int, groups, xp: torch.Tensor, h: torch.Tensor,
               out: torch.Tensor, path: int = _lib.FFN_AUTO, stream=None) -> None:
    """groups: iterable of (slot, row_begin, row_count)."""
    groups = list(groups)
    arr = groups_array(groups)
    check(lib.hm_expert_ffn(_p(pool), n_slots, H, I, arr, len(groups), _p(xp), xp.shape[0], _p(h), _p(out), path,
                            _stream(stream)))


def combine(out: torch.Tensor, pos: torch.Tensor, w: torch.Tensor, residual: torch.Tensor | None = None,
            y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    T, kp = pos.shape
    H = out.shape[1]
    y = y if y is not None else torch.empty((T, H), dtype=torch.bfloat16, device=out.device)
    check(lib.hm_combine(_p(out), _p(pos), _p(w), T, kp, H, _p(residual), _p(y), _stream(stream)))
    return y


def mrs_update_dev(S: torch.Tensor, scores: torch.Tensor, layer: int, p: int, alpha: float, stream=None) -> None:
    N = S.shape[1]
    check(lib.hm_mrs_update_dev(_p(S), _p(scores), int(layer), N, int(p), float(alpha), _stream(stream)))
