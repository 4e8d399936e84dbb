"""Expert weight images: the slot layout shared by the HBM pool, the pinned
host master store and the host worker (see include/hybrimoe.h, hm_group).

  [0, 2IH)   W13: gate/up rows interleaved in 128-row blocks
  [2IH, 3IH) W2 [H, I]
"""
from __future__ import annotations

import numpy as np

ILV = 128


def w13_row_of_gate(i: int) -> int:
    return (i // ILV) * 2 * ILV + i % ILV


def pack_expert(gate: np.ndarray, up: np.ndarray, down: np.ndarray) -> np.ndarray:
    """gate/up [I, H], down [H, I] (same dtype) -> flat slot image [3*H*I]."""
    I, H = gate.shape
    if I % ILV:
        raise ValueError(f"intermediate size {I} must be a multiple of {ILV}")
    w13 = np.empty((2 * I, H), dtype=gate.dtype)
    g3 = gate.reshape(I // ILV, ILV, H)
    u3 = up.reshape(I // ILV, ILV, H)
    w13.reshape(I // ILV, 2, ILV, H)[:, 0] = g3
    w13.reshape(I // ILV, 2, ILV, H)[:, 1] = u3
    return np.concatenate([w13.reshape(-1), np.ascontiguousarray(down).reshape(-1)])


def unpack_expert(img: np.ndarray, H: int, I: int):
    """Inverse of pack_expert -> (gate [I, H], up [I, H], down [H, I])."""
    w13 = img[: 2 * I * H].reshape(I // ILV, 2, ILV, H)
    gate = w13[:, 0].reshape(I, H)
    up = w13[:, 1].reshape(I, H)
    down = img[2 * I * H: 3 * I * H].reshape(H, I)
    return gate, up, down
