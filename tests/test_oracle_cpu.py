"""The plain-C oracle expert (oracle/cpu_moe.c, the reference arm's CPU path)
against the fp32 numpy oracle (oracle/moe_ref.py): bf16 weights/activations,
fp32 accumulation, h rounded to bf16 -> max|c - ref| / max|ref| <= 1e-2."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import cpu_moe, moe_ref as ref


@pytest.mark.parametrize("H,I,M", [(256, 384, 1), (512, 256, 4), (2048, 1408, 2), (130, 70, 3)])
def test_c_oracle_expert_matches_numpy_oracle(H, I, M):
    rng = np.random.default_rng(H + I + M)
    w13 = ref.f32_to_bf16((rng.standard_normal((2 * I, H)) * 0.02).astype(np.float32))
    w2 = ref.f32_to_bf16((rng.standard_normal((H, I)) * 0.02).astype(np.float32))
    x = ref.f32_to_bf16(rng.standard_normal((M, H)).astype(np.float32))
    out = np.empty((M, H), np.float32)
    cpu_moe.expert(w13.ctypes.data, w2.ctypes.data, H, I, x.ctypes.data, M, out.ctypes.data, cpu_moe.Scratch())
    f = ref.bf16_to_f32
    want = ref.expert(f(x), f(w13[:I]), f(w13[I:]), f(w2))
    assert np.abs(out - want).max() / np.abs(want).max() <= 1e-2
    assert cpu_moe.threads() >= 1
