"""Qwen2-57B-A14B expert shape on both FFN paths, with its shared expert.

Routed experts at the released dims (H, I) = (3584, 2560) and
the (3584, 20480) shared expert scaled by sigmoid(x . w_sg) (transformers
qwen2_moe/modeling_qwen2_moe.py:346-370), executed as 8 always-resident chunks
of the routed shape (csrc: SwiGLU is separable along I).  The oracle computes
the shared expert as ONE (3584, 20480) SwiGLU from the concatenated chunk
weights, so the test also pins the chunk decomposition.  Decode (T=1: the
weight-streaming GEMV) and prefill (T=128: the tcgen05 grouped GEMM) go
through router -> permute -> expert FFN -> combine.  Top-8 of 16 routed
experts keeps the pool at 24 images (1.3 GB).  Bar: max|gpu-ref|/max|ref| <= 1e-2.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_ref as ref
from test_kernels_gpu import TOL, bf16_numpy, make_pool, rel_err

from paper_2504_05897_b200 import _lib, kernels as K

pytestmark = pytest.mark.gpu

H, I, N, KK, CHUNKS = 3584, 2560, 16, 8, 8


@pytest.fixture(scope="module")
def pool():
    return make_pool(N + CHUNKS, H, I, 17)


@pytest.mark.parametrize("T,path", [(1, _lib.FFN_AUTO), (4, _lib.FFN_GEMV), (128, _lib.FFN_AUTO)])
def test_qwen2_layer_with_shared_expert(pool, T, path):
    pool_t, experts = pool
    rng = np.random.default_rng(T)
    logits = rng.standard_normal((T, N + 1)).astype(np.float32)   # column N: the shared-expert gate logit
    x = torch.randn((T, H), device="cuda").to(torch.bfloat16)
    sel, w, probs, counts = K.router_topk(torch.from_numpy(logits).cuda(), N, KK, False, CHUNKS, N)
    offs = K.offsets(counts)
    pos, row_src = K.permute(sel, offs, N + CHUNKS)
    xp = K.gather_rows(x, row_src, KK + CHUNKS)
    rows = T * (KK + CHUNKS)
    h = torch.empty((rows, I), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((rows, H), device="cuda")
    o = offs.cpu().numpy()
    groups = [(e, int(o[e]), int(o[e + 1] - o[e])) for e in range(N + CHUNKS)]
    K.expert_ffn(pool_t, N + CHUNKS, H, I, groups, xp, h, out, path)
    y = K.combine(out, pos, w)
    torch.cuda.synchronize()
    # the shared expert as one (H, 8*I) SwiGLU
    sh = experts[N:]
    shared = (np.concatenate([e[0] for e in sh], 0), np.concatenate([e[1] for e in sh], 0),
              np.concatenate([e[2] for e in sh], 1))
    want = ref.moe_layer(bf16_numpy(x), logits, experts[:N] + [shared], N, KK, False, 1, N)
    err = rel_err(bf16_numpy(y), want)
    assert err <= TOL, err
