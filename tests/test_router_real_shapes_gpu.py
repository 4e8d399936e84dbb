"""GPU router at the real model shapes against the unmodified reference's loads.

For Mixtral-8x7B (N=8, K=2), DeepSeek-V2-Lite (N=64, K=6, 2 shared) and
Qwen2-57B-A14B (N=64, K=8, 1 shared of 8 chunks, sigmoid gate column) at
generator seeds 0-4: the 1024-token prefill logits go through the prefill
router kernel (hm_router_topk) and every decode pass's logits through the
fused one-block decode router (hm_router_fused_small), each with the family's
conventions; the routed-expert counts must equal the loads the reference's
generate_trace recorded (tests/golden/router_real_shapes.json,
tracegen.py:137-148).  The logits themselves are pinned to the reference by
tests/test_router_real_shapes.py.  Rows whose K/K+1 margin is below the fp32
cast error are reported (see AMBIGUOUS there): they must not change any load.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from test_router_real_shapes import AMBIGUOUS, CASES, GOLD, ambiguous_rows

from paper_2504_05897_b200 import _lib, kernels as K
from paper_2504_05897_b200.moe import FAMILIES, SHAPES, shared_chunks
from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits

pytestmark = pytest.mark.gpu


def fused_decode_counts(lg: np.ndarray, N: int, k: int, S: int, renorm: bool, gate: int, H: int = 256) -> list:
    T, ld = lg.shape
    kp, E = k + S, N + S
    dev = "cuda"
    logits = torch.from_numpy(np.ascontiguousarray(lg, dtype=np.float32)).to(dev)
    x = torch.zeros((T, H), dtype=torch.bfloat16, device=dev)
    sel = torch.empty((T, kp), dtype=torch.int32, device=dev)
    w = torch.empty((T, kp), device=dev)
    pos = torch.empty((T, kp), dtype=torch.int32, device=dev)
    row_src = torch.empty((T * kp,), dtype=torch.int32, device=dev)
    xp = torch.empty((T * kp, H), dtype=torch.bfloat16, device=dev)
    mi = torch.empty((2 * E + 2,), dtype=torch.int32, device=dev)
    md = torch.empty((2 * N,), dtype=torch.float64, device=dev)
    f = _lib.lib.hm_router_fused_small
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                  C.c_int] + [C.c_void_p] * 8
    _lib.check(f(logits.data_ptr(), T, N, ld, k, int(renorm), S, gate, x.data_ptr(), H, sel.data_ptr(), w.data_ptr(),
                 pos.data_ptr(), row_src.data_ptr(), xp.data_ptr(), mi.data_ptr(), md.data_ptr(),
                 torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return mi[:N].cpu().tolist()


@pytest.mark.parametrize("shape,seed", CASES)
def test_gpu_router_loads_equal_reference_trace(shape, seed):
    cfg = SHAPES[shape]
    fam = FAMILIES[shape]
    N, k, S = cfg.num_routed, cfg.num_activated, shared_chunks(cfg)
    gate = N if fam.shared_gate else -1
    run = GOLD["shapes"][shape]["runs"][seed]
    _, logits = generate_router_logits(cfg, GenParams(seed=seed), GOLD["prefill"], GOLD["decode"])
    report = []
    for l in range(cfg.num_layers):
        z = logits[0][l]
        lg = z.astype(np.float32)
        if fam.shared_gate:  # the runtime's [T, N+1] layout: gate logit in column N
            lg = np.concatenate([lg, np.zeros((lg.shape[0], 1), np.float32)], axis=1)
        sel, w, probs, counts = K.router_topk(torch.from_numpy(np.ascontiguousarray(lg)).cuda(), N, k,
                                              fam.renormalize, S, gate)
        torch.cuda.synchronize()
        c = counts.cpu().numpy()
        assert c[:N].tolist() == run["prefill_loads"][l], (shape, seed, "prefill", l)
        assert c[N:].tolist() == [GOLD["prefill"]] * S  # every token routes to every shared chunk
        for row in ambiguous_rows(z, k):
            report.append((l, int(row)))
    for p in range(GOLD["decode"]):
        for l in range(cfg.num_layers):
            lg = logits[1 + p][l].astype(np.float32)
            if fam.shared_gate:
                lg = np.concatenate([lg, np.zeros((1, 1), np.float32)], axis=1)
            got = fused_decode_counts(lg, N, k, S, fam.renormalize, gate)
            assert got == run["decode_loads"][p][l], (shape, seed, "decode", p, l)
    print(f"{shape} seed {seed}: ambiguous K/K+1 rows (layer, token) = {report}; all loads equal the reference")
    assert len(report) == AMBIGUOUS.get((shape, seed), 0)
