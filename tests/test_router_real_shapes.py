"""Router inputs at the real model shapes, pinned to the unmodified reference.

tests/golden/router_real_shapes.json was written by running the reference's
trace generator (moesim.tracegen.generate_trace, tracegen.py:100-163) with its
`_softmax` wrapped to record the exact fp64 logits it routes on
(tests/golden/make_router_golden.py).  Here, on CPU:
  * this package's generator reproduces those logits bit for bit (SHA-256 per
    layer) and the loads, for the Mixtral / DeepSeek-V2-Lite / Qwen2-57B shapes
    at seeds 0-4 (1024-token prefill + 4 decode passes);
  * the tie-margin report: rows whose K-th vs (K+1)-th fp64 logit margin is
    below the fp64->fp32 cast error (where fp32 top-K could legitimately differ
    from the reference's fp64 argpartition, tracegen.py:147), and the fp32
    (value desc, index asc) rule of the oracle router still giving the
    reference's loads on every layer, ambiguous rows included.
The GPU router is checked against the same loads in test_router_real_shapes_gpu.py.
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import moe_ref as ref

from paper_2504_05897_b200.moe import FAMILIES, SHAPES
from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "router_real_shapes.json").read_text())
CASES = [(s, r["seed"]) for s in GOLD["shapes"] for r in GOLD["shapes"][s]["runs"]]
# (shape, seed) -> rows whose K/K+1 margin is below the cast error (computed once, frozen here)
AMBIGUOUS = {("deepseek", 1): 1, ("qwen2", 0): 1}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def ambiguous_rows(z: np.ndarray, k: int) -> np.ndarray:
    """Rows where fp32 rounding could reorder the K-th and (K+1)-th logits."""
    s = -np.sort(-z, axis=1)
    margin = s[:, k - 1] - s[:, k]
    bound = np.ldexp(np.maximum(np.abs(s[:, k - 1]), np.abs(s[:, k])), -23)
    return np.flatnonzero(margin <= bound)


@pytest.mark.parametrize("shape,seed", CASES)
def test_generator_reproduces_reference_logits(shape, seed):
    cfg = SHAPES[shape]
    run = GOLD["shapes"][shape]["runs"][seed]
    trace, logits = generate_router_logits(cfg, GenParams(seed=seed), GOLD["prefill"], GOLD["decode"])
    assert [sha(logits[0][l]) for l in range(cfg.num_layers)] == run["prefill_logits_sha"]
    assert [list(r.loads) for r in trace.passes[0].layers] == run["prefill_loads"]
    for p in range(GOLD["decode"]):
        assert [sha(logits[1 + p][l]) for l in range(cfg.num_layers)] == run["decode_logits_sha"][p]
        assert [list(r.loads) for r in trace.passes[1 + p].layers] == run["decode_loads"][p]


@pytest.mark.parametrize("shape,seed", CASES)
def test_tie_margin_report_and_fp32_rule(shape, seed):
    cfg = SHAPES[shape]
    fam = FAMILIES[shape]
    run = GOLD["shapes"][shape]["runs"][seed]
    _, logits = generate_router_logits(cfg, GenParams(seed=seed), GOLD["prefill"], 0)
    n_amb = 0
    for l in range(cfg.num_layers):
        z = logits[0][l]
        n_amb += len(ambiguous_rows(z, cfg.num_activated))
        _, _, _, counts, _ = ref.router(z.astype(np.float32), cfg.num_routed, cfg.num_activated, fam.renormalize)
        assert counts[: cfg.num_routed].tolist() == run["prefill_loads"][l], (shape, seed, l)
    assert n_amb == AMBIGUOUS.get((shape, seed), 0)
