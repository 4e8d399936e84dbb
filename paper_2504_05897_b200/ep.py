"""Expert parallelism across the GPUs of one box.

Expert (l, e) is homed on rank ``e % G`` (shared chunk c on ``c % G``).  Each
rank owns its home experts' pinned host images, a share of the *global*
cache budget floor(ratio * L * N) (split as evenly as possible), its own host
worker cores and its own decision core, which sees the rank-masked
LayerRequest: loads of non-home experts zeroed, scores kept whole so every
rank's MRS table is the same.  Per-rank decisions therefore equal the
reference's ``run_trace`` on the rank-masked trace (tests/test_ep.py).

Exchange: the hidden state of the sequence is replicated; every rank routes
it identically, computes the partial ``sum_k w_k E_k(x)`` over its home
experts and the partials are summed with one all-reduce per layer (NCCL over
NVLink on the GPUs; gloo in the CPU tests), then the residual is added.
"""
from __future__ import annotations

import math

from .core import ForwardPass, LayerRequest, ModelConfig, Trace


def home_rank(expert: int, world: int) -> int:
    return expert % world


def home_experts(n_routed: int, rank: int, world: int) -> list[int]:
    return [e for e in range(n_routed) if e % world == rank]


def rank_capacity(config: ModelConfig, ratio: float, rank: int, world: int) -> int:
    """This rank's share of the global budget floor(ratio * L * N) (engine.py:401-404)."""
    if not 0.0 < ratio <= 1.0:
        raise ValueError(f"capacity_ratio must be in (0, 1], got {ratio}")
    total = math.floor(ratio * config.total_routed_experts)
    return total // world + (1 if rank < total % world else 0)


def mask_request(req: LayerRequest, rank: int, world: int) -> LayerRequest:
    """Loads of experts homed elsewhere zeroed; scores untouched."""
    loads = tuple(v if i % world == rank else 0 for i, v in enumerate(req.loads))
    return LayerRequest(layer=req.layer, loads=loads, scores=req.scores,
                        activated=frozenset(i for i in req.activated if i % world == rank))


def mask_trace(trace: Trace, rank: int, world: int) -> Trace:
    """The rank-masked trace (run_trace never validates, so masked requests are legal)."""
    return Trace(config=trace.config, metadata=dict(trace.metadata),
                 passes=tuple(ForwardPass(f.stage, f.token_count, tuple(mask_request(r, rank, world) for r in f.layers))
                              for f in trace.passes))


def rank_ratio(config: ModelConfig, ratio: float, rank: int, world: int) -> float:
    """A capacity ratio whose floor(ratio * L * N) is exactly this rank's slot count."""
    cap = rank_capacity(config, ratio, rank, world)
    return min(1.0, (cap + 0.5) / config.total_routed_experts)
