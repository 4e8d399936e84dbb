"""Expert parallelism on CPU: per-rank decision parity on the
rank-masked traces, and a world-size-2 gloo run of the exchange (partial
expert sums all-reduced across ranks) against the single-process layer."""
from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import decisions as od
from oracle import moe_ref as ref

import paper_2504_05897_b200.core as mcore
import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.engine as me
from paper_2504_05897_b200 import ep
from paper_2504_05897_b200.tracegen import GenParams, generate_trace


def _profile(cfg):
    eb = mcore.expert_bytes(cfg)
    return mcost.HardwareProfile(gpu_time_per_expert=1, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)


@pytest.mark.parametrize("world", [2, 4])
def test_rank_capacities_sum_to_global_budget(world):
    cfg = mcore.ModelConfig(32, 8, 0, 2, (4096, 14336), None, 2)
    caps = [ep.rank_capacity(cfg, 0.25, r, world) for r in range(world)]
    assert sum(caps) == math.floor(0.25 * 32 * 8) and max(caps) - min(caps) <= 1
    for r in range(world):
        assert math.floor(ep.rank_ratio(cfg, 0.25, r, world) * cfg.total_routed_experts) == caps[r]


@pytest.mark.parametrize("world,policy,prefetch", [(2, "mrs", True), (2, "lru", False), (4, "lfu", True)])
def test_per_rank_decisions_equal_oracle_on_masked_trace(world, policy, prefetch):
    cfg = mcore.ModelConfig(4, 16, 0, 4, (128, 256), None, 2)
    prof = _profile(cfg)
    tr = generate_trace(cfg, GenParams(seed=4), 96, 24)
    pdict = {k: getattr(prof, k) for k in prof.__dataclass_fields__}
    for r in range(world):
        masked = ep.mask_trace(tr, r, world)
        ratio = ep.rank_ratio(cfg, 0.5, r, world)
        m = me.run_trace(masked, me.EnginePolicy(cache_policy=policy, prefetch=prefetch), ratio, prof, 3).to_record()
        passes = [(f.stage, [(q.layer, list(q.loads), list(q.scores)) for q in f.layers]) for f in masked.passes]
        o = od.run(passes, cfg.num_layers, cfg.num_routed, cfg.num_activated, mcore.expert_bytes(cfg), pdict,
                   ep.rank_capacity(cfg, 0.5, r, world), policy, prefetch,
                   predict=lambda pi, l: od.predictions(passes[pi][1], pi, l, 3))
        for k in ("ttft", "mean_tbt", "hits", "inserts", "evictions", "prefetch_issued", "elapsed"):
            assert m[k] == o[k], (r, k)
        # every activated expert of the full trace is planned by exactly one rank
    total = sum(len(q.activated) for f in tr.passes for q in f.layers)
    planned = sum(len(q.activated) for r in range(world) for f in ep.mask_trace(tr, r, world).passes
                  for q in f.layers)
    assert planned == total


@pytest.mark.reference
def test_per_rank_decisions_equal_reference_on_masked_trace(moesim):
    import moesim.core as rc
    import moesim.costs as rco
    import moesim.engine as re_
    import moesim.tracegen as rt

    cfg = rc.ModelConfig(num_layers=4, num_routed=16, num_shared=0, num_activated=4, routed_expert_dims=(128, 256),
                         bytes_per_weight=2)
    eb = rc.expert_bytes(cfg)
    rprof = rco.HardwareProfile(gpu_time_per_expert=1, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                cpu_first_expert_penalty=1.4)
    rtr = rt.generate_trace(cfg, rt.GenParams(seed=4), 96, 24)
    mine_cfg = mcore.ModelConfig(4, 16, 0, 4, (128, 256), None, 2)
    tr = generate_trace(mine_cfg, GenParams(seed=4), 96, 24)
    for r in range(2):
        rm = rc.Trace(config=cfg, passes=tuple(
            rc.ForwardPass(f.stage, f.token_count, tuple(
                rc.LayerRequest(q.layer, tuple(v if i % 2 == r else 0 for i, v in enumerate(q.loads)), q.scores,
                                frozenset(i for i in q.activated if i % 2 == r)) for q in f.layers))
            for f in rtr.passes))
        ratio = ep.rank_ratio(mine_cfg, 0.5, r, 2)
        want = re_.run_trace(rm, re_.EnginePolicy(prefetch=True), ratio, rprof, 3).to_record()
        got = me.run_trace(ep.mask_trace(tr, r, 2), me.EnginePolicy(prefetch=True), ratio, _profile(mine_cfg),
                           3).to_record()
        assert got == want


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)          # identical on every rank: replicated x and router
        T, N, K, S, H, I = 12, 8, 2, 2, 64, 128
        x = rng.standard_normal((T, H)).astype(np.float32)
        logits = rng.standard_normal((T, N)).astype(np.float32)
        experts = [tuple(rng.standard_normal(s).astype(np.float32) * 0.05 for s in ((I, H), (I, H), (H, I)))
                   for _ in range(N + S)]
        sel, w, *_ = ref.router(logits, N, K, False, S)
        part = np.zeros((T, H), dtype=np.float32)
        for t in range(T):
            for k in range(K + S):
                e = int(sel[t, k])
                owner = (e if e < N else e - N) % world
                if owner == rank:                # this rank's home experts only
                    part[t] += w[t, k] * ref.expert(x[t:t + 1], *experts[e])[0]
        pt = torch.from_numpy(part)
        dist.all_reduce(pt)                      # the combine exchange
        y = x + pt.numpy()
        want = ref.moe_layer(x, logits, experts, N, K, False, S, residual=True)
        q.put((rank, float(np.abs(y - want).max() / np.abs(want).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partial_sums_equal_full_layer():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert max(res.values()) < 1e-5
