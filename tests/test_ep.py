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


def _dispatch_worker(rank, world, port, q):
    """Token-sharded mode's algorithm (csrc/ep_exchange.cu) restated on CPU:
    local routing of this rank's tokens, all-gather of per-expert counts and
    fp64 score sums, home layout (experts in index order, rows by source rank
    then source order), all-to-all of rows to home ranks, expert compute at
    home, all-to-all back, local combine."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1)
        T, N, K, S, H, I = 13, 8, 2, 1, 32, 128
        E, Kp = N + S, K + S
        x = rng.standard_normal((T, H)).astype(np.float32)
        logits = rng.standard_normal((T, N)).astype(np.float32)
        experts = [tuple(rng.standard_normal(s).astype(np.float32) * 0.05 for s in ((I, H), (I, H), (H, I)))
                   for _ in range(E)]
        home = [(e if e < N else e - N) % world for e in range(E)]
        a, b = rank * T // world, (rank + 1) * T // world
        xl, ll = x[a:b], logits[a:b]
        sel, w, probs, counts, _ = ref.router(ll, N, K, False, S)
        counts = np.asarray(counts, dtype=np.int64)
        sums = probs.astype(np.float64).sum(axis=0) if len(ll) else np.zeros(N)
        # all-gather counts and score sums; global LayerRequest in rank order
        ca = [torch.zeros(E, dtype=torch.int64) for _ in range(world)]
        sa = [torch.zeros(N, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ca, torch.from_numpy(counts))
        dist.all_gather(sa, torch.from_numpy(sums))
        ca = np.stack([c.numpy() for c in ca])
        gsum = np.zeros(N)
        for s in range(world):
            gsum = gsum + sa[s].numpy()
        # local permutation: rows grouped by expert, token order inside
        order = sorted(range(len(xl) * Kp), key=lambda j: (int(sel.reshape(-1)[j]), j))
        lrows = [(int(sel.reshape(-1)[j]), j // Kp) for j in order]
        local_off = np.concatenate([[0], np.cumsum(counts)])
        # home layout and destinations
        run = [0] * world
        recv_base = np.zeros(E, dtype=np.int64)
        for e in range(E):
            recv_base[e] = run[home[e]]
            run[home[e]] += int(ca[:, e].sum())
        src_base = np.concatenate([np.zeros((1, E), np.int64), np.cumsum(ca, axis=0)])
        send = [[] for _ in range(world)]
        for p, (e, t) in enumerate(lrows):
            send[home[e]].append((int(recv_base[e] + src_base[rank, e] + p - local_off[e]), e, xl[t]))
        # all-to-all of rows (object lists stand in for the P2P stores)
        got = [None] * world
        for dst in range(world):
            gl = [None] * world
            dist.all_gather_object(gl, send[dst])
            if dst == rank:
                got = gl
        recv = {}
        for s in range(world):
            for pos, e, row in got[s]:
                recv[pos] = (s, e, row)
        assert sorted(recv) == list(range(run[rank]))
        # experts at home, then back to the sources' permuted positions
        back = [[] for _ in range(world)]
        for pos, (s, e, row) in recv.items():
            r = pos - recv_base[e]
            lo = ca[s, :e].sum()
            back[s].append((int(lo + r - src_base[s, e]), ref.expert(row[None], *experts[e])[0]))
        ret = {}
        for src in range(world):
            gl = [None] * world
            dist.all_gather_object(gl, back[src])
            if src == rank:
                for lst in gl:
                    ret.update(dict(lst))
        # local combine
        pos_of = {(t, e): p for p, (e, t) in enumerate(lrows)}
        y = xl.copy()
        for t in range(len(xl)):
            for k in range(Kp):
                e = int(sel[t, k])
                y[t] += w[t, k] * ret[pos_of[(t, e)]]
        want = ref.moe_layer(x, logits, experts, N, K, False, S, residual=True)[a:b]
        ref_sel, _, ref_probs, ref_counts, _ = ref.router(logits, N, K, False, S)
        ok_counts = list(ca.sum(axis=0)) == [int(v) for v in ref_counts]
        err = float(np.abs(y - want).max() / np.abs(want).max()) if len(y) else 0.0
        q.put((rank, err, ok_counts, float(np.abs(gsum - ref_probs.astype(np.float64).sum(axis=0)).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_token_sharded_dispatch_equals_full_layer():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dispatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = {r: (e, ok, ds) for r, e, ok, ds in (q.get(timeout=5) for _ in range(2))}
    assert all(p.exitcode == 0 for p in procs)
    for r, (err, ok_counts, dsum) in res.items():
        assert ok_counts and err < 1e-5 and dsum < 1e-12, (r, err, ok_counts, dsum)


def _a2a_worker(rank, world, port, q):
    """The NCCL transport's schedule (native hm_ep_a2a_plan) executed with gloo
    point-to-point ops in the same issue order: every rank's rows must land in
    the home layout the peer-memory kernels write, and come back."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, S, Hs = 10, 2, 3
        E = N + S
        rng = np.random.default_rng(100 + world)
        counts = rng.integers(0, 4, size=(world, E)).astype(np.int32)   # same draw on every rank
        counts[world - 1] = 0                                            # one rank holds no tokens
        mine = torch.from_numpy(counts[rank].copy())
        gathered = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gathered, mine)                                  # the all-gathered count matrix
        cnt = torch.stack(gathered).numpy()
        assert (cnt == counts).all()
        home = lambda e: (e if e < N else e - N) % world                # noqa: E731
        # local permuted rows: expert-contiguous, value = (rank, expert, index)
        local = np.array([[rank, e, i] for e in range(E) for i in range(cnt[rank, e])], dtype=np.float32)
        local = torch.from_numpy(local.reshape(-1, Hs))

        def run(plan, src, n_dst):
            dst = torch.full((n_dst, Hs), -1.0)
            reqs = []
            for kind, peer, s0, d0, n in plan:
                if kind == 2:
                    dst[d0:d0 + n] = src[s0:s0 + n]
                elif kind == 0:
                    reqs.append(dist.isend(src[s0:s0 + n].contiguous(), peer))
                else:
                    buf = torch.empty((n, Hs))
                    reqs.append((dist.irecv(buf, peer), buf, d0, n))
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    dst[r[2]:r[2] + r[3]] = r[1]
                else:
                    r.wait()
            return dst

        # dispatch: home layout = my experts in index order, rows by source rank then source order
        want = np.array([[s, e, i] for e in range(E) if home(e) == rank for s in range(world)
                         for i in range(cnt[s, e])], dtype=np.float32).reshape(-1, Hs)
        recv = run(ep.a2a_plan(cnt, world, E, N, rank, 0), local, len(want))
        assert np.array_equal(recv.numpy(), want)
        # "experts" on the home rank, then the return all-to-all to the source positions
        back = run(ep.a2a_plan(cnt, world, E, N, rank, 1), recv * 2 + 1, local.shape[0])
        assert torch.equal(back, local * 2 + 1)
        q.put((rank, True))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_nccl_a2a_schedule_moves_rows_to_home_layout_and_back(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(q.get(timeout=5) for _ in range(world)) == {r: True for r in range(world)}


def test_a2a_plan_validates_and_counts():
    cnt = np.array([[1, 0, 2], [0, 3, 1]], dtype=np.int32)
    ops0 = ep.a2a_plan(cnt, 2, 3, 3, 0, 0)
    # rank 0: expert 0 (home 0) local copy, expert 2 (home 0) local copy; receives expert 2 from rank 1
    assert ops0 == [(2, 0, 0, 0, 1), (2, 0, 1, 1, 2), (1, 1, 3, 3, 1)]
    from paper_2504_05897_b200 import _lib
    with pytest.raises(ValueError):
        ep.a2a_plan(-cnt, 2, 3, 3, 0, 0)
    assert "negative" in _lib.last_error()
