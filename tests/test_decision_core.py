"""Native decision core vs the reference's golden fixtures (bit-exact, CPU only)."""
from __future__ import annotations

import pytest

import paper_2504_05897_b200.caching as mc
import paper_2504_05897_b200.core as mcore
import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.engine as me
import paper_2504_05897_b200.prefetch as mp
import paper_2504_05897_b200.scheduling as ms
import paper_2504_05897_b200.tracegen as mt
from stream import digest, fx, from_records, plan_item

R = mcore.ExpertRef


def _cfg(d):
    d = dict(d)
    d["routed_expert_dims"] = tuple(d["routed_expert_dims"])
    if d.get("shared_expert_dims"):
        d["shared_expert_dims"] = tuple(d["shared_expert_dims"])
    return mcore.ModelConfig(**d)


def test_kats(golden):
    k = golden["kats"]
    C = mcore.ModelConfig
    assert mcore.expert_bytes(C(1, 8, 0, 2, (4096, 14336), None, 0.5)) == k["expert_bytes"][0]
    assert mcore.expert_bytes(C(1, 1, 0, 1, (1, 1), None, 1)) == k["expert_bytes"][1]
    assert mcore.expert_bytes(C(1, 64, 0, 6, (2048, 1408), None, 0.5)) == k["expert_bytes"][2]
    HP = mcost.HardwareProfile
    g = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1.0, gpu_saturation_load=128, gpu_slope=0.01)
    assert [mcost.gpu_time(g, x) for x in (1, 64, 228)] == k["gpu_time"]
    c = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.4)
    c1 = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    assert [mcost.cpu_time(c, 2, 0), mcost.cpu_time(c, 2, 3), mcost.cpu_time(c1, 1, 5)] == k["cpu_time"]
    t0 = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1e9)
    t1 = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1e9, transfer_latency=0.5)
    assert [mcost.transfer_time(t0, 3e9), mcost.transfer_time(t1, 1e9)] == k["transfer_time"]
    req = mcore.make_layer_request(0, [5, 1, 4, 2], [0.4, 0.1, 0.3, 0.2])
    cache = mcore.CacheState(4)
    cache.resident = {R(0, 0), R(0, 1)}
    gq, cq = ms.build_queues(req, cache)
    assert [[[t.ref[1], t.load] for t in gq], [[t.ref[1], t.load] for t in cq]] == k["build_queues"]
    p = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    assert plan_item(ms.select_plan(mcore.make_layer_request(0, [2], [1.0]), mcore.CacheState(1), p, 3.0)) == \
        k["single_uncached"]
    st = mc.MrsState(scores={R(0, 0): 0.4, R(0, 1): 0.2, R(0, 2): 0.0}, alpha=0.5, p=2)
    mc.mrs_update(st, 0, [0.6, 0.3, 0.1])
    assert [st.scores[R(0, i)] for i in range(3)] == k["mrs_update"]
    assert mc.top_p_filter([0.25] * 4, 2) == k["top_p_ties"]
    p = HP(gpu_time_per_expert=1.0, cpu_slope=5.0, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    assert mp.evaluate_gain(R(1, 0), mcore.make_layer_request(1, [1, 0], [0.9, 0.1]), mcore.CacheState(2),
                            ms.MakespanEvaluator(p, 3.0)) == k["evaluate_gain"]
    PC = mp.PrefetchCandidate
    cands = [PC(R(1, 0), 1, 5.0, 3.0, 1), PC(R(1, 1), 1, 3.0, 3.0, 1), PC(R(1, 2), 1, 1.0, 3.0, 1)]
    assert [list(r) for r in mp.select_prefetches(cands, 6.0)] == k["select_prefetches"]
    tie = [PC(R(2, 0), 1, 2.0, 1.0, 2), PC(R(1, 5), 1, 2.0, 1.0, 1)]
    assert [list(r) for r in mp.select_prefetches(tie, 1.0)] == k["select_prefetches_tie"]
    cache = mcore.CacheState(2)
    mc.insert_with_eviction(cache, R(0, 0), "lru")
    mc.insert_with_eviction(cache, R(0, 1), "lru")
    assert mc.lookup(cache, R(0, 0), "lru")
    assert list(mc.insert_with_eviction(cache, R(0, 2), "lru")) == k["lru_sequence"]
    cache = mcore.CacheState(2)
    cache.resident = {R(0, 0), R(0, 1)}
    st = mc.MrsState(scores={R(0, 0): 0.5, R(0, 1): 0.2}, alpha=0.5, p=2)
    assert list(mc.insert_with_eviction(cache, R(0, 2), "mrs", st)) == k["mrs_victim"]


def test_eviction_error_when_all_pinned():
    cache = mcore.CacheState(1)
    mc.insert_with_eviction(cache, R(0, 0), "lru")
    cache.pinned.add(R(0, 0))
    with pytest.raises(mc.EvictionError):
        mc.insert_with_eviction(cache, R(0, 1), "lru")
    with pytest.raises(ValueError):
        mc.insert_with_eviction(cache, R(0, 0), "lru")


def test_random_plans(golden):
    for case in golden["plans"]:
        prof = mcost.HardwareProfile(**case["profile"])
        layer, loads = case["layer"], case["loads"]
        req = mcore.make_layer_request(layer, loads, [1.0 / len(loads)] * len(loads))
        cache = mcore.CacheState(len(loads))
        cache.resident = {R(layer, i) for i in case["cached"]}
        plan = ms.select_plan(req, cache, prof, case["bytes"])
        assert plan_item(plan) == case["plan"]
        assert fx(ms.pcie_idle_budget(plan)) == case["budget"]
        ms.check_plan(plan)
        # the same instance through the generic (non-native cache) path
        class Plain:
            resident = {R(layer, i) for i in case["cached"]}
        assert plan_item(ms.select_plan(req, Plain(), prof, case["bytes"])) == case["plan"]
        if case["oracle"] is not None:
            assert fx(ms.oracle_optimal(req, cache, prof, case["bytes"])) == case["oracle"]


def test_tracegen_reproduces_reference(golden):
    cfg = mcore.ModelConfig(4, 8, 0, 2, (128, 256), None, 2)
    tr = mt.generate_trace(cfg, mt.GenParams(seed=5), 48, 6)
    got = [{"pass": p, "stage": f.stage, "layer": r.layer, "loads": list(r.loads), "scores": [fx(v) for v in r.scores]}
           for p, f in enumerate(tr.passes) for r in f.layers]
    assert got == golden["traces"]


def _run(entry):
    cfg = _cfg(entry["config"])
    tr = mt.generate_trace(cfg, mt.GenParams(seed=entry["gen_seed"]), entry["prefill"], entry["decode"])
    pol = me.EnginePolicy(scheduling=entry.get("scheduling", "hybrid"), cache_policy=entry["policy"],
                          prefetch=entry["prefetch"])
    return me.run_trace(tr, pol, entry["ratio"], mcost.HardwareProfile(**entry["profile"]), entry["seed"],
                        decision_log=True), pol


@pytest.mark.parametrize("idx", range(19))
def test_run_trace_records_and_streams(golden, idx):
    runs = golden["runs"]
    if idx >= len(runs):
        pytest.skip("no such run")
    entry = runs[idx]
    m, pol = _run(entry)
    assert m.to_record() == entry["record"], entry["name"]
    stream = from_records(m.decisions, pol.cache_policy == "mrs" and pol.scheduling != "static_layer_split")
    if entry["name"] in golden["streams"]:
        ref = golden["streams"][entry["name"]]
        for i, (a, b) in enumerate(zip(stream, ref)):
            assert a == b, (entry["name"], i)
    assert len(stream) == entry["stream_len"], entry["name"]
    assert digest(stream) == entry["stream_sha"], entry["name"]


def test_expected_eviction_errors(golden):
    cfg = mcore.ModelConfig(4, 8, 0, 2, (128, 256), None, 2)
    for case in golden["errors"]:
        tr = mt.generate_trace(cfg, mt.GenParams(seed=case["gen_seed"]), case["prefill"], case["decode"])
        prof = mcost.HardwareProfile(**case["profile"])
        if case["outcome"] == "EvictionError":
            with pytest.raises(mc.EvictionError):
                me.run_trace(tr, me.EnginePolicy(prefetch=True), case["ratio"], prof, case["seed"])
        else:
            m = me.run_trace(tr, me.EnginePolicy(prefetch=True), case["ratio"], prof, case["seed"])
            assert m.to_record() == case["record"]


def test_replay_trace_matches_oracle_properties():
    cfg = mcore.ModelConfig(4, 8, 0, 2, (128, 256), None, 2)
    tr = mt.generate_trace(cfg, mt.GenParams(seed=3), 32, 40)
    for pol in mc.POLICIES:
        st = mc.replay_trace(tr, pol, 8)
        assert st.lookups == sum(len(r.activated) for f in tr.passes for r in f.layers)
        assert 0 <= st.hits <= st.lookups and st.evictions <= st.inserts


def test_cache_views_behave_like_sets():
    cache = mcore.CacheState(3)
    for i in range(3):
        mc.insert_with_eviction(cache, R(1, i), "lfu")
    assert set(cache.resident) == {R(1, 0), R(1, 1), R(1, 2)}
    pins = {R(1, 0)}
    cache.pinned |= pins
    assert R(1, 0) in cache.pinned and len(cache.pinned) == 1
    cache.pinned -= pins
    assert len(cache.pinned) == 0
    assert cache.frequency[R(1, 2)] == 1
    assert mc.lookup(cache, R(1, 2), "lfu") and cache.frequency[R(1, 2)] == 2
    assert (cache.resident | {R(2, 0)}) == {R(1, 0), R(1, 1), R(1, 2), R(2, 0)}
    assert sorted(cache.slot_of(R(1, i)) for i in range(3)) == [0, 1, 2]
    v = mc.insert_with_eviction(cache, R(3, 3), "lfu")
    assert v == R(1, 0) and cache.slot_of(R(3, 3)) == 0 and cache.slot_of(R(1, 0)) == -1
