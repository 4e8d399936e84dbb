"""Generate the golden fixtures by running the UNMODIFIED reference (moesim).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/decisions.json.  Contents:
  kats      SPEC.md known-answer examples evaluated by moesim
  runs      run_trace records + SHA-256 of the canonical decision stream
            (tests/golden/stream.py) for the stress grid of SURVEY.md §4.4 and
            for Mixtral / DeepSeek-V2-Lite / Qwen2-57B shaped traces
  streams   two full decision streams (for debugging a hash mismatch)
  errors    runs that must raise EvictionError on a demand insert (§4.4)
  plans     random select_plan instances: inputs and the exact plan
  traces    generate_trace outputs (loads, scores as float.hex) for tracegen parity
numpy's Generator streams are version-dependent, so the fixtures are frozen
here rather than regenerated at test time.
"""
from __future__ import annotations

import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import moesim.caching as mc  # noqa: E402
import moesim.core as mcore  # noqa: E402
import moesim.costs as mcost  # noqa: E402
import moesim.engine as me  # noqa: E402
import moesim.prefetch as mp  # noqa: E402
import moesim.scheduling as ms  # noqa: E402
import moesim.tracegen as mt  # noqa: E402
from stream import digest, fx, insert_item, plan_item, row_hash  # noqa: E402

TINY = dict(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(128, 256),
            bytes_per_weight=2)
SHAPES = {
    "mixtral": dict(num_layers=32, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(4096, 14336),
                    bytes_per_weight=2),
    "deepseek": dict(num_layers=26, num_routed=64, num_shared=2, num_activated=6, routed_expert_dims=(2048, 1408),
                     shared_expert_dims=(2048, 1408), bytes_per_weight=2),
    "qwen2": dict(num_layers=28, num_routed=64, num_shared=1, num_activated=8, routed_expert_dims=(3584, 2560),
                  shared_expert_dims=(3584, 20480), bytes_per_weight=2),
}
PROFILE_FIELDS = [f for f in mcost.HardwareProfile.__dataclass_fields__]


def prof_dict(p) -> dict:
    return {k: getattr(p, k) for k in PROFILE_FIELDS}


def stress_profile(cfg) -> mcost.HardwareProfile:
    eb = mcore.expert_bytes(cfg)
    return mcost.HardwareProfile(gpu_time_per_expert=1, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)


def b200_like_profile(cfg) -> mcost.HardwareProfile:
    """Seconds; a plausible B200 host: 6.4 TB/s HBM, 100 GB/s host DRAM, 55 GB/s PCIe."""
    eb = mcore.expert_bytes(cfg)
    return mcost.HardwareProfile(gpu_time_per_expert=eb / 6.4e12 + 4e-6, cpu_slope=eb / 100e9,
                                 transfer_bandwidth=55e9, transfer_latency=1e-5, gpu_saturation_load=256,
                                 gpu_slope=2.0 * 3 * cfg.routed_expert_dims[0] * cfg.routed_expert_dims[1] / 1.2e15,
                                 cpu_first_expert_penalty=1.15)


class Recorder:
    """Wraps the engine-level names of moesim.engine (engine.py:27-64) to log decisions."""

    NAMES = ("lookup", "insert_with_eviction", "mrs_update", "evaluate_gain", "select_prefetches", "_build_plan")

    def __init__(self) -> None:
        self.stream: list = []
        self.saved = {n: getattr(me, n) for n in self.NAMES}

    def __enter__(self):
        s = self.saved
        st = self.stream

        def lookup(cache, ref, policy):
            h = s["lookup"](cache, ref, policy)
            st.append(["L", ref[0], ref[1], int(h)])
            return h

        def insert(cache, ref, policy, mrs=None):
            try:
                v = s["insert_with_eviction"](cache, ref, policy, mrs)
            except mc.EvictionError:
                st.append(insert_item(ref, "E"))
                raise
            st.append(insert_item(ref, v))
            return v

        def mrs_update(state, layer, scores):
            out = s["mrs_update"](state, layer, scores)
            n = len(scores)
            st.append(["M", layer, row_hash([state.scores[mcore.ExpertRef(layer, i)] for i in range(n)])])
            return out

        def evaluate_gain(cand, pred, cache, evaluator):
            g = s["evaluate_gain"](cand, pred, cache, evaluator)
            st.append(["G", cand[0], cand[1], fx(g)])
            return g

        def select_prefetches(cands, budget):
            out = s["select_prefetches"](cands, budget)
            st.append(["S", fx(budget), [[r[0], r[1]] for r in out]])
            return out

        def build_plan(*a, **k):
            plan = s["_build_plan"](*a, **k)
            st.append(plan_item(plan))
            return plan

        me.lookup, me.insert_with_eviction, me.mrs_update = lookup, insert, mrs_update
        me.evaluate_gain, me.select_prefetches, me._build_plan = evaluate_gain, select_prefetches, build_plan
        return self

    def __exit__(self, *exc):
        for n, f in self.saved.items():
            setattr(me, n, f)
        return False


def record_run(trace, policy, ratio, profile, seed):
    with Recorder() as rec:
        m = me.run_trace(trace, policy, ratio, profile, seed)
    # validate replans (policy.validate) would log extra plans; keep validate off
    return m.to_record(), rec.stream


def kats() -> dict:
    out = {}
    C = mcore.ModelConfig
    out["expert_bytes"] = [
        mcore.expert_bytes(C(num_layers=1, num_routed=8, num_shared=0, num_activated=2,
                             routed_expert_dims=(4096, 14336), bytes_per_weight=0.5)),
        mcore.expert_bytes(C(num_layers=1, num_routed=1, num_shared=0, num_activated=1, routed_expert_dims=(1, 1),
                             bytes_per_weight=1)),
        mcore.expert_bytes(C(num_layers=1, num_routed=64, num_shared=0, num_activated=6,
                             routed_expert_dims=(2048, 1408), bytes_per_weight=0.5)),
    ]
    HP = mcost.HardwareProfile
    g = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1.0, gpu_saturation_load=128, gpu_slope=0.01)
    out["gpu_time"] = [mcost.gpu_time(g, 1), mcost.gpu_time(g, 64), mcost.gpu_time(g, 228)]
    c = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.4)
    c1 = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    out["cpu_time"] = [mcost.cpu_time(c, 2, 0), mcost.cpu_time(c, 2, 3), mcost.cpu_time(c1, 1, 5)]
    t0 = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1e9)
    t1 = HP(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1e9, transfer_latency=0.5)
    out["transfer_time"] = [mcost.transfer_time(t0, 3e9), mcost.transfer_time(t1, 1e9)]
    # build_queues: A:5,B:1 cached; C:4,D:2 uncached
    req = mcore.make_layer_request(0, [5, 1, 4, 2], [0.4, 0.1, 0.3, 0.2])
    cache = mcore.CacheState(4)
    cache.resident |= {mcore.ExpertRef(0, 0), mcore.ExpertRef(0, 1)}
    gq, cq = ms.build_queues(req, cache)
    out["build_queues"] = [[[t.ref[1], t.load] for t in gq], [[t.ref[1], t.load] for t in cq]]
    # single uncached expert
    p = HP(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    plan = ms.select_plan(mcore.make_layer_request(0, [2], [1.0]), mcore.CacheState(1), p, 3.0)
    out["single_uncached"] = plan_item(plan)
    # mrs_update and the TopP tie rule
    st = mc.MrsState(scores={mcore.ExpertRef(0, 0): 0.4, mcore.ExpertRef(0, 1): 0.2, mcore.ExpertRef(0, 2): 0.0},
                     alpha=0.5, p=2)
    mc.mrs_update(st, 0, [0.6, 0.3, 0.1])
    out["mrs_update"] = [st.scores[mcore.ExpertRef(0, i)] for i in range(3)]
    out["top_p_ties"] = mc.top_p_filter([0.25, 0.25, 0.25, 0.25], 2)
    # evaluate_gain: transfer 3, gpu 1, cpu 5
    p = HP(gpu_time_per_expert=1.0, cpu_slope=5.0, transfer_bandwidth=1.0, cpu_first_expert_penalty=1.0)
    ev = ms.MakespanEvaluator(p, 3.0)
    out["evaluate_gain"] = mp.evaluate_gain(mcore.ExpertRef(1, 0), mcore.make_layer_request(1, [1, 0], [0.9, 0.1]),
                                            mcore.CacheState(2), ev)
    # select_prefetches
    R = mcore.ExpertRef
    cands = [mp.PrefetchCandidate(R(1, 0), 1, 5.0, 3.0, 1), mp.PrefetchCandidate(R(1, 1), 1, 3.0, 3.0, 1),
             mp.PrefetchCandidate(R(1, 2), 1, 1.0, 3.0, 1)]
    out["select_prefetches"] = [[r[0], r[1]] for r in mp.select_prefetches(cands, 6.0)]
    tie = [mp.PrefetchCandidate(R(2, 0), 1, 2.0, 1.0, 2), mp.PrefetchCandidate(R(1, 5), 1, 2.0, 1.0, 1)]
    out["select_prefetches_tie"] = [[r[0], r[1]] for r in mp.select_prefetches(tie, 1.0)]
    # LRU sequence: insert A, insert B, lookup A, insert C -> evicts B
    cache = mcore.CacheState(2)
    A, B, Cc = R(0, 0), R(0, 1), R(0, 2)
    mc.insert_with_eviction(cache, A, "lru")
    mc.insert_with_eviction(cache, B, "lru")
    mc.lookup(cache, A, "lru")
    out["lru_sequence"] = list(mc.insert_with_eviction(cache, Cc, "lru"))
    # MRS min-S
    cache = mcore.CacheState(2)
    cache.resident |= {A, B}
    st = mc.MrsState(scores={A: 0.5, B: 0.2}, alpha=0.5, p=2)
    out["mrs_victim"] = list(mc.insert_with_eviction(cache, Cc, "mrs", st))
    return out


def random_plans(n: int = 400, seed: int = 7) -> list:
    rnd = random.Random(seed)
    out = []
    for k in range(n):
        nexp = rnd.randint(1, 12)
        N = rnd.randint(nexp, 16)
        layer = rnd.randint(0, 3)
        chosen = rnd.sample(range(N), nexp)
        loads = [0] * N
        for i in chosen:
            loads[i] = rnd.choice([1, 1, 2, 3, 5, 8, 16, 64, 300]) if k % 3 else rnd.randint(1, 4)
        scores = [1.0 / N] * N
        cached = sorted(rnd.sample(chosen, rnd.randint(0, nexp)))
        prof = mcost.HardwareProfile(
            gpu_time_per_expert=rnd.choice([1.0, 0.5, 0.1, 2.0]), cpu_slope=rnd.choice([0.05, 0.2, 0.5, 1.0, 2.0]),
            transfer_bandwidth=rnd.choice([1.0, 2.0, 0.25]), transfer_latency=rnd.choice([0.0, 0.1]),
            gpu_saturation_load=rnd.choice([4, 64, 256]), gpu_slope=rnd.choice([0.0, 0.01, 0.1]),
            cpu_first_expert_penalty=rnd.choice([1.0, 1.2, 1.4, 2.0]))
        nbytes = rnd.choice([1.0, 2.5, 3.0, 7.0])
        req = mcore.make_layer_request(layer, loads, scores)
        cache = mcore.CacheState(N)
        cache.resident |= {mcore.ExpertRef(layer, i) for i in cached}
        plan = ms.select_plan(req, cache, prof, nbytes)
        out.append({"layer": layer, "loads": loads, "cached": cached, "profile": prof_dict(prof), "bytes": nbytes,
                    "plan": plan_item(plan), "budget": fx(ms.pcie_idle_budget(plan)),
                    "oracle": fx(ms.oracle_optimal(req, cache, prof, nbytes)) if nexp <= 10 else None})
    return out


def main() -> None:
    golden = {"numpy": np.__version__, "kats": kats(), "runs": [], "streams": {}, "errors": [], "plans": [],
              "traces": []}
    tiny = mcore.ModelConfig(**TINY)
    tr = mt.generate_trace(tiny, mt.GenParams(seed=2), 64, 32)
    hp = stress_profile(tiny)
    for pol in ("mrs", "lru", "lfu"):
        for pf in (False, True):
            rec, stream = record_run(tr, me.EnginePolicy(cache_policy=pol, prefetch=pf), 0.25, hp, 2)
            name = f"tiny-{pol}-{'pf' if pf else 'nopf'}"
            golden["runs"].append({"name": name, "config": TINY, "gen_seed": 2, "prefill": 64, "decode": 32,
                                   "ratio": 0.25, "profile": prof_dict(hp), "policy": pol, "prefetch": pf, "seed": 2,
                                   "record": rec, "stream_sha": digest(stream), "stream_len": len(stream)})
            if name in ("tiny-mrs-pf", "tiny-lfu-pf"):
                golden["streams"][name] = stream
    # baselines (engine.py:171-252): same trace, fixed residency / on-demand
    for sched in ("static_layer_split", "fixed_frequency_map", "gpu_ondemand"):
        rec, stream = record_run(tr, me.EnginePolicy(scheduling=sched, cache_policy="lru"), 0.5, hp, 2)
        golden["runs"].append({"name": f"tiny-{sched}", "config": TINY, "gen_seed": 2, "prefill": 64, "decode": 32,
                               "ratio": 0.5, "profile": prof_dict(hp), "policy": "lru", "prefetch": False, "seed": 2,
                               "scheduling": sched, "record": rec, "stream_sha": digest(stream),
                               "stream_len": len(stream)})
    for name, cfgd in SHAPES.items():
        cfg = mcore.ModelConfig(**cfgd)
        trs = mt.generate_trace(cfg, mt.GenParams(seed=0), 256, 16)
        hpb = b200_like_profile(cfg)
        ratios = (0.1, 0.25, 0.5) if name == "qwen2" else (0.25,)
        for ratio in ratios:
            for pf in (False, True):
                rec, stream = record_run(trs, me.EnginePolicy(prefetch=pf), ratio, hpb, 0)
                golden["runs"].append({"name": f"{name}-{ratio}-{'pf' if pf else 'nopf'}", "config": cfgd,
                                       "gen_seed": 0, "prefill": 256, "decode": 16, "ratio": ratio,
                                       "profile": prof_dict(hpb), "policy": "mrs", "prefetch": pf, "seed": 0,
                                       "record": rec, "stream_sha": digest(stream), "stream_len": len(stream)})
        print(name, "done", flush=True)
    # expected EvictionError on demand inserts
    for seed in (1, 2, 3, 4, 5):
        trs = mt.generate_trace(tiny, mt.GenParams(seed=seed), 1024, 8)
        try:
            rec, stream = record_run(trs, me.EnginePolicy(prefetch=True), 0.25, hp, seed)
            outcome = "ok"
        except mc.EvictionError:
            outcome, rec = "EvictionError", None
        golden["errors"].append({"gen_seed": seed, "prefill": 1024, "decode": 8, "ratio": 0.25, "seed": seed,
                                 "profile": prof_dict(hp), "outcome": outcome, "record": rec})
    golden["plans"] = random_plans()
    trt = mt.generate_trace(tiny, mt.GenParams(seed=5), 48, 6)
    for p, fwd in enumerate(trt.passes):
        for r in fwd.layers:
            golden["traces"].append({"pass": p, "stage": fwd.stage, "layer": r.layer, "loads": list(r.loads),
                                     "scores": [fx(v) for v in r.scores]})
    (HERE / "decisions.json").write_text(json.dumps(golden, separators=(",", ":")))
    print("wrote", HERE / "decisions.json", (HERE / "decisions.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
