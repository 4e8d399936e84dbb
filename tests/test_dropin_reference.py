"""Drop-in test: the UNMODIFIED reference run_trace, with
its engine-level names patched to this package's native implementations, must
give identical RunMetrics and an identical decision stream.  Build container only."""
from __future__ import annotations

import sys

import pytest

from stream import digest

import paper_2504_05897_b200.caching as nc
import paper_2504_05897_b200.core as ncore
import paper_2504_05897_b200.prefetch as npf
import paper_2504_05897_b200.scheduling as ns

pytestmark = pytest.mark.reference

PATCH = {
    "CacheState": ncore.CacheState, "make_mrs_state": nc.make_mrs_state, "lookup": nc.lookup,
    "insert_with_eviction": nc.insert_with_eviction, "mrs_update": nc.mrs_update, "select_plan": ns.select_plan,
    "plan_all_gpu": ns.plan_all_gpu, "plan_all_cpu": ns.plan_all_cpu, "pcie_idle_budget": ns.pcie_idle_budget,
    "MakespanEvaluator": ns.MakespanEvaluator, "evaluate_gain": npf.evaluate_gain,
    "select_prefetches": npf.select_prefetches, "EvictionError": nc.EvictionError,
}


@pytest.mark.parametrize("name", ["tiny-mrs-pf", "tiny-lru-pf", "tiny-lfu-nopf", "tiny-gpu_ondemand",
                                  "deepseek-0.25-pf", "qwen2-0.25-nopf"])
def test_patched_reference_run_trace(golden, moesim, name):
    import moesim.core as rc
    import moesim.costs as rco
    import moesim.engine as re_
    import moesim.tracegen as rt
    sys.path.insert(0, __import__("os").path.dirname(__file__) + "/golden")
    from make_golden import Recorder

    entry = next(r for r in golden["runs"] if r["name"] == name)
    d = dict(entry["config"])
    d["routed_expert_dims"] = tuple(d["routed_expert_dims"])
    if d.get("shared_expert_dims"):
        d["shared_expert_dims"] = tuple(d["shared_expert_dims"])
    tr = rt.generate_trace(rc.ModelConfig(**d), rt.GenParams(seed=entry["gen_seed"]), entry["prefill"], entry["decode"])
    pol = re_.EnginePolicy(scheduling=entry.get("scheduling", "hybrid"), cache_policy=entry["policy"],
                           prefetch=entry["prefetch"])
    saved = {k: getattr(re_, k) for k in PATCH}
    try:
        for k, v in PATCH.items():
            setattr(re_, k, v)
        with Recorder() as rec:
            m = re_.run_trace(tr, pol, entry["ratio"], rco.HardwareProfile(**entry["profile"]), entry["seed"])
    finally:
        for k, v in saved.items():
            setattr(re_, k, v)
    assert m.to_record() == entry["record"]
    assert digest(rec.stream) == entry["stream_sha"]
