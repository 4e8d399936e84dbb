"""Pin the CPU oracle (oracle/decisions.py) against the reference's golden fixtures."""
from __future__ import annotations

import pytest

from oracle import decisions as od
from stream import fx

import paper_2504_05897_b200.core as mcore
import paper_2504_05897_b200.tracegen as mt

KEYS = ("ttft", "mean_tbt", "lookups", "hits", "inserts", "evictions", "prefetch_issued", "prefetch_hits",
        "prefetch_expired", "elapsed", "gpu_util", "cpu_util", "pcie_util")


def _passes(entry):
    d = dict(entry["config"])
    d["routed_expert_dims"] = tuple(d["routed_expert_dims"])
    if d.get("shared_expert_dims"):
        d["shared_expert_dims"] = tuple(d["shared_expert_dims"])
    cfg = mcore.ModelConfig(**d)
    tr = mt.generate_trace(cfg, mt.GenParams(seed=entry["gen_seed"]), entry["prefill"], entry["decode"])
    return cfg, [(f.stage, [(r.layer, list(r.loads), list(r.scores)) for r in f.layers]) for f in tr.passes]


def test_oracle_random_plans(golden):
    for case in golden["plans"]:
        layer, loads = case["layer"], case["loads"]
        cached = [((layer, i), loads[i]) for i in sorted(case["cached"])]
        unc = [((layer, i), loads[i]) for i in range(len(loads)) if loads[i] > 0 and i not in case["cached"]]
        ev, asg, mk = od.best_plan(cached, unc, case["profile"], case["bytes"])
        assert fx(mk) == case["plan"][1]
        assert [[e[0], e[1][0], e[1][1], e[2], fx(e[3]), fx(e[4])] for e in ev] == case["plan"][2]
        assert sorted([[r[0], r[1], h] for r, h in asg.items()]) == case["plan"][3]
        assert fx(od.idle_budget((ev, asg, mk))) == case["budget"]


@pytest.mark.parametrize("name", ["tiny-mrs-nopf", "tiny-mrs-pf", "tiny-lru-nopf", "tiny-lru-pf", "tiny-lfu-nopf",
                                  "tiny-lfu-pf", "mixtral-0.25-pf", "deepseek-0.25-nopf", "qwen2-0.1-nopf"])
def test_oracle_runs(golden, name):
    entry = next(r for r in golden["runs"] if r["name"] == name)
    cfg, passes = _passes(entry)
    import math
    cap = math.floor(entry["ratio"] * cfg.num_layers * cfg.num_routed)
    pred = lambda pi, layer: od.predictions(passes[pi][1], pi, layer, entry["seed"])  # noqa: E731
    rec = od.run(passes, cfg.num_layers, cfg.num_routed, cfg.num_activated, mcore.expert_bytes(cfg),
                 entry["profile"], cap, entry["policy"], entry["prefetch"], predict=pred)
    for k in KEYS:
        assert rec[k] == entry["record"][k], (name, k)


def test_oracle_kats(golden):
    k = golden["kats"]
    p = dict(gpu_time_per_expert=1.0, cpu_slope=0.5, transfer_bandwidth=1.0, transfer_latency=0.0,
             gpu_saturation_load=256, gpu_slope=0.0, cpu_first_expert_penalty=1.4, shared_expert_time=0.0,
             non_expert_time=0.0)
    assert od.cpu_time(p, 2, 0) == k["cpu_time"][0] and od.cpu_time(p, 2, 3) == k["cpu_time"][1]
    assert od.top_p([0.25] * 4, 2) == k["top_p_ties"]
    c = od.Cache(2, "mrs", 1, 3, 0.5, 2)
    c.S.update({(0, 0): 0.4, (0, 1): 0.2, (0, 2): 0.0})
    c.mrs_update(0, [0.6, 0.3, 0.1])
    assert [c.S[(0, i)] for i in range(3)] == k["mrs_update"]
