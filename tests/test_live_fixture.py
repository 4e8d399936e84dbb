"""Decision parity on a LIVE B200 run (tests/golden/live_runs.json, made by
tools/live_fixture.py on the GPU box): the runtime's routing came from its own
GPU router in model mode (logits = x . W_g per layer), its LayerRequests were
written in the reference's trace format, and the runtime's decision stream was
hashed.  Replaying that trace through the UNMODIFIED reference run_trace (build
container) and through the native decision core must give the same stream."""
from __future__ import annotations

import json
from pathlib import Path

import pytest

from stream import digest, from_records

import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.engine as me
from paper_2504_05897_b200.tracegen import load_trace

LIVE = json.loads((Path(__file__).resolve().parent / "golden" / "live_runs.json").read_text())


@pytest.mark.parametrize("policy", sorted(LIVE))
def test_live_run_replays_through_decision_core(policy, tmp_path):
    case = LIVE[policy]
    p = tmp_path / "live.jsonl"
    p.write_text(case["trace_jsonl"])
    trace = load_trace(p)
    assert trace.metadata.get("source", "").startswith("live B200 run")
    assert trace.config.num_routed in (8, 64)
    m = me.run_trace(trace, me.EnginePolicy(cache_policy=case["policy"], prefetch=case["prefetch"]), case["ratio"],
                     mcost.HardwareProfile(**case["profile"]), case["seed"], decision_log=True)
    assert digest(from_records(m.decisions, case["policy"] == "mrs")) == case["runtime_stream_sha256"]


@pytest.mark.reference
@pytest.mark.parametrize("policy", sorted(LIVE))
def test_live_run_replays_through_reference(policy, moesim, tmp_path):
    import make_golden as mg          # the Recorder wraps the reference's own engine-level names
    import moesim.costs as rcost
    import moesim.engine as reng
    import moesim.tracegen as rtrace

    case = LIVE[policy]
    p = tmp_path / "live.jsonl"
    p.write_text(case["trace_jsonl"])
    trace = rtrace.load_trace(str(p))
    with mg.Recorder() as rec:
        reng.run_trace(trace, reng.EnginePolicy(cache_policy=case["policy"], prefetch=case["prefetch"]), case["ratio"],
                       rcost.HardwareProfile(**case["profile"]), case["seed"])
    assert digest(rec.stream) == case["runtime_stream_sha256"]


LIVE_EP = json.loads((Path(__file__).resolve().parent / "golden" / "live_ep.json").read_text())


@pytest.mark.parametrize("rank", sorted(LIVE_EP))
def test_live_ep_rank_replays_through_decision_core(rank, tmp_path):
    """Per-rank parity on a live two-rank run: the rank's own
    masked LayerRequests at its share of the global budget."""
    case = LIVE_EP[rank]
    p = tmp_path / "live.jsonl"
    p.write_text(case["trace_jsonl"])
    trace = load_trace(p)
    m = me.run_trace(trace, me.EnginePolicy(cache_policy=case["policy"], prefetch=case["prefetch"]), case["ratio"],
                     mcost.HardwareProfile(**case["profile"]), case["seed"], decision_log=True)
    assert digest(from_records(m.decisions, True)) == case["runtime_stream_sha256"]


@pytest.mark.reference
@pytest.mark.parametrize("rank", sorted(LIVE_EP))
def test_live_ep_rank_replays_through_reference(rank, moesim, tmp_path):
    import make_golden as mg
    import moesim.costs as rcost
    import moesim.engine as reng
    import moesim.tracegen as rtrace

    case = LIVE_EP[rank]
    p = tmp_path / "live.jsonl"
    p.write_text(case["trace_jsonl"])
    trace = rtrace.load_trace(str(p))
    assert reng.cache_capacity(trace.config, case["ratio"]) == case["capacity"]
    with mg.Recorder() as rec:
        reng.run_trace(trace, reng.EnginePolicy(cache_policy=case["policy"], prefetch=case["prefetch"]), case["ratio"],
                       rcost.HardwareProfile(**case["profile"]), case["seed"])
    assert digest(rec.stream) == case["runtime_stream_sha256"]
