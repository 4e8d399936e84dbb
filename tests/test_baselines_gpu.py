"""The comparison schedulings executed for real by the runtime, and runtime edge cases.

* static_layer_split (llama.cpp-like), fixed_frequency_map (kTransformers-like)
  and gpu_ondemand (AdapMoE-like) (reference engine.py:171-252) on the tiny
  stack of the golden fixtures: the GPU router's LayerRequests, the decision
  stream the runtime executed (every lookup, plan, insert) hashes to the
  stream the UNMODIFIED reference produced for the same trace
  (tests/golden/decisions.json, runs "tiny-<scheduling>", make_golden.py), and
  the layer outputs match the fp32 oracle (1e-2).
* a budget that floors the cache to 0 slots: the plan's transferred experts
  are still copied and computed (through the staging slot), so the outputs
  match the oracle and the decisions match the decision core's replay.
* switching compute streams between passes is ordered after the previous
  stream's combine / MRS work (same outputs as one stream).
* static_layer_split needs no explicit preload (HybridMoE keeps the layers
  below the split resident itself).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_ref as ref
from stream import digest, from_records
from test_runtime_gpu import _experts, bf

import paper_2504_05897_b200.core as mcore
import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.engine as me
from paper_2504_05897_b200.moe import HybridMoE
from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits

pytestmark = pytest.mark.gpu


def _gold_run(golden, name):
    return next(r for r in golden["runs"] if r["name"] == name)


def _run_stack(moe, cfg, trace, logits, check_layers=(0, -1), stream=None):
    recs, reqs, n_xfer, n_gpu, n_cpu = [], [], 0, 0, 0
    g = torch.Generator(device="cuda").manual_seed(0)
    outs = []
    for p, fwd in enumerate(trace.passes):
        lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda()
              for l in range(cfg.num_layers)]
        x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
        st = stream(p) if stream else None
        y, info = moe.forward_pass(x, lg, decision_log=True, keep_layers=True, stream=st)
        torch.cuda.synchronize()
        outs.append(y.float().cpu().numpy())
        for l, (loads, scores) in enumerate(info["requests"]):
            assert list(loads) == list(fwd.layers[l].loads), (p, l)
            reqs.append((l, loads, scores))
        recs.extend(info["records"])
        n_xfer += sum(s.n_transfer for s in info["stats"])
        n_gpu += sum(s.n_gpu for s in info["stats"])
        n_cpu += sum(s.n_cpu for s in info["stats"])
        if p in [c % len(trace.passes) for c in check_layers]:
            for l, (xi, lgi, yo) in enumerate(info["layers"]):
                want = ref.moe_layer(bf(xi), lgi.cpu().numpy(), _experts(moe, l), moe.N, moe.K, True, 0, -1)
                err = np.abs(bf(yo) - want).max() / np.abs(want).max()
                assert err <= 1e-2, (p, l, err)
    return recs, reqs, outs, (n_gpu, n_cpu, n_xfer)


@pytest.mark.parametrize("sched", ["static_layer_split", "fixed_frequency_map", "gpu_ondemand"])
def test_baseline_scheduling_executed_matches_reference(golden, sched):
    entry = _gold_run(golden, f"tiny-{sched}")
    cfg = mcore.ModelConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in entry["config"].items()})
    prof = mcost.HardwareProfile(**entry["profile"])
    policy = me.EnginePolicy(scheduling=sched, cache_policy=entry["policy"])
    trace, logits = generate_router_logits(cfg, GenParams(seed=entry["gen_seed"]), entry["prefill"], entry["decode"])
    moe = HybridMoE(cfg, "tiny", policy, entry["ratio"], prof, max_tokens=entry["prefill"], residual=False)
    moe.init_random_weights(5)
    if sched == "fixed_frequency_map":
        fixed = me.compute_fixed_pinned_set(trace, moe.capacity, policy.calibration_prefix_fraction, None)
        moe.set_fixed_gpu_set(sorted(fixed))
    recs, _, _, (n_gpu, n_cpu, n_xfer) = _run_stack(moe, cfg, trace, logits)
    stream = from_records(recs, False)
    assert len(stream) == entry["stream_len"]
    assert digest(stream) == entry["stream_sha"]
    if sched == "gpu_ondemand":
        assert n_cpu == 0 and n_xfer > 0
    else:
        assert n_xfer == 0 and n_gpu > 0 and n_cpu > 0


@pytest.mark.parametrize("sched", ["hybrid", "gpu_ondemand"])
def test_zero_capacity_budget_still_computes_transfers(sched):
    cfg = mcore.ModelConfig(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(256, 256),
                            bytes_per_weight=2)
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)
    policy = me.EnginePolicy(scheduling=sched)
    moe = HybridMoE(cfg, "tiny", policy, 0.02, prof, max_tokens=32, residual=False)
    assert moe.capacity == 0
    moe.init_random_weights(2)
    trace, logits = generate_router_logits(cfg, GenParams(seed=3), 32, 4)
    recs, reqs, _, (n_gpu, n_cpu, n_xfer) = _run_stack(moe, cfg, trace, logits, check_layers=range(5))
    assert n_xfer > 0 and 0 < n_gpu <= n_xfer  # every GPU expert arrived by a transfer, none was kept
    passes, i = [], 0
    for fwd in trace.passes:
        layers = []
        for l in range(cfg.num_layers):
            _, loads, scores = reqs[i]
            i += 1
            layers.append(mcore.make_layer_request(l, loads.tolist(), scores.tolist()))
        passes.append(mcore.ForwardPass(fwd.stage, fwd.token_count, tuple(layers)))
    m = me.run_trace(mcore.Trace(cfg, tuple(passes)), policy, 0.02, prof, 2, decision_log=True)
    assert digest(from_records(recs, True)) == digest(from_records(m.decisions, True))


def test_stream_switch_between_passes_is_ordered():
    cfg = mcore.ModelConfig(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(256, 256),
                            bytes_per_weight=2)
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5)
    trace, logits = generate_router_logits(cfg, GenParams(seed=5), 32, 6)
    results = []
    for switching in (False, True):
        moe = HybridMoE(cfg, "tiny", me.EnginePolicy(prefetch=True), 0.5, prof, max_tokens=32, residual=False)
        moe.init_seeded_weights(1)
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        pick = (lambda p: streams[p % 2]) if switching else None
        _, _, outs, _ = _run_stack(moe, cfg, trace, logits, check_layers=(), stream=pick)
        results.append(outs)
    for a, b in zip(*results):
        assert np.array_equal(a, b)


def test_static_layer_split_needs_no_explicit_preload():
    cfg = mcore.ModelConfig(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(256, 256),
                            bytes_per_weight=2)
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5)
    moe = HybridMoE(cfg, "tiny", me.EnginePolicy(scheduling="static_layer_split"), 0.5, prof, max_tokens=32,
                    residual=False)
    moe.init_random_weights(4)
    trace, logits = generate_router_logits(cfg, GenParams(seed=1), 16, 2)
    _, _, _, (n_gpu, n_cpu, _) = _run_stack(moe, cfg, trace, logits, check_layers=(0, 1, 2))
    assert n_gpu > 0 and n_cpu > 0
