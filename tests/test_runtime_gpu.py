"""End-to-end HybriMoE layer stack on the GPU: router parity against the
reference's traces, decision parity against the decision core replayed on the
same LayerRequests, numerics against the fp32 oracle, GPU MRS table bit-exact."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_ref as ref
from stream import digest, from_records

import paper_2504_05897_b200.core as mcore
import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.engine as me
from paper_2504_05897_b200.moe import SHAPES, HybridMoE, shared_chunks
from paper_2504_05897_b200.prefetch import predict_layers
from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits
from paper_2504_05897_b200.weights import unpack_expert

pytestmark = pytest.mark.gpu


def stress_profile(cfg):
    eb = mcore.expert_bytes(cfg)
    return mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)


def family_cfg(family: str):
    """The tiny stack, or a 3-layer stack of 64 routed experts with the family's
    shared experts (DeepSeek: 2 chunk-sized, top-6; Qwen2: 1 four-chunk, top-8)."""
    if family == "tiny":
        return SHAPES["tiny"]
    n_shared, k = (2, 6) if family == "deepseek" else (1, 8)
    return mcore.ModelConfig(num_layers=3, num_routed=64, num_shared=n_shared, num_activated=k,
                             routed_expert_dims=(256, 256),
                             shared_expert_dims=(256, 256 if family == "deepseek" else 4 * 256), bytes_per_weight=2)


def bf(t: torch.Tensor) -> np.ndarray:
    return ref.bf16_to_f32(t.view(torch.int16).cpu().numpy().view(np.uint16))


def _experts(moe, layer):
    ex = []
    for e in range(moe.N):
        g, u, d = unpack_expert(moe.expert_image(layer, e), moe.H, moe.I)
        ex.append((ref.bf16_to_f32(g), ref.bf16_to_f32(u), ref.bf16_to_f32(d)))
    for c in range(moe.S):
        g, u, d = unpack_expert(moe.shared_image(layer, c), moe.H, moe.I)
        ex.append((ref.bf16_to_f32(g), ref.bf16_to_f32(u), ref.bf16_to_f32(d)))
    return ex


@pytest.mark.parametrize("policy_name,prefetch,ratio", [("mrs", True, 0.5), ("lru", False, 0.25), ("lfu", True, 0.75)])
def test_tiny_stack_parity(policy_name, prefetch, ratio):
    cfg = SHAPES["tiny"]
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(cache_policy=policy_name, prefetch=prefetch)
    moe = HybridMoE(cfg, "tiny", policy, ratio, prof, max_tokens=64, residual=False)
    moe.init_random_weights(3)
    trace, logits = generate_router_logits(cfg, GenParams(seed=2), 48, 6)
    g = torch.Generator(device="cuda").manual_seed(0)
    recs, reqs = [], []
    for p, fwd in enumerate(trace.passes):
        lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
        x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
        y, info = moe.forward_pass(x, lg, predict=lambda l, p=p, fwd=fwd: predict_layers(
            fwd.layers, cfg.num_layers, p, l, policy.prediction, 2), decision_log=True, keep_layers=True)
        torch.cuda.synchronize()
        for l, (loads, scores) in enumerate(info["requests"]):
            assert list(loads) == list(fwd.layers[l].loads), (p, l)      # router == reference trace
            reqs.append((l, loads, scores))
        recs.extend(info["records"])
        if p in (0, len(trace.passes) - 1):
            for l, (xi, lgi, yo) in enumerate(info["layers"]):
                want = ref.moe_layer(bf(xi), lgi.cpu().numpy(), _experts(moe, l), moe.N, moe.K, True, 0, -1)
                err = np.abs(bf(yo) - want).max() / np.abs(want).max()
                assert err <= 1e-2, (p, l, err)
    # the decision core replayed on the runtime's own LayerRequests gives the same decision stream
    passes, i = [], 0
    for fwd in trace.passes:
        layers = []
        for l in range(cfg.num_layers):
            _, loads, scores = reqs[i]
            i += 1
            layers.append(mcore.make_layer_request(l, loads.tolist(), scores.tolist()))
        passes.append(mcore.ForwardPass(fwd.stage, fwd.token_count, tuple(layers)))
    replay = mcore.Trace(cfg, tuple(passes))
    m = me.run_trace(replay, policy, ratio, prof, 2, decision_log=True)
    mrs = policy_name == "mrs"
    assert digest(from_records(recs, mrs)) == digest(from_records(m.decisions, mrs))
    if mrs:
        assert np.array_equal(moe.device_mrs().view(np.uint64), moe.mrs.table().view(np.uint64))


@pytest.mark.parametrize("shape", ["deepseek", "qwen2"])
def test_shared_expert_families_one_layer(shape):
    base = SHAPES[shape]
    # two layers of the family's routing/shared structure at a reduced hidden size
    H = 256
    I = base.routed_expert_dims[1] if base.routed_expert_dims[1] <= 2560 else 256
    I = 256 if shape == "qwen2" else 384
    shared = (H, I * (8 if shape == "qwen2" else 1))
    cfg = mcore.ModelConfig(num_layers=2, num_routed=16, num_shared=base.num_shared, num_activated=base.num_activated,
                            routed_expert_dims=(H, I), shared_expert_dims=shared, bytes_per_weight=2)
    prof = stress_profile(cfg)
    moe = HybridMoE(cfg, shape, me.EnginePolicy(), 0.5, prof, max_tokens=128, residual=False)
    moe.init_random_weights(1)
    rng = np.random.default_rng(0)
    T = 96
    lg = [torch.from_numpy(rng.standard_normal((T, moe.ld)).astype(np.float32)).cuda() for _ in range(2)]
    x = torch.randn((T, H), device="cuda").to(torch.bfloat16)
    y, info = moe.forward_pass(x, lg, keep_layers=True)
    torch.cuda.synchronize()
    fam = moe.family
    for l, (xi, lgi, yo) in enumerate(info["layers"]):
        want = ref.moe_layer(bf(xi), lgi.cpu().numpy(), _experts(moe, l), moe.N, moe.K, fam.renormalize,
                             shared_chunks(cfg), moe.gate_col)
        err = np.abs(bf(yo) - want).max() / np.abs(want).max()
        assert err <= 1e-2, (l, err)


def test_live_lookahead_prefetch_model_mode():
    """Model mode with the paper's live predictor (future gates on the current
    hidden state): predictions equal the routing those gates produce, and the
    decisions replay exactly through the decision core with those predictions."""
    cfg = SHAPES["tiny"]
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    moe = HybridMoE(cfg, "tiny", policy, 0.5, prof, max_tokens=32)
    moe.init_random_weights(11)
    x = torch.randn((1, moe.H), device="cuda").to(torch.bfloat16)
    preds = moe.lookahead(x, 0)
    assert [p.layer for p in preds] == [1, 2, 3]
    from paper_2504_05897_b200.kernels import router_logits, router_topk
    for p in preds:
        _, _, _, c = router_topk(router_logits(x, moe.gate_w[p.layer]), moe.N, moe.K, True)
        assert list(p.loads) == c.cpu().tolist() and sum(p.loads) == moe.K
    for _ in range(4):
        y, info = moe.forward_pass(x, None, predict="live", decision_log=True)
        x = y.clone()
    torch.cuda.synchronize()
    assert torch.isfinite(x.float()).all()


@pytest.mark.parametrize("zero_copy,family", [("1", "tiny"), ("0", "tiny"), ("1", "deepseek"), ("1", "qwen2")])
def test_native_live_lookahead_matches_python_lookahead(monkeypatch, zero_copy, family):
    """The runtime's live predictor (one look-ahead kernel ahead of the router,
    loads published with the LayerRequest) makes the same decisions as the
    Python look-ahead (router_logits + router_topk per future layer): model
    mode per layer, and the one-call native pass in trace mode."""
    monkeypatch.setenv("HM_ZERO_COPY", zero_copy)
    cfg = family_cfg(family)
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    trace, logits = generate_router_logits(cfg, GenParams(seed=8), 24, 4)
    runs = {}
    for mode in ("live_py", "live", "live_native_pass"):
        moe = HybridMoE(cfg, family, policy, 0.5, prof, max_tokens=64)
        moe.init_seeded_weights(6)
        g = torch.Generator(device="cuda").manual_seed(2)
        recs, ys, res = [], [], []
        for p, fwd in enumerate(trace.passes):  # model mode: logits from each layer's live input
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            y, info = moe.forward_pass(x, None, predict=mode.replace("_native_pass", ""), decision_log=True)
            recs.extend(info["records"])
            ys.append(y.float().cpu().numpy())
            r = info["pass"]
            res.append((r.latency, r.lookups, r.hits, r.inserts, r.evictions, r.prefetch_issued))
        g = torch.Generator(device="cuda").manual_seed(3)
        for p, fwd in enumerate(trace.passes):  # trace mode, per layer vs one native call
            lg = [torch.from_numpy(np.ascontiguousarray(np.pad(logits[p][l], ((0, 0), (0, moe.ld - moe.N))),
                                                        dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            pred = "live" if mode == "live_native_pass" else mode
            y, info = moe.forward_pass(x, lg, predict=pred, decision_log=mode != "live_native_pass")
            torch.cuda.synchronize()
            ys.append(y.float().cpu().numpy())
            r = info["pass"]
            res.append((r.latency, r.lookups, r.hits, r.inserts, r.evictions, r.prefetch_issued))
        runs[mode] = (digest(from_records(recs, True)), ys, res)
    assert runs["live_py"][0] == runs["live"][0] == runs["live_native_pass"][0]
    assert runs["live_py"][2] == runs["live"][2]
    assert runs["live_py"][2] == runs["live_native_pass"][2]
    assert sum(r[-1] for r in runs["live"][2]) > 0  # the predictions drove prefetches
    for a, b in zip(runs["live_py"][1], runs["live"][1]):
        assert np.array_equal(a, b)
    for a, b in zip(runs["live_py"][1], runs["live_native_pass"][1]):
        assert np.array_equal(a, b)


def test_native_trace_predictor_matches_python_predictor():
    """forward_pass with the native prediction model makes the same decisions
    as with the Python (numpy) prediction model."""
    from paper_2504_05897_b200.moe import TracePredictor
    cfg = SHAPES["tiny"]
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    trace, logits = generate_router_logits(cfg, GenParams(seed=4), 32, 4)
    streams = []
    for native in (False, True):
        moe = HybridMoE(cfg, "tiny", policy, 0.5, prof, max_tokens=64)
        moe.init_seeded_weights(2)
        recs = []
        g = torch.Generator(device="cuda").manual_seed(1)
        for p, fwd in enumerate(trace.passes):
            lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda()
                  for l in range(cfg.num_layers)]
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            pred = (TracePredictor(trace, p, 9) if native else
                    (lambda l, p=p, fwd=fwd: predict_layers(fwd.layers, cfg.num_layers, p, l, policy.prediction, 9)))
            _, info = moe.forward_pass(x, lg, predict=pred, decision_log=True)
            recs.extend(info["records"])
        streams.append(digest(from_records(recs, True)))
    assert streams[0] == streams[1]


def test_native_pass_equals_per_layer_pass():
    """hm_runtime_forward_pass (one call per pass) == the Python per-layer loop:
    same outputs and the same PassResult (decisions)."""
    from paper_2504_05897_b200.moe import TracePredictor
    cfg = SHAPES["tiny"]
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    trace, logits = generate_router_logits(cfg, GenParams(seed=6), 32, 4)
    outs = []
    for native in (False, True):
        moe = HybridMoE(cfg, "tiny", policy, 0.5, prof, max_tokens=64)
        moe.init_seeded_weights(4)
        g = torch.Generator(device="cuda").manual_seed(3)
        ys, results = [], []
        for p, fwd in enumerate(trace.passes):
            lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda()
                  for l in range(cfg.num_layers)]
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            y, info = moe.forward_pass(x, lg, predict=TracePredictor(trace, p, 5), decision_log=not native)
            torch.cuda.synchronize()
            ys.append(y.float().cpu().numpy())
            r = info["pass"]
            results.append((r.latency, r.lookups, r.hits, r.inserts, r.evictions, r.prefetch_issued))
        outs.append((ys, results))
    assert outs[0][1] == outs[1][1]
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)


def test_model_mode_runs_and_is_deterministic():
    cfg = SHAPES["tiny"]
    moe = HybridMoE(cfg, "tiny", me.EnginePolicy(), 0.25, stress_profile(cfg), max_tokens=32)
    moe.init_random_weights(5)
    x = torch.randn((16, moe.H), device="cuda").to(torch.bfloat16)
    y1, _ = moe.forward_pass(x, None)
    y1 = y1.clone()
    torch.cuda.synchronize()
    assert torch.isfinite(y1.float()).all()


@pytest.mark.parametrize("family", ["tiny", "deepseek", "qwen2"])
def test_zero_copy_path_equals_copy_path(monkeypatch, family):
    """The zero-copy decode path (router mirrors the LayerRequest and the routed
    rows into mapped host memory, host spins on a flag; the combine reads the
    host worker's rows over PCIe and folds the MRS update into the same launch)
    gives bit-identical outputs, decisions and MRS table to the copy path --
    also with 64 routed experts and shared experts (DeepSeek / Qwen2 families)."""
    from paper_2504_05897_b200.moe import TracePredictor
    cfg = family_cfg(family)
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    trace, logits = generate_router_logits(cfg, GenParams(seed=8), 24, 6)
    outs = []
    for zc in ("0", "1"):
        monkeypatch.setenv("HM_ZERO_COPY", zc)
        moe = HybridMoE(cfg, family, policy, 0.5, prof, max_tokens=64)
        moe.init_seeded_weights(6)
        g = torch.Generator(device="cuda").manual_seed(5)
        ys, recs, ncpu = [], [], 0
        for p, fwd in enumerate(trace.passes):
            lg = [torch.from_numpy(np.ascontiguousarray(np.pad(logits[p][l], ((0, 0), (0, moe.ld - moe.N))),
                                                        dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            y, info = moe.forward_pass(x, lg, predict=TracePredictor(trace, p, 5), decision_log=True)
            torch.cuda.synchronize()
            ys.append(y.float().cpu().numpy())
            recs.extend(info["records"])
            ncpu += sum(s.n_cpu for s in info["stats"])
        outs.append((ys, digest(from_records(recs, True)), moe.device_mrs(), ncpu))
    assert outs[0][3] > 0  # the host worker ran experts (zero-copy rows exercised)
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][2].view(np.uint64), outs[1][2].view(np.uint64))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)


def test_q4_stack_parity():
    """4-bit experts end to end (the paper's setting, bytes_per_weight 0.5):
    GPU GEMV/GEMM and host worker on 4-bit images match the fp32 oracle on the
    dequantized weights, and the decisions replay exactly through the decision
    core (expert_bytes at 0.5 bytes per weight)."""
    from dataclasses import replace
    cfg = replace(SHAPES["tiny"], bytes_per_weight=0.5)
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    moe = HybridMoE(cfg, "tiny", policy, 0.5, prof, max_tokens=64, residual=False, weight_bits=4)
    moe.init_random_weights(3)
    trace, logits = generate_router_logits(cfg, GenParams(seed=2), 48, 4)
    g = torch.Generator(device="cuda").manual_seed(0)
    recs, reqs, n_cpu, n_gpu = [], [], 0, 0
    for p, fwd in enumerate(trace.passes):
        lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
        x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
        y, info = moe.forward_pass(x, lg, predict=lambda l, p=p, fwd=fwd: predict_layers(
            fwd.layers, cfg.num_layers, p, l, policy.prediction, 2), decision_log=True, keep_layers=True)
        torch.cuda.synchronize()
        n_cpu += sum(s.n_cpu for s in info["stats"])
        n_gpu += sum(s.n_gpu for s in info["stats"])
        for l, (loads, scores) in enumerate(info["requests"]):
            reqs.append((l, loads, scores))
        recs.extend(info["records"])
        for l, (xi, lgi, yo) in enumerate(info["layers"]):
            ex = [ref.q4_expert(moe.expert_image(l, e), moe.H, moe.I) for e in range(moe.N)]
            want = ref.moe_layer(bf(xi), lgi.cpu().numpy(), ex, moe.N, moe.K, True, 0, -1)
            err = np.abs(bf(yo) - want).max() / np.abs(want).max()
            assert err <= 1e-2, (p, l, err)
    assert n_cpu > 0 and n_gpu > 0
    passes, i = [], 0
    for fwd in trace.passes:
        layers = []
        for l in range(cfg.num_layers):
            _, loads, scores = reqs[i]
            i += 1
            layers.append(mcore.make_layer_request(l, loads.tolist(), scores.tolist()))
        passes.append(mcore.ForwardPass(fwd.stage, fwd.token_count, tuple(layers)))
    m = me.run_trace(mcore.Trace(cfg, tuple(passes)), policy, 0.5, prof, 2, decision_log=True)
    assert digest(from_records(recs, True)) == digest(from_records(m.decisions, True))


@pytest.mark.parametrize("family", ["tiny", "deepseek"])
def test_gpu_mrs_rows_drive_decisions_bit_identically(family):
    """Score updates on the GPU (zero-copy decode path): the router computes each
    layer's new MRS row from the decision core's mapped table and the decision
    core consumes it at step (5).  Against the host recurrence (gpu_mrs=False):
    identical decision streams, MRS tables and outputs over prefill + decode
    passes -- and both equal the reference's decisions replayed on the same
    LayerRequests."""
    from paper_2504_05897_b200.moe import TracePredictor
    cfg = family_cfg(family)
    prof = stress_profile(cfg)
    policy = me.EnginePolicy(prefetch=True)
    trace, logits = generate_router_logits(cfg, GenParams(seed=12), 24, 8)
    outs = []
    for gpu_mrs in (False, True):
        moe = HybridMoE(cfg, family, policy, 0.5, prof, max_tokens=64, gpu_mrs=gpu_mrs)
        moe.init_seeded_weights(4)
        g = torch.Generator(device="cuda").manual_seed(3)
        ys, recs, reqs = [], [], []
        for p, fwd in enumerate(trace.passes):
            lg = [torch.from_numpy(np.ascontiguousarray(np.pad(logits[p][l], ((0, 0), (0, moe.ld - moe.N))),
                                                        dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
            x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            y, info = moe.forward_pass(x, lg, predict=TracePredictor(trace, p, 5), decision_log=True)
            torch.cuda.synchronize()
            ys.append(y.float().cpu().numpy())
            recs.extend(info["records"])
            reqs.append([(lo.tolist(), sc.tolist()) for lo, sc in info["requests"]])
        outs.append((ys, digest(from_records(recs, True)), moe.mrs.table().copy(), reqs))
        del moe
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][2].view(np.uint64), outs[1][2].view(np.uint64))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)
    # the decision core alone on the runtime's LayerRequests (host recurrence throughout)
    passes = [mcore.ForwardPass(f.stage, f.token_count, tuple(mcore.make_layer_request(l, lo, sc)
                                                             for l, (lo, sc) in enumerate(outs[1][3][p])))
              for p, f in enumerate(trace.passes)]
    replay = mcore.Trace(cfg, tuple(passes))
    m = me.run_trace(replay, policy, 0.5, prof, 5, decision_log=True)
    assert digest(from_records(m.decisions, True)) == outs[1][1]
