"""Live-run decision fixture (run on the GPU box; commits tests/golden/live_*.json).

A tiny HybriMoE stack runs in MODEL MODE on the B200: every layer's router
logits are x . W_g computed on the GPU from that layer's live input, so the
LayerRequests come from this implementation's kernels, not from the
reference's trace generator.  The runtime's per-layer LayerRequests are
written in the reference's trace format (tracegen.save_trace, byte-identical
to the reference writer) together with the SHA-256 of the runtime's decision
stream.  tests/test_live_fixture.py replays the trace through the UNMODIFIED
reference run_trace (build container) and through the native decision core,
and requires the same stream: decision parity on a live B200 run.

    python tools/live_fixture.py
"""
from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

import paper_2504_05897_b200.core as mcore  # noqa: E402
import paper_2504_05897_b200.costs as mcost  # noqa: E402
import paper_2504_05897_b200.engine as me  # noqa: E402
from paper_2504_05897_b200.moe import SHAPES, HybridMoE  # noqa: E402
from paper_2504_05897_b200.tracegen import save_trace  # noqa: E402
from stream import digest, from_records  # noqa: E402


def run(policy_name: str, seed: int) -> dict:
    cfg = SHAPES["tiny"]
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)
    policy = me.EnginePolicy(cache_policy=policy_name, prefetch=False)
    ratio = 0.5
    moe = HybridMoE(cfg, "tiny", policy, ratio, prof, max_tokens=64)
    moe.init_random_weights(seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    passes, recs = [], []
    stages = [("prefill", 48)] + [("decode", 1)] * 12
    for stage, T in stages:
        x = torch.randn((T, moe.H), generator=g, device="cuda").to(torch.bfloat16)
        _, info = moe.forward_pass(x, None, decision_log=True)  # model mode: logits = x . W_g per layer
        torch.cuda.synchronize()
        recs.extend(info["records"])
        layers = tuple(mcore.make_layer_request(l, loads.tolist(), scores.tolist())
                       for l, (loads, scores) in enumerate(info["requests"]))
        passes.append(mcore.ForwardPass(stage, T, layers))
    trace = mcore.Trace(cfg, tuple(passes), {"source": "live B200 run, model-mode routing"})
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "t.jsonl"
        save_trace(trace, p)
        text = p.read_text()
    return {"policy": policy_name, "prefetch": False, "ratio": ratio, "seed": 2,
            "profile": {k: getattr(prof, k) for k in prof.__dataclass_fields__},
            "trace_jsonl": text, "runtime_stream_sha256": digest(from_records(recs, policy_name == "mrs")),
            "gpu": torch.cuda.get_device_name(0)}


def run_prefetch(seed: int) -> dict:
    """Impact-driven prefetch on live routing: phase 1 runs the stack in model
    mode and keeps every layer's GPU-computed logits; phase 2 (a fresh stack,
    same weights) runs trace mode on exactly those logits with prefetch on and
    the reference's prediction model fed with the phase-1 loads, so its
    decisions must equal the reference replaying the recorded trace."""
    from paper_2504_05897_b200.moe import TracePredictor
    cfg = SHAPES["tiny"]
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                 cpu_first_expert_penalty=1.4)
    stages = [("prefill", 48)] + [("decode", 1)] * 12
    g = torch.Generator(device="cuda").manual_seed(seed)
    xs = [torch.randn((T, cfg.routed_expert_dims[0]), generator=g, device="cuda").to(torch.bfloat16)
          for _, T in stages]
    moe = HybridMoE(cfg, "tiny", me.EnginePolicy(), 0.5, prof, max_tokens=64)
    moe.init_seeded_weights(seed)
    passes, logits = [], []
    for (stage, T), x in zip(stages, xs):
        _, info = moe.forward_pass(x, None, decision_log=True, keep_layers=True)
        torch.cuda.synchronize()
        logits.append([lg.clone() for _, lg, _ in info["layers"]])
        passes.append(mcore.ForwardPass(stage, T, tuple(mcore.make_layer_request(l, lo.tolist(), sc.tolist())
                                                         for l, (lo, sc) in enumerate(info["requests"]))))
    trace = mcore.Trace(cfg, tuple(passes), {"source": "live B200 run, model-mode routing"})
    del moe
    policy = me.EnginePolicy(cache_policy="mrs", prefetch=True)
    moe2 = HybridMoE(cfg, "tiny", policy, 0.5, prof, max_tokens=64)
    moe2.init_seeded_weights(seed)
    recs, pseed = [], 2
    for p, x in enumerate(xs):
        _, info = moe2.forward_pass(x, logits[p], predict=TracePredictor(trace, p, pseed), decision_log=True)
        torch.cuda.synchronize()
        recs.extend(info["records"])
        assert [list(lo) for lo, _ in info["requests"]] == [list(r.loads) for r in trace.passes[p].layers]
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "t.jsonl"
        save_trace(trace, f)
        text = f.read_text()
    return {"policy": "mrs", "prefetch": True, "ratio": 0.5, "seed": pseed,
            "profile": {k: getattr(prof, k) for k in prof.__dataclass_fields__},
            "trace_jsonl": text, "runtime_stream_sha256": digest(from_records(recs, True)),
            "gpu": torch.cuda.get_device_name(0)}


def run_shape(shape: str, seed: int, ratio: float, n_decode: int, prefill: int) -> dict:
    """A full-size shape (DeepSeek: 64 experts, top-6 + 2 shared) planned with
    the profile the bench calibrated on a B200 box.  The logits come from the
    reference's trace generator (the MoE-only stack has no normalisation, so a
    26-layer model-mode residual stream diverges); the LayerRequests -- counts
    and fp64 score sums -- are the GPU router's."""
    from paper_2504_05897_b200.moe import with_shared_time
    from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits
    cfg = SHAPES[shape]
    base = json.loads((ROOT / "profiles" / "r01c_configs" / f"{shape}_25.json").read_text())["profile"]
    prof = with_shared_time(mcost.HardwareProfile(**base), cfg)
    policy = me.EnginePolicy(cache_policy="mrs", prefetch=False)
    moe = HybridMoE(cfg, shape, policy, ratio, prof, max_tokens=prefill, host_images=64)
    moe.init_random_weights(seed)
    gen, logits = generate_router_logits(cfg, GenParams(seed=seed), prefill, n_decode)
    g = torch.Generator(device="cuda").manual_seed(seed)
    passes, recs = [], []
    for p, fwd in enumerate(gen.passes):
        lg = []
        for l in range(cfg.num_layers):
            a = logits[p][l].astype(np.float32)
            if moe.family.shared_gate:
                a = np.concatenate([a, np.zeros((a.shape[0], 1), np.float32)], axis=1)
            lg.append(torch.from_numpy(np.ascontiguousarray(a)).cuda())
        x = torch.randn((fwd.token_count, moe.H), generator=g, device="cuda").to(torch.bfloat16)
        _, info = moe.forward_pass(x, lg, decision_log=True)
        torch.cuda.synchronize()
        recs.extend(info["records"])
        passes.append(mcore.ForwardPass(fwd.stage, fwd.token_count,
                                        tuple(mcore.make_layer_request(l, lo.tolist(), sc.tolist())
                                              for l, (lo, sc) in enumerate(info["requests"]))))
    trace = mcore.Trace(cfg, tuple(passes), {"source": "live B200 run, GPU router on generator logits"})
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "t.jsonl"
        save_trace(trace, f)
        text = f.read_text()
    return {"policy": "mrs", "prefetch": False, "ratio": ratio, "seed": 2,
            "profile": {k: getattr(prof, k) for k in prof.__dataclass_fields__},
            "trace_jsonl": text, "runtime_stream_sha256": digest(from_records(recs, True)),
            "gpu": torch.cuda.get_device_name(0)}


if __name__ == "__main__":
    out = {p: run(p, 5 + i) for i, p in enumerate(("mrs", "lru", "lfu"))}
    out["mrs_prefetch"] = run_prefetch(9)
    out["deepseek_mrs"] = run_shape("deepseek", 11, 0.25, 6, 256)
    dst = ROOT / "gpurun_out" / "live_fixture.json"
    dst.parent.mkdir(exist_ok=True)
    dst.write_text(json.dumps(out))
    print(dst, {k: v["runtime_stream_sha256"][:16] for k, v in out.items()})
