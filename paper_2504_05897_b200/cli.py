"""Command line (SPEC.md:585-655 names the reference's intended CLI; the
reference never shipped it).  Decision commands run the native decision core;
``measure`` calibrates and runs the real layer stack on the GPU.

  python -m paper_2504_05897_b200.cli generate --model qwen2 --decode-steps 100 --seed 7 --out t.jsonl
  python -m paper_2504_05897_b200.cli run --trace t.jsonl --ratio 0.25 [--profile p.txt] [--policy mrs] [--prefetch]
  python -m paper_2504_05897_b200.cli sweep --model mixtral --ratios 0.25,0.5 --policies mrs,lru --seeds 0,1
  python -m paper_2504_05897_b200.cli calibrate --samples s.txt --out p.txt
  python -m paper_2504_05897_b200.cli measure --model mixtral --out p.txt      (GPU box: warm-up calibration)

Exit codes: 0 success, 1 usage, 2 data error, 3 internal invariant violation.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys

from .costs import CalibrationError, HardwareProfile, calibrate, load_profile, load_samples, save_profile
from .core import expert_bytes
from .engine import EnginePolicy, run_trace
from .errors import PlanInvariantError, TraceFormatError
from .prefetch import PredictionModel
from .tracegen import GenParams, generate_trace, load_trace, save_trace

PRESETS = {"mixtral", "deepseek", "qwen2", "tiny"}


def _model(name: str):
    from .moe import SHAPES
    return SHAPES[name]


def _default_profile(cfg) -> HardwareProfile:
    """A B200-host profile in seconds (6.4 TB/s HBM, 200 GB/s host DRAM, 55 GB/s PCIe)."""
    eb = expert_bytes(cfg)
    return HardwareProfile(gpu_time_per_expert=eb / 6.4e12 + 4e-6, cpu_slope=eb / 200e9, transfer_bandwidth=55e9,
                           transfer_latency=1e-5, cpu_first_expert_penalty=1.1)


def _policy(a) -> EnginePolicy:
    return EnginePolicy(scheduling=a.scheduling, cache_policy=a.policy, prefetch=a.prefetch,
                        prediction=PredictionModel(horizon=a.horizon, accuracy=a.accuracy))


def cmd_generate(a) -> int:
    cfg = _model(a.model)
    tr = generate_trace(cfg, GenParams(skew=a.skew, temporal_rho=a.rho, layer_sim=a.layer_sim, seed=a.seed),
                        a.prefill_tokens, a.decode_steps)
    save_trace(tr, a.out)
    print(f"wrote {a.out}: {len(tr.passes)} passes x {cfg.num_layers} layers")
    return 0


def cmd_run(a) -> int:
    tr = load_trace(a.trace)
    prof = load_profile(a.profile) if a.profile else _default_profile(tr.config)
    m = run_trace(tr, _policy(a), a.ratio, prof, a.seed)
    print(json.dumps(m.to_record()))
    return 0


def cmd_sweep(a) -> int:
    cfg = _model(a.model)
    rows = []
    print("policy\tratio\tseed\tttft\tmean_tbt\thit_rate")
    for seed in [int(s) for s in a.seeds.split(",")]:
        tr = generate_trace(cfg, GenParams(seed=seed), a.prefill_tokens, a.decode_steps)
        prof = load_profile(a.profile) if a.profile else _default_profile(cfg)
        for pol in a.policies.split(","):
            for ratio in [float(r) for r in a.ratios.split(",")]:
                m = run_trace(tr, EnginePolicy(cache_policy=pol, prefetch=a.prefetch), ratio, prof, seed)
                rows.append((pol, ratio, seed, m.ttft, m.mean_tbt, m.hit_rate))
                print(f"{pol}\t{ratio}\t{seed}\t{m.ttft}\t{m.mean_tbt}\t{m.hit_rate}")
    print("\n| policy | ratio | mean TTFT | mean TBT | hit rate |\n|---|---|---|---|---|")
    for pol in a.policies.split(","):
        for ratio in [float(r) for r in a.ratios.split(",")]:
            cell = [r for r in rows if r[0] == pol and r[1] == ratio]
            print(f"| {pol} | {ratio} | {statistics.mean(r[3] for r in cell):.6g} | "
                  f"{statistics.mean(r[4] for r in cell):.6g} | {statistics.mean(r[5] for r in cell):.4f} |")
    return 0


def cmd_calibrate(a) -> int:
    res = calibrate(load_samples(a.samples))
    save_profile(res.profile, a.out)
    print(res.report())
    return 0


def cmd_measure(a) -> int:
    from .calibration import calibrate_shape
    cfg = _model(a.model)
    res, samples = calibrate_shape(*cfg.routed_expert_dims)
    save_profile(res.profile, a.out)
    if a.samples_out:
        with open(a.samples_out, "w") as f:
            f.write("# device load position duration_s\n")
            for s in samples:
                f.write(f"{s.device} {s.load} {s.position} {s.duration!r}\n")
    print(res.report())
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="hybrimoe")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--model", choices=sorted(PRESETS), default="mixtral")
    g.add_argument("--prefill-tokens", type=int, default=1024)
    g.add_argument("--decode-steps", type=int, default=128)
    g.add_argument("--skew", type=float, default=1.0)
    g.add_argument("--rho", type=float, default=0.85)
    g.add_argument("--layer-sim", type=float, default=0.6)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out", required=True)
    for name in ("run", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("--profile")
        p.add_argument("--policy", default="mrs")
        p.add_argument("--prefetch", action="store_true")
        if name == "run":
            p.add_argument("--trace", required=True)
            p.add_argument("--ratio", type=float, default=0.25)
            p.add_argument("--seed", type=int, default=0)
            p.add_argument("--scheduling", default="hybrid")
            p.add_argument("--horizon", type=int, default=3)
            p.add_argument("--accuracy", type=float, default=0.85)
        else:
            p.add_argument("--model", choices=sorted(PRESETS), default="mixtral")
            p.add_argument("--ratios", default="0.25,0.5,0.75")
            p.add_argument("--policies", default="mrs,lru")
            p.add_argument("--seeds", default="0")
            p.add_argument("--prefill-tokens", type=int, default=1024)
            p.add_argument("--decode-steps", type=int, default=32)
    c = sub.add_parser("calibrate")
    c.add_argument("--samples", required=True)
    c.add_argument("--out", required=True)
    m = sub.add_parser("measure")
    m.add_argument("--model", choices=sorted(PRESETS), default="mixtral")
    m.add_argument("--out", required=True)
    m.add_argument("--samples-out")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 1 if e.code else 0
    try:
        return {"generate": cmd_generate, "run": cmd_run, "sweep": cmd_sweep, "calibrate": cmd_calibrate,
                "measure": cmd_measure}[a.cmd](a)
    except (ValueError, TraceFormatError, CalibrationError, FileNotFoundError) as exc:
        if isinstance(exc, PlanInvariantError):
            print(f"invariant violation: {exc}", file=sys.stderr)
            return 3
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
