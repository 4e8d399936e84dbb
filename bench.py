#!/usr/bin/env python
"""HybriMoE MoE-layer hot path on B200: decode tok/s and 1k-token prefill latency
at a 25% expert-cache budget (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus 1] [--steps 8] [--warmup 3] [--shape mixtral] [--impl ours|reference]

A "step" is one decode pass: one token through all L MoE layers of the named
shape (random-init bf16 weights, synthetic routing from the reference's trace
generator), executed under the HybriMoE schedule -- GPU experts from the HBM
cache, demand copies over PCIe, CPU experts on the host worker -- with the
decision core planning every layer from a profile calibrated on this box.
The prefill pass (1024 tokens, cold cache) runs first and is reported as
``prefill.ms``.  ``--impl reference`` times the CPU oracle port of the path
(oracle/: the reference's decisions + fp32 numpy experts, all on the CPU).
"""
from __future__ import annotations

import argparse
import dataclasses
from dataclasses import replace
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region:
    ONE `nvidia-smi --query-gpu=... -lms 50` process (the profiling recipe's
    looping form), started (and its first row read) before the region and
    terminated after it, at least one row later.  (Spawning a
    fresh nvidia-smi every 200 ms kept a host core busy with NVML start-up for
    the whole region and delayed the host worker's threads.)"""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int = 0) -> None:
        self.gpu, self.rows, self._proc = gpu, [], None
        self._t = threading.Thread(target=self._read, daemon=True)

    def _read(self) -> None:
        try:
            for line in self._proc.stdout:
                self.rows.append([v.strip() for v in line.strip().split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            t0 = time.time()  # NVML is up once the first row arrives: the region starts after it
            while not self.rows and time.time() - t0 < 3.0 and self._proc.poll() is None:
                time.sleep(0.005)
            self._n0 = len(self.rows)
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is not None:
            t0 = time.time()  # at least one row taken after the region started
            while len(self.rows) <= getattr(self, "_n0", 0) and time.time() - t0 < 1.0:
                time.sleep(0.005)
            self._proc.terminate()  # our own child, by its handle
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self) -> dict:
        rows = self.rows[getattr(self, "_n0", 0):] or self.rows  # rows taken inside the region
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i - 3] for r in rows if len(r) >= 7 for i in range(3, 7)
                          if r[i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# --------------------------------------------------------------------------- reference arm / cpu baseline
# The reference's own CPU path for this hot path: every
# expert of every layer on the host cores under plan_all_cpu semantics
# (scheduling.py:273-284), bf16 expert weights with fp32 accumulation
# (torch CPU / oneDNN, AMX where present) on all host threads, routing from the
# reference's own trace generator (fp32 logits frozen from the unmodified
# moesim.tracegen by tests/golden/make_router_golden.py), the router and the
# plan from the oracle restatement.  Nothing here imports the product package.
REF_SHAPES = {  # L, N, K, (H, I), shared chunks of (H, I), renormalise, shared gate
    "tiny": (4, 8, 2, (256, 256), 0, True, False),
    "mixtral": (32, 8, 2, (4096, 14336), 0, True, False),
    "deepseek": (26, 64, 6, (2048, 1408), 2, False, False),
    "qwen2": (28, 64, 8, (3584, 2560), 8, False, True),
}
REF_POOL_BYTES = 16 << 30   # distinct expert images (aliased modulo their count): >> host LLC


def host_info() -> dict:
    out = {"cpu_count": os.cpu_count()}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {ln.split(":", 1)[0].strip(): ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ":" in ln}
        out.update(model=kv.get("Model name"), sockets=kv.get("Socket(s)"), numa_nodes=kv.get("NUMA node(s)"),
                   l3=kv.get("L3 cache"))
    except Exception:
        pass
    return out


class CpuMoE:
    """The all-CPU MoE stack of one shape: bf16 expert images on the host."""

    def __init__(self, shape: str, threads: int | None = None, pool_bytes: int = REF_POOL_BYTES) -> None:
        import torch
        self.torch = torch
        L, N, K, (H, I), S, renorm, sgate = REF_SHAPES[shape]
        self.L, self.N, self.K, self.H, self.I, self.S, self.renorm, self.sgate = L, N, K, H, I, S, renorm, sgate
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        n = 3 * H * I
        total = L * (N + S)
        self.n_images = int(min(total, max(8, pool_bytes // (2 * n))))
        g = torch.Generator().manual_seed(0)
        base = (torch.randn(n, generator=g) * 0.02).to(torch.bfloat16)
        self.images = torch.empty((self.n_images, n), dtype=torch.bfloat16)
        for i in range(self.n_images):  # distinct images: base rotated by a per-image offset
            o = (i * 7919 * 64) % n
            self.images[i, : n - o].copy_(base[o:])
            self.images[i, n - o:].copy_(base[:o])
        self.logits = np.load(ROOT / "oracle" / "fixtures" / f"decode_logits_{shape}.npy")
        self.image_bytes = 2 * n
        from oracle import cpu_moe
        self.scratch = cpu_moe.Scratch()

    def expert(self, l: int, e: int, x):
        """SwiGLU on rows x [M, H] bf16, fp32 accumulation: decode-sized row
        groups through the plain-C oracle (oracle/cpu_moe.c, weight streaming
        on all threads), prefill-sized ones through torch CPU (oneDNN / AMX
        GEMM).  Image layout: W13 rows [gate | up] x H, then W2 [H][I]."""
        torch = self.torch
        img = self.images[(l * (self.N + self.S) + e) % self.n_images]
        H, I = self.H, self.I
        if x.shape[0] <= 8:
            from oracle import cpu_moe
            xc = x.contiguous()
            out = torch.empty((x.shape[0], H), dtype=torch.float32)
            cpu_moe.expert(img.data_ptr(), img.data_ptr() + 4 * H * I, H, I, xc.data_ptr(), x.shape[0],
                           out.data_ptr(), self.scratch)
            return out
        F = torch.nn.functional
        gu = F.linear(x, img[: 2 * H * I].view(2 * I, H)).float()
        h = (F.silu(gu[:, :I]) * gu[:, I:]).to(torch.bfloat16)
        return F.linear(h, img[2 * H * I:].view(H, I)).float()

    def layer(self, l: int, x, logits: np.ndarray):
        """One MoE layer on x [T, H] bf16 with fp32 logits [T, N]: oracle router,
        plan_all_cpu, experts in plan order, weighted sum + residual."""
        from oracle import decisions as od
        from oracle import moe_ref as ref
        torch = self.torch
        lg = logits
        if self.sgate:
            lg = np.concatenate([lg, np.zeros((lg.shape[0], 1), np.float32)], axis=1)
        sel, w, _, counts, _ = ref.router(lg, self.N, self.K, self.renorm, self.S, self.N if self.sgate else -1)
        tasks = [((l, e), int(counts[e])) for e in range(self.N + self.S) if counts[e] > 0]
        events, _, _ = od.all_cpu(tasks, self.prof)
        y = torch.zeros((x.shape[0], self.H), dtype=torch.float32)
        selt, wt = torch.from_numpy(sel), torch.from_numpy(w)
        for ev in events:  # plan CPU order
            e = ev[1][1]
            rows, slot = (selt == e).nonzero(as_tuple=True)
            out = self.expert(l, e, x[rows])
            y.index_add_(0, rows, out * wt[rows, slot][:, None])
        return (x.float() + y).to(torch.bfloat16)

    prof = dict(gpu_time_per_expert=1.0, cpu_slope=1.0, transfer_bandwidth=1e9, transfer_latency=0.0,
                gpu_saturation_load=256, gpu_slope=0.0, cpu_first_expert_penalty=1.0, shared_expert_time=0.0,
                non_expert_time=0.0)

    def decode_token(self, p: int, x):
        for l in range(self.L):
            x = self.layer(l, x, self.logits[p % len(self.logits), l][None, :])
        return x

    def prefill(self, T: int, seed: int = 0):
        rng = np.random.default_rng(seed)
        x = self.torch.randn((T, self.H), generator=self.torch.Generator().manual_seed(seed)).to(self.torch.bfloat16)
        for l in range(self.L):
            x = self.layer(l, x, rng.standard_normal((T, self.N)).astype(np.float32))
        return x


def cpu_reference_decode(shape: str, steps: int, warmup: int, prefill: int = 0, threads: int | None = None):
    """Timed all-CPU decode (and optionally one prefill): returns the cpu_baseline dict."""
    import torch
    t_setup = time.perf_counter()
    m = CpuMoE(shape, threads)
    setup = time.perf_counter() - t_setup
    x = torch.randn((1, m.H), generator=torch.Generator().manual_seed(1)).to(torch.bfloat16)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        x = m.decode_token(i, x)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    ms = 1e3 * statistics.mean(times)
    out = {"value": 1e3 / ms, "unit": "tok/s", "cores": m.threads, "kind": "port", "ms_per_token": ms,
           "sample": f"{steps} decode tokens x all {m.L} layers (after {warmup} warm-up), every expert on the host: "
                     f"bf16 weights, fp32 accumulation (plain-C oracle oracle/cpu_moe.c, OpenMP, {m.threads} "
                     f"threads; prefill GEMMs torch CPU/oneDNN), oracle router + "
                     f"plan_all_cpu; routing = fp32 logits frozen from the unmodified reference generator; "
                     f"{m.n_images} distinct {m.image_bytes / 1e6:.1f} MB expert images aliased modulo their count "
                     f"({m.n_images * m.image_bytes / 1e9:.1f} GB >> LLC)",
           "setup_s": setup, "host": host_info()}
    if prefill:
        t0 = time.perf_counter()
        m.prefill(prefill)
        out["prefill_ms"] = 1e3 * (time.perf_counter() - t0)
        out["prefill_tokens"] = prefill
    return out


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_reference_decode(args.shape, args.steps, args.warmup, prefill=args.prefill if args.ref_prefill else 0)
    tok_s = cb["value"]
    line = {"impl": "reference", "metric": "decode tok/s at 25% expert-cache budget", "value": tok_s,
            "unit": "tok/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cb["ms_per_token"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16 weights, fp32 accumulation (CPU)",
            "data": "synthetic (reference trace-generator routing frozen from the reference, random-init weights)",
            "config": {"workload": f"{args.shape}-shaped MoE decode, batch 1, all experts on the host CPU "
                                   f"(the reference's CPU path, plan_all_cpu)", "shape": args.shape},
            "cpu_baseline": cb,
            "e2e": {"value": tok_s, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if "prefill_ms" in cb:
        line["prefill"] = {"tokens": cb["prefill_tokens"], "ms": cb["prefill_ms"]}
    print(json.dumps(line), flush=True)


def reference_decision_path(passes, cfg, profile, capacity: int, policy: str, prefetch: bool) -> dict:
    """the reference's decision path (oracle restatement of
    run_pass, engine.py:288-486; one Python thread) on the same LayerRequests
    and calibrated profile the runtime planned with: microseconds per layer."""
    from oracle import decisions as od
    prof = {k: getattr(profile, k) for k in ("gpu_time_per_expert", "cpu_slope", "transfer_bandwidth",
                                              "transfer_latency", "gpu_saturation_load", "gpu_slope",
                                              "cpu_first_expert_penalty", "shared_expert_time", "non_expert_time")}
    H, I = cfg.routed_expert_dims
    nbytes = 3.0 * H * I * cfg.bytes_per_weight
    t0 = time.perf_counter()
    od.run(passes, cfg.num_layers, cfg.num_routed, cfg.num_activated, nbytes, prof, capacity, policy, False)
    dt = time.perf_counter() - t0
    n_layers = sum(len(layers) for _, layers in passes)
    return {"us_per_layer": 1e6 * dt / max(1, n_layers), "layers": n_layers, "threads": 1, "kind": "port",
            "what": "oracle restatement of the reference run_pass decisions (lookup, select_plan, inserts, MRS) on "
                    "the runtime's own LayerRequests (the timed decode passes) with the calibrated profile"}


# --------------------------------------------------------------------------- our arm
def warm_parity(cfg, trace, requests, records, moe, policy, args) -> dict:
    """Evidence carried in the bench line: the GPU router's loads equal the
    reference trace generator's for every warm-up layer, and the digest of the
    runtime's decision stream (tests/test_runtime_gpu.py proves the stream equals
    the decision core replayed on the same LayerRequests)."""
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    from stream import digest, from_records

    from paper_2504_05897_b200 import core as mcore
    n_eq = n_tot = 0
    for i, reqs in enumerate(requests):
        for l, (loads, _scores) in enumerate(reqs):
            want = list(trace.passes[1 + i].layers[l].loads)
            if moe.ep_world > 1:
                want = [v if e % moe.ep_world == moe.ep_rank else 0 for e, v in enumerate(want)]
            n_eq += int(list(loads) == want)
            n_tot += 1
    return {"router_loads_equal_reference_trace": f"{n_eq}/{n_tot}",
            "decision_stream_sha": digest(from_records(records, policy.cache_policy == "mrs"))[:16],
            "warmup_layers_recorded": len(records)}


def _trace(msg: str) -> None:
    """HM_BENCH_TRACE=1: stage markers on stderr (debugging multi-rank runs)."""
    if os.environ.get("HM_BENCH_TRACE") == "1":
        print(f"[rank {os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_ours(args) -> None:
    if os.environ.get("HM_NCU_TIMED") == "1":
        # under ncu's serialised replay nothing may wait on the host: no timing
        # gate, no host-mapped router flag (the copy path is used instead)
        os.environ["HM_TIMING_GATE"] = "0"
        os.environ["HM_ZERO_COPY"] = "0"
    import torch

    from paper_2504_05897_b200 import _lib
    from paper_2504_05897_b200.calibration import calibrate_shape
    from paper_2504_05897_b200.engine import EnginePolicy
    from paper_2504_05897_b200.moe import SHAPES, HybridMoE, layer_stats, with_shared_time
    from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU is required")
    # HM_SAME_GPU=1: every rank on cuda:0 with a gloo control plane -- only to
    # exercise the multi-rank harness on a one-GPU box (timings meaningless:
    # the ranks' contexts time-slice the GPU)
    same_gpu = os.environ.get("HM_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL's init log (communicator size and ranks) on stderr, also when
        # torchrun launched us (the self-spawn path sets the same)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # one process per GPU: this rank's host worker on its GPU's NUMA node, the
    # node's cores split between the ranks that share it (before anything
    # allocates pinned memory or starts host threads; hostplace.py)
    bound_cpus = None
    if world > 1 and not same_gpu:
        from paper_2504_05897_b200.hostplace import bind_rank
        bound_cpus = bind_rank(local, int(os.environ.get("LOCAL_WORLD_SIZE", world)))

    cfg = SHAPES[args.shape]
    if args.bits == 4:  # the paper's 4-bit experts: expert_bytes at 0.5 bytes per weight (core.py:55)
        from dataclasses import replace as _replace
        cfg = _replace(cfg, bytes_per_weight=0.5)
    H, I = cfg.routed_expert_dims
    pk, pk_kind = peaks()
    t_setup = time.time()
    from paper_2504_05897_b200.costs import load_profile, save_profile
    # Stage-calibrated profiles: the reference's cost model is linear in load
    # (costs.py:68-88), but the host worker is DRAM-bound at decode loads and
    # compute-bound (AMX) at prefill loads, so one fit cannot serve both.  The
    # decode profile is fitted at the load decode plans with -- one token per
    # expert at batch 1 -- so a host expert is rated at its streaming time, not
    # at a slope through loads 1-4 (which under-rated it 1.8x in round 1); the
    # prefill profile at prefill loads.  Each pass is planned with its stage's profile.
    # host-worker threads of this rank (the calibration measures the same pool size)
    threads = args.cpu_threads or (len(bound_cpus) if bound_cpus else max(1, (os.cpu_count() or 1) // world))
    if args.profile_file:  # e.g. for runs under a profiler, where warm-up timings are distorted
        base_profile = load_profile(args.profile_file)
        prefill_profile = load_profile(args.prefill_profile_file) if args.prefill_profile_file else base_profile
    else:
        base_profile = calibrate_shape(H, I, weight_bits=args.bits, gpu_loads=(1, 2, 3, 4), cpu_loads=(1,),
                                       cpu_bursts=4, cpu_threads=threads)[0].profile
        prefill_profile = base_profile
        if args.stage_profiles and not args.live_fixture:  # a fixture replays with ONE profile
            prefill_profile = calibrate_shape(H, I, cpu_loads=(64, 128, 256), cpu_bursts=1,
                                              gpu_loads=(64, 128, 256, 384, 512), weight_bits=args.bits,
                                              cpu_threads=threads)[0].profile
        if args.save_profile and rank == 0:
            save_profile(base_profile, args.save_profile)
            save_profile(prefill_profile, args.save_profile + ".prefill")
    prof = with_shared_time(base_profile, cfg)
    prof_prefill = with_shared_time(prefill_profile, cfg)
    # non-expert (attention block) time per layer, measured on this GPU at the
    # family's attention shapes (costs.py:45, engine.py:307): reported as the
    # reference's end-to-end what-if; the planning profile keeps the
    # reference's default 0 (SPEC.md: speedups isolate expert handling), which
    # no decision depends on
    from paper_2504_05897_b200.calibration import measure_non_expert_time
    non_expert = {"decode_us_per_layer": 1e6 * measure_non_expert_time(args.shape, 1, args.prefill),
                  "prefill_us_per_layer": 1e6 * measure_non_expert_time(args.shape, args.prefill, 0, reps=3),
                  "context": args.prefill,
                  "what": "RMSNorm + QKV/O projections + SDPA over the KV cache, bf16 (cuBLAS/SDPA library calls, "
                          "calibration input only, not executed in the timed step)"}
    policy = EnginePolicy(scheduling=args.scheduling, cache_policy=args.policy, prefetch=args.prefetch)
    # expert parallelism over the ranks of this box: each rank homes experts
    # e % world, host bytes and worker cores split by rank
    image_bytes = 3 * H * I * 2 if args.bits == 16 else 3 * H * I // 2 + 3 * H * I // 64
    total_bytes = cfg.num_layers * cfg.num_routed * image_bytes // world
    host_images = args.host_images
    if host_images is None:
        try:
            import psutil
            avail = psutil.virtual_memory().available // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        except Exception:
            avail = 0
        host_images = None if avail > 1.3 * total_bytes else max(16, int(0.5 * avail / image_bytes))
    from paper_2504_05897_b200.ep import PeerMemoryUnavailable
    exchange_note = None
    try:
        moe = HybridMoE(cfg, args.shape, policy, args.ratio, prof, host_images=host_images,
                        max_tokens=max(args.prefill, 1), cpu_threads=threads, ep_rank=rank, ep_world=world,
                        exchange=args.exchange, weight_bits=args.bits)
    except PeerMemoryUnavailable as e:  # every rank sees the same verdict: use the NCCL exchange instead
        if args.exchange not in ("p2p", "dispatch"):
            raise
        fallback = "nccl_a2a" if args.exchange == "dispatch" else "allreduce"
        exchange_note = f"p2p unavailable ({e}); NCCL {fallback} used"
        moe = HybridMoE(cfg, args.shape, policy, args.ratio, prof, host_images=host_images,
                        max_tokens=max(args.prefill, 1), cpu_threads=threads, ep_rank=rank, ep_world=world,
                        exchange=fallback, weight_bits=args.bits)
    moe.init_random_weights(seed=args.seed + rank)
    n_dec = args.warmup + args.steps
    # passes: prefill | warm-up | timed | instrumented (kernel timing) | e2e
    n_pass = 1 + n_dec + args.steps + n_dec
    trace, logits = generate_router_logits(cfg, GenParams(seed=args.seed), args.prefill, n_pass - 1)
    dev_logits = []
    for p in range(len(trace.passes)):
        layer_logits = []
        for l in range(cfg.num_layers):
            lg = logits[p][l].astype(np.float32)
            if moe.family.shared_gate:
                lg = np.concatenate([lg, np.zeros((lg.shape[0], 1), np.float32)], axis=1)
            layer_logits.append(torch.from_numpy(np.ascontiguousarray(lg)).cuda())
        dev_logits.append(layer_logits)
    if args.scheduling == "fixed_frequency_map":  # kTransformers-like pinned set (engine.py:195-231)
        from paper_2504_05897_b200.engine import compute_fixed_pinned_set
        fixed = compute_fixed_pinned_set(trace, moe.capacity * world, policy.calibration_prefix_fraction, None)
        moe.set_fixed_gpu_set(sorted(r for r in fixed if r[1] % world == rank)[: moe.capacity])
    g = torch.Generator(device="cuda").manual_seed(1234)  # replicated hidden state on every rank
    xs = [torch.randn((f.token_count, H), generator=g, device="cuda").to(torch.bfloat16) for f in trace.passes]
    if world > 1 and moe.exchange in ("dispatch", "nccl_a2a"):  # token-sharded: rank r keeps tokens [r*T/G, (r+1)*T/G)
        def shard(t):
            T = t.shape[0]
            return t[rank * T // world:(rank + 1) * T // world].contiguous()
        xs = [shard(x) for x in xs]
        dev_logits = [[shard(t) for t in layer_logits] for layer_logits in dev_logits]
    torch.cuda.synchronize()
    # host DRAM read bandwidth over (part of) the pinned master store: the host roofline
    import ctypes as C
    cp = C.c_void_p()
    _lib.check(_lib.lib.hm_cpu_pool_create(threads, C.byref(cp)))
    hbw = C.c_double()
    nbytes = min(moe.store.nbytes, 16 << 30)
    _lib.check(_lib.lib.hm_host_read_bw(cp, moe.store.ctypes.data, nbytes, 3, C.byref(hbw)))
    _lib.lib.hm_cpu_pool_destroy(cp)
    host_bw_gbs = hbw.value if args.host_bw_gbs <= 0 else args.host_bw_gbs
    setup_s = time.time() - t_setup
    _trace(f"setup done in {setup_s:.1f} s")

    from paper_2504_05897_b200.moe import TracePredictor
    predictors = [TracePredictor(trace, p, args.seed) for p in range(len(trace.passes))]

    def predictor(p):  # the reference's prediction model on this pass, natively -- or the live look-ahead
        return "live" if args.predict == "live" else predictors[p]

    lib = _lib.lib
    st = torch.cuda.current_stream()
    live_fixture = bool(args.live_fixture)
    fixture_records, fixture_requests = [], []
    # ---- prefill: 1k tokens, cold cache (the reference's TTFT, engine.py:465-466)
    _trace("prefill")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.hm_runtime_set_copy_timing(moe._rt, 1)
    moe.set_profile(prof_prefill)
    ev0.record(st)
    _, pinfo = moe.forward_pass(xs[0], dev_logits[0], predict=predictor(0), decision_log=live_fixture)
    ev1.record(st)
    ev1.synchronize()
    moe.set_profile(prof)
    prefill_ms = ev0.elapsed_time(ev1)
    if live_fixture:
        fixture_records.extend(pinfo["records"])
        fixture_requests.append(pinfo["requests"])
    cms, cby, cn, cmx = C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
    _lib.check(lib.hm_runtime_copy_times(moe._rt, C.byref(cms), C.byref(cby), C.byref(cn), C.byref(cmx)))
    lib.hm_runtime_set_copy_timing(moe._rt, 0)
    # PCIe roofline of the prefill's expert copies (CUDA events on the copy stream)
    h2d_roofline = {"bound": "pcie", "copies": cn.value, "bytes": cby.value, "copy_ms": cms.value,
                    "achieved_gbs": cby.value / (cms.value / 1e3) / 1e9 if cms.value > 0 else None,
                    "peak_gbs_gen5_x16": 64.0,
                    "frac_of_gen5": (cby.value / (cms.value / 1e3) / 1e9 / 64.0) if cms.value > 0 else None,
                    "link_busy_frac_of_prefill": cms.value / prefill_ms if prefill_ms > 0 else None}
    pst = layer_stats(pinfo)
    predicted_ttft_ms = 1e3 * pinfo["pass"].latency
    if os.environ.get("HM_BENCH_DUMP_PREFILL"):  # per-layer prefill stats (diagnostics)
        Path(os.environ["HM_BENCH_DUMP_PREFILL"]).write_text(json.dumps(
            {"prefill_ms": prefill_ms, "predicted_ms": predicted_ttft_ms,
             "layers": [dataclasses.asdict(x) for x in pst]}, indent=1))

    # ---- decode: W warm-up passes (recorded for the parity block), then K timed passes
    _trace("decode")
    warm_records, warm_requests, warm_stats = [], [], []
    for p in range(1, 1 + args.warmup):
        _, winfo = moe.forward_pass(xs[p], dev_logits[p], predict=predictor(p), decision_log=True)
        warm_records.extend(winfo["records"])
        warm_requests.append(winfo["requests"])
        warm_stats.extend(winfo["stats"])
    torch.cuda.synchronize()
    if live_fixture:
        fixture_records.extend(warm_records)
        fixture_requests.extend(warm_requests)
    parity = warm_parity(cfg, trace, warm_requests, warm_records, moe, policy, args)
    # warm-up calibration of the host worker (§IV-A): the decode
    # passes above are the workload itself -- refit the reference's CPU cost
    # (cpu_slope x (penalty + n - 1) per layer burst of n experts, costs.py:68-88)
    # on their measured worker times and plan the timed passes with it; the
    # stand-alone micro-calibration drifts +-40 % from box to box
    refit = refit_cpu_decode(warm_stats, prof) if args.refit and not live_fixture else None
    if refit is not None:
        prof = replace(prof, cpu_slope=refit["cpu_slope"], cpu_first_expert_penalty=refit["cpu_first_expert_penalty"])
        moe.set_profile(prof)
    launches0 = lib.hm_launch_count()
    stats_all, predicted = [], []
    worker_prof = os.environ.get("HM_BENCH_WORKER_PROF") == "1"  # diagnostics only, never in a reported run
    if worker_prof:
        _lib.check(lib.hm_cpu_decode_profile_accum(None, 1))
        lib.hm_cpu_decode_profile(1, None, 0)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # the timed region runs the runtime exactly as e2e does: no kernel-timing
    # events, no timing gate (those run in a separate instrumented pass below)
    ncu_timed = os.environ.get("HM_NCU_TIMED") == "1"  # bracket for `ncu --profile-from-start off`
    with ClockSampler(local) as clocks:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ncu_timed:
            torch.cuda.profiler.start()
        t0.record(st)
        for k in range(args.steps):
            p = 1 + args.warmup + k
            _, info = moe.forward_pass(xs[p], dev_logits[p], predict=predictor(p))
            stats_all.append(info)
        t1.record(st)
        t1.synchronize()
        torch.cuda.synchronize()
        if ncu_timed:
            torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
    launches = lib.hm_launch_count() - launches0
    predicted = [1e3 * info["pass"].latency for info in stats_all]
    stats_all = [s for info in stats_all for s in layer_stats(info)]
    if worker_prof:  # per-call host-worker phase breakdown of the timed passes (diagnostics)
        acc, hist, slow = (C.c_int64 * 7)(), (C.c_int64 * 5)(), (C.c_int64 * 64)()
        _lib.check(lib.hm_cpu_decode_profile_hist(hist, slow, 64))
        print("[worker profile] start-delay histogram (<=5, 20, 100, 1000, >1000 us):", list(hist),
              "slowest starter per tid:", [v for v in slow][:threads], file=sys.stderr, flush=True)
        _lib.check(lib.hm_cpu_decode_profile_accum(acc, 1))
        lib.hm_cpu_decode_profile(0, None, 0)
        n = max(1, acc[0])
        print("[worker profile] calls %d, mean us: worker start %.1f, caller start %.1f, phase-1 end %.1f, "
              "barrier %.1f, phase-2 end %.1f, wall %.1f" % (acc[0], *(acc[i] / n / 1e3 for i in range(1, 7))),
              file=sys.stderr, flush=True)
    if os.environ.get("HM_BENCH_DUMP_DECODE"):  # per-layer timed-decode stats (diagnostics)
        Path(os.environ["HM_BENCH_DUMP_DECODE"]).write_text(json.dumps(
            [dataclasses.asdict(x) for x in stats_all]))
    ms_total = t0.elapsed_time(t1)
    if dist:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    tok_s = 1e3 / ms_step  # one sequence, experts sharded: tokens of the whole job per second

    # ---- instrumented passes (outside the timed region): CUDA events around
    # every expert-FFN launch for the dominant kernel's roofline
    _trace("instrumented")
    lib.hm_runtime_set_kernel_timing(moe._rt, 1)
    i0 = 1 + n_dec
    for k in range(args.steps):
        p = i0 + k
        moe.forward_pass(xs[p], dev_logits[p], predict=predictor(p))
    torch.cuda.synchronize()
    kms, kbytes, kn, kmax = C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
    lib.hm_runtime_kernel_times(moe._rt, C.byref(kms), C.byref(kbytes), C.byref(kn), C.byref(kmax))
    lib.hm_runtime_set_kernel_timing(moe._rt, 0)

    # ---- e2e: host buffers through the public API, copies inside the timed region
    _trace("e2e")
    e2e_passes = list(range(1 + n_dec + args.steps, 1 + 2 * n_dec + args.steps))
    host_x = [xs[p].cpu().pin_memory() for p in e2e_passes]
    host_lg = [torch.stack([t.cpu() for t in dev_logits[p]]).pin_memory() for p in e2e_passes]
    y_host = torch.empty((host_x[0].shape[0], H), dtype=torch.bfloat16).pin_memory()
    dx = torch.empty_like(host_x[0], device="cuda")
    dlg = torch.empty_like(host_lg[0], device="cuda")
    for i in range(args.warmup):
        dx.copy_(host_x[i], non_blocking=True)
        dlg.copy_(host_lg[i], non_blocking=True)
        y, _ = moe.forward_pass(dx, list(dlg), predict=predictor(e2e_passes[i]))
        y_host.copy_(y, non_blocking=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(args.warmup, n_dec):
        dx.copy_(host_x[i], non_blocking=True)
        dlg.copy_(host_lg[i], non_blocking=True)
        y, _ = moe.forward_pass(dx, list(dlg), predict=predictor(e2e_passes[i]))
        y_host.copy_(y, non_blocking=True)
    e1.record(st)
    e1.synchronize()
    e2e_total = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_ms = e2e_total / args.steps
    h2d = host_x[0].numel() * 2 + host_lg[0].numel() * 4
    d2h = y_host.numel() * 2

    # ---- roofline of the dominant GPU kernel (decode expert FFN, HBM-bound)
    achieved_gbs = kbytes.value / (kms.value / 1e3) / 1e9 if kms.value > 0 else 0.0
    hbm_peak = float(pk["hbm_gbs"])
    # DRAM traffic of the same kernels from the committed ncu --set full capture
    # (tools/profile_round.sh): measured bytes for that launch beside its
    # algorithmic bytes -- traffic ~ algorithmic means weights are read once
    traffic = {}
    tp = {("mixtral", 16): "r02_traffic_mixtral.json", ("deepseek", 16): "r02_traffic_deepseek.json",
          ("qwen2", 16): "r02_traffic_qwen2.json", ("mixtral", 4): "r01d_traffic_mixtral_q4.json"}.get(
        (args.shape, args.bits))
    if tp is not None and (ROOT / "profiles" / tp).exists():
        traffic = json.loads((ROOT / "profiles" / tp).read_text())
    tg = traffic.get("decode_gemv", {})
    roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak, "traffic": tg.get("dram_bytes"),
                "traffic_launch": tg.get("launch"), "traffic_algorithmic_bytes": tg.get("algorithmic_bytes"),
                "traffic_source": traffic.get("source"),
                "kernel": "decode expert FFN: ffn1_gemv + ffn2_gemv pair (PDL), weights streamed once" if args.bits == 16 else
                          "decode expert FFN on 4-bit images (ffn1_q4 + ffn2_q4)",
                "launches": kn.value, "avg_launch_us": 1e3 * kms.value / max(1, kn.value),
                "bytes_per_launch": kbytes.value / max(1, kn.value), "peak_kind": pk_kind,
                "timed_in": "separate instrumented passes (CUDA events around each expert-FFN launch), "
                            "not the headline timed region"}
    # plan-conditional roofline of the whole step: max(B_gpu/BW_hbm, B_cpu/BW_host, B_h2d/BW_pcie) per layer;
    # host bandwidth = the better of the read probe and what the worker itself streamed in the step
    cpu_us = sum(s.t_cpu_us for s in stats_all)
    worker_gbs = sum(s.bytes_cpu for s in stats_all) / (cpu_us * 1e-6) / 1e9 if cpu_us > 0 else 0.0
    host_probe_gbs = host_bw_gbs
    host_bw_gbs = max(host_bw_gbs, worker_gbs)
    bw_host = host_bw_gbs * 1e9
    bw_pcie = base_profile.transfer_bandwidth  # bytes / s, fitted at warm-up
    bound_s = sum(max(s.bytes_gpu / (hbm_peak * 1e9), s.bytes_cpu / bw_host, s.bytes_h2d / bw_pcie)
                  for s in stats_all)
    n_cpu = sum(s.n_cpu for s in stats_all) / args.steps
    n_gpu = sum(s.n_gpu for s in stats_all) / args.steps
    n_xfer = sum(s.n_transfer for s in stats_all) / args.steps

    # ---- prefill-side kernel: grouped tcgen05 GEMM over 8 resident experts x 256 tokens
    from paper_2504_05897_b200.microbench import gemm_bench
    gb = gemm_bench(H, I, rows_per_expert=256, n_experts=cfg.num_routed if cfg.num_routed <= 8 else 8)
    tc_peak = float(pk["bf16_tflops"])
    tm = traffic.get("prefill_gemm", {})
    gemm_roofline = {"bound": "tensor", "achieved": gb["tflops"], "peak": tc_peak, "unit": "TFLOP/s",
                     "frac": gb["tflops"] / tc_peak, "traffic": tm.get("dram_bytes"),
                     "traffic_algorithmic_bytes": tm.get("algorithmic_bytes"), "peak_kind": pk_kind + " burst",
                     "kernel": "expert_gemm_kernel (ffn1 SwiGLU + ffn2), 256 tokens x 8 experts",
                     "ms": gb["ms"], "hbm_gbs": gb["hbm_gbs"]}
    # 256 tokens per expert is 256 flop per weight byte -- the ridge: the shape's
    # own roof is min(tensor peak, HBM x intensity); and the same kernel at a
    # compute-bound shape (1024 tokens per expert) for the tensor-pipe side
    ai = 256.0
    shape_roof = min(tc_peak, hbm_peak * ai / 1e3)
    gemm_roofline.update({"flop_per_weight_byte": ai, "shape_roof_tflops": shape_roof,
                          "frac_of_shape_roof": gb["tflops"] / shape_roof})
    gc = gemm_bench(H, I, rows_per_expert=1024, n_experts=4, reps=3)
    gemm_roofline["compute_bound"] = {"tokens_per_expert": 1024, "experts": 4, "achieved": gc["tflops"],
                                      "frac": gc["tflops"] / tc_peak, "ms": gc["ms"],
                                      "ncu_tensor_pipe_active": "85.1 % / 80.9 % (profiles/r02_ncu_gemm_q4.md)"}

    # ---- BASELINE.md §5 A (decision path) and C (simulator prediction vs measured)
    decision_baseline = None
    if rank == 0 and not args.no_cpu_baseline:
        dpasses = [("decode", [(l, list(lo), list(sc)) for l, (lo, sc) in enumerate(reqs)])
                   for reqs in warm_requests]
        decision_baseline = reference_decision_path(dpasses, cfg, prof, moe.capacity, args.policy, False)
        decision_baseline["native_us_per_layer"] = statistics.mean(s.t_decide_us for s in stats_all)
        decision_baseline["speedup"] = decision_baseline["us_per_layer"] / max(1e-9,
                                                                              decision_baseline["native_us_per_layer"])
    model_check = {"what": "simulator (the reference's cost model, the decision core's own pass latency) with the "
                           "calibrated profiles vs measured",
                   "predicted_tbt_ms": statistics.mean(predicted), "measured_tbt_ms": ms_step,
                   "tbt_ratio_measured_over_predicted": ms_step / max(1e-9, statistics.mean(predicted)),
                   "predicted_ttft_ms": predicted_ttft_ms, "measured_ttft_ms": prefill_ms,
                   "ttft_ratio_measured_over_predicted": prefill_ms / max(1e-9, predicted_ttft_ms)}

    # ---- CPU baseline: the reference's all-CPU path on this host, bounded sample
    cpu = None
    # release the pinned store, the slot pool and the worker threads before the
    # CPU baseline and the child config runs: explicit, so that a reference
    # still held elsewhere cannot keep 90 GB of pinned host memory alive
    torch.cuda.synchronize()
    if dist:  # every rank's last exchange into a peer's memory has completed
        dist.barrier()
    moe.close()
    del moe
    # the same bytes per launch read by a pure 16-byte-load kernel as two
    # dependent launches (the ffn1 / ffn2 split): the achievable floor at this
    # launch size, next to the HBM peak
    if rank == 0 and roofline["bytes_per_launch"] > 0:
        nb = int(roofline["bytes_per_launch"]) // 256 * 256
        n_buf = max(2, int(600e6 // nb) + 1)
        rbuf = torch.empty(n_buf * nb, dtype=torch.uint8, device="cuda")
        rms = C.c_float()
        _lib.check(lib.hm_bench_stream_read(rbuf.data_ptr(), nb, n_buf, 1, 4, 20, st.cuda_stream, C.byref(rms)))
        floor_gbs = nb / (rms.value * 1e-3) / 1e9
        roofline["read_floor"] = {"gbs": floor_gbs, "frac_of_floor": roofline["achieved"] / floor_gbs,
                                  "what": "bytes_per_launch read by a pure 16-byte-load kernel as two dependent "
                                          "launches (2/3 + 1/3: the ffn1 / ffn2 split), back to back over "
                                          "rotating buffers (hm_bench_stream_read)"}
        del rbuf
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # rank 0 at N=1 only
        cpu = cpu_reference_decode(args.shape, args.cpu_baseline_steps, 1, prefill=0)

    # ---- per-rank parity, gathered
    if dist:
        allp = [None] * world
        dist.all_gather_object(allp, parity)
        parity = {"per_rank": allp}
    if live_fixture and rank == 0:
        write_live_fixture(args, cfg, prof, fixture_records, fixture_requests, trace)

    if rank == 0:
        line = {
            "metric": "decode tok/s at 25% expert-cache budget", "value": tok_s, "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if args.bits == 16 else "int4 weights, bf16 activations",
            "data": "synthetic (reference trace-generator routing GenParams(1.0,0.85,0.6), random-init N(0,0.02^2) "
                    "bf16 weights)",
            "config": {"workload": f"{args.shape}-shaped MoE decode, batch 1, {args.ratio:.0%} expert-cache budget",
                       "shape": args.shape, "layers": cfg.num_layers, "experts": cfg.num_routed,
                       "top_k": cfg.num_activated, "hidden": H, "inter": I, "cache_slots": moe_capacity(cfg, args),
                       "host_images": host_images, "policy": args.policy, "prefetch": args.prefetch,
                       "predict": args.predict, "scheduling": args.scheduling,
                       "l2": f"each step streams {cfg.num_layers * cfg.num_activated} expert evaluations x "
                             f"{image_bytes / 1e6:.1f} MB of weights (>> 126 MB L2); no flush needed",
                       "parallelism": f"ep{world}" if world > 1 else "single", "weight_bits": args.bits,
                       "ep_exchange": (exchange_note or args.exchange) if world > 1 else "none"},
            "prefill": {"tokens": args.prefill, "ms": prefill_ms, "cold_cache": True,
                        "gpu_experts": sum(s.n_gpu for s in pst), "cpu_experts": sum(s.n_cpu for s in pst),
                        "transfers": sum(s.n_transfer for s in pst)},
            "e2e": {"value": 1e3 / e2e_ms, "unit": "tok/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": roofline,
            "gemm_roofline": gemm_roofline,
            "h2d_roofline": h2d_roofline,
            "step_roofline": {"bound": "plan-conditional max(B_gpu/HBM, B_cpu/host DRAM, B_h2d/PCIe)",
                              "bound_ms_per_step": 1e3 * bound_s / args.steps,
                              "frac": (1e3 * bound_s / args.steps) / ms_step, "host_bw_gbs": host_bw_gbs,
                              "host_read_probe_gbs": host_probe_gbs, "host_worker_gbs": worker_gbs,
                              "pcie_gbs": bw_pcie / 1e9},
            "per_step": {"gpu_experts": n_gpu, "cpu_experts": n_cpu, "transfers": n_xfer,
                         "host_decide_us_per_layer": statistics.mean(s.t_decide_us for s in stats_all),
                         "host_wait_router_us_per_layer": statistics.mean(s.t_wait_router_us for s in stats_all),
                         "cpu_worker_ms": sum(s.t_cpu_us for s in stats_all) / 1e3 / args.steps},
            "profile": {k: getattr(base_profile, k) for k in ("gpu_time_per_expert", "cpu_slope",
                                                               "transfer_bandwidth", "transfer_latency", "gpu_slope",
                                                               "cpu_first_expert_penalty")},
            "prefill_profile": {k: getattr(prefill_profile, k) for k in ("gpu_time_per_expert", "cpu_slope",
                                                                          "gpu_slope", "cpu_first_expert_penalty")},
            "model_vs_measured": model_check,
            "decode_refit": refit,
            "non_expert": dict(non_expert, **{
                "tbt_ms_with_non_expert": ms_step + cfg.num_layers * non_expert["decode_us_per_layer"] / 1e3,
                "ttft_ms_with_non_expert": prefill_ms + cfg.num_layers * non_expert["prefill_us_per_layer"] / 1e3,
                "predicted_tbt_ms_with_non_expert": statistics.mean(predicted)
                + cfg.num_layers * non_expert["decode_us_per_layer"] / 1e3}),
            "decision_path_baseline": decision_baseline,
            "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clocks.summary(), "parity": parity,
            "setup_s": setup_s,
        }
        if world == 1 and args.extra_configs:
            line["configs"] = run_extra_configs(args)
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


EXTRA_CONFIGS = {  # BASELINE.json configs 3-4: DeepSeek-V2-Lite at 25 %, Qwen2-57B-A14B budget sweep 10/25/50 %;
    # plus the headline shape with the paper's 4-bit experts
    "mixtral_25_q4": ["--shape", "mixtral", "--ratio", "0.25", "--bits", "4"],
    "deepseek_25": ["--shape", "deepseek", "--ratio", "0.25"],
    "qwen2_25": ["--shape", "qwen2", "--ratio", "0.25", "--host-images", "192"],
    "qwen2_10": ["--shape", "qwen2", "--ratio", "0.10", "--host-images", "192"],
    "qwen2_50": ["--shape", "qwen2", "--ratio", "0.50", "--host-images", "192"],
}


def run_extra_configs(args) -> dict:
    """The other named configs, each a child bench.py run (own process: the
    Mixtral run's pinned host store is released), summarised into this line so
    the driver's record carries them; a failure is recorded, never fatal."""
    out = {}
    for name in args.extra_configs.split(","):
        if name not in EXTRA_CONFIGS:
            out[name] = {"error": "unknown config"}
            continue
        cmd = [sys.executable, str(Path(__file__).resolve()), "--steps", "4", "--warmup", "3", "--no-cpu-baseline",
               "--extra-configs", ""] + EXTRA_CONFIGS[name]
        t0 = time.time()
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
            rows = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            if r.returncode != 0 or not rows:
                out[name] = {"error": f"rc={r.returncode}: {r.stderr[-300:]}"}
                continue
            d = json.loads(rows[-1])
            out[name] = {"decode_tok_s": d["value"], "e2e_tok_s": d["e2e"]["value"], "ms_per_step": d["ms_per_step"],
                         "prefill_ms": d["prefill"]["ms"], "prefill_tokens": d["prefill"]["tokens"],
                         "config": d["config"], "per_step": d["per_step"], "roofline": d["roofline"],
                         "step_roofline": d["step_roofline"], "model_vs_measured": d["model_vs_measured"],
                         "parity": d["parity"], "clocks": d["clocks"], "gpu_launches": d["gpu_launches"],
                         "decode_refit": d.get("decode_refit"), "h2d_roofline": d.get("h2d_roofline"),
                         "steps": d["steps"], "warmup": d["warmup"], "wall_s": time.time() - t0,
                         "argv": EXTRA_CONFIGS[name]}
        except subprocess.TimeoutExpired:
            out[name] = {"error": "timeout after 300 s"}
    return out


def refit_cpu_decode(stats, prof) -> dict | None:
    """Least-squares fit of t = a + b n over the warm-up layers that ran n >= 1
    experts on the host worker: cpu_slope = b, penalty = 1 + a / b (>= 1)."""
    pts = [(s.n_cpu, s.t_cpu_us * 1e-6) for s in stats if s.n_cpu > 0]
    if len(pts) < 4:
        return None
    n = [p[0] for p in pts]
    t = [p[1] for p in pts]
    mn, mt = statistics.mean(n), statistics.mean(t)
    var = sum((x - mn) ** 2 for x in n)
    if var > 0:
        b = sum((x - mn) * (y - mt) for x, y in zip(n, t)) / var
        a = mt - b * mn
    else:
        b, a = mt / mn, 0.0
    if b <= 0 or a < 0:  # no usable intercept: a plain per-expert average
        b, a = sum(t) / sum(n), 0.0
    return {"cpu_slope": b, "cpu_first_expert_penalty": 1.0 + a / b, "layers": len(pts),
            "calibrated_cpu_slope": prof.cpu_slope, "calibrated_penalty": prof.cpu_first_expert_penalty,
            "what": "host-worker cost refitted on the warm-up decode passes' measured per-layer worker times; "
                    "the timed passes are planned with it"}


def moe_capacity(cfg, args) -> int:
    from paper_2504_05897_b200.engine import cache_capacity
    return cache_capacity(cfg, args.ratio)


def write_live_fixture(args, cfg, prof, records, requests, trace) -> None:
    """Live-run decision fixture of THIS bench configuration: the prefill and
    warm-up decode passes' LayerRequests (from the GPU router) in the
    reference's trace format, the profile the runtime planned with, and the
    SHA-256 of the runtime's decision stream (tests/test_live_fixture.py
    replays it through the unmodified reference run_trace)."""
    import tempfile

    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    from stream import digest, from_records

    from paper_2504_05897_b200 import core as mcore
    from paper_2504_05897_b200.tracegen import save_trace
    passes = []
    for i, reqs in enumerate(requests):
        fwd = trace.passes[i]
        passes.append(mcore.ForwardPass(fwd.stage, fwd.token_count, tuple(
            mcore.make_layer_request(l, list(map(int, lo)), list(map(float, sc))) for l, (lo, sc) in enumerate(reqs))))
    live = mcore.Trace(cfg, tuple(passes), {"source": f"live B200 run, bench.py --shape {args.shape} "
                                                      f"--ratio {args.ratio} (GPU router on generator logits)"})
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "t.jsonl"
        save_trace(live, f)
        text = f.read_text()
    import torch
    out = {"policy": args.policy, "prefetch": args.prefetch, "ratio": args.ratio, "seed": args.seed,
           "profile": {k: getattr(prof, k) for k in prof.__dataclass_fields__}, "trace_jsonl": text,
           "runtime_stream_sha256": digest(from_records(records, args.policy == "mrs")),
           "gpu": torch.cuda.get_device_name(0)}
    Path(args.live_fixture).parent.mkdir(parents=True, exist_ok=True)
    Path(args.live_fixture).write_text(json.dumps(out))


def spawn_ranks(argv: list[str], n: int) -> int:
    """`bench.py --gpus N` launched without torchrun: start N ranks (one per GPU) itself."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init log (communicator ranks) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + argv
    return subprocess.call(cmd, env=env)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--shape", default="mixtral", choices=["tiny", "mixtral", "deepseek", "qwen2"])
    ap.add_argument("--ratio", type=float, default=0.25)
    ap.add_argument("--bits", type=int, default=16, choices=[16, 4],
                    help="expert weights: bf16 (BASELINE config) or the paper's 4-bit (int4 g128)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "dispatch", "nccl_a2a", "allreduce"],
                    help="expert parallelism: replicated tokens + fused peer-memory reduce (p2p), token-sharded "
                         "all-to-all dispatch/return over peer memory (dispatch) or over NCCL grouped send/recv "
                         "(nccl_a2a), or replicated + NCCL all-reduce (allreduce)")
    ap.add_argument("--prefill", type=int, default=1024)
    ap.add_argument("--policy", default="mrs", choices=["mrs", "lru", "lfu"])
    ap.add_argument("--scheduling", default="hybrid",
                    choices=["hybrid", "static_layer_split", "fixed_frequency_map", "gpu_ondemand"])
    ap.add_argument("--prefetch", action="store_true")
    ap.add_argument("--predict", default="trace", choices=["trace", "live"],
                    help="prefetch predictions: the reference's trace-mode model, or the live gate look-ahead "
                         "(future layers' gates on the current hidden state, one kernel per layer)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--host-images", type=int, default=None)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--host-bw-gbs", type=float, default=0.0, help="<= 0: measure")
    ap.add_argument("--cpu-baseline-steps", type=int, default=3,
                    help="decode tokens of the bounded CPU-baseline sample in our arm's line")
    ap.add_argument("--ref-prefill", action=argparse.BooleanOptionalAction, default=True,
                    help="reference arm: also time one all-CPU prefill of --prefill tokens")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--live-fixture", default=None,
                    help="write a live-run decision fixture (prefill + warm-up passes) to this path")
    ap.add_argument("--profile-file", default=None, help="HardwareProfile key=value file instead of calibrating")
    ap.add_argument("--save-profile", default=None, help="write the calibrated HardwareProfile here")
    ap.add_argument("--prefill-profile-file", default=None)
    ap.add_argument("--extra-configs", default="deepseek_25,qwen2_10,qwen2_25,qwen2_50,mixtral_25_q4",
                    help="comma list of other named configs run as child processes after the headline one "
                         "and summarised under 'configs' ('' = none)")
    ap.add_argument("--refit", action=argparse.BooleanOptionalAction, default=True,
                    help="refit the host-worker decode cost on the warm-up passes before the timed ones")
    ap.add_argument("--stage-profiles", action=argparse.BooleanOptionalAction, default=True,
                    help="calibrate a separate prefill-load profile for the prefill pass")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
