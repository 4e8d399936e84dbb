"""Per-layer orchestration (drop-in for ``moesim.engine``).

``run_pass`` / ``run_trace`` keep the reference's signatures and results
(engine.py:255-486), but every per-layer step -- lookups, pinning, plan
selection, demand inserts, MRS update, prefetch gain evaluation / selection /
inserts, pin expiry -- executes inside one native call (``hm_engine_run_layer``)
in the exact engine.py:288-389 order.  Python only supplies the predicted
requests of the prediction model (numpy RNG, prefetch.py:54-101) and
aggregates metrics with the reference's float summation order.

``decision_log=True`` additionally returns, per (pass, layer), the record the
parity tests compare bit-for-bit against the reference.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib, pack
from .caching import POLICIES, POLICY_CODE, POLICY_MRS, CacheStats, MrsState, make_mrs_state
from .core import CacheState, ExpertRef, LayerRequest, ModelConfig, STAGE_PREFILL, Trace, _ref_of, expert_bytes
from .costs import HardwareProfile, gpu_time, to_native, transfer_time
from .prefetch import PredictionModel, predict_layers, predict_layers_native
from .scheduling import (ASSIGN_GPU_CACHED, DEVICE_CPU, DEVICE_GPU, DEVICE_PCIE, KIND_COMPUTE, MakespanEvaluator,
                         SchedulePlan, TimelineEvent, activated_tasks, plan_all_cpu, plan_from_native)

SCHED_HYBRID = "hybrid"
SCHED_STATIC_SPLIT = "static_layer_split"
SCHED_FIXED_MAP = "fixed_frequency_map"
SCHED_GPU_ONDEMAND = "gpu_ondemand"
SCHEDULINGS = (SCHED_HYBRID, SCHED_STATIC_SPLIT, SCHED_FIXED_MAP, SCHED_GPU_ONDEMAND)
_STATIC_SCHEDULINGS = (SCHED_STATIC_SPLIT, SCHED_FIXED_MAP)
_SCHED_CODE = {SCHED_HYBRID: 0, SCHED_STATIC_SPLIT: 1, SCHED_FIXED_MAP: 2, SCHED_GPU_ONDEMAND: 3}


@dataclass(frozen=True)
class EnginePolicy:
    """Scheduling, cache policy and prefetch settings of one run (engine.py:76-103)."""

    scheduling: str = SCHED_HYBRID
    cache_policy: str = POLICY_MRS
    prefetch: bool = False
    prediction: PredictionModel = field(default_factory=PredictionModel)
    static_split_point: int | None = None
    pin_top_fraction: float | None = None
    mrs_alpha: float = 0.5
    mrs_p: int | None = None
    calibration_prefix_fraction: float = 0.1
    validate: bool = False

    def __post_init__(self) -> None:
        if self.scheduling not in SCHEDULINGS:
            raise ValueError(f"unknown scheduling {self.scheduling!r}")
        if self.cache_policy not in POLICIES:
            raise ValueError(f"unknown cache policy {self.cache_policy!r}")
        if self.pin_top_fraction is not None and not 0.0 <= self.pin_top_fraction <= 1.0:
            raise ValueError(f"pin_top_fraction must be in [0, 1], got {self.pin_top_fraction}")
        if not 0.0 < self.calibration_prefix_fraction <= 1.0:
            raise ValueError("calibration_prefix_fraction must be in (0, 1]")
        if self.prefetch and self.scheduling in _STATIC_SCHEDULINGS:
            raise ValueError(f"prefetch is meaningless with {self.scheduling} (fixed residency)")
        if not 0.0 <= self.mrs_alpha <= 1.0:
            raise ValueError(f"mrs_alpha must be in [0, 1], got {self.mrs_alpha}")


@dataclass
class RunMetrics:
    """Aggregated outcome of one run (engine.py:106-156)."""

    ttft: float | None
    tbt: tuple[float, ...]
    cache: CacheStats
    device_busy: dict[str, float]
    device_idle: dict[str, float]
    prefetch_issued: int
    prefetch_hits: int
    prefetch_expired: int
    elapsed: float
    plans: list[SchedulePlan] | None = None
    decisions: list[dict] | None = None

    @property
    def mean_tbt(self) -> float | None:
        return sum(self.tbt) / len(self.tbt) if self.tbt else None

    @property
    def median_tbt(self) -> float | None:
        if not self.tbt:
            return None
        v = sorted(self.tbt)
        m = len(v) // 2
        return v[m] if len(v) % 2 else (v[m - 1] + v[m]) / 2

    @property
    def hit_rate(self) -> float | None:
        return self.cache.hits / self.cache.lookups if self.cache.lookups else None

    def to_record(self) -> dict:
        total = self.elapsed if self.elapsed > 0 else 1.0
        return {
            "ttft": self.ttft, "mean_tbt": self.mean_tbt, "median_tbt": self.median_tbt,
            "decode_passes": len(self.tbt), "hit_rate": self.hit_rate, "lookups": self.cache.lookups,
            "hits": self.cache.hits, "inserts": self.cache.inserts, "evictions": self.cache.evictions,
            "gpu_util": self.device_busy[DEVICE_GPU] / total, "cpu_util": self.device_busy[DEVICE_CPU] / total,
            "pcie_util": self.device_busy[DEVICE_PCIE] / total, "prefetch_issued": self.prefetch_issued,
            "prefetch_hits": self.prefetch_hits, "prefetch_expired": self.prefetch_expired,
            "elapsed": self.elapsed,
        }


@dataclass
class PassResult:
    latency: float
    layer_makespans: list[float]
    cache_stats: CacheStats
    busy: dict[str, float]
    prefetch_issued: int = 0
    prefetch_hits: int = 0
    prefetch_expired: int = 0
    plans: list[SchedulePlan] | None = None
    decisions: list[dict] | None = None


# ------------------------------------------------------------------ baselines
# The planners of the comparison baselines (engine.py:171-231).  The engine
# runs them natively; these Python entry points exist for API parity.


def static_layer_split_plan(request: LayerRequest, profile: HardwareProfile, split_point: int) -> SchedulePlan:
    """GPU below the split (serial, load-descending), CPU above (engine.py:185-192)."""
    return _single_layer_plan(request, profile, SCHED_STATIC_SPLIT, split_point=split_point)


def fixed_frequency_map_plan(request: LayerRequest, pinned_set, profile: HardwareProfile) -> SchedulePlan:
    """Pinned experts on the GPU, the rest on the CPU, no transfers (engine.py:195-205)."""
    return _single_layer_plan(request, profile, SCHED_FIXED_MAP, fixed=pinned_set)


def _single_layer_plan(request, profile, scheduling, split_point=0, fixed=frozenset()) -> SchedulePlan:
    n = len(request.loads)
    cfg = ModelConfig(num_layers=request.layer + 1, num_routed=n, num_shared=0, num_activated=1,
                      routed_expert_dims=(1, 1), bytes_per_weight=1.0)
    eng = _NativeEngine(cfg, EnginePolicy(scheduling=scheduling), CacheState(0), None,
                        MakespanEvaluator(profile, 3.0), profile, split_point, fixed, collect=True)
    eng.begin_pass()
    eng.run_layer(request, [])
    plan = eng.plan()
    eng.end_pass()
    return plan


def compute_fixed_pinned_set(trace: Trace, capacity: int, prefix_fraction: float,
                             pin_top_fraction: float | None) -> frozenset[ExpertRef]:
    """Top experts by activation count over a calibration prefix (engine.py:208-231)."""
    n_prefix = max(1, math.floor(prefix_fraction * len(trace.passes)))
    counts: dict[ExpertRef, int] = {}
    for fwd in trace.passes[:n_prefix]:
        for req in fwd.layers:
            for i in req.activated:
                r = ExpertRef(req.layer, i)
                counts[r] = counts.get(r, 0) + 1
    size = capacity
    if pin_top_fraction is not None:
        size = min(capacity, math.floor(pin_top_fraction * trace.config.total_routed_experts))
    cfg = trace.config
    universe = [ExpertRef(l, e) for l in range(cfg.num_layers) for e in range(cfg.num_routed)]
    return frozenset(sorted(universe, key=lambda r: (-counts.get(r, 0), r))[:size])


# --------------------------------------------------------------- native engine


class _NativeEngine:
    """One hm_engine bound to a run's cache / MRS state / evaluator."""

    def __init__(self, config: ModelConfig, policy: EnginePolicy, cache: CacheState, mrs: MrsState | None,
                 evaluator: MakespanEvaluator, profile: HardwareProfile, split_point: int,
                 fixed_pinned, collect: bool) -> None:
        if not isinstance(cache, CacheState):
            raise TypeError("run_pass needs this package's native CacheState")
        if mrs is not None and not isinstance(mrs, MrsState):
            raise TypeError("run_pass needs this package's native MrsState")
        if not isinstance(evaluator, MakespanEvaluator):
            raise TypeError("run_pass needs this package's native MakespanEvaluator")
        self.n = config.num_routed
        self.policy = policy
        self.collect = collect
        cfg = _lib.EngineConfig(
            num_layers=config.num_layers, num_routed=config.num_routed, num_activated=config.num_activated,
            scheduling=_SCHED_CODE[policy.scheduling], cache_policy=POLICY_CODE[policy.cache_policy],
            prefetch=int(policy.prefetch), validate=int(policy.validate), split_point=int(split_point),
            capacity=cache.capacity, expert_bytes=float(expert_bytes(config)), collect=int(collect))
        h = C.c_void_p()
        check(lib.hm_engine_create(C.byref(cfg), C.byref(to_native(profile)), cache._h,
                                   mrs._h if mrs is not None else None, evaluator._h, C.byref(h)))
        self._h = h.value
        self._keep = (cache, mrs, evaluator)  # the engine borrows these
        if fixed_pinned:
            refs = (C.c_uint32 * len(fixed_pinned))(*[pack(*r) for r in fixed_pinned])
            check(lib.hm_engine_set_fixed_pinned(self._h, refs, len(fixed_pinned)))
        self._loads = np.zeros(self.n, dtype=np.int64)
        self._scores = np.zeros(self.n, dtype=np.float64)

    def __del__(self) -> None:
        if getattr(self, "_h", None):
            lib.hm_engine_destroy(self._h)
            self._h = None

    def begin_pass(self) -> None:
        check(lib.hm_engine_begin_pass(self._h))

    def run_layer_arrays(self, layer: int, loads: np.ndarray, scores: np.ndarray, pred_layers: np.ndarray,
                         pred_loads: np.ndarray) -> None:
        check(lib.hm_engine_run_layer(self._h, int(layer), _lib.ptr(loads, C.c_int64), _lib.ptr(scores, C.c_double),
                                      self.n, _lib.ptr(pred_layers, C.c_int32), _lib.ptr(pred_loads, C.c_int64),
                                      len(pred_layers)))

    def run_layer(self, request: LayerRequest, predicted: list[LayerRequest]) -> None:
        loads = self._loads
        loads[:] = 0
        for i in request.activated:
            loads[i] = request.loads[i]
        self._scores[:] = request.scores
        pl = np.array([p.layer for p in predicted], dtype=np.int32)
        pload = np.zeros((max(1, len(predicted)), self.n), dtype=np.int64)
        for d, p in enumerate(predicted):
            for i in p.activated:
                pload[d, i] = p.loads[i]
        self.run_layer_arrays(request.layer, loads, self._scores, pl, pload)

    def _sizes(self) -> _lib.RecordSizes:
        s = _lib.RecordSizes()
        check(lib.hm_engine_record_sizes(self._h, C.byref(s)))
        return s

    def plan(self) -> SchedulePlan:
        s = self._sizes()
        ev = (_lib.Event * max(1, s.n_events))()
        asg = (_lib.Assign * max(1, s.n_assign))()
        check(lib.hm_engine_record(self._h, None, None, ev, asg, None, None, None, None, None, None, None, None))
        return plan_from_native(ev, s.n_events, asg, s.n_assign, s.makespan)

    def record(self) -> dict:
        """The cache-decision record of the last layer."""
        s = self._sizes()
        lr = (C.c_uint32 * max(1, s.n_lookups))()
        lh = (C.c_uint8 * max(1, s.n_lookups))()
        ev = (_lib.Event * max(1, s.n_events))()
        asg = (_lib.Assign * max(1, s.n_assign))()
        dr = (C.c_uint32 * max(1, s.n_demand))()
        dv = (C.c_uint32 * max(1, s.n_demand))()
        dh = (C.c_uint8 * max(1, s.n_demand))()
        cd = (_lib.Candidate * max(1, s.n_candidates))()
        cr = (C.c_uint32 * max(1, s.n_chosen))()
        cv = (C.c_uint32 * max(1, s.n_chosen))()
        ch = (C.c_uint8 * max(1, s.n_chosen))()
        sl = (C.c_uint32 * max(1, s.n_selected))()
        check(lib.hm_engine_record(self._h, lr, lh, ev, asg, dr, dv, dh, cd, cr, cv, ch, sl))
        plan = plan_from_native(ev, s.n_events, asg, s.n_assign, s.makespan)
        return {
            "lookups": [(_ref_of(lr[i]), bool(lh[i])) for i in range(s.n_lookups)],
            "plan": plan,
            "demand_inserts": [(_ref_of(dr[i]), _ref_of(dv[i]) if dh[i] else None) for i in range(s.n_demand)],
            "candidates": [(_ref_of(cd[i].ref), cd[i].predicted_load, cd[i].gain, cd[i].layer_distance)
                           for i in range(s.n_candidates)],
            "budget": s.budget if self.policy.prefetch else None,
            "selected": [_ref_of(sl[i]) for i in range(s.n_selected)],
            "chosen": [(_ref_of(cr[i]), _ref_of(cv[i]) if ch[i] else None) for i in range(s.n_chosen)],
            "prefetch_evict_error": bool(s.prefetch_evict_error),
            "expired": s.expired,
        }

    def end_pass(self) -> _lib.PassResult:
        out = _lib.PassResult()
        check(lib.hm_engine_end_pass(self._h, C.byref(out)))
        return out

    def layer_makespans(self, n_layers: int) -> list[float]:
        buf = (C.c_double * max(1, n_layers))()
        k = C.c_int()
        check(lib.hm_engine_layer_makespans(self._h, buf, n_layers, C.byref(k)))
        return list(buf[: k.value])


def run_pass(trace: Trace, pass_index: int, policy: EnginePolicy, cache: CacheState, profile: HardwareProfile,
             mrs: MrsState | None, seed: int, *, split_point: int = 0, fixed_pinned=frozenset(),
             evaluator: MakespanEvaluator | None = None, collect_plans: bool = False,
             decision_log: bool = False, _engine: _NativeEngine | None = None) -> PassResult:
    """Replay one forward pass; mutates cache and mrs (engine.py:255-398)."""
    fwd = trace.passes[pass_index]
    cfg = trace.config
    size_bytes = expert_bytes(cfg)
    if evaluator is None:
        evaluator = MakespanEvaluator(profile, size_bytes)
    eng = _engine or _NativeEngine(cfg, policy, cache, mrs, evaluator, profile, split_point, fixed_pinned,
                                   collect_plans or decision_log)
    eng.begin_pass()
    predicting = policy.prefetch and policy.scheduling not in _STATIC_SCHEDULINGS and cache.capacity > 0
    plans: list[SchedulePlan] | None = [] if collect_plans else None
    decisions: list[dict] | None = [] if decision_log else None
    pass_loads = (np.ascontiguousarray([r.loads for r in fwd.layers], dtype=np.int64) if predicting else None)
    for request in fwd.layers:
        # the prediction model (prefetch.py:54-101) through its native restatement
        # of numpy's stream; tests/test_predict_native.py pins it to numpy itself
        predicted = (predict_layers_native(fwd.layers, cfg.num_layers, pass_index, request.layer, policy.prediction,
                                           seed, pass_loads) if predicting else [])
        eng.run_layer(request, predicted)
        if collect_plans:
            plans.append(eng.plan())
        if decision_log:
            rec = eng.record()
            rec["layer"] = request.layer
            rec["mrs_row"] = (mrs.table()[request.layer].copy()
                              if mrs is not None and policy.cache_policy == POLICY_MRS else None)
            decisions.append(rec)
    r = eng.end_pass()
    stats = CacheStats(lookups=r.lookups, hits=r.hits, inserts=r.inserts, evictions=r.evictions)
    return PassResult(latency=r.latency, layer_makespans=eng.layer_makespans(cfg.num_layers), cache_stats=stats,
                      busy={DEVICE_CPU: r.busy[0], DEVICE_GPU: r.busy[1], DEVICE_PCIE: r.busy[2]},
                      prefetch_issued=r.prefetch_issued, prefetch_hits=r.prefetch_hits,
                      prefetch_expired=r.prefetch_expired, plans=plans, decisions=decisions)


def cache_capacity(config: ModelConfig, capacity_ratio: float) -> int:
    """floor(ratio * L * N) (engine.py:401-404)."""
    if not 0.0 < capacity_ratio <= 1.0:
        raise ValueError(f"capacity_ratio must be in (0, 1], got {capacity_ratio}")
    return math.floor(capacity_ratio * config.total_routed_experts)


def run_trace(trace: Trace, policy: EnginePolicy, capacity_ratio: float, profile: HardwareProfile, seed: int, *,
              collect_plans: bool = False, decision_log: bool = False) -> RunMetrics:
    """Replay a whole trace under one policy (engine.py:407-486)."""
    cfg = trace.config
    capacity = cache_capacity(cfg, capacity_ratio)
    cache = CacheState(capacity)
    mrs = make_mrs_state(cfg, alpha=policy.mrs_alpha, p=policy.mrs_p)
    evaluator = MakespanEvaluator(profile, expert_bytes(cfg))
    split_point = policy.static_split_point
    if split_point is None:
        split_point = math.floor(capacity_ratio * cfg.num_layers)
    if not 0 <= split_point <= cfg.num_layers:
        raise ValueError(f"static_split_point must be in [0, num_layers], got {split_point}")
    fixed: frozenset[ExpertRef] = frozenset()
    if policy.scheduling == SCHED_FIXED_MAP:
        fixed = compute_fixed_pinned_set(trace, capacity, policy.calibration_prefix_fraction,
                                         policy.pin_top_fraction)
        cache.resident = set(fixed)
    eng = _NativeEngine(cfg, policy, cache, mrs, evaluator, profile, split_point, fixed,
                        collect_plans or decision_log)

    ttft = None
    tbt: list[float] = []
    stats = CacheStats()
    busy = {DEVICE_CPU: 0.0, DEVICE_GPU: 0.0, DEVICE_PCIE: 0.0}
    issued = hits = expired = 0
    elapsed = 0.0
    all_plans: list[SchedulePlan] = []
    all_dec: list[dict] = []
    for p, fwd in enumerate(trace.passes):
        res = run_pass(trace, p, policy, cache, profile, mrs, seed, split_point=split_point, fixed_pinned=fixed,
                       evaluator=evaluator, collect_plans=collect_plans, decision_log=decision_log, _engine=eng)
        elapsed += res.latency
        stats.merge(res.cache_stats)
        for d in busy:
            busy[d] += res.busy[d]
        issued += res.prefetch_issued
        hits += res.prefetch_hits
        expired += res.prefetch_expired
        if fwd.stage == STAGE_PREFILL and ttft is None:
            ttft = res.latency
        elif fwd.stage != STAGE_PREFILL:
            tbt.append(res.latency)
        if collect_plans:
            all_plans.extend(res.plans)
        if decision_log:
            all_dec.extend(res.decisions)
    m = RunMetrics(ttft=ttft, tbt=tuple(tbt), cache=stats, device_busy=busy,
                   device_idle={d: elapsed - busy[d] for d in busy}, prefetch_issued=issued, prefetch_hits=hits,
                   prefetch_expired=expired, elapsed=elapsed)
    if collect_plans:
        m.plans = all_plans
    if decision_log:
        m.decisions = all_dec
    return m
