"""Intra-layer hybrid CPU/GPU/PCIe scheduler (drop-in for ``moesim.scheduling``).

All plan construction runs in the native decision core (include/hybrimoe.h,
scheduling section): the greedy three-timeline fill (scheduling.py:160-270),
the two degenerate guard plans (273-317), best-of-three selection (320-350),
plan validation (80-124) and the memoised makespan evaluator (433-465).  This
module only converts between the reference's Python types and flat arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, NamedTuple

import numpy as np

from . import _lib
from ._lib import check, lib, pack
from .core import CacheState, ExpertRef, LayerRequest, _ref_of
from .costs import HardwareProfile, to_native
from .errors import PlanInvariantError

DEVICE_CPU = "cpu"
DEVICE_GPU = "gpu"
DEVICE_PCIE = "pcie"
KIND_COMPUTE = "compute"
KIND_TRANSFER = "transfer"
ASSIGN_CPU = "cpu"
ASSIGN_GPU_CACHED = "gpu_cached"
ASSIGN_GPU_TRANSFER = "gpu_after_transfer"
_TIE_ORDER = {DEVICE_PCIE: 0, DEVICE_GPU: 1, DEVICE_CPU: 2}
ORACLE_LIMIT = 12

_DEV_NAME = {_lib.DEV_CPU: DEVICE_CPU, _lib.DEV_GPU: DEVICE_GPU, _lib.DEV_PCIE: DEVICE_PCIE}
_DEV_CODE = {v: k for k, v in _DEV_NAME.items()}
_KIND_NAME = {_lib.KIND_COMPUTE: KIND_COMPUTE, _lib.KIND_TRANSFER: KIND_TRANSFER}
_KIND_CODE = {v: k for k, v in _KIND_NAME.items()}
_ASSIGN_NAME = {_lib.ASSIGN_CPU: ASSIGN_CPU, _lib.ASSIGN_GPU_CACHED: ASSIGN_GPU_CACHED,
                _lib.ASSIGN_GPU_TRANSFER: ASSIGN_GPU_TRANSFER}
_ASSIGN_CODE = {v: k for k, v in _ASSIGN_NAME.items()}


class ExpertTask(NamedTuple):
    ref: ExpertRef
    load: int


class TimelineEvent(NamedTuple):
    device: str
    expert: ExpertRef
    kind: str
    start: float
    end: float


@dataclass(frozen=True)
class SchedulePlan:
    """Committed layer schedule (scheduling.py:61-73)."""

    events: tuple[TimelineEvent, ...]
    assignment: dict[ExpertRef, str]
    makespan: float

    def compute_events(self) -> list[TimelineEvent]:
        return [e for e in self.events if e.kind == KIND_COMPUTE]

    def transfer_events(self) -> list[TimelineEvent]:
        return [e for e in self.events if e.kind == KIND_TRANSFER]


# ---------------------------------------------------------------- marshalling


def _tasks(tasks: Iterable[ExpertTask]):
    ts = list(tasks)
    arr = (_lib.Task * max(1, len(ts)))()
    for i, t in enumerate(ts):
        layer, expert = t[0]
        arr[i].ref = pack(int(layer), int(expert))
        arr[i].load = int(t[1])
    return arr, len(ts)


def plan_from_native(ev, n_ev: int, asg, n_as: int, makespan: float) -> SchedulePlan:
    events = tuple(TimelineEvent(_DEV_NAME[ev[i].device], _ref_of(ev[i].ref), _KIND_NAME[ev[i].kind],
                                 ev[i].start, ev[i].end) for i in range(n_ev))
    assignment = {_ref_of(asg[i].ref): _ASSIGN_NAME[asg[i].how] for i in range(n_as)}
    return SchedulePlan(events=events, assignment=assignment, makespan=makespan)


def _plan_call(fn, n_tasks: int, *args) -> SchedulePlan:
    ev = (_lib.Event * max(1, 2 * n_tasks))()
    asg = (_lib.Assign * max(1, n_tasks))()
    n_ev, n_as, mk = C.c_int(), C.c_int(), C.c_double()
    check(fn(*args, ev, C.byref(n_ev), asg, C.byref(n_as), C.byref(mk)))
    return plan_from_native(ev, n_ev.value, asg, n_as.value, mk.value)


def _plan_to_native(plan: SchedulePlan):
    n_ev, n_as = len(plan.events), len(plan.assignment)
    ev = (_lib.Event * max(1, n_ev))()
    for i, e in enumerate(plan.events):
        ev[i].device = _DEV_CODE[e.device]
        ev[i].kind = _KIND_CODE[e.kind]
        ev[i].ref = pack(*e.expert)
        ev[i].start, ev[i].end = float(e.start), float(e.end)
    asg = (_lib.Assign * max(1, n_as))()
    for i, (ref, how) in enumerate(plan.assignment.items()):
        asg[i].ref = pack(*ref)
        asg[i].how = _ASSIGN_CODE[how]
    return ev, n_ev, asg, n_as


# ------------------------------------------------------------------ the API


def check_plan(plan: SchedulePlan) -> None:
    """Per-device non-overlap, transfer-before-compute, one compute per expert,
    makespan = latest end (scheduling.py:80-124); raises PlanInvariantError."""
    if any(e.device not in _DEV_CODE or e.kind not in _KIND_CODE for e in plan.events):
        raise PlanInvariantError("unknown device or kind in plan")
    ev, n_ev, asg, n_as = _plan_to_native(plan)
    check(lib.hm_check_plan(ev, n_ev, asg, n_as, float(plan.makespan)))


def activated_tasks(request: LayerRequest) -> list[ExpertTask]:
    """(ref, load) of every activated expert in ref order (scheduling.py:127-132)."""
    return [ExpertTask(ExpertRef(request.layer, i), request.loads[i]) for i in sorted(request.activated)]


def build_queues(request: LayerRequest, cache) -> tuple[list[ExpertTask], list[ExpertTask]]:
    """GPU queue: cached, (-load, ref); CPU queue: uncached, (load, ref) (scheduling.py:135-147)."""
    tasks = activated_tasks(request)
    res = cache.resident
    gpu_q = sorted((t for t in tasks if t.ref in res), key=lambda t: (-t.load, t.ref))
    cpu_q = sorted((t for t in tasks if t.ref not in res), key=lambda t: (t.load, t.ref))
    return gpu_q, cpu_q


def simulate_schedule(gpu_queue: Iterable[ExpertTask], cpu_queue: Iterable[ExpertTask],
                      profile: HardwareProfile, expert_size_bytes: float) -> SchedulePlan:
    """Greedy three-timeline fill (scheduling.py:160-270), native."""
    g, ng = _tasks(gpu_queue)
    c, nc = _tasks(cpu_queue)
    return _plan_call(lib.hm_simulate_schedule, ng + nc, g, ng, c, nc, C.byref(to_native(profile)),
                      float(expert_size_bytes))


def plan_all_cpu(tasks: Iterable[ExpertTask], profile: HardwareProfile) -> SchedulePlan:
    t, n = _tasks(tasks)
    return _plan_call(lib.hm_plan_all_cpu, n, t, n, C.byref(to_native(profile)))


def plan_all_gpu(cached: Iterable[ExpertTask], uncached: Iterable[ExpertTask], profile: HardwareProfile,
                 expert_size_bytes: float) -> SchedulePlan:
    c, nc = _tasks(cached)
    u, nu = _tasks(uncached)
    return _plan_call(lib.hm_plan_all_gpu, nc + nu, c, nc, u, nu, C.byref(to_native(profile)),
                      float(expert_size_bytes))


def _select_plan_tasks(cached, uncached, profile, expert_size_bytes) -> SchedulePlan:
    c, nc = _tasks(cached)
    u, nu = _tasks(uncached)
    return _plan_call(lib.hm_select_plan_tasks, nc + nu, c, nc, u, nu, C.byref(to_native(profile)),
                      float(expert_size_bytes))


def select_plan(request: LayerRequest, cache, profile: HardwareProfile, expert_size_bytes: float) -> SchedulePlan:
    """Best of greedy / all-CPU / all-GPU, ties keep greedy (scheduling.py:338-350)."""
    if isinstance(cache, CacheState) and all((v > 0) == (i in request.activated)
                                             for i, v in enumerate(request.loads)):
        loads = np.ascontiguousarray(request.loads, dtype=np.int64)
        n = len(loads)
        return _plan_call(lib.hm_select_plan, n, cache._h, int(request.layer), _lib.ptr(loads, C.c_int64), n,
                          C.byref(to_native(profile)), float(expert_size_bytes))
    gpu_q, cpu_q = build_queues(request, cache)
    return _select_plan_tasks(gpu_q, cpu_q, profile, expert_size_bytes)


def oracle_optimal(request: LayerRequest, cache, profile: HardwareProfile, expert_size_bytes: float,
                   limit: int = ORACLE_LIMIT) -> float:
    """Exhaustive minimum makespan (scheduling.py:356-402); test oracle."""
    tasks = activated_tasks(request)
    t, n = _tasks(tasks)
    res = cache.resident
    cached = (C.c_uint8 * max(1, n))(*[1 if x.ref in res else 0 for x in tasks])
    out = C.c_double()
    check(lib.hm_oracle_optimal(t, n, cached, C.byref(to_native(profile)), float(expert_size_bytes),
                                int(limit), C.byref(out)))
    return out.value


def pcie_idle_budget(plan: SchedulePlan) -> float:
    """max(0, makespan - sum of transfer durations) (scheduling.py:405-412)."""
    ev, n_ev, _, _ = _plan_to_native(SchedulePlan(plan.events, {}, plan.makespan))
    out = C.c_double()
    check(lib.hm_pcie_idle_budget(ev, n_ev, float(plan.makespan), C.byref(out)))
    return out.value


def device_busy(plan: SchedulePlan) -> dict[str, float]:
    busy = {DEVICE_CPU: 0.0, DEVICE_GPU: 0.0, DEVICE_PCIE: 0.0}
    for ev in plan.events:
        busy[ev.device] += ev.end - ev.start
    return busy


def format_plan(plan: SchedulePlan) -> str:
    """One event per line: device layer expert kind start end (scheduling.py:422-430)."""
    return "\n".join(f"{e.device}\t{e.expert.layer}\t{e.expert.expert}\t{e.kind}\t{e.start:.6f}\t{e.end:.6f}"
                     for e in plan.events)


class MakespanEvaluator:
    """Memoised select-plan makespans keyed by load multisets (scheduling.py:433-465), native."""

    def __init__(self, profile: HardwareProfile, expert_size_bytes: float) -> None:
        self.profile = profile
        self.expert_size_bytes = expert_size_bytes
        h = C.c_void_p()
        check(lib.hm_evaluator_create(C.byref(to_native(profile)), float(expert_size_bytes), C.byref(h)))
        self._h = h.value

    def __del__(self) -> None:
        if getattr(self, "_h", None):
            lib.hm_evaluator_destroy(self._h)
            self._h = None

    def __len__(self) -> int:
        v = C.c_int64()
        check(lib.hm_evaluator_size(self._h, C.byref(v)))
        return v.value

    def makespan(self, cached_loads: Iterable[int], uncached_loads: Iterable[int]) -> float:
        c = np.ascontiguousarray(list(cached_loads), dtype=np.int64)
        u = np.ascontiguousarray(list(uncached_loads), dtype=np.int64)
        out = C.c_double()
        check(lib.hm_evaluator_makespan(self._h, _lib.ptr(c, C.c_int64), len(c), _lib.ptr(u, C.c_int64), len(u),
                                        C.byref(out)))
        return out.value

    def makespan_for_request(self, request: LayerRequest, resident) -> float:
        cached, uncached = [], []
        for i in sorted(request.activated):
            (cached if ExpertRef(request.layer, i) in resident else uncached).append(request.loads[i])
        return self.makespan(cached, uncached)
