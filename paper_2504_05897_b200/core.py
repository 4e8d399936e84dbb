"""Domain types of the MoE-layer hot path (drop-in for ``moesim.core``).

Types keep the reference's names, fields and validation (core.py:19-265) so
code written against ``moesim`` runs unchanged.  ``CacheState`` is backed by
the native cache (include/hybrimoe.h ``hm_cache_*``): its ``resident`` and
``pinned`` attributes are live set views over the C++ state, so the
reference's engine idioms (``ref in cache.resident``, ``cache.pinned |= s``,
``cache.pinned.discard(r)``) operate on the native object directly.
"""
from __future__ import annotations

import ctypes as C
import math
from collections.abc import Mapping, MutableSet, Set
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple

from . import _lib
from ._lib import check, lib, pack

STAGE_PREFILL = "prefill"
STAGE_DECODE = "decode"
STAGES = (STAGE_PREFILL, STAGE_DECODE)
SCORE_SUM_TOL = 1e-9  # core.py:23-24


class ExpertRef(NamedTuple):
    """(layer, expert); tuple order is the global tie-break (core.py:27-36)."""

    layer: int
    expert: int


def _ref_of(packed: int) -> ExpertRef:
    return ExpertRef(packed >> 16, packed & 0xFFFF)


@dataclass(frozen=True)
class ModelConfig:
    """Static MoE shape (core.py:39-81); bytes_per_weight may be fractional."""

    num_layers: int
    num_routed: int
    num_shared: int
    num_activated: int
    routed_expert_dims: tuple[int, int]
    shared_expert_dims: tuple[int, int] | None = None
    bytes_per_weight: float = 0.5

    def __post_init__(self) -> None:
        checks = [
            (self.num_layers >= 1, f"num_layers must be >= 1, got {self.num_layers}"),
            (self.num_routed >= 1, f"num_routed must be >= 1, got {self.num_routed}"),
            (1 <= self.num_activated <= self.num_routed,
             f"num_activated must be in [1, num_routed], got {self.num_activated} "
             f"with num_routed={self.num_routed}"),
            (self.num_shared >= 0, f"num_shared must be >= 0, got {self.num_shared}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        h, i = self.routed_expert_dims
        if h < 1 or i < 1:
            raise ValueError(f"expert dims must be >= 1, got {self.routed_expert_dims}")
        if self.shared_expert_dims is not None and min(self.shared_expert_dims) < 1:
            raise ValueError(f"shared dims must be >= 1, got {self.shared_expert_dims}")
        if self.bytes_per_weight <= 0:
            raise ValueError(f"bytes_per_weight must be > 0, got {self.bytes_per_weight}")

    @property
    def total_routed_experts(self) -> int:
        return self.num_layers * self.num_routed


def expert_bytes(config: ModelConfig) -> float:
    """3 * hidden * intermediate * bytes_per_weight (core.py:84-91)."""
    h, i = config.routed_expert_dims
    return 3 * h * i * config.bytes_per_weight


def rank_by_score(scores: Iterable[float]) -> list[int]:
    """Indices by score descending, lower index first on ties (core.py:94-97)."""
    s = list(scores)
    return sorted(range(len(s)), key=lambda i: (-s[i], i))


@dataclass(frozen=True)
class LayerRequest:
    """One layer's work in one pass (core.py:100-112)."""

    layer: int
    loads: tuple[int, ...]
    scores: tuple[float, ...]
    activated: frozenset[int]


def make_layer_request(layer: int, loads: Iterable[int], scores: Iterable[float]) -> LayerRequest:
    lt = tuple(int(v) for v in loads)
    st = tuple(float(v) for v in scores)
    return LayerRequest(layer=layer, loads=lt, scores=st,
                        activated=frozenset(i for i, v in enumerate(lt) if v > 0))


@dataclass(frozen=True)
class ForwardPass:
    stage: str
    token_count: int
    layers: tuple[LayerRequest, ...]


@dataclass(frozen=True)
class Trace:
    config: ModelConfig
    passes: tuple[ForwardPass, ...]
    metadata: dict[str, str] = field(default_factory=dict)


@dataclass(frozen=True)
class Violation:
    pass_index: int
    layer: int
    rule: str
    detail: str

    def __str__(self) -> str:
        return f"pass {self.pass_index} layer {self.layer}: {self.rule}: {self.detail}"


def _request_violations(cfg: ModelConfig, p: int, fwd: ForwardPass, req: LayerRequest) -> list[Violation]:
    """Trace invariants of one request (core.py:153-209)."""
    out: list[Violation] = []
    n = cfg.num_routed

    def add(rule: str, detail: str) -> None:
        out.append(Violation(p, req.layer, rule, detail))

    if len(req.loads) != n:
        add("loads-length", f"expected {n} entries, got {len(req.loads)}")
        return out
    if len(req.scores) != n:
        add("scores-length", f"expected {n} entries, got {len(req.scores)}")
        return out
    if min(req.loads) < 0:
        add("negative-load", f"loads={req.loads}")
    nz = frozenset(i for i, v in enumerate(req.loads) if v > 0)
    if nz != req.activated:
        add("activated-load-mismatch", f"activated={sorted(req.activated)} but loads>0 at {sorted(nz)}")
    if min(req.scores) < 0:
        add("negative-score", "scores must be nonnegative")
    total = math.fsum(req.scores)
    if abs(total - 1.0) > SCORE_SUM_TOL:
        add("score-normalization", f"scores sum to {total!r}")
    k = len(req.activated)
    if 0 < k <= n:
        top = set(rank_by_score(req.scores)[:k])
        if top != set(req.activated):
            add("activated-not-top-scores", f"activated={sorted(req.activated)} but top-{k} scores at {sorted(top)}")
    if fwd.stage == STAGE_DECODE and fwd.token_count == 1:
        if k != cfg.num_activated:
            add("decode-activated-count", f"expected {cfg.num_activated} activated experts, got {k}")
        if any(req.loads[i] != 1 for i in req.activated):
            add("decode-unit-load", "every activated load must be 1 in single-token decode")
    want = fwd.token_count * cfg.num_activated
    got = sum(req.loads[i] for i in req.activated)
    if got != want:
        add("load-total", f"activated loads sum to {got}, expected token_count*K={want}")
    return out


def validate_trace(trace: Trace) -> list[Violation]:
    """Every trace invariant as data (core.py:212-232)."""
    out: list[Violation] = []
    cfg = trace.config
    for p, fwd in enumerate(trace.passes):
        if fwd.stage not in STAGES:
            out.append(Violation(p, -1, "bad-stage", f"stage={fwd.stage!r}"))
            continue
        if fwd.token_count < 1:
            out.append(Violation(p, -1, "bad-token-count", f"token_count={fwd.token_count}"))
        if len(fwd.layers) != cfg.num_layers:
            out.append(Violation(p, -1, "layer-count", f"expected {cfg.num_layers}, got {len(fwd.layers)}"))
            continue
        for idx, req in enumerate(fwd.layers):
            if req.layer != idx:
                out.append(Violation(p, idx, "layer-order", f"request carries layer={req.layer}"))
                continue
            out.extend(_request_violations(cfg, p, fwd, req))
    return out


# --------------------------------------------------------------------------
# Native cache container


def _members(fn, handle) -> list[int]:
    n = C.c_int64(0)
    check(fn(handle, None, 0, C.byref(n)))
    buf = (C.c_uint32 * max(1, n.value))()
    check(fn(handle, buf, n.value, C.byref(n)))
    return list(buf[: n.value])


def _as_ref(x) -> ExpertRef:
    layer, expert = x
    return ExpertRef(int(layer), int(expert))


class _ResidentView(Set):
    """Live read-only view of CacheState.resident (a set of ExpertRef)."""

    __slots__ = ("_c",)

    def __init__(self, cache: "CacheState") -> None:
        self._c = cache

    def __contains__(self, x) -> bool:
        try:
            r = pack(*_as_ref(x))
        except (TypeError, ValueError):
            return False
        out = C.c_int(0)
        check(lib.hm_cache_is_resident(self._c._h, r, C.byref(out)))
        return bool(out.value)

    def __iter__(self):
        return iter([_ref_of(r) for r in _members(lib.hm_cache_resident, self._c._h)])

    def __len__(self) -> int:
        n = C.c_int64(0)
        check(lib.hm_cache_counts(self._c._h, C.byref(n), None))
        return n.value

    @classmethod
    def _from_iterable(cls, it):
        return set(it)

    def __repr__(self) -> str:
        return f"resident({sorted(self)})"


class _PinnedView(MutableSet):
    """Live mutable view of CacheState.pinned; supports |=, -=, add, discard."""

    __slots__ = ("_c",)

    def __init__(self, cache: "CacheState") -> None:
        self._c = cache

    def __contains__(self, x) -> bool:
        try:
            r = pack(*_as_ref(x))
        except (TypeError, ValueError):
            return False
        out = C.c_int(0)
        check(lib.hm_cache_is_pinned(self._c._h, r, C.byref(out)))
        return bool(out.value)

    def __iter__(self):
        return iter([_ref_of(r) for r in _members(lib.hm_cache_pinned, self._c._h)])

    def __len__(self) -> int:
        n = C.c_int64(0)
        check(lib.hm_cache_counts(self._c._h, None, C.byref(n)))
        return n.value

    def add(self, x) -> None:
        check(lib.hm_cache_pin(self._c._h, pack(*_as_ref(x))))

    def discard(self, x) -> None:
        check(lib.hm_cache_unpin(self._c._h, pack(*_as_ref(x))))

    def clear(self) -> None:
        check(lib.hm_cache_clear_pinned(self._c._h))

    def update(self, items) -> None:
        for x in items:
            self.add(x)

    def difference_update(self, items) -> None:
        for x in items:
            self.discard(x)

    @classmethod
    def _from_iterable(cls, it):
        return set(it)

    def __repr__(self) -> str:
        return f"pinned({sorted(self)})"


class _MetaView(Mapping):
    """LRU ticks / LFU counts of resident experts (core.py:253-254)."""

    __slots__ = ("_c", "_get", "_set")

    def __init__(self, cache: "CacheState", getter, setter) -> None:
        self._c, self._get, self._set = cache, getter, setter

    def _lookup(self, x):
        v, has = C.c_int64(0), C.c_int(0)
        check(self._get(self._c._h, pack(*_as_ref(x)), C.byref(v), C.byref(has)))
        return v.value if has.value else None

    def __getitem__(self, x) -> int:
        v = self._lookup(x)
        if v is None:
            raise KeyError(x)
        return v

    def __setitem__(self, x, v: int) -> None:
        check(self._set(self._c._h, pack(*_as_ref(x)), int(v)))

    def __iter__(self):
        return iter([r for r in self._c.resident if self._lookup(r) is not None])

    def __len__(self) -> int:
        return sum(1 for _ in self)


class CacheState:
    """GPU-resident expert set + pins + policy metadata (core.py:235-265).

    Native: the state lives in C++ (``hm_cache``), which also tracks the HBM
    slot each resident expert occupies for the real executor.
    """

    __slots__ = ("_h", "_owned", "__weakref__")

    def __init__(self, capacity: int, _handle: int | None = None) -> None:
        if _handle is not None:
            self._h, self._owned = _handle, False
            return
        if capacity < 0:
            raise ValueError(f"capacity must be >= 0, got {capacity}")
        h = C.c_void_p()
        check(lib.hm_cache_create(int(capacity), C.byref(h)))
        self._h, self._owned = h.value, True

    def __del__(self) -> None:
        if getattr(self, "_owned", False) and self._h:
            lib.hm_cache_destroy(self._h)
            self._h = None

    @property
    def capacity(self) -> int:
        v = C.c_int64(0)
        check(lib.hm_cache_capacity(self._h, C.byref(v)))
        return v.value

    @property
    def resident(self) -> _ResidentView:
        return _ResidentView(self)

    @resident.setter
    def resident(self, refs) -> None:
        check(lib.hm_cache_clear_resident(self._h))
        for r in refs:
            check(lib.hm_cache_add_resident(self._h, pack(*_as_ref(r))))

    @property
    def pinned(self) -> _PinnedView:
        return _PinnedView(self)

    @pinned.setter
    def pinned(self, refs) -> None:
        if isinstance(refs, _PinnedView) and refs._c is self:
            return  # `cache.pinned |= s` rebinds the same live view
        check(lib.hm_cache_clear_pinned(self._h))
        for r in refs:
            check(lib.hm_cache_pin(self._h, pack(*_as_ref(r))))

    @property
    def last_access(self) -> _MetaView:
        return _MetaView(self, lib.hm_cache_last_access, lib.hm_cache_set_last_access)

    @property
    def frequency(self) -> _MetaView:
        return _MetaView(self, lib.hm_cache_frequency, lib.hm_cache_set_frequency)

    @property
    def _tick(self) -> int:
        v = C.c_int64(0)
        check(lib.hm_cache_tick(self._h, C.byref(v)))
        return v.value

    def next_tick(self) -> int:
        v = C.c_int64(0)
        check(lib.hm_cache_next_tick(self._h, C.byref(v)))
        return v.value

    def slot_of(self, ref) -> int:
        """HBM slot index of a resident expert (-1 if not resident)."""
        v = C.c_int64(0)
        check(lib.hm_cache_slot(self._h, pack(*_as_ref(ref)), C.byref(v)))
        return v.value

    def check(self) -> None:
        if len(self.resident) > self.capacity:
            raise ValueError(f"resident set ({len(self.resident)}) exceeds capacity {self.capacity}")
        if not set(self.pinned) <= set(self.resident):
            raise ValueError("pinned experts must be resident")
