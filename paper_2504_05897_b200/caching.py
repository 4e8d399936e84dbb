"""Expert-cache policies: MRS (Eq. 3), LRU, LFU (drop-in for ``moesim.caching``).

The cache container and the MRS score table are native (``hm_cache``,
``hm_mrs``); lookups, victim selection, insert/evict and the MRS update run in
C++ with the reference's exact tie rules and fp64 arithmetic
(caching.py:58-128).  ``MrsState.scores`` is a live mapping view of the table.
The GPU copy of the table used by the real executor is updated with the
``hm_mrs_update_dev`` kernel, bit-identical to this one.
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib, pack
from .core import CacheState, ExpertRef, ModelConfig, Trace, _as_ref
from .errors import EvictionError

POLICY_MRS = "mrs"
POLICY_LRU = "lru"
POLICY_LFU = "lfu"
POLICIES = (POLICY_MRS, POLICY_LRU, POLICY_LFU)
POLICY_CODE = {POLICY_MRS: 0, POLICY_LRU: 1, POLICY_LFU: 2}

__all__ = ["POLICY_MRS", "POLICY_LRU", "POLICY_LFU", "POLICIES", "EvictionError", "MrsState",
           "make_mrs_state", "top_p_filter", "mrs_update", "lookup", "insert_with_eviction",
           "CacheStats", "hit_rate", "replay_trace"]


def _policy(policy: str) -> int:
    try:
        return POLICY_CODE[policy]
    except KeyError:
        raise ValueError(f"unknown policy {policy!r}") from None


class _ScoreView(Mapping):
    """Live view of the native S table as {ExpertRef: float}."""

    __slots__ = ("_m",)

    def __init__(self, m: "MrsState") -> None:
        self._m = m

    def __getitem__(self, ref) -> float:
        layer, expert = _as_ref(ref)
        if not (0 <= layer < self._m.num_layers and 0 <= expert < self._m.num_routed):
            raise KeyError(ref)
        out = C.c_double()
        check(lib.hm_mrs_get(self._m._h, pack(layer, expert), C.byref(out)))
        return out.value

    def __setitem__(self, ref, v: float) -> None:
        check(lib.hm_mrs_set(self._m._h, pack(*_as_ref(ref)), float(v)))

    def __iter__(self):
        return (ExpertRef(l, e) for l in range(self._m.num_layers) for e in range(self._m.num_routed))

    def __len__(self) -> int:
        return self._m.num_layers * self._m.num_routed


class MrsState:
    """Per-expert score S plus (alpha, p) (caching.py:30-42), native table."""

    def __init__(self, scores=None, alpha: float = 0.5, p: int = 4, *, num_layers: int | None = None,
                 num_routed: int | None = None) -> None:
        if not 0.0 <= alpha <= 1.0:
            raise ValueError(f"alpha must be in [0, 1], got {alpha}")
        if p < 1:
            raise ValueError(f"p must be >= 1, got {p}")
        if num_layers is None or num_routed is None:
            keys = list(scores or {})
            num_layers = 1 + max((k[0] for k in keys), default=0)
            num_routed = 1 + max((k[1] for k in keys), default=0)
        h = C.c_void_p()
        check(lib.hm_mrs_create(int(num_layers), int(num_routed), float(alpha), int(p), C.byref(h)))
        self._h = h.value
        self.num_layers, self.num_routed = int(num_layers), int(num_routed)
        if scores is not None:
            for l in range(self.num_layers):
                for e in range(self.num_routed):
                    check(lib.hm_mrs_set(self._h, pack(l, e), float(scores.get(ExpertRef(l, e), 0.0))))

    def __del__(self) -> None:
        if getattr(self, "_h", None):
            lib.hm_mrs_destroy(self._h)
            self._h = None

    @property
    def alpha(self) -> float:
        a = C.c_double()
        check(lib.hm_mrs_params(self._h, C.byref(a), None, None, None))
        return a.value

    @property
    def p(self) -> int:
        v = C.c_int()
        check(lib.hm_mrs_params(self._h, None, C.byref(v), None, None))
        return v.value

    @property
    def scores(self) -> _ScoreView:
        return _ScoreView(self)

    def table(self) -> np.ndarray:
        """S as an [L, N] fp64 array (a copy)."""
        out = np.empty((self.num_layers, self.num_routed), dtype=np.float64)
        check(lib.hm_mrs_table(self._h, _lib.ptr(out, C.c_double)))
        return out


def make_mrs_state(config: ModelConfig, alpha: float = 0.5, p: int | None = None) -> MrsState:
    """Uniform prior 1/N, p defaults to 2K (caching.py:45-55)."""
    if p is None:
        p = 2 * config.num_activated
    return MrsState(None, alpha=alpha, p=p, num_layers=config.num_layers, num_routed=config.num_routed)


def top_p_filter(scores, p: int) -> list[float]:
    """Zero all but the p largest; ties keep the lower index (caching.py:58-62)."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    out = np.empty_like(s)
    check(lib.hm_top_p_filter(_lib.ptr(s, C.c_double), len(s), int(p), _lib.ptr(out, C.c_double)))
    return out.tolist()


def mrs_update(state: MrsState, layer: int, scores) -> MrsState:
    """S[i] <- a*TopP(s)[i] + (1-a)*S[i] for this layer (caching.py:65-76), in place."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    check(lib.hm_mrs_update(state._h, int(layer), _lib.ptr(s, C.c_double), len(s)))
    return state


def _native_cache(cache) -> CacheState:
    if not isinstance(cache, CacheState):
        raise TypeError("the cache operations act on the native CacheState of this package")
    return cache


def lookup(cache: CacheState, expert: ExpertRef, policy: str) -> bool:
    """Hit iff resident; LRU refreshes, LFU counts on hit (caching.py:79-91)."""
    hit = C.c_int()
    check(lib.hm_cache_lookup(_native_cache(cache)._h, pack(*_as_ref(expert)), _policy(policy), C.byref(hit)))
    return bool(hit.value)


def insert_with_eviction(cache: CacheState, expert: ExpertRef, policy: str,
                         mrs: MrsState | None = None) -> ExpertRef | None:
    """Insert a non-resident expert, evicting the policy's victim when full (caching.py:111-128)."""
    v, has = C.c_uint32(), C.c_int()
    check(lib.hm_cache_insert(_native_cache(cache)._h, pack(*_as_ref(expert)), _policy(policy),
                              mrs._h if mrs is not None else None, C.byref(v), C.byref(has)))
    return ExpertRef(v.value >> 16, v.value & 0xFFFF) if has.value else None


@dataclass
class CacheStats:
    lookups: int = 0
    hits: int = 0
    inserts: int = 0
    evictions: int = 0

    def merge(self, other: "CacheStats") -> None:
        self.lookups += other.lookups
        self.hits += other.hits
        self.inserts += other.inserts
        self.evictions += other.evictions

    def check(self) -> None:
        if self.hits > self.lookups:
            raise ValueError("hits exceed lookups")
        if self.evictions > self.inserts:
            raise ValueError("evictions exceed inserts")


def hit_rate(stats: CacheStats) -> float | None:
    return stats.hits / stats.lookups if stats.lookups >= 1 else None


def replay_trace(trace: Trace, policy: str, capacity: int, alpha: float = 0.5, p: int | None = None) -> CacheStats:
    """Cache-only replay (caching.py:158-197): lookups, pin hits, insert and pin
    misses while an unpinned slot remains, MRS update, clear pins."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}")
    cache = CacheState(capacity)
    mrs = make_mrs_state(trace.config, alpha=alpha, p=p) if policy == POLICY_MRS else None
    stats = CacheStats()
    for fwd in trace.passes:
        for req in fwd.layers:
            refs = [ExpertRef(req.layer, i) for i in sorted(req.activated)]
            cache.pinned.update(r for r in refs if r in cache.resident)
            misses = []
            for r in refs:
                stats.lookups += 1
                if lookup(cache, r, policy):
                    stats.hits += 1
                else:
                    misses.append(r)
            for r in misses:
                if len(cache.pinned) >= cache.capacity:
                    break
                if insert_with_eviction(cache, r, policy, mrs) is not None:
                    stats.evictions += 1
                stats.inserts += 1
                cache.pinned.add(r)
            if policy == POLICY_MRS:
                mrs_update(mrs, req.layer, req.scores)
            cache.pinned.clear()
    stats.check()
    return stats
