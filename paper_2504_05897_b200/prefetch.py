"""Impact-driven inter-layer prefetch (drop-in for ``moesim.prefetch``).

``evaluate_gain`` and ``select_prefetches`` run in the native core
(prefetch.py:104-143).  ``predict_activations`` is the reference's prediction
model -- noisy ground truth drawn from numpy's PCG64 stream seeded with
[seed, pass, layer, 0x5EED] (prefetch.py:54-101) -- used in trace (parity)
mode; the live B200 path predicts with the next layers' gate kernels instead
(``moe.MoEModel.lookahead``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib, pack
from .core import CacheState, ExpertRef, LayerRequest, Trace, _as_ref
from .scheduling import MakespanEvaluator

_PREDICT_STREAM = 0x5EED


@dataclass(frozen=True)
class PredictionModel:
    horizon: int = 3
    accuracy: float = 0.85

    def __post_init__(self) -> None:
        if self.horizon < 1:
            raise ValueError(f"horizon must be >= 1, got {self.horizon}")
        if not 0.0 <= self.accuracy <= 1.0:
            raise ValueError(f"accuracy must be in [0, 1], got {self.accuracy}")


@dataclass(frozen=True)
class PrefetchCandidate:
    expert: ExpertRef
    predicted_load: int
    gain: float
    cost: float
    layer_distance: int


def predict_layers(layers, n_layers: int, pass_index: int, current_layer: int, model: PredictionModel,
                   seed: int) -> list[LayerRequest]:
    """The prediction model over a pass's list of LayerRequests (prefetch.py:54-101).

    Each activated expert of a future layer (horizon truncated at the last
    layer) is, with probability 1 - accuracy, swapped -- load and score --
    with a uniformly drawn expert that is not activated at that moment.
    """
    if not 0 <= current_layer < n_layers:
        raise ValueError(f"layer {current_layer} out of range")
    last = min(current_layer + model.horizon, n_layers - 1)
    rng = np.random.default_rng([seed, pass_index, current_layer, _PREDICT_STREAM])
    miss = 1.0 - model.accuracy
    out: list[LayerRequest] = []
    for layer in range(current_layer + 1, last + 1):
        req = layers[layer]
        if model.accuracy >= 1.0:
            out.append(req)
            continue
        loads, scores = list(req.loads), list(req.scores)
        active = set(req.activated)
        n = len(loads)
        for i in sorted(req.activated):
            if rng.random() < miss:
                pool = [j for j in range(n) if j not in active]
                if not pool:
                    continue
                j = pool[int(rng.integers(len(pool)))]
                loads[i], loads[j] = loads[j], loads[i]
                scores[i], scores[j] = scores[j], scores[i]
                active.discard(i)
                active.add(j)
        out.append(LayerRequest(layer=layer, loads=tuple(loads), scores=tuple(scores), activated=frozenset(active)))
    return out


def predict_layers_native(layers, n_layers: int, pass_index: int, current_layer: int, model: PredictionModel,
                          seed: int, pass_loads: np.ndarray | None = None) -> list[LayerRequest]:
    """predict_layers through the native restatement of numpy's stream
    (csrc/predict.cpp); loads only -- the scores of predicted requests are never
    read by the prefetch decision.  pass_loads: the pass's [L, N] loads, if cached."""
    n = len(layers[0].loads)
    if pass_loads is None:
        pass_loads = np.ascontiguousarray([r.loads for r in layers], dtype=np.int64)
    hz = model.horizon
    out_layers = np.empty(hz, dtype=np.int32)
    out_loads = np.empty((hz, n), dtype=np.int64)
    k = C.c_int()
    check(lib.hm_predict_layers(_lib.ptr(pass_loads, C.c_int64), n_layers, n, int(pass_index), int(current_layer),
                                int(seed), hz, float(model.accuracy), _lib.ptr(out_layers, C.c_int32),
                                _lib.ptr(out_loads, C.c_int64), C.byref(k)))
    return [LayerRequest(layer=int(out_layers[d]), loads=tuple(int(v) for v in out_loads[d]), scores=(),
                         activated=frozenset(int(i) for i in np.nonzero(out_loads[d])[0])) for d in range(k.value)]


def predict_activations(trace: Trace, pass_index: int, current_layer: int, model: PredictionModel,
                        seed: int) -> list[LayerRequest]:
    """Future layer requests of this pass, perturbed per the model accuracy (prefetch.py:54-101)."""
    return predict_layers(trace.passes[pass_index].layers, trace.config.num_layers, pass_index, current_layer,
                          model, seed)


def evaluate_gain(candidate: ExpertRef, predicted_request: LayerRequest, cache, evaluator: MakespanEvaluator) -> float:
    """Makespan of the predicted layer without minus with the candidate resident (prefetch.py:104-121)."""
    if candidate in cache.resident:
        raise ValueError(f"{candidate} is already resident")
    if isinstance(cache, CacheState) and isinstance(evaluator, MakespanEvaluator):
        n = len(predicted_request.loads)
        loads = np.zeros(n, dtype=np.int64)
        for i in predicted_request.activated:
            loads[i] = predicted_request.loads[i]
        out = C.c_double()
        check(lib.hm_evaluate_gain(pack(*_as_ref(candidate)), int(predicted_request.layer),
                                   _lib.ptr(loads, C.c_int64), n, cache._h, evaluator._h, C.byref(out)))
        return out.value
    base = evaluator.makespan_for_request(predicted_request, cache.resident)
    with_it = evaluator.makespan_for_request(predicted_request, set(cache.resident) | {candidate})
    return base - with_it


def select_prefetches(candidates: list[PrefetchCandidate], idle_budget: float) -> list[ExpertRef]:
    """Admit by (-gain, layer distance, ref) while the cost fits; stop at the first miss (prefetch.py:124-143)."""
    n = len(candidates)
    arr = (_lib.Candidate * max(1, n))()
    for i, c in enumerate(candidates):
        arr[i].ref = pack(*_as_ref(c.expert))
        arr[i].layer_distance = int(c.layer_distance)
        arr[i].predicted_load = int(c.predicted_load)
        arr[i].gain = float(c.gain)
        arr[i].cost = float(c.cost)
    out = (C.c_uint32 * max(1, n))()
    k = C.c_int()
    check(lib.hm_select_prefetches(arr, n, float(idle_budget), out, C.byref(k)))
    return [ExpertRef(out[i] >> 16, out[i] & 0xFFFF) for i in range(k.value)]
