"""The native prediction model (csrc/predict.cpp) against numpy's own stream
(prefetch.py:54-101 via this package's predict_layers): identical predicted
loads for every (pass, layer) of several traces and accuracies."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2504_05897_b200 import _lib
from paper_2504_05897_b200.core import ModelConfig
from paper_2504_05897_b200.prefetch import PredictionModel, predict_layers, predict_layers_native
from paper_2504_05897_b200.tracegen import GenParams, generate_trace


@pytest.mark.parametrize("N,K,acc,seed", [(8, 2, 0.85, 0), (64, 6, 0.85, 3), (64, 8, 0.5, 11), (16, 4, 0.0, 7),
                                          (8, 2, 1.0, 1), (5, 4, 0.2, 2)])
def test_native_predictions_equal_numpy(N, K, acc, seed):
    cfg = ModelConfig(6, N, 0, K, (64, 128), None, 2)
    tr = generate_trace(cfg, GenParams(seed=seed), 24, 5)
    model = PredictionModel(horizon=3, accuracy=acc)
    for p, fwd in enumerate(tr.passes):
        for l in range(cfg.num_layers):
            want = predict_layers(fwd.layers, cfg.num_layers, p, l, model, seed)
            got = predict_layers_native(fwd.layers, cfg.num_layers, p, l, model, seed)
            assert [(r.layer, r.loads) for r in got] == [(r.layer, r.loads) for r in want], (p, l)


def test_big_seeds_and_indices():
    cfg = ModelConfig(4, 64, 0, 8, (64, 128), None, 2)
    tr = generate_trace(cfg, GenParams(seed=5), 0, 2)
    model = PredictionModel(horizon=2, accuracy=0.3)
    for seed in (0, 1, 2**31 - 1, 2**32 + 5, 123456789012):
        for l in range(3):
            want = predict_layers(tr.passes[1].layers, 4, 1, l, model, seed)
            got = predict_layers_native(tr.passes[1].layers, 4, 1, l, model, seed)
            assert [r.loads for r in got] == [r.loads for r in want], seed
