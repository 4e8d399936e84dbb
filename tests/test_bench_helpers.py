"""bench.py host-side helpers (CPU): the warm-up refit of the host-worker
decode cost and the extra-config table."""
from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    argv = sys.argv
    sys.argv = ["bench.py"]
    try:
        spec.loader.exec_module(mod)
    finally:
        sys.argv = argv
    return mod


class _S:
    def __init__(self, n, us):
        self.n_cpu, self.t_cpu_us = n, us


def test_refit_recovers_slope_and_penalty(bench):
    from paper_2504_05897_b200.costs import HardwareProfile
    prof = HardwareProfile(gpu_time_per_expert=1e-4, cpu_slope=2.7e-3, transfer_bandwidth=5e10)
    slope, pen = 1.9e-3, 1.2
    stats = [_S(n, 1e6 * slope * (pen + n - 1)) for n in (1, 2, 1, 3, 2, 1, 0)]
    r = bench.refit_cpu_decode(stats, prof)
    assert r["cpu_slope"] == pytest.approx(slope, rel=1e-9)
    assert r["cpu_first_expert_penalty"] == pytest.approx(pen, rel=1e-9)
    assert r["calibrated_cpu_slope"] == 2.7e-3 and r["layers"] == 6


def test_refit_falls_back_to_mean_and_needs_samples(bench):
    from paper_2504_05897_b200.costs import HardwareProfile
    prof = HardwareProfile(gpu_time_per_expert=1e-4, cpu_slope=2.7e-3, transfer_bandwidth=5e10)
    # every layer ran one expert: no intercept can be fitted -> per-expert mean, penalty 1
    r = bench.refit_cpu_decode([_S(1, 2000.0), _S(1, 2200.0), _S(1, 1800.0), _S(1, 2000.0)], prof)
    assert r["cpu_slope"] == pytest.approx(2.0e-3) and r["cpu_first_expert_penalty"] == 1.0
    assert bench.refit_cpu_decode([_S(1, 2000.0)] * 3, prof) is None


def test_extra_configs_are_named_configs(bench):
    assert set(bench.EXTRA_CONFIGS) == {"deepseek_25", "qwen2_10", "qwen2_25", "qwen2_50", "mixtral_25_q4"}
    for argv in bench.EXTRA_CONFIGS.values():
        assert "--shape" in argv and "--ratio" in argv
