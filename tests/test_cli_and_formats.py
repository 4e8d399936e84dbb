"""CLI and the file formats it uses: trace JSONL round trip
byte-identical with the reference's writer, profile key=value files,
calibration samples -> profile (the reference's fits, costs.py:134-219)."""
from __future__ import annotations

import math

import pytest

import paper_2504_05897_b200.costs as mcost
import paper_2504_05897_b200.tracegen as mt
from paper_2504_05897_b200 import cli
from paper_2504_05897_b200.moe import SHAPES


def test_trace_roundtrip_and_determinism(tmp_path):
    cfg = SHAPES["tiny"]
    tr = mt.generate_trace(cfg, mt.GenParams(seed=3), 16, 4)
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    mt.save_trace(tr, a)
    mt.save_trace(mt.generate_trace(cfg, mt.GenParams(seed=3), 16, 4), b)
    assert a.read_bytes() == b.read_bytes()
    back = mt.load_trace(a)
    assert [[(r.loads, r.scores) for r in f.layers] for f in back.passes] == \
        [[(r.loads, r.scores) for r in f.layers] for f in tr.passes]


@pytest.mark.reference
def test_trace_file_byte_identical_to_reference_writer(moesim, tmp_path):
    import moesim.core as rc
    import moesim.tracegen as rt
    cfg = dict(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(128, 256),
               bytes_per_weight=2)
    rt.save_trace(rt.generate_trace(rc.ModelConfig(**cfg), rt.GenParams(seed=4), 32, 5), tmp_path / "ref.jsonl")
    from paper_2504_05897_b200.core import ModelConfig
    mt.save_trace(mt.generate_trace(ModelConfig(**cfg), mt.GenParams(seed=4), 32, 5), tmp_path / "ours.jsonl")
    assert (tmp_path / "ref.jsonl").read_bytes() == (tmp_path / "ours.jsonl").read_bytes()
    # and the reference can read what we write
    assert len(rt.load_trace(tmp_path / "ours.jsonl").passes) == 6


def test_bad_trace_file_errors(tmp_path):
    p = tmp_path / "bad.jsonl"
    p.write_text('{"record": "layer"}\n')
    with pytest.raises(mt.TraceFormatError):
        mt.load_trace(p)


def test_profile_and_calibration_files(tmp_path):
    true = mcost.HardwareProfile(gpu_time_per_expert=2e-4, cpu_slope=1.5e-3, transfer_bandwidth=5e10,
                                 transfer_latency=1e-5, cpu_first_expert_penalty=1.2)
    lines = []
    for load in (1, 2, 4):
        for pos in (0, 1, 2):
            lines.append(f"cpu {load} {pos} {mcost.cpu_time(true, load, pos)!r}")
    for load in (1, 64, 200):
        lines.append(f"gpu {load} 0 {mcost.gpu_time(true, load)!r}")
    for nbytes in (1e8, 2e8, 3.5e8):
        lines.append(f"pcie {nbytes} 0 {mcost.transfer_time(true, nbytes)!r}")
    samples = tmp_path / "s.txt"
    samples.write_text("# device load position duration\n" + "\n".join(lines) + "\n")
    out = tmp_path / "p.txt"
    assert cli.main(["calibrate", "--samples", str(samples), "--out", str(out)]) == 0
    got = mcost.load_profile(out)
    for k in ("gpu_time_per_expert", "cpu_slope", "transfer_latency", "cpu_first_expert_penalty"):
        assert math.isclose(getattr(got, k), getattr(true, k), rel_tol=1e-6, abs_tol=1e-12), k
    assert math.isclose(got.transfer_bandwidth, true.transfer_bandwidth, rel_tol=1e-6)
    bad = tmp_path / "bad.txt"
    bad.write_text("cpu 1 0 0.1\ncpu 2 1 0.2\n")
    assert cli.main(["calibrate", "--samples", str(bad), "--out", str(out)]) == 2


def test_cli_generate_run_sweep(tmp_path, capsys):
    t = tmp_path / "t.jsonl"
    assert cli.main(["generate", "--model", "tiny", "--prefill-tokens", "16", "--decode-steps", "3", "--seed", "7",
                     "--out", str(t)]) == 0
    assert cli.main(["run", "--trace", str(t), "--ratio", "0.5", "--prefetch"]) == 0
    assert cli.main(["sweep", "--model", "tiny", "--ratios", "0.25,0.5", "--policies", "mrs,lru", "--seeds", "0,1",
                     "--prefill-tokens", "16", "--decode-steps", "3"]) == 0
    out = capsys.readouterr().out
    assert out.count("\nmrs\t") + out.count("\nlru\t") == 8
    assert cli.main(["generate", "--rho", "1.5", "--out", str(tmp_path / "x.jsonl")]) == 2
