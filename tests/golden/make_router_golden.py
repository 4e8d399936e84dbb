"""Router fixtures from the UNMODIFIED reference trace generator (moesim.tracegen).

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_router_golden.py

For the three model shapes of BASELINE.json (Mixtral-8x7B, DeepSeek-V2-Lite,
Qwen2-57B-A14B) and generator seeds 0-4, `generate_trace(cfg, GenParams(seed),
1024, 4)` is run with `moesim.tracegen._softmax` wrapped, which records the
exact fp64 logits the reference routes on (tracegen.py:137-151: the decode
latent z[layer], the prefill per-token `tok` matrix).  Written:

  tests/golden/router_real_shapes.json
      per (shape, seed): the 1024-token prefill pass's loads [L][N]
      (tracegen.py:147-148) and a SHA-256 of each layer's fp64 logits, plus
      the decode passes' loads -- the GPU router must reproduce these loads
      from the same logits (tests/test_router_real_shapes_gpu.py), and this
      package's generator must reproduce the logits bit for bit
      (tests/test_router_real_shapes.py).
  oracle/fixtures/decode_logits_<shape>.npy
      fp32 [P, L, N] decode logits of seed 0 (P = 32 passes): the routing
      input of bench.py's reference arm, so that arm imports nothing from the
      product package.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

import moesim.core as mcore  # noqa: E402
import moesim.tracegen as mt  # noqa: E402

SHAPES = {
    "mixtral": dict(num_layers=32, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(4096, 14336),
                    bytes_per_weight=2),
    "deepseek": dict(num_layers=26, num_routed=64, num_shared=2, num_activated=6, routed_expert_dims=(2048, 1408),
                     shared_expert_dims=(2048, 1408), bytes_per_weight=2),
    "qwen2": dict(num_layers=28, num_routed=64, num_shared=1, num_activated=8, routed_expert_dims=(3584, 2560),
                  shared_expert_dims=(3584, 20480), bytes_per_weight=2),
}
PREFILL, DECODE, SEEDS, BENCH_PASSES = 1024, 4, (0, 1, 2, 3, 4), 32


def capture(cfg, seed, prefill, decode):
    """generate_trace with the logits it routes on, in call order."""
    seen = []
    orig = mt._softmax

    def spy(z):
        seen.append(np.array(z, dtype=np.float64, copy=True))
        return orig(z)

    mt._softmax = spy
    try:
        tr = mt.generate_trace(cfg, mt.GenParams(seed=seed), prefill, decode)
    finally:
        mt._softmax = orig
    L = cfg.num_layers
    assert len(seen) == L * len(tr.passes)
    logits = [[seen[p * L + l] for l in range(L)] for p in range(len(tr.passes))]
    return tr, logits


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def main() -> None:
    out = {"numpy": np.__version__, "prefill": PREFILL, "decode": DECODE, "shapes": {}}
    for name, d in SHAPES.items():
        cfg = mcore.ModelConfig(**d)
        entries = []
        for seed in SEEDS:
            tr, logits = capture(cfg, seed, PREFILL, DECODE)
            entries.append({
                "seed": seed,
                "prefill_loads": [list(r.loads) for r in tr.passes[0].layers],
                "prefill_logits_sha": [sha(logits[0][l]) for l in range(cfg.num_layers)],
                "decode_loads": [[list(r.loads) for r in f.layers] for f in tr.passes[1:]],
                "decode_logits_sha": [[sha(logits[p][l]) for l in range(cfg.num_layers)]
                                      for p in range(1, len(tr.passes))],
            })
        out["shapes"][name] = {"config": d, "runs": entries}
        # bench reference arm: frozen decode routing (seed 0, no prefill pass)
        tr, logits = capture(cfg, 0, 0, BENCH_PASSES)
        arr = np.stack([np.stack([logits[p][l] for l in range(cfg.num_layers)]) for p in range(BENCH_PASSES)])
        np.save(ROOT / "oracle" / "fixtures" / f"decode_logits_{name}.npy", arr.astype(np.float32))
        print(name, "done", flush=True)
    tiny = mcore.ModelConfig(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(256, 256),
                             bytes_per_weight=2)
    tr, logits = capture(tiny, 0, 0, BENCH_PASSES)
    arr = np.stack([np.stack([logits[p][l] for l in range(4)]) for p in range(BENCH_PASSES)])
    np.save(ROOT / "oracle" / "fixtures" / "decode_logits_tiny.npy", arr.astype(np.float32))
    (HERE / "router_real_shapes.json").write_text(json.dumps(out, separators=(",", ":")))


if __name__ == "__main__":
    main()
