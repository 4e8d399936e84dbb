"""Routing workload: the reference's synthetic router + trace JSONL format.

``generate_trace`` reproduces ``moesim.tracegen.generate_trace``
(tracegen.py:100-163) draw for draw from numpy's PCG64 stream, so the same
(config, GenParams) yields the same ``Trace``.  ``generate_router_logits``
additionally returns the per-token router logits behind that trace -- the
latent z for decode, z + token noise for prefill (tracegen.py:123-147) --
which the B200 path feeds to its router kernel ("trace mode").
``save_trace`` / ``load_trace`` read and write the reference's line-delimited
JSON format (tracegen.py:284-426) so B200 runs can be replayed by ``moesim``.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .core import STAGE_DECODE, STAGE_PREFILL, ForwardPass, LayerRequest, ModelConfig, Trace, make_layer_request
from .errors import TraceFormatError

_TOKEN_NOISE = 0.5   # tracegen.py:45
_TIE_JITTER = 1e-9   # tracegen.py:48


@dataclass(frozen=True)
class GenParams:
    skew: float = 1.0
    temporal_rho: float = 0.85
    layer_sim: float = 0.6
    seed: int = 0

    def __post_init__(self) -> None:
        if self.skew < 0:
            raise ValueError(f"skew must be >= 0, got {self.skew}")
        if not 0.0 <= self.temporal_rho < 1.0:
            raise ValueError(f"temporal_rho must be in [0, 1), got {self.temporal_rho}")
        if not 0.0 <= self.layer_sim < 1.0:
            raise ValueError(f"layer_sim must be in [0, 1), got {self.layer_sim}")


def _softmax_rows(z: np.ndarray) -> np.ndarray:
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def _repair(scores: np.ndarray, activated: np.ndarray) -> np.ndarray:
    """Swap score values so the activated set is the top-|A| set (tracegen.py:74-97)."""
    m, n = int(activated.sum()), len(scores)
    if m == 0 or m == n:
        return scores
    vals = np.sort(scores)[::-1]
    act = np.flatnonzero(activated)
    rest = np.flatnonzero(~activated)
    act = act[np.argsort(-scores[act], kind="stable")]
    rest = rest[np.argsort(-scores[rest], kind="stable")]
    out = np.empty_like(scores)
    out[act] = vals[:m]
    out[rest] = vals[m:]
    if vals[m - 1] <= vals[m]:
        out[act[-1]] += 1e-12
        out[rest[0]] -= 1e-12
    return out


def _walk(config: ModelConfig, params: GenParams, num_prefill_tokens: int, num_decode_steps: int, keep_logits: bool):
    if num_prefill_tokens < 0 or num_decode_steps < 0:
        raise ValueError("token and step counts must be >= 0")
    rng = np.random.default_rng(params.seed)
    n, L, k = config.num_routed, config.num_layers, config.num_activated
    rho, sim = params.temporal_rho, params.layer_sim
    fresh_keep = math.sqrt(1.0 - sim * sim)
    rho_keep = math.sqrt(1.0 - rho * rho)
    schedule = ([(STAGE_PREFILL, num_prefill_tokens)] if num_prefill_tokens > 0 else []) + \
               [(STAGE_DECODE, 1)] * num_decode_steps
    z = np.zeros((L, n))
    passes, logits = [], []
    for p, (stage, tokens) in enumerate(schedule):
        nz = np.empty_like(z)
        for l in range(L):  # latent AR(1) across passes, mixed across layers (tracegen.py:124-133)
            eps = params.skew * rng.standard_normal(n)
            fresh = eps if l == 0 else sim * nz[l - 1] + fresh_keep * eps
            nz[l] = fresh if p == 0 else rho * z[l] + rho_keep * fresh
            nz[l] += _TIE_JITTER * rng.standard_normal(n)
        z = nz
        reqs, pass_logits = [], []
        for l in range(L):
            if stage == STAGE_DECODE:  # tracegen.py:137-142
                scores = _softmax_rows(z[l])
                order = np.lexsort((np.arange(n), -scores))
                loads = np.zeros(n, dtype=int)
                loads[order[:k]] = 1
                if keep_logits:
                    pass_logits.append(z[l][None, :].copy())
            else:  # tracegen.py:144-151
                tok = z[l][None, :] + _TOKEN_NOISE * params.skew * rng.standard_normal((tokens, n))
                top = np.argpartition(-tok, k - 1, axis=1)[:, :k]
                loads = np.bincount(top.ravel(), minlength=n)
                scores = _softmax_rows(tok).mean(axis=0)
                scores = scores / scores.sum()
                scores = _repair(scores, loads > 0)
                if keep_logits:
                    pass_logits.append(tok)
            reqs.append(make_layer_request(l, loads.tolist(), scores.tolist()))
        passes.append(ForwardPass(stage=stage, token_count=tokens, layers=tuple(reqs)))
        if keep_logits:
            logits.append(pass_logits)
    meta = {"seed": str(params.seed), "skew": repr(params.skew), "temporal_rho": repr(params.temporal_rho),
            "layer_sim": repr(params.layer_sim), "prefill_tokens": str(num_prefill_tokens),
            "decode_steps": str(num_decode_steps)}
    return Trace(config=config, passes=tuple(passes), metadata=meta), logits


def generate_trace(config: ModelConfig, params: GenParams, num_prefill_tokens: int, num_decode_steps: int) -> Trace:
    """One optional prefill pass plus decode passes (tracegen.py:100-163)."""
    return _walk(config, params, num_prefill_tokens, num_decode_steps, keep_logits=False)[0]


def generate_router_logits(config: ModelConfig, params: GenParams, num_prefill_tokens: int,
                           num_decode_steps: int) -> tuple[Trace, list[list[np.ndarray]]]:
    """The trace plus, per pass and layer, the fp64 router logits [tokens, N] behind it."""
    return _walk(config, params, num_prefill_tokens, num_decode_steps, keep_logits=True)


# ------------------------------------------------------------- JSONL format


def save_trace(trace: Trace, path: str | Path) -> None:
    """Config record then one record per (pass, layer), fixed key order (tracegen.py:302-336)."""
    cfg = trace.config
    head = {"record": "config", "num_layers": cfg.num_layers, "num_routed": cfg.num_routed,
            "num_shared": cfg.num_shared, "num_activated": cfg.num_activated,
            "routed_expert_dims": list(cfg.routed_expert_dims),
            "shared_expert_dims": list(cfg.shared_expert_dims) if cfg.shared_expert_dims else None,
            "bytes_per_weight": cfg.bytes_per_weight, "metadata": dict(sorted(trace.metadata.items()))}
    out = [json.dumps(head)]
    for p, fwd in enumerate(trace.passes):
        out.extend(json.dumps({"record": "layer", "pass": p, "stage": fwd.stage, "token_count": fwd.token_count,
                               "layer": r.layer, "loads": list(r.loads), "scores": list(r.scores)})
                   for r in fwd.layers)
    Path(path).write_text("\n".join(out) + "\n")


def _field(rec: dict, key: str, lineno: int):
    if key not in rec:
        raise TraceFormatError(f"line {lineno}: missing field {key!r}")
    return rec[key]


def _record(lineno: int, text: str) -> dict:
    try:
        rec = json.loads(text)
    except json.JSONDecodeError as exc:
        raise TraceFormatError(f"line {lineno}: invalid record: {exc}") from exc
    if not isinstance(rec, dict):
        raise TraceFormatError(f"line {lineno}: record must be an object")
    return rec


def load_trace(path: str | Path) -> Trace:
    """Parse a trace file; TraceFormatError carries the line and field (tracegen.py:345-426)."""
    lines = Path(path).read_text().splitlines()
    if not lines:
        raise TraceFormatError("line 1: empty trace file")
    head = _record(1, lines[0])
    if _field(head, "record", 1) != "config":
        raise TraceFormatError("line 1: first record must be the config")
    try:
        shared = head.get("shared_expert_dims")
        cfg = ModelConfig(num_layers=int(_field(head, "num_layers", 1)), num_routed=int(_field(head, "num_routed", 1)),
                          num_shared=int(_field(head, "num_shared", 1)),
                          num_activated=int(_field(head, "num_activated", 1)),
                          routed_expert_dims=tuple(_field(head, "routed_expert_dims", 1)),
                          shared_expert_dims=tuple(shared) if shared else None,
                          bytes_per_weight=float(_field(head, "bytes_per_weight", 1)))
    except ValueError as exc:
        raise TraceFormatError(f"line 1: bad config: {exc}") from exc
    meta = {str(k): str(v) for k, v in head.get("metadata", {}).items()}
    by_pass: dict[int, dict] = {}
    for lineno, text in enumerate(lines[1:], start=2):
        if not text.strip():
            continue
        rec = _record(lineno, text)
        if _field(rec, "record", lineno) != "layer":
            raise TraceFormatError(f"line {lineno}: expected a layer record")
        p = int(_field(rec, "pass", lineno))
        layer = int(_field(rec, "layer", lineno))
        loads, scores = _field(rec, "loads", lineno), _field(rec, "scores", lineno)
        for name, vals in (("loads", loads), ("scores", scores)):
            if len(vals) != cfg.num_routed:
                raise TraceFormatError(f"line {lineno}: field {name!r} has {len(vals)} entries, "
                                       f"config says {cfg.num_routed}")
        slot = by_pass.setdefault(p, {"stage": _field(rec, "stage", lineno),
                                      "token_count": int(_field(rec, "token_count", lineno)), "layers": {}})
        if layer in slot["layers"]:
            raise TraceFormatError(f"line {lineno}: duplicate layer {layer} in pass {p}")
        slot["layers"][layer] = make_layer_request(layer, loads, scores)
    passes = []
    for p in range(len(by_pass)):
        if p not in by_pass:
            raise TraceFormatError(f"pass indices not contiguous: missing pass {p}")
        slot = by_pass[p]
        if set(slot["layers"]) != set(range(cfg.num_layers)):
            missing = sorted(set(range(cfg.num_layers)) - set(slot["layers"]))
            raise TraceFormatError(f"pass {p}: missing layers {missing} (truncated file?)")
        passes.append(ForwardPass(stage=slot["stage"], token_count=slot["token_count"],
                                  layers=tuple(slot["layers"][i] for i in range(cfg.num_layers))))
    return Trace(config=cfg, passes=tuple(passes), metadata=meta)
