"""Canonical cache-decision stream ("the record to compare bit-for-bit").

One flat list of JSON-able items per run, in engine.py:288-389 call order:

  ["L", layer, expert, hit]                       lookup
  ["P", makespan, events, assignment]             plan (floats as float.hex())
  ["I", layer, expert, victim_layer, victim_exp]  insert (-1,-1: no victim; "E": EvictionError)
  ["M", layer, sha256(S row fp64)[:16]]           MRS row after mrs_update
  ["G", layer, expert, gain]                      evaluate_gain
  ["S", budget, [[layer, expert], ...]]           select_prefetches

Both the reference (wrapped moesim.engine names) and this package's native
engine (its per-layer decision records) are reduced to this form.
"""
from __future__ import annotations

import hashlib
import json
import struct


def fx(v: float) -> str:
    return float(v).hex()


def plan_item(plan) -> list:
    evs = [[e.device, int(e.expert[0]), int(e.expert[1]), e.kind, fx(e.start), fx(e.end)] for e in plan.events]
    asg = sorted([[int(r[0]), int(r[1]), how] for r, how in plan.assignment.items()])
    return ["P", fx(plan.makespan), evs, asg]


def row_hash(values) -> str:
    return hashlib.sha256(struct.pack(f"<{len(values)}d", *[float(v) for v in values])).hexdigest()[:16]


def insert_item(ref, victim) -> list:
    if victim == "E":
        return ["I", int(ref[0]), int(ref[1]), "E"]
    if victim is None:
        return ["I", int(ref[0]), int(ref[1]), -1, -1]
    return ["I", int(ref[0]), int(ref[1]), int(victim[0]), int(victim[1])]


def digest(stream: list) -> str:
    return hashlib.sha256(json.dumps(stream, separators=(",", ":")).encode()).hexdigest()


def from_records(records: list[dict], mrs_policy: bool) -> list:
    """Stream from this package's per-layer decision records (engine.run_trace(decision_log=True))."""
    out: list = []
    for rec in records:
        out.extend(["L", int(r[0]), int(r[1]), int(h)] for r, h in rec["lookups"])
        out.append(plan_item(rec["plan"]))
        out.extend(insert_item(r, v) for r, v in rec["demand_inserts"])
        if mrs_policy:
            if "layer" in rec:
                layer = rec["layer"]
            else:
                layer = rec["plan"].events[0].expert[0] if rec["plan"].events else rec["lookups"][0][0][0]
            out.append(["M", int(layer), row_hash(rec["mrs_row"])])
        if rec["budget"] is not None:
            out.extend(["G", int(r[0]), int(r[1]), fx(g)] for r, _, g, _ in rec["candidates"])
            out.append(["S", fx(rec["budget"]), [[int(r[0]), int(r[1])] for r in rec["selected"]]])
            out.extend(insert_item(r, v) for r, v in rec["chosen"])
            if rec["prefetch_evict_error"]:
                nxt = rec["selected"][len(rec["chosen"])]
                out.append(insert_item(nxt, "E"))
    return out
