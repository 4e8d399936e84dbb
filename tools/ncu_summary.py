"""Summarise ncu reports / launch lists into profiles/*.md (run in the build container).

  python tools/ncu_summary.py gpurun_out/prof_gemv1.ncu-rep ... --launches gpurun_out/launches_decode.csv --out profiles/r01_summary.md
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__t_bytes.sum",
    "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3,
        "MB": 1e6, "GB": 1e9}


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        d["__units__"] = dict(zip(head, units))
        recs.append(d)
    return recs


def num(rec: dict, key: str) -> float | None:
    v = rec.get(key)
    if v is None:
        return None
    try:
        f = float(v.replace(",", ""))
    except ValueError:
        return None
    return f * UNIT.get(rec["__units__"].get(key, ""), 1.0)


def fmt(v: str) -> str:
    try:
        f = float(v.replace(",", ""))
    except ValueError:
        return v
    return f"{f:,.4g}"


def summarise_rep(rep: str) -> str:
    recs = raw(rep)
    lines = [f"### `{Path(rep).name}` ({len(recs)} profiled launches)", ""]
    for i, r in enumerate(recs):
        name = r.get("Kernel Name", r.get("Function Name", "?"))
        lines.append(f"**launch {i}: `{name[:120]}`**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m in METRICS:
            for k in r:
                if k == m or k.startswith(m + " "):
                    lines.append(f"| {k} | {fmt(r[k])} {r['__units__'].get(k, '')} |")
                    break
        rd, wr, t = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum"), num(r, "gpu__time_duration.sum")
        if rd is not None and wr is not None:
            lines.append(f"| **dram traffic (read+write)** | **{rd + wr:,.0f} B** |")
            if t:
                lines.append(f"| dram GB/s (traffic / duration) | {(rd + wr) / t / 1e9:,.1f} |")
        lines.append("")
    return "\n".join(lines)


def summarise_launches(path: str) -> str:
    text = Path(path).read_text().splitlines()
    start = next((i for i, l in enumerate(text) if l.startswith('"ID"')), None)
    if start is None:
        return f"(no launch table in {path})"
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:80]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        per[name][0] += 1
        per[name][1] += v
        total += v
    lines = [f"### launch list `{Path(path).name}`: {sum(c for c, _ in per.values())} launches, "
             f"{total / 1e3:,.2f} ms of kernel time (cold-cache, serialised by ncu)", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for name, (c, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {c} | {us:,.1f} | {us / c:,.2f} | {us / total:.1%} |")
    return "\n".join(lines)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    parts = [f"# {a.title}", ""]
    for l in a.launches:
        parts += [summarise_launches(l), ""]
    for r in a.reps:
        parts += [summarise_rep(r), ""]
    Path(a.out).write_text("\n".join(parts))
    print(a.out)


if __name__ == "__main__":
    main()
