"""Summarise an ncu --csv launch list (long format) per kernel.

usage: python tools/ncu_summary.py LAUNCHES.csv [--tasks T] [--json OUT.json] [--md OUT.md]

Per kernel name: launches, total / mean device time, share of the total, and --
when the capture has them -- dram__bytes_read.sum + dram__bytes_write.sum in
total, per launch and per task (T tasks in the captured solve).
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import re

SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
           "s": 1e3, "second": 1e3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
           "B": 1}


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::|unnamed>::|void ", "", name)
    return name.split("(")[0].strip()


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ix["ID"]])
        names[lid] = short(r[ix["Kernel Name"]])
        v = float(r[ix["Metric Value"]].replace(",", ""))
        m, u = r[ix["Metric Name"]], r[ix["Metric Unit"]]
        if m == "gpu__time_duration.sum":
            per[lid]["ms"] = v * SCALE_T[u]
        elif m.startswith("dram__bytes_"):
            per[lid]["bytes"] = per[lid].get("bytes", 0.0) + v * SCALE_B.get(u, 1)
    return names, per


def summarise(path, tasks=None):
    names, per = load(path)
    agg = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "bytes": 0.0})
    for lid, d in per.items():
        a = agg[names[lid]]
        a["launches"] += 1
        a["ms"] += d.get("ms", 0.0)
        a["bytes"] += d.get("bytes", 0.0)
    tot = sum(a["ms"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        e = {"kernel": k, "launches": a["launches"], "total_ms": a["ms"],
             "mean_us": 1e3 * a["ms"] / a["launches"], "share": a["ms"] / tot if tot else 0.0}
        if a["bytes"]:
            e["dram_bytes"] = a["bytes"]
            e["dram_GBps"] = a["bytes"] / (a["ms"] * 1e-3) / 1e9 if a["ms"] else None
            if tasks:
                e["dram_bytes_per_task"] = a["bytes"] / tasks
        out.append(e)
    return {"source": path, "total_ms": tot, "kernels": out}


def to_md(s):
    lines = [f"Source: `{s['source']}` (ncu, serialised launches; total {s['total_ms']:.2f} ms)", "",
             "| kernel | launches | total ms | mean us | share | DRAM GB/s | DRAM B/task |",
             "|---|---|---|---|---|---|---|"]
    for e in s["kernels"]:
        lines.append(f"| {e['kernel']} | {e['launches']} | {e['total_ms']:.3f} | {e['mean_us']:.1f} | "
                     f"{100 * e['share']:.1f}% | {e.get('dram_GBps') or '':.6} | "
                     f"{e.get('dram_bytes_per_task', '')} |")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tasks", type=int, default=None)
    ap.add_argument("--json")
    ap.add_argument("--md")
    a = ap.parse_args()
    s = summarise(a.csv, a.tasks)
    if a.json:
        json.dump(s, open(a.json, "w"), indent=1)
    md = to_md(s)
    if a.md:
        open(a.md, "w").write(md)
    print(md)


if __name__ == "__main__":
    main()
