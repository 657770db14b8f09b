"""Copy the GPU-box evidence of a round into profiles/ (tracked).

usage: python tools/update_profiles.py TAG
Reads gpurun_out/{bench_TAG.log | bench.log, launches_TAG.csv, dram_TAG.csv,
full_TAG_*.ncu-rep} and writes profiles/TAG_bench.json, TAG_launches.md/json,
TAG_dram.md/json, TAG_full_<kernel>.csv (ncu --set full details),
TAG_sass_<kernel>.txt (tools/sass_hot.py) and profiles/ncu_summary.json (the LU
walk's DRAM bytes per task per launch, DRAM throughput fraction and FP64 pipe
utilisation, read by bench.py's roofline object).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

tag = sys.argv[1]
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)
for b in (os.path.join(G, f"bench_{tag}.log"), os.path.join(G, "bench.log")):
    if os.path.exists(b):
        lines = [ln for ln in open(b) if ln.startswith("{")]
        if lines:
            open(os.path.join(P, f"{tag}_bench.json"), "w").write(lines[-1])
            break


def raw_metrics(rep):
    """name -> (unit, value) of one kernel's --page raw."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


summary = {}
for kind in ("launches", "dram"):
    f = os.path.join(G, f"{kind}_{tag}.csv")
    if os.path.exists(f):
        s = ncu_summary.summarise(f, 10000)
        s["source"] = f"gpurun_out/{kind}_{tag}.csv"
        json.dump(s, open(os.path.join(P, f"{tag}_{kind}.json"), "w"), indent=1)
        open(os.path.join(P, f"{tag}_{kind}.md"), "w").write(ncu_summary.to_md(s))
        if kind == "dram":
            k = {e["kernel"]: e for e in s["kernels"]}
            lu = [e for n, e in k.items() if n.startswith("lu_walk_kernel")]
            if lu:
                e = lu[0]
                summary = {"source": f"profiles/{tag}_dram.json (ncu dram__bytes_read.sum + dram__bytes_write.sum "
                                     "over every launch of one synth9241 x 10000 solve) and "
                                     f"profiles/{tag}_full_lu_walk_kernel.csv",
                           "lu_kernel": {"kernel": e["kernel"], "launches": e["launches"],
                                         "dram_bytes_per_task": e["dram_bytes_per_task"] / e["launches"]}}
for rep in glob.glob(os.path.join(G, f"full_{tag}_*.ncu-rep")):
    name = os.path.basename(rep)[len(f"full_{tag}_"):-len(".ncu-rep")]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True)
    open(os.path.join(P, f"{tag}_full_{name}.csv"), "w").write(out.stdout)
    sass = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_hot.py"), rep, "30"],
                          capture_output=True, text=True).stdout
    open(os.path.join(P, f"{tag}_sass_{name}.txt"), "w").write(sass)
    if name == "lu_walk_kernel" and summary:
        m = raw_metrics(rep)
        pick = lambda k: float(m[k][1]) if k in m and m[k][1] not in ("", "n/a") else None  # noqa: E731
        rd, wr = pick("dram__bytes_read.sum"), pick("dram__bytes_write.sum")
        ms = pick("gpu__time_duration.sum")
        rate = pick("dram__bytes.sum.per_second")  # TB/s
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
        summary["lu_kernel"].update({
            "full_capture_ms": ms, "full_dram_gb": (rd + wr) if rd and wr else None,
            "dram_tbs": rate,
            "dram_frac": rate * 1e3 / peak if rate and peak else None,
            "fp64_pipe_pct": pick("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "smem_wavefront_pct": pick("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "issue_ipc": None})
if summary:
    json.dump(summary, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
print(sorted(x for x in os.listdir(P) if x.startswith(tag)))
