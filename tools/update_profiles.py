"""Copy the GPU-box evidence of a round into profiles/ (tracked).

usage: python tools/update_profiles.py TAG
Reads gpurun_out/{bench.log, launches_TAG.csv, dram_TAG.csv, full_TAG_*.ncu-rep}
and writes profiles/TAG_bench.json, TAG_launches.md/json, TAG_dram.md/json,
TAG_full_<kernel>.csv (ncu --set full details) and profiles/ncu_summary.json
(per-task DRAM bytes of one LU-walk launch, read by bench.py's roofline).
"""
import glob
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
b = os.path.join(G, "bench.log")
if os.path.exists(b):
    lines = [ln for ln in open(b) if ln.startswith("{")]
    if lines:
        open(os.path.join(P, f"{tag}_bench.json"), "w").write(lines[-1])
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
                json.dump({"source": f"profiles/{tag}_dram.json (ncu dram__bytes_read.sum + "
                                     "dram__bytes_write.sum over every launch of one synth9241 x 10000 solve)",
                           "lu_kernel": {"kernel": e["kernel"], "launches": e["launches"],
                                         "dram_bytes_per_task": e["dram_bytes_per_task"] / e["launches"]}},
                          open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
for rep in glob.glob(os.path.join(G, f"full_{tag}_*.ncu-rep")):
    name = os.path.basename(rep)[len(f"full_{tag}_"):-len(".ncu-rep")]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True)
    open(os.path.join(P, f"{tag}_full_{name}.csv"), "w").write(out.stdout)
print(sorted(os.listdir(P)))
