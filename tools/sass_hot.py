"""Summarise an ncu --set full report at SASS level: top blocks by instructions
and stall samples.  usage: python tools/sass_hot.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: sum(int(r[hdr.index(h)] or 0) for r in data) for h in reasons}
print("stalls:", sorted(((k, v) for k, v in tot.items() if v), key=lambda x: -x[1]))
blocks, cur = [], None
for i, r in enumerate(data):
    e, s = int(r[iE] or 0), int(r[iS] or 0)
    if cur is None or e != cur[1]:
        cur = [i, e, 0, 0, r[1].strip()[:48]]
        blocks.append(cur)
    cur[2] += s
    cur[3] += 1
ti = sum(b[1] * b[3] for b in blocks)
ts = sum(b[2] for b in blocks)
print(f"instructions {ti:.4g}  samples {ts}")
for b in sorted(blocks, key=lambda b: -(b[1] * b[3] / ti + b[2] / ts))[:N]:
    print(f"@{b[0]:5d} exec={b[1]:>11d} n={b[3]:3d} inst={b[1]*b[3]/ti*100:5.1f}% "
          f"samp={b[2]/ts*100:5.1f}%  {b[4]}")
