"""Per-phase timeline of one LU walk launch (library built with make GBNR_TRACE=1,
run with GBNR_DBG=4): parses the device printf of tile 0 and summarises, per
walker, the time from kernel start to each phase barrier and to the end.
usage: GBNR_DBG=4 GBNR_LIB=ab/trace.so python tools/trace_phases.py [CASE] [TASKS]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
case = sys.argv[1] if len(sys.argv) > 1 else "synth9241"
T = sys.argv[2] if len(sys.argv) > 2 else "10000"
code = f"""
import sys; sys.path.insert(0, {ROOT!r})
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
gc = load_case({ROOT!r} + '/cases/{case}.m'); vm0, va0 = gc.v_start(); p0, q0 = montecarlo(gc, {T})
plan = S.NrPlan.from_case(gc, device=0); plan.stage(p0, q0, vm0, va0)
plan.refactor(reps=1, want_lu=False)
"""
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout
ev = [(int(a), int(b), c, int(d)) for a, b, c, d in
      re.findall(r"\[walk\] tile (\d+) warp (\d+) (start|reached sync|done) at (\d+) ns", out)]
for tile in sorted({e[0] for e in ev}):
    es = [e for e in ev if e[0] == tile]
    t0 = min(e[3] for e in es)
    print(f"tile {tile}:")
    for w in sorted({e[1] for e in es}):
        ts = [(e[2], (e[3] - t0) / 1e6) for e in es if e[1] == w]
        print(f"  warp {w}: " + "  ".join(f"{k[:4]} {t:.2f}" for k, t in ts))
