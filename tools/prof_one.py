"""The ncu capture target of tools/gpu_round.sh and gpu_full.sh: one staged solve.

usage: prof_one.py CASE TASKS [key=val ...]  (key=val are gbnr_options fields)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

name, T = sys.argv[1], int(sys.argv[2])
opts = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[3:])}
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
plan = S.NrPlan.from_case(gc, device=0, **opts)
plan.stage(p0, q0, vm0, va0)
plan.run()
print(plan.fetch().iterations[:8])
