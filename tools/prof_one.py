"""One staged solve (for ncu): prof_one.py CASE TASKS [LU_WARPS] [FS_WARPS]"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from paper_2101_02270_b200 import solver as S

name, T = sys.argv[1], int(sys.argv[2])
lw = int(sys.argv[3]) if len(sys.argv) > 3 else 8
fw = int(sys.argv[4]) if len(sys.argv) > 4 else 8
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
plan = S.NrPlan.from_case(gc, device=0, lu_warps=lw, fs_warps=fw)
plan.stage(p0, q0, vm0, va0)
plan.run()
print(plan.fetch().iterations[:8])
