"""Stage + one refactorization (for ncu on the LU level kernels): prof_lu.py CASE TASKS"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from paper_2101_02270_b200 import solver as S
gc = load_case(os.path.join(ROOT, "cases", sys.argv[1] + ".m"))
T = int(sys.argv[2])
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
plan = S.NrPlan.from_case(gc, device=0)
plan.stage(p0, q0, vm0, va0)
plan.run()
plan.stage(p0, q0, vm0, va0)
plan.refactor(reps=1, want_lu=False)
