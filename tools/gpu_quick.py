"""Quick GPU timing probe (not the bench): solve a batch and print per-kernel times."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from paper_2101_02270_b200 import solver as S

name = sys.argv[1] if len(sys.argv) > 1 else "synth9241"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
warps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
gc = load_case(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "cases", name + ".m"))
plan = S.NrPlan.from_case(gc, device=0, profile=1, lu_warps=warps)
print(plan.stats())
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
plan.stage(p0, q0, vm0, va0)
for rep in range(3):
    t = time.time(); plan.run(); dt = time.time() - t
    tm = plan.timing()
    print(f"run {rep}: wall {dt*1e3:.1f} ms  {T/dt:.0f} PF/s", {k: round(v, 3) if isinstance(v, float) else v for k, v in tm.items()})
r = plan.fetch()
print("iters", np.bincount(r.iterations), "status", np.bincount(r.status))
plan.stage(p0, q0, vm0, va0)
_, fl, ms = plan.refactor(reps=5, want_lu=False)
st = plan.stats()
b_lu = 8 * (2 * st["nnzLU"] + st["D"]) * T
print(f"refactor {ms:.3f} ms  -> {b_lu/ms/1e6:.1f} GB/s algorithmic")
