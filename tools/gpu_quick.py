"""Quick GPU timing probe (not the bench): per-kernel device times of one solve
and of the LU-only refactorization.  usage: gpu_quick.py CASE TASKS [key=val ...]
(key=val are gbnr_options fields, e.g. ring_rows=256 prefetch=12)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "synth9241"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
opts = dict(kv.split("=") for kv in sys.argv[3:])
opts = {k: int(v) for k, v in opts.items()}
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
plan = S.NrPlan.from_case(gc, device=0, profile=1, **opts)
st = plan.stats()
plan.stage(p0, q0, vm0, va0)
best = None
for rep in range(3):
    plan.run()
    tm = plan.timing()
    best = tm if best is None or tm["total_ms"] < best["total_ms"] else best
print(f"{name} T={T} {opts}: total {best['total_ms']:.2f} ms ({T / best['total_ms'] * 1e3:.0f} PF/s) "
      f"it={best['iterations']} | " + " ".join(
          f"{k}={best[k + '_ms'] / max(best[k + '_launches'], 1):.3f}" for k in
          ("npm", "jacobian", "lu", "fsbs", "vupdate")), flush=True)
_, fl, ms = plan.refactor(reps=5, want_lu=False)
b_lu = 8 * (2 * st["nnzLU"] + st["D"]) * T
print(f"   refactor {ms:.3f} ms -> {b_lu / ms / 1e6:.1f} GB/s algorithmic", flush=True)
plan.close()
