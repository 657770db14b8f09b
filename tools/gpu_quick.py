"""Quick GPU timing probe (not the bench): per-kernel times over a config sweep.
usage: gpu_quick.py CASE TASKS LU_WARPS[,..] FS_WARPS[,..]"""
import sys, time, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from paper_2101_02270_b200 import solver as S

name = sys.argv[1] if len(sys.argv) > 1 else "synth9241"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
lws = [tuple(int(y) for y in x.split(":")) for x in (sys.argv[3] if len(sys.argv) > 3 else "8:32").split(",")]
fws = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "16").split(",")]
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
for lw, cap in lws:
    for fw in fws:
        plan = S.NrPlan.from_case(gc, device=0, profile=1, fs_warps=fw,
                                  bulk_min=int(os.environ.get("BULK", "0")))
        st = plan.stats()
        plan.stage(p0, q0, vm0, va0)
        best = None
        for rep in range(3):
            t = time.time(); plan.run(); dt = time.time() - t
            tm = plan.timing()
            best = tm if best is None or tm["total_ms"] < best["total_ms"] else best
        it = best["iterations"]
        print(f"lu_warps={lw} cap={cap} fs_warps={fw}: total {best['total_ms']:.1f} ms ({T/best['total_ms']*1e3:.0f} PF/s) it={it} | "
              + " ".join(f"{k}={best[k+'_ms']/max(best[k+'_launches'],1):.3f}" for k in ("npm", "jacobian", "lu", "fsbs", "vupdate")), flush=True)
        _, fl, ms = plan.refactor(reps=5, want_lu=False)
        b_lu = 8 * (2 * st["nnzLU"] + st["D"]) * T
        print(f"   refactor {ms:.3f} ms -> {b_lu/ms/1e6:.1f} GB/s algorithmic", flush=True)
        plan.close()
r = None
