"""Every BASELINE.json config on one B200 (not the driver's bench line).

  configs[0] case14, 1000 scenarios      -- GPU solve and the CPU oracle port
  configs[1] synth300 (case300-sized), 10k Monte-Carlo load/PV scenarios
  configs[2] synth2383 (case2383wp-sized), 10k: batched LU refactorization microbenchmark
  configs[3] synth9241 (case9241pegase-sized), 10k (the headline; bench.py)
  configs[4] synth9241, 100k over N GPUs -- per-GPU 12.5k slice at N = 8 (weak-scaled here)

Device times are CUDA events on the solver stream (best of 3 after a warm-up);
CPU numbers are the oracle with all host threads.  Writes one JSON object.
usage: python tools/bench_configs.py [OUT.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402


def gpu_solve(name, T, mode="load"):
    gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
    vm0, va0 = gc.v_start()
    p0, q0 = montecarlo(gc, T, mode=mode)
    plan = S.NrPlan.from_case(gc, device=0, profile=1)
    st = plan.stats()
    plan.stage(p0, q0, vm0, va0)
    plan.run()
    best = None
    for _ in range(3):
        plan.run()
        tm = plan.timing()
        best = tm if best is None or tm["total_ms"] < best["total_ms"] else best
    out = {"case": name, "tasks": T, "scenario_mode": mode, "nJ": st["nJ"], "nnzLU": st["nnzLU"], "D": st["D"],
           "ms": best["total_ms"], "pf_per_s": best["converged"] / (best["total_ms"] / 1e3),
           "iterations": best["iterations"], "converged": best["converged"],
           "per_launch_ms": {k: best[k + "_ms"] / max(best[k + "_launches"], 1)
                             for k in ("npm", "jacobian", "lu", "fsbs", "vupdate")}}
    return gc, plan, out


def cpu_solve(gc, T, threads, mode="load"):
    orc = po.Oracle()
    ip, ix, _, yr, yi = orc.build_ybus(gc)
    vm0, va0 = gc.v_start()
    op = orc.plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    p0, q0 = montecarlo(gc, T, mode=mode)
    t = time.perf_counter()
    r = op.solve(p0, q0, vm0[:, None], va0[:, None], n_threads=threads)
    dt = time.perf_counter() - t
    return {"tasks": T, "threads": threads, "s": dt, "pf_per_s": int((r["status"] == 0).sum()) / dt}


def main():
    threads = os.cpu_count() or 1
    res = {"host_threads": threads}
    gc, plan, res["config0_case14_1000"] = gpu_solve("case14", 1000)
    res["config0_case14_1000"]["cpu_oracle"] = cpu_solve(gc, 1000, threads)
    plan.close()
    # configs[1]: 10k Monte-Carlo load/PV scenarios (PV set-points drawn per task too)
    gc, plan, res["config1_synth300_10k_loadpv"] = gpu_solve("synth300", 10000, mode="loadpv")
    res["config1_synth300_10k_loadpv"]["cpu_oracle"] = cpu_solve(gc, 10000, threads, mode="loadpv")
    plan.close()
    # configs[2]: LU-only microbenchmark, J frozen at each task's start voltages
    gc = load_case(os.path.join(ROOT, "cases", "synth2383.m"))
    vm0, va0 = gc.v_start()
    p0, q0 = montecarlo(gc, 10000)
    plan = S.NrPlan.from_case(gc, device=0)
    st = plan.stats()
    plan.stage(p0, q0, vm0, va0)
    _, _, ms = plan.refactor(reps=10, want_lu=False)
    b = 8 * (2 * st["nnzLU"] + st["D"]) * 10000
    res["config2_synth2383_lu_refactor_10k"] = {
        "ms_per_refactorization": ms, "algorithmic_GBps": b / ms / 1e6, "nnzLU": st["nnzLU"], "D": st["D"]}
    plan.close()
    gc, plan, res["config3_synth9241_10k"] = gpu_solve("synth9241", 10000)
    plan.close()
    gc, plan, res["config4_synth9241_12500_per_gpu"] = gpu_solve("synth9241", 12500)
    plan.close()
    res["config4_synth9241_12500_per_gpu"]["note"] = ("100k scenarios over 8 GPUs = 12.5k per GPU; "
                                                       "tasks are independent (no collective)")
    out = json.dumps(res, indent=1)
    print(out)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(out)


if __name__ == "__main__":
    main()
