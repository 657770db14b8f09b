"""Probe: one 10k batch through gbnr_solve on one plan vs split over k plans
sharing the GPU (n_devices=k, device_step=0: concurrent half/third batches on
their own streams).  usage: split_probe.py CASE TASKS"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

name, T = sys.argv[1], int(sys.argv[2])
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
for k in (1, 2, 3, 1, 2, 3):
    plan = S.NrPlan.from_case(gc, device=0, n_devices=k, device_step=0)
    plan.solve(p0, q0, vm0, va0)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        r = plan.solve(p0, q0, vm0, va0)
        best = min(best, time.perf_counter() - t0)
    print(f"{name} T={T} plans={k}: {best * 1e3:.1f} ms per gbnr_solve ({T / best:.0f} PF/s e2e, "
          f"device {plan.timing()['total_ms']:.1f} ms max shard)", flush=True)
    plan.close()
