"""Probe: one synth9241 batch as k concurrent slices on one GPU (k plans, each
its own stream, driven from k host threads), device-resident (staged), timed by
wall clock around synchronised runs.  usage: stream_probe.py CASE TASKS"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

name, T = sys.argv[1], int(sys.argv[2])
ks = [int(x) for x in sys.argv[3:]] or [1, 2, 3, 4]
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
p0, q0 = montecarlo(gc, T)
for k in ks:
    plans = []
    for i in range(k):
        a, b = T * i // k, T * (i + 1) // k
        pl = S.NrPlan.from_case(gc, device=0, profile=0)
        pl.stage(np.ascontiguousarray(p0[:, a:b]), np.ascontiguousarray(q0[:, a:b]), vm0, va0)
        plans.append(pl)

    def job():
        th = [threading.Thread(target=pl.run) for pl in plans]
        for t in th:
            t.start()
        for t in th:
            t.join()
    job()
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        job()
        best = min(best, time.perf_counter() - t0)
    conv = sum(pl.timing()["converged"] for pl in plans)
    dev = [pl.timing()["total_ms"] for pl in plans]
    print(f"{name} T={T} k={k}: {best * 1e3:.1f} ms wall per batch ({conv / best:.0f} PF/s), "
          f"per-slice device ms {[round(d, 1) for d in dev]}, tw {[pl.walk_info(0)['rows'] for pl in plans]}", flush=True)
    for pl in plans:
        pl.close()
