"""Probe: several independent solves sharing one GPU from concurrent host threads.
usage: concurrency_probe.py CASE TOTAL_TASKS PARTS"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

name, total, parts = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
stagger = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0  # ms between thread starts
gc = load_case(os.path.join(ROOT, "cases", name + ".m"))
vm0, va0 = gc.v_start()
T = total // parts
plans = []
for i in range(parts):
    p = S.NrPlan.from_case(gc, device=0, profile=0)
    p0, q0 = montecarlo(gc, T, task0=i * T)
    p.stage(p0, q0, vm0, va0)
    plans.append(p)
for p in plans:
    p.run()
for rep in range(3):
    th = [threading.Thread(target=p.run) for p in plans]
    t = time.perf_counter()
    for x in th:
        x.start()
        time.sleep(stagger / 1e3)
    for x in th:
        x.join()
    dt = time.perf_counter() - t
    conv = sum(p.timing()["converged"] for p in plans)
    print(f"{name} {parts} x {T}: {dt * 1e3:.1f} ms wall, {conv / dt:.0f} PF/s, per-plan device ms "
          f"{[round(p.timing()['total_ms'], 1) for p in plans]}", flush=True)
