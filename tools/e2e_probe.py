"""Probe: host<->device copy rates and pipelined batch throughput (not the bench)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2101_02270_b200 import solver as S  # noqa: E402
from paper_2101_02270_b200.case import load_case  # noqa: E402
from paper_2101_02270_b200.scenarios import montecarlo  # noqa: E402

gc = load_case(os.path.join(ROOT, "cases", "synth9241.m"))
T = 10000
n = gc.n_bus
h = torch.empty((n, T), dtype=torch.float64).pin_memory()
d = torch.empty((n, T), dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D {h.numel() * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print(f"D2H {h.numel() * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
del d
vm0, va0 = gc.v_start()
plan = S.NrPlan.from_case(gc, device=0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
ins = [tuple(pin(x) for x in montecarlo(gc, T, task0=i * T)) for i in range(2)]
outs = [S.TaskResults(pin(np.empty((n, T))), pin(np.empty((n, T))), np.empty(T, np.int32),
                      np.empty(T, np.uint8), np.empty(T, np.int32), np.empty(T)) for _ in range(2)]
for K in (1, 2, 4, 8):
    sel = [i % 2 for i in range(K)]
    plan.solve_batches([ins[j][0] for j in sel], [ins[j][1] for j in sel], vm0, va0, [outs[j] for j in sel])
    t = time.perf_counter()
    plan.solve_batches([ins[j][0] for j in sel], [ins[j][1] for j in sel], vm0, va0, [outs[j] for j in sel])
    dt = time.perf_counter() - t
    print(f"solve_batches K={K}: {dt * 1e3:.1f} ms, {K * T / dt:.0f} PF/s, {dt / K * 1e3:.1f} ms/batch", flush=True)
plan.stage(ins[0][0], ins[0][1], vm0, va0)
t = time.perf_counter(); plan.run(); print(f"device solve {1e3 * (time.perf_counter() - t):.1f} ms")
for K in (4,):
    sel = [i % 2 for i in range(K)]
    t = time.perf_counter()
    plan.solve_batches([ins[j][0] for j in sel], [ins[j][1] for j in sel], vm0, va0, [outs[j] for j in sel])
    dt = time.perf_counter() - t
    print(f"again K={K}: {dt * 1e3:.1f} ms; last batch device {plan.timing()['total_ms']:.1f} ms")
# pure compute back to back
plan.stage(ins[0][0], ins[0][1], vm0, va0)
torch.cuda.synchronize()
for _ in range(3):
    t = time.perf_counter(); plan.run(); print(f"run wall {1e3 * (time.perf_counter() - t):.1f} ms device {plan.timing()['total_ms']:.1f}")
