#!/usr/bin/env python
"""bench.py -- converged power flows per second of the batched Newton-Raphson
solver (BASELINE.json metric) on a case9241pegase-sized grid, 10k Monte-Carlo
load scenarios per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

A *step* is one full batched NR solve of the per-GPU batch (every task from its
V0 until converged / diverged / max_iter), inputs resident in HBM.  `value` is
converged PFs of all ranks / max-over-ranks device time (CUDA events on the
solver stream).  `e2e` is the same metric through the C ABI call with pinned
host buffers (gbnr_solve: H2D of Sbus, solve, D2H of V / iterations / status).
`--impl reference` times the CPU restatement of the reference path (the
oracle, oracle/oracle.c -- the reference itself has no NR/LU code, SURVEY.md
§0.1) with all host threads on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "converged power flows/sec (10k-scenario batch) at 1/2/4/8 B200 vs CPU ref"
UNIT = "PF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--case", default="synth9241")
    ap.add_argument("--tasks", type=int, default=10000, help="tasks per GPU (weak scaling)")
    ap.add_argument("--total-tasks", type=int, default=0, help="strong scaling: total tasks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample budget")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="batches in the pipelined e2e call (0 = --steps, at least 10: every step one "
                         "10k batch in, its voltages out)")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def ensure_built():
    need = [os.path.join(ROOT, "paper_2101_02270_b200", "libgbnr.so"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-s", "-C", ROOT], check=True)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_lu_summary():
    """The LU walk's ncu figures from the committed capture (profiles/ncu_summary.json):
    DRAM bytes per task per launch, DRAM throughput fraction, FP64 pipe %."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        lu = d["lu_kernel"]
        return {"dram_bytes_per_task": float(lu["dram_bytes_per_task"]),
                "dram_frac": lu.get("dram_frac"), "fp64_pipe_pct": lu.get("fp64_pipe_pct"),
                "source": d.get("source")}
    except Exception:
        return {}


def host_info():
    """Host cores and CPU model of the box (reported beside every CPU number)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def workload_config(case, nJ, T, world):
    """The `config` object of both arms (same workload, same keys)."""
    return {"workload": f"{case} (case9241pegase-sized synthetic grid, {nJ}-dim Jacobian), "
                        "Monte-Carlo loads U(0.8,1.2)",
            "case": case, "tasks_per_gpu": T, "global_batch": T * world,
            "parallelism": f"scenario-sharded x{world}, no collective", "tol": 1e-8, "max_iter": 10}


def oracle_plan(gc):
    """The CPU restatement (test oracle) on the case's representative task; Ybus
    from the oracle's own build_ybus (nothing of the product on this path)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    orc = po.Oracle()
    ip, ix, _, yr, yi = orc.build_ybus(gc)
    vm0, va0 = gc.v_start()
    return orc.plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0), vm0, va0


def cpu_baseline(gc, case, p0, q0, budget_s, threads):
    """Oracle (CPU restatement of the reference path) on the SAME pre-generated
    batch the GPU arm solves: whole-batch calls repeated until budget_s, input
    generation outside the timed region (as in --impl reference)."""
    oplan, vm0, va0 = oracle_plan(gc)
    T = p0.shape[1]
    done = conv = 0
    t0 = time.perf_counter()
    while True:
        r = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T, n_threads=threads)
        conv += int((r["status"] == 0).sum())
        done += T
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": conv / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{done // T} x the GPU arm's batch ({T} tasks, ids 0..{T - 1}) of the {case} "
                      f"Monte-Carlo workload, inputs pre-generated, {dt:.1f} s on {threads} threads",
            **host_info()}


def run_reference(a, rk):
    """--impl reference: the oracle port with all host threads on the same
    workload as our arm (same case, same tasks per step, same scenario ids),
    rank 0 only.  Inputs are generated once, before warm-up."""
    from paper_2101_02270_b200.case import load_case
    from paper_2101_02270_b200.scenarios import montecarlo
    if not rk.is_root:
        return None
    gc = load_case(os.path.join(ROOT, "cases", a.case + ".m"))
    threads = os.cpu_count() or 1
    oplan, vm0, va0 = oracle_plan(gc)
    T = a.tasks
    p0, q0 = montecarlo(gc, T)
    for _ in range(a.warmup):
        oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T, n_threads=threads)
    conv = 0
    t0 = time.perf_counter()
    for _ in range(a.steps):
        r = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T, n_threads=threads)
        conv += int((r["status"] == 0).sum())
    dt = time.perf_counter() - t0
    value = conv / dt
    sample = (f"the full {T}-task batch (ids 0..{T - 1}) of the {a.case} workload per step, "
              "inputs pre-generated")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload_config(a.case, oplan.stats()["nJ"], T, 1), "same_config": True,
                       "threads": threads},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample, **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    a = parse()
    ensure_built()
    from paper_2101_02270_b200 import dist
    rk = dist.init()
    if a.impl == "reference":
        out = run_reference(a, rk)
        if out is not None:
            print(json.dumps(out), flush=True)
        dist.finalize(rk)
        return

    import torch
    from paper_2101_02270_b200 import solver as S
    from paper_2101_02270_b200.case import load_case
    from paper_2101_02270_b200.scenarios import montecarlo

    dev = dist.device_of(rk)
    gc = load_case(os.path.join(ROOT, "cases", a.case + ".m"))
    if a.total_tasks:
        task0, T = dist.shard(a.total_tasks, rk.world, rk.rank)
        scaling = "strong"
    else:
        task0, T = rk.rank * a.tasks, a.tasks
        scaling = "weak"
    torch.cuda.init()
    # load the library and its modules once (a case14 plan), so init_ms is the plan
    # build of the benchmark case itself, not the process's first CUDA use
    S.NrPlan.from_case(load_case(os.path.join(ROOT, "cases", "case14.m")), device=dev).close()
    i0 = time.perf_counter()
    plan = S.NrPlan.from_case(gc, device=dev, profile=1)  # one-time init
    init_ms = (time.perf_counter() - i0) * 1e3
    st = plan.stats()
    vm0, va0 = gc.v_start()
    p0, q0 = montecarlo(gc, T, task0=task0)
    plan.stage(p0, q0, vm0, va0, n_tasks=T)

    for _ in range(a.warmup):
        plan.run()
    dist.barrier(rk)
    torch.cuda.synchronize(dev)
    dev_ms = lu_ms = 0.0
    conv = launches = lu_launches = lu_tasks = npm_tasks = 0
    iters = []
    with ClockSampler(dev) as clk:
        w0 = time.perf_counter()
        for _ in range(a.steps):
            plan.run()
            tm = plan.timing()
            dev_ms += tm["total_ms"]
            lu_ms += tm["lu_ms"]
            conv += tm["converged"]
            lu_launches += tm["lu_launches"]
            lu_tasks += tm["lu_task_launches"]
            npm_tasks += tm["tasks"] + tm["lu_task_launches"]  # the V0 check + one per update
            launches += tm["kernels"]
            iters.append(tm["iterations"])
        wall = time.perf_counter() - w0
    torch.cuda.synchronize(dev)
    dist.barrier(rk)
    job_ms = dist.reduce_max(rk, dev_ms)
    job_conv = dist.reduce_sum(rk, conv)
    value = job_conv / (job_ms / 1e3)

    # end to end through the C ABI with pinned host buffers: gbnr_solve_batches
    # over e2e_steps batches (alternating two distinct scenario batches), every
    # batch's H2D of Sbus and D2H of V / iterations / status inside the timed
    # region, pipelined against the neighbouring batches' solves
    n = gc.n_bus
    import ctypes as C
    lib = S.lib()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    pb, qb = montecarlo(gc, T, task0=task0 + T)
    ins = [(pin(p0), pin(q0)), (pin(pb), pin(qb))]
    outs = [S.TaskResults(pin(np.empty((n, T))), pin(np.empty((n, T))), np.empty(T, np.int32),
                          np.empty(T, np.uint8), np.empty(T, np.int32), np.empty(T)) for _ in range(2)]
    K = max(a.e2e_steps, 1) if a.e2e_steps > 0 else max(a.steps, 10)
    P = C.c_void_p * K
    arr = lambda xs: P(*[x.ctypes.data for x in xs])  # noqa: E731
    sel = [i % 2 for i in range(K)]
    def solve_e2e():
        rc = lib.gbnr_solve_batches(
            plan.h, K, T, arr([ins[j][0] for j in sel]), arr([ins[j][1] for j in sel]),
            vm0.ctypes.data, va0.ctypes.data, arr([outs[j].vm for j in sel]), arr([outs[j].va for j in sel]),
            arr([outs[j].iterations for j in sel]), arr([outs[j].converged for j in sel]),
            arr([outs[j].status for j in sel]), arr([outs[j].max_mismatch for j in sel]))
        S._check(rc)
    solve_e2e()  # warm
    e2e_runs = []
    for _ in range(3):  # median of three jobs (host-side PCIe / pinned-memory jitter)
        dist.barrier(rk)
        e0 = time.perf_counter()
        solve_e2e()
        e2e_runs.append(dist.reduce_max(rk, time.perf_counter() - e0))
    e2e_s = sorted(e2e_runs)[1]
    e2e_conv = dist.reduce_sum(rk, sum(int(outs[j].converged.sum()) for j in sel))
    h2d = 2 * n * T * 8
    d2h = 2 * n * T * 8 + T * (4 + 4 + 8)

    # roofline of the dominant kernel: the LU walk (frozen-pattern G-P
    # refactorization fused with the forward substitution), DESIGN.md §5:
    # 8(2 zLU + D) bytes of Alg. 2 + 16 nJ of right-hand side in / y out
    b_lu_task = 8 * (2 * st["nnzLU"] + st["D"]) + 16 * st["nJ"]
    peak, peak_kind = measured_peaks()
    achieved = b_lu_task * lu_tasks / (lu_ms / 1e3) / 1e9 if lu_ms > 0 else None
    ncu = ncu_lu_summary()
    tr = ncu.get("dram_bytes_per_task")
    # whole solve: every kernel's algorithmic bytes (DESIGN.md §5 table) over the
    # whole device time -- mismatch sweeps for every check, the rest per LU launch
    n_, nJ_, zLU_, zL_ = gc.n_bus, st["nJ"], st["nnzLU"], st["nnzL"]
    b_npm = 32 * n_ + 8 * nJ_
    b_iter = (16 * n_ + 8 * zLU_) + b_lu_task + (8 * (zLU_ - zL_) + 16 * nJ_) + (8 * nJ_ + 32 * n_)
    solve_bytes = b_npm * npm_tasks + b_iter * lu_tasks
    solve_gbs = solve_bytes / (dev_ms / 1e3) / 1e9 if dev_ms > 0 else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "traffic": tr * (lu_tasks / max(lu_launches, 1)) if tr else None,
            "kernel": "lu_walk_kernel<FS> (batched frozen-pattern G-P refactorization + forward "
                      "substitution, tile walks)",
            "algorithmic_bytes_per_task": b_lu_task, "peak_kind": peak_kind,
            # also against the nominal HBM3e figure (7.7 TB/s HGX B200)
            "peak_nominal": 7700.0, "frac_nominal": achieved / 7700.0 if achieved else None,
            "lu_ms_per_launch": lu_ms / max(lu_launches, 1),
            "lu_share_of_step": lu_ms / dev_ms if dev_ms else None,
            # ncu (profiles/ncu_summary.json): DRAM bytes actually moved by one LU launch
            # and its rate over the ncu-timed launch, FP64 pipe utilisation
            "ncu_dram_frac": ncu.get("dram_frac"), "ncu_fp64_pipe_pct": ncu.get("fp64_pipe_pct"),
            "ncu_source": ncu.get("source"),
            "whole_solve": {"achieved": solve_gbs, "peak": peak, "unit": "GB/s",
                            "frac": solve_gbs / peak if solve_gbs else None,
                            "bytes_per_task_iteration": b_iter + b_npm,
                            "note": "algorithmic bytes of every kernel (DESIGN.md §5) over the whole "
                                    "device time of the solve"}}

    cpu = None
    if rk.is_root and rk.world == 1 and not a.no_cpu:
        cpu = cpu_baseline(gc, a.case, p0, q0, a.cpu_seconds, os.cpu_count() or 1)

    if rk.is_root:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": rk.world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": job_ms / a.steps,
               "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
               "dtype": "f64", "data": "synthetic",
               "config": {**workload_config(a.case, st["nJ"], T, rk.world),
                          "newton_iterations_per_step": iters,
                          "l2": "inputs larger than L2 (LU tape "
                                f"{st['nnzLU'] * 8 * T / 1e9:.1f} GB per GPU)",
                          "wall_s_timed": wall},
               "init_ms": init_ms,
               "init_note": "one-time plan create of the case (symbolic analysis, walk programs, upload), "
                            "excluded from value; library loaded beforehand",
               "clocks": clk.summary(),
               "e2e": {"value": e2e_conv / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "steps": K, "jobs_timed": 3, "statistic": "median",
                       "call": "gbnr_solve_batches (pinned host buffers, per-batch H2D/D2H pipelined "
                               "against the neighbouring batches' solves)"},
               "gpu_launches": int(launches),
               "roofline": roof,
               "cpu_baseline": cpu}
        print(json.dumps(out), flush=True)
    plan.close()
    dist.finalize(rk)


if __name__ == "__main__":
    main()
