"""Job front end: the reference's batch_runtime modes over the GPU solver.

``batch_runtime.run`` takes a JobSpec with a
mode in {montecarlo, timeseries, contingency, single} and hands each mini-batch
of tasks to ``nr_solve_batch``.  Here every mode reduces to per-task inputs for
one ``gbnr_solve`` call (host arrays, the C ABI of include/gbnr.h):

* montecarlo  -- seeded U(0.8, 1.2) load scenarios (scenarios.py);
* timeseries  -- one task per row of a scenario CSV (case_io.hpp:368-447), "a thin
                 wrapper over montecarlo plumbing (profiles per step)";
* contingency -- one branch outage per task (an outage list, case_io.hpp:449-471):
                 per-task Ybus value sets on the fixed pattern, and the islanding
                 pre-check (grid.hpp:257-261) -- islanded tasks are not solved and
                 report status ``ISLANDED``;
* single      -- the case loads, one task.

No numerics here: inputs are assembled on the host exactly as the reference's
``assemble_profiles`` does (grid.hpp:299-344), and every solve runs on the GPU.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import solver as S
from .case import parse_outage_list, parse_scenario_csv
from .scenarios import SEED, montecarlo

CONVERGED, DIVERGED, SINGULAR, FALLBACK_CONVERGED, ISLANDED = 0, 1, 2, 3, 4
MODES = ("montecarlo", "timeseries", "contingency", "single")


@dataclass
class JobInputs:
    p0: np.ndarray            # [n_bus][T] p.u.
    q0: np.ndarray
    y: tuple | None           # per-task Ybus value sets (y_re, y_im) [nnzY][T], or None
    islanded: np.ndarray      # [T] bool: excluded by the islanding pre-check
    outages: np.ndarray | None


@dataclass
class JobResult:
    status: np.ndarray        # [T] CONVERGED / DIVERGED / SINGULAR / FALLBACK_CONVERGED / ISLANDED
    iterations: np.ndarray
    vm: np.ndarray            # [n_bus][T]
    va: np.ndarray
    max_mismatch: np.ndarray
    report: dict              # RunReport subset: phase times, counts


def job_inputs(gc, mode: str, n_tasks: int | None = None, scenario_csv: str | None = None,
               outages=None, seed: int = SEED, scenario_mode: str = "load") -> JobInputs:
    """Per-task solver inputs of one job (JobSpec invariants)."""
    if mode not in MODES:
        raise ValueError(f"unknown job mode {mode!r}; expected one of {MODES}")
    y = None
    out = None
    if mode == "montecarlo":
        if not n_tasks or n_tasks < 1:
            raise ValueError("montecarlo mode needs n_tasks >= 1")
        p0, q0 = montecarlo(gc, n_tasks, seed=seed, mode=scenario_mode)
    elif mode == "timeseries":
        if scenario_csv is None:
            raise ValueError("timeseries mode needs a scenario CSV (one row per step)")
        p0, q0 = gc.profiles(*parse_scenario_csv(scenario_csv, gc))
    elif mode == "contingency":
        if outages is None:
            raise ValueError("contingency mode requires an outage list")
        out = parse_outage_list(outages, gc) if isinstance(outages, str) else np.asarray(outages, np.int32)
        yre, yim, isl = S.contingency_values(gc, out)
        y = (yre, yim)
        p0, q0 = gc.profiles(np.repeat(gc.pd[:, None], len(out), 1), np.repeat(gc.qd[:, None], len(out), 1))
        return JobInputs(p0, q0, y, isl.astype(bool), out)
    else:
        p0, q0 = gc.profiles(gc.pd, gc.qd)
    return JobInputs(p0, q0, y, np.zeros(p0.shape[1], bool), out)


def run(plan: S.NrPlan, gc, mode: str, batch_size: int | None = None, **kw) -> JobResult:
    """batch_runtime.run for one job on one plan.  Tasks removed by the islanding
    pre-check keep status ISLANDED and zero voltages; all others go through
    gbnr_solve (second chance and re-derivation included) in mini-batches of
    ``batch_size`` tasks (JobSpec.batch_size; None = one batch --
    the library itself still splits a batch that exceeds device memory).
    Results do not depend on the batch size."""
    if batch_size is not None and batch_size < 1:
        raise ValueError("batch_size must be >= 1 (JobSpec invariant, SPEC.md:380)")
    t0 = time.perf_counter()
    inp = job_inputs(gc, mode, **kw)
    t_init = time.perf_counter() - t0
    T = inp.p0.shape[1]
    vm0, va0 = gc.v_start()
    keep = np.nonzero(~inp.islanded)[0]
    n = gc.n_bus
    status = np.full(T, ISLANDED, np.int32)
    iters = np.zeros(T, np.int32)
    vm = np.zeros((n, T))
    va = np.zeros((n, T))
    mm = np.full(T, np.inf)
    t1 = time.perf_counter()
    step = int(keep.size) if batch_size is None else int(batch_size)
    device_ms, batches = 0.0, 0
    for b0 in range(0, int(keep.size), max(step, 1)):
        ids = keep[b0:b0 + step]
        y = None if inp.y is None else (np.ascontiguousarray(inp.y[0][:, ids]),
                                        np.ascontiguousarray(inp.y[1][:, ids]))
        r = plan.solve(np.ascontiguousarray(inp.p0[:, ids]), np.ascontiguousarray(inp.q0[:, ids]),
                       vm0, va0, n_tasks=int(ids.size), y=y)
        status[ids], iters[ids], mm[ids] = r.status, r.iterations, r.max_mismatch
        vm[:, ids], va[:, ids] = r.vm, r.va
        device_ms += plan.timing()["total_ms"]
        batches += 1
    t_solve = time.perf_counter() - t1
    report = {"mode": mode, "tasks": T, "solved": int(keep.size), "batches": batches,
              "init_s": t_init, "solve_wall_s": t_solve,
              "device_ms": device_ms,
              "counts": {name: int((status == code).sum()) for name, code in
                         (("converged", CONVERGED), ("diverged", DIVERGED), ("singular", SINGULAR),
                          ("fallback_converged", FALLBACK_CONVERGED), ("islanded", ISLANDED))}}
    return JobResult(status, iters, vm, va, mm, report)
