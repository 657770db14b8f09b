"""Seeded Monte-Carlo load scenarios (SPEC.md:410-418 ``sample_montecarlo``).

Counter-based: every draw is splitmix64 of (seed, stream, task, bus), so any
rank or GPU can generate exactly its own slice of a batch:

* per-bus load multiplier s ~ U(lo, hi), the same factor on P and Q;
* generator P scaled per task by the batch's total-load ratio so the
  dispatch stays balanced before losses (the slack absorbs losses);
* ``mode="loadpv"`` additionally scales each PV-bus generator by U(0.5, 1.0).

``montecarlo`` is the benchmark workload.  Its generator
rescaling is this repo's choice, not the reference's: SPEC.md's
``sample_montecarlo`` only replaces bus loads and lets the slack absorb the
change.  ``sample_montecarlo`` below is that operation as specified, with the
per-bus distribution table {normal(mu, sigma), uniform(lo, hi), fixed}.

Outputs are element-major [n_bus][n_tasks] (task innermost), the BatchTape
layout of batch_tape.hpp:6-9 and the C ABI.
"""
from __future__ import annotations

import numpy as np

SEED = 210102270
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, stream: int, task: np.ndarray, bus: np.ndarray) -> np.ndarray:
    """U[0,1) keyed by (seed, stream, task, bus); broadcasts task x bus."""
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) + np.uint64(stream))
        h = splitmix64(h + np.asarray(task, np.uint64))
        h = splitmix64(h + np.asarray(bus, np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def montecarlo(gc, n_tasks: int, task0: int = 0, seed: int = SEED, lo: float = 0.8,
               hi: float = 1.2, mode: str = "load"):
    """Returns (p0, q0) [n_bus][n_tasks] in p.u. for tasks task0 .. task0+n_tasks-1."""
    n = gc.n_bus
    tasks = np.arange(task0, task0 + n_tasks, dtype=np.uint64)[None, :]
    buses = np.arange(n, dtype=np.uint64)[:, None]
    s = lo + (hi - lo) * uniform(seed, 0, tasks, buses)         # [n][T]
    p_mw = gc.pd[:, None] * s
    q_mvar = gc.qd[:, None] * s
    tot = gc.pd.sum()
    ratio = (p_mw.sum(axis=0) / tot) if tot != 0.0 else np.ones(n_tasks)
    gen_scale = np.broadcast_to(ratio[None, :], (n, n_tasks)).copy()
    if mode == "loadpv":
        pvmask = np.zeros(n, bool)
        pvmask[gc.pv] = True
        u = 0.5 + 0.5 * uniform(seed, 1, tasks, buses)
        gen_scale = np.where(pvmask[:, None], gen_scale * u, gen_scale)
    elif mode != "load":
        raise ValueError(f"unknown scenario mode {mode!r}")
    gen_scale[gc.slack, :] = 1.0
    return gc.profiles(p_mw, q_mvar, gen_scale)


_KINDS = ("normal", "uniform", "fixed")


def _spec_table(spec, n: int):
    """Per-bus (kind, a, b) arrays from one tuple (every bus) or a list of n tuples."""
    rows = [spec] * n if isinstance(spec, tuple) else list(spec)
    if len(rows) != n:
        raise ValueError(f"distribution table needs {n} rows (one per bus), got {len(rows)}")
    kind = np.empty(n, np.int8)
    a = np.zeros(n)
    b = np.zeros(n)
    for i, r in enumerate(rows):
        k = r[0]
        if k not in _KINDS:
            raise ValueError(f"bus {i}: unknown distribution {k!r}; expected one of {_KINDS}")
        if k == "fixed":
            if len(r) != 2:
                raise ValueError(f"bus {i}: fixed takes one value")
            kind[i], a[i] = 2, float(r[1])
        else:
            if len(r) != 3:
                raise ValueError(f"bus {i}: {k} takes two parameters")
            x, y = float(r[1]), float(r[2])
            if k == "normal" and not (y >= 0.0 and np.isfinite(x) and np.isfinite(y)):
                raise ValueError(f"bus {i}: normal needs finite mu and sigma >= 0")
            if k == "uniform" and not (np.isfinite(x) and np.isfinite(y) and x <= y):
                raise ValueError(f"bus {i}: uniform needs lo <= hi")
            kind[i], a[i], b[i] = (0 if k == "normal" else 1), x, y
    return kind, a, b


def sample_montecarlo(gc, spec, n_tasks: int, task0: int = 0, seed: int = SEED):
    """``sample_montecarlo``: per-bus load multipliers drawn from
    a distribution table -- ('normal', mu, sigma), ('uniform', lo, hi) or
    ('fixed', value); one tuple applies to every bus, else one per bus.  The
    multiplier scales the bus's P and Q load; generator dispatch is unchanged
    (the slack absorbs the difference).  Counter-based and seeded, so the same
    seed gives the same table and any slice of tasks can be drawn on its own.
    Returns (p0, q0) [n_bus][n_tasks] p.u. for tasks task0 .. task0+n_tasks-1."""
    if n_tasks < 1:
        raise ValueError("n_tasks must be >= 1")
    n = gc.n_bus
    kind, a, b = _spec_table(spec, n)
    tasks = np.arange(task0, task0 + n_tasks, dtype=np.uint64)[None, :]
    buses = np.arange(n, dtype=np.uint64)[:, None]
    u0 = uniform(seed, 2, tasks, buses)
    u1 = uniform(seed, 3, tasks, buses)
    # Box-Muller on (0, 1] x [0, 1)
    z = np.sqrt(-2.0 * np.log1p(-u0)) * np.cos(2.0 * np.pi * u1)
    s = np.where(kind[:, None] == 0, a[:, None] + b[:, None] * z,
                 np.where(kind[:, None] == 1, a[:, None] + (b - a)[:, None] * u0,
                          np.broadcast_to(a[:, None], (n, n_tasks))))
    return gc.profiles(gc.pd[:, None] * s, gc.qd[:, None] * s)
