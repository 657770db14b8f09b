"""Python mirror of the reference solver interface over libgbnr.so (ctypes).

The reference exposes ``nr_solve_batch(case, symbolic, tapes, cfg) ->
TaskResult[]`` after ``initialize``; the
paper's Python front end hands numpy buffers to the C++/CUDA solver through
Cython.  ``NrPlan`` is ``initialize``; ``NrPlan.solve`` is
``nr_solve_batch`` returning the TaskResult fields as arrays; ``newtonpf_batch``
is the MATPOWER-style entry point (Ybus, Sbus, V0, ref, pv, pq).

There is no CPU fallback: if the CUDA library is missing this module raises on
import of the library, and a plan on a machine without a GPU can only be a
host-only (symbolic) plan.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GBNR_LIB", os.path.join(HERE, "libgbnr.so"))

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")

CONVERGED, DIVERGED, SINGULAR = 0, 1, 2
STAT_KEYS = ("nJ", "nnzJ", "nnzLU", "nnzL", "nnzU", "D", "flops_lu", "levels_lu", "levels_fs",
             "levels_bs", "offdiag_pivots", "npvpq", "n_fill", "max_col", "max_udeps", "nnzY")
EXPORTS = ("gbnr_default_options", "gbnr_last_error", "gbnr_version", "gbnr_build_ybus",
           "gbnr_amd_order", "gbnr_plan_create", "gbnr_plan_destroy", "gbnr_plan_stats",
           "gbnr_plan_export", "gbnr_solve", "gbnr_stage", "gbnr_run", "gbnr_fetch",
           "gbnr_last_timing", "gbnr_refactor", "gbnr_walk_info", "gbnr_walk_export",
           "gbnr_solve_batches", "gbnr_contingency_values", "gbnr_branch_admittances",
           "gbnr_branch_flows")


class GbnrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"gbnr error {code}: {msg}")
        self.code = code


class Options(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32), ("pivot_tol", C.c_double),
                ("singular_tol", C.c_double), ("device", C.c_int32), ("ring_rows", C.c_int32),
                ("profile", C.c_int32), ("stage_rows", C.c_int32),
                ("prefetch", C.c_int32), ("headroom", C.c_int32), ("walkers", C.c_int32),
                ("jacobian", C.c_int32), ("second_chance", C.c_int32),
                ("n_devices", C.c_int32), ("device_step", C.c_int32), ("chunk_tasks", C.c_int32),
                ("tile_width", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Load libgbnr.so (built in-tree by ``make``); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built -- run `make` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    L.gbnr_default_options.argtypes = [C.POINTER(Options)]
    L.gbnr_last_error.restype = C.c_char_p
    L.gbnr_version.restype = C.c_char_p
    L.gbnr_build_ybus.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                  _f64p, _u8p, _f64p, _f64p, C.c_double, _i32p, _i32p, _i32p,
                                  _f64p, _f64p, C.POINTER(C.c_int32)]
    L.gbnr_amd_order.argtypes = [C.c_int32, _i32p, _i32p, _i32p]
    L.gbnr_branch_admittances.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                          _f64p, _u8p, _f64p, _f64p, C.c_double, _f64p]
    L.gbnr_branch_flows.argtypes = [C.c_void_p, C.c_int32, _i32p, _i32p, _f64p, C.c_void_p] + [C.c_void_p] * 4
    L.gbnr_contingency_values.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                          _f64p, _u8p, _f64p, _f64p, C.c_double, _i32p, C.c_int32,
                                          _f64p, _f64p, _u8p]
    L.gbnr_plan_create.argtypes = [C.c_int32, _i32p, _i32p, _f64p, _f64p, C.c_int32, _i32p,
                                   C.c_int32, _i32p, C.c_int32, _f64p, _f64p, C.POINTER(Options),
                                   C.POINTER(C.c_void_p)]
    L.gbnr_plan_destroy.argtypes = [C.c_void_p]
    L.gbnr_plan_stats.argtypes = [C.c_void_p, _i64p]
    L.gbnr_plan_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]
    L.gbnr_solve.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                             C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_void_p]
    L.gbnr_stage.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                             C.c_void_p, C.c_void_p, C.c_int32]
    L.gbnr_run.argtypes = [C.c_void_p]
    L.gbnr_fetch.argtypes = [C.c_void_p] + [C.c_void_p] * 6
    L.gbnr_last_timing.argtypes = [C.c_void_p, _f64p]
    L.gbnr_refactor.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_double)]
    L.gbnr_walk_info.argtypes = [C.c_void_p, C.c_int32, _i64p]
    L.gbnr_solve_batches.argtypes = [C.c_void_p, C.c_int32, C.c_int32] + [C.c_void_p] * 10
    L.gbnr_walk_export.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise GbnrError(rc, lib().gbnr_last_error().decode())


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_options(**kw) -> Options:
    o = Options()
    lib().gbnr_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def build_ybus(gc):
    """grid.hpp:208-243 via the C++ host library: (indptr, indices, diag, y_re, y_im)."""
    n, nb = gc.n_bus, gc.n_branch
    cap = n + 2 * nb
    indptr = np.zeros(n + 1, np.int32)
    indices = np.zeros(cap, np.int32)
    diag = np.zeros(n, np.int32)
    yre = np.zeros(cap)
    yim = np.zeros(cap)
    nnz = C.c_int32()
    _check(lib().gbnr_build_ybus(n, nb, _i32(gc.br_f), _i32(gc.br_t), _f64(gc.br_r), _f64(gc.br_x),
                                 _f64(gc.br_b), _f64(gc.br_tap), _f64(gc.br_shift),
                                 np.ascontiguousarray(gc.br_on, np.uint8), _f64(gc.gs),
                                 _f64(gc.bs), float(gc.base_mva), indptr, indices, diag, yre, yim,
                                 C.byref(nnz)))
    m = nnz.value
    return indptr, indices[:m].copy(), diag, yre[:m].copy(), yim[:m].copy()


def contingency_values(gc, outages):
    """N-1 value sets (grid.hpp:245-261 via the C++ host): for every task the base
    Ybus pattern's values with branch outages[t] removed (-1 = base case).
    Returns (y_re, y_im) [nnzY][T] and islanded [T] (bool)."""
    outages = _i32(outages)
    T = len(outages)
    nnz = int(build_ybus(gc)[0][-1])
    yre = np.empty((nnz, T))
    yim = np.empty((nnz, T))
    isl = np.zeros(T, np.uint8)
    _check(lib().gbnr_contingency_values(
        gc.n_bus, gc.n_branch, _i32(gc.br_f), _i32(gc.br_t), _f64(gc.br_r), _f64(gc.br_x),
        _f64(gc.br_b), _f64(gc.br_tap), _f64(gc.br_shift), np.ascontiguousarray(gc.br_on, np.uint8),
        _f64(gc.gs), _f64(gc.bs), float(gc.base_mva), outages, T, yre, yim, isl))
    return yre, yim, isl.astype(bool)


def branch_admittances(gc) -> np.ndarray:
    """[n_branch][8] (ff, ft, tf, tt) as (re, im) -- grid.hpp:195-206 via the C++ host."""
    adm = np.zeros((gc.n_branch, 8))
    _check(lib().gbnr_branch_admittances(
        gc.n_bus, gc.n_branch, _i32(gc.br_f), _i32(gc.br_t), _f64(gc.br_r), _f64(gc.br_x),
        _f64(gc.br_b), _f64(gc.br_tap), _f64(gc.br_shift), np.ascontiguousarray(gc.br_on, np.uint8),
        _f64(gc.gs), _f64(gc.bs), float(gc.base_mva), adm))
    return adm


def amd_order(n, col_ptr, row_ix) -> np.ndarray:
    fwd = np.zeros(n, np.int32)
    _check(lib().gbnr_amd_order(n, _i32(col_ptr), _i32(row_ix), fwd))
    return fwd


@dataclass
class TaskResults:
    """TaskResult fields for a batch, element-major V."""
    vm: np.ndarray
    va: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray
    status: np.ndarray
    max_mismatch: np.ndarray


class NrPlan:
    """``initialize``: frozen symbolic state on one device."""

    def __init__(self, n_bus, indptr, indices, y_re, y_im, ref, pv, pq, vm0, va0,
                 device: int = 0, **opts):
        self.n_bus = int(n_bus)
        self.h = C.c_void_p()
        self.opts = default_options(device=device, **opts)
        self._y = (_f64(y_re), _f64(y_im))
        _check(lib().gbnr_plan_create(self.n_bus, _i32(indptr), _i32(indices), self._y[0],
                                      self._y[1], int(ref), _i32(pv), len(pv), _i32(pq), len(pq),
                                      _f64(vm0), _f64(va0), C.byref(self.opts), C.byref(self.h)))
        self._n_tasks = 0

    @classmethod
    def from_case(cls, gc, device: int = 0, **opts):
        ip, ix, _, yr, yi = build_ybus(gc)
        vm0, va0 = gc.v_start()
        return cls(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, device=device,
                   **opts)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().gbnr_plan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        out = np.zeros(16, np.int64)
        _check(lib().gbnr_plan_stats(self.h, out))
        return {k: int(out[i]) for i, k in enumerate(STAT_KEYS)}

    def export(self) -> dict:
        st = self.stats()
        nJ, z = st["nJ"], st["nnzLU"]
        d = dict(row_fwd=np.zeros(nJ, np.int32), col_fwd=np.zeros(nJ, np.int32),
                 col_ptr=np.zeros(nJ + 1, np.int32), row_ix=np.zeros(z, np.int32),
                 level=np.zeros(nJ, np.int32))
        _check(lib().gbnr_plan_export(self.h, *(_ptr(d[k]) for k in
                                               ("row_fwd", "col_fwd", "col_ptr", "row_ix", "level"))))
        return d

    def _sets(self, a, n_tasks, name="array"):
        a = _f64(a)
        if a.shape[0] != self.n_bus:
            raise ValueError(f"{name} must have n_bus = {self.n_bus} rows, got {a.shape[0]}")
        if a.ndim == 1:
            return a, 1
        if a.ndim != 2 or a.shape[1] not in (1, n_tasks):
            raise ValueError(f"{name}: set count must be 1 or n_tasks")
        return a, a.shape[1]

    def _inputs(self, p0, q0, vm0, va0, n_tasks):
        """Validated (p0, q0, n_ssets, vm0, va0, n_vsets): q0 must have p0's set
        count and va0 vm0's, or the C side would read past a host array."""
        p0 = _f64(p0); vm0 = _f64(vm0)
        if n_tasks is None:
            n_tasks = max(p0.shape[1] if p0.ndim == 2 else 1, vm0.shape[1] if vm0.ndim == 2 else 1)
        p0, ns = self._sets(p0, n_tasks, "p0")
        q0, nq = self._sets(q0, n_tasks, "q0")
        vm0, nv = self._sets(vm0, n_tasks, "vm0")
        va0, na = self._sets(va0, n_tasks, "va0")
        if nq != ns:
            raise ValueError(f"q0 has {nq} sets but p0 has {ns}")
        if na != nv:
            raise ValueError(f"va0 has {na} sets but vm0 has {nv}")
        return n_tasks, p0, q0, ns, vm0, va0, nv

    def stage(self, p0, q0, vm0, va0, n_tasks: int | None = None):
        n_tasks, p0, q0, ns, vm0, va0, nv = self._inputs(p0, q0, vm0, va0, n_tasks)
        self._keep = (p0, q0, vm0, va0)
        _check(lib().gbnr_stage(self.h, n_tasks, _ptr(p0), _ptr(q0), ns, _ptr(vm0), _ptr(va0), nv))
        self._n_tasks = n_tasks

    def run(self):
        _check(lib().gbnr_run(self.h))

    def fetch(self) -> TaskResults:
        n, T = self.n_bus, self._n_tasks
        r = TaskResults(np.empty((n, T)), np.empty((n, T)), np.empty(T, np.int32),
                        np.empty(T, np.uint8), np.empty(T, np.int32), np.empty(T))
        _check(lib().gbnr_fetch(self.h, _ptr(r.vm), _ptr(r.va), _ptr(r.iterations),
                                _ptr(r.converged), _ptr(r.status), _ptr(r.max_mismatch)))
        return r

    def solve(self, p0, q0, vm0, va0, n_tasks: int | None = None, y=None) -> TaskResults:
        """``nr_solve_batch`` through gbnr_solve: H2D, solve, D2H.
        ``y`` = (y_re, y_im) [nnzY] (a new shared value set) or [nnzY][T] (one per
        task, e.g. N-1 contingencies from ``contingency_values``)."""
        n_tasks, p0, q0, ns, vm0, va0, nv = self._inputs(p0, q0, vm0, va0, n_tasks)
        yre = yim = None
        ny = 1
        if y is not None:
            yre, yim = _f64(y[0]), _f64(y[1])
            ny = yre.shape[1] if yre.ndim == 2 else 1
            if yre.shape != yim.shape or ny not in (1, n_tasks):
                raise ValueError("y_re / y_im must share one shape [nnzY] or [nnzY][n_tasks]")
        n, T = self.n_bus, n_tasks
        r = TaskResults(np.empty((n, T)), np.empty((n, T)), np.empty(T, np.int32),
                        np.empty(T, np.uint8), np.empty(T, np.int32), np.empty(T))
        _check(lib().gbnr_solve(self.h, T, _ptr(yre), _ptr(yim), ny, _ptr(p0), _ptr(q0), ns,
                                _ptr(vm0), _ptr(va0), nv, _ptr(r.vm), _ptr(r.va), _ptr(r.iterations),
                                _ptr(r.converged), _ptr(r.status), _ptr(r.max_mismatch)))
        self._n_tasks = T
        return r

    def solve_batches(self, p0s, q0s, vm0, va0, outs=None):
        """Pipelined sequence of batches (gbnr_solve_batches): per-task injections
        p0s[i]/q0s[i] [n][T], shared start voltages; returns a list of TaskResults
        (or fills the preallocated `outs`)."""
        nb = len(p0s)
        if nb == 0 or len(q0s) != nb:
            raise ValueError("solve_batches needs one q0 per p0 and at least one batch")
        T = p0s[0].shape[1]
        n = self.n_bus
        p0s = [_f64(a) for a in p0s]
        q0s = [_f64(a) for a in q0s]
        for a in p0s + q0s:
            if a.shape != (n, T):
                raise ValueError(f"every batch's p0/q0 must be [n_bus][T] = {(n, T)}, got {a.shape}")
        if _f64(vm0).shape != (n,) or _f64(va0).shape != (n,):
            raise ValueError("solve_batches takes shared start voltages vm0/va0 [n_bus]")
        if outs is None:
            outs = [TaskResults(np.empty((n, T)), np.empty((n, T)), np.empty(T, np.int32),
                                np.empty(T, np.uint8), np.empty(T, np.int32), np.empty(T))
                    for _ in range(nb)]
        P = C.c_void_p * nb
        arr = lambda xs: P(*[x.ctypes.data for x in xs])  # noqa: E731
        self._keep = (p0s, q0s)
        _check(lib().gbnr_solve_batches(
            self.h, nb, T, arr(p0s), arr(q0s), _ptr(_f64(vm0)), _ptr(_f64(va0)),
            arr([o.vm for o in outs]), arr([o.va for o in outs]), arr([o.iterations for o in outs]),
            arr([o.converged for o in outs]), arr([o.status for o in outs]),
            arr([o.max_mismatch for o in outs])))
        return outs

    def branch_flows(self, gc, outages=None):
        """calc_branch_flows on the last solve: (S_from, S_to)
        complex [n_branch][T]; loading percent = 100 |S| / (rateA / baseMVA)."""
        nb, T = gc.n_branch, self._n_tasks
        adm = branch_admittances(gc)
        out = [np.empty((nb, T)) for _ in range(4)]
        oa = None if outages is None else _i32(outages)
        _check(lib().gbnr_branch_flows(self.h, nb, _i32(gc.br_f), _i32(gc.br_t), adm, _ptr(oa),
                                       *[_ptr(o) for o in out]))
        return out[0] + 1j * out[1], out[2] + 1j * out[3]

    def timing(self) -> dict:
        out = np.zeros(24)
        _check(lib().gbnr_last_timing(self.h, out))
        keys = ("npm", "jacobian", "lu", "fsbs", "vupdate", "total")
        d = {f"{k}_ms": float(out[i]) for i, k in enumerate(keys)}
        d.update({f"{k}_launches": int(out[6 + i]) for i, k in enumerate(keys[:5])})
        d["iterations"] = int(out[12])
        d["tasks"] = int(out[13])
        d["lu_tile_launches"] = int(out[14])
        d["lu_task_launches"] = int(out[15])
        d["converged"] = int(out[16])
        d["diverged"] = int(out[17])
        d["singular"] = int(out[18])
        d["fallback_converged"] = int(out[20])  # second-chance successes (included in converged)
        d["rederived"] = int(out[21])  # batch restarted from a re-derived representative task
        d["kernels"] = int(out[19])
        return d

    WALK_KEYS = ("steps", "walkers", "phases", "rows", "page_words", "pages", "barriers",
                 "stream_words", "events", "ring_dep_rows", "fetched_rows", "n_ops", "n_copies",
                 "smem_bytes", "ring_rows", "stage_rows", "global_steps", "global_deps",
                 "scratch_rows")

    def walk_info(self, which: int) -> dict:
        out = np.zeros(20, np.int64)
        _check(lib().gbnr_walk_info(self.h, int(which), out))
        return {k: int(out[i]) for i, k in enumerate(self.WALK_KEYS)}

    def walk_export(self, which: int) -> dict:
        """The device program of a tile walk (walk.hpp) as numpy arrays."""
        info = self.walk_info(which)
        st = self.stats()
        sizes = (info["stream_words"], info["walkers"] + 1, st["nJ"], st["nnzLU"], st["nJ"],
                 st["nJ"] + 1)
        names = ("stream", "wpage0", "owner", "tape_of_ccs", "lslot", "ucrs0")
        d = dict(info=info)
        for part, nm in enumerate(names):
            a = np.zeros(sizes[part], np.int32)
            _check(lib().gbnr_walk_export(self.h, int(which), part, a.ctypes.data_as(C.c_void_p)))
            d[nm] = a
        return d

    def refactor(self, reps: int = 1, want_lu: bool = True):
        """LU-only pass on the staged voltages; returns (lu [nnzLU][T] or None, flags, ms/rep)."""
        T = self._n_tasks
        lu = np.empty((self.stats()["nnzLU"], T)) if want_lu else None
        flags = np.empty(T, np.uint8)
        ms = C.c_double()
        _check(lib().gbnr_refactor(self.h, int(reps), _ptr(lu), _ptr(flags), C.byref(ms)))
        return lu, flags, ms.value


def newtonpf_batch(Ybus, Sbus, V0, ref, pv, pq, tol=1e-8, max_it=10, device=0):
    """MATPOWER ``newtonpf`` semantics, batched: Ybus (scipy CSR, shared pattern and
    values), Sbus [n][T] complex, V0 [n] or [n][T] complex -> (V [n][T], success [T],
    iterations [T])."""
    Y = Ybus.tocsr()
    Y.sort_indices()
    n = Y.shape[0]
    V0 = np.asarray(V0)
    vm0, va0 = np.abs(V0), np.angle(V0)
    rep_vm = vm0 if vm0.ndim == 1 else vm0[:, 0]
    rep_va = va0 if va0.ndim == 1 else va0[:, 0]
    plan = NrPlan(n, Y.indptr, Y.indices, Y.data.real.copy(), Y.data.imag.copy(), ref, pv, pq,
                  rep_vm, rep_va, device=device, tol=tol, max_iter=max_it)
    S = np.asarray(Sbus)
    r = plan.solve(S.real.copy(), S.imag.copy(), vm0, va0)
    plan.close()
    return r.vm * np.exp(1j * r.va), r.converged.astype(bool), r.iterations
