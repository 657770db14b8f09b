"""ctypes bindings for the parity oracle -- TEST INFRASTRUCTURE ONLY.

``Oracle`` wraps oracle/liboracle.so (the C restatement, oracle.c);
``Reference`` wraps oracle/_ref/libgbref.so (the reference's own headers built
in place by ``make -C oracle ref``; present only where /root/reference exists).
Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU arms.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libgbref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, msg, code=0):
        super().__init__(msg)
        self.code = code


class Oracle:
    def __init__(self, path: str = LIB):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_sincos.argtypes = [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_build_ybus.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                     _f64p, _u8p, _f64p, _f64p, C.c_double, _i32p, _i32p, _i32p,
                                     _f64p, _f64p, C.POINTER(C.c_int32)]
        L.orc_amd.argtypes = [C.c_int32, _i32p, _i32p, _i32p]
        L.orc_plan_create.argtypes = [C.c_int32, _i32p, _i32p, _f64p, _f64p, C.c_int32, _i32p,
                                      C.c_int32, _i32p, C.c_int32, _f64p, _f64p, C.c_double,
                                      C.POINTER(C.c_void_p)]
        L.orc_plan_destroy.argtypes = [C.c_void_p]
        L.orc_plan_stats.argtypes = [C.c_void_p, _i64p]
        L.orc_plan_export.argtypes = [C.c_void_p, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.orc_solve.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p, C.c_int32, _f64p, _f64p,
                                C.c_int32, _f64p, _f64p, C.c_int32, C.c_double, C.c_int32,
                                C.c_double, _f64p, _f64p, _i32p, _u8p, _i32p, _f64p, C.c_int32]
        L.orc_refactor.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p, C.c_double, _f64p, _u8p,
                                   C.c_int32]
        L.orc_mismatch.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.orc_branch_flows.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, C.c_int32, _f64p,
                                       _f64p, C.c_void_p, _f64p, _f64p, _f64p, _f64p]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(f"oracle error {rc}: {self.lib.orc_last_error().decode()}", rc)

    def sincos(self, x):
        s, c = C.c_double(), C.c_double()
        out_s = np.empty(len(x)); out_c = np.empty(len(x))
        for i, v in enumerate(np.asarray(x, np.float64)):
            self.lib.orc_sincos(float(v), C.byref(s), C.byref(c))
            out_s[i], out_c[i] = s.value, c.value
        return out_s, out_c

    def build_ybus(self, gc):
        n, nb = gc.n_bus, gc.n_branch
        cap = n + 2 * nb
        indptr = np.zeros(n + 1, np.int32); indices = np.zeros(cap, np.int32)
        diag = np.zeros(n, np.int32); yre = np.zeros(cap); yim = np.zeros(cap)
        nnz = C.c_int32()
        self._check(self.lib.orc_build_ybus(
            n, nb, _i32(gc.br_f), _i32(gc.br_t), _f64(gc.br_r), _f64(gc.br_x), _f64(gc.br_b),
            _f64(gc.br_tap), _f64(gc.br_shift), np.ascontiguousarray(gc.br_on, np.uint8),
            _f64(gc.gs), _f64(gc.bs), float(gc.base_mva), indptr, indices, diag, yre, yim,
            C.byref(nnz)))
        m = nnz.value
        return indptr, indices[:m].copy(), diag, yre[:m].copy(), yim[:m].copy()

    def branch_flows(self, gc, adm, vm, va, outage=None):
        """calc_branch_flows: (S_from, S_to) complex [n_branch][T]."""
        vm = _f64(vm); va = _f64(va)
        T = vm.shape[1]
        nb = gc.n_branch
        out = [np.zeros((nb, T)) for _ in range(4)]
        oa = None if outage is None else _i32(outage)
        self._check(self.lib.orc_branch_flows(
            gc.n_bus, nb, _i32(gc.br_f), _i32(gc.br_t), _f64(adm), T, vm, va,
            None if oa is None else oa.ctypes.data_as(C.c_void_p), *out))
        return out[0] + 1j * out[1], out[2] + 1j * out[3]

    def amd(self, n, col_ptr, row_ix):
        fwd = np.zeros(n, np.int32)
        self._check(self.lib.orc_amd(n, _i32(col_ptr), _i32(row_ix), fwd))
        return fwd

    def plan(self, n_bus, indptr, indices, yre, yim, ref, pv, pq, vm0, va0, pivot_tol=1e-3):
        return OraclePlan(self, n_bus, indptr, indices, yre, yim, ref, pv, pq, vm0, va0, pivot_tol)


class OraclePlan:
    STAT_KEYS = ("nJ", "nnzJ", "nnzLU", "nnzL", "nnzU", "D", "flops_lu", "levels_lu",
                 "levels_fs", "levels_bs", "offdiag_pivots", "npvpq", "n_fill", "max_col",
                 "max_udeps")

    def __init__(self, orc, n_bus, indptr, indices, yre, yim, ref, pv, pq, vm0, va0, pivot_tol):
        self.o = orc
        self.n_bus = n_bus
        self.h = C.c_void_p()
        self._keep = (_i32(indptr), _i32(indices), _f64(yre), _f64(yim), _i32(pv), _i32(pq))
        self.ref, self.pivot_tol = int(ref), float(pivot_tol)
        orc._check(orc.lib.orc_plan_create(
            n_bus, self._keep[0], self._keep[1], self._keep[2], self._keep[3], int(ref),
            self._keep[4], len(pv), self._keep[5], len(pq), _f64(vm0), _f64(va0),
            float(pivot_tol), C.byref(self.h)))
        self.nnzY = int(indptr[-1])

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.o.lib.orc_plan_destroy(self.h)
            self.h = C.c_void_p()

    def stats(self) -> dict:
        out = np.zeros(16, np.int64)
        self.o.lib.orc_plan_stats(self.h, out)
        return {k: int(out[i]) for i, k in enumerate(self.STAT_KEYS)}

    def export(self):
        st = self.stats()
        nJ, z = st["nJ"], st["nnzLU"]
        rf = np.zeros(nJ, np.int32); cf = np.zeros(nJ, np.int32)
        cp = np.zeros(nJ + 1, np.int32); ri = np.zeros(z, np.int32); lev = np.zeros(nJ, np.int32)
        self.o.lib.orc_plan_export(self.h, rf, cf, cp, ri, lev)
        return dict(row_fwd=rf, col_fwd=cf, col_ptr=cp, row_ix=ri, level=lev)

    def solve(self, p0, q0, vm0, va0, n_tasks=None, y=None, tol=1e-8, max_iter=10,
              singular_tol=1e-14, n_threads=None, second_chance=True, _rederive=True):
        p0 = _f64(p0); q0 = _f64(q0); vm0 = _f64(vm0); va0 = _f64(va0)
        if n_tasks is None:
            n_tasks = max(p0.shape[1] if p0.ndim == 2 else 1, vm0.shape[1] if vm0.ndim == 2 else 1)
        ns = p0.shape[1] if p0.ndim == 2 else 1
        nv = vm0.shape[1] if vm0.ndim == 2 else 1
        if y is None:
            yre, yim, ny = _f64(self._keep[2]), _f64(self._keep[3]), 1
        else:
            yre, yim = _f64(y[0]), _f64(y[1])
            ny = yre.shape[1] if yre.ndim == 2 else 1
        n = self.n_bus
        vm = np.zeros((n, n_tasks)); va = np.zeros((n, n_tasks))
        it = np.zeros(n_tasks, np.int32); cv = np.zeros(n_tasks, np.uint8)
        st = np.zeros(n_tasks, np.int32); mm = np.zeros(n_tasks)
        nt = n_threads or os.cpu_count() or 1
        self.o._check(self.o.lib.orc_solve(self.h, n_tasks, yre, yim, ny, p0, q0, ns, vm0, va0, nv,
                                           tol, max_iter, singular_tol, vm, va, it, cv, st, mm, nt))
        second_chance = bool(second_chance)
        if second_chance and _rederive and ny == 1 and int(((st == 2) & (it == 1)).sum()) * 20 > n_tasks:
            # representative re-derivation (SPEC.md DESIGN DECISIONS): the frozen
            # pivots failed for more than 5% of the tasks at their first solve ->
            # restart the batch once from the task with the worst mismatch at V0
            full = lambda a, k: a if (a.ndim == 2 and a.shape[1] == n_tasks) else np.repeat(
                a.reshape(a.shape[0], -1)[:, :1], n_tasks, axis=1)
            f0 = self.mismatch(full(p0, ns), full(q0, ns), full(vm0, nv), full(va0, nv))
            m0 = np.where(np.isnan(f0), np.inf, np.abs(f0)).max(axis=0)
            w = int(np.argmax(m0))
            vw = 0 if nv == 1 else w
            v_m = vm0.reshape(self.n_bus, -1)[:, vw].copy()
            v_a = va0.reshape(self.n_bus, -1)[:, vw].copy()
            ip, ix, _, _, pv, pq = self._keep
            try:
                alt = OraclePlan(self.o, self.n_bus, ip, ix, yre.reshape(-1), yim.reshape(-1), self.ref, pv, pq,
                                 v_m, v_a, self.pivot_tol)
            except OracleError as e:
                if e.code != 4:
                    raise
            else:
                return alt.solve(p0, q0, vm0, va0, n_tasks=n_tasks, tol=tol, max_iter=max_iter,
                                 singular_tol=singular_tol, n_threads=n_threads, second_chance=second_chance,
                                 _rederive=False)
        if second_chance:
            self._second_chance(n_tasks, yre, yim, ny, p0, q0, ns, tol, max_iter, singular_tol,
                                vm, va, it, cv, st, mm)
        return dict(vm=vm, va=va, iterations=it, converged=cv, status=st, max_mismatch=mm)

    def _second_chance(self, n_tasks, yre, yim, ny, p0, q0, ns, tol, max_iter, singular_tol,
                       vm, va, it, cv, st, mm):
        """second_chance_refactorize (open question :436): a task
        whose frozen pivot collapsed (status singular after `it` linear solves) gets a
        fresh threshold-pivoting factorization at its current voltages, kept for the
        rest of its Newton loop, and continues with the remaining budget
        max_iter - (it - 1).  Converged -> status 3 (fallback_converged);
        otherwise the re-run's status.  As the product's plan.cu second_chance: one
        fresh plan from the flagged task with the largest mismatch at its failure
        (first of the largest) re-runs every flagged task, grouped by budget; the
        tasks its pivots do not carry (flagged again) each get their own fresh plan.
        A task whose own fresh factorization is singular stays singular."""
        ip, ix, _, _, pv, pq = self._keep
        col = lambda a, sets, t: (a[:, t] if sets > 1 else (a[:, 0] if a.ndim == 2 else a))  # noqa: E731
        flagged = [int(t) for t in np.nonzero(st == 2)[0] if max_iter - (int(it[t]) - 1) >= 1]
        if not flagged:
            return
        fail = {t: (vm[:, t].copy(), va[:, t].copy(), int(it[t])) for t in flagged}
        w = max(flagged, key=lambda t: (float(mm[t]), -t))  # first of the largest

        def fresh(t):
            try:
                return OraclePlan(self.o, self.n_bus, ip, ix, col(yre, ny, t), col(yim, ny, t), self.ref, pv, pq,
                                  fail[t][0], fail[t][1], self.pivot_tol)
            except OracleError as e:
                if e.code != 4:  # only a numerically singular fresh factorization leaves it failed
                    raise
                return None

        def rerun(sub, grp, b, self_t):
            """grp through sub's pivots; returns the tasks not carried (flagged again)."""
            pp = np.stack([col(p0, ns, t) for t in grp], axis=1)
            qq = np.stack([col(q0, ns, t) for t in grp], axis=1)
            vmg = np.stack([fail[t][0] for t in grp], axis=1)
            vag = np.stack([fail[t][1] for t in grp], axis=1)
            y = None if ny == 1 else (np.ascontiguousarray(yre[:, grp]), np.ascontiguousarray(yim[:, grp]))
            r = sub.solve(pp, qq, vmg, vag, n_tasks=len(grp), y=y, tol=tol, max_iter=b,
                          singular_tol=singular_tol, n_threads=1, second_chance=False)
            left = []
            for j, t in enumerate(grp):
                s2 = int(r["status"][j])
                if s2 == 2 and t != self_t:
                    left.append(t)
                    continue
                st[t] = 3 if s2 == 0 else s2
                cv[t] = 1 if s2 == 0 else 0
                it[t] = fail[t][2] - 1 + int(r["iterations"][j])
                vm[:, t], va[:, t], mm[t] = r["vm"][:, j], r["va"][:, j], r["max_mismatch"][j]
            return left

        # one fresh plan from the worst flagged task for all of them, in one batch per budget
        sub = fresh(w)
        rest = [t for t in flagged if t != w] if sub is None else []
        if sub is not None:
            for b in sorted({max_iter - (fail[t][2] - 1) for t in flagged}):
                rest += rerun(sub, [t for t in flagged if max_iter - (fail[t][2] - 1) == b], b, w)
        # the tasks its pivots did not carry: each its own fresh plan
        for t in sorted(rest):
            own = fresh(t)
            if own is not None:
                rerun(own, [t], max_iter - (fail[t][2] - 1), t)

    def refactor(self, vm, va, singular_tol=1e-14, n_threads=None):
        vm = _f64(vm); va = _f64(va)
        nt_ = vm.shape[1]
        z = self.stats()["nnzLU"]
        lu = np.zeros((z, nt_)); fl = np.zeros(nt_, np.uint8)
        self.o._check(self.o.lib.orc_refactor(self.h, nt_, vm, va, singular_tol, lu, fl,
                                              n_threads or os.cpu_count() or 1))
        return lu, fl

    def mismatch(self, p0, q0, vm, va):
        vm = _f64(vm); nt_ = vm.shape[1]
        f = np.zeros((self.stats()["nJ"], nt_))
        self.o._check(self.o.lib.orc_mismatch(self.h, nt_, _f64(p0), _f64(q0), vm, _f64(va), f))
        return f


class Reference:
    """The reference's own substrate (parse_case, build_ybus, assemble_profiles, amd_order)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_parse_case.restype = C.c_void_p
        L.ref_parse_case.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_free_case.argtypes = [C.c_void_p]
        L.ref_case_dims.argtypes = [C.c_void_p, _i64p]
        L.ref_case_sets.argtypes = [C.c_void_p, _i32p, _i32p]
        L.ref_build_ybus.argtypes = [C.c_void_p, _i32p, _i32p, _i32p, _f64p, _f64p]
        L.ref_profiles.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _f64p, _f64p, _f64p, _f64p,
                                   _f64p, _f64p, _f64p]
        L.ref_case_loads.argtypes = [C.c_void_p, _f64p, _f64p]
        L.ref_ybus_outage.argtypes = [C.c_void_p, C.c_int32, _f64p, _f64p, C.POINTER(C.c_int32)]
        L.ref_amd_order.argtypes = [C.c_int32, _i32p, _i32p, _i32p]
        L.ref_crs_from_coords.argtypes = [C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32,
                                          _i32p, _i32p, _i32p, C.POINTER(C.c_int32)]
        L.ref_crs_to_ccs.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.ref_scatter_lookup.argtypes = [C.c_int32, _i32p, _i32p, _i32p, _i32p, C.c_int32, _i32p,
                                         _i32p, _i32p, _i32p, _i32p]
        L.ref_parse_scenario.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32), C.c_void_p,
                                         C.c_void_p]
        L.ref_parse_outages.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int32), C.c_void_p]

    def err(self):
        return self.lib.ref_last_error().decode()

    def parse(self, text: str):
        rc = C.c_int()
        h = self.lib.ref_parse_case(text.encode(), C.byref(rc))
        if rc.value != 0:
            raise OracleError(f"ref parse error {rc.value}: {self.err()}")
        return RefCase(self, h)

    def branch_flows(self, gc, adm, vm, va, outage=None):
        """calc_branch_flows: (S_from, S_to) complex [n_branch][T]."""
        vm = _f64(vm); va = _f64(va)
        T = vm.shape[1]
        nb = gc.n_branch
        out = [np.zeros((nb, T)) for _ in range(4)]
        oa = None if outage is None else _i32(outage)
        self._check(self.lib.orc_branch_flows(
            gc.n_bus, nb, _i32(gc.br_f), _i32(gc.br_t), _f64(adm), T, vm, va,
            None if oa is None else oa.ctypes.data_as(C.c_void_p), *out))
        return out[0] + 1j * out[1], out[2] + 1j * out[3]

    def amd(self, n, col_ptr, row_ix):
        fwd = np.zeros(n, np.int32)
        if self.lib.ref_amd_order(n, _i32(col_ptr), _i32(row_ix), fwd) != 0:
            raise OracleError(self.err())
        return fwd


class RefCase:
    def __init__(self, ref: Reference, h):
        self.r, self.h = ref, h
        d = np.zeros(6, np.int64)
        ref.lib.ref_case_dims(h, d)
        self.n_bus, self.n_branch, self.slack, self.n_pv, self.n_pq, self.nnzY = map(int, d)

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_free_case(self.h)
            self.h = None

    def sets(self):
        pv = np.zeros(self.n_pv, np.int32); pq = np.zeros(self.n_pq, np.int32)
        self.r.lib.ref_case_sets(self.h, pv, pq)
        return pv, pq

    def ybus(self):
        n, z = self.n_bus, self.nnzY
        ip = np.zeros(n + 1, np.int32); ix = np.zeros(z, np.int32); dg = np.zeros(n, np.int32)
        yr = np.zeros(z); yi = np.zeros(z)
        self.r.lib.ref_build_ybus(self.h, ip, ix, dg, yr, yi)
        return ip, ix, dg, yr, yi

    def outage(self, branch):
        """(y_re, y_im, islands) of ybus_values_with_outage / outage_islands_grid."""
        yr = np.zeros(self.nnzY); yi = np.zeros(self.nnzY); isl = C.c_int32()
        if self.r.lib.ref_ybus_outage(self.h, int(branch), yr, yi, C.byref(isl)) != 0:
            raise OracleError(self.r.err())
        return yr, yi, bool(isl.value)

    def scenario(self, text: str):
        """parse_scenario_csv (case_io.hpp:368-447) -> (p_mw, q_mvar) [n_bus][n_tasks];
        raises OracleError with the reference's error code."""
        nt = C.c_int32()
        rc = self.r.lib.ref_parse_scenario(self.h, text.encode(), C.byref(nt), None, None)
        if rc != 0:
            raise OracleError(self.r.err(), rc)
        p = np.zeros((self.n_bus, nt.value)); q = np.zeros((self.n_bus, nt.value))
        self.r.lib.ref_parse_scenario(self.h, text.encode(), C.byref(nt), p.ctypes.data, q.ctypes.data)
        return p, q

    def outages(self, text: str):
        """parse_outage_list (case_io.hpp:449-471) -> int32 branch indices."""
        n = C.c_int32()
        rc = self.r.lib.ref_parse_outages(self.h, text.encode(), C.byref(n), None)
        if rc != 0:
            raise OracleError(self.r.err(), rc)
        out = np.zeros(n.value, np.int32)
        self.r.lib.ref_parse_outages(self.h, text.encode(), C.byref(n), out.ctypes.data)
        return out

    def loads(self):
        p = np.zeros(self.n_bus); q = np.zeros(self.n_bus)
        self.r.lib.ref_case_loads(self.h, p, q)
        return p, q

    def profiles(self, p_mw, q_mvar):
        p_mw = _f64(p_mw); q_mvar = _f64(q_mvar)
        if p_mw.ndim == 1:
            p_mw = p_mw[:, None].copy(); q_mvar = q_mvar[:, None].copy()
        ns = p_mw.shape[1]
        n = self.n_bus
        p0 = np.zeros((n, ns)); q0 = np.zeros((n, ns))
        vm = np.zeros(n); va = np.zeros(n); vs = np.zeros(n)
        rc = self.r.lib.ref_profiles(self.h, ns, ns, p_mw, q_mvar, p0, q0, vm, va, vs)
        if rc != 0:
            raise OracleError(self.r.err())
        return p0, q0, vm, va
