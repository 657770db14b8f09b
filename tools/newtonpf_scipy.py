"""Independent cross-check: MATPOWER ``newtonpf`` in scipy (SuperLU).

Not the oracle and not the product -- a third implementation used (a) by
tools/gen_cases.py to solve the synthetic base cases and (b) by tests to
cross-check the oracle on real data.  Algorithm as published in MATPOWER
(newtonpf.m / dSbus_dV.m), the pandapower baseline the paper compares against
(PAPER.md:504).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def ybus_matrix(indptr, indices, yre, yim, n):
    return sp.csr_matrix((np.asarray(yre) + 1j * np.asarray(yim), indices, indptr), shape=(n, n))


def dsbus_dv(Y, V):
    n = V.shape[0]
    Ibus = Y @ V
    diagV = sp.diags(V)
    diagI = sp.diags(Ibus)
    diagVn = sp.diags(V / np.abs(V))
    dS_dVm = diagV @ np.conj(Y @ diagVn) + np.conj(diagI) @ diagVn
    dS_dVa = 1j * diagV @ np.conj(diagI - Y @ diagV)
    return dS_dVm, dS_dVa


def newtonpf(Y, Sbus, V0, ref, pv, pq, tol=1e-8, max_it=10):
    """Returns (V, success, iterations) with MATPOWER's iteration convention."""
    V = V0.astype(np.complex128).copy()
    Va = np.angle(V)
    Vm = np.abs(V)
    pvpq = np.r_[pv, pq]
    npv, npq = len(pv), len(pq)
    j1, j2 = 0, npv + npq
    mis = V * np.conj(Y @ V) - Sbus
    F = np.r_[mis[pvpq].real, mis[pq].imag]
    it = 0
    converged = np.max(np.abs(F)) < tol
    while not converged and it < max_it:
        it += 1
        dS_dVm, dS_dVa = dsbus_dv(Y, V)
        J11 = dS_dVa[np.ix_(pvpq, pvpq)].real
        J12 = dS_dVm[np.ix_(pvpq, pq)].real
        J21 = dS_dVa[np.ix_(pq, pvpq)].imag
        J22 = dS_dVm[np.ix_(pq, pq)].imag
        J = sp.vstack([sp.hstack([J11, J12]), sp.hstack([J21, J22])], format="csc")
        dx = -spla.spsolve(J, F)
        Va[pvpq] += dx[j1:j2]
        Vm[pq] += dx[j2:]
        V = Vm * np.exp(1j * Va)
        Vm = np.abs(V)
        Va = np.angle(V)
        mis = V * np.conj(Y @ V) - Sbus
        F = np.r_[mis[pvpq].real, mis[pq].imag]
        converged = np.max(np.abs(F)) < tol
    return V, bool(converged), it
