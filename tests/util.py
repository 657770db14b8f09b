"""Shared test helpers (pure numpy; no product or oracle logic)."""
from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = os.path.join(ROOT, "cases")


def case_path(name: str) -> str:
    return os.path.join(CASES, f"{name}.m")


def j_pattern_ccs(n, indptr, indices, ref, pv, pq):
    """Reduced Jacobian pattern in CCS, MATPOWER ordering
    rows/cols [th(pv;pq), |V|(pq)], structural diagonal included."""
    jth = -np.ones(n, np.int64); jvm = -np.ones(n, np.int64)
    npv, npq = len(pv), len(pq)
    jth[pv] = np.arange(npv); jth[pq] = npv + np.arange(npq)
    jvm[pq] = npv + npq + np.arange(npq)
    nJ = npv + 2 * npq
    rows, cols = [], []
    for r in range(n):
        for q in range(indptr[r], indptr[r + 1]):
            k = indices[q]
            for a in (jth[r], jvm[r]):
                for b in (jth[k], jvm[k]):
                    if a >= 0 and b >= 0:
                        rows.append(a); cols.append(b)
    rows += list(range(nJ)); cols += list(range(nJ))
    key = np.unique(np.array(cols, np.int64) * nJ + np.array(rows, np.int64))
    c = key // nJ; r = key % nJ
    col_ptr = np.zeros(nJ + 1, np.int32)
    np.add.at(col_ptr, c + 1, 1)
    col_ptr = np.cumsum(col_ptr).astype(np.int32)
    return nJ, col_ptr, r.astype(np.int32)
