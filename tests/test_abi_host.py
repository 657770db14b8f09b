"""The C-ABI library on a machine without a GPU (CPU-only checks).

* libgbnr.so loads and exports every entry point include/gbnr.h declares;
* the host-only (device = -1) plan runs the C++ symbolic stage, and its
  structure (permutations, LU pattern, level schedule, counters) equals the
  oracle's restatement of SPEC.md:292-309 exactly;
* there is no CPU fallback: a solve on a host-only plan fails loudly (GBNR_ECONFIG);
* error taxonomy of core.hpp:32-65 at the boundary (codes 2 structural, 3 config).
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import pyoracle as po
import util
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case

HEADER = os.path.join(util.ROOT, "include", "gbnr.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gbnr_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 14
    L = S.lib()
    for nm in names:
        assert hasattr(L, nm), f"{nm} declared in gbnr.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", S.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gbnr_\w+)", out))
    assert set(names) <= exported
    assert set(S.EXPORTS) <= exported


def test_version_and_defaults():
    assert b"sm_100a" in S.lib().gbnr_version()
    o = S.default_options()
    assert o.tol == 1e-8 and o.max_iter == 10 and o.pivot_tol == 1e-3 and o.singular_tol == 1e-14
    assert o.second_chance == 1 and o.jacobian == 0 and o.walkers == 8 and o.headroom == 1
    assert o.n_devices == 1 and o.device_step == 1 and o.chunk_tasks == 0 and o.tile_width == 0


def host_plan(name, **kw):
    gc = load_case(util.case_path(name))
    return gc, S.NrPlan.from_case(gc, device=-1, **kw)


@pytest.mark.parametrize("name", ["case14", "synth118", "synth300", "synth2383", "synth9241"])
def test_symbolic_equals_oracle(name):
    gc, plan = host_plan(name)
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    op = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    a, b = plan.stats(), op.stats()
    for k in po.OraclePlan.STAT_KEYS:
        assert a[k] == b[k], k
    assert a["nnzY"] == ip[-1]
    ea, eb = plan.export(), op.export()
    for k in ("row_fwd", "col_fwd", "col_ptr", "row_ix", "level"):
        np.testing.assert_array_equal(ea[k], eb[k], err_msg=k)
    plan.close()


def test_case14_counters_match_survey():
    """case14 nJ 22, zJ 146, zLU 162, fill 16, D 250, 13 levels."""
    _, plan = host_plan("case14")
    st = plan.stats()
    assert (st["nJ"], st["nnzJ"], st["nnzLU"], st["n_fill"]) == (22, 146, 162, 16)
    assert st["D"] == 250 and st["levels_lu"] == 13 and st["offdiag_pivots"] == 0
    plan.close()


def test_no_cpu_fallback():
    gc, plan = host_plan("case14")
    vm0, va0 = gc.v_start()
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    with pytest.raises(S.GbnrError) as e:
        plan.solve(p0, q0, vm0, va0, n_tasks=4)
    assert e.value.code == 3 and "host-only" in str(e.value)
    plan.close()


def test_config_and_structural_errors():
    gc = load_case(util.case_path("case14"))
    for bad in (dict(max_iter=0), dict(max_iter=31), dict(jacobian=3), dict(second_chance=-1),
                dict(walkers=9), dict(prefetch=-1), dict(n_devices=-1), dict(chunk_tasks=-2),
                dict(tile_width=3), dict(tile_width=34)):
        with pytest.raises(S.GbnrError) as e:
            S.NrPlan.from_case(gc, device=-1, **bad)
        assert e.value.code == 3, bad
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    bad_pq = gc.pq.copy()
    bad_pq[0] = gc.slack  # slack listed as PQ: structural error
    with pytest.raises(S.GbnrError) as e:
        S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, bad_pq, vm0, va0, device=-1)
    assert e.value.code == 2
    assert S.lib().gbnr_last_error()


def test_singular_representative_is_error_4():
    """A structurally present but numerically singular Jacobian at the representative
    V0 cannot be factorized (SingularError, core.hpp:32-65 -> code 4)."""
    gc = load_case(util.case_path("case14"))
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    z = np.zeros_like(yr)
    with pytest.raises(S.GbnrError) as e:
        S.NrPlan(gc.n_bus, ip, ix, z, z, gc.slack, gc.pv, gc.pq, vm0, va0, device=-1)
    assert e.value.code == 4


def test_plan_stats_null_safety():
    _, plan = host_plan("case14")
    out = np.zeros(16, np.int64)
    assert S.lib().gbnr_plan_stats(plan.h, out) == 0
    # export tolerates NULL outputs
    assert S.lib().gbnr_plan_export(plan.h, None, None, None, None, None) == 0
    plan.close()
