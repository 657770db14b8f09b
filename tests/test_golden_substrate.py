"""Substrate parity against golden vectors produced by the REFERENCE ITSELF.

tests/golden/*.npz were written by tools/make_golden.py from the reference's own
headers (parse_case, build_ybus, assemble_profiles, amd_order -- compiled in
place into oracle/_ref).  Checked here, bit for bit:
  * the oracle's restatement (oracle.c: orc_build_ybus, orc_amd),
  * the product's host side (libgbnr.so: gbnr_build_ybus, gbnr_amd_order --
    CPU-only entry points of the C ABI, no device needed),
  * the Python case parser / profile assembly (paper_2101_02270_b200.case).
Where oracle/_ref is present (this container) the fixtures are re-derived from
the live reference as well, so a stale fixture cannot hide a regression.
"""
import os

import numpy as np
import pytest

import pyoracle as po
import util
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case

GOLD = os.path.join(util.ROOT, "tests", "golden")
CASES = ("case14", "synth30", "synth118", "synth300", "synth2383", "synth9241")


def gold(name):
    return dict(np.load(os.path.join(GOLD, f"{name}.npz")))


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


@pytest.mark.parametrize("name", CASES)
def test_case_parse_and_sets(name):
    g = gold(name)
    gc = load_case(util.case_path(name))
    assert gc.n_bus == g["n_bus"] and gc.n_branch == g["n_branch"]
    assert gc.slack == g["slack"]
    np.testing.assert_array_equal(gc.pv, g["pv"])
    np.testing.assert_array_equal(gc.pq, g["pq"])


@pytest.mark.parametrize("name", CASES)
def test_ybus_bitwise(name, orc):
    g = gold(name)
    gc = load_case(util.case_path(name))
    for impl in (S.build_ybus, orc.build_ybus):
        ip, ix, dg, yr, yi = impl(gc)
        np.testing.assert_array_equal(ip, g["indptr"])
        np.testing.assert_array_equal(ix, g["indices"])
        np.testing.assert_array_equal(dg, g["diag"])
        np.testing.assert_array_equal(yr, g["y_re"])
        np.testing.assert_array_equal(yi, g["y_im"])


@pytest.mark.parametrize("name", CASES)
def test_profiles_and_v0_bitwise(name):
    g = gold(name)
    gc = load_case(util.case_path(name))
    np.testing.assert_array_equal(gc.pd, g["p_mw"])
    np.testing.assert_array_equal(gc.qd, g["q_mvar"])
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    np.testing.assert_array_equal(p0[:, 0], g["p0"])
    np.testing.assert_array_equal(q0[:, 0], g["q0"])
    s = g["scale_3"]
    p3, q3 = gc.profiles(gc.pd[:, None] * s, gc.qd[:, None] * s)
    np.testing.assert_array_equal(p3, g["p0_3"])
    np.testing.assert_array_equal(q3, g["q0_3"])
    vm0, va0 = gc.v_start()
    np.testing.assert_array_equal(vm0, g["vm_start"])
    np.testing.assert_array_equal(va0, g["va_start"])


@pytest.mark.parametrize("name", CASES)
def test_jacobian_pattern_and_amd(name, orc):
    g = gold(name)
    nJ, cp, ri = util.j_pattern_ccs(int(g["n_bus"]), g["indptr"], g["indices"], int(g["slack"]),
                                    g["pv"], g["pq"])
    assert nJ == g["nJ"]
    np.testing.assert_array_equal(cp, g["j_col_ptr"])
    np.testing.assert_array_equal(ri, g["j_row_ix"])
    np.testing.assert_array_equal(orc.amd(nJ, cp, ri), g["amd_fwd"])
    np.testing.assert_array_equal(S.amd_order(nJ, cp, ri), g["amd_fwd"])


@pytest.mark.parametrize("name", CASES)
def test_contingency_values_bitwise(name):
    """N-1 value sets on the fixed pattern (ybus_values_with_outage, grid.hpp:245-255)
    and the islanding pre-check (outage_islands_grid, grid.hpp:257-261) against the
    reference's own functions."""
    g = gold(name)
    gc = load_case(util.case_path(name))
    br = g["outage_branches"]
    yre, yim, isl = S.contingency_values(gc, np.r_[br, -1])
    np.testing.assert_array_equal(yre[:, :-1], g["outage_y_re"])
    np.testing.assert_array_equal(yim[:, :-1], g["outage_y_im"])
    np.testing.assert_array_equal(isl[:-1], g["outage_islands"].astype(bool))
    np.testing.assert_array_equal(yre[:, -1], g["y_re"])  # -1 = the base case
    np.testing.assert_array_equal(yim[:, -1], g["y_im"])
    if len(g["islands_all"]):
        _, _, isl_all = S.contingency_values(gc, np.arange(gc.n_branch))
        np.testing.assert_array_equal(isl_all, g["islands_all"].astype(bool))


def test_amd_kats():
    """SPEC.md:289 (diagonal -> identity) and :290 (arrow: zero fill; the reference
    puts the hub at n-2 because of its lowest-index tie-break)."""
    k = dict(np.load(os.path.join(GOLD, "sparse_kats.npz")))
    n = 10
    ident = np.arange(n, dtype=np.int32)
    np.testing.assert_array_equal(S.amd_order(n, np.arange(n + 1, dtype=np.int32), ident),
                                  k["amd_diag_fwd"])
    np.testing.assert_array_equal(k["amd_diag_fwd"], ident)
    fwd = S.amd_order(n, k["amd_arrow_col_ptr"], k["amd_arrow_row_ix"])
    np.testing.assert_array_equal(fwd, k["amd_arrow_fwd"])
    assert fwd[0] == n - 2


def test_sparse_kats_values():
    """The SPEC.md sparse_core examples as the reference evaluates them."""
    k = dict(np.load(os.path.join(GOLD, "sparse_kats.npz")))
    assert k["crs_n2_row_ptr"].tolist() == [0, 2, 3]
    assert k["crs_n2_col_ix"].tolist() == [0, 1, 1]
    assert k["crs_n2_diag"].tolist() == [0, 2]
    assert k["crs_n1_empty_col_ix"].tolist() == [0]
    assert k["crs_fig4a_diag"].tolist() == [0, 4, 6]
    assert k["ccs_upper2_col_ptr"].tolist() == [0, 1, 3]
    assert k["scatter_swap_lookup"].tolist() == [3, 1, 2, 0]


@pytest.mark.skipif(not os.path.exists(po.REF_LIB), reason="oracle/_ref (reference build) absent")
@pytest.mark.parametrize("name", ("case14", "synth300"))
def test_golden_is_the_live_reference(name):
    ref = po.Reference()
    g = gold(name)
    with open(util.case_path(name)) as fh:
        rc = ref.parse(fh.read())
    ip, ix, dg, yr, yi = rc.ybus()
    np.testing.assert_array_equal(ip, g["indptr"])
    np.testing.assert_array_equal(yr, g["y_re"])
    np.testing.assert_array_equal(yi, g["y_im"])
    np.testing.assert_array_equal(ref.amd(int(g["nJ"]), g["j_col_ptr"], g["j_row_ix"]),
                                  g["amd_fwd"])


@pytest.mark.skipif(not os.path.exists(po.REF_LIB), reason="oracle/_ref (reference build) absent")
def test_reference_error_taxonomy():
    """SPEC.md:129 duplicate slack -> StructuralError; malformed number -> ParseError
    naming its line; the Python parser raises the same categories."""
    from paper_2101_02270_b200.case import CaseError, parse_matpower
    ref = po.Reference()
    with open(util.case_path("case14")) as fh:
        txt = fh.read()
    import re
    dup = re.sub(r"^(\s*2\s+)2(\s+21\.7)", r"\g<1>3\2", txt, count=1, flags=re.M)
    assert dup != txt
    with pytest.raises(po.OracleError, match="error 2"):
        ref.parse(dup)
    with pytest.raises(CaseError) as e:
        parse_matpower(dup)
    assert e.value.code == 2
    bad = txt.replace("47.8", "47.8x", 1)
    with pytest.raises(po.OracleError, match="error 1"):
        ref.parse(bad)
    with pytest.raises(CaseError) as e:
        parse_matpower(bad)
    assert e.value.code == 1
