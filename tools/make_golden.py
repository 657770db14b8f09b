"""Generate tests/golden/*.npz from the REFERENCE ITSELF (test fixtures).

Runs the reference's own header-only substrate, compiled in place from
/root/reference/proj/include by `make -C oracle ref` into oracle/_ref/libgbref.so
(oracle/ref_shim.cpp), on every case under cases/ and stores what it returns:

  * parse_case      case_io.hpp:345-351 -> n_bus, n_branch, slack, pv, pq
                    (typing rule case_io.hpp:228-236, finalize_case grid.hpp:123-173)
  * build_ybus      grid.hpp:208-243   -> indptr, indices, diag_ptr, y_re, y_im
  * assemble_profiles grid.hpp:299-344 -> p0, q0 (case loads and a 3-set scaled
                    table), vm_start, va_start (the V0 rule :331-342)
  * amd_order       amd.hpp:29-157     -> forward permutation of the reduced
                    Jacobian pattern (built by tests/util.py)
  * ybus_values_with_outage grid.hpp:245-255 -> N-1 value sets for a few branches,
    outage_islands_grid grid.hpp:257-261 -> the islanding pre-check (every branch
    where the case is small enough)
  * the SPEC.md known-answer examples of sparse_core

/root/reference does not exist on the GPU box; the fixtures are committed and
the tests only read them.  Usage:  python tools/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import pyoracle as po  # noqa: E402
import util  # noqa: E402

CASES = ("case14", "synth30", "synth118", "synth300", "synth2383", "synth9241")
OUT = os.path.join(ROOT, "tests", "golden")


def case_golden(ref: po.Reference, name: str) -> dict:
    with open(util.case_path(name)) as fh:
        rc = ref.parse(fh.read())
    pv, pq = rc.sets()
    ip, ix, dg, yr, yi = rc.ybus()
    p_mw, q_mvar = rc.loads()
    p0, q0, vm0, va0 = rc.profiles(p_mw, q_mvar)
    scale = np.array([0.8, 1.0, 1.2])
    p3, q3, _, _ = rc.profiles(p_mw[:, None] * scale, q_mvar[:, None] * scale)
    nJ, cp, ri = util.j_pattern_ccs(rc.n_bus, ip, ix, rc.slack, pv, pq)
    fwd = ref.amd(nJ, cp, ri)
    # N-1: ybus_values_with_outage for some branches, islanding for every branch
    nb = rc.n_branch
    pick = np.arange(nb) if nb <= 64 else np.unique(np.r_[0, 1, nb // 2, nb - 1,
                                                          np.random.default_rng(7).integers(0, nb, 4)])
    outs = [rc.outage(int(b)) for b in pick]
    islands = np.array([rc.outage(b)[2] for b in range(nb)], np.uint8) if nb <= 4096 else \
        np.array([], np.uint8)
    return dict(n_bus=rc.n_bus, n_branch=rc.n_branch, slack=rc.slack, pv=pv, pq=pq,
                indptr=ip, indices=ix, diag=dg, y_re=yr, y_im=yi, p_mw=p_mw, q_mvar=q_mvar,
                p0=p0[:, 0], q0=q0[:, 0], p0_3=p3, q0_3=q3, scale_3=scale, vm_start=vm0,
                va_start=va0, nJ=nJ, j_col_ptr=cp, j_row_ix=ri, amd_fwd=fwd,
                outage_branches=pick.astype(np.int32),
                outage_y_re=np.stack([o[0] for o in outs], 1), outage_y_im=np.stack([o[1] for o in outs], 1),
                outage_islands=np.array([o[2] for o in outs], np.uint8), islands_all=islands)


def sparse_kats(ref: po.Reference) -> dict:
    """SPEC.md sparse_core examples, evaluated by the reference."""
    L = ref.lib
    out = {}

    def crs(n_rows, n_cols, entries):
        r = np.array([e[0] for e in entries], np.int32)
        c = np.array([e[1] for e in entries], np.int32)
        cap = len(entries) + n_rows
        rp = np.zeros(n_rows + 1, np.int32); ci = np.zeros(cap, np.int32)
        dg = np.zeros(n_rows, np.int32); nnz = po.C.c_int32()
        assert L.ref_crs_from_coords(n_rows, n_cols, len(entries), r, c, cap, rp, ci, dg,
                                     po.C.byref(nnz)) == 0, ref.err()
        return rp, ci[:nnz.value].copy(), dg

    # SPEC.md:52 n=2 {(0,0),(0,1),(1,1)}; :53 n=1 empty (diagonal inserted);
    # :54 Fig. 4a 3x3 shape
    for key, (n, ent) in {"n2": (2, [(0, 0), (0, 1), (1, 1)]), "n1_empty": (1, []),
                          "fig4a": (3, [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (2, 0), (2, 2)])}.items():
        rp, ci, dg = crs(n, n, ent)
        out[f"crs_{key}_row_ptr"], out[f"crs_{key}_col_ix"], out[f"crs_{key}_diag"] = rp, ci, dg
    # SPEC.md:61 upper-triangular 2x2 -> CCS col_ptr [0,1,3]
    rp, ci, _ = crs(2, 2, [(0, 0), (0, 1), (1, 1)])
    cp = np.zeros(3, np.int32); rix = np.zeros(3, np.int32); mp = np.zeros(3, np.int32)
    assert L.ref_crs_to_ccs(2, 2, rp, ci, cp, rix, mp) == 0, ref.err()
    out["ccs_upper2_col_ptr"], out["ccs_upper2_row_ix"], out["ccs_upper2_map"] = cp, rix, mp
    # SPEC.md:71 scatter lookup with the swap permutation on a full 2x2
    rp, ci, _ = crs(2, 2, [(0, 0), (0, 1), (1, 0), (1, 1)])
    cp = np.zeros(3, np.int32); rix = np.zeros(4, np.int32); mp = np.zeros(4, np.int32)
    assert L.ref_crs_to_ccs(2, 2, rp, ci, cp, rix, mp) == 0, ref.err()
    swap = np.array([1, 0], np.int32); ident = np.array([0, 1], np.int32)
    lk = np.zeros(4, np.int32)
    assert L.ref_scatter_lookup(2, rp, ci, swap, swap, 2, cp, rix, ident, ident, lk) == 0, ref.err()
    out["scatter_swap_lookup"] = lk
    # SPEC.md:289 AMD of a diagonal matrix; SPEC.md:290 arrow matrix (hub = 0)
    n = 10
    out["amd_diag_fwd"] = ref.amd(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32))
    cols = [[0] + list(range(1, n))] + [[0, j] for j in range(1, n)]
    cp = np.cumsum([0] + [len(c) for c in cols]).astype(np.int32)
    out["amd_arrow_col_ptr"] = cp
    out["amd_arrow_row_ix"] = np.concatenate([np.array(c, np.int32) for c in cols])
    out["amd_arrow_fwd"] = ref.amd(n, cp, out["amd_arrow_row_ix"])
    return out


SCENARIO_TEXTS = {
    "valid_two_rows": "bus:4:p,bus:4:q,bus:14:p\n10,2,5\n11,3,6\n",
    "valid_crlf_blank": "bus:9:q\r\n\r\n16.6\r\n  \n17\n",
    "valid_neg_exp": "bus:2:p,bus:3:q\n-1.5e1,0.25\n",
    "bad_field": "bus:4:x\n1\n",
    "unknown_bus": "bus:99:p\n1\n",
    "cell_count": "bus:4:p,bus:5:p\n1\n",
    "no_rows": "bus:4:p\n",
    "empty": "",
    "bad_number": "bus:4:p\n1e\n",
    "plus_id": "bus:+4:p\n1\n",
    "short_header": "bus:4p\n1\n",
}
OUTAGE_TEXTS = {
    "valid_comments": "0 3 # comment\n5\n\n19\n",
    "valid_float_int": "2.0 7\n",
    "only_comment": "# nothing\n",
    "out_of_range": "20\n",
    "fractional": "1.5\n",
    "negative": "-1\n",
    "bad_token": "3 x\n",
}


def io_kats(ref: po.Reference) -> dict:
    """parse_scenario_csv / parse_outage_list (case_io.hpp:368-471) on case14, as the
    reference returns them (values, or the error category code)."""
    with open(util.case_path("case14")) as fh:
        rc = ref.parse(fh.read())
    out = {"case": "case14", "scenario": {}, "outages": {}}
    for k, text in SCENARIO_TEXTS.items():
        try:
            p, q = rc.scenario(text)
            out["scenario"][k] = {"text": text, "p_mw": p.tolist(), "q_mvar": q.tolist()}
        except po.OracleError as e:
            out["scenario"][k] = {"text": text, "error": e.code}
    for k, text in OUTAGE_TEXTS.items():
        try:
            out["outages"][k] = {"text": text, "branches": rc.outages(text).tolist()}
        except po.OracleError as e:
            out["outages"][k] = {"text": text, "error": e.code}
    return out


def main():
    po.build(ref=True)
    ref = po.Reference()
    os.makedirs(OUT, exist_ok=True)
    manifest = {"generator": "tools/make_golden.py",
                "source": "reference headers /root/reference/proj/include/gridbatch compiled "
                          "in place via oracle/ref_shim.cpp (oracle/_ref/libgbref.so)",
                "cases": {}}
    for name in CASES:
        g = case_golden(ref, name)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **g)
        manifest["cases"][name] = {k: int(g[k]) for k in ("n_bus", "n_branch", "slack", "nJ")}
        manifest["cases"][name].update(n_pv=len(g["pv"]), n_pq=len(g["pq"]),
                                       nnzY=int(g["indptr"][-1]))
        print(name, manifest["cases"][name], flush=True)
    np.savez_compressed(os.path.join(OUT, "sparse_kats.npz"), **sparse_kats(ref))
    with open(os.path.join(OUT, "io_kats.json"), "w") as fh:
        json.dump(io_kats(ref), fh, indent=1)
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)


if __name__ == "__main__":
    main()
