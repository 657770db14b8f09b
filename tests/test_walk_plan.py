"""Host replay of the tile-walk copy programs (walk.hpp) -- CPU only.

The LU+FS and BS walks are driven by a static program of TMA copies planned on
the host (which step's block lives where in shared memory, which dependency is
still resident, which must be re-fetched, and after which consumer event each
copy may be issued).  This test replays that program exactly as the kernels do
-- copies take effect when issued, the warp consumes in order -- on a 32-lane
tile, with numpy standing in for shared memory and the tapes.  A copy issued
too early (before its producer wrote the data) or a ring row overwritten while
still needed shows up as a wrong factor, so the result is compared BITWISE with
a plain sequential Alg. 2 / FS / BS over the same numbers (both sides use the
same unfused arithmetic here; the GPU's fused arithmetic is checked against the
oracle by the -m gpu parity tests).
"""
import numpy as np
import pytest

import util
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from newtonpf_scipy import dsbus_dv, ybus_matrix

TAPE_A, TAPE_LU, TAPE_B = 0, 1, 2


def jacobian_tape(gc, plan, lanes=32, seed=0):
    """A values (LU CCS slot order) of `lanes` tasks at perturbed voltages."""
    ip, ix, _, yr, yi = S.build_ybus(gc)
    Y = ybus_matrix(ip, ix, yr, yi, gc.n_bus)
    ex = plan.export()
    cp, ri = ex["col_ptr"], ex["row_ix"]
    nJ = len(ex["row_fwd"])
    pos = {}
    for j in range(nJ):
        for s in range(cp[j], cp[j + 1]):
            pos[(ri[s], j)] = s
    vm0, va0 = gc.v_start()
    rng = np.random.default_rng(seed)
    pvpq = np.r_[gc.pv, gc.pq]
    A = np.zeros((cp[-1], lanes))
    for t in range(lanes):
        V = vm0 * (1 + 0.01 * rng.standard_normal(gc.n_bus)) * np.exp(1j * (va0 + 0.02 * rng.standard_normal(gc.n_bus)))
        dVm, dVa = dsbus_dv(Y, V)
        J = np.block([[dVa[np.ix_(pvpq, pvpq)].real.toarray(), dVm[np.ix_(pvpq, gc.pq)].real.toarray()],
                      [dVa[np.ix_(gc.pq, pvpq)].imag.toarray(), dVm[np.ix_(gc.pq, gc.pq)].imag.toarray()]])
        rr, cc = np.nonzero(J)
        for a, b in zip(rr, cc):
            A[pos[(ex["row_fwd"][a], ex["col_fwd"][b])], t] = J[a, b]
    b = rng.standard_normal((nJ, lanes))
    return ex, A, b


def sequential(ex, A, b):
    """Alg. 2 + push FS + push BS, CCS storage (the oracle's operation order)."""
    cp, ri = ex["col_ptr"], ex["row_ix"]
    nJ = len(cp) - 1
    lu = A.copy()
    dpos = np.zeros(nJ, np.int64)
    for k in range(nJ):
        rows = ri[cp[k]:cp[k + 1]]
        dpos[k] = cp[k] + int(np.searchsorted(rows, k))
        posm = {r: z for z, r in enumerate(rows)}
        x = lu[cp[k]:cp[k + 1]]
        for z in range(dpos[k] - cp[k]):
            j = rows[z]
            xj = x[z].copy()
            for zz in range(dpos[j] + 1, cp[j + 1]):
                d = posm[ri[zz]]
                x[d] = x[d] - xj * lu[zz]
        dp = dpos[k] - cp[k]
        inv = 1.0 / x[dp]
        x[dp + 1:] = x[dp + 1:] * inv
    y = b.copy()
    for k in range(nJ):
        for z in range(dpos[k] + 1, cp[k + 1]):
            y[ri[z]] = y[ri[z]] - lu[z] * y[k]
    x = y.copy()
    for k in range(nJ - 1, -1, -1):
        x[k] = x[k] / lu[dpos[k]]
        for z in range(cp[k], dpos[k]):
            x[ri[z]] = x[ri[z]] - lu[z] * x[k]
    return lu, y, x


REC_ISSUE, REC_STEP, REC_DEP, REC_END, REC_PAGE, REC_DONE, REC_SYNC, REC_DEP2, REC_DEPN = 1, 2, 3, 4, 5, 6, 7, 8, 9
REC_STEPG, REC_DEPG, REC_ENDG, REC_ENDU, REC_DEPNG, REC_PAIR = 10, 11, 12, 13, 14, 15


class Machine:
    """One walker as the kernels see it: its paged program words, its op barriers,
    and the CTA's shared rows R (shared with the other walkers of the tile)."""

    def __init__(self, w, walker, R, tapes):
        info = w["info"]
        self.tapes, self.R = tapes, R
        self.W, self.NP, self.NB = info["page_words"], info["pages"], info["barriers"]
        p0, p1 = w["wpage0"][walker], w["wpage0"][walker + 1]
        self.gs = w["stream"][p0 * self.W:p1 * self.W].astype(np.int64)
        self.n_pages = p1 - p0
        self.pages = np.zeros((self.NP, self.W), np.int64)
        for p in range(min(self.NP, self.n_pages)):
            self.pages[p] = self.gs[p * self.W:(p + 1) * self.W]
        self.page, self.off = 0, 0
        self.issued = set()
        self.n_issued = 0
        self.done = False

    def rec(self):
        return self.pages[self.page % self.NP, self.off:]

    def next_page(self):
        if self.page + self.NP < self.n_pages:
            q = self.page + self.NP
            self.pages[self.page % self.NP] = self.gs[q * self.W:(q + 1) * self.W]
        self.page += 1
        self.off = 0

    def issue(self, r):
        ncopy = (int(r[0]) >> 4) & 0xFFF
        op = int(r[1])
        assert op == self.n_issued, "ops must be issued in order"
        nbytes = 0
        for i in range(ncopy):
            c, slot = int(r[3 + 2 * i]), int(r[4 + 2 * i])
            tape, rows, smem = c & 3, (c >> 2) & 1023, c >> 12
            self.R[smem:smem + rows] = self.tapes[tape][slot:slot + rows]
            nbytes += rows
        assert nbytes == r[2]  # expect_tx in rows (the kernel scales by its row bytes)
        self.issued.add(op)
        self.n_issued += 1
        return 3 + 2 * ncopy

    def wait(self, op):
        assert op in self.issued, f"waits on unissued op {op}"
        assert self.n_issued <= op + self.NB, "barrier re-armed before its wait"


def run_phases(w, tapes, step_fn):
    """Run every walker's program phase by phase (walkers of a phase are
    independent, so running them one after another is a valid interleaving)."""
    info = w["info"]
    R = np.full((info["rows"], 32), np.nan)
    ms = [Machine(w, k, R, tapes) for k in range(info["walkers"])]
    while not all(m.done for m in ms):
        for m in ms:
            state = {}
            while True:
                r = m.rec()
                t = int(r[0]) & 15
                if t == REC_ISSUE:
                    m.off += m.issue(r)
                elif t == REC_PAGE:
                    m.next_page()
                elif t == REC_SYNC:
                    m.off += 1
                    break
                elif t == REC_DONE:
                    m.done = True
                    break
                else:
                    m.off += step_fn(m, r, t, state)
    return R


def replay_forward(w, A_tape, nrows, fs=True):
    LU = np.full((nrows, 32), np.nan)
    tapes = {TAPE_A: A_tape, TAPE_LU: LU, TAPE_B: None}

    def step(M, r, t, S):
        R = M.R
        h = int(r[0])
        if t == REC_STEPG:  # column too large for the pool: its A rows + F in a global scratch
            ln, dp = int(r[1]) & 0xFFFF, int(r[1]) >> 16
            a0 = int(r[2])
            S.update(ring=None, ln=ln, dp=dp, lslot=int(r[3]), uy=int(r[4]), gmax=0.0)
            S["x"] = A_tape[a0:a0 + ln + 1].copy()  # the scratch (the A tape stays intact)
            S["acc"] = S["x"][ln].copy() if fs else None
            return 5
        if t == REC_DEPG:  # dependency read from the LU tape
            op = (h >> 4) - 1
            if op >= 0:
                M.wait(op)
            kpos_fs, n, slot, nl = int(r[1]), int(r[2]), int(r[3]), int(r[4])
            x = S["x"]
            if n > 0:
                mult = x[kpos_fs & 0xFFFF].copy()
                for q in range(n):
                    wq = int(r[5 + q // 2])
                    d = (wq >> 16) & 0xFFFF if q & 1 else wq & 0xFFFF
                    x[d] = x[d] - mult * LU[slot + q]
            fsp = (kpos_fs >> 16) & 0xFFFF
            if fs and fsp != 0xFFFF:
                S["acc"] = S["acc"] - LU[slot + fsp] * LU[slot + nl]
            return 5 + (n + 1) // 2
        if t == REC_ENDU:
            cnt, z0 = (h >> 4) & 0xFFFFF, int(r[1])
            for i in range(cnt):
                LU[int(r[2 + i])] = S["x"][z0 + i]
            return 2 + cnt
        if t == REC_ENDG:
            x, dp, ln, lslot = S["x"], S["dp"], S["ln"], S["lslot"]
            piv = x[dp].copy()
            inv = 1.0 / piv
            for z in range(dp + 1, ln):
                LU[lslot + z - dp - 1] = x[z] * inv
            LU[S["uy"] + 1] = piv
            if fs:
                LU[lslot + ln - dp - 1] = S["acc"]
                LU[S["uy"]] = S["acc"]
            return 1
        if t == REC_DEP:
            op = (h >> 4) - 1
            kpos_fs, nrows, src, ysrc = int(r[1]), int(r[2]) & 0xFFFF, (int(r[2]) >> 16) & 0xFFFF, int(r[3])
            if op >= 0:
                M.wait(op)
            x = S["x"]
            if nrows > 0:
                mult = x[kpos_fs & 0xFFFF].copy()
                for q in range(nrows):
                    wq = int(r[4 + q // 2])
                    d = (wq >> 16) & 0xFFFF if q & 1 else wq & 0xFFFF
                    x[d] = x[d] - mult * R[src + q]
            fsp = (kpos_fs >> 16) & 0xFFFF
            if fs and fsp != 0xFFFF:
                S["acc"] = S["acc"] - R[src + fsp] * R[ysrc]
            return 4 + ((nrows + 3) & ~3) // 2
        if t == REC_DEP2:  # supernode pair k, k+1 in one pass, k's update first per element
            op = (h >> 4) - 1
            w1, w2, w3, w4, w5 = (int(v) for v in r[1:6])
            fs2, op2 = w5 & 0xFFFF, (w5 >> 16) - 1
            if op >= 0:
                M.wait(op)
            if op2 >= 0:
                M.wait(op2)
            x = S["x"]
            kpos1, kpos2, nrows, s1 = w1 & 0xFFFF, w1 >> 16, w2 & 0xFFFF, w2 >> 16
            s2, fs1, y1, y2 = w3 & 0xFFFF, w3 >> 16, w4 & 0xFFFF, w4 >> 16
            m1 = x[kpos1].copy()
            x[kpos2] = x[kpos2] - m1 * R[s1]
            m2 = x[kpos2].copy()
            for q in range(nrows):
                wq = int(r[6 + q // 2])
                d = (wq >> 16) & 0xFFFF if q & 1 else wq & 0xFFFF
                x[d] = (x[d] - m1 * R[s1 + 1 + q]) - m2 * R[s2 + q]
            if fs and fs1 != 0xFFFF:
                S["acc"] = S["acc"] - R[s1 + fs1] * R[y1]
            if fs and fs2 != 0xFFFF:
                S["acc"] = S["acc"] - R[s2 + fs2] * R[y2]
            return 6 + ((nrows + 3) & ~3) // 2
        if t == REC_STEP:
            ring, ln = int(r[1]) & 0xFFFF, int(r[1]) >> 16
            S.update(ring=ring, ln=ln, dp=int(r[2]), lslot=int(r[3]), uy=int(r[4]))
            M.wait(int(r[5]))
            S["x"] = R[ring:ring + ln]
            S["acc"] = R[ring + ln].copy() if fs else None
            return 6
        assert t == REC_END
        x, dp, ln, lslot = S["x"], S["dp"], S["ln"], S["lslot"]
        piv = x[dp].copy()
        inv = 1.0 / piv
        for z in range(dp + 1, ln):
            x[z] = x[z] * inv
            LU[lslot + z - dp - 1] = x[z]
        for z in range(dp):
            LU[int(r[1 + z])] = x[z]
        LU[S["uy"] + 1] = piv  # U(m,m) closing the backward block
        if fs:  # y_m after the L rows and in the backward block
            R[S["ring"] + ln] = S["acc"]
            LU[lslot + ln - dp - 1] = S["acc"]
            LU[S["uy"]] = S["acc"]
        return 1 + dp

    run_phases(w, tapes, step)
    return LU


def replay_backward(w, LU, b_tape):
    tapes = {TAPE_A: None, TAPE_LU: LU, TAPE_B: b_tape}

    def step(M, r, t, S):
        R = M.R
        h = int(r[0])
        if t == REC_STEPG:  # row block read in place from the LU tape
            ne, slot = int(r[1]), int(r[2])
            S.update(ring=None, ne=ne, brow=int(r[3]), gslot=slot, e=0)
            S["acc"] = LU[slot + ne].copy()
            return 4
        if t == REC_PAIR:  # two independent rows in one record (their order is free)
            nA, nw = (h >> 4) & 0xFFF, (h >> 16) & 0xFF
            wa, wb, bra, brb, ops, nB = (int(x) for x in r[1:7])
            for op in ((ops & 0xFFFF) - 1, (ops >> 16) - 1, *[int(x) - 1 for x in r[7:7 + nw]]):
                if op >= 0:
                    M.wait(op)
            ya = 7 + nw
            yb = ya + (nA + 1) // 2
            xs = []
            for (w_, n_, y0) in ((wa, nA, ya), (wb, nB, yb)):
                ring, ne = w_ & 0xFFFF, w_ >> 16
                acc = R[ring + ne].copy()
                for i in range(n_):
                    wq = int(r[y0 + i // 2])
                    ysrc = (wq >> 16) & 0xFFFF if i & 1 else wq & 0xFFFF
                    acc = acc - R[ring + i] * R[ysrc]
                xs.append((ring, ne, acc / R[ring + ne + 1]))
            for (ring, ne, x), br in zip(xs, (bra, brb)):
                R[ring + ne] = x
                b_tape[br] = x
            return yb + (nB + 1) // 2
        if t == REC_DEPNG:
            n = (h >> 4) & 0xFFFFF
            for i in range(n):
                S["acc"] = S["acc"] - LU[S["gslot"] + S["e"]] * b_tape[int(r[1 + i])]
                S["e"] += 1
            return 1 + n
        if t == REC_ENDG:
            b_tape[S["brow"]] = S["acc"] / LU[S["gslot"] + S["ne"] + 1]
            return 1
        if t == REC_DEPN:
            op = (h >> 4) - 1
            if op >= 0:
                M.wait(op)
            n = int(r[1])
            for i in range(n):
                wq = int(r[2 + i // 2])
                ysrc = (wq >> 16) & 0xFFFF if i & 1 else wq & 0xFFFF
                S["acc"] = S["acc"] - R[S["ring"] + S["e"]] * R[ysrc]
                S["e"] += 1
            return 2 + (n + 1) // 2
        if t == REC_STEP:
            ring, ne = int(r[1]) & 0xFFFF, int(r[1]) >> 16
            S.update(ring=ring, ne=ne, brow=int(r[4]), e=0)
            M.wait(int(r[5]))
            S["acc"] = R[ring + ne].copy()
            return 6
        assert t == REC_END
        ring, ne = S["ring"], S["ne"]
        xi = S["acc"] / R[ring + ne + 1]
        R[ring + ne] = xi
        b_tape[S["brow"]] = xi
        return 1

    run_phases(w, tapes, step)


@pytest.mark.parametrize("name,opts", [("case14", {}), ("synth118", {}), ("synth300", {}),
                                       ("synth300", dict(walkers=1)),
                                       ("synth300", dict(walkers=8)),
                                       ("synth300", dict(walkers=2, ring_rows=40, stage_rows=24, prefetch=3)),
                                       ("synth300", dict(walkers=1, ring_rows=200, stage_rows=80, prefetch=20)),
                                       ("synth2383", dict(walkers=3, prefetch=5, headroom=1))])
@pytest.mark.parametrize("unified", ["1", "0"])
def test_walk_replay_bitwise(name, opts, unified, monkeypatch):
    """Both planners: the unified block/staging pool (default) and the split
    ring + staging plan it falls back to (GBNR_UNIFIED=0)."""
    monkeypatch.setenv("GBNR_UNIFIED", unified)
    gc = load_case(util.case_path(name))
    plan = S.NrPlan.from_case(gc, device=-1, **opts)
    check_replay(gc, plan)


@pytest.mark.parametrize("name,frac,opts", [("synth118", "0.1", {}), ("synth300", "0.05", {}),
                                            ("synth300", "0.2", dict(walkers=2)),
                                            ("synth300", "0.001", dict(walkers=1)),
                                            ("synth2383", "0.08", {})])
@pytest.mark.parametrize("unified", ["1", "0"])
def test_walk_replay_global_forms(name, frac, opts, unified, monkeypatch):
    """Blocks / fetches moved to global memory (the fallback for columns too large
    for a walker's shared-memory pool, forced here on small grids by
    GBNR_GLOBAL_FRAC) keep every element's operation order: bitwise equal."""
    monkeypatch.setenv("GBNR_UNIFIED", unified)
    monkeypatch.setenv("GBNR_GLOBAL_FRAC", frac)
    gc = load_case(util.case_path(name))
    plan = S.NrPlan.from_case(gc, device=-1, **opts)
    infos = [plan.walk_info(w) for w in (0, 1, 2)]
    assert infos[0]["global_steps"] > 0 and infos[0]["scratch_rows"] > 0
    if frac == "0.001":  # everything global: no copies at all
        assert all(i["global_steps"] == i["steps"] and i["n_copies"] == 0 for i in infos)
    check_replay(gc, plan)


def check_replay(gc, plan):
    ex, A, b = jacobian_tape(gc, plan)
    lu_ref, y_ref, x_ref = sequential(ex, A, b)
    wf, wl, wb = plan.walk_export(0), plan.walk_export(1), plan.walk_export(2)
    toc, lslot, ucrs0 = wf["tape_of_ccs"], wf["lslot"], wf["ucrs0"]
    cp, ri = ex["col_ptr"], ex["row_ix"]
    nJ = len(cp) - 1
    nrows = len(toc) + 2 * nJ
    assert ucrs0[-1] == nrows
    # A tape: every column's CCS entries followed by its F row (walk.hpp LuLayout)
    A_tape = np.full((len(toc) + nJ, 32), np.nan)
    for m in range(nJ):
        A_tape[cp[m] + m:cp[m + 1] + m] = A[cp[m]:cp[m + 1]]
        A_tape[cp[m + 1] + m] = b[m]
    LU = replay_forward(wf, A_tape, nrows, fs=True)
    np.testing.assert_array_equal(LU[toc], lu_ref)
    dpos = np.array([cp[k] + np.searchsorted(ri[cp[k]:cp[k + 1]], k) for k in range(nJ)])
    np.testing.assert_array_equal(LU[lslot + cp[1:] - dpos - 1], y_ref)  # y_k after L(:,k)
    np.testing.assert_array_equal(LU[ucrs0[1:] - 2], y_ref)  # and in row k's backward block
    np.testing.assert_array_equal(toc[dpos], ucrs0[1:] - 1)  # U(k,k) closing it
    b_tape = np.full((nJ, 32), np.nan)
    replay_backward(wb, LU, b_tape)
    np.testing.assert_array_equal(b_tape[::-1], x_ref)  # x_k at b-tape row nJ-1-k
    LU2 = replay_forward(wl, A_tape, nrows, fs=False)
    np.testing.assert_array_equal(LU2[toc], lu_ref)
    plan.close()


def test_walk_stats_and_layout():
    gc = load_case(util.case_path("synth2383"))
    plan = S.NrPlan.from_case(gc, device=-1)
    st = plan.stats()
    for which in (0, 1, 2):
        info = plan.walk_info(which)
        assert info["steps"] == st["nJ"]
        assert info["walkers"] == 8 and info["phases"] >= 3  # 8, 4, 2, then 1 walker
        assert info["smem_bytes"] + 1024 <= 228 * 1024 // 3  # three tiles per SM
    w = plan.walk_export(0)
    toc = w["tape_of_ccs"]
    # the pattern's slots plus, per column, y after L(:,k) and y before U(k,k) closing row k
    extra = np.r_[w["lslot"] + np.diff(w["lslot"], append=w["ucrs0"][0]) - 1, w["ucrs0"][1:] - 2]
    assert sorted(np.r_[toc, extra].tolist()) == list(range(st["nnzLU"] + 2 * st["nJ"]))
    own = w["owner"]
    level, walker = own >> 4, own & 15
    assert set(np.unique(level)) <= {0, 1, 2, 3}
    assert (walker < np.array([8, 4, 2, 1])[level]).all()
    # most columns are walked by eight concurrent walkers; the serial top is small
    assert (level == 0).mean() > 0.7 and (level == level.max()).sum() < 0.02 * len(own)
    # the backward walk has its own (lighter) blocks, so more of it runs at level 0
    bl = plan.walk_export(2)["owner"] >> 4
    assert (bl == 0).mean() >= (level == 0).mean()
    plan.close()


def test_sequential_reference_kat():
    """SPEC.md:335 known answer for the sequential Alg. 2 + FS/BS the replays are
    compared with: L = [[1], [2, 1], [0, 3, 1]] (unit lower triangular, so U = I),
    b = [1, 4, 11] -> y = x = [1, 2, 5]."""
    ex = {"col_ptr": np.array([0, 2, 4, 5]), "row_ix": np.array([0, 1, 1, 2, 2])}
    A = np.array([[1.0], [2.0], [1.0], [3.0], [1.0]])
    b = np.array([[1.0], [4.0], [11.0]])
    lu, y, x = sequential(ex, A, b)
    np.testing.assert_array_equal(y[:, 0], [1.0, 2.0, 5.0])
    np.testing.assert_array_equal(x[:, 0], [1.0, 2.0, 5.0])
    np.testing.assert_array_equal(lu, A)  # already factored: L unchanged, U = I


def test_unified_pool_planner_is_used(monkeypatch):
    """The default plans come from the unified pool planner (its placements differ
    from the split ring + staging plans), not from its silent fallback."""
    gc = load_case(util.case_path("synth2383"))
    infos = {}
    for u in ("1", "0"):
        monkeypatch.setenv("GBNR_UNIFIED", u)
        plan = S.NrPlan.from_case(gc, device=-1)
        infos[u] = [plan.walk_info(w) for w in (0, 1, 2)]
        plan.close()
    for a, b in zip(infos["1"], infos["0"]):
        assert a["steps"] == b["steps"]
        assert (a["n_ops"], a["ring_dep_rows"], a["stream_words"]) != (b["n_ops"], b["ring_dep_rows"], b["stream_words"])
