"""Pinning the oracle's Newton-Raphson / LU restatement (CPU only).

The reference has no NR or LU code, so the oracle's numeric
half is pinned against
  * the published IEEE case14 solution (MATPOWER case14.m),
  * an independent MATPOWER ``newtonpf`` in scipy/SuperLU (tools/newtonpf_scipy.py,
    the pandapower baseline of PAPER.md:504),
  * the SPEC's invariants: dense(L)·dense(U) = P·J·Q, solo == batch
    (SPEC.md:244, :409), worker-count invariance, a diverging
    task never affects its peers, F = S_calc - S_spec.
"""
import numpy as np
import pytest

import pyoracle as po
import util
from newtonpf_scipy import dsbus_dv, newtonpf, ybus_matrix
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo

VM_PUB = [1.06, 1.045, 1.01, 1.018, 1.02, 1.07, 1.062, 1.09, 1.056, 1.051, 1.057, 1.055, 1.05,
          1.036]
VA_PUB = [0, -4.98, -12.73, -10.31, -8.77, -14.22, -13.36, -13.36, -14.94, -15.10, -14.79, -15.08,
          -15.16, -16.03]


def setup(name):
    orc = po.Oracle()
    gc = load_case(util.case_path(name))
    ip, ix, _, yr, yi = orc.build_ybus(gc)
    vm0, va0 = gc.v_start()
    plan = orc.plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    Y = ybus_matrix(ip, ix, yr, yi, gc.n_bus)
    return gc, plan, Y, vm0, va0


def test_case14_published_solution():
    gc, plan, Y, vm0, va0 = setup("case14")
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    assert r["status"][0] == 0 and r["iterations"][0] == 2  # reference V0 rule: warm start
    np.testing.assert_allclose(r["vm"][:, 0], VM_PUB, atol=1.5e-3)
    np.testing.assert_allclose(np.degrees(r["va"][:, 0]), VA_PUB, atol=2e-2)
    vflat = np.where(np.isin(np.arange(14), gc.pq), 1.0, vm0)
    flat = plan.solve(p0, q0, vflat[:, None], np.zeros((14, 1)))
    _, ok, it = newtonpf(Y, p0[:, 0] + 1j * q0[:, 0], vflat.astype(complex), gc.slack, gc.pv, gc.pq)
    assert ok and it == 4  # 4 iterations from flat start
    assert flat["status"][0] == 0 and flat["iterations"][0] == it
    np.testing.assert_allclose(flat["vm"], r["vm"], atol=1e-8)


@pytest.mark.parametrize("name,T", [("case14", 40), ("synth118", 12), ("synth300", 8),
                                    ("synth2383", 6), ("synth9241", 4)])
def test_matches_scipy_newtonpf(name, T):
    gc, plan, Y, vm0, va0 = setup(name)
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    for t in range(T):
        V, ok, it = newtonpf(Y, p0[:, t] + 1j * q0[:, t], vm0 * np.exp(1j * va0), gc.slack,
                             gc.pv, gc.pq)
        assert ok == bool(r["converged"][t])
        assert it == r["iterations"][t]
        assert np.abs(np.abs(V) - r["vm"][:, t]).max() < 1e-8
        assert np.abs(np.angle(V) - r["va"][:, t]).max() < 1e-8


def test_iteration_convention_zero_and_max():
    """MATPOWER convention: 0 iterations if V0 already converged;
    max_iter and converged=0 when the budget runs out."""
    gc, plan, Y, vm0, va0 = setup("case14")
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    again = plan.solve(p0, q0, r["vm"], r["va"])
    assert again["iterations"][0] == 0 and again["status"][0] == 0
    short = plan.solve(p0, q0, vm0[:, None], va0[:, None], max_iter=1)
    assert short["iterations"][0] == 1 and short["converged"][0] == 0 and short["status"][0] == 1


def test_mismatch_is_s_calc_minus_spec():
    gc, plan, Y, vm0, va0 = setup("synth118")
    T = 5
    p0, q0 = montecarlo(gc, T)
    rng = np.random.default_rng(3)
    vm = vm0[:, None] * (1 + 0.01 * rng.standard_normal((gc.n_bus, T)))
    va = va0[:, None] + 0.02 * rng.standard_normal((gc.n_bus, T))
    f = plan.mismatch(p0, q0, vm, va)
    pvpq = np.r_[gc.pv, gc.pq]
    for t in range(T):
        V = vm[:, t] * np.exp(1j * va[:, t])
        mis = V * np.conj(Y @ V) - (p0[:, t] + 1j * q0[:, t])
        F = np.r_[mis[pvpq].real, mis[gc.pq].imag]
        np.testing.assert_allclose(f[:, t], F, rtol=0, atol=1e-11)


@pytest.mark.parametrize("name", ["synth30", "synth300"])
def test_refactor_dense_lu_equals_permuted_jacobian(name):
    gc, plan, Y, vm0, va0 = setup(name)
    T = 3
    rng = np.random.default_rng(5)
    vm = vm0[:, None] * (1 + 0.02 * rng.standard_normal((gc.n_bus, T)))
    va = va0[:, None] + 0.05 * rng.standard_normal((gc.n_bus, T))
    lu, flags = plan.refactor(vm, va)
    assert not flags.any()
    ex = plan.export()
    nJ = len(ex["row_fwd"])
    cp, ri = ex["col_ptr"], ex["row_ix"]
    pvpq = np.r_[gc.pv, gc.pq]
    for t in range(T):
        V = vm[:, t] * np.exp(1j * va[:, t])
        dVm, dVa = dsbus_dv(Y, V)
        J = np.block([[dVa[np.ix_(pvpq, pvpq)].real.toarray(), dVm[np.ix_(pvpq, gc.pq)].real.toarray()],
                      [dVa[np.ix_(gc.pq, pvpq)].imag.toarray(), dVm[np.ix_(gc.pq, gc.pq)].imag.toarray()]])
        A = np.zeros((nJ, nJ))
        A[np.ix_(ex["row_fwd"], ex["col_fwd"])] = J
        L = np.eye(nJ)
        U = np.zeros((nJ, nJ))
        for j in range(nJ):
            for s in range(cp[j], cp[j + 1]):
                i = ri[s]
                if i > j:
                    L[i, j] = lu[s, t]
                else:
                    U[i, j] = lu[s, t]
        np.testing.assert_allclose(L @ U, A, rtol=0, atol=1e-10 * np.abs(A).max())


def test_level_schedule_is_topological():
    """level(c) = 1 + max level(U-deps of c), 0 without deps."""
    gc, plan, Y, vm0, va0 = setup("synth300")
    ex = plan.export()
    cp, ri, lev = ex["col_ptr"], ex["row_ix"], ex["level"]
    for j in range(len(lev)):
        deps = [i for i in ri[cp[j]:cp[j + 1]] if i < j]
        assert lev[j] == (1 + max(lev[d] for d in deps) if deps else 0)
    st = plan.stats()
    assert st["levels_lu"] == lev.max() + 1


def test_batch_solo_and_thread_invariance_and_divergence_isolated():
    gc, plan, Y, vm0, va0 = setup("synth118")
    T = 24
    p0, q0 = montecarlo(gc, T)
    p0 = p0.copy(); q0 = q0.copy()
    p0[:, 7] *= 100.0
    q0[:, 7] *= 100.0
    ref = plan.solve(p0, q0, vm0[:, None], va0[:, None], n_threads=1)
    assert ref["status"][7] != 0
    assert (ref["status"][np.arange(T) != 7] == 0).all()
    for nt in (2, 4, 8):
        r = plan.solve(p0, q0, vm0[:, None], va0[:, None], n_threads=nt)
        for k in ("vm", "va", "iterations", "status", "max_mismatch"):
            np.testing.assert_array_equal(r[k], ref[k])
    for t in (0, 7, 13, 23):
        s = plan.solve(p0[:, t:t + 1], q0[:, t:t + 1], vm0[:, None], va0[:, None])
        np.testing.assert_array_equal(s["vm"][:, 0], ref["vm"][:, t])
        np.testing.assert_array_equal(s["va"][:, 0], ref["va"][:, t])
        assert s["iterations"][0] == ref["iterations"][t]


def test_case14_montecarlo_iteration_split():
    """BASELINE configs[0]: case14, 1000 U(0.8,1.2) scenarios; all converge in 2-3
    iterations from the reference's warm start (SURVEY.md §8a probe)."""
    gc, plan, Y, vm0, va0 = setup("case14")
    p0, q0 = montecarlo(gc, 1000)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    assert (r["status"] == 0).all()
    assert set(np.unique(r["iterations"])) <= {2, 3}
    assert (r["max_mismatch"] < 1e-8).all()


def test_branch_flows_oracle_kats():
    """calc_branch_flows in the oracle: dense restatement, lossless
    lines conserve real power, the whole grid balances, an outaged branch carries 0."""
    from paper_2101_02270_b200 import solver as S
    gc, plan, Y, vm0, va0 = setup("case14")
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    adm = S.branch_admittances(gc)
    sf, st = po.Oracle().branch_flows(gc, adm, r["vm"], r["va"])
    V = r["vm"][:, 0] * np.exp(1j * r["va"][:, 0])
    a = adm[:, 0::2] + 1j * adm[:, 1::2]  # ff, ft, tf, tt
    Vf, Vt = V[gc.br_f], V[gc.br_t]
    np.testing.assert_allclose(sf[:, 0], Vf * np.conj(a[:, 0] * Vf + a[:, 1] * Vt), rtol=0, atol=1e-12)
    np.testing.assert_allclose(st[:, 0], Vt * np.conj(a[:, 2] * Vf + a[:, 3] * Vt), rtol=0, atol=1e-12)
    lossless = (gc.br_r == 0) & (gc.br_b == 0)
    assert lossless.any()
    np.testing.assert_allclose(sf[lossless, 0].real, -st[lossless, 0].real, atol=1e-12)
    Sbus = V * np.conj(Y @ V)  # injections = branch flows + shunts
    shunt = np.conj((gc.gs + 1j * gc.bs) / gc.base_mva) * np.abs(V) ** 2
    total = np.zeros(gc.n_bus, complex)
    np.add.at(total, gc.br_f, sf[:, 0])
    np.add.at(total, gc.br_t, st[:, 0])
    np.testing.assert_allclose(total + shunt, Sbus, atol=1e-10)
    sf2, st2 = po.Oracle().branch_flows(gc, adm, r["vm"], r["va"], outage=np.array([3], np.int32))
    assert sf2[3, 0] == 0 and st2[3, 0] == 0 and sf2[2, 0] == sf[2, 0]


def _two_bus_instability(T=8, special=3, angle=np.pi / 2):
    """SPEC.md:342 example: a task whose frozen pivot collapses but is well
    conditioned under fresh pivoting.  Slack + one PQ bus on a lossless line
    (x = 0.1): dP1/dtheta1 = V1 V0 B10 cos(theta1), so a task starting at
    theta1 = 90 degrees has a zero frozen (diagonal) pivot while J stays
    nonsingular ([[0, a], [b, c]])."""
    ip = np.array([0, 2, 4], np.int32)
    ix = np.array([0, 1, 0, 1], np.int32)
    yr, yi = np.zeros(4), np.array([-10.0, 10.0, 10.0, -10.0])
    vm0, va0 = np.ones(2), np.zeros(2)
    p0 = np.tile(np.array([0.0, -0.5])[:, None], (1, T))
    q0 = np.tile(np.array([0.0, -0.2])[:, None], (1, T))
    vm, va = np.ones((2, T)), np.zeros((2, T))
    va[1, special] = angle
    pq = np.array([1], np.int32)
    return (ip, ix, yr, yi, 0, np.array([], np.int32), pq, vm0, va0), p0, q0, vm, va


def test_second_chance_fallback_oracle():
    """second_chance_refactorize: the flagged task is re-planned
    with fresh pivoting and converges as fallback_converged (status 3); batch peers
    are unaffected (solo-run comparison, SPEC.md:502 criterion 7); without the
    second chance it stays singular."""
    T = 40  # one flagged task in 40: below the 5% re-derivation threshold
    args, p0, q0, vm, va = _two_bus_instability(T)
    op = po.Oracle().plan(2, *args)
    off = op.solve(p0, q0, vm, va, n_tasks=T, second_chance=False)
    assert off["status"][3] == 2 and off["iterations"][3] == 1
    r = op.solve(p0, q0, vm, va, n_tasks=T)
    assert r["status"][3] == 3 and r["converged"][3] == 1 and r["max_mismatch"][3] < 1e-8
    assert r["iterations"][3] > 1
    peers = [t for t in range(T) if t != 3]
    assert (r["status"][peers] == 0).all()
    solo = op.solve(p0[:, :1], q0[:, :1], vm[:, :1], va[:, :1], n_tasks=1)
    np.testing.assert_array_equal(r["vm"][:, peers], np.repeat(solo["vm"], T - 1, axis=1))
    np.testing.assert_array_equal(r["iterations"][peers], solo["iterations"][0])


def test_representative_rederivation_oracle():
    """SPEC.md DESIGN DECISIONS: when the frozen pivots fail for more than 5% of the
    tasks at their first solve (here 1 of 8), the batch restarts once from a plan
    whose pivots come from the task with the worst mismatch at V0 -- the 90-degree
    task itself, which then converges normally while the flat-start tasks now hit
    a zero frozen pivot and take the second chance."""
    args, p0, q0, vm, va = _two_bus_instability(8)
    r = po.Oracle().plan(2, *args).solve(p0, q0, vm, va, n_tasks=8)
    assert r["status"][3] == 0
    assert (np.delete(r["status"], 3) == 3).all() and r["converged"].all()
