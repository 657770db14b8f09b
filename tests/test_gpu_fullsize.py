"""GPU parity at the BASELINE configs' full sizes (BASELINE.json configs[1..3]).

Same bar as test_gpu_parity.py -- statuses / iteration counts identical,
voltages and LU factors bit-identical to the oracle -- but on the
whole benchmark batches, not samples: the oracle runs on every host thread
(about 6 s for synth9241 x 10k on the GPU box's 16 cores).  The MATPOWER-signature
entry point is checked against an independent scipy newtonpf (tools/newtonpf_scipy.py).
"""
import numpy as np
import pytest

import pyoracle as po
import util
from newtonpf_scipy import newtonpf, ybus_matrix
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from test_gpu_parity import _compare, _setup

pytestmark = pytest.mark.gpu


def test_headline_batch_synth9241_10k_bitwise():
    """configs[3] (the headline): every one of the 10k synth9241 Monte-Carlo tasks
    the bench solves equals the oracle bitwise (statuses, iterations, V, mismatch)."""
    gc, plan, oplan, vm0, va0 = _setup("synth9241")
    T = 10000
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    assert (r.status == 0).all()
    _compare(r, o)


def test_loadpv_synth300_10k_bitwise():
    """configs[1]: IEEE-300-sized grid, 10k Monte-Carlo load/PV scenarios (loads and
    PV generator set-points both drawn per task)."""
    gc, plan, oplan, vm0, va0 = _setup("synth300")
    T = 10000
    p0, q0 = montecarlo(gc, T, mode="loadpv")
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    assert (r.status == 0).mean() > 0.99
    _compare(r, o)


def test_refactor_synth2383_10k_bitwise():
    """configs[2]: the batched LU refactorization microbenchmark, synth2383 x 10k,
    each task's Jacobian at its own perturbed voltages: every L/U value and pivot
    flag of every task equals orc_refactor's."""
    gc, plan, oplan, vm0, va0 = _setup("synth2383")
    T = 10000
    rng = np.random.default_rng(23)
    vm = vm0[:, None] * (1 + 0.01 * rng.standard_normal((gc.n_bus, T)))
    va = va0[:, None] + 0.02 * rng.standard_normal((gc.n_bus, T))
    p0, q0 = montecarlo(gc, T)
    plan.stage(p0, q0, vm, va)
    lu, flags, ms = plan.refactor(reps=1)
    olu, oflags = oplan.refactor(vm, va)
    np.testing.assert_array_equal(flags, oflags)
    assert np.array_equal(lu, olu), "LU factors differ from the oracle"
    assert ms > 0.0


@pytest.mark.parametrize("name,T", [("case14", 64), ("synth300", 48), ("synth2383", 12)])
def test_newtonpf_batch_matches_scipy_newtonpf(name, T):
    """PAPER.md:193-195 / :504: the MATPOWER-signature call (Ybus, Sbus, V0, ref, pv,
    pq -> V, success, iterations) against MATPOWER newtonpf in scipy, task by task:
    identical success flags and iteration counts, |dV| <= 1e-8 p.u. (north star);
    and bit-identical to the oracle on the same inputs."""
    gc = load_case(util.case_path(name))
    ip, ix, _, yr, yi = S.build_ybus(gc)
    Y = ybus_matrix(ip, ix, yr, yi, gc.n_bus)
    vm0, va0 = gc.v_start()
    p0, q0 = montecarlo(gc, T)
    Sbus = p0 + 1j * q0
    V0 = vm0 * np.exp(1j * va0)
    V, ok, it = S.newtonpf_batch(Y, Sbus, V0, gc.slack, gc.pv, gc.pq)
    assert V.shape == (gc.n_bus, T) and ok.all()
    for t in range(T):
        Vs, oks, its = newtonpf(Y, Sbus[:, t], V0, gc.slack, gc.pv, gc.pq)
        assert oks == bool(ok[t]) and its == int(it[t])
        assert np.abs(np.abs(Vs) - np.abs(V[:, t])).max() <= 1e-8
        assert np.abs(np.angle(Vs) - np.angle(V[:, t])).max() <= 1e-8
    o = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0).solve(
        p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    np.testing.assert_array_equal(it, o["iterations"])
    np.testing.assert_array_equal(V, o["vm"] * np.exp(1j * o["va"]))
