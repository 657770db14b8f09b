"""GPU parity: the CUDA path (through the C ABI) against the C oracle.

Bar: iteration counts, convergence flags and statuses identical; voltages
bit-identical (the arithmetic contract of DESIGN.md §4 makes the two
implementations perform the same IEEE operations) -- the north star's 1e-8 p.u.
tolerance is asserted as well so a contract break shows up as a bound, not
just an inequality.
"""
import numpy as np
import pytest

import pyoracle as po
import util
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo
from paper_2101_02270_b200 import solver as S

pytestmark = pytest.mark.gpu
TOL_V = 1e-8  # p.u. / rad, BASELINE.json north_star


def _setup(name):
    gc = load_case(util.case_path(name))
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    plan = S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, device=0)
    oplan = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    return gc, plan, oplan, vm0, va0


def _compare(r, o, exact=True):
    np.testing.assert_array_equal(r.status, o["status"])
    np.testing.assert_array_equal(r.iterations, o["iterations"])
    np.testing.assert_array_equal(r.converged, o["converged"])
    ok = (r.status == 0) | (r.status == 3)  # converged, incl. second chance
    assert np.abs(r.vm[:, ok] - o["vm"][:, ok]).max(initial=0) <= TOL_V
    assert np.abs(r.va[:, ok] - o["va"][:, ok]).max(initial=0) <= TOL_V
    if exact:
        np.testing.assert_array_equal(r.vm[:, ok], o["vm"][:, ok])
        np.testing.assert_array_equal(r.va[:, ok], o["va"][:, ok])
        np.testing.assert_array_equal(r.max_mismatch[ok], o["max_mismatch"][ok])


@pytest.mark.parametrize("name,T", [("case14", 1000), ("synth30", 333), ("synth118", 256),
                                    ("synth300", 2000), ("synth2383", 200), ("synth9241", 96)])
def test_montecarlo_matches_oracle(name, T):
    gc, plan, oplan, vm0, va0 = _setup(name)
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    assert (r.status == 0).mean() > 0.99
    _compare(r, o)


@pytest.mark.parametrize("name,T", [("synth300", 130), ("synth2383", 700)])
def test_loadpv_mode_and_per_task_v0(name, T):
    gc, plan, oplan, vm0, va0 = _setup(name)
    p0, q0 = montecarlo(gc, T, mode="loadpv")
    rng = np.random.default_rng(1)
    vmT = vm0[:, None] * (1 + 0.001 * rng.standard_normal((gc.n_bus, T)))
    vaT = va0[:, None] + 0.001 * rng.standard_normal((gc.n_bus, T))
    r = plan.solve(p0, q0, vmT, vaT)
    o = oplan.solve(p0, q0, vmT, vaT)
    _compare(r, o)


def test_shared_injection_set_broadcast():
    gc, plan, oplan, vm0, va0 = _setup("case14")
    p0, q0 = gc.profiles(gc.pd, gc.qd)
    r = plan.solve(p0[:, 0], q0[:, 0], vm0, va0, n_tasks=77)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=77)
    _compare(r, o)
    assert (r.iterations == 2).all()
    assert np.abs(r.vm - r.vm[:, :1]).max() == 0.0  # identical tasks -> identical results


def test_diverging_task_isolated_and_batch_invariance():
    gc, plan, oplan, vm0, va0 = _setup("synth118")
    T = 64
    p0, q0 = montecarlo(gc, T)
    p0 = p0.copy(); q0 = q0.copy()
    p0[:, 5] *= 100.0
    q0[:, 5] *= 100.0
    r = plan.solve(p0, q0, vm0, va0)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None])
    _compare(r, o)
    assert r.status[5] != 0 and not r.converged[5]
    # solo runs of a few tasks are bit-identical to their batch results
    for t in (0, 6, 33, 63):
        rs = plan.solve(p0[:, t:t + 1], q0[:, t:t + 1], vm0, va0, n_tasks=1)
        np.testing.assert_array_equal(rs.vm[:, 0], r.vm[:, t])
        np.testing.assert_array_equal(rs.va[:, 0], r.va[:, t])
        assert rs.iterations[0] == r.iterations[t]


def test_refactor_matches_oracle_bitwise():
    gc, plan, oplan, vm0, va0 = _setup("synth300")
    T = 70
    rng = np.random.default_rng(7)
    vm = vm0[:, None] * (1 + 0.02 * rng.standard_normal((gc.n_bus, T)))
    va = va0[:, None] + 0.05 * rng.standard_normal((gc.n_bus, T))
    p0, q0 = montecarlo(gc, T)
    plan.stage(p0, q0, vm, va)
    lu, flags, ms = plan.refactor(reps=2)
    olu, oflags = oplan.refactor(vm, va)
    np.testing.assert_array_equal(flags, oflags)
    np.testing.assert_array_equal(lu, olu)
    assert ms > 0.0


def test_refactor_flags_singular_task_only():
    """a batch with one task whose frozen pivot is exactly zero (the
    two-bus 90-degree instance) -> that task flagged, every other task's factors
    identical to a solo refactorization and to the oracle."""
    from test_oracle_nr import _two_bus_instability
    args, p0, q0, vm, va = _two_bus_instability(T=40, special=3)
    ip, ix, yr, yi, ref, pv, pq, vm0, va0 = args
    plan = S.NrPlan(2, ip, ix, yr, yi, ref, pv, pq, vm0, va0, device=0)
    plan.stage(p0, q0, vm, va)
    lu, flags, _ = plan.refactor(reps=1)
    olu, oflags = po.Oracle().plan(2, *args).refactor(vm, va)
    np.testing.assert_array_equal(flags, oflags)
    assert flags[3] == 1 and flags.sum() == 1
    np.testing.assert_array_equal(lu, olu)
    plan.stage(p0[:, :1], q0[:, :1], vm[:, :1], va[:, :1])
    solo, _, _ = plan.refactor(reps=1)
    np.testing.assert_array_equal(np.delete(lu, 3, axis=1), np.repeat(solo, 39, axis=1))


def test_repeat_solve_is_deterministic():
    gc, plan, oplan, vm0, va0 = _setup("synth300")
    p0, q0 = montecarlo(gc, 300)
    a = plan.solve(p0, q0, vm0, va0)
    b = plan.solve(p0, q0, vm0, va0)
    np.testing.assert_array_equal(a.vm, b.vm)
    np.testing.assert_array_equal(a.iterations, b.iterations)


@pytest.mark.parametrize("opts", [dict(walkers=4, ring_rows=36, stage_rows=24, prefetch=3),
                                  dict(walkers=1, ring_rows=64, stage_rows=40, prefetch=1, headroom=1),
                                  dict(walkers=1),
                                  dict(walkers=8, prefetch=16, headroom=4),
                                  dict(walkers=8, split=True)])
def test_walk_plan_invariance(opts, monkeypatch):
    """execute_schedule == refactorize_batch bitwise for any execution plan:
    changing the number of walkers per tile (how the elimination tree is split into
    concurrently walked subtrees) or shrinking / growing the shared-memory rings moves
    dependencies between ring residency and TMA re-fetches and changes every copy's
    issue point, never a bit."""
    opts = dict(opts)
    if opts.pop("split", False):  # the split ring + staging planner (GBNR_UNIFIED=0)
        monkeypatch.setenv("GBNR_UNIFIED", "0")
    gc, plan, oplan, vm0, va0 = _setup("synth300")
    ip, ix, _, yr, yi = S.build_ybus(gc)
    plan2 = S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, **opts)
    p0, q0 = montecarlo(gc, 100)
    _compare(plan2.solve(p0, q0, vm0, va0), oplan.solve(p0, q0, vm0[:, None], va0[:, None]))


@pytest.mark.parametrize("jacobian", [0, 1, 2])
def test_jacobian_policy_invariance(jacobian):
    """Where the next Jacobian is built -- speculatively inside the mismatch sweep
    (0), always there (1), or after the convergence check as the reference orders
    it (2, every Jacobian through the skipped-task launch) -- never changes a bit."""
    gc, plan, oplan, vm0, va0 = _setup("synth2383")
    ip, ix, _, yr, yi = S.build_ybus(gc)
    plan2 = S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, jacobian=jacobian)
    p0, q0 = montecarlo(gc, 150)
    p0[:, 7] *= 40.0  # one task that does not converge
    r = plan2.solve(p0, q0, vm0, va0)
    assert r.status[7] != 0 and (r.status == 0).sum() >= 140
    _compare(r, oplan.solve(p0, q0, vm0[:, None], va0[:, None]))


def test_solve_batches_pipeline_matches_single_solves():
    """gbnr_solve_batches (H2D / D2H overlapped with neighbouring solves) returns
    exactly what one gbnr_solve per batch returns."""
    gc, plan, oplan, vm0, va0 = _setup("synth300")
    T = 160
    batches = [montecarlo(gc, T, task0=i * T) for i in range(3)]
    outs = plan.solve_batches([b[0] for b in batches], [b[1] for b in batches], vm0, va0)
    for (p0, q0), r in zip(batches, outs):
        s = plan.solve(p0, q0, vm0, va0)
        for k in ("vm", "va", "iterations", "converged", "status", "max_mismatch"):
            np.testing.assert_array_equal(getattr(r, k), getattr(s, k))
        _compare(r, oplan.solve(p0, q0, vm0[:, None], va0[:, None]))


@pytest.mark.parametrize("name,T", [("case14", 0), ("synth300", 256), ("synth2383", 0), ("synth9241", 96)])
def test_n1_contingency_matches_oracle(name, T):
    """N-1 mode: one branch outage per task on the fixed
    pattern (per-task Ybus value sets, n_ysets = n_tasks), bit-identical to the
    oracle; tasks whose outage islands the grid are reported by the pre-check."""
    gc, plan, oplan, vm0, va0 = _setup(name)
    outages = np.arange(gc.n_branch) if T == 0 else \
        np.random.default_rng(11).integers(0, gc.n_branch, T).astype(np.int32)
    T = len(outages)
    yre, yim, islanded = S.contingency_values(gc, outages)
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0, va0, y=(yre, yim))
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], y=(yre, yim))
    _compare(r, o)
    assert (r.status[~islanded] == 0).mean() > 0.8
    if name == "synth2383":  # every branch: second chances capped per solve, islanded ones fail
        assert islanded.any() and (r.status[islanded] != 0).all()
    # the shared-Ybus path is untouched afterwards
    rs = plan.solve(p0, q0, vm0, va0)
    _compare(rs, oplan.solve(p0, q0, vm0[:, None], va0[:, None]))


@pytest.mark.parametrize("name,n1", [("case14", False), ("synth300", False), ("synth300", True)])
def test_branch_flows_match_oracle(name, n1):
    """calc_branch_flows on the device voltages of the last solve, bit-identical to
    the oracle (N-1: the outaged branch carries no flow)."""
    gc, plan, oplan, vm0, va0 = _setup(name)
    T = 96
    p0, q0 = montecarlo(gc, T)
    outages = np.random.default_rng(5).integers(0, gc.n_branch, T).astype(np.int32) if n1 else None
    y = None
    if n1:
        yre, yim, _ = S.contingency_values(gc, outages)
        y = (yre, yim)
    r = plan.solve(p0, q0, vm0, va0, y=y)
    sf, st = plan.branch_flows(gc, outages)
    osf, ost = po.Oracle().branch_flows(gc, S.branch_admittances(gc), r.vm, r.va, outage=outages)
    np.testing.assert_array_equal(sf, osf)
    np.testing.assert_array_equal(st, ost)
    if n1:
        assert (sf[outages, np.arange(T)] == 0).all()


@pytest.mark.parametrize("second_chance", [1, 0])
def test_second_chance_matches_oracle(second_chance):
    """a task whose frozen pivot collapses (here: a zero diagonal
    at a 90-degree start angle, test_oracle_nr._two_bus_instability) is re-planned
    alone with fresh pivoting at its current voltages and continues on the GPU;
    status, iterations and voltages match the oracle's second chance bitwise, and
    its batch peers match a solo run.  With second_chance = 0 it stays singular."""
    from test_oracle_nr import _two_bus_instability
    args, p0, q0, vm, va = _two_bus_instability(T=40, special=3)
    ip, ix, yr, yi, ref, pv, pq, vm0, va0 = args
    plan = S.NrPlan(2, ip, ix, yr, yi, ref, pv, pq, vm0, va0, device=0, second_chance=second_chance)
    r = plan.solve(p0, q0, vm, va, n_tasks=40)
    o = po.Oracle().plan(2, *args).solve(p0, q0, vm, va, n_tasks=40, second_chance=second_chance)
    _compare(r, o)
    assert r.status[3] == (3 if second_chance else 2)
    if second_chance:
        assert r.converged[3] and plan.timing()["fallback_converged"] == 1
    peers = np.r_[0:3, 4:40]
    assert (r.status[peers] == 0).all()
    solo = plan.solve(p0[:, :1], q0[:, :1], vm[:, :1], va[:, :1], n_tasks=1)
    np.testing.assert_array_equal(r.vm[:, peers], np.repeat(solo.vm, len(peers), axis=1))


def test_representative_rederivation_matches_oracle():
    """More than 5% of the tasks flagged at their first solve: gbnr_solve restarts
    the batch once from the worst-V0-mismatch task's pivots (SPEC.md DESIGN
    DECISIONS), exactly as the oracle does, then second chances what still fails."""
    from test_oracle_nr import _two_bus_instability
    args, p0, q0, vm, va = _two_bus_instability(T=8, special=3)
    ip, ix, yr, yi, ref, pv, pq, vm0, va0 = args
    plan = S.NrPlan(2, ip, ix, yr, yi, ref, pv, pq, vm0, va0, device=0)
    r = plan.solve(p0, q0, vm, va, n_tasks=8)
    o = po.Oracle().plan(2, *args).solve(p0, q0, vm, va, n_tasks=8)
    _compare(r, o)
    tm = plan.timing()
    assert tm["rederived"] == 1 and r.status[3] == 0 and tm["fallback_converged"] == 7


def test_runtime_modes_match_oracle():
    """batch_runtime modes through paper_2101_02270_b200.runtime:
    contingency over every case14 branch (islanded outages excluded by the
    pre-check, status ISLANDED) and a 24-step time series from a scenario CSV,
    each bit-identical to the oracle on the solved tasks."""
    from paper_2101_02270_b200 import runtime
    for name in ("synth30", "case14"):  # every outage of a 30-bus case
        gc, plan, oplan, vm0, va0 = _setup(name)
        inp = runtime.job_inputs(gc, "contingency", outages=np.arange(gc.n_branch))
        res = runtime.run(plan, gc, "contingency", outages=np.arange(gc.n_branch))
        keep = ~inp.islanded
        assert (res.status[~keep] == runtime.ISLANDED).all()
        assert (res.status[keep] == 0).mean() > 0.9
    assert (~keep).sum() == 1
    o = oplan.solve(inp.p0[:, keep], inp.q0[:, keep], vm0[:, None], va0[:, None],
                    y=(np.ascontiguousarray(inp.y[0][:, keep]), np.ascontiguousarray(inp.y[1][:, keep])))
    np.testing.assert_array_equal(res.status[keep], o["status"])
    np.testing.assert_array_equal(res.iterations[keep], o["iterations"])
    np.testing.assert_array_equal(res.vm[:, keep], o["vm"])
    assert res.report["counts"]["islanded"] == 1
    csv = "bus:4:p,bus:4:q,bus:9:p\n" + "\n".join(f"{40 + i},{-3 + 0.1 * i},{20 + i}" for i in range(24)) + "\n"
    ts = runtime.run(plan, gc, "timeseries", scenario_csv=csv)
    ti = runtime.job_inputs(gc, "timeseries", scenario_csv=csv)
    o = oplan.solve(ti.p0, ti.q0, vm0[:, None], va0[:, None])
    np.testing.assert_array_equal(ts.status, o["status"])
    np.testing.assert_array_equal(ts.va, o["va"])
    assert ts.report["counts"]["converged"] == 24


def test_full_size_batch_sampled_parity():
    """BASELINE configs[4] per-GPU slice at full size (synth9241 x 12.5k tasks, past
    the 2^31-element mark of a [zLU][B] tape, 64-bit tile offsets): tasks sampled
    across the batch -- first, last, both sides of tile boundaries -- match the
    oracle run on just those tasks bitwise (solo == batch)."""
    gc, plan, oplan, vm0, va0 = _setup("synth9241")
    T = 12500
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    assert (r.status == 0).all()
    pick = np.array([0, 1, 31, 32, 4095, 4096, 6250, 9999, 10000, 12287, 12288, 12479, 12480, 12498, 12499])
    o = oplan.solve(p0[:, pick], q0[:, pick], vm0[:, None], va0[:, None], n_tasks=len(pick))
    np.testing.assert_array_equal(r.iterations[pick], o["iterations"])
    np.testing.assert_array_equal(r.vm[:, pick], o["vm"])
    np.testing.assert_array_equal(r.va[:, pick], o["va"])
    np.testing.assert_array_equal(r.max_mismatch[pick], o["max_mismatch"])


def test_nonfinite_task_isolated():
    """A task with a NaN / inf injection (a corrupted scenario row) never converges
    (the max-norm treats NaN as inf), ends diverged after max_iter like the
    oracle's, and leaves every other task bit-identical (per-task independence,
    SPEC.md:216)."""
    gc, plan, oplan, vm0, va0 = _setup("synth118")
    T = 70
    p0, q0 = montecarlo(gc, T)
    p0[5, 10] = np.nan
    q0[7, 41] = np.inf
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    _compare(r, o)
    assert r.status[10] != 0 and r.status[41] != 0
    assert (np.delete(r.status, [10, 41]) == 0).all()


def _setup_case(gc, **opts):
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    plan = S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, device=0, **opts)
    oplan = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    return plan, oplan, vm0, va0


@pytest.mark.parametrize("name,extra,T", [("synth9241x", 0, 64), ("synth9241", 50, 64), ("synth9241", 100, 64),
                                          ("synth9241", 200, 64), ("synth9241", 1000, 32)])
def test_dense_grids_plan_and_match_oracle(name, extra, T):
    """execute_schedule for ANY frozen pattern: denser grids whose
    LU columns outgrow a walker's shared-memory pool (synth9241x: 250 long tie
    lines, nnzLU 341k, max_col 462; synth9241 + 50..1000 random branches, up to
    nnzLU 1.6M, max_col 1321) plan -- the too-large blocks and fetches run from
    global memory -- and solve bit-identically to the oracle."""
    from gen_cases import add_random_branches
    gc = load_case(util.case_path(name))
    if extra:
        gc = add_random_branches(gc, extra)
    # full-width tiles: the smallest per-walker pools, so the global forms run (a
    # narrower automatic width for 64 tasks would give every column shared rows)
    plan, oplan, vm0, va0 = _setup_case(gc, tile_width=32)
    p0, q0 = montecarlo(gc, T)
    r = plan.solve(p0, q0, vm0, va0, n_tasks=T)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None], n_tasks=T)
    assert (r.status == 0).mean() > 0.9
    _compare(r, o)
    if extra >= 100 or name == "synth9241x":
        assert plan.walk_info(0)["global_steps"] > 0


@pytest.mark.parametrize("frac", ["0.2", "0.05"])
def test_global_forms_match_oracle(frac, monkeypatch):
    """Blocks / fetches forced into global memory on a grid that fits (the
    fallback's code paths, GBNR_GLOBAL_FRAC): NR solve and the LU-only
    refactorization stay bit-identical to the oracle."""
    monkeypatch.setenv("GBNR_GLOBAL_FRAC", frac)
    gc = load_case(util.case_path("synth2383"))
    plan, oplan, vm0, va0 = _setup_case(gc)
    assert plan.walk_info(0)["global_steps"] > 0 and plan.walk_info(2)["global_steps"] > 0
    T = 100
    p0, q0 = montecarlo(gc, T)
    _compare(plan.solve(p0, q0, vm0, va0), oplan.solve(p0, q0, vm0[:, None], va0[:, None]))
    rng = np.random.default_rng(3)
    vm = vm0[:, None] * (1 + 0.02 * rng.standard_normal((gc.n_bus, 40)))
    va = va0[:, None] + 0.05 * rng.standard_normal((gc.n_bus, 40))
    plan.stage(p0[:, :40], q0[:, :40], vm, va)
    lu, flags, _ = plan.refactor(reps=2)
    olu, oflags = oplan.refactor(vm, va)
    np.testing.assert_array_equal(flags, oflags)
    np.testing.assert_array_equal(lu, olu)


@pytest.mark.parametrize("tw", [2, 8, 16, 24, 32, 14])
def test_tile_width_invariance(tw):
    """gbnr_options.tile_width (tasks per tile; the walk programs re-planned for the
    row budget of that width, lanes >= width shadowing the last real lane) never
    changes a bit: NR solve, N-1 per-task Ybus sets and the LU-only refactorization
    against the oracle.  14 is not one of the automatic widths (generic kernels)."""
    gc = load_case(util.case_path("synth2383"))
    plan, oplan, vm0, va0 = _setup_case(gc, tile_width=tw)
    T = 77
    p0, q0 = montecarlo(gc, T)
    _compare(plan.solve(p0, q0, vm0, va0), oplan.solve(p0, q0, vm0[:, None], va0[:, None]))
    outages = np.random.default_rng(4).integers(0, gc.n_branch, T).astype(np.int32)
    yre, yim, _ = S.contingency_values(gc, outages)
    _compare(plan.solve(p0, q0, vm0, va0, y=(yre, yim)),
             oplan.solve(p0, q0, vm0[:, None], va0[:, None], y=(yre, yim)))
    rng = np.random.default_rng(9)
    vm = vm0[:, None] * (1 + 0.02 * rng.standard_normal((gc.n_bus, 30)))
    va = va0[:, None] + 0.05 * rng.standard_normal((gc.n_bus, 30))
    plan.stage(p0[:, :30], q0[:, :30], vm, va)
    lu, flags, _ = plan.refactor(reps=1)
    olu, oflags = oplan.refactor(vm, va)
    np.testing.assert_array_equal(flags, oflags)
    np.testing.assert_array_equal(lu, olu)
