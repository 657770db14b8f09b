"""Scenario CSV and outage-list front ends (case_io.hpp:368-471),
checked against the reference's own parsers on committed fixtures
(tests/golden/io_kats.json, made by tools/make_golden.py from oracle/_ref)."""
import json
import os

import numpy as np
import pytest

import util
from paper_2101_02270_b200.case import CaseError, load_case, parse_outage_list, parse_scenario_csv
from paper_2101_02270_b200 import runtime

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "io_kats.json")))
GC = load_case(util.case_path(KATS["case"]))


@pytest.mark.parametrize("key", sorted(KATS["scenario"]))
def test_scenario_csv_matches_reference(key):
    k = KATS["scenario"][key]
    if "error" in k:
        with pytest.raises(CaseError) as e:
            parse_scenario_csv(k["text"], GC)
        assert e.value.code == k["error"]
    else:
        p, q = parse_scenario_csv(k["text"], GC)
        np.testing.assert_array_equal(p, np.array(k["p_mw"]))
        np.testing.assert_array_equal(q, np.array(k["q_mvar"]))


@pytest.mark.parametrize("key", sorted(KATS["outages"]))
def test_outage_list_matches_reference(key):
    k = KATS["outages"][key]
    if "error" in k:
        with pytest.raises(CaseError) as e:
            parse_outage_list(k["text"], GC)
        assert e.value.code == k["error"]
    else:
        np.testing.assert_array_equal(parse_outage_list(k["text"], GC), k["branches"])


def test_job_inputs_per_mode():
    """batch_runtime modes (JobSpec): the per-task inputs each mode
    hands to the solver."""
    T = 5
    mc = runtime.job_inputs(GC, "montecarlo", n_tasks=T)
    assert mc.p0.shape == (GC.n_bus, T) and mc.y is None and not mc.islanded.any()
    ts = runtime.job_inputs(GC, "timeseries", scenario_csv=KATS["scenario"]["valid_two_rows"]["text"])
    p_mw, q_mvar = parse_scenario_csv(KATS["scenario"]["valid_two_rows"]["text"], GC)
    p0, q0 = GC.profiles(p_mw, q_mvar)
    np.testing.assert_array_equal(ts.p0, p0)
    np.testing.assert_array_equal(ts.q0, q0)
    one = runtime.job_inputs(GC, "single")
    assert one.p0.shape == (GC.n_bus, 1)
    ct = runtime.job_inputs(GC, "contingency", outages="0 1 2 13\n")
    assert ct.y[0].shape == (int(GC.ybus()[0][-1]), 4)
    # case14 branch 13 (7-8) is the only line to bus 8: its outage islands the grid
    np.testing.assert_array_equal(ct.islanded, [False, False, False, True])
    with pytest.raises(ValueError):
        runtime.job_inputs(GC, "contingency")


def test_sample_montecarlo_distribution_table():
    """sample_montecarlo: per-bus {normal, uniform, fixed}
    multipliers on the loads, seeded and counter-based; generator dispatch untouched."""
    from paper_2101_02270_b200.scenarios import sample_montecarlo
    T = 10000
    p_fix, q_fix = sample_montecarlo(GC, ("fixed", 1.0), 7)
    p_base, q_base = GC.profiles(GC.pd, GC.qd)
    np.testing.assert_array_equal(p_fix, np.repeat(p_base, 7, 1))  # all fixed -> n identical tasks
    np.testing.assert_array_equal(q_fix, np.repeat(q_base, 7, 1))
    a = sample_montecarlo(GC, ("normal", 1.0, 0.1), T, seed=5)
    b = sample_montecarlo(GC, ("normal", 1.0, 0.1), T, seed=5)
    np.testing.assert_array_equal(a[0], b[0])  # same seed -> identical tables
    load = np.nonzero(GC.pd)[0][0]
    gen_p = GC.gen_injection()[0][load] / GC.base_mva
    s = (gen_p - a[0][load]) / (GC.pd[load] / GC.base_mva)  # the drawn multipliers
    assert abs(s.mean() - 1.0) < 0.01 and abs(s.std() - 0.1) < 0.01  # 3 sigma / sqrt(n) bounds
    # a slice drawn on its own equals the same tasks of the full table
    sl = sample_montecarlo(GC, ("normal", 1.0, 0.1), 5, task0=100, seed=5)
    np.testing.assert_array_equal(sl[0], a[0][:, 100:105])
    u = sample_montecarlo(GC, [("uniform", 0.9, 1.1)] * GC.n_bus, 1000)
    su = (gen_p - u[0][load]) / (GC.pd[load] / GC.base_mva)
    assert su.min() >= 0.9 - 1e-12 and su.max() <= 1.1 + 1e-12
    for bad in (("normal", 1.0, -0.1), ("uniform", 1.2, 0.8), ("weird", 1.0), ("fixed", 1.0, 2.0)):
        with pytest.raises(ValueError):
            sample_montecarlo(GC, bad, 3)
    with pytest.raises(ValueError):
        sample_montecarlo(GC, [("fixed", 1.0)] * (GC.n_bus - 1), 3)


def test_solver_rejects_mismatched_set_counts():
    """Host-side argument checks of NrPlan (no compute): q0 must carry p0's set
    count and va0 vm0's, otherwise the C side would read past a host array."""
    from paper_2101_02270_b200 import solver as S
    plan = S.NrPlan.from_case(GC, device=-1)
    n, T = GC.n_bus, 4
    vm0, va0 = GC.v_start()
    p = np.zeros((n, T))
    with pytest.raises(ValueError):
        plan.solve(p, np.zeros(n), vm0, va0)          # q0 shared, p0 per task
    with pytest.raises(ValueError):
        plan.stage(p, p, np.ones((n, T)), va0)        # va0 shared, vm0 per task
    with pytest.raises(ValueError):
        plan.solve(p, p, vm0, va0, y=(np.zeros(3), np.zeros(4)))
    with pytest.raises(ValueError):
        plan.solve(np.zeros((n + 1, T)), np.zeros((n + 1, T)), vm0, va0)
    with pytest.raises(ValueError):
        plan.solve_batches([p, p], [p], vm0, va0)
    with pytest.raises(ValueError):
        plan.solve_batches([p, np.zeros((n, T + 1))], [p, np.zeros((n, T + 1))], vm0, va0)
    with pytest.raises(ValueError):
        runtime.run(plan, GC, "single", batch_size=0)
    plan.close()
