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
