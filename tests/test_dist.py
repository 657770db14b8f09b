"""Multi-GPU host logic on CPU: world_size 2 over gloo.

Scenarios shard with no collective in the solve; the only communication is the
max-over-ranks time and the sum of converged counts around the timed region.
Each rank generates exactly its own slice with the counter-based RNG, so the
sharded batch is the same batch as the single-process one.  The per-rank solve
here is the oracle (this container has no GPU); the GPU path runs the same
dist plumbing in bench.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import util
from paper_2101_02270_b200 import dist
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo


def test_shard_partitions():
    for total in (1, 7, 10000, 100000):
        for world in (1, 2, 3, 8):
            spans = [dist.shard(total, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (a0, n0), (a1, _) in zip(spans, spans[1:]):
                assert a0 + n0 == a1
            assert sum(n for _, n in spans) == total
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_scenario_slices_are_counter_based():
    gc = load_case(util.case_path("synth118"))
    p, q = montecarlo(gc, 40)
    ps, qs = montecarlo(gc, 15, task0=10)
    np.testing.assert_array_equal(ps, p[:, 10:25])
    np.testing.assert_array_equal(qs, q[:, 10:25])
    p2, _ = montecarlo(gc, 40, mode="loadpv")
    assert not np.array_equal(p2, p)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import pyoracle as po
    rk = dist.init("gloo")
    gc = load_case(util.case_path("case14"))
    ip, ix, _, yr, yi = po.Oracle().build_ybus(gc)
    vm0, va0 = gc.v_start()
    plan = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    t0, n = dist.shard(total, rk.world, rk.rank)
    p0, q0 = montecarlo(gc, n, task0=t0)
    dist.barrier(rk)
    r = plan.solve(p0, q0, vm0[:, None], va0[:, None], n_threads=1)
    conv = dist.reduce_sum(rk, int(r["converged"].sum()))
    tmax = dist.reduce_max(rk, float(rk.rank + 1))
    g = dist.gather_columns(rk, [r["vm"], r["va"], r["iterations"]], total)
    if rk.is_root:
        np.save(os.path.join(os.environ["GBNR_TEST_OUT"], "gathered.npy"), np.concatenate([g[0], g[1]]))
    q.put((rk.rank, t0, r["iterations"].tolist(), conv, tmax))
    dist.finalize(rk)


def test_gloo_world2_sharded_solve_equals_single(tmp_path, monkeypatch):
    monkeypatch.setenv("GBNR_TEST_OUT", str(tmp_path))
    total, world = 101, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import pyoracle as po
    gc = load_case(util.case_path("case14"))
    ip, ix, _, yr, yi = po.Oracle().build_ybus(gc)
    vm0, va0 = gc.v_start()
    plan = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    p0, q0 = montecarlo(gc, total)
    full = plan.solve(p0, q0, vm0[:, None], va0[:, None])
    its = sum((r[2] for r in res), [])
    assert its == full["iterations"].tolist()
    assert all(r[3] == int(full["converged"].sum()) for r in res)
    assert all(r[4] == float(world) for r in res)
    # the final gather on rank 0 reassembles the whole batch's voltages
    np.testing.assert_array_equal(np.load(tmp_path / "gathered.npy"), np.concatenate([full["vm"], full["va"]]))
