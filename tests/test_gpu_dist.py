"""The product under two ranks: world_size 2 over gloo, both ranks
on cuda:0 (the box has one GPU; dist.device_of wraps local ranks onto the devices
present).  Each rank generates its own slice of the batch with the counter-based
RNG, solves it through the CUDA library with no collective on the data path, and
rank 0 gathers the voltages (dist.gather_columns).  The reassembled batch must
equal a single-process GPU solve and the oracle bit for bit; the rank timings and
converged counts go through the same max / sum reductions bench.py uses.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import pyoracle as po
import util
from paper_2101_02270_b200 import dist
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo

pytestmark = pytest.mark.gpu

CASE, TOTAL, WORLD = "synth2383", 301, 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan(gc):
    ip, ix, _, yr, yi = S.build_ybus(gc)
    vm0, va0 = gc.v_start()
    return S.NrPlan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0, device=0), vm0, va0


def _worker(rank, port, out_dir, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(WORLD), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    rk = dist.init("gloo")
    gc = load_case(util.case_path(CASE))
    plan, vm0, va0 = _plan(gc)
    t0, n = dist.shard(TOTAL, rk.world, rk.rank)
    p0, q0 = montecarlo(gc, n, task0=t0)
    dist.barrier(rk)
    r = plan.solve(p0, q0, vm0, va0)
    conv = dist.reduce_sum(rk, int(r.converged.sum()))
    g = dist.gather_columns(rk, [r.vm, r.va, r.iterations, r.status], TOTAL)
    if rk.is_root:
        np.savez(os.path.join(out_dir, "gathered.npz"), vm=g[0], va=g[1], it=g[2], st=g[3])
    q.put((rk.rank, t0, n, conv))
    dist.finalize(rk)


def test_two_ranks_on_the_gpu_equal_single_process_and_oracle(tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, str(tmp_path), q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [0, dist.shard(TOTAL, WORLD, 1)[0]]
    g = np.load(tmp_path / "gathered.npz")

    gc = load_case(util.case_path(CASE))
    plan, vm0, va0 = _plan(gc)
    p0, q0 = montecarlo(gc, TOTAL)
    single = plan.solve(p0, q0, vm0, va0)
    assert all(r[3] == int(single.converged.sum()) for r in res)
    np.testing.assert_array_equal(g["it"], single.iterations)
    np.testing.assert_array_equal(g["st"], single.status)
    np.testing.assert_array_equal(g["vm"], single.vm)
    np.testing.assert_array_equal(g["va"], single.va)

    ip, ix, _, yr, yi = po.Oracle().build_ybus(gc)
    oplan = po.Oracle().plan(gc.n_bus, ip, ix, yr, yi, gc.slack, gc.pv, gc.pq, vm0, va0)
    o = oplan.solve(p0, q0, vm0[:, None], va0[:, None])
    np.testing.assert_array_equal(g["st"], o["status"])
    np.testing.assert_array_equal(g["it"], o["iterations"])
    ok = g["st"] == 0
    np.testing.assert_array_equal(g["vm"][:, ok], o["vm"][:, ok])
    np.testing.assert_array_equal(g["va"][:, ok], o["va"][:, ok])
