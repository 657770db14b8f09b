"""The product under two ranks (one process per GPU), on the GPU
box's single B200: both ranks' plans on cuda:0, gloo for the plumbing.  Each rank
solves its contiguous shard through the C ABI with no collective in the solve;
the final gather on rank 0 equals a single-process solve of the whole batch bit
for bit, and the max-over-ranks time / summed converged counts are consistent."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import util
from paper_2101_02270_b200 import dist
from paper_2101_02270_b200 import solver as S
from paper_2101_02270_b200.case import load_case
from paper_2101_02270_b200.scenarios import montecarlo

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, total, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    rk = dist.init("gloo")
    gc = load_case(util.case_path("synth2383"))
    plan = S.NrPlan.from_case(gc, device=0)
    vm0, va0 = gc.v_start()
    t0, n = dist.shard(total, rk.world, rk.rank)
    p0, q0 = montecarlo(gc, n, task0=t0)
    dist.barrier(rk)
    r = plan.solve(p0, q0, vm0, va0)
    ms = dist.reduce_max(rk, plan.timing()["total_ms"])
    conv = dist.reduce_sum(rk, int(r.converged.sum()))
    g = dist.gather_columns(rk, [r.vm, r.va, r.iterations, r.status], total)
    if rk.is_root:
        np.savez(os.path.join(out, "gathered.npz"), vm=g[0], va=g[1], it=g[2], st=g[3], ms=ms, conv=conv)
    plan.close()
    dist.finalize(rk)


def test_two_ranks_on_one_gpu_equal_single_process(tmp_path):
    total, world = 1000, 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, total, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    g = np.load(tmp_path / "gathered.npz")
    gc = load_case(util.case_path("synth2383"))
    plan = S.NrPlan.from_case(gc, device=0)
    vm0, va0 = gc.v_start()
    p0, q0 = montecarlo(gc, total)
    full = plan.solve(p0, q0, vm0, va0)
    np.testing.assert_array_equal(g["vm"], full.vm)
    np.testing.assert_array_equal(g["va"], full.va)
    np.testing.assert_array_equal(g["it"], full.iterations)
    np.testing.assert_array_equal(g["st"], full.status)
    assert int(g["conv"]) == int(full.converged.sum()) and float(g["ms"]) > 0.0
