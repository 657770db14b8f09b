"""Multi-GPU plumbing: one process per GPU, scenarios sharded, no collective in the solve.

Tasks are independent, so a batch is split into contiguous
per-rank slices of task ids; each rank generates its own slice with the
counter-based scenario RNG and runs its own plan on its own device.  The only
communication is outside the timed solve: a barrier before and after, and a
max-reduction of the per-rank device times (the job is as slow as its slowest
rank) plus a sum of the per-rank converged counts.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class Rank:
    rank: int = 0
    world: int = 1
    local_rank: int = 0

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def from_env() -> Rank:
    return Rank(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                int(os.environ.get("LOCAL_RANK", 0)))


def shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [task0, task0 + count) of n_total tasks for rank."""
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    task0 = rank * base + min(rank, extra)
    return task0, count


def init(backend: str | None = None) -> Rank:
    """Join the job.  Backend: nccl when GPUs are visible, else gloo;
    GBNR_DIST_BACKEND overrides (gloo lets several ranks share one GPU in tests)."""
    r = from_env()
    if r.world > 1:
        import torch.distributed as td
        if not td.is_initialized():
            backend = backend or os.environ.get("GBNR_DIST_BACKEND")
            if backend is None:
                import torch
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                import torch
                torch.cuda.set_device(device_of(r))
            td.init_process_group(backend=backend)
    return r


def device_of(r: Rank) -> int:
    """CUDA ordinal of a rank: one GPU per rank (wrapping when ranks outnumber GPUs)."""
    import torch
    n = torch.cuda.device_count()
    return r.local_rank % n if n else 0


def _device():
    import torch
    import torch.distributed as td
    return torch.device("cuda", torch.cuda.current_device()) \
        if td.get_backend() == "nccl" else torch.device("cpu")


def barrier(r: Rank) -> None:
    if r.world > 1:
        import torch.distributed as td
        td.barrier()


def reduce_max(r: Rank, x: float) -> float:
    if r.world == 1:
        return float(x)
    import torch
    import torch.distributed as td
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(r: Rank, x: float) -> float:
    if r.world == 1:
        return float(x)
    import torch
    import torch.distributed as td
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    td.all_reduce(t, op=td.ReduceOp.SUM)
    return float(t.item())


def gather_columns(r: Rank, arrays, total: int):
    """The final host gather: every rank's result arrays, columns
    [task0, task0 + count) of its shard (2-D [rows][count] or 1-D [count]), are
    assembled on rank 0 into arrays over all `total` tasks; other ranks get None.
    Runs once after the solve, outside any timed region."""
    import numpy as np
    if r.world == 1:
        return list(arrays)
    import torch.distributed as td
    task0, count = shard(total, r.world, r.rank)
    parts = [None] * r.world if r.is_root else None
    td.gather_object((task0, [np.asarray(a) for a in arrays]), parts, dst=0)
    if not r.is_root:
        return None
    out = []
    for i, a in enumerate(arrays):
        a = np.asarray(a)
        full = np.empty(a.shape[:-1] + (total,), a.dtype)
        for t0, arrs in parts:
            full[..., t0:t0 + arrs[i].shape[-1]] = arrs[i]
        out.append(full)
    return out


def finalize(r: Rank) -> None:
    if r.world > 1:
        import torch.distributed as td
        if td.is_initialized():
            td.destroy_process_group()
