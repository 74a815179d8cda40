"""Multi-GPU replicas over right-hand-side columns.

The butterfly apply shards by right-hand sides: every rank holds the whole
plan and transforms its own columns, so there is no data-path collective
("replicas only"; SURVEY.md §8(e) first bullet).  The process group is only
used for the bench barrier and the max-over-ranks timing.  Host logic only —
works with NCCL (one process per GPU) and with gloo (CPU tests).
"""
from __future__ import annotations

import os

import numpy as np

import mht_inputs as mi


def env_world():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_seed(base: int, rank: int) -> int:
    """Distinct seeded streams per replica; rank 0 reproduces the single-GPU inputs."""
    return base + 1000 * rank


def rank_coefficients(w: mi.Workload, nrhs: int, rank: int) -> np.ndarray:
    if rank == 0:
        return mi.workload_coefficients(w, nrhs)
    if w.dtype == "complex128":
        return mi.complex_gaussian(nrhs, w.m, rank_seed(mi.SEED_COEF, rank))
    return mi.real_gaussian(nrhs, w.m, rank_seed(mi.SEED_COEF, rank))


def rank_adjoint_inputs(w: mi.Workload, nrhs: int, rank: int) -> np.ndarray:
    if rank == 0:
        return mi.workload_adjoint_input(w, nrhs)
    if w.dtype == "complex128":
        return mi.complex_gaussian(nrhs, w.n, rank_seed(mi.SEED_ADJ, rank))
    return mi.real_gaussian(nrhs, w.n, rank_seed(mi.SEED_ADJ, rank))


def split_columns(total_nrhs: int, world: int, rank: int):
    """Contiguous [start, stop) block of a global RHS batch owned by `rank`
    (used when a fixed global batch is spread over replicas)."""
    base, extra = divmod(total_nrhs, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allreduce_max(x: float, world: int, device=None) -> float:
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def job_throughput(units_per_rank: int, world: int, max_seconds: float) -> float:
    """Whole-job rate: units all ranks processed / the slowest rank's time."""
    return units_per_rank * world / max_seconds
