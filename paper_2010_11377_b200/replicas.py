"""Multi-GPU = independent replicas.

The IRK solve does not shard (sequential time steps, global GMRES dot
products, stage-sequential LD sweep), so `bench.py --gpus N` runs one
independent trajectory per GPU.  This module holds the host-side aggregation
shared by the bench and the gloo tests: a barrier, the max of the per-rank
device times, and the whole-job throughput.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def max_over_ranks(value: float, device: str = "cpu") -> float:
    """Maximum of a per-rank scalar (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def whole_job_throughput(steps_per_rank: int, world_size: int, max_ms: float) -> float:
    """Solves/s of the whole job: every rank's steps over the slowest rank's time."""
    if max_ms <= 0.0:
        raise ValueError("whole_job_throughput: time must be positive")
    return world_size * steps_per_rank / (max_ms / 1e3)
