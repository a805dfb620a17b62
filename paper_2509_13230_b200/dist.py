"""Multi-GPU plumbing for the sampler.

The samples of an ensemble are independent (counter-based Philox keyed by the sample index,
DESIGN.md R1), so the path shards by samples with NO data-path collective: rank r draws sample
indices [r*R, (r+1)*R) of the same plan (weak scaling).  The only collectives are for timing
and accounting (max of elapsed time, sum of counters) over torch.distributed (NCCL on GPUs,
gloo on CPU in tests).
"""
from __future__ import annotations

import os


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def shard_samples(rank: int, world: int, samples_per_rank: int, first: int = 0):
    """(first_sample, n_samples) of rank `rank`: contiguous, disjoint, covering world*R samples."""
    if not (0 <= rank < world) or samples_per_rank < 0:
        raise ValueError("bad shard arguments")
    return first + rank * samples_per_rank, samples_per_rank


def reduce_max(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(values, device=None):
    import torch
    import torch.distributed as dist
    vals = [float(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]
