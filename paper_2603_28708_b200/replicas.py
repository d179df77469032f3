"""Multi-GPU replica plumbing ("replicas only").

The forward has no exchange step: batch rows are independent (reference
src/model.cpp:397 loops b; SPEC.md:210 batch consistency), so N GPUs run N
independent model replicas -- one process per GPU, each with its own arena,
stream and CUDA graphs.  torch.distributed is used only for host plumbing:
a barrier around the timed region and the max-over-ranks of its duration.
No collective ever touches the data path.
"""
from __future__ import annotations


def shard_batch(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Strong scaling: contiguous share (start, count) of a fixed global batch;
    the first `global_batch % world` ranks take one extra sequence."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def replica_token_seed(base_seed: int, rank: int) -> int:
    """Weak scaling: each replica draws its own synthetic token batch."""
    return base_seed + rank


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Timing reduction: the slowest rank defines the step time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: int, world: int, seconds: float) -> float:
    """Whole-job units/s: every rank processed `units_per_rank` in `seconds` (max over ranks)."""
    return world * units_per_rank / seconds
