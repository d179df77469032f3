"""Multi-GPU replica plumbing ("replicas only").

The forward has no exchange step: batch rows are independent (reference
src/model.cpp:397 loops b; SPEC.md:210 batch consistency), so N GPUs run N
independent model replicas -- one process per GPU, each with its own arena,
stream and CUDA graphs.  torch.distributed is used only for host plumbing:
a barrier around the timed region and the max-over-ranks of its duration.
No collective ever touches the data path.

bench.py drives every multi-rank run through this module (`ReplicaEnv`,
`rank_batch`, `timed_steps`, `max_over_ranks`, `aggregate_throughput`), and
tests/test_replicas_gloo.py runs bench.py itself under a 2-rank gloo launch with
a CPU stand-in for the device step.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass


@dataclass(frozen=True)
class ReplicaEnv:
    """One process per GPU (torchrun): RANK / WORLD_SIZE / LOCAL_RANK from the env."""
    rank: int = 0
    world: int = 1
    local: int = 0

    @classmethod
    def from_env(cls) -> "ReplicaEnv":
        return cls(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                   int(os.environ.get("LOCAL_RANK", "0")))


def shard_batch(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Strong scaling: contiguous share (start, count) of a fixed global batch;
    the first `global_batch % world` ranks take one extra sequence."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def rank_batch(batch: int, world: int, rank: int, strong: bool) -> tuple[int, int]:
    """Sequences this rank runs per step: weak scaling = `batch` per replica (global batch
    world * batch); strong = this rank's shard of a fixed global `batch`.  (start, count)."""
    if strong:
        return shard_batch(batch, world, rank)
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return rank * batch, batch


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


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """Units processed by the whole job (strong scaling: the shards differ by <= 1)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def aggregate_throughput(units_per_rank: int, world: int, seconds: float) -> float:
    """Whole-job units/s: every rank processed `units_per_rank` in `seconds` (max over ranks)."""
    return world * units_per_rank / seconds


class WallTimer:
    """Host wall-clock marks (the CPU stand-in used by the gloo test)."""

    def mark(self):
        return time.perf_counter()

    def elapsed_ms(self, a, b) -> float:
        return 1000.0 * (b - a)

    def sync(self):
        pass


class CudaEventTimer:
    """CUDA events recorded on the stream the step launches on (device time)."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream

    def mark(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def elapsed_ms(self, a, b) -> float:
        return a.elapsed_time(b)

    def sync(self):
        self.torch.cuda.synchronize()


def timed_steps(step, steps: int, warmup: int, timer, dist=None, device=None, before_timed=None):
    """W untimed warm-up steps, then EXACTLY `steps` timed steps bracketed by a barrier and a
    device synchronize on both sides.  Returns (per-step ms list, this rank's total ms,
    max-over-ranks total ms)."""
    for _ in range(warmup):
        step()
    timer.sync()

    def barrier():
        if dist is not None and dist.is_initialized():
            dist.barrier()
        timer.sync()

    if before_timed is not None:
        before_timed()
    barrier()
    marks = [timer.mark()]
    for _ in range(steps):
        step()
        marks.append(timer.mark())
    timer.sync()
    barrier()
    per = [timer.elapsed_ms(marks[i], marks[i + 1]) for i in range(steps)]
    total = timer.elapsed_ms(marks[0], marks[-1])
    return per, total, max_over_ranks(total, dist, device)
