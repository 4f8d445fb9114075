"""Replica bookkeeping for `bench.py --gpus N` (the path does not shard; N GPUs
run N independent replicas of the config-5 batch).  The only cross-rank step is the timing:
every figure is taken as the maximum over ranks (the slowest replica bounds the job), and the
whole-job throughput is N x batch / that time.  Works on any process group: NCCL (CUDA
tensors) on the GPU box, gloo (CPU tensors) in the CPU tests."""

from __future__ import annotations

import torch


def max_over_ranks(x: float) -> float:
    """max of a per-rank scalar over the default process group (x itself without one)."""
    import torch.distributed as tdist

    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if tdist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(per_rank_units: int, per_rank_seconds: float) -> tuple[float, float]:
    """(whole-job units/s, slowest rank's seconds): world x units / max-over-ranks time."""
    import torch.distributed as tdist

    world = tdist.get_world_size() if (tdist.is_available() and tdist.is_initialized()) else 1
    t = max_over_ranks(per_rank_seconds)
    return world * per_rank_units / t, t
