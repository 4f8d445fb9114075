"""`bench.py --gpus N` bookkeeping on CPU: two gloo ranks (replicas only, the
one cross-rank step is max-over-ranks timing and the whole-job throughput)."""

import os
import socket

import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2408_03571_b200.replicas import job_throughput, max_over_ranks

        t = 0.010 * (rank + 1)  # rank 1 is the slow replica
        out[rank] = (max_over_ranks(t), *job_throughput(32, t))
    finally:
        tdist.destroy_process_group()


def test_two_replicas_take_the_slowest_rank():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        mx, value, t = out[rank]
        assert mx == pytest.approx(0.020) and t == pytest.approx(0.020)
        assert value == pytest.approx(world * 32 / 0.020)  # whole-job units/s over the slowest rank


def test_single_process_is_identity():
    from paper_2408_03571_b200.replicas import job_throughput, max_over_ranks

    assert not tdist.is_initialized()
    assert max_over_ranks(0.5) == 0.5
    assert job_throughput(32, 0.5) == (64.0, 0.5)
