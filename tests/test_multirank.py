"""The N>1 bench path on CPU: two gloo ranks (127.0.0.1) aggregate their
device-timed totals the way bench.py does under torchrun (max over ranks of the
time, sum of the units; every rank owns an independent system)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms_total = [10.0, 14.0][rank]  # rank 1 is the slowest
    ms_step, units, value = bench.aggregate(ms_total, 1 << 26, 2, dist, "cpu")
    out[rank] = (ms_step, units, value)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_aggregation():
    world, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        ms_step, units, value = out[r]
        assert ms_step == pytest.approx(7.0)          # max(10, 14) / 2 steps
        assert units == 2 * (1 << 26)                 # both ranks' systems
        assert value == pytest.approx(units / 7e-3)


def test_single_rank_aggregation():
    import bench
    ms_step, units, value = bench.aggregate(5.0, 100, 5)
    assert (ms_step, units, value) == (1.0, 100.0, 100000.0)
