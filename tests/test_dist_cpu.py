"""The N>1 bench path (independent replicas; the job time is the max over ranks) on CPU
with the gloo backend, world size 2."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ms = bench.max_over_ranks(10.0 + 5.0 * rank, world, "cpu")
    steps = 100
    value = world * steps / (ms / 1000.0)  # whole-job throughput of the replicas
    out[rank] = (ms, value)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == 15.0
    assert abs(out[0][1] - 2 * 100 / 0.015) < 1e-6


def _gather_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1812_08324_b200.hmatrix import allgather_varlen

    buf = torch.arange(3 + 2 * rank, dtype=torch.float64) + 100.0 * rank
    parts = allgather_varlen(buf)
    out[rank] = [p.tolist() for p in parts]
    dist.barrier()
    dist.destroy_process_group()


def test_allgather_varlen_gloo_world2():
    """The sharded-assembly exchange (variable-length factor buffers) on gloo, world 2."""
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29600 + os.getpid() % 1000
    mp.spawn(_gather_worker, args=(2, port, out), nprocs=2, join=True)
    want = [[0.0, 1.0, 2.0], [100.0, 101.0, 102.0, 103.0, 104.0]]
    assert out[0] == want and out[1] == want
