"""bench.py's multi-rank aggregation on CPU (gloo, world_size 2): the N > 1
path runs independent replicas (replicas only) and reports
value = (sum of iterations over ranks) / (max device time over ranks)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = [1200.0, 1500.0][rank]
    iters = [6000, 5800][rank]
    out[rank] = bench.combine_ranks(ms, iters, dist, torch.device("cpu"))
    dist.destroy_process_group()


def test_combine_ranks_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1] == (1500.0, 11800.0)


def test_combine_ranks_single():
    import bench
    assert bench.combine_ranks(10.0, 7, None, None) == (10.0, 7.0)
