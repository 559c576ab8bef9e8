"""Multi-rank path of bench.py on CPU (gloo, world_size 2): replicas, max-over-ranks time, summed work
(DESIGN.md §8 "replicas only"; the sharded solver is NEXT-3)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, iters = bench.aggregate(10.0 + 5 * rank, 100 + rank, world, device="cpu")
    out[rank] = (ms, iters)
    dist.barrier()
    dist.destroy_process_group()


def test_aggregate_world2_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        ms, iters = out[r]
        assert ms == 15.0          # max over ranks
        assert iters == 201.0      # work of all replicas


def test_aggregate_single_rank():
    import bench
    assert bench.aggregate(3.0, 7, 1) == (3.0, 7)
