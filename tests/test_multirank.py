"""The N>1 bench path on CPU (gloo, world_size 2): every rank solves its own
right-hand sides; whole-job time is the max over ranks, work the sum."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    # rank r: 100*(r+1) ms of device time for 10*(r+1) applies
    res = bench.aggregate(100.0 * (rank + 1), 10 * (rank + 1), 1.0 + rank, 7, dist=dist, device="cpu")
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_aggregate_two_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        dev_ms, applies, e2e_s, e2e_applies = out[r]
        assert dev_ms == 200.0 and applies == 30.0
        assert e2e_s == 2.0 and e2e_applies == 14.0


def test_aggregate_single_rank():
    assert bench.aggregate(5.0, 3, 1.5, 2) == (5.0, 3.0, 1.5, 2.0)
