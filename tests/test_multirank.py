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


def _worker_rhs(rank, ws, port, out):
    import numpy as np

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    assert bench.dist_env() == (ws, rank, rank)
    b0 = np.linspace(-1.0, 1.0, 64)
    b = bench.rank_rhs(b0, rank)
    # every rank's unit of work is its own: gather the vectors and compare
    gathered = [torch.zeros(64, dtype=torch.float64) for _ in range(ws)]
    dist.all_gather(gathered, torch.tensor(b))
    out[rank] = [g.numpy().tolist() for g in gathered]
    dist.barrier()
    dist.destroy_process_group()


def test_ranks_solve_distinct_right_hand_sides():
    """N > 1 shards right-hand sides: rank 0 keeps the config's b, the others
    draw their own seeded vectors; every rank sees the same assignment."""
    import numpy as np

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_rhs, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]
    b0, b1 = np.array(out[0][0]), np.array(out[0][1])
    assert np.array_equal(b0, np.linspace(-1.0, 1.0, 64))
    assert not np.allclose(b0, b1) and np.all(np.abs(b1) <= 1.0)
    assert np.array_equal(b1, bench.rank_rhs(b0, 1))  # deterministic per rank


def test_aggregate_single_rank():
    assert bench.aggregate(5.0, 3, 1.5, 2) == (5.0, 3.0, 1.5, 2.0)
