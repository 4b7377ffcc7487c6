"""World-size-2 gloo run of the histogram all-reduce the sharded Refine-and-Prune
uses (reduce_hist): exact integer SUM of the bins, SUM of invalid counts, MAX of
max_len — so every rank then partitions the same summed histogram."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_21758_b200.ewsjf import reduce_hist
    h = workload.heavy(50_000, 5)
    a, b = workload.shard_range(len(h), rank, world)
    mine = np.bincount(h[a:b], minlength=(1 << 20) + 1).astype(np.int32)
    hist, info = reduce_hist(torch.from_numpy(mine), {"invalid": rank, "over": 0, "max_len": int(h[a:b].max())})
    out[rank] = (hist.numpy().copy(), info)
    dist.destroy_process_group()


def test_reduce_hist_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    h = workload.heavy(50_000, 5)
    ref = np.bincount(h, minlength=(1 << 20) + 1)
    for r in range(world):
        hist, info = out[r]
        np.testing.assert_array_equal(hist, ref)
        assert info == {"invalid": 1, "over": 0, "max_len": int(h.max())}


def _worker_over(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_21758_b200.ewsjf import EwsjfError, check_reduced, reduce_hist
    h = workload.heavy(20_000, 6)
    a, b = workload.shard_range(len(h), rank, world)
    mine = h[a:b].copy()
    if rank == 1:
        mine[7] = 1 << 21            # one over-long prompt on one shard only
    over = int((mine >= (1 << 20)).sum())
    binned = np.bincount(mine[mine < (1 << 20)], minlength=(1 << 20) + 1).astype(np.int32)
    hist, info = reduce_hist(torch.from_numpy(binned), {"invalid": 0, "over": over, "max_len": int(mine.max())})
    try:
        check_reduced(info)
        out[rank] = ("ok", info["over"])
    except EwsjfError as e:
        out[rank] = ("raised", e.status)
    dist.destroy_process_group()


def test_over_long_length_on_one_shard_raises_on_every_rank():
    """a shard with a length >= 2^20 must not leave the other ranks
    blocked in the all-reduce; all ranks reduce, then all refuse together."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_over, args=(world, port, out), nprocs=world, join=True, )
    from paper_2601_21758_b200 import _lib as L
    assert out[0] == ("raised", L.UNSUPPORTED) and out[1] == ("raised", L.UNSUPPORTED)
