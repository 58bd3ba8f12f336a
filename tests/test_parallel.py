"""Multi-GPU host logic on CPU: member sharding and the single sketch
exchange (all-reduce of the owned Gamma rows), world_size 2 over gloo."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23571_b200.parallel import gather_sketch_rows, max_over_ranks, shard


def test_shard_partitions():
    for total in (0, 1, 7, 200, 401):
        for world in (1, 2, 3, 8):
            parts = [shard(total, world, r) for r in range(world)]
            assert sum(c for _, c in parts) == total
            off = 0
            for o, c in parts:
                assert o == off
                off += c


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total, n, ell = 7, 5, 5
    off, cnt = shard(total, world, rank)
    # member j's Gamma row is filled with j (+ a column ramp)
    rows = torch.stack([torch.full((n,), float(off + i)) + torch.arange(n) for i in range(cnt)])
    g = gather_sketch_rows(rows, off, ell)
    t = max_over_ranks(1.0 + rank, torch.device("cpu"))
    out[rank] = (g.tolist(), t)
    dist.destroy_process_group()


def test_gloo_sketch_exchange():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    expect = [[float(j + c) for c in range(5)] for j in range(5)]
    for r in range(world):
        assert res[r][0] == expect
        assert res[r][1] == 2.0
