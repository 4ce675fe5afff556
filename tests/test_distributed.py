"""Multi-process host logic with the gloo backend (world size 2, CPU): view
sharding covers every view once, and the gradient exchange returns the mean
over all views on every rank with replicas in sync."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_11752_b200.parallel import allreduce_mean_, params_checksum, shard_views


def test_shard_views_partition():
    for world in (1, 2, 3, 8):
        for costs in (None, np.random.default_rng(world).uniform(1, 5, 64)):
            owned = sorted(v for r in range(world) for v in shard_views(64, world, r, costs))
            assert owned == list(range(64))
    costs = np.array([10.0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1])
    loads = [costs[shard_views(11, 2, r, costs)].sum() for r in range(2)]
    assert max(loads) - min(loads) <= 1.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, views, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_views(views, world, rank)
    # per-view "gradients" are deterministic functions of the view id
    g = torch.zeros(6, 5, dtype=torch.float32)
    for v in mine:
        g += torch.full((6, 5), float(v + 1))
    allreduce_mean_(g, views)
    p = torch.ones(6, 5) - 0.01 * g  # identical update on every rank
    q.put((rank, mine, g.numpy().copy(), params_checksum(p)))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_two_ranks_gradient_mean():
    world, views = 2, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, views, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    res.sort()
    assert sorted(res[0][1] + res[1][1]) == list(range(views))
    expect = np.mean(np.arange(1, views + 1))
    for _, _, g, _ in res:
        assert np.allclose(g, expect)
    assert res[0][3] == res[1][3]
