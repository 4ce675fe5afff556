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


# --- render -> backward -> all-reduce -> Adam across two ranks ---------------
# One training step of config 4's structure on a small scene: each rank renders
# its shard of the views, accumulates the raw gradients of the L1 loss, the
# ranks all-reduce (sum) and divide by the total view count (allreduce_mean_),
# and every rank applies the same Adam step.  The result must equal one process
# doing the same over all views, and the replicas must stay identical.

VIEWS = 4
LRS = [1e-3, 1e-3, 1e-3, 1e-3, 1e-3]


def _small_training_setup():
    from paper_2412_11752_b200 import scenes
    sc = scenes.random_scene(60, seed=21, sh_degree=1, clusters=3)
    cams = [scenes.look_at_camera(48, 32, (3.2 * np.cos(a), 0.4, 3.2 * np.sin(a))) for a in np.linspace(0.3, 2.2, VIEWS)]
    tgts = [scenes.config_target(2, c, view=i) for i, c in enumerate(cams)]
    return sc, cams, tgts


def _grads_cpu(sc, cams, tgts, views):
    """Sum over `views` of the reference's raw gradients of the L1 loss (oracle/_ref train_step)."""
    from oracle import ref
    g = np.zeros_like(sc.raw)
    for v in views:
        g += ref.train_step(sc, cams[v], tgts[v], ref.Options(sh_degree=1))["raw"]
    return g


def _adam_cpu(sc, g_mean):
    from oracle import ref
    p = sc.raw.astype(np.float64).copy()
    m, vv = np.zeros_like(p), np.zeros_like(p)
    ref.adam_step(p, g_mean, m, vv, sc.k, sc.terms, 0, LRS, 100, 2.0)
    return p


def _train_worker_cpu(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, cams, tgts = _small_training_setup()
    g = torch.from_numpy(_grads_cpu(sc, cams, tgts, shard_views(VIEWS, world, rank)))
    allreduce_mean_(g, VIEWS)
    p = _adam_cpu(sc, g.numpy())
    q.put((rank, p, params_checksum(torch.from_numpy(p))))
    dist.destroy_process_group()


def _run_two(target):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(600)
def test_gloo_two_ranks_training_step_matches_single_process():
    """CPU: the reference's per-view gradients (the oracle), gloo all-reduce, reference Adam."""
    res = _run_two(_train_worker_cpu)
    sc, cams, tgts = _small_training_setup()
    want = _adam_cpu(sc, _grads_cpu(sc, cams, tgts, range(VIEWS)) / VIEWS)
    assert res[0][2] == res[1][2]  # replicas in sync
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert np.abs(res[0][1] - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def _train_worker_gpu(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q.put((rank,) + _gpu_step(shard_views(VIEWS, world, rank), world))
    dist.destroy_process_group()


def _gpu_step(views, world):
    """GPU training step over `views`: render -> L1 -> deterministic backward
    (accumulated) -> all-reduce mean (CPU copy over gloo when world > 1) -> Adam."""
    from paper_2412_11752_b200.api import FrameGrad, OptState, Rasterizer, RenderOptions, TrainConfig
    sc, cams, tgts = _small_training_setup()
    r = Rasterizer(0)
    p = torch.from_numpy(sc.f32()).cuda()
    g = torch.zeros_like(p)
    opt = RenderOptions(sh_degree=1)
    for v in views:
        fb = r.render(p, cams[v], opt)
        _, dcol = r.l1_loss(fb.color, torch.from_numpy(tgts[v].astype(np.float32)).cuda())
        r.backward_render(p, FrameGrad(d_color=dcol), grad_out=g, accumulate=True, deterministic=True)
    gc = g.cpu()
    allreduce_mean_(gc, VIEWS)
    g.copy_(gc)
    st = OptState.zeros_like(p)
    cfg = TrainConfig(steps=100, lr_drk=1e-3, lr_position=1e-3, lr_rotation=1e-3, lr_opacity=1e-3, lr_sh=1e-3)
    r.adam_step(p, g, st, cfg, scene_extent=2.0)
    out = p.cpu().numpy().copy()
    r.close()
    return out, params_checksum(torch.from_numpy(out)), gc.numpy().copy()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_gloo_two_ranks_gpu_training_step():
    """GPU kernels in two ranks (both on cuda:0, gradients exchanged over gloo on
    host copies; the ranks never wait on each other's kernels): same parameters
    on both replicas, equal to one process over all views up to the fp32
    summation order of the per-view gradients, and the mean gradient within the
    parity tolerance of the reference's (oracle/_ref)."""
    res = _run_two(_train_worker_gpu)
    assert res[0][2] == res[1][2]
    np.testing.assert_array_equal(res[0][1], res[1][1])
    single, _, g_single = _gpu_step(range(VIEWS), 1)
    rel = np.linalg.norm(res[0][1] - single) / np.linalg.norm(single)
    assert rel <= 1e-6, rel
    sc, cams, tgts = _small_training_setup()
    g_ref = _grads_cpu(sc, cams, tgts, range(VIEWS)) / VIEWS
    assert np.linalg.norm(res[0][3] - g_ref) / np.linalg.norm(g_ref) <= 1e-3
