"""Native NCCL gradient exchange (csrc/drk_comm.cu): reduce-scatter of the raw
gradients, drk::adam_step on the rank's shard, all-gather of the parameters.

On one GPU the communicator has one rank: the exchange must then equal a plain
drk_adam_step bitwise (same kernel, same scalars).  The multi-rank arithmetic
is the same code with shards of total / N scalars; its host logic (sharding,
mean over views) is covered by tests/test_distributed.py."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2412_11752_b200 import scenes

pytestmark = pytest.mark.gpu


def test_single_rank_allreduce_adam_equals_adam(rast):
    from paper_2412_11752_b200.api import OptState, TrainConfig
    from paper_2412_11752_b200.parallel import NcclComm
    comm = NcclComm(rast, 0, 1)
    try:
        sc = scenes.random_scene(1001, seed=3, sh_degree=3)  # total scalars not a multiple of the shard size
        p_a = torch.from_numpy(sc.f32()).cuda()
        p_b = p_a.clone()
        st_a, st_b = OptState.zeros_like(p_a), OptState.zeros_like(p_b)
        cfg = TrainConfig(steps=100, lr_drk=1e-3, lr_position=1e-3, lr_rotation=1e-3, lr_opacity=1e-3, lr_sh=1e-3)
        rng = np.random.default_rng(1)
        for _ in range(3):
            g = torch.from_numpy(rng.normal(0, 1, p_a.shape).astype(np.float32)).cuda()
            rast.adam_step(p_a, g.clone(), st_a, cfg, scene_extent=2.0, grad_scale=0.25)
            rast.allreduce_adam(comm, p_b, g.clone(), st_b, cfg, scene_extent=2.0, grad_scale=0.25)
        torch.cuda.synchronize()
        assert st_a.step == st_b.step == 3
        assert torch.equal(p_a, p_b) and torch.equal(st_a.m, st_b.m) and torch.equal(st_a.v, st_b.v)
        x = torch.arange(1000, dtype=torch.float32, device="cuda")
        y = comm.allreduce_sum_(x.clone())
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        comm.close()
