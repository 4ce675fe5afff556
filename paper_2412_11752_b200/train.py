"""The reference's fitting loop, drk::train (optimize.cpp:390-470), driven from the
host over the device path: per step one view (std::mt19937_64 draw, like the
reference), SH-degree warm-up, render -> loss (L1 + D-SSIM) -> backward_render ->
DensifyStats::accumulate -> adam_step, periodic densify_and_prune and checkpoints
(DRKSCENE), PSNR of the 8-bit quantised render at the evaluation cadence and at
the end.  Every per-pixel / per-primitive stage runs in this package's CUDA
kernels (the host only sequences the calls and reads the scalar loss / PSNR);
parameters, Adam moments and density statistics stay on the device.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .api import (DensifyStats, DeviceScene, FrameGrad, KernelConfig, OptState, Rasterizer, RenderOptions,
                  TrainConfig)
from .scenes import Camera


class MT19937_64:
    """std::mt19937_64 (the C++ standard fixes its output sequence): the view sampler
    of train (optimize.cpp:396, 407)."""

    N, M = 312, 156
    MATRIX_A, UPPER, LOWER = 0xB5026F5AA96619E9, 0xFFFFFFFF80000000, 0x7FFFFFFF
    MASK = (1 << 64) - 1

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.i = self.N

    def __call__(self) -> int:
        if self.i >= self.N:
            mt = self.mt
            for k in range(self.N):
                x = (mt[k] & self.UPPER) | (mt[(k + 1) % self.N] & self.LOWER)
                xa = x >> 1
                if x & 1:
                    xa ^= self.MATRIX_A
                mt[k] = mt[(k + self.M) % self.N] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEB88A000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK


@dataclass
class TrainView:
    """drk::TrainView (optimize.hpp:90-93): target image H x W x 3 (device f32) and camera."""

    image: torch.Tensor
    camera: Camera


@dataclass
class MetricRow:
    """drk::MetricRow (optimize.hpp:95-100)."""

    step: int = 0
    loss: float = 0.0
    psnr: float = -1.0
    count: int = 0


@dataclass
class TrainResult:
    """drk::TrainResult (optimize.hpp:102-106): params f32 [S, n] on the device."""

    params: torch.Tensor = None
    log: list = field(default_factory=list)
    final_psnr: float = 0.0


def train(views: list[TrainView], init: torch.Tensor, cfg: TrainConfig, k: int = 8,
          rast: Rasterizer | None = None) -> TrainResult:
    """drk::train (reference optimize.cpp:390-470) on raw parameters f32 [S, n]."""
    if not views:
        raise RuntimeError("training needs at least one posed view")  # optimize.cpp:392
    rast = rast or Rasterizer()
    dev = rast.device
    params = init.to(dev, torch.float32).contiguous().clone()
    S, n = params.shape
    state = OptState.zeros_like(params)
    stats = DensifyStats.zeros(n, dev)
    rng = MT19937_64(cfg.seed)
    extent = rast.scene_extent(params)
    kernel = cfg.kernel or KernelConfig(basis_count=k)
    ropt = RenderOptions(kernel=kernel, background=tuple(cfg.background), threads=cfg.threads)
    result = TrainResult()
    targets = [v.image.to(dev, torch.float32).contiguous() for v in views]
    terms = (S - (3 + 4 + 2 * k + 3)) // 3
    sh_deg_stored = int(round(terms ** 0.5)) - 1
    for step in range(cfg.steps):
        vi = 0 if len(views) == 1 else rng() % len(views)  # optimize.cpp:407
        view = views[vi]
        ropt.sh_degree = (min(cfg.max_sh_degree, step // cfg.sh_degree_warmup_interval)
                          if cfg.sh_degree_warmup_interval > 0 else cfg.max_sh_degree)
        fb = rast.render(params, view.camera, ropt, k=k)
        out, d_color = rast.loss(fb.color, targets[vi], cfg.dssim_weight)
        grads = rast.backward_render(params, FrameGrad(d_color=d_color))
        rast.densify_accumulate(grads, stats)
        rast.adam_step(params, grads.raw, state, cfg, extent, k=k)
        row = MetricRow(step=step, loss=float(out[0]), count=params.shape[1])
        if cfg.eval_interval > 0 and (step % cfg.eval_interval == 0 or step + 1 == cfg.steps):
            row.psnr = float(rast.psnr_quantized(fb.color, targets[vi]))
        result.log.append(row)
        done = step + 1
        if (cfg.densify_interval > 0 and done % cfg.densify_interval == 0 and
                done >= cfg.densify_start_step and done <= cfg.densify_stop_step):
            params = rast.densify_and_prune(params, state, stats, cfg, extent, k=k)
            stats = DensifyStats.zeros(params.shape[1], dev)
        elif params.shape[1] != stats.screen_grad_accum.numel():
            stats = DensifyStats.zeros(params.shape[1], dev)
        if (cfg.checkpoint_interval > 0 and cfg.checkpoint_path and params.shape[1] > 0 and
                done % cfg.checkpoint_interval == 0 and done < cfg.steps):
            rast.save_scene(DeviceScene(k, sh_deg_stored, params), f"{cfg.checkpoint_path}.{done}")
    ropt.sh_degree = cfg.max_sh_degree
    total = 0.0
    for vi, view in enumerate(views):
        fb = rast.render(params, view.camera, ropt, k=k)
        total += float(rast.psnr_quantized(fb.color, targets[vi]))
    result.final_psnr = total / len(views)
    result.params = params
    return result
