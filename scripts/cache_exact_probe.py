"""Diagnostic: the reference raster suite's "cache-sorted render equals the exact-sort
oracle under low overlap" scene (test_raster.cpp:199-220) through render_prims in
reference precision (fp64 alpha): cache vs exact-sort fp64 framebuffers."""
import ctypes as C
import math
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2412_11752_b200 import _lib, scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions

rng_vals = [float(x) for x in sys.argv[1:]] or None
g = np.random.default_rng(97)
K = 8
n = 6
mu = np.zeros((n, 3)); sc = np.zeros((n, K)); op = np.zeros(n); col = np.zeros((n, 3))
for i in range(n):
    u = g.uniform(size=8)
    mu[i] = [0.4 * (u[0] - 0.5), 0.4 * (u[1] - 0.5), 0.8 + 0.3 * u[2]]
    sc[i] = 0.2 + 0.2 * u[3]
    op[i] = 0.3 + 0.5 * u[4]
    col[i] = u[5:8]
steps = np.full(K, 0.5 + 1.0 / (K - 2))
th = np.cumsum(steps) * (2 * math.pi / steps.sum()); th[-1] = 2 * math.pi
tau = -0.1 + 1.09 * 0.36697247706422015
prims = dict(mu=torch.tensor(mu), rot=torch.eye(3, dtype=torch.float64).repeat(n, 1, 1),
             scales=torch.tensor(sc), angles=torch.tensor(np.tile(th, (n, 1))), eta=torch.full((n,), 0.5, dtype=torch.float64),
             tau=torch.full((n,), tau, dtype=torch.float64), opacity=torch.tensor(op),
             sh=torch.tensor(((col - 0.5) / 0.28209479177387814)[:, None, :]))
cam = scenes.simple_camera(48, 48)
r = Rasterizer(0)
r.set_counters(True)


def fb64():
    H = W = 48
    out = [np.zeros((H, W, 3)), np.zeros((H, W)), np.zeros((H, W, 3)), np.zeros((H, W))]
    _lib.check(_lib.lib().drk_get_framebuffers_f64(r._h, *[o.ctypes.data_as(C.c_void_p) for o in out]))
    return out


res = {}
for name, kw in (("cache", {}), ("exact", dict(exact_sort=True)), ("list", dict(use_cache=False))):
    for f64 in (True, False):
        r.render_prims(prims, cam, RenderOptions(sh_degree=0, fp64_alpha=f64, **kw))
        res[(name, f64)] = fb64()
        print(name, 'fp64' if f64 else 'fast', {k: r.stats()[k] for k in ('popped', 'composited', 'fp64_pixels')})
for f64 in (True, False):
    a, b = res[("cache", f64)], res[("exact", f64)]
    for nm, x, y in zip(("color", "depth", "normal", "alpha"), a, b):
        d = np.abs(x - y)
        print('fp64' if f64 else 'fast', nm, 'max diff', d.max(), 'n diff', int((d > 0).sum()),
              'at', np.unravel_index(np.argmax(d), d.shape))
