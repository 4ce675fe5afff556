"""Shared fixtures-as-functions for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from paper_2412_11752_b200 import scenes
from oracle import ref


def opt_for(sh_degree=0, **kw):
    return ref.Options(sh_degree=sh_degree, **kw)


def api_options(o: ref.Options):
    from paper_2412_11752_b200.api import KernelConfig, PresortMode, RenderOptions
    return RenderOptions(kernel=KernelConfig(lowpass_radius=o.lowpass_radius, alpha_min=o.alpha_min,
                                             grazing_eps=o.grazing_eps),
                         background=tuple(o.background), sh_degree=o.sh_degree, use_cache=o.use_cache,
                         exact_sort=o.exact_sort, presort=PresortMode(o.presort),
                         early_stop_transmittance=o.early_stop_transmittance)


def small_scene(seed=0, n=60, sh_degree=0, k=8, clusters=0):
    sc = scenes.random_scene(n, seed=seed, k=k, sh_degree=sh_degree, clusters=clusters)
    cam = scenes.look_at_camera(64, 48, (0.3, -0.2, -3.5))
    return sc, cam


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
