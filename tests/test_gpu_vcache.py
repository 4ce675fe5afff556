"""K1 vertex cache (several views of one activation): the second forward of an
activation builds the cache of the wedge-tree leaves' world-space vertices,
later ones project it instead of expanding the tree.  Tile lists and
framebuffers must be the bits of a cold render of the same view, including
views where primitives are near-clipped (the serial K1 path)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions

pytestmark = pytest.mark.gpu


def _frame(r):
    b = r.tile_binning()
    st = r.stats()
    return b, st


def test_vertex_cache_views_bit_identical():
    sc = scenes.random_scene(12000, seed=41, sh_degree=3, clusters=10)
    raw = torch.from_numpy(sc.f32()).cuda()
    opt = RenderOptions(sh_degree=3)
    # orbit views, the last ones close enough that primitives cross the near plane
    cams = [scenes.look_at_camera(192, 128, (3.2 * np.cos(a), 0.4, 3.2 * np.sin(a))) for a in np.linspace(0, 5, 4)]
    cams += [scenes.look_at_camera(192, 128, (0.3, 0.1, -0.6)), scenes.look_at_camera(192, 128, (-0.2, 0.0, 0.5))]
    warm = Rasterizer(0)
    cold = Rasterizer(0)
    try:
        got, want = [], []
        for v, cam in enumerate(cams):
            fb = warm.render(raw, cam, opt) if v == 0 else warm.render_again(cam, opt)
            got.append(([t.clone() for t in (fb.color, fb.depth, fb.normal, fb.alpha)], _frame(warm)))
            fc = cold.render(raw, cam, opt)  # a fresh activation each time: plain K1
            want.append(([t.clone() for t in (fc.color, fc.depth, fc.normal, fc.alpha)], _frame(cold)))
        overflow_views = 0
        for (g_img, (g_b, g_st)), (w_img, (w_b, w_st)) in zip(got, want):
            for a, b in zip(g_img, w_img):
                assert torch.equal(a, b)
            assert np.array_equal(g_b.offsets, w_b.offsets)
            assert np.array_equal(g_b.prim_ids, w_b.prim_ids)
            assert np.array_equal(g_b.keys, w_b.keys)
            assert g_st["pairs"] == w_st["pairs"]
            assert g_st["poly_overflow"] == w_st["poly_overflow"]
            overflow_views += g_st["poly_overflow"] > 0
        assert overflow_views > 0  # the near-clip (serial) path is exercised with a built cache
    finally:
        warm.close()
        cold.close()
