"""Parity at BASELINE scale: the CUDA path against the reference build
(oracle/_ref, the unmodified reference sources, all host threads) on full
config-1 and config-2 frames, config-3 orbit views (near-clipped primitives:
the K1 large-polygon path k_prep1) and a config-4 view binned in bands.

Reference tile lists come from ref_bin_parallel (the reference bin_primitives
on chunks of the primitives, merged with its own comparator; equal to one call,
tests/test_oracle.py::test_reference_parallel_binning_is_exact).  Crops
(configs 3 and 4, where one reference render of every primitive would take
minutes) are rendered by the reference on the primitives of the crop's tile
lists, in id order: render reads primitives only through the tile lists, and
the (key, id) order is preserved, so the crop's framebuffers are the full
scene's.  Bars (BASELINE.json north_star): tile lists bit-exact, framebuffers
within 1e-4 max abs, gradients within 1e-3 relative L2, touched equal.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ref
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import FrameGrad
from tests.helpers import api_options, rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FB_TOL = 1e-4
GRAD_TOL = 1e-3


def _bins_equal(gpu_bins, orc_bins):
    off, ids, keys = orc_bins
    np.testing.assert_array_equal(gpu_bins.offsets, off)
    np.testing.assert_array_equal(gpu_bins.prim_ids, ids)
    np.testing.assert_array_equal(gpu_bins.keys.view(np.uint64), keys.view(np.uint64))


def _fb_close(fb, orc):
    for f in ("color", "depth", "normal", "alpha"):
        err = float(np.abs(getattr(fb, f).cpu().numpy().astype(np.float64) - orc[f]).max())
        assert err <= FB_TOL, (f, err)


def _subset(sc, ids):
    keep = np.unique(ids)
    return scenes.Scene(raw=np.ascontiguousarray(sc.raw[:, keep]), k=sc.k, sh_degree=sc.sh_degree), keep


def test_config1_full_frame(rast):
    sc = scenes.config_scene(1)
    cam = scenes.config_cameras(1)[0]
    o = ref.Options(sh_degree=3, threads=0)
    fb = rast.render(sc.f32(), cam, api_options(o))
    bins = rast.tile_binning()
    orc_bins = ref.bin_primitives_parallel(sc, cam, o)
    assert len(orc_bins[1]) > 10_000_000
    _bins_equal(bins, orc_bins)
    _fb_close(fb, ref.render(sc, cam, o))


def test_config2_full_frame_forward_backward(rast):
    sc = scenes.config_scene(2)
    cam = scenes.config_cameras(2)[0]
    tgt = scenes.config_target(2, cam)
    o = ref.Options(sh_degree=3, threads=0)
    fb = rast.render(sc.f32(), cam, api_options(o))
    bins = rast.tile_binning()
    _bins_equal(bins, ref.bin_primitives_parallel(sc, cam, o))
    orc = ref.fwd_bwd(sc, cam, tgt, o)
    _fb_close(fb, orc)
    loss, dcol = rast.l1_loss(fb.color, torch.from_numpy(tgt.astype(np.float32)).cuda())
    assert abs(float(loss) - orc["loss"]) <= 1e-6
    # the same frame gradient (the reference's dL/dC, f32) into both backward passes
    fg = FrameGrad(d_color=torch.from_numpy(orc["d_color"].astype(np.float32)))
    for det in (False, True):
        g = rast.backward_render(sc.f32(), fg, deterministic=det)
        assert rel_l2(g.raw.cpu().numpy(), orc["raw"]) <= GRAD_TOL
        assert rel_l2(g.d_center_world.cpu().numpy(), orc["d_center_world"]) <= GRAD_TOL
        assert rel_l2(g.screen_grad.cpu().numpy(), orc["screen_grad"]) <= GRAD_TOL
        np.testing.assert_array_equal(g.touched.cpu().numpy(), orc["touched"])


def _crop_parity(rast, sc, cam, o, band_limit_div=0):
    """GPU render of the crop (full scene) vs the reference: bit-exact tile lists
    (all primitives, parallel reference binning), framebuffers of the reference
    render of the crop's primitives."""
    if band_limit_div:
        rast.render(sc.f32(), cam, api_options(o))
        pairs = rast.stats()["pairs"]
        rast.set_band_limit(max(1, pairs // band_limit_div))
    try:
        fb = rast.render(sc.f32(), cam, api_options(o))
        st = rast.stats()
        bands = rast.bands()
        bins = rast.tile_binning()
    finally:
        if band_limit_div:
            rast.set_band_limit(0)
    orc_bins = ref.bin_primitives_parallel(sc, cam, o)
    _bins_equal(bins, orc_bins)
    sub, keep = _subset(sc, orc_bins[1])
    _fb_close(fb, ref.render(sub, cam, o))
    return st, bands, len(orc_bins[1])


def _centre_crop(cam0, size):
    return cam0.crop(cam0.width // 2 // 16 * 16 - size // 2, cam0.height // 2 // 16 * 16 - size // 2, size, size)


def test_config3_orbit_view_crops(rast):
    """Two orbit views of the 1M-primitive scene whose binning sends primitives
    through the large-polygon path (k_prep1: polygons clipped at the near plane,
    raster.cpp:15-30 / :209, or too many vertices for the warp path): the first
    two of the 64 views where that counter is nonzero, on a centred 128 x 128
    crop; at least one of them has such a primitive (centre within 6 largest
    scales of the camera plane) in the crop's tile lists."""
    sc = scenes.config_scene(3)
    cams = scenes.config_cameras(3)
    o = ref.Options(sh_degree=3, threads=0)
    raw = torch.from_numpy(sc.f32()).cuda()
    picked = []
    for v, cam0 in enumerate(cams):
        rast.render(raw, _centre_crop(cam0, 128), api_options(o))
        if rast.stats()["poly_overflow"] > 0:
            picked.append(v)
        if len(picked) == 2:
            break
    assert len(picked) == 2, "no orbit view exercises the large-polygon path"
    smax = np.exp(sc.raw[7:15].max(axis=0))
    near_in_lists = 0
    for v in picked:
        cam = _centre_crop(cams[v], 128)
        st, _, pairs = _crop_parity(rast, sc, cam, o)
        assert st["poly_overflow"] > 0 and pairs > 0
        z = sc.raw[0:3].T @ np.asarray(cam.R)[2] + np.asarray(cam.t)[2]
        near = np.nonzero(np.abs(z) < 6 * smax)[0]
        near_in_lists += int(np.isin(near, rast.tile_binning().prim_ids).any())
    assert near_in_lists >= 1


def test_config4_band(rast):
    """A 64x64 crop of a config-4 view (4M primitives, 3840x2160), binned in >= 3
    bands of tile rows (the memory path of config 4)."""
    sc = scenes.config_scene(4)
    cam0 = scenes.config_cameras(4)[0]
    cam = cam0.crop(cam0.width // 2 // 16 * 16 - 32, cam0.height // 2 // 16 * 16 - 32, 64, 64)
    st, bands, pairs = _crop_parity(rast, sc, cam, ref.Options(sh_degree=3, threads=0), band_limit_div=4)
    assert bands >= 3 and pairs > 100_000
