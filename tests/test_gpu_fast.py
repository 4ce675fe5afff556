"""The fp32 interval forward kernel (drk_raster_fast.cu) against the legacy fp64-depth
kernel and against its own fp64 re-evaluation.

- Every fp32 alpha of a frame is re-evaluated in fp64 (drk_set_validation): the
  observed error must stay inside the bound that gates the fp64 fallbacks.
- Full BASELINE frames (configs 1 and 2, where the CPU oracle is too slow): both
  kernels make the reference's discrete decisions, so their framebuffers agree
  within the parity tolerance and their work counters agree.
- Backward after the fast forward: gradients match the oracle (termination is
  taken from the forward's per-pixel composite count).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

from oracle import port
from paper_2412_11752_b200 import scenes
from tests.helpers import api_options, opt_for, rel_l2, small_scene

pytestmark = pytest.mark.gpu


def _render(rast, sc, cam, opt, kernel):
    fb = rast.render(sc.f32(), cam, dataclasses.replace(opt, raster_kernel=kernel))
    return fb, rast.stats()


@pytest.mark.parametrize("cfg,crop", [(0, None), (1, 256), (2, 192), (1, None), (2, None)])
def test_fast_alpha_bound_in_situ(rast, cfg, crop):
    sc = scenes.config_scene(cfg)
    cam = scenes.config_cameras(cfg)[0]
    if crop:
        cam = cam.crop((cam.width // 2 - crop // 2) // 16 * 16, (cam.height // 2 - crop // 2) // 16 * 16, crop, crop)
    opt = api_options(opt_for(scenes.CONFIGS[cfg]["sh_degree"]))
    rast.set_validation(True)
    try:
        rast.render(sc.f32(), cam, opt)
        ratio, max_abs = rast.validation()
    finally:
        rast.set_validation(False)
    st = rast.stats()
    assert st["popped"] > 0
    assert ratio < 1.0, (ratio, max_abs)


@pytest.mark.parametrize("cfg", [1, 2])
def test_fast_matches_legacy_full_frame(rast, cfg):
    sc = scenes.config_scene(cfg)
    cam = scenes.config_cameras(cfg)[0]
    opt = api_options(opt_for(3))
    fb_l, st_l = _render(rast, sc, cam, opt, 1)
    legacy = {f: getattr(fb_l, f).clone() for f in ("color", "depth", "normal", "alpha")}
    fb_f, st_f = _render(rast, sc, cam, opt, 0)
    for f, v in legacy.items():
        err = float((getattr(fb_f, f) - v).abs().max())
        assert err <= 1e-4, (f, err)
    # identical decisions: the same entries stream, pop and composite (up to the
    # pixels either kernel hands to the fp64 re-render)
    for k in ("streamed", "popped", "composited"):
        assert abs(st_f[k] - st_l[k]) <= 1e-4 * st_l[k], (k, st_f[k], st_l[k])
    assert st_f["fp64_pixels"] <= 0.02 * cam.width * cam.height


def test_fast_small_scenes_vs_oracle(rast):
    for seed in range(4):
        sc, cam = small_scene(seed=20 + seed, n=120, sh_degree=3, clusters=3)
        o = opt_for(3, background=(0.1, 0.7, 0.3))
        fb = rast.render(sc.f32(), cam, api_options(o))
        orc = port.render(sc, cam, o)
        for f in ("color", "depth", "normal", "alpha"):
            err = float(np.abs(getattr(fb, f).cpu().numpy().astype(np.float64) - orc[f]).max())
            assert err <= 1e-4, (seed, f, err)


def test_fast_backward_termination_from_forward(rast):
    from paper_2412_11752_b200.api import FrameGrad
    sc, cam = small_scene(seed=31, n=150, sh_degree=3, clusters=2)
    o = opt_for(3)
    rast.render(sc.f32(), cam, api_options(o))
    rng = np.random.default_rng(3)
    dc = rng.uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)
    g = rast.backward_render(sc.f32(), FrameGrad(d_color=torch.from_numpy(dc)))
    og = port.backward(sc, cam, o, dc, None, None, None)
    assert rel_l2(g.raw.cpu().numpy(), og["raw"]) <= 1e-3
    np.testing.assert_array_equal(g.touched.cpu().numpy(), og["touched"])


def test_legacy_backward_kernel_parity(rast):
    """The legacy warp-reduced backward (raster_kernel=5) against the oracle."""
    import dataclasses
    from paper_2412_11752_b200.api import FrameGrad
    sc, cam = small_scene(seed=41, n=150, sh_degree=3, clusters=2)
    o = opt_for(3)
    opt = dataclasses.replace(api_options(o), raster_kernel=5)
    rast.render(sc.f32(), cam, opt)
    rng = np.random.default_rng(5)
    dc = rng.uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)
    dd = rng.uniform(-0.1, 0.1, (cam.height, cam.width)).astype(np.float32)
    g = rast.backward_render(sc.f32(), FrameGrad(d_color=torch.from_numpy(dc), d_depth=torch.from_numpy(dd)))
    og = port.backward(sc, cam, o, dc, dd, None, None)
    assert rel_l2(g.raw.cpu().numpy(), og["raw"]) <= 1e-3
    np.testing.assert_array_equal(g.touched.cpu().numpy(), og["touched"])


def test_banded_binning_matches_single_band(rast):
    """Bands of tile rows (config 4's memory path) give the same frame as one band,
    and the banded backward the same gradients (up to atomic summation order)."""
    from paper_2412_11752_b200.api import FrameGrad
    sc = scenes.config_scene(2, n=30000)
    cam = scenes.config_cameras(2)[0].crop(0, 0, 320, 256)
    opt = api_options(opt_for(3))
    rng = np.random.default_rng(9)
    dc = torch.from_numpy(rng.uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32))
    fb1 = rast.render(sc.f32(), cam, opt)
    ref = {f: getattr(fb1, f).clone() for f in ("color", "depth", "normal", "alpha")}
    g1 = rast.backward_render(sc.f32(), FrameGrad(d_color=dc)).raw.clone()
    pairs = rast.stats()["pairs"]
    assert rast.bands() == 1
    try:
        rast.set_band_limit(max(1, pairs // 4))
        fb4 = rast.render(sc.f32(), cam, opt)
        assert rast.bands() >= 3
        for f, v in ref.items():
            assert torch.equal(getattr(fb4, f), v), f
        assert rast.stats()["pairs"] == pairs
        g4 = rast.backward_render(sc.f32(), FrameGrad(d_color=dc)).raw
        assert rel_l2(g4.cpu().numpy(), g1.cpu().numpy()) <= 1e-5
    finally:
        rast.set_band_limit(0)


@pytest.mark.parametrize("cfg", [0, 1])
def test_forward_host_matches_device(rast, cfg):
    """drk_forward_host: page-locked outputs written in place by the kernels (zero-copy,
    the fp64 re-render included), pageable ones copied out: bitwise the device frame."""
    sc = scenes.config_scene(cfg)
    cam = scenes.config_cameras(cfg)[0]
    opt = api_options(opt_for(scenes.CONFIGS[cfg]["sh_degree"]))
    fb = rast.render(sc.f32(), cam, opt)
    dev = {f: getattr(fb, f).cpu().numpy().copy() for f in ("color", "depth", "normal", "alpha")}
    flagged = rast.stats()["fp64_pixels"]
    if cfg == 1:
        assert flagged > 0  # the fp64 re-render writes host memory too
    for pinned in (False, True):
        if pinned:
            outs = {f: torch.empty(v.shape, dtype=torch.float32).pin_memory() for f, v in dev.items()}
            raw = torch.from_numpy(sc.f32()).pin_memory()
            rast.render_host_ptrs(raw, outs, cam, opt)
            torch.cuda.synchronize()
            out = {f: t.numpy() for f, t in outs.items()}
        else:
            out = rast.render_host(sc.f32(), cam, opt)
        assert rast.stats()["fp64_pixels"] == flagged
        for f, v in dev.items():
            np.testing.assert_array_equal(out[f], v, err_msg=f"{f} pinned={pinned}")


@pytest.mark.gpu
def test_multiview_renderer_matches_single_context(rast):
    """Two in-flight contexts on their own streams / host threads render each view
    bit-identically to one context rendering the views in turn."""
    import torch

    from paper_2412_11752_b200 import scenes
    from paper_2412_11752_b200.api import RenderOptions
    from paper_2412_11752_b200.parallel import MultiViewRenderer
    sc = scenes.random_scene(3000, seed=17, sh_degree=3, clusters=8)
    raw = torch.from_numpy(sc.f32()).cuda()
    cams = [scenes.look_at_camera(160, 96, (3.5 * np.cos(a), 0.3, 3.5 * np.sin(a))) for a in np.linspace(0, 5, 7)]
    opt = RenderOptions(sh_degree=3)
    want = [rast.render(raw, c, opt).color.clone() for c in cams]
    mv = MultiViewRenderer(inflight=2)
    got = mv.render(raw, cams, opt)
    torch.cuda.synchronize()
    for g, w in zip(got, want):
        assert torch.equal(g.color, w)
    mv.close()


@pytest.mark.gpu
def test_half_tile_ctas_bit_identical(rast):
    """The fast forward's half-tile CTAs (8 x 16 pixels, chosen for long tile lists)
    give the same framebuffers and per-pixel composite counts as whole-tile CTAs,
    through the host-buffer entry too."""
    from paper_2412_11752_b200 import scenes
    from paper_2412_11752_b200.api import RenderOptions
    sc = scenes.random_scene(20000, seed=29, sh_degree=3, clusters=12)
    cam = scenes.look_at_camera(300, 170, (0.3, 0.2, -3.2))
    raw = torch.from_numpy(sc.f32()).cuda()
    out = {}
    from paper_2412_11752_b200.api import FrameGrad
    dcol = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32))
    grads = {}
    for rk in (7, 6):
        fb = rast.render(raw, cam, RenderOptions(sh_degree=3, raster_kernel=rk))
        out[rk] = [t.clone() for t in (fb.color, fb.depth, fb.normal, fb.alpha)]
        st = rast.stats()
        out[rk].append(st["streamed"]), out[rk].append(st["composited"])
        grads[rk] = rast.backward_render(raw, FrameGrad(d_color=dcol.cuda())).raw.clone()
        host = rast.render_host(sc.f32(), cam, RenderOptions(sh_degree=3, raster_kernel=rk))
        assert np.array_equal(host["color"], out[rk][0].cpu().numpy())
    for a, b in zip(out[7][:4], out[6][:4]):
        assert torch.equal(a, b)
    assert out[7][4:] == out[6][4:]
    # backward with the same CTA shape: equal up to the order of the f32 atomics
    rel = float((grads[7] - grads[6]).norm() / grads[7].norm())
    assert rel < 1e-5, rel


@pytest.mark.gpu
def test_counters_off_same_frame(rast):
    """drk_set_counters(0) launches the counter-free fast kernel: same frame, zero work counts."""
    from paper_2412_11752_b200.api import RenderOptions
    sc = scenes.random_scene(5000, seed=31, sh_degree=3, clusters=6)
    cam = scenes.look_at_camera(160, 112, (0.2, -0.3, -3.4))
    raw = torch.from_numpy(sc.f32()).cuda()
    a = rast.render(raw, cam, RenderOptions(sh_degree=3)).color.clone()
    assert rast.stats()["popped"] > 0
    try:
        rast.set_counters(False)
        b = rast.render(raw, cam, RenderOptions(sh_degree=3)).color
        assert rast.stats()["popped"] == 0
    finally:
        rast.set_counters(True)
    assert torch.equal(a, b)
