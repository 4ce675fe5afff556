"""The C restatement oracle (oracle/drk_oracle.c) against the UNMODIFIED reference
build (oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile.ref):
bit-exact tile lists, framebuffers, replay records and gradients on seeded inputs.
CPU only."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import port, ref
from paper_2412_11752_b200 import scenes

pytestmark = pytest.mark.skipif(not (ref.available() and port.available()),
                                reason="oracle libraries not built (run __graft_entry__.build())")


def _same(a, b):
    return all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(a, b))


def _render_equal(sc, cam, opt, replay=True):
    a = ref.render(sc, cam, opt, replay=replay)
    b = port.render(sc, cam, opt, replay=replay)
    for f in ("color", "depth", "normal", "alpha"):
        assert np.array_equal(a[f], b[f]), f
    if replay:
        assert _same(a["replay"], b["replay"])
    return b


def test_config0_bit_exact():
    sc = scenes.config_scene(0)
    cam = scenes.config_cameras(0)[0]
    opt = ref.Options(sh_degree=0)
    assert _same(ref.bin_primitives(sc, cam, opt), port.bin_primitives(sc, cam, opt))
    out = _render_equal(sc, cam, opt)
    st = out["stats"]
    assert st["pairs"] == 19505 and st["composited"] > 0


@pytest.mark.parametrize("presort", [0, 1, 2])
@pytest.mark.parametrize("use_cache,exact", [(True, False), (False, False), (True, True)])
def test_modes_bit_exact(presort, use_cache, exact):
    sc = scenes.random_scene(60, seed=10 + presort, sh_degree=1)
    cam = scenes.look_at_camera(48, 40, (0.4, 0.2, -3.2))
    opt = ref.Options(sh_degree=1, presort=presort, use_cache=use_cache, exact_sort=exact,
                      background=(0.1, 0.7, 0.3))
    assert _same(ref.bin_primitives(sc, cam, opt), port.bin_primitives(sc, cam, opt))
    _render_equal(sc, cam, opt)


def test_k4_sh3_and_crop():
    sc = scenes.random_scene(90, seed=3, k=4, sh_degree=3, clusters=4)
    cam = scenes.look_at_camera(96, 64, (0.0, -0.5, -3.0)).crop(16, 16, 64, 32)
    for deg in (0, 2, 3):
        opt = ref.Options(sh_degree=deg)
        assert _same(ref.bin_primitives(sc, cam, opt), port.bin_primitives(sc, cam, opt))
        _render_equal(sc, cam, opt)


def test_edge_cases():
    # empty scene, primitives behind the camera, a camera inside the cloud (near clip)
    cam = scenes.simple_camera(32, 32)
    empty = scenes.random_scene(0, seed=1)
    out = _render_equal(empty, cam, ref.Options(sh_degree=0, background=(0.2, 0.4, 0.6)))
    assert np.allclose(out["color"], [0.2, 0.4, 0.6]) and not out["alpha"].any()
    behind = scenes.random_scene(25, seed=2)
    behind.raw[2] = -3.0
    off, ids, keys = port.bin_primitives(behind, cam, ref.Options(sh_degree=0))
    assert len(ids) == 0
    inside = scenes.random_scene(80, seed=5, sh_degree=0)
    cam_in = scenes.look_at_camera(40, 40, (0.05, 0.02, -0.3))
    opt = ref.Options(sh_degree=0)
    assert _same(ref.bin_primitives(inside, cam_in, opt), port.bin_primitives(inside, cam_in, opt))
    _render_equal(inside, cam_in, opt, replay=False)


def test_backward_bit_exact():
    sc = scenes.random_scene(30, seed=8, sh_degree=1)
    cam = scenes.look_at_camera(40, 32, (0.2, 0.1, -3.0))
    opt = ref.Options(sh_degree=1, background=(0.3, 0.5, 0.2))
    rng = np.random.default_rng(3)
    H, W = cam.height, cam.width
    args = (rng.uniform(-1, 1, (H, W, 3)), rng.uniform(-.1, .1, (H, W)), rng.uniform(-.1, .1, (H, W, 3)),
            rng.uniform(-.5, .5, (H, W)))
    a = ref.backward(sc, cam, opt, *args)
    b = port.backward(sc, cam, opt, *args)
    for f in ("raw", "d_center_world", "screen_grad", "touched"):
        assert np.array_equal(a[f], b[f]), f
    assert np.abs(a["raw"]).sum() > 0


def test_activation_loss_adam():
    sc = scenes.random_scene(40, seed=9, sh_degree=3)
    a, b = ref.activate(sc), port.activate(sc)
    for f in a:
        assert np.array_equal(a[f], b[f]), f
    rng = np.random.default_rng(1)
    r, t = rng.uniform(0, 1, (8, 9, 3)), rng.uniform(0, 1, (8, 9, 3))
    t[0, 0, 0] = r[0, 0, 0]
    va, da = ref.loss_l1(r, t)
    vb, db = port.loss_l1(r, t)
    assert va == vb and np.array_equal(da, db)
    pa, pb = sc.raw.copy(), sc.raw.copy()
    ma, va_, mb, vb_ = (np.zeros_like(sc.raw) for _ in range(4))
    sa = sb = 0
    for _ in range(3):
        g = rng.normal(0, 1, sc.raw.shape)
        sa = ref.adam_step(pa, g, ma, va_, 8, 16, sa, [1e-3, 2e-4, 1e-3, 5e-2, 2.5e-3], 100, 2.0)
        sb = port.adam_step(pb, g, mb, vb_, 8, 16, sb, [1e-3, 2e-4, 1e-3, 5e-2, 2.5e-3], 100, 2.0)
    assert sa == sb == 3 and np.array_equal(pa, pb) and np.array_equal(ma, mb) and np.array_equal(va_, vb_)


@pytest.mark.slow
def test_config1_crop_bit_exact():
    sc = scenes.config_scene(1)
    cam0 = scenes.config_cameras(1)[0]
    cam = cam0.crop(928, 512, 48, 48)
    opt = ref.Options(sh_degree=3)
    assert _same(ref.bin_primitives(sc, cam, opt), port.bin_primitives(sc, cam, opt))
    _render_equal(sc, cam, opt, replay=False)


@pytest.mark.parametrize("cfg,n,threads", [(0, None, 3), (1, 6000, 4)])
def test_reference_parallel_binning_is_exact(cfg, n, threads):
    """ref_bin_parallel (the reference bin_primitives on chunks of the primitives,
    merged with its own comparator) equals one reference bin_primitives call."""
    sc = scenes.config_scene(cfg, n=n)
    cam = scenes.config_cameras(cfg)[0]
    if cfg:
        cam = cam.crop(640, 320, 320, 256)
    opt = ref.Options(sh_degree=scenes.CONFIGS[cfg]["sh_degree"])
    a = ref.bin_primitives(sc, cam, opt)
    b = ref.bin_primitives_parallel(sc, cam, opt, threads=threads)
    assert len(a[1]) > 1000
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
