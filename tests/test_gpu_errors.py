"""Error statuses of the GPU path against the reference's exceptions
(errors.hpp:9-97; SURVEY.md §8(b) "Errors"): NonFinite and DegenerateQuaternion
from activate (core.cpp:134, geometry.cpp:23), DegenerateBasis from the kernel
evaluation (core.cpp:191: |det [e_lo e_hi]| < 1e-12), ReplayMismatch from
backward_render (grad.cpp:311-314).  The same inputs make the reference build
(oracle/_ref) raise the same class (its status codes 2 / 3 / 4)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ref
from paper_2412_11752_b200 import _lib, scenes
from paper_2412_11752_b200.api import FrameGrad, Rasterizer, RenderOptions

pytestmark = pytest.mark.gpu


def _one(center, scale_raw=-2.0, quat=(1.0, 0.0, 0.0, 0.0)):
    sc = scenes.random_scene(1, seed=3, sh_degree=0)
    sc.raw[0:3, 0] = center
    sc.raw[3:7, 0] = quat
    sc.raw[7:15, 0] = scale_raw
    sc.raw[7 + 2 * 8 + 2, 0] = 3.0  # opacity sigmoid(3)
    sc.raw = sc.raw.astype(np.float32).astype(np.float64)
    return sc


def _ref_status(sc, cam):
    try:
        ref.render(sc, cam, ref.Options(sh_degree=0))
    except RuntimeError as e:
        return int(str(e).split()[2].rstrip(":"))
    return 0


@pytest.mark.parametrize("case,status,exc", [
    ("nonfinite", 2, _lib.NonFiniteError),
    ("quaternion", 3, _lib.DegenerateQuaternionError),
    ("basis", 4, _lib.DegenerateBasisError),
])
def test_error_statuses_match_reference(case, status, exc):
    cam = scenes.simple_camera(64, 64)
    # the ray of pixel (32, 32) meets z = 1 at (2^-7, 2^-7)
    c = [2.0 ** -7 + 3e-7, 2.0 ** -7 + 2e-7, 1.0]
    if case == "nonfinite":
        sc = _one(c)
        sc.raw[9, 0] = np.nan
    elif case == "quaternion":
        sc = _one(c, quat=(0.0, 0.0, 0.0, 0.0))
    else:
        # scales 1e-6: det = s_lo s_hi sin(gap) < 1e-12 for every bracket; the
        # pixel's ray passes 0.36 s from the centre, so its alpha is evaluated
        sc = _one(c, scale_raw=float(np.log(1e-6)))
    assert _ref_status(sc, cam) == status
    r = Rasterizer(0)
    try:
        with pytest.raises(exc):
            r.render(sc.f32(), cam, RenderOptions(sh_degree=0))
        # the context stays usable after an error
        ok = scenes.random_scene(20, seed=1, sh_degree=0)
        fb = r.render(ok.f32(), scenes.look_at_camera(32, 32, (0.0, 0.0, -3.0)), RenderOptions(sh_degree=0))
        assert torch.isfinite(fb.color).all()
    finally:
        r.close()


def test_replay_mismatch():
    """backward_render without the forward it replays (grad.cpp:311-314)."""
    r = Rasterizer(0)
    try:
        sc = scenes.random_scene(10, seed=2, sh_degree=0)
        with pytest.raises(_lib.ReplayMismatchError):
            r.backward_render(sc.f32(), FrameGrad(d_color=torch.zeros(8, 8, 3)))
        # the C-ABI itself reports it (the Python check above is only a shortcut)
        import ctypes as C
        st = _lib.lib().drk_backward(r._h, None, C.byref(_lib.FrameGrad_()), None, None, None, None, 0, 0)
        assert st == _lib.ReplayMismatchError.status
    finally:
        r.close()


@pytest.mark.parametrize("bad", ["nonfinite", "quaternion"])
def test_host_pipeline_errors(bad):
    """drk_forward_host on page-locked parameters of a large scene (the chunked
    upload that overlaps activation and K1) reports the activation's errors
    after the fact, like the device path, and leaves the context usable."""
    sc = scenes.random_scene(70000, seed=5, sh_degree=0)
    raw = sc.f32().copy()
    if bad == "nonfinite":
        raw[9, 65000] = np.nan  # a primitive in the last chunk
    else:
        raw[3:7, 12345] = 0.0
    cam = scenes.look_at_camera(96, 64, (0.0, 0.0, -3.0))
    host = torch.from_numpy(raw).pin_memory()
    outs = {"color": torch.empty(cam.height, cam.width, 3, pin_memory=True),
            "depth": torch.empty(cam.height, cam.width, pin_memory=True),
            "normal": torch.empty(cam.height, cam.width, 3, pin_memory=True),
            "alpha": torch.empty(cam.height, cam.width, pin_memory=True)}
    exc = _lib.NonFiniteError if bad == "nonfinite" else _lib.DegenerateQuaternionError
    r = Rasterizer(0)
    try:
        with pytest.raises(exc):
            r.render_host_ptrs(host, outs, cam, RenderOptions(sh_degree=0))
        good = torch.from_numpy(sc.f32()).pin_memory()
        r.render_host_ptrs(good, outs, cam, RenderOptions(sh_degree=0))
        torch.cuda.synchronize()
        fb = r.render(sc.f32(), cam, RenderOptions(sh_degree=0))
        assert torch.equal(fb.color.cpu(), outs["color"])
    finally:
        r.close()
