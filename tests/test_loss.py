"""Image losses of the training step: drk::loss with the D-SSIM term, drk::ssim,
drk::psnr (reference optimize.cpp:14-204).

CPU: the numpy restatement (oracle/loss_np.py) against the reference build.
GPU: drk_loss / drk_ssim / drk_psnr against the reference build on the same f32
images: the value within 1e-12 relative (only the mean reductions are
reordered), d_color equal to the reference's double rounded to f32 (the SSIM
taps, map and adjoint are evaluated in the reference's op order)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import loss_np, ref

CASES = [  # (H, W, C, dssim_weight)
    (40, 53, 3, 0.2), (11, 11, 3, 0.2), (12, 30, 1, 0.5), (64, 48, 3, 1.0), (37, 29, 3, 0.0), (10, 40, 3, 0.2),
    (5, 3, 3, 0.2),
]


def images(H, W, C, seed):
    rng = np.random.default_rng(seed)
    r = rng.uniform(0, 1, (H, W, C)).astype(np.float32)
    t = rng.uniform(0, 1, (H, W, C)).astype(np.float32)
    r[::7, ::5] = t[::7, ::5]  # exact ties: sign(0) = 0 (optimize.cpp:184)
    return r, t


needs_ref = pytest.mark.skipif(not ref.available(), reason="reference build (oracle/_ref) missing")


@needs_ref
@pytest.mark.parametrize("H,W,C,w", CASES)
def test_restatement_matches_reference(H, W, C, w):
    r, t = images(H, W, C, H * 1000 + W)
    r64, t64 = r.astype(np.float64), t.astype(np.float64)
    v_ref, d_ref = ref.loss(r64, t64, w)
    v, d = loss_np.loss(r64, t64, w)
    assert abs(v - v_ref) <= 1e-13 * max(1.0, abs(v_ref))
    assert np.abs(d - d_ref).max() <= 1e-13 * max(np.abs(d_ref).max(), 1e-30)
    assert loss_np.psnr(r64, t64) == pytest.approx(ref.psnr(r64, t64), rel=1e-13)
    if H >= 11 and W >= 11:
        assert loss_np.ssim(r64, t64) == pytest.approx(ref.ssim(r64, t64), rel=1e-12, abs=1e-15)


@needs_ref
def test_reference_edge_cases():
    r, _ = images(16, 16, 3, 1)
    r64 = r.astype(np.float64)
    assert ref.psnr(r64, r64) == 100.0 and loss_np.psnr(r64, r64) == 100.0  # mse < 1e-10
    assert ref.ssim(r64, r64) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(RuntimeError):  # DimensionMismatchError: image smaller than the window
        ref.ssim(r64[:10], r64[:10])


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("H,W,C,w", CASES + [(720, 1280, 3, 0.2)])
def test_device_loss_matches_reference(rast, H, W, C, w):
    import torch
    r, t = images(H, W, C, H * 1000 + W)
    v_ref, d_ref = ref.loss(r.astype(np.float64), t.astype(np.float64), w)
    shape = (H, W, C) if C > 1 else (H, W, 1)
    out, d = rast.loss(torch.from_numpy(r.reshape(shape)).cuda(), torch.from_numpy(t.reshape(shape)).cuda(), w)
    out = out.cpu().numpy()
    d = d.cpu().numpy().reshape(H, W, C)
    assert abs(out[0] - v_ref) <= 1e-12 * max(1.0, abs(v_ref)), (out, v_ref)
    # taps / SSIM map / adjoint in the reference's op order: identical doubles, rounded once to f32
    assert np.array_equal(d, d_ref.astype(np.float32)), np.abs(d - d_ref).max()
    if H >= 11 and W >= 11 and w > 0:  # loss() evaluates SSIM only when it is weighted (optimize.cpp:173-175)
        assert out[2] == pytest.approx(ref.ssim(r.astype(np.float64), t.astype(np.float64)), rel=1e-12, abs=1e-15)


@pytest.mark.gpu
@needs_ref
def test_device_ssim_psnr(rast):
    import torch

    from paper_2412_11752_b200.api import DimensionMismatchError
    for (H, W) in ((16, 16), (45, 80), (1080, 1920)):
        a, b = images(H, W, 3, H + W)
        A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        assert float(rast.ssim(A, B)) == pytest.approx(ref.ssim(a64, b64), rel=1e-12, abs=1e-15)
        assert float(rast.psnr(A, B)) == pytest.approx(ref.psnr(a64, b64), rel=1e-11)  # reordered mse sum
        assert float(rast.psnr(A, A)) == 100.0
        assert float(rast.ssim(A, A)) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(DimensionMismatchError):
        rast.ssim(A[:10], B[:10])
