"""numpy restatement of the reference's image losses (optimize.cpp:14-204):
ssim_kernel, correlate_valid, scatter_full, ssim_channel, psnr, ssim, loss.

TEST INFRASTRUCTURE ONLY (checker of paper_2412_11752_b200/csrc/drk_loss.cu);
pinned against the reference build (oracle/ref.py: ref_loss / ref_ssim /
ref_psnr) in tests/test_loss.py.  Images are float64 [H, W, C]."""
from __future__ import annotations

import numpy as np

WIN, SIGMA = 11, 1.5            # optimize.cpp:14-15
C1, C2 = 0.01 * 0.01, 0.03 * 0.03  # optimize.cpp:16-17


def ssim_kernel():
    """optimize.cpp:23-33"""
    d = np.arange(WIN) - (WIN - 1) / 2.0
    g = np.exp(-d * d / (2.0 * SIGMA * SIGMA))
    s = 0.0
    for v in g:  # sequential sum like the reference
        s += v
    return g / s


def correlate_valid(p, g):
    """optimize.cpp:45-60 (taps summed i ascending)"""
    H, W = p.shape
    vw, vh = W - WIN + 1, H - WIN + 1
    tmp = np.zeros((H, vw))
    for i in range(WIN):
        tmp = tmp + g[i] * p[:, i:i + vw]
    out = np.zeros((vh, vw))
    for i in range(WIN):
        out = out + g[i] * tmp[i:i + vh, :]
    return out


def scatter_full(f, W, H, g):
    """optimize.cpp:63-80: adjoint of correlate_valid"""
    vh, vw = f.shape
    tmp = np.zeros((vh, W))
    for i in range(WIN):
        tmp[:, i:i + vw] += g[i] * f
    out = np.zeros((H, W))
    for i in range(WIN):
        out[i:i + vh, :] += g[i] * tmp
    return out


def ssim_channel(x, y, with_grad):
    """optimize.cpp:97-143 -> (mean, d_x or None)"""
    g = ssim_kernel()
    mx, my = correlate_valid(x, g), correlate_valid(y, g)
    mxx, myy, mxy = correlate_valid(x * x, g), correlate_valid(y * y, g), correlate_valid(x * y, g)
    ux, uy = mx, my
    vx, vy, vxy = mxx - ux * ux, myy - uy * uy, mxy - ux * uy
    a1, a2 = 2 * ux * uy + C1, 2 * vxy + C2
    b1, b2 = ux * ux + uy * uy + C1, vx + vy + C2
    s = (a1 * a2) / (b1 * b2)
    inv_n = 1.0 / s.size
    mean = s.sum() * inv_n
    if not with_grad:
        return mean, None
    ds_dvx = -s / b2
    ds_dvxy = 2 * a1 / (b1 * b2)
    ds_dux = 2 * uy * a2 / (b1 * b2) - 2 * ux * s / b1 - 2 * ux * ds_dvx - uy * ds_dvxy
    H, W = x.shape
    s1, s2, s3 = (scatter_full(f, W, H, g) for f in (ds_dux, ds_dvx, ds_dvxy))
    return mean, inv_n * (s1 + 2.0 * x * s2 + y * s3)


def psnr(a, b):
    """optimize.cpp:145-155"""
    mse = float(np.mean((a - b) ** 2))
    return 100.0 if mse < 1e-10 else -10.0 * np.log10(mse)


def ssim(a, b):
    """optimize.cpp:157-166"""
    H, W, C = a.shape
    if W < WIN or H < WIN:
        raise ValueError("image smaller than the SSIM window")
    return sum(ssim_channel(a[..., c], b[..., c], False)[0] for c in range(C)) / C


def loss(r, t, dssim_weight):
    """optimize.cpp:171-204 -> (value, d_color)"""
    H, W, C = r.shape
    use = dssim_weight > 0 and W >= WIN and H >= WIN
    w = dssim_weight if use else 0.0
    inv_n = 1.0 / r.size
    d = r - t
    dcol = (1.0 - w) * inv_n * np.sign(d)
    value = (1.0 - w) * (np.abs(d).sum() * inv_n)
    if use:
        ms = 0.0
        for c in range(C):
            m, dx = ssim_channel(r[..., c], t[..., c], True)
            ms += m
            dcol[..., c] += (-w / C) * dx
        value += w * (1.0 - ms / C)
    return value, dcol
