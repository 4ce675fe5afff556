"""Seeded synthetic DRK scenes and cameras for BASELINE.json configs 0-4.

The reference's own tests draw from ``std::mt19937_64`` through
``std::uniform_real_distribution``, whose output is implementation-defined, so
the generator here uses numpy's PCG64 *raw* 64-bit stream with explicit
transforms (u = (x >> 11) * 2^-53; Box-Muller normals) — portable and stable
across numpy versions.  Every value is rounded to float32 and the same arrays
feed the oracle, the reference build and the CUDA path.

Field recipe (BASELINE.json configs):
  * centre: C0 U[-1,1]^3; C1-C4 a 32-cluster Gaussian mixture, cluster centres
    U[-2,2]^3, sigma 0.15.
  * quat_raw = normalize(N(0,1)^4); scale_raw = log sigma ~ U(-3,-1).
  * angles: 8 gaps = spacings of 7 sorted U(0,1) (plus the endpoints), mapped to
    raws with the inverse of ``angle_activation`` (reference mesh.cpp:101-123
    restated; nearest representable when the gap ratio exceeds 7).
  * eta_raw, tau_raw = logit(U(0,1)) (BASELINE's "remap knots" map to the single
    sharpness tau, core.cpp:142); opacity_raw ~ N(0,1).
  * colour: DC coefficient so that rgb = U(0,1) (geometry.cpp:130-132
    convention); SH degree 3 higher coefficients ~ N(0, 0.2^2).
  * camera: hfov 50 deg, fx = fy = W / (2 tan 25 deg), principal point at the
    image centre, looking at the origin from (0,0,-4) (C0-C2) or from a seeded
    orbit of radius U(3,5) (C3/C4).  "near 0.01" has no slot in the reference
    Camera and is ignored.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SH_C0 = 0.28209479177387814


def sh_terms(degree: int) -> int:
    return (degree + 1) * (degree + 1)


def scalar_count(k: int, terms: int) -> int:
    """Reference types.hpp:74."""
    return 3 + 4 + 2 * k + 3 + 3 * terms


class Rng:
    """Portable PCG64 raw stream with explicit float transforms."""

    def __init__(self, seed: int):
        self._bg = np.random.PCG64(seed)

    def uniform(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        x = self._bg.random_raw(n).astype(np.uint64)
        u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * u

    def normal(self, n: int, std: float = 1.0) -> np.ndarray:
        m = (n + 1) // 2
        u1 = self.uniform(m)
        u2 = self.uniform(m)
        r = np.sqrt(-2.0 * np.log1p(-u1))
        z = np.concatenate([r * np.cos(2 * math.pi * u2), r * np.sin(2 * math.pi * u2)])
        return std * z[:n]

    def integers(self, n: int, hi: int) -> np.ndarray:
        x = self._bg.random_raw(n).astype(np.uint64)
        return (x % np.uint64(hi)).astype(np.int64)


def _logit(p: np.ndarray) -> np.ndarray:
    p = np.clip(p, 1e-12, 1 - 1e-12)
    return np.log(p / (1.0 - p))


def angles_to_raw(gaps: np.ndarray) -> np.ndarray:
    """Inverse of angle_activation for rows of gap ratios summing to 1.

    Restates reference mesh.cpp:101-123: scale the ratios by sqrt(d_lo*d_hi)
    when representable (ratio spread < 7 for K=8), else by the midpoint, clamp
    the sigmoid to [1e-9, 1-1e-9] and take the logit.
    """
    k = gaps.shape[1]
    residual = 1.0 / (k - 2)
    rmin = gaps.min(axis=1, keepdims=True)
    rmax = gaps.max(axis=1, keepdims=True)
    d_lo = residual / rmin
    d_hi = (1.0 + residual) / rmax
    exact = d_lo < d_hi
    total = np.where(exact, np.sqrt(d_lo * d_hi), 0.5 * (d_lo + d_hi))
    s = np.clip(gaps * total - residual, 1e-9, 1.0 - 1e-9)
    return np.log(s / (1.0 - s))


@dataclass
class Scene:
    """Raw DRK parameters in the ABI layout: scalar-major SoA, raw[s, i]."""

    raw: np.ndarray  # float64 [scalar_count, n], values exactly representable in f32
    k: int
    sh_degree: int

    @property
    def n(self) -> int:
        return self.raw.shape[1]

    @property
    def terms(self) -> int:
        return sh_terms(self.sh_degree)

    def f32(self) -> np.ndarray:
        return np.ascontiguousarray(self.raw.astype(np.float32))


@dataclass
class Camera:
    """Mirror of drk::Camera (reference geometry.hpp:9-19)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray = field(default_factory=lambda: np.eye(3))  # world->cam, row-major
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def position(self) -> np.ndarray:
        return -self.R.T @ self.t

    def crop(self, x0: int, y0: int, w: int, h: int) -> "Camera":
        """Sub-window camera (SURVEY.md §8(d) crops); x0, y0 multiples of 16."""
        return Camera(self.fx, self.fy, self.cx - x0, self.cy - y0, w, h, self.R.copy(), self.t.copy())


def look_at_camera(width: int, height: int, pos, target=(0.0, 0.0, 0.0), hfov_deg: float = 50.0) -> Camera:
    pos = np.asarray(pos, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - pos
    f /= np.linalg.norm(f)
    up = np.array([0.0, -1.0, 0.0])
    x = np.cross(f, up)
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f])
    t = -R @ pos
    fx = width / (2.0 * math.tan(math.radians(hfov_deg) / 2.0))
    return Camera(fx, fx, width / 2.0, height / 2.0, width, height, R, t)


def simple_camera(size: int = 64, focal: float = 64.0) -> Camera:
    """Reference tests/test_util.hpp:38-44."""
    return Camera(focal, focal, size / 2.0, size / 2.0, size, size, np.eye(3), np.zeros(3))


def random_scene(n: int, seed: int, k: int = 8, sh_degree: int = 0, clusters: int = 0,
                 extent: float = 1.0, cluster_sigma: float = 0.15) -> Scene:
    rng = Rng(seed)
    terms = sh_terms(sh_degree)
    S = scalar_count(k, terms)
    raw = np.zeros((S, n), dtype=np.float64)
    if clusters > 0:
        cc = rng.uniform(3 * clusters, -2.0, 2.0).reshape(clusters, 3)
        lab = rng.integers(n, clusters)
        ctr = cc[lab] + rng.normal(3 * n, cluster_sigma).reshape(n, 3)
    else:
        ctr = rng.uniform(3 * n, -extent, extent).reshape(n, 3)
    raw[0:3] = ctr.T
    q = rng.normal(4 * n).reshape(n, 4)
    q /= np.maximum(np.linalg.norm(q, axis=1, keepdims=True), 1e-12)
    raw[3:7] = q.T
    raw[7:7 + k] = rng.uniform(k * n, -3.0, -1.0).reshape(k, n)
    cuts = np.sort(rng.uniform((k - 1) * n).reshape(n, k - 1), axis=1)
    edges = np.concatenate([np.zeros((n, 1)), cuts, np.ones((n, 1))], axis=1)
    gaps = np.maximum(np.diff(edges, axis=1), 1e-6)
    gaps /= gaps.sum(axis=1, keepdims=True)
    raw[7 + k:7 + 2 * k] = angles_to_raw(gaps).T
    o = 7 + 2 * k
    raw[o] = _logit(rng.uniform(n))        # eta
    raw[o + 1] = _logit(rng.uniform(n))    # tau
    raw[o + 2] = rng.normal(n)             # opacity
    sh = np.zeros((n, terms, 3))
    sh[:, 0, :] = (rng.uniform(3 * n).reshape(n, 3) - 0.5) / SH_C0
    if terms > 1:
        sh[:, 1:, :] = rng.normal(n * (terms - 1) * 3, 0.2).reshape(n, terms - 1, 3)
    raw[o + 3:] = sh.reshape(n, terms * 3).T
    raw = raw.astype(np.float32).astype(np.float64)
    return Scene(raw=raw, k=k, sh_degree=sh_degree)


# BASELINE.json configs (index = config number).
CONFIGS = {
    0: dict(n=1_000, width=256, height=256, sh_degree=0, clusters=0, views=1, backward=False),
    1: dict(n=100_000, width=1920, height=1080, sh_degree=3, clusters=32, views=1, backward=False),
    2: dict(n=300_000, width=1280, height=720, sh_degree=3, clusters=32, views=1, backward=True),
    3: dict(n=1_000_000, width=1920, height=1080, sh_degree=3, clusters=32, views=64, backward=False),
    4: dict(n=4_000_000, width=3840, height=2160, sh_degree=3, clusters=32, views=8, backward=True),
}


def orbit_cameras(views: int, width: int, height: int, seed: int) -> list[Camera]:
    rng = Rng(seed ^ 0x5EED)
    cams = []
    while len(cams) < views:
        d = rng.normal(3)
        d /= np.linalg.norm(d)
        if abs(d[1]) > 0.999:  # parallel to the up vector
            continue
        r = float(rng.uniform(1, 3.0, 5.0)[0])
        cams.append(look_at_camera(width, height, r * d))
    return cams


def config_scene(cfg: int, seed: int = 0, n: int | None = None) -> Scene:
    c = CONFIGS[cfg]
    return random_scene(n or c["n"], seed=seed * 1000 + cfg, sh_degree=c["sh_degree"],
                        clusters=c["clusters"])


def config_cameras(cfg: int, seed: int = 0) -> list[Camera]:
    c = CONFIGS[cfg]
    if c["views"] == 1:
        return [look_at_camera(c["width"], c["height"], (0.0, 0.0, -4.0))]
    return orbit_cameras(c["views"], c["width"], c["height"], seed * 1000 + cfg)


def config_target(cfg: int, cam: Camera, seed: int = 0, view: int = 0) -> np.ndarray:
    """Seeded U(0,1) H x W x 3 target image (configs 2 and 4)."""
    rng = Rng(seed * 1000 + cfg + 7919 * (view + 1))
    return rng.uniform(cam.height * cam.width * 3).reshape(cam.height, cam.width, 3)
