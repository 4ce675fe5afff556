"""Seeded synthetic inputs (BASELINE.json distributions) and the angle inverse."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2412_11752_b200 import scenes


def test_deterministic_and_f32_representable():
    a = scenes.config_scene(0)
    b = scenes.config_scene(0)
    assert np.array_equal(a.raw, b.raw)
    assert np.array_equal(a.raw, a.raw.astype(np.float32).astype(np.float64))
    assert a.raw.shape == (scenes.scalar_count(8, 1), 1000)
    c = scenes.config_scene(1, n=2000)
    assert c.raw.shape == (scenes.scalar_count(8, 16), 2000)


def test_distributions_config0():
    sc = scenes.config_scene(0)
    k = sc.k
    assert np.all(np.abs(sc.raw[0:3]) <= 1.0)
    q = sc.raw[3:7]
    assert np.allclose(np.linalg.norm(q, axis=0), 1.0, atol=1e-6)
    assert np.all((sc.raw[7:7 + k] >= -3.0) & (sc.raw[7:7 + k] <= -1.0))
    rgb = 0.5 + scenes.SH_C0 * sc.raw[10 + 2 * k:13 + 2 * k]
    assert np.all((rgb > -1e-6) & (rgb < 1 + 1e-6))


def test_cameras():
    cam = scenes.config_cameras(1)[0]
    assert (cam.width, cam.height) == (1920, 1080)
    assert np.allclose(cam.R @ cam.R.T, np.eye(3), atol=1e-12)
    assert np.allclose(cam.position(), [0, 0, -4])
    orbit = scenes.config_cameras(3)
    assert len(orbit) == 64
    r = np.array([np.linalg.norm(c.position()) for c in orbit])
    assert np.all((r >= 3 - 1e-9) & (r <= 5 + 1e-9))
    crop = cam.crop(16, 32, 64, 48)
    assert crop.cx == cam.cx - 16 and crop.cy == cam.cy - 32


def test_angles_inverse_roundtrip():
    oracle = pytest.importorskip("oracle.port")
    if not oracle.available():
        pytest.skip("oracle not built")
    sc = scenes.random_scene(200, seed=4)
    th = oracle.activate(sc)["angles"]
    gaps = np.diff(np.concatenate([np.zeros((200, 1)), th], axis=1), axis=1)
    assert np.all(gaps > 0) and np.all(gaps < np.pi)
    assert np.allclose(th[:, -1], 2 * np.pi)
