"""DRKSCENE v1 scene files (reference io.cpp:40-97).

CPU: the numpy restatement (oracle/scene_io.py) against the unmodified
reference save_scene / load_scene (oracle/_ref/libdrk_refio.so) and the golden
files it wrote (tests/golden/make_golden_scenes.py); the C-ABI header checks
(drk_scene_read_header, host-only) against both on malformed files — the
reference suite's cases (test_io.cpp:65-94) and more.
GPU: drk_scene_load / drk_scene_save (device transpose) bit-exact against the
golden files and the restatement, up to config-1 size."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import scene_io

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ("k8_sh2", "k5_sh0", "k8_sh3_empty")
HEADERS = {"k8_sh2": (8, 2, 100), "k5_sh0": (5, 0, 37), "k8_sh3_empty": (8, 3, 0)}


def golden_path(name):
    return os.path.join(GOLDEN, f"scene_{name}.drk")


def golden_inputs():
    return dict(np.load(os.path.join(GOLDEN, "scene_inputs.npz")))


def malformed_files(tmp):
    """(name, path, expected_k): truncated payload, K mismatch, bad magic
    (test_io.cpp:65-94) plus header variants the reference parses by istream."""
    good = open(golden_path("k8_sh2"), "rb").read()
    body = good[good.index(b"\n") + 1:]
    rec = 4 * scene_io.scalar_count(8, 2)
    cases = {
        "truncated": good[:-7],
        "extra_byte": good + b"\0",
        "bad_magic": b"NOTASCENE 1 8 0 0\n",
        "empty": b"",
        "version2": b"DRKSCENE 2 8 2 100\n" + body,
        "k2": b"DRKSCENE 1 2 0 0\n",
        "deg4": b"DRKSCENE 1 8 4 0\n",
        "neg_count": b"DRKSCENE 1 8 2 -1\n",
        "short_header": b"DRKSCENE 1 8 2\n",
        "junk_in_k": b"DRKSCENE 1 8x 2 100\n" + body,
        "junk_after_count": b"DRKSCENE 1 8 2 100junk\n" + body,
        "extra_tokens": b"DRKSCENE 1 8 2 100 7 7\n" + body,
        "tabs_plus": b"DRKSCENE\t+1  8\t2 +100\r\n" + body,
        "no_newline_empty": b"DRKSCENE 1 8 2 0",
        "count_mismatch": b"DRKSCENE 1 8 2 99\n" + body,
        "one_record": b"DRKSCENE 1 8 2 1\n" + body[:rec],
        "huge_count": b"DRKSCENE 1 8 2 99999999999999\n" + body,
        "int_overflow_k": b"DRKSCENE 1 99999999999 2 0\n",
    }
    out = []
    for name, data in cases.items():
        p = os.path.join(tmp, f"{name}.drk")
        with open(p, "wb") as fh:
            fh.write(data)
        out.append((name, p, -1))
    out.append(("k_expected_5", golden_path("k8_sh2"), 5))  # VersionMismatchError (test_io.cpp:85)
    out.append(("k_expected_8", golden_path("k8_sh2"), 8))
    out.append(("missing", os.path.join(tmp, "does_not_exist.drk"), -1))
    return out


def oracle_status(path, k):
    try:
        scene_io.read_header(path, k)
        return 0
    except scene_io.SceneError as e:
        return e.status


needs_ref = pytest.mark.skipif(not scene_io.reference_available(), reason="oracle/_ref/libdrk_refio.so not built")


# --- CPU: restatement pinned against the reference ------------------------------
def test_golden_files_restatement():
    inp = golden_inputs()
    for name in NAMES:
        k, deg, raw = scene_io.load_scene(golden_path(name))
        assert (k, deg, raw.shape[1]) == HEADERS[name]
        assert np.array_equal(raw.view(np.uint32), inp[name].view(np.uint32))


def test_restatement_save_matches_golden_bytes(tmp_path):
    inp = golden_inputs()
    for name in NAMES:
        k, deg, _ = HEADERS[name]
        p = str(tmp_path / f"{name}.drk")
        scene_io.save_scene(p, inp[name], k, deg)
        assert open(p, "rb").read() == open(golden_path(name), "rb").read()


@needs_ref
def test_restatement_matches_reference_round_trip(tmp_path):
    # values not representable in f32: both narrow with round-to-nearest (io.cpp:26)
    rng = np.random.default_rng(5)
    for k, deg, n in ((8, 3, 64), (3, 0, 5), (16, 1, 9), (8, 0, 0)):
        raw = rng.normal(0, 3, (scene_io.scalar_count(k, deg), n))
        a, b = str(tmp_path / "ref.drk"), str(tmp_path / "ours.drk")
        assert scene_io.ref_save_scene(a, raw, k, deg) == 0
        scene_io.save_scene(b, raw, k, deg)
        assert open(a, "rb").read() == open(b, "rb").read()
        st, k2, d2, r2 = scene_io.ref_load_scene(a)
        assert st == 0 and (k2, d2) == (k, deg)
        k3, d3, r3 = scene_io.load_scene(a)
        assert np.array_equal(r2.astype(np.float32).view(np.uint32), r3.view(np.uint32))
        # save -> load -> save reproduces the bytes (test_io.cpp:56-62)
        assert scene_io.ref_save_scene(b, r2, k, deg) == 0
        assert open(a, "rb").read() == open(b, "rb").read()


@needs_ref
def test_restatement_matches_reference_on_malformed_files(tmp_path):
    for name, path, k in malformed_files(str(tmp_path)):
        st_ref = scene_io.ref_load_scene(path, k)[0]
        assert oracle_status(path, k) == st_ref, name


def test_reference_suite_rejection_cases(tmp_path):
    # test_io.cpp:65-94: truncation -> CorruptFileError, K mismatch -> VersionMismatchError,
    # bad magic -> CorruptFileError
    cases = {n: (p, k) for n, p, k in malformed_files(str(tmp_path))}
    assert oracle_status(*cases["truncated"]) == scene_io.CORRUPT
    assert oracle_status(*cases["k_expected_5"]) == scene_io.VERSION
    assert oracle_status(*cases["bad_magic"]) == scene_io.CORRUPT
    assert oracle_status(*cases["k_expected_8"]) == 0


# --- CPU: the C-ABI header checks (host-only entry point) ---------------------------
@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLDEN), "..", "paper_2412_11752_b200",
                                                    "libdrk_b200.so")), reason="CUDA extension not built")
def test_cabi_header_checks_match_oracle(tmp_path):
    import ctypes as C

    from paper_2412_11752_b200 import _lib
    for name, path, k in malformed_files(str(tmp_path)) + [(n, golden_path(n), -1) for n in NAMES]:
        h = _lib.SceneHeader_()
        st = _lib.lib().drk_scene_read_header(os.fsencode(path), k, C.byref(h))
        assert st == oracle_status(path, k), name
        if st == 0:
            kk, deg, count, payload, _ = scene_io.read_header(path, k)
            assert (h.basis_count, h.sh_degree, h.count, h.scalar_count) == \
                (kk, deg, count, scene_io.scalar_count(kk, deg)), name


# --- GPU: device loader / saver ------------------------------------------------------
@pytest.mark.gpu
def test_device_load_golden(rast):
    inp = golden_inputs()
    for name in NAMES:
        sc = rast.load_scene(golden_path(name))
        assert (sc.basis_count, sc.sh_degree, sc.params.shape[1]) == HEADERS[name]
        got = sc.params.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), inp[name].view(np.uint32)), name


@pytest.mark.gpu
def test_device_save_matches_golden_bytes(rast, tmp_path):
    import torch

    from paper_2412_11752_b200.api import DeviceScene
    inp = golden_inputs()
    for name in NAMES:
        k, deg, _ = HEADERS[name]
        p = str(tmp_path / f"{name}.drk")
        rast.save_scene(DeviceScene(k, deg, torch.from_numpy(inp[name]).cuda()), p)
        assert open(p, "rb").read() == open(golden_path(name), "rb").read(), name


@pytest.mark.gpu
def test_device_load_errors(rast, tmp_path):
    from paper_2412_11752_b200 import _lib
    classes = {scene_io.IO: _lib.IoError, scene_io.CORRUPT: _lib.CorruptFileError,
               scene_io.VERSION: _lib.VersionMismatchError}
    for name, path, k in malformed_files(str(tmp_path)):
        st = oracle_status(path, k)
        if st == 0:
            sc = rast.load_scene(path, k)
            _, _, raw = scene_io.load_scene(path, k)
            assert np.array_equal(sc.params.cpu().numpy().view(np.uint32), raw.view(np.uint32)), name
        else:
            with pytest.raises(classes[st]):
                rast.load_scene(path, k)


@pytest.mark.gpu
def test_device_round_trip_config1(rast, tmp_path):
    """Config-1 size (100k DRKs, SH 3): device save == restatement bytes, device load
    == the saved parameters bit for bit, and the loaded scene renders identically."""
    import torch

    from paper_2412_11752_b200 import scenes
    from paper_2412_11752_b200.api import DeviceScene, RenderOptions
    sc = scenes.config_scene(1)
    raw = sc.f32()
    p_dev, p_orc = str(tmp_path / "dev.drk"), str(tmp_path / "orc.drk")
    rast.save_scene(DeviceScene(8, 3, torch.from_numpy(raw).cuda()), p_dev)
    scene_io.save_scene(p_orc, raw, 8, 3)
    assert open(p_dev, "rb").read() == open(p_orc, "rb").read()
    loaded = rast.load_scene(p_dev, 8)
    assert np.array_equal(loaded.params.cpu().numpy().view(np.uint32), raw.view(np.uint32))
    cam = scenes.config_cameras(1)[0]
    cam_small = scenes.Camera(fx=cam.fx / 4, fy=cam.fy / 4, cx=cam.cx / 4, cy=cam.cy / 4, width=480, height=270,
                              R=cam.R, t=cam.t)
    opt = RenderOptions(sh_degree=3)
    a = rast.render(torch.from_numpy(raw).cuda(), cam_small, opt).color.clone()
    b = rast.render(loaded.params, cam_small, opt).color
    assert torch.equal(a, b)
