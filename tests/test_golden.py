"""Golden fixtures generated from the unmodified reference build
(tests/golden/make_golden.py): the C oracle reproduces them bit for bit (CPU),
and the CUDA path matches them within the parity tolerances (GPU).  The
fixtures travel to the GPU box; /root/reference is not needed there."""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from oracle import port, ref
from paper_2412_11752_b200 import scenes

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(f for f in glob.glob(os.path.join(HERE, "golden", "*.npz"))
                  if not os.path.basename(f).startswith("scene_"))  # scene files: test_scene_io.py


def load(path):
    z = np.load(path)
    sc = scenes.Scene(raw=z["raw"], k=int(z["k"]), sh_degree=int(z["sh_degree"]))
    fx, fy, cx, cy = z["cam_f"]
    w, h = (int(v) for v in z["cam_wh"])
    cam = scenes.Camera(fx, fy, cx, cy, w, h, z["cam_R"], z["cam_t"])
    deg, cache, exact, presort = (int(v) for v in z["opt"])
    opt = ref.Options(sh_degree=deg, use_cache=bool(cache), exact_sort=bool(exact), presort=presort,
                      background=tuple(z["background"]))
    return z, sc, cam, opt


@pytest.mark.skipif(not port.available(), reason="oracle not built")
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_oracle_reproduces_reference_fixture(path):
    z, sc, cam, opt = load(path)
    off, ids, keys = port.bin_primitives(sc, cam, opt)
    assert np.array_equal(off, z["tile_off"]) and np.array_equal(ids, z["tile_ids"])
    assert np.array_equal(keys.view(np.uint64), z["tile_keys"].view(np.uint64))
    fb = port.render(sc, cam, opt, replay=True)
    for f in ("color", "depth", "normal", "alpha"):
        assert np.array_equal(fb[f], z[f]), f
    roff, rids, rvals = fb["replay"]
    assert np.array_equal(roff, z["replay_off"]) and np.array_equal(rids, z["replay_ids"])
    assert np.array_equal(rvals, z["replay_vals"])
    g = port.backward(sc, cam, opt, z["d_color"], z["d_depth"], None, None)
    assert np.array_equal(g["raw"], z["grad_raw"]) and np.array_equal(g["touched"], z["grad_touched"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_cuda_matches_reference_fixture(rast, path):
    import torch

    from paper_2412_11752_b200.api import FrameGrad
    from tests.helpers import api_options, rel_l2
    z, sc, cam, opt = load(path)
    fb = rast.render(sc.f32(), cam, api_options(opt), k=sc.k)
    b = rast.tile_binning()
    assert np.array_equal(b.offsets, z["tile_off"]) and np.array_equal(b.prim_ids, z["tile_ids"])
    assert np.array_equal(b.keys.view(np.uint64), z["tile_keys"].view(np.uint64))
    for f in ("color", "depth", "normal", "alpha"):
        err = np.abs(getattr(fb, f).cpu().numpy().astype(np.float64) - z[f]).max()
        assert err <= 1e-4, (f, err)
    g = rast.backward_render(sc.f32(), FrameGrad(d_color=torch.from_numpy(z["d_color"].astype(np.float32)),
                                                 d_depth=torch.from_numpy(z["d_depth"].astype(np.float32))))
    assert rel_l2(g.raw.cpu().numpy(), z["grad_raw"]) <= 1e-3
    assert np.array_equal(g.touched.cpu().numpy(), z["grad_touched"])
