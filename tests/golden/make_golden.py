"""Generates the golden fixtures of tests/golden/ from the UNMODIFIED reference
build (oracle/_ref/libdrk_refcapi.so, compiled from /root/reference/proj/src by
oracle/Makefile.ref).  Run from the repo root:  python tests/golden/make_golden.py

Each fixture holds the seeded inputs (raw parameters in the ABI layout, camera,
options) and the reference outputs: tile lists (ids + f64 keys per tile),
framebuffers, per-pixel replay records and backward_render gradients for a
fixed random frame gradient.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2412_11752_b200 import scenes  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (scene kwargs, camera (w, h, pos), options)
    "small_sh1": (dict(n=150, seed=21, sh_degree=1), (64, 48, (0.3, -0.2, -3.4)),
                  dict(sh_degree=1, background=(0.3, 0.5, 0.2))),
    "cluster_sh3": (dict(n=400, seed=22, sh_degree=3, clusters=6), (48, 32, (0.0, 0.4, -3.8)), dict(sh_degree=3)),
    "k4_list_order": (dict(n=120, seed=23, k=4, sh_degree=0), (48, 48, (-0.5, 0.1, -3.0)),
                      dict(sh_degree=0, use_cache=False, presort=1)),
}


def make(name):
    skw, (w, h, pos), okw = CASES[name]
    sc = scenes.random_scene(**skw)
    cam = scenes.look_at_camera(w, h, pos)
    opt = ref.Options(**okw)
    off, ids, keys = ref.bin_primitives(sc, cam, opt)
    fb = ref.render(sc, cam, opt, replay=True)
    roff, rids, rvals = fb["replay"]
    rng = np.random.default_rng(7)
    dc = rng.uniform(-1, 1, (h, w, 3)).astype(np.float32).astype(np.float64)
    dd = rng.uniform(-0.1, 0.1, (h, w)).astype(np.float32).astype(np.float64)
    g = ref.backward(sc, cam, opt, dc, dd, None, None)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), raw=sc.raw, k=sc.k, sh_degree=sc.sh_degree,
                        cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]), cam_wh=np.array([w, h]), cam_R=cam.R,
                        cam_t=cam.t, opt=np.array([opt.sh_degree, int(opt.use_cache), int(opt.exact_sort),
                                                   opt.presort]),
                        background=np.array(opt.background), tile_off=off, tile_ids=ids, tile_keys=keys,
                        color=fb["color"], depth=fb["depth"], normal=fb["normal"], alpha=fb["alpha"],
                        replay_off=roff, replay_ids=rids, replay_vals=rvals, d_color=dc, d_depth=dd,
                        grad_raw=g["raw"], grad_dcw=g["d_center_world"], grad_screen=g["screen_grad"],
                        grad_touched=g["touched"])
    print(name, "pairs", len(ids), "records", len(rids))


if __name__ == "__main__":
    for n in CASES:
        make(n)
