"""Golden DRKSCENE files written by the UNMODIFIED reference drk::save_scene
(oracle/_ref/libdrk_refio.so, built from /root/reference/proj/src/io.cpp by
oracle/Makefile.ref).  Run from the repo root:
    python tests/golden/make_golden_scenes.py
Writes tests/golden/scene_<name>.drk and scene_inputs.npz (the raw parameters,
C-ABI layout f32 [S, n], that were saved)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import scene_io  # noqa: E402
from paper_2412_11752_b200 import scenes  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = {"k8_sh2": dict(n=100, seed=123, k=8, sh_degree=2), "k5_sh0": dict(n=37, seed=124, k=5, sh_degree=0),
         "k8_sh3_empty": dict(n=0, seed=125, k=8, sh_degree=3)}


def main():
    assert scene_io.reference_available(), "build oracle/_ref first (make -f oracle/Makefile.ref)"
    arrays = {}
    for name, kw in CASES.items():
        if kw["n"] > 0:
            raw = scenes.random_scene(kw["n"], seed=kw["seed"], k=kw["k"], sh_degree=kw["sh_degree"]).f32()
        else:
            raw = np.zeros((scene_io.scalar_count(kw["k"], kw["sh_degree"]), 0), np.float32)
        path = os.path.join(OUT, f"scene_{name}.drk")
        st = scene_io.ref_save_scene(path, raw.astype(np.float64), kw["k"], kw["sh_degree"])
        assert st == 0, st
        arrays[name] = raw
        print(name, raw.shape, os.path.getsize(path), "bytes")
    np.savez_compressed(os.path.join(OUT, "scene_inputs.npz"), **arrays)


if __name__ == "__main__":
    main()
