"""Mesh2DRK (reference mesh.cpp): the OBJ / MTL loader
(host, through the C-ABI) against the reference's load_mesh, and the device
face -> DRK conversion and Lambert shading against the reference's convert /
shade_lambert (oracle/_ref/libdrk_refio.so, mesh.cpp built unmodified)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import scene_io

needs_ref = pytest.mark.skipif(not scene_io.reference_available(), reason="oracle/_ref/libdrk_refio.so not built")

OBJ = """# test mesh
mtllib mats.mtl
v 0 0 0
v 1 0 0
v 1 1 0
v 0 1 0
v 0.5 0.5 1
v 2 0 0.3
v 2.5 0.2 0.1
v 2.2 1.1 0.5
vt 0 0
usemtl red
f 1 2 3 4
f 1/1 2/1 5/1
usemtl blue
f -7 -6 5
f 6 7 8
f 2 3 5 1
usemtl none
f 1 2 2
f 1 3 2 4
v 3 0 0
v 4 0 0
v 4 1 0
v 4.5 0.5 0
v 3 1 0
f 9 10 12 11 13
f 9 11 10 12 13
"""
MTL = """newmtl red
Kd 0.9 0.1 0.2
newmtl blue
Kd 0.1 0.2 0.95
"""


def write_mesh(tmp, obj=OBJ, mtl=MTL):
    with open(os.path.join(tmp, "mats.mtl"), "w") as fh:
        fh.write(mtl)
    p = os.path.join(tmp, "m.obj")
    with open(p, "w") as fh:
        fh.write(obj)
    return p


BAD = {  # reference error statuses: 11 IoError, 16 ParseError, 17 EmptyMeshError
    "bad_vertex": ("v 0 0\nf 1 2 3\n", 16),
    "zero_index": ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", 16),
    "out_of_range": ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 4\n", 16),
    "bad_token": ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 x 3\n", 16),
    "two_vertices": ("v 0 0 0\nv 1 0 0\nf 1 2\n", 16),
    "no_faces": ("v 0 0 0\n", 17),
}


def mesh_dict(m):
    return dict(vertices=m.vertices, face_offsets=m.face_offsets, indices=m.indices, colors=m.colors,
                warnings=m.warnings)


@needs_ref
def test_load_mesh_matches_reference(tmp_path):
    from paper_2412_11752_b200.api import load_mesh
    p = write_mesh(str(tmp_path))
    st, want = scene_io.ref_load_mesh(p)
    assert st == 0
    got = mesh_dict(load_mesh(p))
    for key in ("vertices", "face_offsets", "indices", "colors"):
        assert np.array_equal(got[key], want[key]), key
    assert got["warnings"] == want["warnings"] > 0
    assert len(got["face_offsets"]) - 1 > 8  # fan-triangulated non-planar / concave faces


@needs_ref
def test_load_mesh_errors_match_reference(tmp_path):
    from paper_2412_11752_b200 import _lib
    from paper_2412_11752_b200.api import load_mesh
    for name, (text, status) in BAD.items():
        p = str(tmp_path / f"{name}.obj")
        with open(p, "w") as fh:
            fh.write(text)
        assert scene_io.ref_load_mesh(p)[0] == status, name
        with pytest.raises(_lib._ERRORS[status]):
            load_mesh(p)
    assert scene_io.ref_load_mesh(str(tmp_path / "missing.obj"))[0] == 11
    with pytest.raises(_lib.IoError):
        load_mesh(str(tmp_path / "missing.obj"))


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("k", [8, 5, 16])
def test_device_convert_and_shade_match_reference(rast, tmp_path, k):
    from paper_2412_11752_b200.api import load_mesh
    m = load_mesh(write_mesh(str(tmp_path)))
    st, want, skipped = scene_io.ref_convert(mesh_dict(m), k)
    assert st == 0
    raw, n_skip = rast.mesh_convert(m, basis_count=k)
    assert n_skip == skipped and n_skip >= 1  # the degenerate "f 1 2 2"
    got = raw.cpu().numpy()
    ref32 = want.astype(np.float32)
    assert got.shape == ref32.shape
    # fp64 in the reference's expression order, device libm (atan2 / cos / sin / log)
    # against glibc: identical after the f32 rounding up to one ulp
    np.testing.assert_array_max_ulp(got, ref32, maxulp=1)
    assert (got == ref32).mean() > 0.97
    light, amb = (0.3, -1.0, 0.5), 0.25
    rast.shade_lambert(raw, light, amb, basis_count=k)
    shaded = scene_io.ref_shade_lambert(got.astype(np.float64), k, light, amb).astype(np.float32)
    np.testing.assert_array_max_ulp(raw.cpu().numpy(), shaded, maxulp=1)


@pytest.mark.gpu
@needs_ref
def test_device_convert_too_many_vertices(rast, tmp_path):
    from paper_2412_11752_b200 import _lib
    from paper_2412_11752_b200.api import load_mesh
    m = load_mesh(write_mesh(str(tmp_path)))
    assert scene_io.ref_convert(mesh_dict(m), 4)[0] == 15
    with pytest.raises(_lib.TooManyVerticesError):
        rast.mesh_convert(m, basis_count=4)


@pytest.mark.gpu
def test_converted_mesh_renders(rast, tmp_path):
    """Converted faces render through the forward path (SH degree 0)."""
    from paper_2412_11752_b200 import scenes
    from paper_2412_11752_b200.api import RenderOptions, load_mesh
    m = load_mesh(write_mesh(str(tmp_path)))
    raw, _ = rast.mesh_convert(m, basis_count=8)
    cam = scenes.look_at_camera(64, 48, (1.5, 0.5, -4.0), target=(1.5, 0.5, 0.3))
    fb = rast.render(raw, cam, RenderOptions(sh_degree=0))
    assert float(fb.alpha.max()) > 0.5
