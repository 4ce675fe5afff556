"""DRKSCENE v1 scene files: numpy restatement of the reference's
drk::save_scene / drk::load_scene (io.cpp:40-97; format io.hpp:20-23), plus a
ctypes binding of the unmodified reference functions built into
oracle/_ref/libdrk_refio.so (oracle/Makefile.ref).

TEST INFRASTRUCTURE ONLY: imported by tests/ (checker of the device loader /
saver in paper_2412_11752_b200/csrc/drk_scene.cu), never by the product.

Arrays use the C-ABI raw layout: float [scalar_count, n] (scalar-major; the
file is record-major in the same for_each_scalar order, types.hpp:48-74).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

SCENE_VERSION = 1  # io.cpp:22
IO, CORRUPT, VERSION, DIMENSION = 11, 12, 13, 6  # include/drk_b200.h status codes


class SceneError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def scalar_count(k: int, sh_degree: int) -> int:
    """types.hpp:74 with terms = (deg + 1)^2 (sh_coeff_count)."""
    return 3 + 4 + 2 * k + 3 + 3 * (sh_degree + 1) ** 2


def save_scene(path: str, raw: np.ndarray, k: int, sh_degree: int) -> None:
    """io.cpp:40-56: header line, then every record's scalars as little-endian f32."""
    S, n = raw.shape
    if S != scalar_count(k, sh_degree):
        raise SceneError(DIMENSION, "primitive layout differs from the scene header")  # io.cpp:46-47
    payload = np.ascontiguousarray(np.asarray(raw).astype("<f4").T).tobytes()  # put_f32: float(v), LE
    with open(path, "wb") as fh:
        fh.write(f"DRKSCENE {SCENE_VERSION} {k} {sh_degree} {n}\n".encode())  # io.cpp:52-53
        fh.write(payload)


def _extract_int(tok: str, last: bool):
    """std::istream >> int/long on one whitespace token: optional sign, digits;
    a non-digit tail makes the following extraction fail (except after the last)."""
    i = 1 if tok[:1] in "+-" else 0
    j = i
    while j < len(tok) and tok[j].isdigit():
        j += 1
    if j == i or (j < len(tok) and not last):
        return None
    return int(tok[:j])


def read_header(path: str, expected_basis_count: int = -1):
    """io.cpp:58-80 header checks, in the reference's order.  Returns
    (k, sh_degree, count, payload_bytes, header_len)."""
    try:
        fh = open(path, "rb")
    except OSError:
        raise SceneError(IO, "cannot open scene file: " + path)  # io.cpp:60
    with fh:
        data = fh.read()
    if not data:
        raise SceneError(CORRUPT, "missing scene header: " + path)  # io.cpp:63
    nl = data.find(b"\n")
    line = data if nl < 0 else data[:nl]
    hlen = len(data) if nl < 0 else nl + 1
    toks = [t for t in re.split(r"[ \t\r\v\f]+", line.decode("latin-1")) if t]
    vals = None
    if len(toks) >= 5:
        vals = [_extract_int(t, i == 3) for i, t in enumerate(toks[1:5])]
        if any(v is None for v in vals) or not all(-2**31 <= v < 2**31 for v in vals[:3]) or \
                not -2**63 <= vals[3] < 2**63:
            vals = None
    if vals is None or toks[0] != "DRKSCENE":
        raise SceneError(CORRUPT, "not a scene file: " + path)  # io.cpp:67-68
    version, k, deg, count = vals
    if version != SCENE_VERSION:
        raise SceneError(VERSION, f"unsupported scene version {version}")  # io.cpp:69-70
    if k < 3 or deg < 0 or deg > 3 or count < 0:
        raise SceneError(CORRUPT, "implausible scene header: " + path)  # io.cpp:71-72
    if expected_basis_count > 0 and k != expected_basis_count:
        raise SceneError(VERSION, f"scene has K={k}, pipeline expects K={expected_basis_count}")  # io.cpp:73-75
    rec = 4 * scalar_count(k, deg)
    if len(data) - hlen != rec * count:
        raise SceneError(CORRUPT, "scene payload size disagrees with the header count: " + path)  # io.cpp:79-80
    return k, deg, count, len(data) - hlen, hlen


def load_scene(path: str, expected_basis_count: int = -1):
    """io.cpp:58-97 -> (k, sh_degree, raw f32 [S, count])."""
    k, deg, count, _, hlen = read_header(path, expected_basis_count)
    with open(path, "rb") as fh:
        fh.seek(hlen)
        body = fh.read()
    S = scalar_count(k, deg)
    raw = np.frombuffer(body, dtype="<f4").reshape(count, S).T.astype(np.float32)
    return k, deg, np.ascontiguousarray(raw)


# --- the reference itself (oracle/_ref/libdrk_refio.so) ----------------------
_REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libdrk_refio.so")
_ref_lib = None


def reference_available() -> bool:
    return os.path.exists(_REF)


def _lib():
    global _ref_lib
    if _ref_lib is None:
        h = C.CDLL(_REF)
        h.refio_save_scene.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        h.refio_load_scene.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_longlong]
        _ref_lib = h
    return _ref_lib


def ref_save_scene(path: str, raw: np.ndarray, k: int, sh_degree: int) -> int:
    """drk::save_scene of the reference build; returns the status code (0 ok)."""
    r = np.ascontiguousarray(raw, dtype=np.float64)
    return _lib().refio_save_scene(os.fsencode(path), r.ctypes.data, r.shape[1], k, sh_degree)


def ref_load_scene(path: str, expected_basis_count: int = -1):
    """drk::load_scene of the reference build -> (status, k, deg, raw f64 [S, n] or None)."""
    hdr = np.zeros(4, np.int64)
    st = _lib().refio_load_scene(os.fsencode(path), expected_basis_count, hdr.ctypes.data, None, 0)
    if st:
        return st, None, None, None
    k, deg, n = int(hdr[0]), int(hdr[1]), int(hdr[2])
    raw = np.zeros((scalar_count(k, deg), n), np.float64)
    st = _lib().refio_load_scene(os.fsencode(path), expected_basis_count, hdr.ctypes.data, raw.ctypes.data, n)
    return st, k, deg, raw


# --- Mesh2DRK of the reference build (mesh.cpp in oracle/_ref/libdrk_refio.so) --------
def ref_load_mesh(path: str):
    """load_mesh (mesh.cpp:134-217) -> (status, dict of arrays or None)."""
    h = _lib()
    h.refmesh_load.argtypes = [C.c_char_p, C.c_void_p]
    sizes = np.zeros(4, np.int64)
    st = h.refmesh_load(os.fsencode(path), sizes.ctypes.data)
    if st:
        return st, None
    nv, nf, ni, nw = (int(x) for x in sizes)
    out = dict(vertices=np.zeros((nv, 3)), face_offsets=np.zeros(nf + 1, np.int32), indices=np.zeros(ni, np.int32),
               colors=np.zeros((nf, 3)), warnings=nw)
    h.refmesh_arrays.argtypes = [C.c_void_p] * 4
    h.refmesh_arrays(out["vertices"].ctypes.data, out["face_offsets"].ctypes.data, out["indices"].ctypes.data,
                     out["colors"].ctypes.data)
    return 0, out


def ref_convert(mesh: dict, k: int):
    """convert (mesh.cpp:326-343) -> (status, raw f64 [S, n], n_skipped)."""
    h = _lib()
    h.refmesh_convert.argtypes = [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                  C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p]
    nf = len(mesh["face_offsets"]) - 1
    S = scalar_count(k, 0)
    raw = np.zeros((S, max(nf, 1)))
    n_out, n_skip = C.c_longlong(0), C.c_longlong(0)
    v = np.ascontiguousarray(mesh["vertices"], np.float64)
    o = np.ascontiguousarray(mesh["face_offsets"], np.int32)
    i = np.ascontiguousarray(mesh["indices"], np.int32)
    c = np.ascontiguousarray(mesh["colors"], np.float64)
    st = h.refmesh_convert(v.ctypes.data, len(v), o.ctypes.data, i.ctypes.data, c.ctypes.data, nf, k, raw.ctypes.data,
                           raw.shape[1], C.byref(n_out), C.byref(n_skip))
    if st:
        return st, None, None
    return 0, np.ascontiguousarray(raw[:, :n_out.value]), n_skip.value


def ref_shade_lambert(raw: np.ndarray, k: int, light, ambient: float) -> np.ndarray:
    """shade_lambert (mesh.cpp:345-357) on a copy of raw f64 [S, n] (SH degree 0)."""
    h = _lib()
    h.refmesh_shade.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_double]
    r = np.ascontiguousarray(raw, np.float64).copy()
    lt = np.asarray(light, np.float64)
    assert h.refmesh_shade(r.ctypes.data, r.shape[1], k, lt.ctypes.data, float(ambient)) == 0
    return r
