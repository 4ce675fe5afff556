"""ctypes bindings to the C restatement oracle (oracle/liboracle.so, built
from oracle/drk_oracle.c).  TEST INFRASTRUCTURE ONLY — same API as
oracle/ref.py; ``render`` additionally returns the work counters used for the
roofline's algorithmic flop count."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import ref as _ref
from .ref import Options, _cam, _opt, _p  # noqa: F401  (re-exported)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")


class Stats(C.Structure):
    _fields_ = [(name, C.c_int64) for name in
                ("pairs", "hits", "streamed", "popped", "composited", "poly_vertices", "max_poly")]


_LIB = _ref._Lib(LIB_PATH, "orc_")


def available() -> bool:
    return _LIB.available()


def _with_lib(fn):
    def wrapped(*a, **kw):
        saved = _ref._LIB
        _ref._LIB = _LIB
        try:
            return fn(*a, **kw)
        finally:
            _ref._LIB = saved
    wrapped.__doc__ = fn.__doc__
    return wrapped


activate = _with_lib(_ref.activate)
bin_primitives = _with_lib(_ref.bin_primitives)
backward = _with_lib(_ref.backward)
loss_l1 = _with_lib(_ref.loss_l1)
adam_step = _with_lib(_ref.adam_step)


def render(scene, cam, opt: Options = Options(), replay: bool = False):
    H, W = cam.height, cam.width
    color = np.zeros((H, W, 3))
    depth = np.zeros((H, W))
    normal = np.zeros((H, W, 3))
    alpha = np.zeros((H, W))
    nrec = C.c_int64(0)
    st = Stats()
    raw = np.ascontiguousarray(scene.raw, dtype=np.float64)
    rc = _LIB.orc_render(_p(raw), scene.n, scene.k, scene.terms, C.byref(_cam(cam)), C.byref(_opt(opt)),
                         _p(color), _p(depth), _p(normal), _p(alpha), int(replay), C.byref(nrec), C.byref(st))
    if rc != 0:
        raise RuntimeError(f"oracle error {rc}: {_LIB.orc_last_error().decode()}")
    out = dict(color=color, depth=depth, normal=normal, alpha=alpha,
               stats={f: getattr(st, f) for f, _ in Stats._fields_})
    if replay:
        off = np.zeros(H * W + 1, dtype=np.int64)
        ids = np.zeros(nrec.value, dtype=np.int32)
        vals = np.zeros((nrec.value, 5))
        _LIB.orc_replay_copy(_p(off), _p(ids), _p(vals))
        out["replay"] = (off, ids, vals)
    return out
