"""ctypes bindings to the reference build (oracle/_ref/libdrk_refcapi.so).

TEST INFRASTRUCTURE ONLY: imported by tests/ (as the checker), by
``__graft_entry__.smoke()`` and by bench.py's ``cpu_baseline`` / ``--impl
reference`` arm.  The library is the UNMODIFIED reference hot path
(/root/reference/proj/src/{core,geometry,raster,grad,image,optimize}.cpp)
compiled by oracle/Makefile.ref against the header shims in oracle/shim/.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libdrk_refcapi.so")


class RefCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_double * 9),
                ("t", C.c_double * 3)]


class RefOptions(C.Structure):
    _fields_ = [("lowpass_radius", C.c_double), ("alpha_min", C.c_double),
                ("grazing_eps", C.c_double), ("background", C.c_double * 3),
                ("early_stop_transmittance", C.c_double), ("sh_degree", C.c_int32),
                ("use_cache", C.c_int32), ("exact_sort", C.c_int32), ("presort", C.c_int32),
                ("threads", C.c_int32), ("pad_", C.c_int32)]


@dataclass
class Options:
    """Mirror of drk::RenderOptions + KernelConfig (reference raster.hpp:81-90, types.hpp:100-105)."""

    lowpass_radius: float = 0.5
    alpha_min: float = 1.0 / 255.0
    grazing_eps: float = 1e-6
    background: tuple = (1.0, 1.0, 1.0)
    early_stop_transmittance: float = 1e-4
    sh_degree: int = 3
    use_cache: bool = True
    exact_sort: bool = False
    presort: int = 2  # 0 None, 1 CenterDepth, 2 NearestDepth
    threads: int = 1


class _Lib:
    """Resolves `<prefix>name` symbols of one of the two CPU libraries."""

    def __init__(self, path: str, prefix: str):
        self.path, self.prefix, self._h = path, prefix, None

    def available(self) -> bool:
        return os.path.exists(self.path)

    def __getattr__(self, name):
        if self._h is None:
            if not self.available():
                raise RuntimeError(f"CPU oracle library missing: {self.path} (run __graft_entry__.build())")
            self._h = C.CDLL(self.path)
            getattr(self._h, self.prefix + "last_error").restype = C.c_char_p
        short = name[4:] if name[:4] in ("ref_", "orc_") else name
        return getattr(self._h, self.prefix + short)


_LIB = _Lib(LIB_PATH, "ref_")


def available() -> bool:
    return _LIB.available()


def lib():
    return _LIB


def _cam(cam) -> RefCamera:
    c = RefCamera()
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    R = np.asarray(cam.R, dtype=np.float64).reshape(9)
    t = np.asarray(cam.t, dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
    return c


def _opt(opt: Options) -> RefOptions:
    o = RefOptions()
    o.lowpass_radius, o.alpha_min, o.grazing_eps = opt.lowpass_radius, opt.alpha_min, opt.grazing_eps
    for i in range(3):
        o.background[i] = opt.background[i]
    o.early_stop_transmittance = opt.early_stop_transmittance
    o.sh_degree, o.use_cache, o.exact_sort = opt.sh_degree, int(opt.use_cache), int(opt.exact_sort)
    o.presort, o.threads = opt.presort, opt.threads
    return o


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _raw(scene) -> np.ndarray:
    return np.ascontiguousarray(scene.raw, dtype=np.float64)


def hardware_threads() -> int:
    return int(lib().ref_hardware_threads())


def activate(scene):
    n, k = scene.n, scene.k
    out = dict(mu=np.zeros((n, 3)), rot=np.zeros((n, 3, 3)), scales=np.zeros((n, k)),
               angles=np.zeros((n, k)), eta=np.zeros(n), tau=np.zeros(n), opacity=np.zeros(n))
    _check(lib().ref_activate(_p(_raw(scene)), n, k, scene.terms, *[_p(out[x]) for x in
                              ("mu", "rot", "scales", "angles", "eta", "tau", "opacity")]))
    return out


def eval_sorting(scene, cam, opt: Options = Options()):
    """drk::eval_sorting (raster.cpp:487-560) -> (accuracy, kendall_tau, mae, pixels)."""
    out = np.zeros(4)
    _check(lib().ref_eval_sorting(_p(_raw(scene)), scene.n, scene.k, scene.terms, C.byref(_cam(cam)),
                                  C.byref(_opt(opt)), _p(out)))
    return float(out[0]), float(out[1]), float(out[2]), int(out[3])


def bin_primitives(scene, cam, opt: Options = Options()):
    """Returns (offsets[T+1], prim_ids[P], keys[P]) of the reference TileBinning."""
    total = C.c_int64(0)
    _check(lib().ref_bin(_p(_raw(scene)), scene.n, scene.k, scene.terms, C.byref(_cam(cam)),
                         C.byref(_opt(opt)), C.byref(total)))
    tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    off = np.zeros(tiles + 1, dtype=np.int64)
    ids = np.zeros(total.value, dtype=np.int32)
    keys = np.zeros(total.value, dtype=np.float64)
    lib().ref_bins_copy(_p(off), _p(ids), _p(keys))
    return off, ids, keys


def bin_primitives_parallel(scene, cam, opt: Options = Options(), threads: int = 0):
    """Reference bin_primitives on `threads` chunks of the primitives, merged with the
    reference comparator (ref_bin_parallel): identical to bin_primitives, faster."""
    total = C.c_int64(0)
    _check(lib().ref_bin_parallel(_p(_raw(scene)), scene.n, scene.k, scene.terms, C.byref(_cam(cam)),
                                  C.byref(_opt(opt)), int(threads), C.byref(total)))
    tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    off = np.zeros(tiles + 1, dtype=np.int64)
    ids = np.zeros(total.value, dtype=np.int32)
    keys = np.zeros(total.value, dtype=np.float64)
    lib().ref_bins_copy(_p(off), _p(ids), _p(keys))
    return off, ids, keys


def fwd_bwd(scene, cam, target, opt: Options = Options()):
    """Reference activate + render(&replay) + L1 loss + backward_render (ref_fwd_bwd):
    framebuffers, loss, d_color, raw grads, d_center_world, screen_grad, touched and
    the wall seconds of the forward and of loss + backward."""
    H, W, n = cam.height, cam.width, scene.n
    out = dict(color=np.zeros((H, W, 3)), depth=np.zeros((H, W)), normal=np.zeros((H, W, 3)),
               alpha=np.zeros((H, W)), d_color=np.zeros((H, W, 3)), raw=np.zeros_like(scene.raw, dtype=np.float64),
               d_center_world=np.zeros((n, 3)), screen_grad=np.zeros(n), touched=np.zeros(n, dtype=np.int8))
    loss = C.c_double(0)
    secs = np.zeros(2)
    tgt = np.ascontiguousarray(target, dtype=np.float64)
    _check(lib().ref_fwd_bwd(_p(_raw(scene)), n, scene.k, scene.terms, C.byref(_cam(cam)), C.byref(_opt(opt)),
                             _p(tgt), *[_p(out[f]) for f in ("color", "depth", "normal", "alpha")], C.byref(loss),
                             _p(out["d_color"]), _p(out["raw"]), _p(out["d_center_world"]), _p(out["screen_grad"]),
                             _p(out["touched"]), _p(secs)))
    out["loss"] = loss.value
    out["seconds_fwd"], out["seconds_bwd"] = float(secs[0]), float(secs[1])
    return out


def render(scene, cam, opt: Options = Options(), replay: bool = False):
    H, W = cam.height, cam.width
    color = np.zeros((H, W, 3))
    depth = np.zeros((H, W))
    normal = np.zeros((H, W, 3))
    alpha = np.zeros((H, W))
    nrec = C.c_int64(0)
    secs = C.c_double(0)
    _check(lib().ref_render(_p(_raw(scene)), scene.n, scene.k, scene.terms, C.byref(_cam(cam)),
                            C.byref(_opt(opt)), _p(color), _p(depth), _p(normal), _p(alpha),
                            int(replay), C.byref(nrec), C.byref(secs)))
    out = dict(color=color, depth=depth, normal=normal, alpha=alpha, seconds=secs.value)
    if replay:
        off = np.zeros(H * W + 1, dtype=np.int64)
        ids = np.zeros(nrec.value, dtype=np.int32)
        vals = np.zeros((nrec.value, 5))
        lib().ref_replay_copy(_p(off), _p(ids), _p(vals))
        out["replay"] = (off, ids, vals)
    return out


def backward(scene, cam, opt: Options = Options(), d_color=None, d_depth=None, d_normal=None,
             d_alpha=None):
    n = scene.n
    g = np.zeros_like(scene.raw, dtype=np.float64)
    dcw = np.zeros((n, 3))
    sg = np.zeros(n)
    touched = np.zeros(n, dtype=np.int8)
    secs = C.c_double(0)

    def arr(a):
        return None if a is None else np.ascontiguousarray(a, dtype=np.float64)

    dc, dd, dn, da = arr(d_color), arr(d_depth), arr(d_normal), arr(d_alpha)
    _check(lib().ref_backward(_p(_raw(scene)), n, scene.k, scene.terms, C.byref(_cam(cam)),
                              C.byref(_opt(opt)), _p(dc), _p(dd), _p(dn), _p(da), _p(g), _p(dcw),
                              _p(sg), _p(touched), C.byref(secs)))
    return dict(raw=g, d_center_world=dcw, screen_grad=sg, touched=touched, seconds=secs.value)


def train_step(scene, cam, target, opt: Options = Options()):
    g = np.zeros_like(scene.raw, dtype=np.float64)
    loss = C.c_double(0)
    secs = C.c_double(0)
    tgt = np.ascontiguousarray(target, dtype=np.float64)
    _check(lib().ref_train_step(_p(_raw(scene)), scene.n, scene.k, scene.terms, C.byref(_cam(cam)),
                                C.byref(_opt(opt)), _p(tgt), C.byref(loss), _p(g), C.byref(secs)))
    return dict(loss=loss.value, raw=g, seconds=secs.value)


def loss_l1(rendered, target):
    H, W = rendered.shape[:2]
    d = np.zeros((H, W, 3))
    v = C.c_double(0)
    _check(lib().ref_loss_l1(_p(np.ascontiguousarray(rendered, dtype=np.float64)),
                             _p(np.ascontiguousarray(target, dtype=np.float64)), W, H, C.byref(v), _p(d)))
    return v.value, d


def loss(rendered, target, dssim_weight):
    """Full drk::loss (optimize.cpp:171-204) -> (value, d_color f64 like rendered)."""
    H, W, Cc = rendered.shape
    d = np.zeros((H, W, Cc))
    v = C.c_double(0)
    _check(lib().ref_loss(_p(np.ascontiguousarray(rendered, dtype=np.float64)),
                          _p(np.ascontiguousarray(target, dtype=np.float64)), W, H, Cc,
                          C.c_double(dssim_weight), C.byref(v), _p(d)))
    return v.value, d


def ssim(a, b):
    """drk::ssim (optimize.cpp:157-166)."""
    H, W, Cc = a.shape
    v = C.c_double(0)
    _check(lib().ref_ssim(_p(np.ascontiguousarray(a, dtype=np.float64)), _p(np.ascontiguousarray(b, dtype=np.float64)),
                          W, H, Cc, C.byref(v)))
    return v.value


def psnr(a, b):
    """drk::psnr (optimize.cpp:145-155)."""
    H, W, Cc = a.shape
    v = C.c_double(0)
    _check(lib().ref_psnr(_p(np.ascontiguousarray(a, dtype=np.float64)), _p(np.ascontiguousarray(b, dtype=np.float64)),
                          W, H, Cc, C.byref(v)))
    return v.value


def densify_and_prune(raw, m, v, k, terms, accum, count, thr, extent):
    """drk::densify_and_prune (optimize.cpp:320-373) on f64 SoA -> (raw, m, v) of the new set."""
    S, n = raw.shape
    cap = 2 * n + 1
    outs = [np.zeros((S, cap)) for _ in range(3)]
    n_out = C.c_longlong(0)
    _check(lib().ref_densify_and_prune(
        _p(np.ascontiguousarray(raw, dtype=np.float64)), _p(np.ascontiguousarray(m, dtype=np.float64)),
        _p(np.ascontiguousarray(v, dtype=np.float64)), n, k, terms, _p(np.ascontiguousarray(accum, dtype=np.float64)),
        _p(np.ascontiguousarray(count, dtype=np.int32)), _p(np.asarray(thr, dtype=np.float64)), C.c_double(extent),
        *[_p(o) for o in outs], C.c_longlong(cap), C.byref(n_out)))
    return tuple(np.ascontiguousarray(o[:, :n_out.value]) for o in outs)


def scene_extent(raw, k, terms):
    """drk::scene_extent (optimize.cpp:375-383)."""
    lib().ref_scene_extent.restype = C.c_double
    return lib().ref_scene_extent(_p(np.ascontiguousarray(raw, dtype=np.float64)), raw.shape[1], k, terms)


def train(raw, k, terms, cams, images, icfg, dcfg):
    """drk::train (optimize.cpp:390-470): icfg = (steps, densify_interval, densify_start,
    densify_stop, sh_warmup, max_sh, eval_interval, seed); dcfg = (lr_drk, lr_position,
    lr_rotation, lr_opacity, lr_sh, densify_grad, prune_opacity, dssim_weight, percent_dense).
    Returns (log [steps, 3] = loss, psnr, count; final_psnr; params f64 [S, n'])."""
    S, n = raw.shape
    steps = int(icfg[0])
    cams_arr = (RefCamera * len(cams))(*[_cam(c) for c in cams])
    imgs = np.concatenate([np.ascontiguousarray(im, dtype=np.float64).ravel() for im in images])
    log = np.zeros((max(steps, 1), 3))
    fin = C.c_double(0)
    cap = n * (2 ** 8) + 16
    out = np.zeros((S, cap))
    n_out = C.c_longlong(0)
    _check(lib().ref_train(_p(np.ascontiguousarray(raw, dtype=np.float64)), n, k, terms, len(cams), cams_arr,
                           _p(imgs), _p(np.asarray(icfg, dtype=np.int32)), _p(np.asarray(dcfg, dtype=np.float64)),
                           _p(log), C.byref(fin), _p(out), C.c_longlong(cap), C.byref(n_out)))
    return log[:steps], fin.value, np.ascontiguousarray(out[:, :n_out.value])


def adam_step(params, grads, m, v, k, terms, step, lrs, steps_total, extent,
              freeze_eta_tau=False, freeze_angles=False):
    """In-place reference adam_step on float64 SoA arrays; returns the new step."""
    st = C.c_int64(step)
    lr = np.asarray(lrs, dtype=np.float64)
    _check(lib().ref_adam_step(_p(params), _p(np.ascontiguousarray(grads, dtype=np.float64)), _p(m),
                               _p(v), params.shape[1], k, terms, C.byref(st), _p(lr), steps_total,
                               C.c_double(extent), int(freeze_eta_tau), int(freeze_angles)))
    return st.value
