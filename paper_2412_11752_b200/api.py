"""Host-side mirror of the reference's render / backward_render interface.

Same names, argument meaning and error behaviour as the reference C++ API
(include/drk/raster.hpp, grad.hpp, optimize.hpp), over the C-ABI of
include/drk_b200.h.  PyTorch supplies device memory and streams; all compute
runs in libdrk_b200.so.  Parameters are the reference's RawDrkParams records
in the ABI's scalar-major SoA layout (``raw[s, i]``, for_each_scalar order,
float32), device-resident between calls.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (DegenerateBasisError, DegenerateQuaternionError, DimensionMismatchError,  # noqa: F401
                   CorruptFileError, DrkError, IoError, NonFiniteError, ReplayMismatchError,
                   VersionMismatchError)
from .scenes import Camera, scalar_count, sh_terms  # noqa: F401


class PresortMode(enum.IntEnum):
    """reference raster.hpp:12"""

    None_ = 0
    CenterDepth = 1
    NearestDepth = 2


@dataclass
class KernelConfig:
    """reference types.hpp:100-105"""

    basis_count: int = 8
    lowpass_radius: float = 0.5
    alpha_min: float = 1.0 / 255.0
    grazing_eps: float = 1e-6


@dataclass
class RenderOptions:
    """reference raster.hpp:81-90 (``threads`` accepted, ignored: deterministic by construction)."""

    kernel: KernelConfig = field(default_factory=KernelConfig)
    background: tuple = (1.0, 1.0, 1.0)
    threads: int = 1
    sh_degree: int = 3
    use_cache: bool = True
    exact_sort: bool = False
    presort: PresortMode = PresortMode.NearestDepth
    early_stop_transmittance: float = 1e-4
    # B200 extension (not in the reference): 0 = fp32 interval forward and
    # backward where eligible (SortCache mode, K = 8), 1 = legacy fp64-depth
    # kernels, 5 = legacy backward only
    raster_kernel: int = 0
    # B200 extension: reference-precision mode (fp64 alpha on every pixel), as the
    # C++ adapter's default; False = fp32 fast path with fp64 fallbacks
    fp64_alpha: bool = False


@dataclass
class FrameBuffers:
    """reference raster.hpp:57-63 (float32 device tensors, H x W x C)."""

    color: torch.Tensor
    depth: torch.Tensor
    normal: torch.Tensor
    alpha: torch.Tensor
    background: tuple = (1.0, 1.0, 1.0)


@dataclass
class TileBinning:
    """reference raster.hpp:19-26 as CSR arrays: tile t holds ids[offsets[t]:offsets[t+1]]."""

    tiles_x: int
    tiles_y: int
    offsets: np.ndarray
    prim_ids: np.ndarray
    keys: np.ndarray
    tile_size: int = 16

    def tile(self, tx: int, ty: int):
        t = ty * self.tiles_x + tx
        s, e = self.offsets[t], self.offsets[t + 1]
        return list(zip(self.prim_ids[s:e].tolist(), self.keys[s:e].tolist()))


@dataclass
class ReplayBuffer:
    """reference raster.hpp:66-79 as CSR arrays; vals columns: u, v, depth, alpha, lowpass_active."""

    width: int
    height: int
    offsets: np.ndarray
    prim_ids: np.ndarray
    vals: np.ndarray

    def at(self, x: int, y: int):
        p = y * self.width + x
        s, e = self.offsets[p], self.offsets[p + 1]
        return [dict(prim_id=int(i), u=v[0], v=v[1], depth=v[2], alpha=v[3], lowpass_active=bool(v[4]))
                for i, v in zip(self.prim_ids[s:e], self.vals[s:e])]


@dataclass
class SortingMetrics:
    """reference raster.hpp:98-103"""

    accuracy: float = 0.0
    kendall_tau: float = 0.0
    mae: float = 0.0
    pixels: int = 0


@dataclass
class FrameGrad:
    """reference grad.hpp:39-45; None = empty image."""

    d_color: torch.Tensor | None = None
    d_depth: torch.Tensor | None = None
    d_normal: torch.Tensor | None = None
    d_alpha: torch.Tensor | None = None


@dataclass
class ParamGrads:
    """reference grad.hpp:48-53 (raw in the SoA layout of the parameters)."""

    raw: torch.Tensor
    d_center_world: torch.Tensor
    screen_grad: torch.Tensor
    touched: torch.Tensor


@dataclass
class TrainConfig:
    """drk::TrainConfig (reference optimize.hpp:30-61), same fields and defaults."""

    steps: int = 35000
    lr_drk: float = 5e-3
    lr_position: float = 1.6e-4
    lr_rotation: float = 1e-3
    lr_opacity: float = 5e-2
    lr_sh: float = 2.5e-3
    densify_grad_threshold: float = 5e-4
    prune_opacity_threshold: float = 5e-2
    densify_interval: int = 100
    densify_start_step: int = 500
    densify_stop_step: int = 15000
    dssim_weight: float = 0.2
    sh_degree_warmup_interval: int = 1000
    max_sh_degree: int = 3
    percent_dense: float = 0.01
    freeze_eta_tau: bool = False
    freeze_angles: bool = False
    seed: int = 0
    threads: int = 1
    background: tuple = (1.0, 1.0, 1.0)
    kernel: "KernelConfig" = None
    eval_interval: int = 250
    checkpoint_interval: int = 0
    checkpoint_path: str = ""


@dataclass
class OptState:
    """reference optimize.hpp:64-70 (SoA moments on the device)."""

    m: torch.Tensor
    v: torch.Tensor
    step: int = 0

    @staticmethod
    def zeros_like(params: torch.Tensor) -> "OptState":
        return OptState(torch.zeros_like(params), torch.zeros_like(params), 0)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _camera(cam: Camera) -> _lib.Camera_:
    c = _lib.Camera_()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    R = np.asarray(cam.R, dtype=np.float64).reshape(9)
    t = np.asarray(cam.t, dtype=np.float64).reshape(3)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = t[i]
    return c


def _options(opt: RenderOptions, replay_cap: int = 0) -> _lib.Options_:
    o = _lib.Options_()
    o.lowpass_radius, o.alpha_min, o.grazing_eps = (opt.kernel.lowpass_radius, opt.kernel.alpha_min,
                                                    opt.kernel.grazing_eps)
    for i in range(3):
        o.background[i] = float(opt.background[i])
    o.early_stop_transmittance = opt.early_stop_transmittance
    o.sh_degree, o.use_cache, o.exact_sort = opt.sh_degree, int(opt.use_cache), int(opt.exact_sort)
    o.presort, o.threads, o.record_replay = int(opt.presort), int(opt.threads), int(replay_cap)
    o.raster_kernel = int(opt.raster_kernel)
    o.fp64_alpha = int(opt.fp64_alpha)
    return o


class Rasterizer:
    """One drk_ctx (device scratch + stream-ordered state of the last forward)."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2412_11752_b200 needs a CUDA device (no CPU fallback)")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           (device.index if isinstance(device, torch.device) else device))
        self.device = dev
        self._h = C.c_void_p()
        _lib.check(_lib.lib().drk_ctx_create(dev.index, C.byref(self._h)))
        self._shape = None

    def close(self):
        if self._h:
            _lib.lib().drk_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        _lib.check(st, self._h)

    def _sync_stream(self):
        _lib.check(_lib.lib().drk_set_stream(self._h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def _raw(self, raw) -> torch.Tensor:
        if isinstance(raw, np.ndarray):
            raw = torch.from_numpy(np.ascontiguousarray(raw, dtype=np.float32))
        return raw.to(self.device, torch.float32).contiguous()

    # --- forward -------------------------------------------------------
    def render(self, raw, cam: Camera, opt: RenderOptions = None, k: int = 8, sh_degree: int | None = None,
               replay: bool | int = False, outputs=("color", "depth", "normal", "alpha")) -> FrameBuffers:
        """drk::render (reference raster.hpp:92-93) from raw parameters (activation included).

        ``replay`` (True or a per-pixel capacity) records the blend lists, read back with
        :meth:`replay_buffer`.
        """
        opt = opt or RenderOptions()
        raw = self._raw(raw)
        S, n = raw.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        if scalar_count(k, terms) != S:
            raise DimensionMismatchError(f"raw has {S} scalars, not scalar_count({k}, terms)")
        H, W = cam.height, cam.width
        kw = dict(device=self.device, dtype=torch.float32)
        fb = FrameBuffers(torch.empty(H, W, 3, **kw) if "color" in outputs else None,
                          torch.empty(H, W, **kw) if "depth" in outputs else None,
                          torch.empty(H, W, 3, **kw) if "normal" in outputs else None,
                          torch.empty(H, W, **kw) if "alpha" in outputs else None, tuple(opt.background))
        cap = (256 if replay is True else int(replay)) if replay else 0
        self._sync_stream()
        self._check(_lib.lib().drk_forward(self._h, _ptr(raw), n, k, terms, C.byref(_camera(cam)),
                                           C.byref(_options(opt, cap)), _ptr(fb.color), _ptr(fb.depth),
                                           _ptr(fb.normal), _ptr(fb.alpha)))
        self._shape = (n, k, terms, H, W)
        return fb

    def render_again(self, cam: Camera, opt: RenderOptions = None,
                     outputs=("color", "depth", "normal", "alpha")) -> FrameBuffers:
        """drk_forward_again: the primitives of the last render on this rasterizer from another
        camera, without re-activating them (multi-view batches; the parameters must be unchanged)."""
        if self._shape is None:
            raise DrkError("render_again without a previous render on this rasterizer")
        opt = opt or RenderOptions()
        n, k, terms, _, _ = self._shape
        H, W = cam.height, cam.width
        kw = dict(device=self.device, dtype=torch.float32)
        fb = FrameBuffers(torch.empty(H, W, 3, **kw) if "color" in outputs else None,
                          torch.empty(H, W, **kw) if "depth" in outputs else None,
                          torch.empty(H, W, 3, **kw) if "normal" in outputs else None,
                          torch.empty(H, W, **kw) if "alpha" in outputs else None, tuple(opt.background))
        self._sync_stream()
        self._check(_lib.lib().drk_forward_again(self._h, C.byref(_camera(cam)), C.byref(_options(opt)),
                                                 _ptr(fb.color), _ptr(fb.depth), _ptr(fb.normal), _ptr(fb.alpha)))
        self._shape = (n, k, terms, H, W)
        return fb

    def render_prims(self, prims: dict, cam: Camera, opt: RenderOptions = None, replay: bool | int = False):
        """drk::render from activated primitives (dict of device tensors: mu [n,3] f64,
        rot [n,3,3] f64, scales/angles [n,K] f64, eta/tau/opacity [n] f64, sh [n,terms,3] f32)."""
        opt = opt or RenderOptions()
        n, k = prims["scales"].shape
        sh = prims["sh"].to(self.device, torch.float32).contiguous()
        # an fp64 SH tensor is also passed as drk_prims.sh64 (fp64 pixel path colours)
        sh64 = prims["sh"].to(self.device).contiguous() if prims["sh"].dtype == torch.float64 else None
        terms = sh.shape[1] if sh.numel() else 0
        keep = {f: prims[f].to(self.device, torch.float64).contiguous()
                for f in ("mu", "rot", "scales", "angles", "eta", "tau", "opacity")}
        p = _lib.Prims_(*[C.c_void_p(keep[f].data_ptr()) for f in
                          ("mu", "rot", "scales", "angles", "eta", "tau", "opacity")], C.c_void_p(sh.data_ptr()),
                        _ptr(sh64))
        H, W = cam.height, cam.width
        kw = dict(device=self.device, dtype=torch.float32)
        fb = FrameBuffers(torch.empty(H, W, 3, **kw), torch.empty(H, W, **kw), torch.empty(H, W, 3, **kw),
                          torch.empty(H, W, **kw), tuple(opt.background))
        cap = (256 if replay is True else int(replay)) if replay else 0
        self._sync_stream()
        self._check(_lib.lib().drk_forward_prims(self._h, C.byref(p), n, k, terms, C.byref(_camera(cam)),
                                                 C.byref(_options(opt, cap)), _ptr(fb.color), _ptr(fb.depth),
                                                 _ptr(fb.normal), _ptr(fb.alpha)))
        self._keep = (keep, sh, sh64)
        self._shape = (n, k, terms, H, W)
        return fb

    def render_host(self, raw_host: np.ndarray, cam: Camera, opt: RenderOptions = None, k: int = 8):
        """Host-buffer entry (drk_forward_host): numpy in, numpy colour/depth/normal/alpha out."""
        opt = opt or RenderOptions()
        raw_host = np.ascontiguousarray(raw_host, dtype=np.float32)
        S, n = raw_host.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        H, W = cam.height, cam.width
        out = dict(color=np.empty((H, W, 3), np.float32), depth=np.empty((H, W), np.float32),
                   normal=np.empty((H, W, 3), np.float32), alpha=np.empty((H, W), np.float32))
        self._check(_lib.lib().drk_forward_host(self._h, raw_host.ctypes.data_as(C.c_void_p), n, k, terms,
                                                C.byref(_camera(cam)), C.byref(_options(opt)),
                                                *[out[f].ctypes.data_as(C.c_void_p) for f in
                                                  ("color", "depth", "normal", "alpha")]))
        self._shape = (n, k, terms, H, W)
        return out

    def render_host_ptrs(self, raw_host: torch.Tensor, outs: dict, cam: Camera, opt: RenderOptions = None,
                         k: int = 8):
        """drk_forward_host with caller-owned (pinned) host tensors: raw [S, n] f32 in,
        outs['color'|'depth'|'normal'|'alpha'] f32 out; ordered on the current torch stream."""
        opt = opt or RenderOptions()
        S, n = raw_host.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        self._sync_stream()
        self._check(_lib.lib().drk_forward_host(self._h, C.c_void_p(raw_host.data_ptr()), n, k, terms,
                                                C.byref(_camera(cam)), C.byref(_options(opt)),
                                                *[_ptr(outs.get(f)) for f in ("color", "depth", "normal", "alpha")]))
        self._shape = (n, k, terms, cam.height, cam.width)

    def tile_binning(self) -> TileBinning:
        """drk::bin_primitives result of the last forward (reference raster.hpp:30-31)."""
        total = C.c_int64(0)
        self._check(_lib.lib().drk_get_tile_lists(self._h, C.byref(total), None, None, None))
        n, k, terms, H, W = self._shape
        tx, ty = (W + 15) // 16, (H + 15) // 16
        off = np.zeros(tx * ty + 1, np.int64)
        ids = np.zeros(total.value, np.int32)
        keys = np.zeros(total.value, np.float64)
        self._check(_lib.lib().drk_get_tile_lists(self._h, C.byref(total), off.ctypes.data_as(C.c_void_p),
                                                  ids.ctypes.data_as(C.c_void_p), keys.ctypes.data_as(C.c_void_p)))
        return TileBinning(tx, ty, off, ids, keys)

    def bin_primitives(self, raw, cam: Camera, cfg: KernelConfig = None,
                       presort: PresortMode = PresortMode.NearestDepth, k: int = 8) -> TileBinning:
        cfg = cfg or KernelConfig()
        opt = RenderOptions(kernel=cfg, presort=presort)
        self.render(raw, cam, opt, k=k, outputs=())
        return self.tile_binning()

    def eval_sorting(self, raw, cam: Camera, cfg: KernelConfig = None, presort=PresortMode.NearestDepth,
                     use_cache: bool = True, k: int = 8) -> "SortingMetrics":
        """drk::eval_sorting (reference raster.cpp:487-560): bins with ``presort`` and
        measures the depth order each pixel would process (SortCache or list order)."""
        cfg = cfg or KernelConfig(basis_count=k)
        opt = RenderOptions(kernel=cfg, presort=presort, use_cache=use_cache, sh_degree=0)
        self.render(raw, cam, opt, k=k)
        out = (C.c_double * 4)()
        self._check(_lib.lib().drk_eval_sorting(self._h, out))
        return SortingMetrics(out[0], out[1], out[2], int(out[3]))

    def replay_buffer(self) -> ReplayBuffer:
        total = C.c_int64(0)
        self._check(_lib.lib().drk_get_replay(self._h, C.byref(total), None, None, None))
        n, k, terms, H, W = self._shape
        off = np.zeros(H * W + 1, np.int64)
        ids = np.zeros(total.value, np.int32)
        vals = np.zeros((total.value, 5), np.float64)
        self._check(_lib.lib().drk_get_replay(self._h, C.byref(total), off.ctypes.data_as(C.c_void_p),
                                              ids.ctypes.data_as(C.c_void_p), vals.ctypes.data_as(C.c_void_p)))
        return ReplayBuffer(W, H, off, ids, vals)

    def alpha_bound_check(self, samples: int = 1 << 22, seed: int = 1):
        """(max error / bound, max abs error) of the fp32 alpha path on the last activated set."""
        r, a = C.c_double(0), C.c_double(0)
        self._check(_lib.lib().drk_debug_alpha_bound(self._h, samples, seed, C.byref(r), C.byref(a)))
        return r.value, a.value

    def stats(self) -> dict:
        s = _lib.Stats_()
        self._check(_lib.lib().drk_get_stats(self._h, C.byref(s)))
        out = {f: getattr(s, f) for f, _ in _lib.Stats_._fields_ if f != "stage_ms"}
        out["stage_ms"] = dict(zip(_lib.STAGES, list(s.stage_ms)))
        return out

    def set_timing(self, enabled: bool = True):
        self._check(_lib.lib().drk_set_timing(self._h, int(enabled)))

    def set_counters(self, enabled: bool = True):
        """drk_set_counters: the fast forward's work counters on, or compiled out (the default)."""
        self._check(_lib.lib().drk_set_counters(self._h, int(enabled)))

    def set_band_limit(self, pairs: int):
        """Force banded binning above `pairs` tile pairs per band (0 = by free device memory)."""
        self._check(_lib.lib().drk_set_band_limit(self._h, int(pairs)))

    def set_det_chunk_limit(self, records: int = 0):
        """Test hook: records per chunk of tile rows in the deterministic backward (0 = memory-based)."""
        self._check(_lib.lib().drk_set_det_chunk_limit(self._h, int(records)))

    def bands(self) -> int:
        v = C.c_int32(0)
        self._check(_lib.lib().drk_get_bands(self._h, C.byref(v)))
        return int(v.value)

    def set_validation(self, enabled: bool = True):
        """Fast forward kernel: check every fp32 alpha against its fp64 value (slow; tests only)."""
        self._check(_lib.lib().drk_set_validation(self._h, int(enabled)))

    def validation(self) -> tuple[float, float]:
        """(max |a32 - a64| / error bound, max |a32 - a64|) since set_validation(True)."""
        v = (C.c_double * 2)()
        self._check(_lib.lib().drk_get_validation(self._h, v))
        return float(v[0]), float(v[1])

    def validation_detail(self) -> list[float]:
        v = (C.c_double * 22)()
        self._check(_lib.lib().drk_get_validation_detail(self._h, v))
        return list(v)

    def fp32_peak_tflops(self) -> float:
        v = C.c_double(0)
        self._check(_lib.lib().drk_measure_fp32_peak(self._h, C.byref(v)))
        return v.value

    # --- backward ------------------------------------------------------
    def backward_render(self, raw, frame_grad: FrameGrad, grad_out: torch.Tensor | None = None,
                        accumulate: bool = False, deterministic: bool = False) -> ParamGrads:
        """drk::backward_render (reference grad.hpp:58-61) for the last forward on this rasterizer."""
        if self._shape is None:
            raise ReplayMismatchError("backward_render without a forward on this rasterizer")
        raw = self._raw(raw)
        n, k, terms, H, W = self._shape
        if raw.shape[1] != n:
            raise ReplayMismatchError("raw and activated primitive counts differ")
        for img, c in ((frame_grad.d_color, 3), (frame_grad.d_depth, 1), (frame_grad.d_normal, 3),
                       (frame_grad.d_alpha, 1)):
            if img is not None and img.numel() != H * W * c:
                raise ReplayMismatchError("frame gradient does not match the camera dimensions")

        def dev(t):
            return None if t is None else t.to(self.device, torch.float32).contiguous()

        fg_t = [dev(frame_grad.d_color), dev(frame_grad.d_depth), dev(frame_grad.d_normal), dev(frame_grad.d_alpha)]
        fg = _lib.FrameGrad_(*[_ptr(t) for t in fg_t])
        g = grad_out if grad_out is not None else torch.zeros_like(raw)
        dcw = torch.empty(n, 3, device=self.device, dtype=torch.float32)
        sg = torch.empty(n, device=self.device, dtype=torch.float32)
        tch = torch.empty(n, device=self.device, dtype=torch.uint8)
        self._sync_stream()
        self._check(_lib.lib().drk_backward(self._h, _ptr(raw), C.byref(fg), _ptr(g), _ptr(dcw), _ptr(sg), _ptr(tch),
                                            int(accumulate), int(deterministic)))
        return ParamGrads(g, dcw, sg, tch)

    # --- loss / optimizer ---------------------------------------------
    def l1_loss(self, rendered: torch.Tensor, target: torch.Tensor):
        """L1 branch of drk::loss (reference optimize.cpp:171-204, dssim_weight = 0)."""
        if rendered.shape != target.shape:
            raise DimensionMismatchError("rendered and target shapes differ")
        H, W = rendered.shape[:2]
        r = rendered.to(self.device, torch.float32).contiguous()
        t = target.to(self.device, torch.float32).contiguous()
        value = torch.empty(1, device=self.device, dtype=torch.float64)
        d = torch.empty_like(r)
        self._sync_stream()
        self._check(_lib.lib().drk_l1_loss(self._h, _ptr(r), _ptr(t), W, H, _ptr(value), _ptr(d)))
        return value, d

    def loss(self, rendered: torch.Tensor, target: torch.Tensor, dssim_weight: float = 0.2):
        """drk::loss (reference optimize.cpp:171-204): (1 - w) L1 + w (1 - mean SSIM) on
        H x W x C images; returns (device f64 [value, l1, mean_ssim], d_color)."""
        if rendered.shape != target.shape:
            raise DimensionMismatchError("image dimensions differ")
        H, W = rendered.shape[:2]
        Cc = rendered.shape[2] if rendered.dim() == 3 else 1
        r = rendered.to(self.device, torch.float32).contiguous()
        t = target.to(self.device, torch.float32).contiguous()
        out = torch.empty(3, device=self.device, dtype=torch.float64)
        d = torch.empty_like(r)
        self._sync_stream()
        self._check(_lib.lib().drk_loss(self._h, _ptr(r), _ptr(t), W, H, Cc, float(dssim_weight), _ptr(out), _ptr(d)))
        return out, d

    def ssim(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        """drk::ssim (reference optimize.cpp:157-166): device f64 scalar tensor."""
        return self._metric(a, b, "drk_ssim", 1)[0]

    def psnr(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        """drk::psnr (reference optimize.cpp:145-155): device f64 scalar tensor."""
        return self._metric(a, b, "drk_psnr", 2)[0]

    def _metric(self, a, b, fn, n_out):
        if a.shape != b.shape:
            raise DimensionMismatchError("image dimensions differ")
        H, W = a.shape[:2]
        Cc = a.shape[2] if a.dim() == 3 else 1
        a = a.to(self.device, torch.float32).contiguous()
        b = b.to(self.device, torch.float32).contiguous()
        out = torch.empty(n_out, device=self.device, dtype=torch.float64)
        self._sync_stream()
        self._check(getattr(_lib.lib(), fn)(self._h, _ptr(a), _ptr(b), W, H, Cc, _ptr(out)))
        return out

    def psnr_quantized(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        """psnr(quantize_8bit(a), b) (reference image.cpp:7-14, optimize.cpp:432)."""
        return self._metric(a, b, "drk_psnr_quantized", 2)[0]

    # --- density control (reference optimize.cpp:309-383) ----------------------
    def scene_extent(self, params: torch.Tensor) -> float:
        out = torch.empty(1, device=self.device, dtype=torch.float64)
        self._sync_stream()
        self._check(_lib.lib().drk_scene_extent(self._h, _ptr(params), params.shape[1], _ptr(out)))
        return float(out)

    def densify_accumulate(self, grads: "ParamGrads", stats: "DensifyStats"):
        """DensifyStats::accumulate (optimize.cpp:309-318) on the device."""
        n = grads.screen_grad.numel()
        if stats.screen_grad_accum.numel() != n:
            raise DimensionMismatchError("densify stats out of sync with the primitive set")
        self._sync_stream()
        self._check(_lib.lib().drk_densify_accumulate(self._h, _ptr(grads.screen_grad), _ptr(grads.touched), n,
                                                      _ptr(stats.screen_grad_accum), _ptr(stats.touch_count)))

    def densify_and_prune(self, params: torch.Tensor, state: "OptState", stats: "DensifyStats", cfg: TrainConfig,
                          extent: float, k: int = 8):
        """densify_and_prune (optimize.cpp:320-373): returns the new params; state's moments follow."""
        S, n = params.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        dc = _lib.DensifyConfig_(cfg.densify_grad_threshold, cfg.prune_opacity_threshold, cfg.percent_dense)
        cap = 2 * n
        outs = [torch.empty(S, max(cap, 1), device=self.device, dtype=torch.float32) for _ in range(3)]
        n_out = C.c_int64(0)
        self._sync_stream()
        self._check(_lib.lib().drk_densify_and_prune(
            self._h, _ptr(params), _ptr(state.m), _ptr(state.v), n, k, terms, _ptr(stats.screen_grad_accum),
            _ptr(stats.touch_count), C.byref(dc), float(extent), *[_ptr(o) for o in outs], cap, C.byref(n_out)))
        m = n_out.value
        p, state.m, state.v = (o[:, :m].contiguous() for o in outs)
        return p

    # --- Mesh2DRK (reference mesh.cpp) ------------------------------------------
    def mesh_convert(self, mesh: "MeshData", basis_count: int = 8):
        """convert (reference mesh.cpp:326-343) on the device -> (raw f32 [S, n], n_skipped):
        one DRK per face, degenerate faces skipped in order, SH degree 0."""
        dev = self.device
        v = torch.from_numpy(np.ascontiguousarray(mesh.vertices, np.float64)).to(dev)
        o = torch.from_numpy(np.ascontiguousarray(mesh.face_offsets, np.int32)).to(dev)
        i = torch.from_numpy(np.ascontiguousarray(mesh.indices, np.int32)).to(dev)
        c = torch.from_numpy(np.ascontiguousarray(mesh.colors, np.float64)).to(dev)
        nf = len(mesh.face_offsets) - 1
        raw = torch.empty(scalar_count(basis_count, 1), max(nf, 1), device=dev, dtype=torch.float32)
        n_out, n_skip = C.c_int64(0), C.c_int64(0)
        self._sync_stream()
        self._check(_lib.lib().drk_mesh_convert(self._h, _ptr(v), len(mesh.vertices), _ptr(o), _ptr(i), _ptr(c), nf,
                                                basis_count, _ptr(raw), raw.shape[1], C.byref(n_out),
                                                C.byref(n_skip)))
        return raw[:, :n_out.value].contiguous(), n_skip.value

    def shade_lambert(self, raw: torch.Tensor, light_dir, ambient: float, basis_count: int = 8):
        """shade_lambert (reference mesh.cpp:345-357), in place on device raw parameters."""
        lt = (C.c_double * 3)(*[float(x) for x in light_dir])
        self._sync_stream()
        self._check(_lib.lib().drk_shade_lambert(self._h, _ptr(raw), raw.shape[1], basis_count, lt, float(ambient)))

    # --- scene files (DRKSCENE v1) -------------------------------------------
    def load_scene(self, path: str, expected_basis_count: int = -1) -> "DeviceScene":
        """drk::load_scene (reference io.cpp:58-97) straight to a device tensor in the
        C-ABI raw layout f32 [scalar_count, n]; raises IoError / CorruptFileError /
        VersionMismatchError like the reference."""
        h = read_scene_header(path, expected_basis_count)
        params = torch.empty(h.scalar_count, h.count, device=self.device, dtype=torch.float32)
        out = _lib.SceneHeader_()
        self._sync_stream()
        self._check(_lib.lib().drk_scene_load(self._h, os.fsencode(path), int(expected_basis_count), _ptr(params),
                                              h.count, C.byref(out)))
        return DeviceScene(out.basis_count, out.sh_degree, params)

    def save_scene(self, scene: "DeviceScene", path: str):
        """drk::save_scene (reference io.cpp:40-56) from device raw parameters."""
        raw = self._raw(scene.params)
        S, n = raw.shape
        if S != scalar_count(scene.basis_count, sh_terms(scene.sh_degree)):
            raise DimensionMismatchError("primitive layout differs from the scene header")
        self._sync_stream()
        self._check(_lib.lib().drk_scene_save(self._h, os.fsencode(path), _ptr(raw), n, scene.basis_count,
                                              scene.sh_degree))

    def adam_step(self, params: torch.Tensor, grads: torch.Tensor, state: OptState, cfg: TrainConfig,
                  scene_extent: float, k: int = 8, grad_scale: float = 1.0):
        """drk::adam_step (reference optimize.cpp:259-307), in place on device tensors."""
        if params.shape != grads.shape or params.shape != state.m.shape:
            raise DimensionMismatchError("optimizer shapes out of sync")
        S, n = params.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        a = _lib.AdamConfig_(cfg.lr_drk, cfg.lr_position, cfg.lr_rotation, cfg.lr_opacity, cfg.lr_sh, cfg.steps,
                             int(cfg.freeze_eta_tau), int(cfg.freeze_angles), 0, float(scene_extent),
                             float(grad_scale))
        step = C.c_int64(state.step)
        self._sync_stream()
        self._check(_lib.lib().drk_adam_step(self._h, _ptr(params), _ptr(grads), _ptr(state.m), _ptr(state.v), n, k,
                                             terms, C.byref(step), C.byref(a)))
        state.step = step.value

    def allreduce_adam(self, comm, params: torch.Tensor, grads: torch.Tensor, state: OptState, cfg: TrainConfig,
                       scene_extent: float, grad_scale: float, k: int = 8):
        """drk_allreduce_adam: gradients summed across the communicator's ranks
        (reduce-scatter), Adam on this rank's shard (gradients x grad_scale, e.g.
        1 / total views), parameters all-gathered; in place, every rank equal."""
        if params.shape != grads.shape or params.shape != state.m.shape:
            raise DimensionMismatchError("optimizer shapes out of sync")
        S, n = params.shape
        terms = (S - (3 + 4 + 2 * k + 3)) // 3
        a = _lib.AdamConfig_(cfg.lr_drk, cfg.lr_position, cfg.lr_rotation, cfg.lr_opacity, cfg.lr_sh, cfg.steps,
                             int(cfg.freeze_eta_tau), int(cfg.freeze_angles), 0, float(scene_extent),
                             float(grad_scale))
        step = C.c_int64(state.step)
        self._sync_stream()
        self._check(_lib.lib().drk_allreduce_adam(self._h, comm.handle, _ptr(params), _ptr(grads), _ptr(state.m),
                                                  _ptr(state.v), n, k, terms, C.byref(step), C.byref(a)))
        state.step = step.value


@dataclass
class DensifyStats:
    """drk::DensifyStats (reference optimize.hpp:78-88) on the device."""

    screen_grad_accum: torch.Tensor  # f64 [n]
    touch_count: torch.Tensor        # i32 [n]

    @staticmethod
    def zeros(n: int, device) -> "DensifyStats":
        return DensifyStats(torch.zeros(n, device=device, dtype=torch.float64),
                            torch.zeros(n, device=device, dtype=torch.int32))


@dataclass
class MeshData:
    """drk::Mesh (reference mesh.hpp:10-18) as host arrays: faces in CSR form."""

    vertices: np.ndarray      # f64 [nv, 3]
    face_offsets: np.ndarray  # i32 [nf + 1]
    indices: np.ndarray       # i32 (0-based)
    colors: np.ndarray        # f64 [nf, 3]
    warnings: int = 0


def load_mesh(path: str) -> MeshData:
    """load_mesh (reference mesh.cpp:134-217) through the C-ABI (host code)."""
    h = C.c_void_p()
    L = _lib.lib()
    st = L.drk_mesh_load(os.fsencode(path), C.byref(h))
    try:
        if st:
            raise _lib._ERRORS.get(st, DrkError)(L.drk_mesh_error(h).decode())
        nv, nf, ni, nw = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        L.drk_mesh_info(h, C.byref(nv), C.byref(nf), C.byref(ni), C.byref(nw))
        m = MeshData(np.zeros((nv.value, 3)), np.zeros(nf.value + 1, np.int32), np.zeros(ni.value, np.int32),
                     np.zeros((nf.value, 3)), nw.value)
        L.drk_mesh_arrays(h, m.vertices.ctypes.data, m.face_offsets.ctypes.data, m.indices.ctypes.data,
                          m.colors.ctypes.data)
        return m
    finally:
        L.drk_mesh_free(h)


@dataclass
class DeviceScene:
    """drk::Scene (reference io.hpp:14-18) with the records on the device, C-ABI raw layout."""

    basis_count: int
    sh_degree: int
    params: torch.Tensor  # f32 [scalar_count(K, terms), n]


def read_scene_header(path: str, expected_basis_count: int = -1) -> _lib.SceneHeader_:
    """Header checks of drk::load_scene (io.cpp:58-80) through the C-ABI; no device work."""
    h = _lib.SceneHeader_()
    _lib.check(_lib.lib().drk_scene_read_header(os.fsencode(path), int(expected_basis_count), C.byref(h)))
    return h


def load_scene(path: str, expected_basis_count: int = -1) -> DeviceScene:
    return default_rasterizer().load_scene(path, expected_basis_count)


def save_scene(scene: DeviceScene, path: str):
    default_rasterizer().save_scene(scene, path)


_default: dict[int, Rasterizer] = {}


def default_rasterizer(device: int | None = None) -> Rasterizer:
    idx = torch.cuda.current_device() if device is None else device
    if idx not in _default:
        _default[idx] = Rasterizer(idx)
    return _default[idx]


def render(raw, cam: Camera, opt: RenderOptions = None, k: int = 8, replay: bool | int = False) -> FrameBuffers:
    return default_rasterizer().render(raw, cam, opt, k=k, replay=replay)


def bin_primitives(raw, cam: Camera, cfg: KernelConfig = None, presort=PresortMode.NearestDepth, k: int = 8):
    return default_rasterizer().bin_primitives(raw, cam, cfg, presort, k=k)


def backward_render(raw, frame_grad: FrameGrad, **kw) -> ParamGrads:
    return default_rasterizer().backward_render(raw, frame_grad, **kw)
