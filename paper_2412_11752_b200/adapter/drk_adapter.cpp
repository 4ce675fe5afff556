// Drop-in adapter: the reference's C++ API (include/drk/raster.hpp,
// include/drk/grad.hpp) implemented on top of the C-ABI of include/drk_b200.h.
//
// A maintainer of the reference replaces three functions by linking this
// translation unit:
//   drk::bin_primitives   (reference raster.hpp:30-31, raster.cpp:119-265)
//   drk::render           (reference raster.hpp:92-93, raster.cpp:440-485)
//   drk::backward_render  (reference grad.hpp:58-61, grad.cpp:307-384)
//   drk::eval_sorting     (reference raster.hpp:105-106, raster.cpp:487-560)
// and the image losses of the training step:
//   drk::loss / drk::ssim / drk::psnr (reference optimize.hpp:6-18,
//   optimize.cpp:145-204) on the device (double images: drk_loss_f64 ...)
// Everything else (SortCache, eval_sorting, backward_alpha,
// finite_diff_check, ...) stays the reference's and calls into these.
//
// Conversions: std::vector<DrkPrimitive> -> activated SoA on the device
// (fp64 centre / rotation / shape, f32 SH); Image (double) <- f32 planes;
// ReplayBuffer <- drk_get_replay; ParamGrads <- f32 SoA gradients.  Status
// codes become the matching drk::Error subclasses.  The backward is always the
// deterministic (fixed-order, parallel) reduction: the reference's contract is
// bitwise equality across thread counts (grad.hpp:55-57).
// Precision: by default the adapter asks for the GPU path's reference-precision
// mode (fp64 alpha everywhere), so that cache-sorted and exact-sort renders are
// bitwise comparable as the reference's raster suite requires
// (test_raster.cpp:199-220); DRK_ADAPTER_PRECISION=fast selects the fp32 fast
// kernels (the benchmarked path; every decision still the reference's).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "drk/errors.hpp"
#include "drk/grad.hpp"
#include "drk/optimize.hpp"
#include "drk/raster.hpp"
#include "drk_b200.h"

namespace {

struct Context {
  drk_ctx* c = nullptr;
  Context() {
    if (drk_ctx_create(0, &c) != DRK_OK) throw drk::Error("drk_b200: no CUDA device");
  }
  ~Context() { drk_ctx_destroy(c); }
};

drk_ctx* ctx() {
  static Context g;
  return g.c;
}

[[noreturn]] void raise(int st) {
  const std::string m = std::string(drk_status_string(st)) + ": " + drk_last_error(ctx());
  switch (st) {
    case DRK_ERR_NONFINITE: throw drk::NonFiniteError(m);
    case DRK_ERR_DEGENERATE_QUAT: throw drk::DegenerateQuaternionError(m);
    case DRK_ERR_DEGENERATE_BASIS: throw drk::DegenerateBasisError(m);
    case DRK_ERR_REPLAY_MISMATCH: throw drk::ReplayMismatchError(m);
    case DRK_ERR_DIMENSION: throw drk::DimensionMismatchError(m);
    default: throw drk::Error(m);
  }
}

void check(int st) {
  if (st != DRK_OK) raise(st);
}

// Grow-only device scratch, one slot per argument role: the reference API is
// called once per training step / finite-difference probe, so per-call
// cudaMalloc / cudaFree (an implicit device synchronisation each) would dominate
// small renders.
void* slot_bytes(int slot, size_t bytes) {
  struct Slot {
    void* p = nullptr;
    size_t bytes = 0;
  };
  static Slot slots[32];
  Slot& s = slots[slot];
  if (s.bytes < bytes) {
    if (s.p) cudaFree(s.p);
    s.p = nullptr;
    const size_t want = bytes + bytes / 4;
    if (cudaMalloc(&s.p, want) != cudaSuccess) throw drk::Error("drk_b200: cudaMalloc");
    s.bytes = want;
  }
  return s.p;
}

enum Slots { kMu, kRot, kS, kTh, kEta, kTau, kO, kSh, kColor, kDepth, kNormal, kAlpha, kRaw, kDC, kDD, kDN, kDA,
             kG, kDcw, kSg, kTch, kLossA, kLossB, kLossOut, kLossD, kSh64 };

// Grow-only page-locked host staging, one slot per role: the conversions write
// into memory that is already mapped (no first-touch page faults per call) and
// the copies run at full link speed.
enum HostSlots { kHMu, kHRot, kHS, kHTh, kHEta, kHTau, kHO, kHSh, kHSh64, kHRaw, kHG, kHDcw, kHSg, kHTch, kHostSlots };
template <class T>
T* pinned(int slot, size_t count) {
  struct Slot {
    void* p = nullptr;
    size_t bytes = 0;
  };
  static Slot slots[kHostSlots];
  Slot& s = slots[slot];
  const size_t bytes = sizeof(T) * (count ? count : 1);
  if (s.bytes < bytes) {
    if (s.p) cudaFreeHost(s.p);
    s.p = nullptr;
    const size_t want = bytes + bytes / 4;
    if (cudaHostAlloc(&s.p, want, cudaHostAllocDefault) != cudaSuccess) throw drk::Error("drk_b200: cudaHostAlloc");
    s.bytes = want;
  }
  return static_cast<T*>(s.p);
}

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  Dev(int slot, size_t count) : p(static_cast<T*>(slot_bytes(slot, sizeof(T) * (count ? count : 1)))), n(count) {}
  Dev(int slot, const T* h, size_t count) : Dev(slot, count) {
    if (count) cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice);
  }
  Dev(int slot, const std::vector<T>& h) : Dev(slot, h.data(), h.size()) {}
  std::vector<T> get() const {
    std::vector<T> h(n);
    if (n) cudaMemcpy(h.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
  }
  const T* get_pinned(int host_slot) const {  // into page-locked staging
    T* h = pinned<T>(host_slot, n);
    if (n) cudaMemcpy(h, p, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
  }
};

// Fingerprint of the host inputs of a forward (64-bit words, multiply-xorshift): the
// backward reuses the device state of the last forward when it saw the same
// primitives, camera and options — the reference's render(&replay) ->
// backward_render sequence — instead of uploading and rendering again.
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void mix(uint64_t w) {
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  }
  void add(const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, b + i, 8);
      mix(w);
    }
    uint64_t tail = n;
    for (; i < n; ++i) tail = (tail << 8) | b[i];
    mix(tail);
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    add(v.data(), v.size() * sizeof(T));
  }
};
uint64_t g_last_forward = 0;  // fingerprint of the context's last forward (0: none)

// Host loops over the primitives / pixels on all cores (the reference API hands
// over host std::vectors; their conversion would otherwise dominate a call).
template <class F>
void parallel_for(size_t n, F f, size_t serial_below = 8192) {
  static const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const unsigned T = n < serial_below ? 1u : (unsigned)std::min<size_t>(hw, n);
  if (T == 1) {
    f(size_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  const size_t chunk = (n + T - 1) / T;
  for (unsigned t = 0; t < T; ++t) {
    const size_t b = t * chunk, e = std::min(n, b + chunk);
    if (b < e) th.emplace_back([=, &f] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// Activated primitives on the device (drk_prims).  One parallel pass fills the
// SoA fields and fingerprints them in blocks of kHashBlock primitives (the block
// hashes combined in order: independent of the thread count).
struct DevPrims {
  static constexpr size_t kHashBlock = 4096;
  int n, k, terms;
  DevPrims(const std::vector<drk::DrkPrimitive>& P, int k_default)
      : n((int)P.size()), k(P.empty() ? k_default : P[0].basis_count()), terms(0) {
    for (const auto& p : P) {
      terms = std::max<int>(terms, (int)p.sh.rows());
      if (p.basis_count() != k) throw drk::DimensionMismatchError("drk_b200 adapter: mixed basis counts");
    }
    const size_t N = P.size(), T3 = 3 * (size_t)terms;
    nmu = 3 * N;
    nrot = 9 * N;
    nk = (size_t)k * N;
    nsh = T3 * N;
    hmu = pinned<double>(kHMu, nmu);
    hrot = pinned<double>(kHRot, nrot);
    hs = pinned<double>(kHS, nk);
    hth = pinned<double>(kHTh, nk);
    heta = pinned<double>(kHEta, N);
    htau = pinned<double>(kHTau, N);
    ho = pinned<double>(kHO, N);
    hsh = pinned<float>(kHSh, nsh);
    hsh64 = pinned<double>(kHSh64, nsh);
    const size_t nblk = (N + kHashBlock - 1) / kHashBlock;
    std::vector<uint64_t> bh(nblk);
    parallel_for(nblk, [&](size_t b0, size_t b1) {
      for (size_t blk = b0; blk < b1; ++blk) {
        const size_t i0 = blk * kHashBlock, i1 = std::min(N, i0 + kHashBlock);
        for (size_t i = i0; i < i1; ++i) {
          const auto& p = P[i];
          for (int a = 0; a < 3; ++a) hmu[3 * i + a] = p.center[a];
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) hrot[9 * i + 3 * r + c] = p.rot(r, c);
          for (int j = 0; j < k; ++j) {
            hs[(size_t)k * i + j] = p.scales[j];
            hth[(size_t)k * i + j] = p.angles[j];
          }
          heta[i] = p.eta;
          htau[i] = p.tau;
          ho[i] = p.opacity;
          for (int t = 0; t < terms; ++t)
            for (int c = 0; c < 3; ++c) {
              const double v = t < p.sh.rows() ? p.sh(t, c) : 0.0;
              hsh64[T3 * i + 3 * t + c] = v;
              hsh[T3 * i + 3 * t + c] = (float)v;
            }
        }
        Fnv f;
        const size_t m = i1 - i0;
        f.add(hmu + 3 * i0, 8 * 3 * m);
        f.add(hrot + 9 * i0, 8 * 9 * m);
        f.add(hs + (size_t)k * i0, 8 * (size_t)k * m);
        f.add(hth + (size_t)k * i0, 8 * (size_t)k * m);
        f.add(heta + i0, 8 * m);
        f.add(htau + i0, 8 * m);
        f.add(ho + i0, 8 * m);
        f.add(hsh64 + T3 * i0, 8 * T3 * m);
        bh[blk] = f.h;
      }
    }, 2);
    Fnv f;
    f.add(&n, sizeof n);
    f.add(&k, sizeof k);
    f.add(&terms, sizeof terms);
    f.vec(bh);
    hash = f.h;
  }
  // device copies (only when a forward must run)
  void upload() {
    const size_t N = (size_t)n;
    Dev<double> mu(kMu, hmu, nmu), rot(kRot, hrot, nrot), s(kS, hs, nk), th(kTh, hth, nk), eta(kEta, heta, N),
        tau(kTau, htau, N), o(kO, ho, N);
    Dev<float> sh(kSh, hsh, nsh);
    Dev<double> sh64(kSh64, hsh64, nsh);  // the fp64 pixel path's colours use the reference's coefficients exactly
    view = drk_prims{mu.p, rot.p, s.p, th.p, eta.p, tau.p, o.p, sh.p, sh64.p};
  }
  // page-locked host copies (adapter staging slots: valid until the next conversion)
  double *hmu, *hrot, *hs, *hth, *heta, *htau, *ho;
  float* hsh;
  double* hsh64;
  size_t nmu, nrot, nk, nsh;
  drk_prims view{};
  uint64_t hash = 0;
};

drk_camera to_cam(const drk::Camera& c) {
  drk_camera d;
  std::memset(&d, 0, sizeof d);  // padding too: the struct is fingerprinted
  d.fx = c.fx;
  d.fy = c.fy;
  d.cx = c.cx;
  d.cy = c.cy;
  d.width = c.width;
  d.height = c.height;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) d.R[3 * r + k] = c.world_to_cam_rot(r, k);
  for (int r = 0; r < 3; ++r) d.t[r] = c.world_to_cam_trans[r];
  return d;
}

// DRK_ADAPTER_TRACE=1: wall time of every adapter call on stderr.
struct Trace {
  const char* what;
  int w, h, n;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  std::string phases;
  Trace(const char* what_, int w_, int h_, int n_) : what(what_), w(w_), h(h_), n(n_) {}
  static bool on() {
    static const bool e = std::getenv("DRK_ADAPTER_TRACE") != nullptr;
    return e;
  }
  void at(const char* phase) {  // checkpoint: time since the previous one
    if (!on()) return;
    const auto now = std::chrono::steady_clock::now();
    char b[64];
    std::snprintf(b, sizeof b, " %s %.2f", phase, std::chrono::duration<double, std::milli>(now - last).count());
    phases += b;
    last = now;
  }
  ~Trace() {
    if (on())
      std::fprintf(stderr, "[drk adapter] %s %dx%d n=%d: %.3f ms |%s\n", what, w, h, n,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
                   phases.c_str());
  }
};

bool fast_precision() {
  static const bool fast = [] {
    const char* e = std::getenv("DRK_ADAPTER_PRECISION");
    return e && std::strcmp(e, "fast") == 0;
  }();
  return fast;
}

drk_options to_opt(const drk::RenderOptions& o, int replay_cap) {
  drk_options d;
  std::memset(&d, 0, sizeof d);
  drk_default_options(&d);
  d.lowpass_radius = o.kernel.lowpass_radius;
  d.alpha_min = o.kernel.alpha_min;
  d.grazing_eps = o.kernel.grazing_eps;
  for (int i = 0; i < 3; ++i) d.background[i] = o.background[i];
  d.early_stop_transmittance = o.early_stop_transmittance;
  d.sh_degree = o.sh_degree;
  d.use_cache = o.use_cache ? 1 : 0;
  d.exact_sort = o.exact_sort ? 1 : 0;
  d.presort = static_cast<int>(o.presort);
  d.threads = o.threads;
  d.record_replay = replay_cap;
  d.fp64_alpha = fast_precision() ? 0 : 1;
  return d;
}

uint64_t forward_hash(const DevPrims& dp, const drk_camera& c, const drk_options& o) {
  drk_options oo = o;
  oo.record_replay = 0;  // the backward does not depend on the replay capacity
  Fnv f;
  f.add(&dp.hash, sizeof dp.hash);
  f.add(&c, sizeof c);
  f.add(&oo, sizeof oo);
  return f.h | 1;
}

void forward(const std::vector<drk::DrkPrimitive>& prims, const drk::Camera& cam, const drk::RenderOptions& opt,
             int replay_cap, float* color, float* depth, float* normal, float* alpha, DevPrims& dp) {
  (void)prims;
  const drk_camera c = to_cam(cam);
  const drk_options o = to_opt(opt, replay_cap);
  g_last_forward = 0;
  dp.upload();
  check(drk_forward_prims(ctx(), &dp.view, dp.n, dp.k, dp.terms, &c, &o, color, depth, normal, alpha));
  g_last_forward = forward_hash(dp, c, o);
}

}  // namespace

namespace drk {

TileBinning bin_primitives(const std::vector<DrkPrimitive>& prims, const Camera& cam, const KernelConfig& cfg,
                           PresortMode presort) {
  DevPrims dp(prims, cfg.basis_count);
  RenderOptions opt;
  opt.kernel = cfg;
  opt.presort = presort;
  forward(prims, cam, opt, 0, nullptr, nullptr, nullptr, nullptr, dp);
  TileBinning b;
  b.tiles_x = (cam.width + b.tile_size - 1) / b.tile_size;
  b.tiles_y = (cam.height + b.tile_size - 1) / b.tile_size;
  b.tiles.assign((size_t)b.tiles_x * b.tiles_y, {});
  int64_t total = 0;
  check(drk_get_tile_lists(ctx(), &total, nullptr, nullptr, nullptr));
  std::vector<int64_t> off(b.tiles.size() + 1);
  std::vector<int32_t> ids(total);
  std::vector<double> keys(total);
  check(drk_get_tile_lists(ctx(), &total, off.data(), ids.data(), keys.data()));
  for (size_t t = 0; t < b.tiles.size(); ++t)
    for (int64_t j = off[t]; j < off[t + 1]; ++j) b.tiles[t].push_back({ids[j], keys[j]});
  return b;
}

// drk::eval_sorting (raster.hpp:105-106): GPU binning + per-pixel order metrics
SortingMetrics eval_sorting(const std::vector<DrkPrimitive>& prims, const Camera& cam, const KernelConfig& cfg,
                            PresortMode presort, bool use_cache) {
  DevPrims dp(prims, cfg.basis_count);
  RenderOptions opt;
  opt.kernel = cfg;
  opt.presort = presort;
  opt.use_cache = use_cache;
  forward(prims, cam, opt, 0, nullptr, nullptr, nullptr, nullptr, dp);
  double out[4];
  check(drk_eval_sorting(ctx(), out));
  SortingMetrics m;
  m.accuracy = out[0];
  m.kendall_tau = out[1];
  m.mae = out[2];
  m.pixels = (long)out[3];
  return m;
}

FrameBuffers render(const std::vector<DrkPrimitive>& prims, const Camera& cam, const RenderOptions& opt,
                    ReplayBuffer* replay) {
  Trace tr{replay ? "render(replay)" : "render", cam.width, cam.height, (int)prims.size()};
  DevPrims dp(prims, opt.kernel.basis_count);
  tr.at("convert+hash");
  const size_t npx = (size_t)cam.width * cam.height;
  Dev<float> color(kColor, 3 * npx), depth(kDepth, npx), normal(kNormal, 3 * npx), alpha(kAlpha, npx);
  forward(prims, cam, opt, replay ? 1024 : 0, color.p, depth.p, normal.p, alpha.p, dp);
  tr.at("upload+forward");
  FrameBuffers fb;
  fb.color = Image(cam.width, cam.height, 3);
  fb.depth = Image(cam.width, cam.height, 1);
  fb.normal = Image(cam.width, cam.height, 3);
  fb.alpha = Image(cam.width, cam.height, 1);
  tr.at("images");
  // the rasterizer's fp64 accumulators (the f32 planes above are their rounding)
  check(drk_get_framebuffers_f64(ctx(), fb.color.data.data(), fb.depth.data.data(), fb.normal.data.data(),
                                 fb.alpha.data.data()));
  tr.at("framebuffers_f64");
  fb.background = opt.background;
  if (replay) {
    replay->width = cam.width;
    replay->height = cam.height;
    replay->pixels.assign(npx, {});
    int64_t total = 0;
    check(drk_get_replay(ctx(), &total, nullptr, nullptr, nullptr));
    std::vector<int64_t> off(npx + 1);
    std::vector<int32_t> ids(total);
    std::vector<double> vals(5 * total);
    check(drk_get_replay(ctx(), &total, off.data(), ids.data(), vals.data()));
    for (size_t p = 0; p < npx; ++p)
      for (int64_t j = off[p]; j < off[p + 1]; ++j) {
        BlendRecord r;
        r.prim_id = ids[j];
        r.u = vals[5 * j];
        r.v = vals[5 * j + 1];
        r.depth = vals[5 * j + 2];
        r.alpha = vals[5 * j + 3];
        r.lowpass_active = vals[5 * j + 4] != 0.0;
        replay->pixels[p].push_back(r);
      }
  }
  return fb;
}

ParamGrads backward_render(const std::vector<RawDrkParams>& raws, const std::vector<DrkPrimitive>& prims,
                           const Camera& cam, const RenderOptions& opt, const ReplayBuffer& replay,
                           const FrameGrad& frame_grad) {
  Trace tr{"backward_render", cam.width, cam.height, (int)prims.size()};
  if (replay.width != cam.width || replay.height != cam.height)
    throw ReplayMismatchError("replay buffer does not match the camera dimensions");
  if (raws.size() != prims.size()) throw ReplayMismatchError("raw and activated primitive counts differ");
  DevPrims dp(prims, opt.kernel.basis_count);
  tr.at("convert+hash");
  // the device keeps the decisions of the forward in place of the ReplayBuffer:
  // the last forward's when it rendered these primitives with this camera and
  // these options (render(&replay) -> backward_render), else a fresh one
  if (g_last_forward != forward_hash(dp, to_cam(cam), to_opt(opt, 0)))
    forward(prims, cam, opt, 0, nullptr, nullptr, nullptr, nullptr, dp);
  tr.at("reforward?");
  const int n = dp.n, k = dp.k, terms = dp.terms;
  const int S = drk_scalar_count(k, terms);
  float* raw_soa = pinned<float>(kHRaw, (size_t)S * n);
  parallel_for((size_t)n, [&](size_t i0, size_t i1) {
    for (int q = 0; q < S; ++q) std::memset(raw_soa + (size_t)q * n + i0, 0, sizeof(float) * (i1 - i0));
    for (size_t i = i0; i < i1; ++i) {
      int s = 0;
      for_each_scalar(raws[i], [&](const double& x, ParamClass) {
        if (s < S) raw_soa[(size_t)s * n + i] = (float)x;
        ++s;
      });
    }
  });
  tr.at("raw_soa");
  Dev<float> raw_d(kRaw, raw_soa, (size_t)S * n);
  auto img = [&](const Image& im, int ch) -> std::vector<float> {
    if (im.empty()) return {};
    if (im.width != cam.width || im.height != cam.height || im.channels != ch)
      throw DimensionMismatchError("frame gradient shape");
    return std::vector<float>(im.data.begin(), im.data.end());
  };
  const std::vector<float> hc = img(frame_grad.d_color, 3), hd = img(frame_grad.d_depth, 1),
                           hn = img(frame_grad.d_normal, 3), ha = img(frame_grad.d_alpha, 1);
  Dev<float> dc(kDC, hc), dd(kDD, hd), dn(kDN, hn), da(kDA, ha);
  drk_frame_grad fg{hc.empty() ? nullptr : dc.p, hd.empty() ? nullptr : dd.p, hn.empty() ? nullptr : dn.p,
                    ha.empty() ? nullptr : da.p};
  Dev<float> g(kG, (size_t)S * n), dcw(kDcw, 3 * (size_t)n), sg(kSg, n);
  Dev<uint8_t> tch(kTch, n);
  tr.at("uploads");
  check(drk_backward(ctx(), raw_d.p, &fg, g.p, dcw.p, sg.p, tch.p, 0, /*deterministic=*/1));
  tr.at("backward");
  const float *gh = g.get_pinned(kHG), *dcwh = dcw.get_pinned(kHDcw), *sgh = sg.get_pinned(kHSg);
  const uint8_t* th = tch.get_pinned(kHTch);
  tr.at("downloads");
  ParamGrads out;
  out.raw.resize(n);
  out.d_center_world.resize(n);
  out.screen_grad.assign(n, 0.0);
  out.touched.assign(n, 0);
  parallel_for((size_t)n, [&](size_t i0, size_t i1) {
    for (size_t i = i0; i < i1; ++i) {
      RawDrkParams r = RawDrkParams::zeros_like(raws[i]);
      int s = 0;
      for_each_scalar(r, [&](double& x, ParamClass) {
        if (s < S) x = gh[(size_t)s * n + i];
        ++s;
      });
      out.raw[i] = std::move(r);
      out.d_center_world[i] = Vec3(dcwh[3 * i], dcwh[3 * i + 1], dcwh[3 * i + 2]);
      out.screen_grad[i] = sgh[i];
      out.touched[i] = (char)th[i];
    }
  });
  tr.at("param_grads");
  return out;
}

// --- image losses (optimize.cpp:145-204) ------------------------------------
namespace {
void same_shape(const Image& a, const Image& b) {
  if (!a.same_shape(b)) throw DimensionMismatchError("image dimensions differ");  // optimize.cpp:19-21
}
// the loss kernels run asynchronously on the context's stream
void done(int st) {
  check(st);
  if (cudaDeviceSynchronize() != cudaSuccess) throw Error("drk_b200: CUDA error in the loss kernels");
}
}  // namespace

double psnr(const Image& a, const Image& b) {
  same_shape(a, b);
  Dev<double> da(kLossA, a.data), db(kLossB, b.data), out(kLossOut, 2);
  done(drk_psnr_f64(ctx(), da.p, db.p, a.width, a.height, a.channels, out.p));
  return out.get()[0];
}

double ssim(const Image& a, const Image& b) {
  same_shape(a, b);
  Dev<double> da(kLossA, a.data), db(kLossB, b.data), out(kLossOut, 1);
  done(drk_ssim_f64(ctx(), da.p, db.p, a.width, a.height, a.channels, out.p));
  return out.get()[0];
}

LossResult loss(const Image& rendered, const Image& target, double dssim_weight) {
  Trace tr{"loss", rendered.width, rendered.height, 0};
  same_shape(rendered, target);
  Dev<double> dr(kLossA, rendered.data), dt(kLossB, target.data), out(kLossOut, 3), dcol(kLossD, rendered.data.size());
  done(drk_loss_f64(ctx(), dr.p, dt.p, rendered.width, rendered.height, rendered.channels, dssim_weight, out.p,
                     dcol.p));
  LossResult res;
  res.value = out.get()[0];
  res.d_color = Image(rendered.width, rendered.height, rendered.channels);
  res.d_color.data = dcol.get();
  return res;
}

}  // namespace drk
