// ctypes-callable C entry points over the UNMODIFIED reference library
// (oracle/_ref/libdrk_refcapi.so) — TEST INFRASTRUCTURE ONLY.
//
// Used by tests/ to pin the C restatement (oracle/drk_oracle.c) and the CUDA
// path against the reference itself, and by bench.py's `--impl reference`
// arm / `cpu_baseline` leg to time the reference CPU renderer.  Never linked
// into the product.
//
// Layouts shared with include/drk_b200.h:
//   raw parameters: scalar-major SoA, raw[s * n + i] for scalar s of primitive i
//     in drk::for_each_scalar order (types.hpp:48-72), s < scalar_count(K, terms);
//   camera: drk_camera (fx, fy, cx, cy, width, height, R row-major world->cam, t);
//   images: row-major interleaved, double here.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "drk/errors.hpp"
#include "drk/grad.hpp"
#include "drk/optimize.hpp"
#include "drk/raster.hpp"

extern "C" {

struct ref_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9];
  double t[3];
};

struct ref_options {
  double lowpass_radius, alpha_min, grazing_eps;
  double background[3];
  double early_stop_transmittance;
  int32_t sh_degree, use_cache, exact_sort, presort, threads, pad_;
};

}  // extern "C"

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  if (dynamic_cast<const drk::NonFiniteError*>(&e)) return 2;
  if (dynamic_cast<const drk::DegenerateQuaternionError*>(&e)) return 3;
  if (dynamic_cast<const drk::DegenerateBasisError*>(&e)) return 4;
  if (dynamic_cast<const drk::ReplayMismatchError*>(&e)) return 5;
  if (dynamic_cast<const drk::DimensionMismatchError*>(&e)) return 6;
  return 1;
}

drk::Camera to_cam(const ref_camera* c) {
  drk::Camera cam;
  cam.fx = c->fx;
  cam.fy = c->fy;
  cam.cx = c->cx;
  cam.cy = c->cy;
  cam.width = c->width;
  cam.height = c->height;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) cam.world_to_cam_rot(r, k) = c->R[3 * r + k];
  for (int r = 0; r < 3; ++r) cam.world_to_cam_trans[r] = c->t[r];
  return cam;
}

drk::RenderOptions to_opt(const ref_options* o, int k) {
  drk::RenderOptions opt;
  opt.kernel.basis_count = k;
  opt.kernel.lowpass_radius = o->lowpass_radius;
  opt.kernel.alpha_min = o->alpha_min;
  opt.kernel.grazing_eps = o->grazing_eps;
  opt.background = drk::Vec3(o->background[0], o->background[1], o->background[2]);
  opt.early_stop_transmittance = o->early_stop_transmittance;
  opt.sh_degree = o->sh_degree;
  opt.use_cache = o->use_cache != 0;
  opt.exact_sort = o->exact_sort != 0;
  opt.presort = static_cast<drk::PresortMode>(o->presort);
  opt.threads = o->threads;
  return opt;
}

std::vector<drk::RawDrkParams> to_raws(const double* soa, int n, int k, int terms) {
  std::vector<drk::RawDrkParams> raws(n);
  const int sc = drk::scalar_count(k, terms);
  (void)sc;
  for (int i = 0; i < n; ++i) {
    drk::RawDrkParams p;
    p.scale_raw = drk::VecX::Zero(k);
    p.angle_raw = drk::VecX::Zero(k);
    p.sh_raw = drk::ShBlock::Zero(terms, 3);
    int s = 0;
    drk::for_each_scalar(p, [&](double& x, drk::ParamClass) { x = soa[static_cast<size_t>(s++) * n + i]; });
    raws[i] = p;
  }
  return raws;
}

void from_raws(const std::vector<drk::RawDrkParams>& raws, double* soa) {
  const int n = static_cast<int>(raws.size());
  for (int i = 0; i < n; ++i) {
    int s = 0;
    drk::for_each_scalar(raws[i], [&](const double& x, drk::ParamClass) {
      soa[static_cast<size_t>(s++) * n + i] = x;
    });
  }
}

void copy_image(const drk::Image& img, double* out) {
  if (out) std::memcpy(out, img.data.data(), img.data.size() * sizeof(double));
}

drk::Image image_from(const double* p, int w, int h, int c) {
  drk::Image img;
  if (!p) return img;
  img = drk::Image(w, h, c);
  std::memcpy(img.data.data(), p, img.data.size() * sizeof(double));
  return img;
}

// Storage of the last binning / replay so the caller can size its buffers.
struct LastBinning {
  std::vector<int64_t> offsets;
  std::vector<int32_t> ids;
  std::vector<double> keys;
} g_bins;

struct LastReplay {
  std::vector<int64_t> offsets;
  std::vector<int32_t> ids;
  std::vector<double> vals;  // u, v, depth, alpha, lowpass per record
} g_replay;

void capture_replay(const drk::ReplayBuffer& rb) {
  g_replay.offsets.assign(rb.pixels.size() + 1, 0);
  g_replay.ids.clear();
  g_replay.vals.clear();
  for (size_t p = 0; p < rb.pixels.size(); ++p) {
    for (const auto& r : rb.pixels[p]) {
      g_replay.ids.push_back(r.prim_id);
      g_replay.vals.insert(g_replay.vals.end(),
                           {r.u, r.v, r.depth, r.alpha, r.lowpass_active ? 1.0 : 0.0});
    }
    g_replay.offsets[p + 1] = static_cast<int64_t>(g_replay.ids.size());
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_hardware_threads() { return drk::resolve_thread_count(0); }

// Activated parameters: mu[3n], rot[9n] (row-major per prim), scales[kn],
// angles[kn], eta[n], tau[n], opacity[n] — all prim-major.
int ref_activate(const double* raw_soa, int n, int k, int terms, double* mu, double* rot,
                 double* scales, double* angles, double* eta, double* tau, double* opacity) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    for (int i = 0; i < n; ++i) {
      const drk::DrkPrimitive p = drk::activate(raws[i]);
      for (int c = 0; c < 3; ++c) mu[3 * i + c] = p.center[c];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) rot[9 * i + 3 * r + c] = p.rot(r, c);
      for (int j = 0; j < k; ++j) {
        scales[k * i + j] = p.scales[j];
        angles[k * i + j] = p.angles[j];
      }
      eta[i] = p.eta;
      tau[i] = p.tau;
      opacity[i] = p.opacity;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// bin_primitives over activated raws; results retrievable with ref_bins_copy.
int ref_bin(const double* raw_soa, int n, int k, int terms, const ref_camera* c,
            const ref_options* o, int64_t* total_pairs) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    const drk::RenderOptions opt = to_opt(o, k);
    const drk::TileBinning b = drk::bin_primitives(prims, to_cam(c), opt.kernel, opt.presort);
    g_bins.offsets.assign(b.tiles.size() + 1, 0);
    g_bins.ids.clear();
    g_bins.keys.clear();
    for (size_t t = 0; t < b.tiles.size(); ++t) {
      for (const auto& e : b.tiles[t]) {
        g_bins.ids.push_back(e.prim_id);
        g_bins.keys.push_back(e.key);
      }
      g_bins.offsets[t + 1] = static_cast<int64_t>(g_bins.ids.size());
    }
    *total_pairs = static_cast<int64_t>(g_bins.ids.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Thread-parallel drk::bin_primitives: the reference function (unmodified) on
// `threads` contiguous chunks of the primitives, then per tile the chunks'
// entries (ids made global) re-sorted with the reference comparator
// (raster.cpp:260-263).  Identical to one call over all primitives — the
// binning is per primitive apart from that final sort — in a fraction of the
// single-threaded time (full BASELINE frames in the parity tests).
int ref_bin_parallel(const double* raw_soa, int n, int k, int terms, const ref_camera* c, const ref_options* o,
                     int threads, int64_t* total_pairs) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    const drk::RenderOptions opt = to_opt(o, k);
    const drk::Camera cam = to_cam(c);
    const int T = std::max(1, std::min(threads > 0 ? threads : drk::resolve_thread_count(0), std::max(1, n)));
    std::vector<drk::TileBinning> parts(T);
    std::vector<std::string> errs(T);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int lo = (int)((long long)n * t / T), hi = (int)((long long)n * (t + 1) / T);
          std::vector<drk::DrkPrimitive> prims;
          prims.reserve(hi - lo);
          for (int i = lo; i < hi; ++i) prims.push_back(drk::activate(raws[i]));
          parts[t] = drk::bin_primitives(prims, cam, opt.kernel, opt.presort);
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw drk::Error(e);
    const size_t tiles = parts[0].tiles.size();
    std::vector<std::vector<drk::TileEntry>> merged(tiles);
    std::vector<std::thread> pool2;
    for (int t = 0; t < T; ++t) {
      pool2.emplace_back([&, t] {
        for (size_t tile = t; tile < tiles; tile += T) {
          auto& m = merged[tile];
          for (int q = 0; q < T; ++q) {
            const int lo = (int)((long long)n * q / T);
            for (const auto& e : parts[q].tiles[tile]) m.push_back({e.prim_id + lo, e.key});
          }
          std::sort(m.begin(), m.end(), [](const drk::TileEntry& a, const drk::TileEntry& b) {
            return a.key < b.key || (a.key == b.key && a.prim_id < b.prim_id);
          });
        }
      });
    }
    for (auto& th : pool2) th.join();
    g_bins.offsets.assign(tiles + 1, 0);
    g_bins.ids.clear();
    g_bins.keys.clear();
    for (size_t t = 0; t < tiles; ++t) {
      for (const auto& e : merged[t]) {
        g_bins.ids.push_back(e.prim_id);
        g_bins.keys.push_back(e.key);
      }
      g_bins.offsets[t + 1] = static_cast<int64_t>(g_bins.ids.size());
    }
    *total_pairs = static_cast<int64_t>(g_bins.ids.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// The reference training-step span of one view: activate + render(&replay) +
// loss (L1, dssim_weight = 0; optimize.cpp:171-204) + backward_render
// (grad.cpp:307-384).  Any output may be null.  seconds2 = {forward
// (activate + render), loss + backward}.
int ref_fwd_bwd(const double* raw_soa, int n, int k, int terms, const ref_camera* c, const ref_options* o,
                const double* target, double* color, double* depth, double* normal, double* alpha, double* loss_out,
                double* d_color, double* grad_soa, double* d_center_world, double* screen_grad, int8_t* touched,
                double* seconds2) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    const drk::Camera cam = to_cam(c);
    const drk::RenderOptions opt = to_opt(o, k);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    drk::ReplayBuffer rb;
    const drk::FrameBuffers fb = drk::render(prims, cam, opt, &rb);
    const auto t1 = std::chrono::steady_clock::now();
    const drk::LossResult lr = drk::loss(fb.color, image_from(target, cam.width, cam.height, 3), 0.0);
    drk::FrameGrad fg;
    fg.d_color = lr.d_color;
    const drk::ParamGrads g = drk::backward_render(raws, prims, cam, opt, rb, fg);
    const auto t2 = std::chrono::steady_clock::now();
    if (seconds2) {
      seconds2[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds2[1] = std::chrono::duration<double>(t2 - t1).count();
    }
    copy_image(fb.color, color);
    copy_image(fb.depth, depth);
    copy_image(fb.normal, normal);
    copy_image(fb.alpha, alpha);
    copy_image(lr.d_color, d_color);
    if (loss_out) *loss_out = lr.value;
    if (grad_soa) from_raws(g.raw, grad_soa);
    for (int i = 0; i < n; ++i) {
      if (d_center_world)
        for (int q = 0; q < 3; ++q) d_center_world[3 * i + q] = g.d_center_world[i][q];
      if (screen_grad) screen_grad[i] = g.screen_grad[i];
      if (touched) touched[i] = g.touched[i];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// drk::eval_sorting (raster.cpp:487-560) over activated raws: out4 = {accuracy,
// kendall_tau, mae, pixels}; presort / use_cache from the options.
int ref_eval_sorting(const double* raw_soa, int n, int k, int terms, const ref_camera* c, const ref_options* o,
                     double* out4) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    const drk::RenderOptions opt = to_opt(o, k);
    const drk::SortingMetrics m = drk::eval_sorting(prims, to_cam(c), opt.kernel, opt.presort, opt.use_cache);
    out4[0] = m.accuracy;
    out4[1] = m.kendall_tau;
    out4[2] = m.mae;
    out4[3] = (double)m.pixels;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

void ref_bins_copy(int64_t* offsets, int32_t* ids, double* keys) {
  std::memcpy(offsets, g_bins.offsets.data(), g_bins.offsets.size() * sizeof(int64_t));
  std::memcpy(ids, g_bins.ids.data(), g_bins.ids.size() * sizeof(int32_t));
  std::memcpy(keys, g_bins.keys.data(), g_bins.keys.size() * sizeof(double));
}

// activate + render.  Any output pointer may be null.  With want_replay the
// per-pixel blend records are kept for ref_replay_copy.  seconds_* report the
// wall time of activate+render (the reference's forward span).
int ref_render(const double* raw_soa, int n, int k, int terms, const ref_camera* c,
               const ref_options* o, double* color, double* depth, double* normal, double* alpha,
               int want_replay, int64_t* replay_records, double* seconds) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    drk::ReplayBuffer rb;
    const drk::FrameBuffers fb = drk::render(prims, to_cam(c), to_opt(o, k), want_replay ? &rb : nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    copy_image(fb.color, color);
    copy_image(fb.depth, depth);
    copy_image(fb.normal, normal);
    copy_image(fb.alpha, alpha);
    if (want_replay) {
      capture_replay(rb);
      if (replay_records) *replay_records = static_cast<int64_t>(g_replay.ids.size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

void ref_replay_copy(int64_t* offsets, int32_t* ids, double* vals) {
  std::memcpy(offsets, g_replay.offsets.data(), g_replay.offsets.size() * sizeof(int64_t));
  std::memcpy(ids, g_replay.ids.data(), g_replay.ids.size() * sizeof(int32_t));
  std::memcpy(vals, g_replay.vals.data(), g_replay.vals.size() * sizeof(double));
}

// activate + render(replay) + backward_render with the given frame gradient
// images (null = empty).  Outputs raw grads in scalar-major SoA, plus
// d_center_world[3n], screen_grad[n], touched[n].
int ref_backward(const double* raw_soa, int n, int k, int terms, const ref_camera* c,
                 const ref_options* o, const double* d_color, const double* d_depth,
                 const double* d_normal, const double* d_alpha, double* grad_soa,
                 double* d_center_world, double* screen_grad, int8_t* touched, double* seconds) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    const drk::Camera cam = to_cam(c);
    const drk::RenderOptions opt = to_opt(o, k);
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    drk::ReplayBuffer rb;
    drk::render(prims, cam, opt, &rb);
    drk::FrameGrad fg;
    fg.d_color = image_from(d_color, cam.width, cam.height, 3);
    fg.d_depth = image_from(d_depth, cam.width, cam.height, 1);
    fg.d_normal = image_from(d_normal, cam.width, cam.height, 3);
    fg.d_alpha = image_from(d_alpha, cam.width, cam.height, 1);
    const auto t0 = std::chrono::steady_clock::now();
    const drk::ParamGrads g = drk::backward_render(raws, prims, cam, opt, rb, fg);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    from_raws(g.raw, grad_soa);
    for (int i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) d_center_world[3 * i + a] = g.d_center_world[i][a];
      screen_grad[i] = g.screen_grad[i];
      touched[i] = g.touched[i];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Full reference training-step span for one view (config 2/4 CPU arm):
// activate, render with replay, L1 loss (dssim_weight 0), backward_render.
int ref_train_step(const double* raw_soa, int n, int k, int terms, const ref_camera* c,
                   const ref_options* o, const double* target, double* loss_out,
                   double* grad_soa, double* seconds) {
  try {
    const auto raws = to_raws(raw_soa, n, k, terms);
    const drk::Camera cam = to_cam(c);
    const drk::RenderOptions opt = to_opt(o, k);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    drk::ReplayBuffer rb;
    const drk::FrameBuffers fb = drk::render(prims, cam, opt, &rb);
    const drk::Image tgt = image_from(target, cam.width, cam.height, 3);
    const drk::LossResult lr = drk::loss(fb.color, tgt, 0.0);
    drk::FrameGrad fg;
    fg.d_color = lr.d_color;
    const drk::ParamGrads g = drk::backward_render(raws, prims, cam, opt, rb, fg);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (loss_out) *loss_out = lr.value;
    if (grad_soa) from_raws(g.raw, grad_soa);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// L1 branch of drk::loss (optimize.cpp:171-204 with dssim_weight = 0).
int ref_loss_l1(const double* rendered, const double* target, int w, int h, double* value,
                double* d_color) {
  try {
    const drk::LossResult lr =
        drk::loss(image_from(rendered, w, h, 3), image_from(target, w, h, 3), 0.0);
    *value = lr.value;
    copy_image(lr.d_color, d_color);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Full drk::loss (optimize.cpp:171-204) on interleaved H x W x c images.
int ref_loss(const double* rendered, const double* target, int w, int h, int c, double dssim_weight,
             double* value, double* d_color) {
  try {
    const drk::LossResult lr = drk::loss(image_from(rendered, w, h, c), image_from(target, w, h, c), dssim_weight);
    *value = lr.value;
    copy_image(lr.d_color, d_color);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// drk::ssim (optimize.cpp:157-166) and drk::psnr (:145-155).
int ref_ssim(const double* a, const double* b, int w, int h, int c, double* out) {
  try {
    *out = drk::ssim(image_from(a, w, h, c), image_from(b, w, h, c));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}
int ref_psnr(const double* a, const double* b, int w, int h, int c, double* out) {
  try {
    *out = drk::psnr(image_from(a, w, h, c), image_from(b, w, h, c));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// densify_and_prune (optimize.cpp:320-373) on SoA raws / moments; outputs
// (capacity cap, SoA with row stride cap) and *n_out.  thr = {densify_grad,
// prune_opacity, percent_dense}.
int ref_densify_and_prune(const double* raw, const double* m, const double* v, int n, int k, int terms,
                          const double* accum, const int* count, const double* thr, double extent, double* raw_out,
                          double* m_out, double* v_out, long long cap, long long* n_out) {
  try {
    std::vector<drk::RawDrkParams> params = to_raws(raw, n, k, terms);
    drk::OptState st;
    st.m = to_raws(m, n, k, terms);
    st.v = to_raws(v, n, k, terms);
    drk::DensifyStats stats;
    stats.resize(n);
    for (int i = 0; i < n; ++i) {
      stats.screen_grad_accum[i] = accum[i];
      stats.touch_count[i] = count[i];
    }
    drk::TrainConfig cfg;
    cfg.densify_grad_threshold = thr[0];
    cfg.prune_opacity_threshold = thr[1];
    cfg.percent_dense = thr[2];
    drk::densify_and_prune(params, st, stats, cfg, extent);
    *n_out = (long long)params.size();
    if ((long long)params.size() > cap) return 0;
    const int no = (int)params.size();
    std::vector<double> tmp((size_t)drk::scalar_count(k, terms) * no);
    auto put = [&](const std::vector<drk::RawDrkParams>& src, double* dst) {
      from_raws(src, tmp.data());
      for (int sc = 0; sc < drk::scalar_count(k, terms); ++sc)
        for (int i = 0; i < no; ++i) dst[(size_t)sc * cap + i] = tmp[(size_t)sc * no + i];
    };
    put(params, raw_out);
    put(st.m, m_out);
    put(st.v, v_out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

double ref_scene_extent(const double* raw, int n, int k, int terms) {
  return drk::scene_extent(to_raws(raw, n, k, terms));
}

// drk::train (optimize.cpp:390-470) over nv views (images H x W x 3 doubles,
// one camera each) from SoA raws.  icfg = {steps, densify_interval,
// densify_start, densify_stop, sh_warmup, max_sh, eval_interval, seed};
// dcfg = {lr_drk, lr_position, lr_rotation, lr_opacity, lr_sh, densify_grad,
// prune_opacity, dssim_weight, percent_dense}.  Outputs: log rows
// (loss, psnr, count) per step, final psnr, final params (cap primitives).
int ref_train(const double* raw, int n, int k, int terms, int nv, const ref_camera* cams, const double* images,
              const int* icfg, const double* dcfg, double* log_out, double* final_psnr, double* raw_out,
              long long cap, long long* n_out) {
  try {
    std::vector<drk::TrainView> views(nv);
    size_t off = 0;
    for (int v = 0; v < nv; ++v) {
      views[v].camera = to_cam(&cams[v]);
      const int w = cams[v].width, h = cams[v].height;
      views[v].image = drk::Image(w, h, 3);
      std::memcpy(views[v].image.data.data(), images + off, sizeof(double) * 3 * w * h);
      off += (size_t)3 * w * h;
    }
    drk::TrainConfig cfg;
    cfg.steps = icfg[0];
    cfg.densify_interval = icfg[1];
    cfg.densify_start_step = icfg[2];
    cfg.densify_stop_step = icfg[3];
    cfg.sh_degree_warmup_interval = icfg[4];
    cfg.max_sh_degree = icfg[5];
    cfg.eval_interval = icfg[6];
    cfg.seed = (unsigned)icfg[7];
    cfg.lr_drk = dcfg[0];
    cfg.lr_position = dcfg[1];
    cfg.lr_rotation = dcfg[2];
    cfg.lr_opacity = dcfg[3];
    cfg.lr_sh = dcfg[4];
    cfg.densify_grad_threshold = dcfg[5];
    cfg.prune_opacity_threshold = dcfg[6];
    cfg.dssim_weight = dcfg[7];
    cfg.percent_dense = dcfg[8];
    cfg.kernel.basis_count = k;
    const drk::TrainResult r = drk::train(views, to_raws(raw, n, k, terms), cfg);
    for (size_t i = 0; i < r.log.size(); ++i) {
      log_out[3 * i] = r.log[i].loss;
      log_out[3 * i + 1] = r.log[i].psnr;
      log_out[3 * i + 2] = (double)r.log[i].count;
    }
    *final_psnr = r.final_psnr;
    *n_out = (long long)r.params.size();
    if ((long long)r.params.size() <= cap) {
      const int no = (int)r.params.size();
      std::vector<double> tmp((size_t)drk::scalar_count(k, terms) * no);
      from_raws(r.params, tmp.data());
      for (int sc = 0; sc < drk::scalar_count(k, terms); ++sc)
        for (int i = 0; i < no; ++i) raw_out[(size_t)sc * cap + i] = tmp[(size_t)sc * no + i];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// drk::adam_step (optimize.cpp:248-307) on SoA raws; m/v are SoA moment
// buffers updated in place; *step is OptState::step (incremented).
// lrs: lr_drk, lr_position, lr_rotation, lr_opacity, lr_sh; steps_total.
int ref_adam_step(double* params_soa, const double* grads_soa, double* m_soa, double* v_soa, int n,
                  int k, int terms, int64_t* step, const double* lrs, int steps_total,
                  double extent, int freeze_eta_tau, int freeze_angles) {
  try {
    auto params = to_raws(params_soa, n, k, terms);
    const auto grads = to_raws(grads_soa, n, k, terms);
    drk::OptState st;
    st.m = to_raws(m_soa, n, k, terms);
    st.v = to_raws(v_soa, n, k, terms);
    st.step = *step;
    drk::TrainConfig cfg;
    cfg.lr_drk = lrs[0];
    cfg.lr_position = lrs[1];
    cfg.lr_rotation = lrs[2];
    cfg.lr_opacity = lrs[3];
    cfg.lr_sh = lrs[4];
    cfg.steps = steps_total;
    cfg.freeze_eta_tau = freeze_eta_tau != 0;
    cfg.freeze_angles = freeze_angles != 0;
    drk::adam_step(params, grads, st, cfg, extent);
    from_raws(params, params_soa);
    from_raws(st.m, m_soa);
    from_raws(st.v, v_soa);
    *step = st.step;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

}  // extern "C"
