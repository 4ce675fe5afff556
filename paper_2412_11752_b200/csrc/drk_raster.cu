// K4 forward rasterizer and K5 backward rasterizer (reference raster.cpp:267-430,
// grad.cpp:16-303), K6 activation backward (grad.cpp:122-159, :370-383),
// K7 L1 loss, K8 Adam.
//
// One CTA per 16x16 tile, one thread per pixel.  The tile list is streamed in
// batches of 256 candidates staged in shared memory (id, ray-plane numerator,
// plane normal: 36 B each); every pixel intersects the batch in fp64 with
// explicitly rounded ops in the reference order (bit-identical depths), runs
// the capacity-8 SortCache (raster.cpp:267-303) in registers, and composites
// popped entries.  A pixel leaves the stream once saturated; the CTA leaves
// once all pixels have (__syncthreads_count).
//
// Alpha of a popped entry is evaluated in fp32 (alpha_f32) with a relative
// error bound.  Decisions that fall inside the bound (alpha_min skip, low-pass
// floor vs kernel, the 1-1e-6 clamp) are re-evaluated in fp64 on the spot; a
// pixel whose transmittance comes within its accumulated error bound of the
// early-stop threshold is flagged and re-rendered entirely in fp64 by a
// second launch (F64 = true).  Composited values are accumulated in fp64.
//
// The backward kernel re-streams the same decisions (no replay buffer) and
// rebuilds `rest` from the forward pass's fp64 per-pixel accumulators.
//
// This translation unit is compiled with --fmad=true: every fp64 value that
// must match the reference bit for bit uses __dmul_rn / __dadd_rn.
#include <algorithm>

#include "drk_internal.h"

#ifndef DRK_RASTER_MIN_BLOCKS
#define DRK_RASTER_MIN_BLOCKS 2
#endif

namespace drk {

// Row stride bound of the activated-gradient buffer (grad_row_stride(16)).
constexpr int kGradSlotStride = 96;
static_assert(kGOffSh + 48 <= kGradSlotStride, "gradient row layout");
#ifndef DRK_BWD_MIN_BLOCKS
#define DRK_BWD_MIN_BLOCKS 2
#endif

// alpha_tilde in fp64 (composite_candidate, raster.cpp:333-345: kernel alpha,
// low-pass floor when the centre projects).  One compiled instance serves the
// cache, list and exact-sort paths, so equal inputs give equal bits in all of
// them (FMA contraction cannot differ between inlined copies).
static __device__ __noinline__ double alpha64(const ShapeView& S, int id, double u, double v, bool has_proj,
                                               double dpw, double dph, double cos_view, double lowpass_radius,
                                               KEval& ev, bool& lp) {
  eval_kernel(u, v, S, id, ev);
  lp = false;
  if (ev.degenerate) return 0.0;
  const double o = S.o[id];
  const double a_kernel = o * sharpen(ev.g, S.tau[id]);
  double a = a_kernel;
  if (has_proj) {
    const double f = low_pass_filter_term(dpw, dph, cos_view, o, lowpass_radius);
    if (f > a_kernel) {
      a = f;
      lp = true;
    }
  }
  return a;
}

template <bool BWD, bool F64>
struct Pixel {
  double dir[3];
  float basis[16];
  double basis64[F64 ? 16 : 1];  // fp64 SH basis of the pixel's ray (sh_basis_d), fp64 paths only
  bool col64;                    // colours in fp64 (reference precision, or fp64 coefficients given)
  double px, py;
  double T, C[3], D, N[3], A;
  float E;  // relative error bound of T (fp32 alphas)
  bool uncertain;
  // backward
  double dC[3], dD, dN[3], dA, rest;
  bool has_dN;
  long long n_pop, n_comp;
  unsigned n_rej1, n_rej2, n_f64;
  int pix, n_rec, stop;
  bool err;

  __device__ void init(const RasterParams& P, int x, int y) {
    n_rej1 = n_rej2 = n_f64 = 0;
    px = x + 0.5;
    py = y + 0.5;
    pixel_dir(P.cam, px, py, dir);
#pragma unroll
    for (int t = 0; t < 16; ++t) basis[t] = 0.f;
    sh_basis_f((float)dir[0], (float)dir[1], (float)dir[2], P.opt.sh_degree, basis);
    col64 = F64 && (P.opt.fp64_alpha || P.sh64 != nullptr);
    if (col64) sh_basis_d(dir[0], dir[1], dir[2], P.opt.sh_degree, basis64);
    T = 1.0;
    C[0] = C[1] = C[2] = D = N[0] = N[1] = N[2] = A = 0;
    E = 0.f;
    uncertain = false;
    n_pop = n_comp = 0;
    n_rec = 0;
    stop = 0x7fffffff;
    err = false;
    pix = y * P.cam.W + x;
  }

  __device__ void init_bwd(const RasterParams& P) {
    const size_t p = (size_t)pix;
    dC[0] = P.dC ? P.dC[3 * p] : 0.f;
    dC[1] = P.dC ? P.dC[3 * p + 1] : 0.f;
    dC[2] = P.dC ? P.dC[3 * p + 2] : 0.f;
    dD = P.dD ? P.dD[p] : 0.f;
    has_dN = P.dN != nullptr;
    dN[0] = P.dN ? P.dN[3 * p] : 0.f;
    dN[1] = P.dN ? P.dN[3 * p + 1] : 0.f;
    dN[2] = P.dN ? P.dN[3 * p + 2] : 0.f;
    dA = P.dA ? P.dA[p] : 0.f;
    const double* st = P.pxstate + 8 * p;
    // total = dC.C + dD D + dN.N + dA A (C includes T_n bg): grad.cpp:210-222
    rest = (dC[0] * st[0] + dC[1] * st[1] + dC[2] * st[2]) + dD * st[3] +
           (dN[0] * st[4] + dN[1] * st[5] + dN[2] * st[6]) + dA * st[7];
  }

  // composite_candidate (raster.cpp:327-362) + backward_pixel (grad.cpp:224-301)
  // for one popped entry.  Returns false once the pixel saturates.
  __device__ bool composite(const RasterParams& P, double rt, int id) {
    const Geo& g = P.geo[id];
    const double rz0 = g.rz[0], rz1 = g.rz[1], rz2 = g.rz[2];
    const double denom = xdot3(dir[0], dir[1], dir[2], rz0, rz1, rz2);
    // u, v (geometry.cpp:48-50)
    const double h0 = xs(xa(P.cam.o[0], xm(rt, dir[0])), g.mu[0]);
    const double h1 = xs(xa(P.cam.o[1], xm(rt, dir[1])), g.mu[1]);
    const double h2 = xs(xa(P.cam.o[2], xm(rt, dir[2])), g.mu[2]);
    const double u = xdot3(g.rx[0], g.rx[1], g.rx[2], h0, h1, h2);
    const double v = xdot3(g.ry[0], g.ry[1], g.ry[2], h0, h1, h2);
    ++n_pop;
    const double cos_view = fabs(denom);
    double dpw = 0, dph = 0;
    if (g.has_proj) {
      dpw = xs(px, g.ppx);
      dph = xs(py, g.ppy);
    }
    // Cheap reject: alpha_kernel < alpha_min whenever r2^2 / s_max^2 > f_vis^2
    // (Q >= r2^2 / s_max^2), and the low-pass floor < alpha_min whenever
    // dp^2 > 2 cos^2 s_l^2 ln(o / alpha_min); both with a 1e-9 margin.
    const double r2 = xa(xm(u, u), xm(v, v));
    const bool lp_possible = g.has_proj && dpw * dpw + dph * dph <= cos_view * cos_view * g.dp2max;
    if (r2 > g.r2max && !lp_possible) {
      ++n_rej1;
      return true;
    }
    double a;
    bool lp = false;
    float rel = 0.f;
    bool use64 = F64;
    KEval ev;
    ev.center = false;
    ev.clamped = false;
    if (!F64) {
      bool degen;
      float relk;
      const float ak = alpha_f32(u, v, r2, P.S, id, 0.f, 0.f, (float)P.S.eta[id], &relk, &degen, !lp_possible);
      if (degen) {
        err = true;
        return false;
      }
      if (ak < 0.f) {  // kernel below alpha_min in its bracket, floor out of reach
        ++n_rej2;
        return true;
      }
      float at = ak, relt = relk;
      // The low-pass floor only matters where it can reach alpha_min
      // (otherwise max(alpha, floor) >= alpha_min <=> alpha >= alpha_min).
      if (lp_possible) {
        const float sl = (float)P.opt.lowpass_radius, cv = (float)cos_view;
        const float ex = fmaxf(-((float)(dpw * dpw + dph * dph)) / (2.0f * cv * cv * sl * sl), -30.0f);
        const float f = (float)P.S.o[id] * expf(ex);
        const float relf = 4e-7f * (1.0f - ex);
        if (fabsf(f - ak) <= relk * ak + relf * f) use64 = true;
        if (f > ak) {
          at = f;
          relt = relf;
          lp = true;
        }
      }
      const float amin = (float)P.opt.alpha_min;
      if (fabsf(at - amin) <= relt * at + 1e-12f) use64 = true;
      if (at >= 0.99f && fabs((double)at - (1.0 - 1e-6)) <= (double)relt * at + 1e-12) use64 = true;
      a = (double)at;
      rel = relt;
    }
    if (use64) {
      ++n_f64;
      a = alpha64(P.S, id, u, v, g.has_proj, dpw, dph, cos_view, P.opt.lowpass_radius, ev, lp);
      if (ev.degenerate) {
        err = true;
        return false;
      }
      rel = 0.f;
    }
    if (a < P.opt.alpha_min) return true;
    a = dmin(a, 1.0 - 1e-6);
    double rgb[3];
    if (F64 && col64) {
      sh_rgb_d(P, id, rgb);
    } else {
      float r0, r1, r2c;
      sh_rgb(P, id, r0, r1, r2c);
      rgb[0] = r0;
      rgb[1] = r1;
      rgb[2] = r2c;
    }
    const bool cl0 = rgb[0] < 0, cl1 = rgb[1] < 0, cl2 = rgb[2] < 0;
    for (int c = 0; c < 3; ++c) rgb[c] = rgb[c] < 0 ? 0.0 : rgb[c];
    const double sgn = denom < 0 ? 1.0 : -1.0;
    const double w = xm(T, a);
    ++n_comp;
    if (!BWD) {
      // raster.cpp:353-357, each op rounded (no contraction): the cache, list
      // and exact-sort paths accumulate bit-identically
      C[0] = xa(C[0], xm(w, rgb[0]));
      C[1] = xa(C[1], xm(w, rgb[1]));
      C[2] = xa(C[2], xm(w, rgb[2]));
      D = xa(D, xm(w, rt));
      N[0] = xa(N[0], xm(w, xm(sgn, rz0)));
      N[1] = xa(N[1], xm(w, xm(sgn, rz1)));
      N[2] = xa(N[2], xm(w, xm(sgn, rz2)));
      A = xa(A, w);
      if (P.replay_cap > 0) {
        if (n_rec < P.replay_cap) {
          const size_t r = (size_t)pix * P.replay_cap + n_rec;
          P.replay_ids[r] = id;
          double* rec = P.replay_rec + 5 * r;
          rec[0] = u;
          rec[1] = v;
          rec[2] = rt;
          rec[3] = a;
          rec[4] = lp ? 1.0 : 0.0;
        }
        ++n_rec;
      }
    } else {
      const bool alpha_clamped = a >= 1.0 - 1e-6 - 1e-12;
      if (!use64 && !lp && !alpha_clamped) {
        eval_kernel(u, v, P.S, id, ev);  // fp64 partials for backward_alpha
      }
      backward_record(P, id, g, rt, u, v, a, lp, ev, rgb, cl0, cl1, cl2, sgn, denom, dpw, dph, w);
    }
    T = xm(T, xs(1.0, a));
    if (!F64) {
      const float af = (float)a;
      E += rel * __fdividef(af, 1.0f - af) + 1e-15f;
      if (fabs(T - P.opt.early_stop) <= T * (double)E) uncertain = true;
    }
    if (T >= P.opt.early_stop) return true;
    stop = (int)n_comp;
    return false;
  }

  __device__ void backward_record(const RasterParams& P, int id, const Geo& g, double rt, double u, double v,
                                  double a, bool lp, const KEval& ev, const double rgb[3], bool cl0, bool cl1,
                                  bool cl2, double sgn, double rdz, double dpw, double dph, double wb) {
    const double rz[3] = {g.rz[0], g.rz[1], g.rz[2]};
    const double cw = (dC[0] * rgb[0] + dC[1] * rgb[1] + dC[2] * rgb[2]) + dD * rt +
                      (dN[0] * (sgn * rz[0]) + dN[1] * (sgn * rz[1]) + dN[2] * (sgn * rz[2])) + dA;
    rest -= wb * cw;
    const double dat = T * cw - rest / (1.0 - a);
    backward_record_dat(P, id, g, rt, u, v, a, lp, ev, rgb, cl0, cl1, cl2, sgn, rdz, dpw, dph, wb, dat, T,
                        (int)n_comp - 1);
  }

  // Gradient of one record given its upstream dL/d(alpha_tilde) (`dat`) and
  // blend weight wb = T alpha (grad.cpp:237-301, :16-101), fp64 atomics.
  __device__ void backward_record_dat(const RasterParams& P, int id, const Geo& g, double rt, double u, double v,
                                      double a, bool lp, const KEval& ev, const double rgb[3], bool cl0, bool cl1,
                                      bool cl2, double sgn, double rdz, double dpw, double dph, double wb,
                                      double dat, double T_i, int comp_idx) const {
    (void)rgb;
    (void)T_i;
    // deterministic mode: the record's own fp64 row (plain adds, fixed order);
    // otherwise fp32 atomics into the primitive's row
    float* pg = P.gact + (size_t)id * P.G;
    double* dr = nullptr;
    float* dr32 = nullptr;
    if (P.det_rec || P.det_rec32) {
      const long long r = det_row(P, pix % P.cam.W, pix / P.cam.W, comp_idx, id);
      if (r < 0) return;
      // the row belongs to this record alone: clear it, then accumulate
      if (P.det_rec) {
        dr = P.det_rec + (size_t)r * P.G;
        for (int c = 0; c < P.G; ++c) dr[c] = 0.0;
      } else {
        dr32 = P.det_rec32 + (size_t)r * P.G;
        for (int c = 0; c < P.G; ++c) dr32[c] = 0.f;
      }
    }
    auto gadd = [dr, dr32, pg](float* a, double v) {
      if (dr) dr[a - pg] += v;
      else if (dr32) dr32[a - pg] += (float)v;
      else atomicAdd(a, (float)v);
    };
    const int K = P.S.K;
    const double rz[3] = {g.rz[0], g.rz[1], g.rz[2]};
    P.touched[id] = 1;
    const int o_rot = 3, o_sc = kGOffSc, o_an = kGOffAn, o_eta = kGOffEta, o_tau = kGOffTau, o_op = kGOffOp,
              o_sh = kGOffSh;
    // SH (linear, clamped channels gated)
    const bool cl[3] = {cl0, cl1, cl2};
    for (int ch = 0; ch < 3; ++ch) {
      if (cl[ch]) continue;
      const double dc = wb * dC[ch];
      if (dc == 0) continue;
      for (int t = 0; t < P.opt.terms_active; ++t)
        gadd(pg + o_sh + 3 * t + ch, dc * (F64 && col64 ? basis64[t < 16 && F64 ? t : 0] : (double)basis[t]));
    }
    if (has_dN)
      for (int q = 0; q < 3; ++q) gadd(pg + o_rot + 3 * q + 2, wb * sgn * dN[q]);
    if (dD != 0) {
      const double d_rt = wb * dD;
      for (int q = 0; q < 3; ++q) {
        const double h = P.cam.o[q] + rt * dir[q] - g.mu[q];
        gadd(pg + q, d_rt * rz[q] / rdz);
        gadd(pg + o_rot + 3 * q + 2, d_rt * (-h / rdz));
      }
    }
    const bool alpha_clamped = a >= 1.0 - 1e-6 - 1e-12;
    if (alpha_clamped) return;
    const double o = P.S.o[id];
    if (lp) {
      const double cv = fabs(rdz), sl = P.opt.lowpass_radius;
      gadd(pg + o_op, dat * a / o);
      const double inv = 1.0 / (cv * cv * sl * sl);
      const double d_dpw = dat * a * (-dpw * inv);
      const double d_dph = dat * a * (-dph * inv);
      const double d_cos = dat * a * (dpw * dpw + dph * dph) * inv / cv;
      double J[6];
      projection_jacobian(P.cam, g.mu, J);
      for (int q = 0; q < 3; ++q) gadd(pg + q, -(J[q] * d_dpw + J[3 + q] * d_dph));
      const double sg = rdz < 0 ? -1.0 : 1.0;
      for (int q = 0; q < 3; ++q) gadd(pg + o_rot + 3 * q + 2, d_cos * sg * dir[q]);
      return;
    }
    // backward_alpha (grad.cpp:16-101)
    const double tau = P.S.tau[id];
    const double d_alpha = dat;
    gadd(pg + o_op, d_alpha * sharpen(ev.g, tau));
    if (ev.center) return;
    const int br = sharpen_branch(ev.g, tau);
    gadd(pg + o_tau, d_alpha * o * sharpen_dtau(br, ev.g, tau));
    if (ev.clamped) return;
    const double d_g = d_alpha * o * sharpen_slope(br, tau);
    const double d_q = d_g * (-0.5 * ev.g);
    const int lo = ev.lo, hi = ev.hi;
    const double* s = P.S.s + (size_t)id * K;
    const double* th = P.S.th + (size_t)id * K;
    const double slo = s[lo], shi = s[hi], eta = P.S.eta[id];
    gadd(pg + o_eta, d_q * (ev.r1 * ev.r1 - ev.r2 * ev.inv_sbar));
    const double d_r1 = d_q * eta * 2.0 * ev.r1;
    const double d_r2sq = d_q * (1.0 - eta) * ev.inv_sbar;
    const double d_inv = d_q * (1.0 - eta) * ev.r2;
    const double c = cos(ev.delta);
    double ds_lo = d_inv * (-(1.0 + c) / (slo * slo * slo));
    double ds_hi = d_inv * (-(1.0 - c) / (shi * shi * shi));
    const double d_c = d_inv * (0.5 / (slo * slo) - 0.5 / (shi * shi));
    const double d_delta = d_c * (-sin(ev.delta));
    double alo = th[lo], ahi = th[hi], theta = ev.theta;
    if (hi == 0) {
      alo -= kTwoPi;
      if (theta > th[K - 1]) theta -= kTwoPi;
    }
    const double gap = ahi - alo;
    const double d_tfd = d_delta * kPi / gap;
    double da_lo = d_delta * kPi * (theta - ahi) / (gap * gap);
    double da_hi = d_delta * (-kPi) * (theta - alo) / (gap * gap);
    const double r2s = dmax(ev.r2, 1e-24);
    double du = d_tfd * (-v / r2s);
    double dv = d_tfd * (u / r2s);
    du += d_r2sq * 2.0 * u;
    dv += d_r2sq * 2.0 * v;
    const double sa = ev.a > 0 ? 1 : (ev.a < 0 ? -1 : 0);
    const double sb = ev.b > 0 ? 1 : (ev.b < 0 ? -1 : 0);
    const double elx = P.S.ex[(size_t)id * K + lo], ely = P.S.ey[(size_t)id * K + lo];
    const double ehx = P.S.ex[(size_t)id * K + hi], ehy = P.S.ey[(size_t)id * K + hi];
    const double det = P.S.det[(size_t)id * K + lo];
    du += d_r1 * (sa * (ehy / det) + sb * (-ely / det));
    dv += d_r1 * (sa * (-ehx / det) + sb * (elx / det));
    const double ca = cos(th[lo]), sa_lo = sin(th[lo]);
    const double cb = cos(th[hi]), sb_hi = sin(th[hi]);
    ds_lo += d_r1 * (-sa * ev.a / slo);
    ds_hi += d_r1 * (-sb * ev.b / shi);
    const double tlx = -slo * sa_lo, tly = slo * ca, thx = -shi * sb_hi, thy = shi * cb;
    const double na = -ev.a, nb = -ev.b;
    const double dtl_x = na * ((ehy * tlx - ehx * tly) / det), dtl_y = na * ((-ely * tlx + elx * tly) / det);
    const double dth_x = nb * ((ehy * thx - ehx * thy) / det), dth_y = nb * ((-ely * thx + elx * thy) / det);
    da_lo += d_r1 * (sa * dtl_x + sb * dtl_y);
    da_hi += d_r1 * (sa * dth_x + sb * dth_y);
    gadd(pg + o_sc + lo, ds_lo);
    gadd(pg + o_sc + hi, ds_hi);
    gadd(pg + o_an + lo, da_lo);
    gadd(pg + o_an + hi, da_hi);
    // (u, v) and r_t chain to centre and rotation columns (grad.cpp:290-300)
    const double h[3] = {P.cam.o[0] + rt * dir[0] - g.mu[0], P.cam.o[1] + rt * dir[1] - g.mu[1],
                         P.cam.o[2] + rt * dir[2] - g.mu[2]};
    const double drx = dir[0] * g.rx[0] + dir[1] * g.rx[1] + dir[2] * g.rx[2];
    const double dry = dir[0] * g.ry[0] + dir[1] * g.ry[1] + dir[2] * g.ry[2];
    for (int q = 0; q < 3; ++q) {
      const double du_dmu = rz[q] * (drx / rdz) - g.rx[q];
      const double dv_dmu = rz[q] * (dry / rdz) - g.ry[q];
      gadd(pg + q, du * du_dmu + dv * dv_dmu);
    }
    const double f = -(du * drx + dv * dry) / rdz;
    for (int q = 0; q < 3; ++q) {
      gadd(pg + o_rot + 3 * q + 0, du * h[q]);
      gadd(pg + o_rot + 3 * q + 1, dv * h[q]);
      gadd(pg + o_rot + 3 * q + 2, f * h[q]);
    }
  }

  // ---- warp-cooperative backward (k_raster_bwd) -------------------------
  // Called by all 32 lanes of a warp together.  `want` lanes replay the
  // forward decision for their popped entry; composited records compute
  // their activated-space gradient (fp32 from the fp32 kernel evaluation, or
  // fp64 in the F64 kernels), and the components are reduced over the lanes
  // whose record hits the same primitive (transpose-reduce, below) and added
  // to HBM with 16-byte vector reductions.  Returns false once this lane's
  // pixel saturates.
  __device__ bool composite_warp(const RasterParams& P, bool want, double rt, int id) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    bool rec = false, cont = true, lp = false, use64 = F64;
    double a = 0, u = 0, v = 0, r2 = 0, denom = 0, dpw = 0, dph = 0, rz[3] = {0, 0, 0};
    float rgbf[3] = {0, 0, 0};
    bool cl[3] = {false, false, false};
    KEval ev;  // fp64 evaluation (F64 kernels; fp32 decisions inside their bound)
    ev.center = ev.clamped = ev.degenerate = false;
    ev.g = 1.0;
    ev.lo = ev.hi = 0;
    KEvalF kf;  // fp32 evaluation, differentiated by the fp32 backward
    kf.center = true;
    kf.clamped = false;
    const Geo* gp = nullptr;
    if (want) {
      const Geo& g = P.geo[id];
      gp = &g;
      rz[0] = g.rz[0];
      rz[1] = g.rz[1];
      rz[2] = g.rz[2];
      denom = xdot3(dir[0], dir[1], dir[2], rz[0], rz[1], rz[2]);
      const double h0 = xs(xa(P.cam.o[0], xm(rt, dir[0])), g.mu[0]);
      const double h1 = xs(xa(P.cam.o[1], xm(rt, dir[1])), g.mu[1]);
      const double h2 = xs(xa(P.cam.o[2], xm(rt, dir[2])), g.mu[2]);
      u = xdot3(g.rx[0], g.rx[1], g.rx[2], h0, h1, h2);
      v = xdot3(g.ry[0], g.ry[1], g.ry[2], h0, h1, h2);
      const double cos_view = fabs(denom);
      if (g.has_proj) {
        dpw = xs(px, g.ppx);
        dph = xs(py, g.ppy);
      }
      r2 = xa(xm(u, u), xm(v, v));
      const bool lp_possible = g.has_proj && dpw * dpw + dph * dph <= cos_view * cos_view * g.dp2max;
      const bool reject = r2 > g.r2max && !lp_possible;
      if (!reject) {
        const double o = P.S.o[id], tau = P.S.tau[id];
        bool skip = false;
        if (!F64) {
          bool degen;
          float relk;
          const float ak = alpha_f32(u, v, r2, P.S, id, (float)o, (float)tau, (float)P.S.eta[id], &relk, &degen,
                                     !lp_possible, &kf);
          if (degen) {
            err = true;
            cont = false;
          }
          skip = ak < 0.f;
          float at = ak, relt = relk;
          if (lp_possible) {
            const float sl = (float)P.opt.lowpass_radius, cv = (float)cos_view;
            const float ex = fmaxf(-((float)(dpw * dpw + dph * dph)) / (2.0f * cv * cv * sl * sl), -30.0f);
            const float f = (float)o * expf(ex);
            const float relf = 4e-7f * (1.0f - ex);
            if (fabsf(f - ak) <= relk * ak + relf * f) use64 = true;
            if (f > ak) {
              at = f;
              relt = relf;
              lp = true;
            }
          }
          const float amin = (float)P.opt.alpha_min;
          if (fabsf(at - amin) <= relt * at + 1e-12f) use64 = true;
          if (at >= 0.99f && fabs((double)at - (1.0 - 1e-6)) <= (double)relt * at + 1e-12) use64 = true;
          a = (double)at;
        }
        if (skip) {
          a = 0;  // alpha < alpha_min: not composited
        } else if (cont && use64) {
          eval_kernel(u, v, P.S, id, ev);
          if (ev.degenerate) {
            err = true;
            cont = false;
          } else {
            const double a_kernel = o * sharpen(ev.g, tau);
            a = a_kernel;
            lp = false;
            if (g.has_proj) {
              const double f = low_pass_filter_term(dpw, dph, cos_view, o, P.opt.lowpass_radius);
              if (f > a_kernel) {
                a = f;
                lp = true;
              }
            }
          }
        }
        if (cont && !skip && a >= P.opt.alpha_min) {
          a = dmin(a, 1.0 - 1e-6);
          rec = true;
          float r0, r1, r2c;
          sh_rgb(P, id, r0, r1, r2c);
          cl[0] = r0 < 0;
          cl[1] = r1 < 0;
          cl[2] = r2c < 0;
          rgbf[0] = cl[0] ? 0.f : r0;
          rgbf[1] = cl[1] ? 0.f : r1;
          rgbf[2] = cl[2] ? 0.f : r2c;
        }
      }
    }
    // upstream scalars (grad.cpp:224-233)
    double wb = 0, dat = 0, sgn = 0;
    if (rec) {
      sgn = denom < 0 ? 1.0 : -1.0;
      wb = T * a;
      const double cw = (dC[0] * rgbf[0] + dC[1] * rgbf[1] + dC[2] * rgbf[2]) + dD * rt +
                        (dN[0] * (sgn * rz[0]) + dN[1] * (sgn * rz[1]) + dN[2] * (sgn * rz[2])) + dA;
      rest -= wb * cw;
      dat = T * cw - rest / (1.0 - a);
      P.touched[id] = 1;
      ++n_comp;
    }
    // per-record activated-space gradient (grad.cpp:237-301, :16-101)
    float dcen[3] = {0, 0, 0}, drot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    float deta = 0, dtau = 0, dop = 0, ds_lo = 0, ds_hi = 0, da_lo = 0, da_hi = 0;
    int lo = 0, hi = 0;
    if (rec) {
      if (F64)
        record_grad_f64(P, id, *gp, rt, u, v, a, lp, ev, denom, dpw, dph, wb, dat, sgn, dcen, drot, deta, dtau, dop,
                        ds_lo, ds_hi, da_lo, da_hi, lo, hi);
      else
        record_grad_f32(P, id, *gp, rt, u, v, r2, a, lp, kf, denom, dpw, dph, wb, dat, sgn, dcen, drot, deta, dtau,
                        dop, ds_lo, ds_hi, da_lo, da_hi, lo, hi);
    }
    const float wc0 = rec && !cl[0] ? (float)(wb * dC[0]) : 0.f;
    const float wc1 = rec && !cl[1] ? (float)(wb * dC[1]) : 0.f;
    const float wc2 = rec && !cl[2] ? (float)(wb * dC[2]) : 0.f;
    // Component c of this lane's gradient row (layout kGOff*); c is a
    // compile-time constant at every call site, so nothing is indexed.
    auto comp = [&](const int c) -> float {
      if (c < 3) return dcen[c];
      if (c < kGOffSc) return drot[c - 3];
      if (c < kGOffAn) return (c - kGOffSc == lo ? ds_lo : 0.f) + (c - kGOffSc == hi ? ds_hi : 0.f);
      if (c < kGOffEta) return (c - kGOffAn == lo ? da_lo : 0.f) + (c - kGOffAn == hi ? da_hi : 0.f);
      if (c == kGOffEta) return deta;
      if (c == kGOffTau) return dtau;
      if (c == kGOffOp) return dop;
      const int t = (c - kGOffSh) / 3, ch = (c - kGOffSh) % 3;
      if (t >= 16) return 0.f;
      return (ch == 0 ? wc0 : (ch == 1 ? wc1 : wc2)) * basis[t];
    };
    // Transpose-reduce: lanes are grouped by primitive (the first remaining
    // record's primitive, twice per step); per chunk of 32 components, 5
    // halving steps (16+8+4+2+1 = 31 shuffles) leave lane l with the group sum
    // of component (chunk + l); lanes 4m gather four and issue one
    // red.global.add.v4.f32.  Records of a third or later primitive in the
    // same step add their own components directly.
    const unsigned recmask = __ballot_sync(FULL, rec);
    unsigned remaining = recmask;
    if (recmask && lane == __ffs(recmask) - 1) ++n_rej1;  // warp steps (backward reuses the counter)
    const int G = P.G;
    for (int pass = 0; pass < 2 && remaining; ++pass) {
      const int lead = __ffs(remaining) - 1;
      const int gid = __shfl_sync(FULL, id, lead);
      const bool in_g = rec && id == gid && ((remaining >> lane) & 1u);
      remaining &= ~__ballot_sync(FULL, in_g);
      if (lane == lead) ++n_rej2;  // groups reduced (backward reuses the counter)
      float* pg = P.gact + (size_t)gid * G;
#pragma unroll
      for (int base = 0; base < kGradSlotStride; base += 32) {
        if (base >= G) break;
        float x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = in_g ? comp(base + i) : 0.f;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < off; ++i) {
            const float send = up ? x[i] : x[i + off];
            const float keep = up ? x[i + off] : x[i];
            x[i] = keep + __shfl_xor_sync(FULL, send, off);
          }
        }
        const float x1 = __shfl_down_sync(FULL, x[0], 1), x2 = __shfl_down_sync(FULL, x[0], 2),
                    x3 = __shfl_down_sync(FULL, x[0], 3);
        const int c = base + lane;
        if ((lane & 3) == 0 && c < G && (x[0] != 0.f || x1 != 0.f || x2 != 0.f || x3 != 0.f))
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(pg + c), "f"(x[0]), "f"(x1), "f"(x2),
                       "f"(x3)
                       : "memory");
      }
    }
    if (rec && ((remaining >> lane) & 1u)) {
      float* po = P.gact + (size_t)id * G;
#pragma unroll
      for (int c = 0; c < kGOffSc; ++c)
        if (comp(c) != 0.f) atomicAdd(po + c, comp(c));
      if (ds_lo != 0.f) atomicAdd(po + kGOffSc + lo, ds_lo);
      if (ds_hi != 0.f) atomicAdd(po + kGOffSc + hi, ds_hi);
      if (da_lo != 0.f) atomicAdd(po + kGOffAn + lo, da_lo);
      if (da_hi != 0.f) atomicAdd(po + kGOffAn + hi, da_hi);
      if (deta != 0.f) atomicAdd(po + kGOffEta, deta);
      if (dtau != 0.f) atomicAdd(po + kGOffTau, dtau);
      if (dop != 0.f) atomicAdd(po + kGOffOp, dop);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        if (t < P.opt.terms_active) {
          if (wc0 != 0.f) atomicAdd(po + kGOffSh + 3 * t, wc0 * basis[t]);
          if (wc1 != 0.f) atomicAdd(po + kGOffSh + 3 * t + 1, wc1 * basis[t]);
          if (wc2 != 0.f) atomicAdd(po + kGOffSh + 3 * t + 2, wc2 * basis[t]);
        }
      }
    }
    if (rec) {
      T = xm(T, xs(1.0, a));
      // the fp32 forward's termination (its count is exact for unflagged
      // pixels); fp64 kernels decide on their own exact T
      cont = (!F64 && P.pxstop) ? n_comp < P.pxstop[pix] : T >= P.opt.early_stop;
    }
    return cont;
  }

  // fp32 gradient of one record (grad.cpp:237-301 and backward_alpha
  // grad.cpp:16-101) differentiating the fp32 evaluation kf: the bracket
  // angle terms use delta (theta - a_lo = delta gap / pi), the endpoint
  // tangents are (-e_y, e_x), and cos/sin(delta) come from the half angle.
  __device__ __forceinline__ void record_grad_f32(const RasterParams& P, int id, const Geo& g, double rt, double u,
                                                  double v, double r2, double a, bool lp, const KEvalF& k,
                                                  double denom, double dpw, double dph, double wb, double dat,
                                                  double sgn, float (&dcen)[3], float (&drot)[9], float& deta,
                                                  float& dtau, float& dop, float& ds_lo, float& ds_hi, float& da_lo,
                                                  float& da_hi, int& lo, int& hi) const {
    const float wbf = (float)wb, denf = (float)denom, datf = (float)dat, af = (float)a;
    const float df[3] = {(float)dir[0], (float)dir[1], (float)dir[2]};
    const float rzf[3] = {(float)g.rz[0], (float)g.rz[1], (float)g.rz[2]};
    float hv[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) hv[q] = (float)(P.cam.o[q] + rt * dir[q] - g.mu[q]);
    if (has_dN)
#pragma unroll
      for (int q = 0; q < 3; ++q) drot[3 * q + 2] += wbf * (float)(sgn * dN[q]);
    if (dD != 0) {
      const float d_rt = wbf * (float)dD;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        dcen[q] += d_rt * rzf[q] / denf;
        drot[3 * q + 2] += d_rt * (-hv[q] / denf);
      }
    }
    if (a >= 1.0 - 1e-6 - 1e-12) return;  // alpha clamped
    const float o = (float)P.S.o[id];
    if (lp) {
      const float cv = fabsf(denf), sl = (float)P.opt.lowpass_radius;
      const float dpwf = (float)dpw, dphf = (float)dph;
      dop += datf * af / o;
      const float inv = 1.0f / (cv * cv * sl * sl);
      const float d_dpw = datf * af * (-dpwf * inv), d_dph = datf * af * (-dphf * inv);
      const float d_cos = datf * af * (dpwf * dpwf + dphf * dphf) * inv / cv;
      double J[6];
      projection_jacobian(P.cam, g.mu, J);
      const float sg = denf < 0 ? -1.0f : 1.0f;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        dcen[q] += -((float)J[q] * d_dpw + (float)J[3 + q] * d_dph);
        drot[3 * q + 2] += d_cos * sg * df[q];
      }
      return;
    }
    const float tau = (float)P.S.tau[id];
    dop += datf * k.P;
    if (k.center) return;
    dtau += datf * o *
            (k.br == 0 ? -2.0f * k.g / ((1.0f + tau) * (1.0f + tau))
                       : (k.br == 1 ? (2.0f * k.g - 1.0f) / ((1.0f - tau) * (1.0f - tau))
                                    : (2.0f - 2.0f * k.g) / ((1.0f + tau) * (1.0f + tau))));
    if (k.clamped) return;
    const int K = P.S.K;
    lo = k.lo;
    hi = k.hi;
    const size_t bl = (size_t)id * K + lo, bh = (size_t)id * K + hi;
    const float eta = (float)P.S.eta[id], r2f = (float)r2;
    const float d_q = datf * o * k.A * (-0.5f * k.g);
    const float hlo = P.S.hf[bl], hhi = P.S.hf[bh];
    const float slo = (float)P.S.s[bl], shi = (float)P.S.s[bh];
    deta += d_q * (k.r1 * k.r1 - r2f * k.inv);
    const float d_r1 = d_q * eta * 2.0f * k.r1;
    const float d_r2sq = d_q * (1.0f - eta) * k.inv;
    const float d_inv = d_q * (1.0f - eta) * r2f;
    ds_lo = d_inv * (-2.0f * k.ch * k.ch * hlo / slo);
    ds_hi = d_inv * (-2.0f * k.sh * k.sh * hhi / shi);
    const float d_delta = -(d_inv * 0.5f * (hlo - hhi)) * (2.0f * k.sh * k.ch);
    const float d_tfd = d_delta * P.S.piogf[bl];
    const float dl = k.delta * (float)(1.0 / kPi);
    da_lo = d_tfd * (dl - 1.0f);
    da_hi = -d_tfd * dl;
    const float uf = (float)u, vf = (float)v, r2s = fmaxf(r2f, 1e-24f);
    const float sa = k.a > 0.f ? 1.f : (k.a < 0.f ? -1.f : 0.f);
    const float sb = k.b > 0.f ? 1.f : (k.b < 0.f ? -1.f : 0.f);
    const float elx = (float)P.S.ex[bl], ely = (float)P.S.ey[bl];
    const float ehx = (float)P.S.ex[bh], ehy = (float)P.S.ey[bh];
    const float invd = P.S.invdetf[bl];
    const float du = d_tfd * (-vf / r2s) + 2.0f * d_r2sq * uf + d_r1 * (sa * ehy - sb * ely) * invd;
    const float dv = d_tfd * (uf / r2s) + 2.0f * d_r2sq * vf + d_r1 * (sb * elx - sa * ehx) * invd;
    ds_lo += d_r1 * (-sa * k.a / slo);
    ds_hi += d_r1 * (-sb * k.b / shi);
    const float cross = ehy * ely + ehx * elx;
    da_lo += d_r1 * invd * (sa * k.a * cross - sb * k.a * slo * slo);
    da_hi += d_r1 * invd * (sa * k.b * shi * shi - sb * k.b * cross);
    // (u, v) and r_t chain to centre and rotation columns (grad.cpp:290-300)
    const float rxf[3] = {(float)g.rx[0], (float)g.rx[1], (float)g.rx[2]};
    const float ryf[3] = {(float)g.ry[0], (float)g.ry[1], (float)g.ry[2]};
    const float drx = df[0] * rxf[0] + df[1] * rxf[1] + df[2] * rxf[2];
    const float dry = df[0] * ryf[0] + df[1] * ryf[1] + df[2] * ryf[2];
    const float f = -(du * drx + dv * dry) / denf;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      dcen[q] += du * (rzf[q] * (drx / denf) - rxf[q]) + dv * (rzf[q] * (dry / denf) - ryf[q]);
      drot[3 * q + 0] += du * hv[q];
      drot[3 * q + 1] += dv * hv[q];
      drot[3 * q + 2] += f * hv[q];
    }
  }

  // fp64 gradient of one record (grad.cpp:237-301, :16-101) from the fp64
  // evaluation ev, in the reference's formulation (F64 kernels).
  __device__ void record_grad_f64(const RasterParams& P, int id, const Geo& g, double rt, double u, double v,
                                  double a, bool lp, const KEval& ev, double denom, double dpw, double dph, double wb,
                                  double dat, double sgn, float (&dcen_o)[3], float (&drot_o)[9], float& deta_o,
                                  float& dtau_o, float& dop_o, float& ds_lo_o, float& ds_hi_o, float& da_lo_o,
                                  float& da_hi_o, int& lo_o, int& hi_o) const {
    const int K = P.S.K;
    const double rz[3] = {g.rz[0], g.rz[1], g.rz[2]};
    double dcen[3] = {0, 0, 0}, drot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double deta = 0, dtau = 0, dop = 0, ds_lo = 0, ds_hi = 0, da_lo = 0, da_hi = 0;
    int lo = 0, hi = 0;
    if (has_dN)
      for (int q = 0; q < 3; ++q) drot[3 * q + 2] += wb * sgn * dN[q];
    if (dD != 0) {
      const double d_rt = wb * dD;
      for (int q = 0; q < 3; ++q) {
        const double h = P.cam.o[q] + rt * dir[q] - g.mu[q];
        dcen[q] += d_rt * rz[q] / denom;
        drot[3 * q + 2] += d_rt * (-h / denom);
      }
    }
    const bool alpha_clamped = a >= 1.0 - 1e-6 - 1e-12;
    const double o = P.S.o[id];
    if (!alpha_clamped && lp) {
      const double cv = fabs(denom), sl = P.opt.lowpass_radius;
      dop += dat * a / o;
      const double inv = 1.0 / (cv * cv * sl * sl);
      const double d_dpw = dat * a * (-dpw * inv);
      const double d_dph = dat * a * (-dph * inv);
      const double d_cos = dat * a * (dpw * dpw + dph * dph) * inv / cv;
      double J[6];
      projection_jacobian(P.cam, g.mu, J);
      for (int q = 0; q < 3; ++q) dcen[q] += -(J[q] * d_dpw + J[3 + q] * d_dph);
      const double sg = denom < 0 ? -1.0 : 1.0;
      for (int q = 0; q < 3; ++q) drot[3 * q + 2] += d_cos * sg * dir[q];
    } else if (!alpha_clamped) {
      const double tau = P.S.tau[id];
      dop += dat * sharpen(ev.g, tau);
      if (!ev.center) {
        const int br = sharpen_branch(ev.g, tau);
        dtau += dat * o * sharpen_dtau(br, ev.g, tau);
        if (!ev.clamped) {
          const double d_g = dat * o * sharpen_slope(br, tau);
          const double d_q = d_g * (-0.5 * ev.g);
          lo = ev.lo;
          hi = ev.hi;
          const double* s = P.S.s + (size_t)id * K;
          const double* th = P.S.th + (size_t)id * K;
          const double slo = s[lo], shi = s[hi], eta = P.S.eta[id];
          deta += d_q * (ev.r1 * ev.r1 - ev.r2 * ev.inv_sbar);
          const double d_r1 = d_q * eta * 2.0 * ev.r1;
          const double d_r2sq = d_q * (1.0 - eta) * ev.inv_sbar;
          const double d_inv = d_q * (1.0 - eta) * ev.r2;
          const double c = cos(ev.delta);
          ds_lo = d_inv * (-(1.0 + c) / (slo * slo * slo));
          ds_hi = d_inv * (-(1.0 - c) / (shi * shi * shi));
          const double d_c = d_inv * (0.5 / (slo * slo) - 0.5 / (shi * shi));
          const double d_delta = d_c * (-sin(ev.delta));
          double alo = th[lo], ahi = th[hi], theta = ev.theta;
          if (hi == 0) {
            alo -= kTwoPi;
            if (theta > th[K - 1]) theta -= kTwoPi;
          }
          const double gap = ahi - alo;
          const double d_tfd = d_delta * kPi / gap;
          da_lo = d_delta * kPi * (theta - ahi) / (gap * gap);
          da_hi = d_delta * (-kPi) * (theta - alo) / (gap * gap);
          const double r2s = dmax(ev.r2, 1e-24);
          double du = d_tfd * (-v / r2s);
          double dv = d_tfd * (u / r2s);
          du += d_r2sq * 2.0 * u;
          dv += d_r2sq * 2.0 * v;
          const double sa = ev.a > 0 ? 1 : (ev.a < 0 ? -1 : 0);
          const double sb = ev.b > 0 ? 1 : (ev.b < 0 ? -1 : 0);
          const double elx = P.S.ex[(size_t)id * K + lo], ely = P.S.ey[(size_t)id * K + lo];
          const double ehx = P.S.ex[(size_t)id * K + hi], ehy = P.S.ey[(size_t)id * K + hi];
          const double det = P.S.det[(size_t)id * K + lo];
          du += d_r1 * (sa * (ehy / det) + sb * (-ely / det));
          dv += d_r1 * (sa * (-ehx / det) + sb * (elx / det));
          const double ca = cos(th[lo]), sa_lo = sin(th[lo]);
          const double cb = cos(th[hi]), sb_hi = sin(th[hi]);
          ds_lo += d_r1 * (-sa * ev.a / slo);
          ds_hi += d_r1 * (-sb * ev.b / shi);
          const double tlx = -slo * sa_lo, tly = slo * ca, thx = -shi * sb_hi, thy = shi * cb;
          const double na = -ev.a, nb = -ev.b;
          da_lo += d_r1 * (sa * (na * ((ehy * tlx - ehx * tly) / det)) + sb * (na * ((-ely * tlx + elx * tly) / det)));
          da_hi += d_r1 * (sa * (nb * ((ehy * thx - ehx * thy) / det)) + sb * (nb * ((-ely * thx + elx * thy) / det)));
          const double hh[3] = {P.cam.o[0] + rt * dir[0] - g.mu[0], P.cam.o[1] + rt * dir[1] - g.mu[1],
                                P.cam.o[2] + rt * dir[2] - g.mu[2]};
          const double drx = dir[0] * g.rx[0] + dir[1] * g.rx[1] + dir[2] * g.rx[2];
          const double dry = dir[0] * g.ry[0] + dir[1] * g.ry[1] + dir[2] * g.ry[2];
          const double f = -(du * drx + dv * dry) / denom;
          for (int q = 0; q < 3; ++q) {
            dcen[q] += du * (rz[q] * (drx / denom) - g.rx[q]) + dv * (rz[q] * (dry / denom) - g.ry[q]);
            drot[3 * q + 0] += du * hh[q];
            drot[3 * q + 1] += dv * hh[q];
            drot[3 * q + 2] += f * hh[q];
          }
        }
      }
    }
    for (int q = 0; q < 3; ++q) dcen_o[q] = (float)dcen[q];
    for (int q = 0; q < 9; ++q) drot_o[q] = (float)drot[q];
    deta_o = (float)deta;
    dtau_o = (float)dtau;
    dop_o = (float)dop;
    ds_lo_o = (float)ds_lo;
    ds_hi_o = (float)ds_hi;
    da_lo_o = (float)da_lo;
    da_hi_o = (float)da_hi;
    lo_o = lo;
    hi_o = hi;
  }

  // SH colour (geometry.cpp:126-138) in fp32, before the clamp at zero.
  // Coefficients are AoS (terms x RGB); groups of 4 terms (12 floats) are
  // read as 3 x float4 when the layout allows it.
  __device__ __forceinline__ void sh_rgb(const RasterParams& P, int id, float& r0, float& r1, float& r2) const {
    const float* shp = P.sh + (size_t)id * P.terms * 3;
    r0 = 0.5f;
    r1 = 0.5f;
    r2 = 0.5f;
    // Loops are fully unrolled over the 16 possible terms (guarded) so that
    // basis[] stays in registers.
    const int ta = P.opt.terms_active;
    if ((P.terms & 3) == 0 && (ta & 3) == 0) {
      const float4* q = reinterpret_cast<const float4*>(shp);
#pragma unroll
      for (int t = 0; t < 16; t += 4) {
        if (t < ta) {
          const float4 a = __ldg(q + 3 * (t / 4)), b = __ldg(q + 3 * (t / 4) + 1), c = __ldg(q + 3 * (t / 4) + 2);
          r0 += basis[t] * a.x;
          r1 += basis[t] * a.y;
          r2 += basis[t] * a.z;
          r0 += basis[t + 1] * a.w;
          r1 += basis[t + 1] * b.x;
          r2 += basis[t + 1] * b.y;
          r0 += basis[t + 2] * b.z;
          r1 += basis[t + 2] * b.w;
          r2 += basis[t + 2] * c.x;
          r0 += basis[t + 3] * c.y;
          r1 += basis[t + 3] * c.z;
          r2 += basis[t + 3] * c.w;
        }
      }
      return;
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      if (t < ta) {
        r0 += basis[t] * __ldg(shp + 3 * t);
        r1 += basis[t] * __ldg(shp + 3 * t + 1);
        r2 += basis[t] * __ldg(shp + 3 * t + 2);
      }
    }
  }

  // SH colour in fp64 (geometry.cpp:126-138, reference op order, rounded
  // explicitly) from the pixel's fp64 ray; coefficients from the fp64 copy when
  // the caller gave one, else the f32 ones widened.  Before the clamp at zero.
  __device__ void sh_rgb_d(const RasterParams& P, int id, double rgb[3]) const {
    const double* b = basis64;
    rgb[0] = rgb[1] = rgb[2] = 0.5;
    const int ta = P.opt.terms_active;
    const size_t base = (size_t)id * P.terms * 3;
    for (int t = 0; t < ta; ++t)
      for (int c = 0; c < 3; ++c) {
        const double s = P.sh64 ? P.sh64[base + 3 * t + c] : (double)P.sh[base + 3 * t + c];
        rgb[c] = xa(rgb[c], xm(b[t], s));
      }
  }

  __device__ void finish_forward(const RasterParams& P) {
    const size_t p = (size_t)pix;
    const double c0 = xa(C[0], xm(T, P.opt.bg[0]));  // raster.cpp:420
    const double c1 = xa(C[1], xm(T, P.opt.bg[1]));
    const double c2 = xa(C[2], xm(T, P.opt.bg[2]));
    if (P.color) {
      P.color[3 * p] = (float)c0;
      P.color[3 * p + 1] = (float)c1;
      P.color[3 * p + 2] = (float)c2;
    }
    if (P.normal) {
      P.normal[3 * p] = (float)N[0];
      P.normal[3 * p + 1] = (float)N[1];
      P.normal[3 * p + 2] = (float)N[2];
    }
    if (P.depth) P.depth[p] = (float)D;
    if (P.alpha) P.alpha[p] = (float)A;
    if (!F64 && P.pxstop) P.pxstop[p] = stop;
    if (P.pxcomp) P.pxcomp[p] = (int)n_comp;
    if (P.pxstate) {
      double* st = P.pxstate + 8 * p;
      st[0] = c0;
      st[1] = c1;
      st[2] = c2;
      st[3] = D;
      st[4] = N[0];
      st[5] = N[1];
      st[6] = N[2];
      st[7] = A;
    }
    if (P.replay_cap > 0) {
      P.replay_cnt[p] = n_rec;
      if (n_rec > P.replay_cap) atomicAdd(&P.counters[C_REPLAY_OVERFLOW], 1ull);
    }
    if (!F64 && P.pxflag) {
      P.pxflag[p] = uncertain ? 1 : 0;
      if (uncertain) P.redo_list[atomicAdd(P.redo_count, 1u)] = pix;
    }
  }
};

// MODE 0: SortCache streaming; MODE 1: list order (use_cache = false).
// F64: re-render of the pixels flagged by the fp32 pass.
template <int MODE, bool BWD, bool F64>
__global__ void __launch_bounds__(256, DRK_RASTER_MIN_BLOCKS) k_raster(RasterParams P) {
  __shared__ int s_id[256];
  __shared__ double s_num[256], s_r0[256], s_r1[256], s_r2[256];
  const int tile = P.tile_base + blockIdx.x;
  const int tx = tile % P.cam.tiles_x, ty = tile / P.cam.tiles_x;
  const int x = tx * kTile + ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7),
            y = ty * kTile + (threadIdx.x >> 6) * 4 + ((threadIdx.x & 31) >> 3);  // 8 x 4 per warp
  bool active = x < P.cam.W && y < P.cam.H;
  if (P.pxflag && (F64 || BWD) && active) {
    const bool flagged = P.pxflag[(size_t)y * P.cam.W + x] != 0;
    active = F64 ? flagged : !flagged;  // the fp64 launch owns the flagged pixels
  }
  if (F64 && __syncthreads_count(active) == 0) return;
  Pixel<BWD, F64> px;
  px.init(P, x, y);
  if (BWD && active) px.init_bwd(P);
  bool done = !active;
  long long streamed = 0;
  double cd[kCacheCap];
  int ci[kCacheCap];
  int csz = 0;
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  const double eps = P.opt.grazing_eps;
  for (long long b0 = beg; b0 < end; b0 += 256) {
    __syncthreads();
    const long long j = b0 + threadIdx.x;
    if (j < end) {
      const int id = P.lid[j];
      const Geo& g = P.geo[id];
      s_id[threadIdx.x] = id;
      s_num[threadIdx.x] = g.num;
      s_r0[threadIdx.x] = g.rz[0];
      s_r1[threadIdx.x] = g.rz[1];
      s_r2[threadIdx.x] = g.rz[2];
    }
    __syncthreads();
    const int cnt = (int)min((long long)256, end - b0);
    if (!done) {
      for (int c = 0; c < cnt; ++c) {
        // classify_intersect (geometry.cpp:40-46)
        const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], s_r0[c], s_r1[c], s_r2[c]);
        if (fabs(denom) < eps) continue;
        const double rt = s_num[c] / denom;
        if (rt <= 0) continue;
        ++streamed;
        const int id = s_id[c];
        if (MODE == 1) {
          if (!px.composite(P, rt, id)) {
            done = true;
            break;
          }
          continue;
        }
        // SortCache::step (raster.cpp:267-303)
        int pos = 0;
#pragma unroll
        for (int q = 0; q < kCacheCap; ++q) pos += (q < csz && cd[q] <= rt) ? 1 : 0;
        if (csz < kCacheCap) {
#pragma unroll
          for (int q = kCacheCap - 1; q > 0; --q)
            if (q > pos) {
              cd[q] = cd[q - 1];
              ci[q] = ci[q - 1];
            }
#pragma unroll
          for (int q = 0; q < kCacheCap; ++q)
            if (q == pos) {
              cd[q] = rt;
              ci[q] = id;
            }
          ++csz;
          continue;
        }
        double prt;
        int pid;
        if (pos == 0) {  // incoming is the new minimum: pops straight through
          prt = rt;
          pid = id;
        } else {
          prt = cd[0];
          pid = ci[0];
#pragma unroll
          for (int q = 0; q < kCacheCap; ++q) {
            if (q < pos - 1) {
              if (q + 1 < kCacheCap) {
                cd[q] = cd[q + 1];
                ci[q] = ci[q + 1];
              }
            } else if (q == pos - 1) {
              cd[q] = rt;
              ci[q] = id;
            }
          }
        }
        if (!px.composite(P, prt, pid)) {
          done = true;
          break;
        }
      }
    }
    if (__syncthreads_count(!done) == 0) break;
  }
  // end marker: drain the cache head first (raster.cpp:410-414)
  if (MODE == 0) {
    while (!done && csz > 0) {
      const double prt = cd[0];
      const int pid = ci[0];
#pragma unroll
      for (int q = 0; q < kCacheCap - 1; ++q) {
        cd[q] = cd[q + 1];
        ci[q] = ci[q + 1];
      }
      --csz;
      if (!px.composite(P, prt, pid)) done = true;
    }
  }
  if (!active) return;
  if (px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  if (!BWD) {
    px.finish_forward(P);
    unsigned long long s = streamed, pp = px.n_pop, cc = px.n_comp;
    if (F64) {
      atomicAdd(&P.counters[C_REDO_PIXELS], 1ull);
    } else {
      atomicAdd(&P.counters[C_STREAMED], s);
      atomicAdd(&P.counters[C_POPPED], pp);
      atomicAdd(&P.counters[C_COMPOSITED], cc);
      atomicAdd(&P.counters[C_REJECT_RADIUS], (unsigned long long)px.n_rej1);
      atomicAdd(&P.counters[C_REJECT_BRACKET], (unsigned long long)px.n_rej2);
      atomicAdd(&P.counters[C_FP64_EVALS], (unsigned long long)px.n_f64);
    }
  }
}

// Backward rasterizer: re-streams the forward decisions with warp-uniform
// control flow so that gradient components can be reduced across lanes
// (Pixel::composite_warp).  MODE / F64 as in k_raster.
template <int MODE, bool F64>
__global__ void __launch_bounds__(256, DRK_BWD_MIN_BLOCKS) k_raster_bwd(RasterParams P) {
  __shared__ int s_id[256];
  __shared__ double s_num[256], s_r0[256], s_r1[256], s_r2[256];
  const unsigned FULL = 0xffffffffu;
  const int tile = P.tile_base + blockIdx.x;
  const int tx = tile % P.cam.tiles_x, ty = tile / P.cam.tiles_x;
  const int x = tx * kTile + ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7),
            y = ty * kTile + (threadIdx.x >> 6) * 4 + ((threadIdx.x & 31) >> 3);  // 8 x 4 per warp
  bool active = x < P.cam.W && y < P.cam.H;
  if (P.pxflag && active) {
    const bool flagged = P.pxflag[(size_t)y * P.cam.W + x] != 0;
    active = F64 ? flagged : !flagged;
  }
  if (__syncthreads_count(active) == 0) return;
  Pixel<true, F64> px;
  px.init(P, x, y);
  px.dC[0] = px.dC[1] = px.dC[2] = px.dD = px.dN[0] = px.dN[1] = px.dN[2] = px.dA = px.rest = 0;
  px.has_dN = P.dN != nullptr;
  if (active) px.init_bwd(P);
  bool done = !active;
  double cd[kCacheCap];
  int ci[kCacheCap];
  int csz = 0;
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  const double eps = P.opt.grazing_eps;
  // Batches of 256 candidates, then (MODE 0) one drain pass over the cache
  // (raster.cpp:410-414) through the same call site, so composite_warp is
  // instantiated once.
  const long long nb = (end - beg + 255) / 256;
  for (long long bi = 0; bi <= nb; ++bi) {
    const bool drain = bi == nb;
    if (drain && MODE != 0) break;
    const long long b0 = beg + bi * 256;
    int cnt = kCacheCap;
    if (!drain) {
      __syncthreads();
      const long long j = b0 + threadIdx.x;
      if (j < end) {
        const int id = P.lid[j];
        const Geo& g = P.geo[id];
        s_id[threadIdx.x] = id;
        s_num[threadIdx.x] = g.num;
        s_r0[threadIdx.x] = g.rz[0];
        s_r1[threadIdx.x] = g.rz[1];
        s_r2[threadIdx.x] = g.rz[2];
      }
      __syncthreads();
      cnt = (int)min((long long)256, end - b0);
    }
    if (__any_sync(FULL, !done)) {
      for (int c = 0; c < cnt; ++c) {
        bool want = false;
        double prt = 0;
        int pid = -1;
        if (drain) {
          if (!done && csz > 0) {
            want = true;
            prt = cd[0];
            pid = ci[0];
#pragma unroll
            for (int q = 0; q < kCacheCap - 1; ++q) {
              cd[q] = cd[q + 1];
              ci[q] = ci[q + 1];
            }
            --csz;
          }
        } else if (!done) {
          const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], s_r0[c], s_r1[c], s_r2[c]);
          if (fabs(denom) >= eps) {
            const double rt = s_num[c] / denom;
            if (rt > 0) {
              const int id = s_id[c];
              if (MODE == 1) {
                want = true;
                prt = rt;
                pid = id;
              } else {
                int pos = 0;
#pragma unroll
                for (int q = 0; q < kCacheCap; ++q) pos += (q < csz && cd[q] <= rt) ? 1 : 0;
                if (csz < kCacheCap) {
#pragma unroll
                  for (int q = kCacheCap - 1; q > 0; --q)
                    if (q > pos) {
                      cd[q] = cd[q - 1];
                      ci[q] = ci[q - 1];
                    }
#pragma unroll
                  for (int q = 0; q < kCacheCap; ++q)
                    if (q == pos) {
                      cd[q] = rt;
                      ci[q] = id;
                    }
                  ++csz;
                } else {
                  want = true;
                  if (pos == 0) {
                    prt = rt;
                    pid = id;
                  } else {
                    prt = cd[0];
                    pid = ci[0];
#pragma unroll
                    for (int q = 0; q < kCacheCap; ++q) {
                      if (q < pos - 1) {
                        if (q + 1 < kCacheCap) {
                          cd[q] = cd[q + 1];
                          ci[q] = ci[q + 1];
                        }
                      } else if (q == pos - 1) {
                        cd[q] = rt;
                        ci[q] = id;
                      }
                    }
                  }
                }
              }
            }
          }
        }
        if (__any_sync(FULL, want)) {
          const bool cont = px.composite_warp(P, want, prt, pid);
          if (want && !cont) done = true;
        }
      }
    }
    if (drain || __syncthreads_count(!done) == 0) break;
  }
  if (active && px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  if (px.n_rej1) atomicAdd(&P.counters[C_BWD_WARPSTEPS], (unsigned long long)px.n_rej1);
  if (px.n_rej2) atomicAdd(&P.counters[C_BWD_LEAD_RECORDS], (unsigned long long)px.n_rej2);
}

// SortCache::step (raster.cpp:267-303) on a register cache; returns true and
// the popped entry when the step pops.
__device__ __forceinline__ bool cache_step(double (&cd)[kCacheCap], int (&ci)[kCacheCap], int& csz, double rt, int id,
                                           double& prt, int& pid) {
  int pos = 0;
#pragma unroll
  for (int q = 0; q < kCacheCap; ++q) pos += (q < csz && cd[q] <= rt) ? 1 : 0;
  if (csz < kCacheCap) {
#pragma unroll
    for (int q = kCacheCap - 1; q > 0; --q)
      if (q > pos) {
        cd[q] = cd[q - 1];
        ci[q] = ci[q - 1];
      }
#pragma unroll
    for (int q = 0; q < kCacheCap; ++q)
      if (q == pos) {
        cd[q] = rt;
        ci[q] = id;
      }
    ++csz;
    return false;
  }
  if (pos == 0) {
    prt = rt;
    pid = id;
    return true;
  }
  prt = cd[0];
  pid = ci[0];
#pragma unroll
  for (int q = 0; q < kCacheCap; ++q) {
    if (q < pos - 1) {
      if (q + 1 < kCacheCap) {
        cd[q] = cd[q + 1];
        ci[q] = ci[q + 1];
      }
    } else if (q == pos - 1) {
      cd[q] = rt;
      ci[q] = id;
    }
  }
  return true;
}

// fp64 re-render of the pixels flagged by the fp32 pass (uncertain
// early-stop decision): one thread per listed pixel streams its tile list
// straight from L2 with fp64 alpha (forward: outputs overwritten; backward:
// per-record atomics).
// One pixel, fp64 alpha, sequential over its tile list.  MODE 0: SortCache,
// 1: list order, 2: exact sort by (depth, list index).
template <int MODE, bool BWD>
__device__ void process_pixel(const RasterParams& P, int pix) {
  const int x = pix % P.cam.W, y = pix / P.cam.W;
  const int tile = (y / kTile) * P.cam.tiles_x + (x / kTile);
  Pixel<BWD, true> px;
  px.init(P, x, y);
  if (BWD) px.init_bwd(P);
  double cd[kCacheCap];
  int ci[kCacheCap];
  int csz = 0;
  bool done = false;
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  if (MODE == 2) {
    double last_d = -1.0;
    long long last_j = -1;
    while (!done) {
      double best_d = 0;
      long long best_j = -1;
      for (long long j = beg; j < end; ++j) {
        const Geo& g = P.geo[P.lid[j]];
        const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], g.rz[0], g.rz[1], g.rz[2]);
        if (fabs(denom) < P.opt.grazing_eps) continue;
        const double rt = g.num / denom;
        if (rt <= 0) continue;
        if (!(rt > last_d || (rt == last_d && j > last_j))) continue;
        if (best_j < 0 || rt < best_d) {
          best_d = rt;
          best_j = j;
        }
      }
      if (best_j < 0) break;
      last_d = best_d;
      last_j = best_j;
      done = !px.composite(P, best_d, P.lid[best_j]);
    }
  } else {
    for (long long j = beg; j < end && !done; ++j) {
      const int id = P.lid[j];
      const Geo& g = P.geo[id];
      const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], g.rz[0], g.rz[1], g.rz[2]);
      if (fabs(denom) < P.opt.grazing_eps) continue;
      const double rt = g.num / denom;
      if (rt <= 0) continue;
      if (MODE == 1) {
        done = !px.composite(P, rt, id);
        continue;
      }
      double prt;
      int pid;
      if (cache_step(cd, ci, csz, rt, id, prt, pid)) done = !px.composite(P, prt, pid);
    }
    if (MODE == 0) {
      while (!done && csz > 0) {
        const double prt = cd[0];
        const int pid = ci[0];
#pragma unroll
        for (int q = 0; q < kCacheCap - 1; ++q) {
          cd[q] = cd[q + 1];
          ci[q] = ci[q + 1];
        }
        --csz;
        done = !px.composite(P, prt, pid);
      }
    }
  }
  if (px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  if (!BWD) px.finish_forward(P);
}

// fp64 evaluation of one popped entry (composite_candidate minus the
// transmittance-dependent part): alpha decision, tangent coordinates,
// colour, kernel partials for the backward.
struct PopEval {
  double a, rt, u, v, denom, dpw, dph;
  double rgb[3];
  bool valid, lp, cl[3];
  KEval ev;
  int id;
};

template <bool BWD>
__device__ void eval_pop(const RasterParams& P, const Pixel<BWD, true>& px, double rt, int id, PopEval& e) {
  const Geo& g = P.geo[id];
  e.valid = false;
  e.lp = false;
  e.id = id;
  e.rt = rt;
  e.denom = xdot3(px.dir[0], px.dir[1], px.dir[2], g.rz[0], g.rz[1], g.rz[2]);
  const double h0 = xs(xa(P.cam.o[0], xm(rt, px.dir[0])), g.mu[0]);
  const double h1 = xs(xa(P.cam.o[1], xm(rt, px.dir[1])), g.mu[1]);
  const double h2 = xs(xa(P.cam.o[2], xm(rt, px.dir[2])), g.mu[2]);
  e.u = xdot3(g.rx[0], g.rx[1], g.rx[2], h0, h1, h2);
  e.v = xdot3(g.ry[0], g.ry[1], g.ry[2], h0, h1, h2);
  const double cos_view = fabs(e.denom);
  e.dpw = e.dph = 0;
  if (g.has_proj) {
    e.dpw = xs(px.px, g.ppx);
    e.dph = xs(px.py, g.ppy);
  }
  const double r2 = xa(xm(e.u, e.u), xm(e.v, e.v));
  const bool lp_possible = g.has_proj && e.dpw * e.dpw + e.dph * e.dph <= cos_view * cos_view * g.dp2max;
  e.ev.center = e.ev.clamped = e.ev.degenerate = false;
  if (r2 > g.r2max && !lp_possible) return;
  const double a = alpha64(P.S, id, e.u, e.v, g.has_proj, e.dpw, e.dph, cos_view, P.opt.lowpass_radius, e.ev, e.lp);
  if (e.ev.degenerate) return;
  if (a < P.opt.alpha_min) return;
  e.a = dmin(a, 1.0 - 1e-6);
  if (px.col64) {
    px.sh_rgb_d(P, id, e.rgb);
  } else {  // fp64 re-render of a fast-path frame: fp32 colours like the fast kernel
    float r0, r1, r2c;
    px.sh_rgb(P, id, r0, r1, r2c);
    e.rgb[0] = r0;
    e.rgb[1] = r1;
    e.rgb[2] = r2c;
  }
  for (int c = 0; c < 3; ++c) {
    e.cl[c] = e.rgb[c] < 0;
    if (e.cl[c]) e.rgb[c] = 0.0;
  }
  e.valid = true;
}

// fp64 re-render, one WARP per flagged pixel: lanes intersect 32 list
// entries at once, lane 0 runs the SortCache over them (in order), lanes
// evaluate the popped entries' alpha in parallel, and lane 0 composites
// them in order until saturation (backward: lanes then compute their
// record's gradient with the transmittance / rest lane 0 produced).
template <int MODE, bool BWD>
__global__ void __launch_bounds__(128) k_raster_pixels_warp(RasterParams P) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  constexpr int kPopVals = BWD ? 3 : 9;
  __shared__ double s_pop[4 * 32 * kPopVals];  // per warp: 32 pops x kPopVals (step 3)
  const unsigned total = *P.redo_count;
  // pixels are fetched dynamically (P.redo_count[1] is the fetch counter, zeroed
  // at launch): a warp that drew a long tile list does not hold back a fixed
  // stride of further pixels
  unsigned* fetch = P.redo_count + 1;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(fetch, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= total) break;
    const int pix = P.redo_list[t];
    const int x = pix % P.cam.W, y = pix / P.cam.W;
    const int tile = (y / kTile) * P.cam.tiles_x + (x / kTile);
    Pixel<BWD, true> px;
    px.init(P, x, y);
    if (BWD) px.init_bwd(P);
    // forward: SortCache distributed over lanes 0..7 (lane q holds entry q);
    // backward: replicated on every lane (faster there, measured).  csz is warp-uniform.
    double cdq = 0;
    int ciq = -1;
    double cd[kCacheCap];
    int ci[kCacheCap];
    int csz = 0;
    bool done = false;
    const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
    long long j = beg;
    // software pipeline over 32-entry chunks: the ray-plane constants (num, R_z:
    // the first 32 bytes of Geo) of the next chunk and the ids of the one after
    // are in flight while the current chunk is sorted, evaluated and composited
    // (a long tile list is walked by one warp: load latency is its critical path)
    auto ld_ray = [&](int id) -> double4 {
      if (id < 0) return make_double4(0, 0, 0, 0);
      const double2* q = reinterpret_cast<const double2*>(P.geo + id);
      const double2 a = __ldg(q), b = __ldg(q + 1);
      return make_double4(a.x, a.y, b.x, b.y);  // num, rz0, rz1, rz2
    };
    int id_a = beg + lane < end ? P.lid[beg + lane] : -1;
    int id_b = beg + 32 + lane < end ? P.lid[beg + 32 + lane] : -1;
    double4 g_a = ld_ray(id_a);
    while (!done) {
      // 1) up to 32 pops: parallel intersections, in-order SortCache on lane 0
      double my_rt = 0;
      int my_id = -1, npop = 0;
      bool list_end = j >= end;
      if (!list_end) {
        const long long jj = j + lane;
        double rt = 0;
        const int id = id_a;
        const double4 g = g_a;
        id_a = id_b;
        g_a = ld_ray(id_b);
        id_b = j + 64 + lane < end ? P.lid[j + 64 + lane] : -1;
        bool hit = false;
        if (jj < end) {
          const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], g.y, g.z, g.w);
          if (fabs(denom) >= P.opt.grazing_eps) {
            rt = g.x / denom;
            hit = rt > 0;
          }
        }
        const unsigned hits = __ballot_sync(FULL, hit);
        unsigned rem = hits;
        while (rem) {
          const int k = __ffs(rem) - 1;
          rem &= rem - 1;
          const double rk = __shfl_sync(FULL, rt, k);
          const int ik = __shfl_sync(FULL, id, k);
          bool pop = false;
          double prt = rk;
          int pid = ik;
          if (MODE == 1) {
            pop = true;
          } else if (BWD) {
            pop = cache_step(cd, ci, csz, rk, ik, prt, pid);  // replicated on all lanes
          } else {
            // SortCache::step (raster.cpp:267-303): entries <= rk form a prefix
            const int pos = __popc(__ballot_sync(FULL, lane < csz && cdq <= rk));
            const double upd = __shfl_up_sync(FULL, cdq, 1), dnd = __shfl_down_sync(FULL, cdq, 1);
            const int upi = __shfl_up_sync(FULL, ciq, 1), dni = __shfl_down_sync(FULL, ciq, 1);
            if (csz < kCacheCap) {
              if (lane > pos && lane <= csz) {
                cdq = upd;
                ciq = upi;
              } else if (lane == pos) {
                cdq = rk;
                ciq = ik;
              }
              ++csz;
            } else {
              pop = true;
              if (pos > 0) {  // head pops; entries 1..pos-1 move down, incoming at pos-1
                prt = __shfl_sync(FULL, cdq, 0);
                pid = __shfl_sync(FULL, ciq, 0);
                if (lane < pos - 1) {
                  cdq = dnd;
                  ciq = dni;
                } else if (lane == pos - 1) {
                  cdq = rk;
                  ciq = ik;
                }
              }  // else: the incoming is strictly shallower than the head and pops through
            }
          }
          if (pop) {
            if (lane == npop) {
              my_rt = prt;
              my_id = pid;
            }
            ++npop;
          }
        }
        j += 32;
      } else if (MODE == 0) {
        // end marker: drain the head (up to 8 pops)
        while (BWD && csz > 0 && npop < 32) {
          if (lane == npop) {
            my_rt = cd[0];
            my_id = ci[0];
          }
#pragma unroll
          for (int q = 0; q < kCacheCap - 1; ++q) {
            cd[q] = cd[q + 1];
            ci[q] = ci[q + 1];
          }
          --csz;
          ++npop;
        }
        while (!BWD && csz > 0 && npop < 32) {
          const double h = __shfl_sync(FULL, cdq, 0);
          const int hi = __shfl_sync(FULL, ciq, 0);
          if (lane == npop) {
            my_rt = h;
            my_id = hi;
          }
          const double dnd = __shfl_down_sync(FULL, cdq, 1);
          const int dni = __shfl_down_sync(FULL, ciq, 1);
          if (lane < kCacheCap - 1) {
            cdq = dnd;
            ciq = dni;
          }
          --csz;
          ++npop;
        }
      }
      if (npop == 0) {
        if (list_end) break;
        continue;
      }
      // 2) parallel fp64 evaluation of the pops
      PopEval e;
      e.valid = false;
      if (lane < npop) eval_pop<BWD>(P, px, my_rt, my_id, e);
      if (lane < npop && e.ev.degenerate) px.err = true;
      // 3) in-order compositing (all lanes replicate the scalar state).  Lane k
      // first lays out what pop k contributes (alpha, 1 - alpha, and the colour /
      // depth / normal factors, or the upstream dot product) in the warp's shared
      // slots; the sequential loop then reads them as broadcasts: its critical path
      // is the transmittance product alone (same explicitly rounded operations,
      // same order as a per-pop loop).
      double* slot = s_pop + (threadIdx.x >> 5) * 32 * kPopVals;
      if (lane < npop) {
        double* row = slot + lane * kPopVals;
        row[0] = e.valid ? e.a : -1.0;  // -1: not composited
        if (e.valid) {
          row[1] = xs(1.0, e.a);
          const Geo& g = P.geo[e.id];
          const double sgn = e.denom < 0 ? 1.0 : -1.0;
          const double n0 = sgn * g.rz[0], n1 = sgn * g.rz[1], n2 = sgn * g.rz[2];
          if (!BWD) {
            row[2] = e.rgb[0];
            row[3] = e.rgb[1];
            row[4] = e.rgb[2];
            row[5] = e.rt;
            row[6] = xm(sgn, g.rz[0]);
            row[7] = xm(sgn, g.rz[1]);
            row[8] = xm(sgn, g.rz[2]);
          } else {
            row[2] = (px.dC[0] * e.rgb[0] + px.dC[1] * e.rgb[1] + px.dC[2] * e.rgb[2]) + px.dD * e.rt +
                     (px.dN[0] * n0 + px.dN[1] * n1 + px.dN[2] * n2) + px.dA;
          }
        }
      }
      __syncwarp();
      double wb_mine = 0, dat_mine = 0, T_mine = 1;
      int idx_mine = 0;
      int last_k = npop - 1;
      for (int k = 0; k < npop && !done; ++k) {
        last_k = k;
        const double* row = slot + k * kPopVals;
        const double a = row[0];
        if (a < 0) continue;
        const double w = xm(px.T, a);
        ++px.n_comp;
        if (!BWD) {
          px.C[0] = xa(px.C[0], xm(w, row[2]));
          px.C[1] = xa(px.C[1], xm(w, row[3]));
          px.C[2] = xa(px.C[2], xm(w, row[4]));
          px.D = xa(px.D, xm(w, row[5]));
          px.N[0] = xa(px.N[0], xm(w, row[6]));
          px.N[1] = xa(px.N[1], xm(w, row[7]));
          px.N[2] = xa(px.N[2], xm(w, row[8]));
          px.A = xa(px.A, w);
        } else {
          const double cw = row[2];
          px.rest -= w * cw;
          if (lane == k) {
            wb_mine = w;
            T_mine = px.T;
            dat_mine = px.T * cw - px.rest / (1.0 - a);
            idx_mine = (int)px.n_comp - 1;
          }
        }
        px.T = xm(px.T, row[1]);
        if (px.T < P.opt.early_stop) done = true;
      }
      __syncwarp();
      if (!BWD && P.replay_cap > 0) {
        // replay records in order (lane k writes its own entry)
        int rec_idx = px.n_rec;
        for (int k = 0; k <= last_k; ++k) {
          const bool valid = __shfl_sync(FULL, e.valid, k);
          if (!valid) continue;
          if (lane == k && rec_idx < P.replay_cap) {
            const size_t r = (size_t)px.pix * P.replay_cap + rec_idx;
            P.replay_ids[r] = e.id;
            double* rec = P.replay_rec + 5 * r;
            rec[0] = e.u;
            rec[1] = e.v;
            rec[2] = e.rt;
            rec[3] = e.a;
            rec[4] = e.lp ? 1.0 : 0.0;
          }
          ++rec_idx;
        }
        px.n_rec = rec_idx;
      }
      if (BWD && lane < npop && e.valid && wb_mine != 0) {
        // this lane's record: gradients with the sequential T / rest
        const Geo& g = P.geo[e.id];
        const double rgb[3] = {(double)e.rgb[0], (double)e.rgb[1], (double)e.rgb[2]};
        const double sgn = e.denom < 0 ? 1.0 : -1.0;
        px.backward_record_dat(P, e.id, g, e.rt, e.u, e.v, e.a, e.lp, e.ev, rgb, e.cl[0], e.cl[1], e.cl[2], sgn,
                               e.denom, e.dpw, e.dph, wb_mine, dat_mine, T_mine, idx_mine);
      }
    }
    if (lane == 0) {
      if (px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
      if (!BWD) {
        px.finish_forward(P);
        atomicAdd(&P.counters[C_REDO_PIXELS], 1ull);
      }
    }
  }
}

template <int MODE, bool BWD>
__global__ void __launch_bounds__(128) k_raster_pixels(RasterParams P) {
  const unsigned total = *P.redo_count;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    process_pixel<MODE, BWD>(P, P.redo_list[t]);
    if (!BWD) atomicAdd(&P.counters[C_REDO_PIXELS], 1ull);
  }
}

// exact_sort oracle mode (raster.cpp:395-401): every hit composited in
// stable depth order (fp64 alpha).  One thread per pixel, selection by
// (depth, list index).
template <bool BWD>
__global__ void __launch_bounds__(128) k_raster_exact(RasterParams P) {
  const int tile = P.tile_base + blockIdx.y;
  const int tx = tile % P.cam.tiles_x, ty = tile / P.cam.tiles_x;
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= 256) return;
  const int x = tx * kTile + (l & 15), y = ty * kTile + (l >> 4);
  if (x >= P.cam.W || y >= P.cam.H) return;
  Pixel<BWD, true> px;
  px.init(P, x, y);
  if (BWD) px.init_bwd(P);
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  double last_d = -1.0;
  long long last_j = -1;
  while (true) {
    double best_d = 0;
    long long best_j = -1;
    for (long long j = beg; j < end; ++j) {
      const int id = P.lid[j];
      const Geo& g = P.geo[id];
      const double denom = xdot3(px.dir[0], px.dir[1], px.dir[2], g.rz[0], g.rz[1], g.rz[2]);
      if (fabs(denom) < P.opt.grazing_eps) continue;
      const double rt = g.num / denom;
      if (rt <= 0) continue;
      const bool after_last = rt > last_d || (rt == last_d && j > last_j);
      if (!after_last) continue;
      if (best_j < 0 || rt < best_d) {
        best_d = rt;
        best_j = j;
      }
    }
    if (best_j < 0) break;
    last_d = best_d;
    last_j = best_j;
    if (!px.composite(P, best_d, P.lid[best_j])) break;
  }
  if (px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  if (!BWD) px.finish_forward(P);
}

// Flagged pixels in decreasing order of their composite count (pxcomp, in
// quarter-octave buckets): the fp64 pass fetches pixels dynamically, so the
// longest walks start first and the short ones fill in behind them instead of
// a few long walks trailing the grid.
__device__ __forceinline__ int redo_bucket(int ncomp) {
  return 63 - min(63, (int)(4.f * __log2f((float)max(ncomp, 0) + 1.f)));
}

__global__ void k_redo_hist(const int* __restrict__ list, const unsigned* count, const int* __restrict__ pxcomp,
                            unsigned* hist) {
  __shared__ unsigned sh[64];
  if (threadIdx.x < 64) sh[threadIdx.x] = 0;
  __syncthreads();
  const unsigned n = *count;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    atomicAdd(&sh[redo_bucket(pxcomp[list[t]])], 1u);
  __syncthreads();
  if (threadIdx.x < 64 && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

__global__ void k_redo_scatter(const int* __restrict__ list, const unsigned* count, const int* __restrict__ pxcomp,
                               const unsigned* hist, unsigned* cursor, int* out) {
  __shared__ unsigned start[64];
  if (threadIdx.x == 0) {
    unsigned a = 0;
    for (int b = 0; b < 64; ++b) {
      start[b] = a;
      a += hist[b];
    }
  }
  __syncthreads();
  const unsigned n = *count;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int p = list[t];
    const int b = redo_bucket(pxcomp[p]);
    out[start[b] + atomicAdd(&cursor[b], 1u)] = p;
  }
}

__global__ void k_redo_copy(const int* __restrict__ src, const unsigned* count, int* dst) {
  const unsigned n = *count;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) dst[t] = src[t];
}

static void order_redo_list(const RasterParams& P, cudaStream_t s) {
  static const bool on = !getenv("DRK_REDO_ORDER") || atoi(getenv("DRK_REDO_ORDER")) != 0;
  if (!on || !P.redo_tmp || !P.redo_hist || !P.pxcomp) return;
  cudaMemsetAsync(P.redo_hist, 0, 128 * sizeof(unsigned), s);
  k_redo_hist<<<148 * 2, 256, 0, s>>>(P.redo_list, P.redo_count, P.pxcomp, P.redo_hist);
  k_redo_scatter<<<148 * 2, 256, 0, s>>>(P.redo_list, P.redo_count, P.pxcomp, P.redo_hist, P.redo_hist + 64,
                                         P.redo_tmp);
  k_redo_copy<<<148 * 2, 256, 0, s>>>(P.redo_tmp, P.redo_count, P.redo_list);
  launch_counter() += 3;
}

void launch_raster(const RasterParams& P, int n_tiles, bool bwd, cudaStream_t s, cudaEvent_t mid) {
  if (n_tiles == 0) return;
  launch_counter() += P.opt.exact_sort ? 1 : 2;
  if (P.opt.exact_sort) {
    RasterParams Q = P;
    Q.pxflag = nullptr;
    dim3 grid(2, n_tiles);
    if (bwd) k_raster_exact<true><<<grid, 128, 0, s>>>(Q);
    else k_raster_exact<false><<<grid, 128, 0, s>>>(Q);
    return;
  }
  // fp32 pass (all pixels; flags uncertain ones), then the fp64 pass over the
  // flagged pixels (CTAs without flagged pixels exit immediately).
  // warp per pixel: 148 SMs x 8 CTAs x 4 warps, grid-stride over the list
  const int redo_blocks = 148 * 8;
  cudaMemsetAsync(P.redo_count + 1, 0, sizeof(unsigned), s);  // k_raster_pixels_warp's fetch counter
  if (P.opt.fp64_alpha) {
    if (!bwd) {
      // reference-precision forward: a thread per pixel over whole tiles, fp64
      // throughout (the fp64 Pixel with the explicitly rounded compositing of the
      // warp-per-pixel kernel: bitwise the same frame, config 2 51.6 ms vs 139 ms)
      RasterParams Q = P;
      Q.pxflag = nullptr;
      if (P.opt.use_cache) k_raster<0, false, true><<<n_tiles, 256, 0, s>>>(Q);
      else k_raster<1, false, true><<<n_tiles, 256, 0, s>>>(Q);
      launch_counter() -= 1;
      if (mid) cudaEventRecord(mid, s);
      return;
    }
    // reference-precision backward (the deterministic one is drk_det.cu's): the
    // warp-reduced backward over whole tiles, fp64 throughout
    RasterParams Q = P;
    Q.pxflag = nullptr;
    if (P.opt.use_cache) k_raster_bwd<0, true><<<n_tiles, 256, 0, s>>>(Q);
    else k_raster_bwd<1, true><<<n_tiles, 256, 0, s>>>(Q);
    launch_counter() -= 1;
    return;
  }
  if (!bwd) cudaMemsetAsync(P.redo_count, 0, sizeof(unsigned), s);
  if (P.opt.use_cache) {
    // fp32 interval backward (drk_raster_bwd.cu) where eligible (config 2: 56.1 ms vs 63.9 ms legacy);
    // raster_kernel 1 / 5 select the legacy warp-reduced kernel
    if (bwd && P.opt.raster_kernel != 1 && P.opt.raster_kernel != 5 && raster_fast_eligible(P))
      launch_raster_bwd_fast(P, n_tiles, s);
    else if (bwd) k_raster_bwd<0, false><<<n_tiles, 256, 0, s>>>(P);
    else if (P.opt.raster_kernel != 1 && raster_fast_eligible(P)) launch_raster_fast(P, n_tiles, P.vstat != nullptr, s);
    else k_raster<0, false, false><<<n_tiles, 256, 0, s>>>(P);
    if (mid) cudaEventRecord(mid, s);
    order_redo_list(P, s);
    if (bwd) k_raster_pixels_warp<0, true><<<redo_blocks, 128, 0, s>>>(P);
    else k_raster_pixels_warp<0, false><<<redo_blocks, 128, 0, s>>>(P);
  } else {
    if (bwd) k_raster_bwd<1, false><<<n_tiles, 256, 0, s>>>(P);
    else k_raster<1, false, false><<<n_tiles, 256, 0, s>>>(P);
    if (mid) cudaEventRecord(mid, s);
    if (bwd) k_raster_pixels_warp<1, true><<<redo_blocks, 128, 0, s>>>(P);
    else k_raster_pixels_warp<1, false><<<redo_blocks, 128, 0, s>>>(P);
  }
}

// Deterministic backward building blocks (drk_det.cu): the fp64 per-pixel
// path over P.redo_list (all pixels of a chunk, or its flagged pixels after the
// fast kernel), and the exact-sort path over a range of tiles.
void launch_pixels_bwd(const RasterParams& P, cudaStream_t s) {
  cudaMemsetAsync(P.redo_count + 1, 0, sizeof(unsigned), s);
  launch_counter() += 1;
  if (P.opt.use_cache) k_raster_pixels_warp<0, true><<<148 * 8, 128, 0, s>>>(P);
  else k_raster_pixels_warp<1, true><<<148 * 8, 128, 0, s>>>(P);
}

void launch_exact_bwd(const RasterParams& P, int n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return;
  launch_counter() += 1;
  RasterParams Q = P;
  Q.pxflag = nullptr;
  k_raster_exact<true><<<dim3(2, n_tiles), 128, 0, s>>>(Q);
}

// FFMA throughput probe (8 independent chains per thread, 148 x 8 CTAs).
__global__ void __launch_bounds__(256) k_ffma(float* out, int iters) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float b = 0.9999f, c = 1e-4f;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678f) out[0] = s;
}

double measure_fp32_peak(cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  cudaMalloc(&out, sizeof(float));
  const int iters = 1 << 16, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma<<<blocks, 256, 0, s>>>(out, iters / 16);  // warm-up
  cudaEventRecord(e0, s);
  k_ffma<<<blocks, 256, 0, s>>>(out, iters);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * iters * (double)blocks * 256;
  return flops / (ms * 1e-3) / 1e12;
}

// Validation of alpha_f32's error bound against the fp64 path: random
// (primitive, u, v) samples over each primitive's support; reports
// max |a32 - a64| / (rel * a32 + 1e-30) and max |a32 - a64|.
__global__ void k_alpha_bound(ShapeView S, int n, long long samples, unsigned long long seed,
                              unsigned long long* max_ratio_bits, unsigned long long* max_abs_bits) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= samples || n == 0) return;
  unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(t + 1));
  auto next = [&]() {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return (double)((x * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
  };
  const int i = (int)(next() * n) % n;
  double smax = 0;
  for (int k = 0; k < S.K; ++k) smax = dmax(smax, S.s[(size_t)i * S.K + k]);
  const double r = 3.5 * smax * sqrt(next());
  const double ang = kTwoPi * next();
  const double u = r * cos(ang), v = r * sin(ang);
  const double r2 = xa(xm(u, u), xm(v, v));
  KEval ev;
  eval_kernel(u, v, S, i, ev);
  if (ev.degenerate) return;
  const double a64 = S.o[i] * sharpen(ev.g, S.tau[i]);
  if (a64 < 1e-4) return;  // far below alpha_min: no decision or composite depends on it
  float rel;
  bool degen;
  const float a32 = alpha_f32(u, v, r2, S, i, (float)S.o[i], (float)S.tau[i], (float)S.eta[i], &rel, &degen);
  if (degen) return;
  const double diff = fabs((double)a32 - a64);
  const double ratio = diff / ((double)rel * a32 + 1e-30);
  atomicMax(max_ratio_bits, (unsigned long long)__double_as_longlong(ratio));
  atomicMax(max_abs_bits, (unsigned long long)__double_as_longlong(diff));
}

void launch_alpha_bound(const ShapeView& S, int n, long long samples, unsigned long long seed,
                        unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, 2 * sizeof(unsigned long long), s);
  if (samples > 0)
    k_alpha_bound<<<(unsigned)((samples + 255) / 256), 256, 0, s>>>(S, n, samples, seed, out, out + 1);
}

// ---------------------------------------------------------------------------
// K6: activation backward (grad.cpp:122-159) + screen_grad (grad.cpp:375-383)
// ---------------------------------------------------------------------------
template <typename GT>
__global__ void k_act_bwd(int n, int K, int terms, const float* __restrict__ raw, const GT* __restrict__ gact,
                          int G, const unsigned char* __restrict__ touched_dev, const Geo* __restrict__ geo, CamD cam,
                          float* grad_raw, float* d_center_world, float* screen_grad, unsigned char* touched_out,
                          int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double g[kGradSlotStride];
  for (int c = 0; c < kGradSlotStride; ++c) g[c] = c < G ? (double)gact[(size_t)i * G + c] : 0.0;
  const int tch = touched_dev[i];
  if (d_center_world)
    for (int a = 0; a < 3; ++a) d_center_world[3 * i + a] = (float)g[a];
  if (touched_out) touched_out[i] = (unsigned char)tch;
  if (screen_grad) {
    double sgv = 0;
    if (tch && geo[i].has_proj) {
      double J[6];
      projection_jacobian(cam, geo[i].mu, J);
      const double jx = J[0] * g[0] + J[1] * g[1] + J[2] * g[2];
      const double jy = J[3] * g[0] + J[4] * g[1] + J[5] * g[2];
      sgv = sqrt(jx * jx + jy * jy);
    }
    screen_grad[i] = (float)sgv;
  }
  if (!grad_raw || !raw) return;
#define RAW(j) ((double)raw[(size_t)(j)*n + i])
  double out[3 + 4 + 2 * kMaxK + 3];
  for (int a = 0; a < 3; ++a) out[a] = g[a];
  // quat_rotation_backward (grad.cpp:122-141)
  const double q[4] = {RAW(3), RAW(4), RAW(5), RAW(6)};
  const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double qh[4] = {q[0] / qn, q[1] / qn, q[2] / qn, q[3] / qn};
  const double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
  const double Ms[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                           {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                           {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                           {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
  const double* dR = g + 3;
  double dqh[4];
  for (int m = 0; m < 4; ++m) {
    double acc = Ms[m][0] * dR[0];
    for (int idx = 1; idx < 9; ++idx) {
      const int r = idx % 3, c = idx / 3;  // column-major storage order of Eigen's sum
      acc = acc + Ms[m][3 * r + c] * dR[3 * r + c];
    }
    dqh[m] = 2.0 * acc;
  }
  const double dd = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
  for (int m = 0; m < 4; ++m) out[3 + m] = (dqh[m] - qh[m] * dd) / qn;
  for (int j = 0; j < K; ++j) out[7 + j] = g[kGOffSc + j] * exp(RAW(7 + j));
  // angle_activation_jacobian (core.cpp:110-131), out = J^T d_angles
  const double residual = 1.0 / (K - 2);
  double dstep[kMaxK], cum[kMaxK], total = 0;
  for (int j = 0; j < K; ++j) {
    const double sg = sigmoid(RAW(7 + K + j));
    const bool clmp = sg < 1e-9 || sg > 1.0 - 1e-9;
    const double sc = sg < 1e-9 ? 1e-9 : (1.0 - 1e-9 < sg ? 1.0 - 1e-9 : sg);
    dstep[j] = clmp ? 0.0 : sg * (1.0 - sg);
    total += sc + residual;
    cum[j] = total;
  }
  for (int c = 0; c < K; ++c) {
    double acc = 0;
    for (int r = 0; r < K; ++r) {
      const double ind = (c <= r) ? 1.0 : 0.0;
      const double jac = (r == K - 1) ? 0.0 : kTwoPi / total * (ind - cum[r] / total) * dstep[c];
      acc = (r == 0) ? jac * g[kGOffAn + r] : acc + jac * g[kGOffAn + r];
    }
    out[7 + K + c] = acc;
  }
  const double eta = sigmoid(RAW(7 + 2 * K));
  out[7 + 2 * K] = g[kGOffEta] * eta * (1.0 - eta);
  const double st = sigmoid(RAW(8 + 2 * K));
  out[8 + 2 * K] = g[kGOffTau] * (kTauHigh - kTauLow) * st * (1.0 - st);
  const double o = sigmoid(RAW(9 + 2 * K));
  out[9 + 2 * K] = g[kGOffOp] * o * (1.0 - o);
#undef RAW
  const int S0 = 10 + 2 * K;
  for (int j = 0; j < S0; ++j) {
    float* dst = grad_raw + (size_t)j * n + i;
    *dst = accumulate ? *dst + (float)out[j] : (float)out[j];
  }
  for (int j = 0; j < 3 * terms; ++j) {
    float* dst = grad_raw + (size_t)(S0 + j) * n + i;
    const float val = (float)g[kGOffSh + j];
    *dst = accumulate ? *dst + val : val;
  }
}

void launch_act_bwd(int n, int K, int terms, const float* raw, const float* gact, int G,
                    const unsigned char* touched_dev, const Geo* geo, const CamD& cam, float* grad_raw,
                    float* d_center_world, float* screen_grad, unsigned char* touched_out, int accumulate,
                    cudaStream_t s) {
  if (n == 0) return;
  k_act_bwd<float><<<(n + 127) / 128, 128, 0, s>>>(n, K, terms, raw, gact, G, touched_dev, geo, cam, grad_raw,
                                                     d_center_world, screen_grad, touched_out, accumulate);
}

// the deterministic backward's fp64 activated-space gradients
void launch_act_bwd(int n, int K, int terms, const float* raw, const double* gact, int G,
                    const unsigned char* touched_dev, const Geo* geo, const CamD& cam, float* grad_raw,
                    float* d_center_world, float* screen_grad, unsigned char* touched_out, int accumulate,
                    cudaStream_t s) {
  if (n == 0) return;
  k_act_bwd<double><<<(n + 127) / 128, 128, 0, s>>>(n, K, terms, raw, gact, G, touched_dev, geo, cam, grad_raw,
                                                      d_center_world, screen_grad, touched_out, accumulate);
}

// ---------------------------------------------------------------------------
// K7: L1 loss (optimize.cpp:171-204 with dssim_weight = 0)
// ---------------------------------------------------------------------------
__global__ void k_l1(long long n, const float* __restrict__ r, const float* __restrict__ t, double inv_n,
                     double* loss, float* dcol) {
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double d = (double)r[i] - (double)t[i];
    acc += fabs(d);
    if (dcol) dcol[i] = (float)(1.0 * inv_n * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0)));
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if (threadIdx.x == 0) atomicAdd(loss, acc * inv_n);
  }
}

void launch_l1(long long n, const float* r, const float* t, double* loss, float* dcol, cudaStream_t s) {
  cudaMemsetAsync(loss, 0, sizeof(double), s);
  if (n == 0) return;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  k_l1<<<blocks, 256, 0, s>>>(n, r, t, 1.0 / (double)n, loss, dcol);
}

// ---------------------------------------------------------------------------
// K8: Adam (optimize.cpp:226-307): beta (0.9, 0.999), eps 1e-15, bias
// corrected, per-class learning rates, SH rows >= 1 at lr_sh / 20.
// ---------------------------------------------------------------------------
// scalars e in [e0, e1) of the SoA parameters (a rank's shard in drk_allreduce_adam);
// the gradient of scalar e is gr[e - g0]
__global__ void k_adam(long long e0, long long e1, long long g0, int n, int K, float* p, const float* __restrict__ gr,
                       float* m, float* v, double bc1, double bc2, double lr_center, double lr_quat, double lr_scale,
                       double lr_angle, double lr_eta, double lr_tau, double lr_op, double lr_sh, double lr_sh_rest,
                       double grad_scale) {
  for (long long e = e0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < e1;
       e += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(e / n);
    double lr;
    if (s < 3) lr = lr_center;
    else if (s < 7) lr = lr_quat;
    else if (s < 7 + K) lr = lr_scale;
    else if (s < 7 + 2 * K) lr = lr_angle;
    else if (s == 7 + 2 * K) lr = lr_eta;
    else if (s == 8 + 2 * K) lr = lr_tau;
    else if (s == 9 + 2 * K) lr = lr_op;
    else lr = (s - (10 + 2 * K)) < 3 ? lr_sh : lr_sh_rest;
    const double g = (double)gr[e - g0] * grad_scale;
    const double mm = 0.9 * (double)m[e] + (1.0 - 0.9) * g;
    const double vv = 0.999 * (double)v[e] + (1.0 - 0.999) * g * g;
    m[e] = (float)mm;
    v[e] = (float)vv;
    const double mh = mm / bc1, vh = vv / bc2;
    p[e] = (float)((double)p[e] - lr * mh / (sqrt(vh) + 1e-15));
  }
}

int run_adam(drk_ctx* c, float* params, const float* grads, float* m, float* v, int n, int K, int terms,
             int64_t step, const drk_adam_config* cfg) {
  const long long total = (long long)(3 + 4 + 2 * K + 3 + 3 * terms) * n;
  return run_adam_range(c, params, grads, 0, m, v, n, K, 0, total, step, cfg);
}

int run_adam_range(drk_ctx* c, float* params, const float* grads, long long g0, float* m, float* v, int n, int K,
                   long long e0, long long e1, int64_t step, const drk_adam_config* cfg) {
  const long long total = e1 - e0;
  const double bc1 = 1.0 - pow(0.9, (double)step);
  const double bc2 = 1.0 - pow(0.999, (double)step);
  const double t = cfg->steps > 0 ? dmin(1.0, (double)step / cfg->steps) : 1.0;
  const double decay = pow(1e-2, t);
  const double lr_drk = cfg->lr_drk * decay;
  const double lr_sh = cfg->lr_sh;
  if (total > 0) {
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    k_adam<<<blocks, 256, 0, c->stream>>>(e0, e1, g0, n, K, params, grads, m, v, bc1, bc2,
                                           cfg->lr_position * cfg->scene_extent * decay, cfg->lr_rotation, lr_drk,
                                           cfg->freeze_angles ? 0.0 : lr_drk, cfg->freeze_eta_tau ? 0.0 : lr_drk,
                                           cfg->freeze_eta_tau ? 0.0 : lr_drk, cfg->lr_opacity, lr_sh, lr_sh / 20.0,
                                           cfg->grad_scale);
  }
  return cuda_check(c, cudaGetLastError(), "adam");
}

// ---------------------------------------------------------------------------
// eval_sorting (reference raster.cpp:487-560): per pixel, the depth sequence
// the renderer would process (SortCache pops, or list order), compared with its
// sorted order: Kendall tau, MAE, fully-ordered flag.  One thread per pixel of
// a chunk of tiles; the sequence lives in a per-pixel scratch row of the tile's
// list length.  Hits and depths are the reference's exact fp64 values
// (classify_intersect op order), concordant / discordant pairs are counted by
// a bottom-up merge sort (O(n log n); strict inequalities only, like the
// reference's O(n^2) loop), so every per-pixel value is the reference's.
// ---------------------------------------------------------------------------
__global__ void k_eval_sorting(const RasterParams P, int tile0, int tile1, const long long* __restrict__ scr_off,
                               double* scratch, int use_cache, double* tau_out, double* mae_out,
                               unsigned char* flag_out) {
  const int t = tile0 + blockIdx.x;
  if (t >= tile1) return;
  const int tx = t % P.cam.tiles_x, ty = t / P.cam.tiles_x;
  const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  if (x >= P.cam.W || y >= P.cam.H) return;
  const size_t pix = (size_t)y * P.cam.W + x;
  flag_out[pix] = 0;
  const long long beg = P.tileoff[t], end = P.tileoff[t + 1];
  const long long L = end - beg;
  if (L == 0) return;
  double* seq = scratch + scr_off[blockIdx.x] + (long long)threadIdx.x * 3 * L;
  double* tmp = seq + L;
  double dir[3];
  pixel_dir(P.cam, x + 0.5, y + 0.5, dir);
  int n = 0;
  double cd[kCacheCap];
  int ci[kCacheCap];
  int csz = 0;
  for (long long j = beg; j < end; ++j) {
    const int id = P.lid[j];
    const Geo& g = P.geo[id];
    const double denom = xdot3(dir[0], dir[1], dir[2], g.rz[0], g.rz[1], g.rz[2]);
    if (fabs(denom) < P.opt.grazing_eps) continue;  // geometry.cpp:40-47
    const double rt = g.num / denom;
    if (!(rt > 0)) continue;
    if (!use_cache) {
      seq[n++] = rt;
      continue;
    }
    double prt;
    int pid;
    if (cache_step(cd, ci, csz, rt, id, prt, pid)) seq[n++] = prt;
  }
  if (use_cache)
    for (int q = 0; q < csz; ++q) seq[n++] = cd[q];  // end marker: drain in order
  if (n < 2) return;
  // discordant pairs (i < j, p_i > p_j) by bottom-up merge sort of a copy
  for (int i = 0; i < n; ++i) tmp[i] = seq[i];
  // the processed order stays in seq; the merge ping-pongs between the row's
  // second and third thirds (scratch row = 3 L doubles)
  double* a = tmp;
  double* c2 = seq + 2 * L;
  long long disc = 0;
  for (int w = 1; w < n; w *= 2) {
    for (int lo = 0; lo < n; lo += 2 * w) {
      const int mid = min(lo + w, n), hi = min(lo + 2 * w, n);
      int i = lo, j = mid, k = lo;
      while (i < mid && j < hi) {
        if (a[j] < a[i]) {
          disc += mid - i;
          c2[k++] = a[j++];
        } else {
          c2[k++] = a[i++];
        }
      }
      while (i < mid) c2[k++] = a[i++];
      while (j < hi) c2[k++] = a[j++];
    }
    double* sw = a;
    a = c2;
    c2 = sw;
  }
  // a = sorted; ties: pairs of equal values are neither concordant nor discordant
  long long ties = 0, run = 1;
  for (int i = 1; i < n; ++i) {
    if (a[i] == a[i - 1]) {
      ++run;
    } else {
      ties += run * (run - 1) / 2;
      run = 1;
    }
  }
  ties += run * (run - 1) / 2;
  const long long total = (long long)n * (n - 1) / 2;
  const long long conc = total - disc - ties;
  const double pairs = 0.5 * n * (n - 1);
  tau_out[pix] = (conc - disc) / pairs;
  double mae = 0;
  for (int i = 0; i < n; ++i) mae += fabs(seq[i] - a[i]);
  mae_out[pix] = mae / n;
  flag_out[pix] = disc == 0 ? 2 : 1;
}

// the reference's accumulation order: tiles row-major, pixels row-major inside
__global__ void k_eval_sorting_reduce(CamD cam, const long long* __restrict__ tileoff, const double* __restrict__ tau,
                                      const double* __restrict__ mae, const unsigned char* __restrict__ flag,
                                      double* out) {
  if (threadIdx.x || blockIdx.x) return;
  double tau_sum = 0, mae_sum = 0;
  long long ordered = 0, counted = 0;
  for (int ty = 0; ty < cam.tiles_y; ++ty)
    for (int tx = 0; tx < cam.tiles_x; ++tx) {
      const int t = ty * cam.tiles_x + tx;
      if (tileoff[t + 1] == tileoff[t]) continue;
      const int x0 = tx * kTile, y0 = ty * kTile;
      const int x1 = min(cam.W, x0 + kTile), y1 = min(cam.H, y0 + kTile);
      for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
          const size_t p = (size_t)y * cam.W + x;
          if (!flag[p]) continue;
          tau_sum += tau[p];
          mae_sum += mae[p];
          if (flag[p] == 2) ++ordered;
          ++counted;
        }
    }
  out[0] = counted > 0 ? (double)ordered / counted : 0.0;
  out[1] = counted > 0 ? tau_sum / counted : 0.0;
  out[2] = counted > 0 ? mae_sum / counted : 0.0;
  out[3] = (double)counted;
}

void launch_eval_sorting(const RasterParams& P, int tile0, int tile1, const long long* scr_off, double* scratch,
                         int use_cache, double* tau, double* mae, unsigned char* flag, cudaStream_t s) {
  if (tile1 > tile0) k_eval_sorting<<<tile1 - tile0, 256, 0, s>>>(P, tile0, tile1, scr_off, scratch, use_cache, tau,
                                                                   mae, flag);
}

void launch_eval_sorting_reduce(const CamD& cam, const long long* tileoff, const double* tau, const double* mae,
                                const unsigned char* flag, double* out, cudaStream_t s) {
  k_eval_sorting_reduce<<<1, 32, 0, s>>>(cam, tileoff, tau, mae, flag, out);
}

}  // namespace drk
