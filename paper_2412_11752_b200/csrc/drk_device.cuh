// Device math for the DRK rasterizer (sm_100a).  Compiled with --fmad=false so
// that every fp64 expression rounds exactly like the reference's x86-64 build
// (no contraction); the op order of each function follows the reference line
// it cites, with Eigen reductions left to right (oracle/shim/Eigen/Core).
// Transcendentals (exp, log, sin, cos, atan2) are CUDA's (<= 2 ulp), so values
// derived from them agree with the reference to ~1e-16 relative; everything
// built from + - * / sqrt only (pixel rays, ray-plane depths, quaternion
// rotation, projection) is bit-identical.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "drk_b200.h"

namespace drk {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kThreeSigmaLevel = 1.2340980408667956e-4;  // core.cpp:14
constexpr double kTauLow = -0.1;
constexpr double kTauHigh = 0.99;
constexpr double kMinExponent = -30.0;
constexpr double kNearClip = 1e-6;  // raster.cpp:12
constexpr int kTile = 16;
constexpr int kCacheCap = 8;  // raster.hpp:37
constexpr int kMaxK = 16;

// Row layout of the activated-space gradient buffer (drk::PrimGrads,
// grad.hpp:19-29), fixed for every K so that the backward's component indices
// are compile-time constants: d_center 0..2, d_rot 3..11 (row-major),
// d_scales [12, 12+kMaxK), d_angles, d_eta, d_tau, d_opacity, d_sh (RGB per
// term).  Rows are padded to a multiple of 4 floats (16-byte vector atomics).
constexpr int kGOffSc = 12, kGOffAn = kGOffSc + kMaxK, kGOffEta = kGOffAn + kMaxK, kGOffTau = kGOffEta + 1,
              kGOffOp = kGOffEta + 2, kGOffSh = kGOffEta + 3;
__host__ __device__ inline int grad_row_stride(int terms) { return (kGOffSh + 3 * terms + 3) & ~3; }

// Device-side error / counter slots (ctx->counters).
enum Counter {
  C_ERR_DEGEN_BASIS = 0,
  C_ERR_NONFINITE,
  C_ERR_DEGEN_QUAT,
  C_POLY_OVERFLOW,
  C_HULL_POOL,        // hull pool cursor
  C_NEAR_TIES,
  C_STREAMED,
  C_POPPED,
  C_COMPOSITED,
  C_REPLAY_OVERFLOW,
  C_VISIBLE,
  C_POLY_FAIL,
  C_REDO_PIXELS,  // pixels re-rendered by the fp64 pass
  C_BWD_WARPSTEPS,     // warp-cooperative backward steps with >= 1 record
  C_BWD_LEAD_RECORDS,  // records reduced in the leader group (rest: direct atomics)
  C_REJECT_RADIUS,     // pops rejected by the isotropic support radius
  C_REJECT_BRACKET,    // pops rejected by the in-bracket Q lower bound
  C_FP64_EVALS,        // pops re-evaluated in fp64 (decision within the fp32 bound)
  C_AMBIGUOUS,         // fast kernel: cache steps with overlapping depth intervals
  C_RING_MISS,         // fast kernel: pops re-staged from HBM (older than the ring)
  C_PTS_POOL,          // K1: sorted-point pool cursor
  C_DET_OVERFLOW,      // deterministic backward: records beyond the forward's composite count (must stay 0)
  C_TIE_RUNS,          // sort: runs of equal packed keys (ordered on the full fp64 key afterwards)
  C_TIE_MEMBERS,       // sort: entries in such runs
  C_TIE_MAXRUN,        // sort: longest run
  C_CACHE_APPEND,      // fast kernel: full-cache steps whose incoming entry is certainly deeper than every cached one
  C_COUNT
};

// Camera + derived constants, passed by value to kernels.
struct CamD {
  double fx, fy, cx, cy;
  double R[9];  // row-major world->cam
  double t[3];
  double o[3];  // camera position, -(R^T) t, op order of geometry.hpp:15
  int W, H, tiles_x, tiles_y;
};

struct OptD {
  double lowpass_radius, alpha_min, grazing_eps;
  double bg[3];
  double early_stop;
  double lp_pad;  // raster.cpp:128-129
  int sh_degree, use_cache, exact_sort, presort, record_replay, terms_active, fp64_alpha, raster_kernel;
};

__host__ __device__ inline double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min
__host__ __device__ inline double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max

// static_cast<int>(double) as compiled for x86-64 (cvttsd2si): NaN and
// out-of-range values give INT_MIN.  raster.cpp:226-231 depends on it.
__host__ __device__ inline int x86_int(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return (int)0x80000000u;
  return (int)v;
}

__host__ __device__ inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// Explicitly rounded fp64 ops: never contracted into FMA, whatever --fmad
// says.  Used for every value that must be bit-identical to the reference
// (ray directions, ray-plane depths, tangent coordinates).
__device__ __forceinline__ double xm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xs(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double xdot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  return xa(xa(xm(a0, b0), xm(a1, b1)), xm(a2, b2));
}

// pixel_ray (geometry.cpp:32-38): dir = normalize(R^T ((px-cx)/fx, (py-cy)/fy, 1)).
__device__ __forceinline__ void pixel_dir(const CamD& c, double px, double py, double d[3]) {
  const double dc0 = xs(px, c.cx) / c.fx, dc1 = xs(py, c.cy) / c.fy, dc2 = 1.0;
  double v0 = xdot3(c.R[0], c.R[3], c.R[6], dc0, dc1, dc2);
  double v1 = xdot3(c.R[1], c.R[4], c.R[7], dc0, dc1, dc2);
  double v2 = xdot3(c.R[2], c.R[5], c.R[8], dc0, dc1, dc2);
  const double sq = xdot3(v0, v1, v2, v0, v1, v2);
  if (sq > 0) {
    const double n = __dsqrt_rn(sq);
    v0 = v0 / n;
    v1 = v1 / n;
    v2 = v2 / n;
  }
  d[0] = v0;
  d[1] = v1;
  d[2] = v2;
}

// Camera::to_camera (geometry.hpp:14): R * w + t.
__device__ __forceinline__ void to_camera(const CamD& c, const double w[3], double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    out[i] = (c.R[3 * i] * w[0] + c.R[3 * i + 1] * w[1] + c.R[3 * i + 2] * w[2]) + c.t[i];
}

// try_project_point (geometry.cpp:67-74).
__device__ __forceinline__ bool try_project(const CamD& c, const double w[3], double out[3]) {
  double p[3];
  to_camera(c, w, p);
  if (p[2] <= 0) return false;
  out[0] = c.fx * p[0] / p[2] + c.cx;
  out[1] = c.fy * p[1] / p[2] + c.cy;
  out[2] = p[2];
  return true;
}

// projection_jacobian (geometry.cpp:82-89), 2x3 row-major.
__device__ __forceinline__ void projection_jacobian(const CamD& c, const double w[3], double J[6]) {
  double p[3];
  to_camera(c, w, p);
  const double z = p[2];
  const double jc[6] = {c.fx / z, 0, -c.fx * p[0] / (z * z), 0, c.fy / z, -c.fy * p[1] / (z * z)};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      J[3 * i + j] = jc[3 * i] * c.R[j] + jc[3 * i + 1] * c.R[3 + j] + jc[3 * i + 2] * c.R[6 + j];
}

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }  // core.cpp:80

// sharpen family (core.cpp:210-245).
__device__ __forceinline__ double sharpen_inverse(double y, double tau) {
  y = dmin(1.0, dmax(0.0, y));
  if (y < (1.0 - tau) / 4.0) return (1.0 + tau) / (1.0 - tau) * y;
  if (y < (3.0 + tau) / 4.0) return ((1.0 - tau) * y + tau) / (1.0 + tau);
  return ((1.0 + tau) * y - 2.0 * tau) / (1.0 - tau);
}
__device__ __forceinline__ int sharpen_branch(double g, double tau) {
  if (g < (1.0 + tau) / 4.0) return 0;
  if (g < (3.0 - tau) / 4.0) return 1;
  return 2;
}
__device__ __forceinline__ double sharpen_slope(int b, double tau) {
  if (b == 1) return (1.0 + tau) / (1.0 - tau);
  return (1.0 - tau) / (1.0 + tau);
}
__device__ __forceinline__ double sharpen_dtau(int b, double g, double tau) {
  if (b == 0) return -2.0 * g / ((1.0 + tau) * (1.0 + tau));
  if (b == 1) return (2.0 * g - 1.0) / ((1.0 - tau) * (1.0 - tau));
  return (2.0 - 2.0 * g) / ((1.0 + tau) * (1.0 + tau));
}
__device__ __forceinline__ double sharpen(double g, double tau) {
  g = dmin(1.0, dmax(0.0, g));
  switch (sharpen_branch(g, tau)) {
    case 0: return (1.0 - tau) / (1.0 + tau) * g;
    case 1: return ((1.0 + tau) * g - tau) / (1.0 - tau);
    default: return ((1.0 - tau) * g + 2.0 * tau) / (1.0 + tau);
  }
}

// binning_radius_factor (core.cpp:305-318); false when never visible.
__device__ __forceinline__ bool binning_radius_factor(double o, double tau, double amin, double* f,
                                                      double* f_vis) {
  const double vis = amin / o;
  if (vis >= 1.0) return false;
  const double gv = sharpen_inverse(vis, tau);
  double fac = sqrt(-2.0 * log(gv));
  *f_vis = fac;
  const double cal = kThreeSigmaLevel / o;
  if (cal < 1.0) {
    const double gc = sharpen_inverse(cal, tau);
    if (gc > 0 && gc < 1) fac = dmax(fac, sqrt(-log(gc)));
  }
  *f = fac;
  return true;
}

// Per-primitive shape constants (view independent), primitive-major with
// stride K: endpoints e_k = s_k (cos th_k, sin th_k) and the determinant of
// the bracket (k, k+1 mod K) as evaluated in core.cpp:188-190.
struct ShapeView {
  const double* s;
  const double* th;
  const double* ex;
  const double* ey;
  const double* det;
  const double* eta;
  const double* tau;
  const double* o;
  // fp32 fast-path constants, stride K: theta_k, 1/det_k, pi/gap_k (bracket
  // k, k+1 mod K), 1/s_k^2
  const float* thf;
  const float* invdetf;
  const float* piogf;
  const float* hf;
  // per primitive, 12 floats: sharpen breakpoints and point-slope form
  // g1, g2, A0, A1, A2, Psi(g1), Psi(g2), opacity, f_vis^2, 0, 0, 0
  // (fp64-derived, rounded once)
  const float* psif;
  int K;
};

struct KEval {
  double g, r2, theta, delta, inv_sbar, a, b, r1;
  int lo, hi;
  bool center, clamped, degenerate;
};

// eval_kernel_detail (core.cpp:148-204) for primitive i.
__device__ __forceinline__ void eval_kernel(double u, double v, const ShapeView& S, int i, KEval& ev) {
  const int K = S.K;
  const double* th = S.th + (size_t)i * K;
  ev.g = 1.0;
  ev.center = false;
  ev.clamped = false;
  ev.degenerate = false;
  ev.r2 = u * u + v * v;
  ev.lo = ev.hi = 0;
  ev.theta = ev.delta = ev.inv_sbar = ev.a = ev.b = ev.r1 = 0;
  if (ev.r2 == 0) {
    ev.center = true;
    return;
  }
  double theta = atan2(v, u);
  if (theta <= 0) theta += kTwoPi;
  ev.theta = theta;
  int lo, hi;
  double alo, ahi;
  const double th0 = th[0], thK = th[K - 1];
  if (theta <= th0 || theta > thK) {
    lo = K - 1;
    hi = 0;
    alo = thK - kTwoPi;
    ahi = th0;
    if (theta > thK) theta -= kTwoPi;
  } else {
    hi = 1;
    while (hi < K && th[hi] < theta) ++hi;  // lower_bound (th[0] < theta here)
    lo = hi - 1;
    alo = th[lo];
    ahi = th[hi];
  }
  ev.lo = lo;
  ev.hi = hi;
  ev.delta = (theta - alo) * kPi / (ahi - alo);
  const double c = cos(ev.delta);
  const double slo = S.s[(size_t)i * K + lo], shi = S.s[(size_t)i * K + hi];
  ev.inv_sbar = (1.0 + c) / (2.0 * slo * slo) + (1.0 - c) / (2.0 * shi * shi);
  const double elx = S.ex[(size_t)i * K + lo], ely = S.ey[(size_t)i * K + lo];
  const double ehx = S.ex[(size_t)i * K + hi], ehy = S.ey[(size_t)i * K + hi];
  const double det = S.det[(size_t)i * K + lo];
  if (fabs(det) < 1e-12) {
    ev.degenerate = true;
    return;
  }
  ev.a = (ehy * u - ehx * v) / det;
  ev.b = (-ely * u + elx * v) / det;
  ev.r1 = fabs(ev.a) + fabs(ev.b);
  const double eta = S.eta[i];
  double e = -0.5 * (eta * ev.r1 * ev.r1 + (1.0 - eta) * ev.r2 * ev.inv_sbar);
  if (e < kMinExponent) {
    e = kMinExponent;
    ev.clamped = true;
  }
  ev.g = exp(e);
}

__device__ __forceinline__ float sharpen_f(float g, float tau) {
  g = fminf(1.0f, fmaxf(0.0f, g));
  if (g < (1.0f + tau) * 0.25f) return (1.0f - tau) / (1.0f + tau) * g;
  if (g < (3.0f - tau) * 0.25f) return ((1.0f + tau) * g - tau) / (1.0f - tau);
  return ((1.0f - tau) * g + 2.0f * tau) / (1.0f + tau);
}

// fp32 fast path of alpha = o * Psi(g(u, v)) (core.cpp:148-204, :229-237,
// :263-265).  Cancellation-prone quantities are formed in fp64 and rounded
// once: the endpoint-basis numerators (a, b) and the angle from the lower
// bracket endpoint (so delta keeps relative precision), with the cosine
// blend written as cos^2(delta/2)/s_lo^2 + sin^2(delta/2)/s_hi^2.  Returns
// alpha and a relative error bound *rel (validated against the fp64 path by
// tests/test_gpu_alpha_bound.py); r2 == 0 gives the exact centre value.
// Psi(g) in point-slope form from fp64-derived per-primitive constants, with
// the condition number A g / Psi that maps the relative error of g onto alpha.
__device__ __forceinline__ float sharpen_ps(const float4 c0, const float4 c1, float g, float relg, float* relP,
                                            float* slope = nullptr, int* branch = nullptr) {
  // c0 = (g1, g2, A0, A1), c1 = (A2, Psi(g1), Psi(g2), o)
  float A, P;
  int br;
  if (g < c0.x) {
    A = c0.z;
    P = c0.z * g;
    br = 0;
  } else if (g < c0.y) {
    A = c0.w;
    P = c1.y + c0.w * (g - c0.x);
    br = 1;
  } else {
    A = c1.x;
    P = c1.z + c1.x * (g - c0.y);
    br = 2;
  }
  // Relative error of P for a relative error relg of g: the largest slope
  // over [g - dg, g + dg] (a breakpoint inside the interval brings the
  // neighbouring branch's slope: for tau -> 0.99 the middle branch is ~200x
  // steeper), the fp32 breakpoint in the point-slope form (<= 2^-25 absolute,
  // times the branch slope), and the roundings of the constants and the FMA.
  const float dg = g * relg + 3.5e-8f;
  float Am = A;
  if (fabsf(g - c0.x) <= dg) Am = fmaxf(Am, fmaxf(c0.z, c0.w));
  if (fabsf(g - c0.y) <= dg) Am = fmaxf(Am, fmaxf(c0.w, c1.x));
  *relP = P > 0.f ? 1.001f * __fdividef(Am * (g * relg) + (br > 0 ? A * 3.5e-8f : 0.f), P) + 1.8e-7f : 1.0f;
  if (slope) *slope = A;
  if (branch) *branch = br;
  return P;
}

// Intermediates of the fp32 kernel evaluation, kept for the fp32 backward
// (grad.cpp:16-101 restated on the fp32 quantities).
struct KEvalF {
  float g, P, A;          // g(u, v), Psi(g), dPsi/dg
  float a, b, r1;         // endpoint-basis coordinates, r1 = |a| + |b|
  float delta, sh, ch;    // bracket angle and sin/cos(delta / 2)
  float inv;              // 1 / s_bar^2
  int lo, hi, br;         // bracket, sharpen branch
  bool center, clamped;
};

// With reject_ok, returns -1 as soon as a lower bound of Q shows
// alpha_kernel < alpha_min with margin: within the bracket, r1 and the
// cosine blend give Q >= eta r1^2 + (1-eta) r2^2 min(1/s_lo^2, 1/s_hi^2), and
// alpha < alpha_min <=> Q > f_vis^2 (core.cpp:305-318 with Psi monotone).
__device__ __forceinline__ float alpha_f32(double u, double v, double r2, const ShapeView& S, int i, float o,
                                           float tau, float eta, float* rel, bool* degenerate,
                                           bool reject_ok = false, KEvalF* kf = nullptr) {
  *degenerate = false;
  (void)o;
  (void)tau;
  const float4* pc = reinterpret_cast<const float4*>(S.psif) + 3 * (size_t)i;
  const float4 c0 = __ldg(pc), c1 = __ldg(pc + 1);
  if (r2 == 0) {
    float relP;
    *rel = 5e-7f;
    if (kf) {
      kf->center = true;
      kf->clamped = false;
      kf->g = 1.0f;
      kf->P = sharpen_ps(c0, c1, 1.0f, 0.f, &relP, &kf->A, &kf->br);
      return c1.w * kf->P;
    }
    return c1.w * sharpen_ps(c0, c1, 1.0f, 0.f, &relP);
  }
  const int K = S.K;
  const float* thf = S.thf + (size_t)i * K;
  const float uf = (float)u, vf = (float)v;
  float th = atan2f(vf, uf);
  if (th <= 0.0f) th += 6.28318530717958647692f;
  int lo, hi;
  if (K == 8) {
    // two vector loads + branchless count instead of a dependent search loop
    const float4 t0 = __ldg(reinterpret_cast<const float4*>(thf)), t1 = __ldg(reinterpret_cast<const float4*>(thf) + 1);
    if (th <= t0.x || th > t1.w) {
      lo = 7;
      hi = 0;
    } else {
      hi = 1 + (t0.y < th) + (t0.z < th) + (t0.w < th) + (t1.x < th) + (t1.y < th) + (t1.z < th);
      lo = hi - 1;
    }
  } else if (th <= thf[0] || th > thf[K - 1]) {
    lo = K - 1;
    hi = 0;
  } else {
    hi = 1;
    while (hi < K && thf[hi] < th) ++hi;
    lo = hi - 1;
  }
  const size_t bl = (size_t)i * K + lo, bh = (size_t)i * K + hi;
  if (fabs(S.det[bl]) < 1e-12) {
    *degenerate = true;
    return 0.0f;
  }
  const double elx = S.ex[bl], ely = S.ey[bl], ehx = S.ex[bh], ehy = S.ey[bh];
  const float invd = S.invdetf[bl];
  const float a = (float)(ehy * u - ehx * v) * invd;
  const float b = (float)(-ely * u + elx * v) * invd;
  const float r1 = fabsf(a) + fabsf(b);
  if (reject_ok) {
    const float fvis2 = __ldg(S.psif + 12 * (size_t)i + 8);
    const float q_lb = eta * r1 * r1 + (1.0f - eta) * (float)r2 * fminf(S.hf[bl], S.hf[bh]);
    if (q_lb > fvis2 * 1.00002f) return -1.0f;
  }
  const float dth = atan2f((float)(elx * v - ely * u), (float)(elx * u + ely * v));
  const float delta = dth * S.piogf[bl];
  float sh, ch;
  sincosf(0.5f * delta, &sh, &ch);
  const float hlo = S.hf[bl], hhi = S.hf[bh];
  const float inv = ch * ch * hlo + sh * sh * hhi;
  const float Q = eta * r1 * r1 + (1.0f - eta) * (float)r2 * inv;
  const float e = fmaxf(-0.5f * Q, -30.0f);
  const float g = expf(e);
  // Relative error bound.  Q: fp32 formation of r1 and the products (~4
  // ulp) plus the cosine blend's sensitivity to delta, |d inv| <=
  // |sin(delta)| |h_lo - h_hi| / 2 * |d delta| with |d delta| <= 8e-7 (1 + delta)
  // (atan2f of the in-bracket angle times pi/gap).  g = exp(-Q/2) adds
  // Q/2 * rel(Q) and expf's ~2 ulp; Psi maps it through its largest slope
  // over g's uncertainty interval (sharpen_ps); the constants add ~4 ulp.
  // Checked against the fp64 path on the GPU
  // (tests/test_gpu_parity.py::test_fp32_alpha_error_bound).
  const float sd = 2.0f * sh * ch;  // sin(delta)
  const float dinv = 0.5f * fabsf(sd) * fabsf(hlo - hhi) * 8e-7f * (1.0f + fabsf(delta));
  const float rel_q = 5e-7f + (1.0f - eta) * (float)r2 * dinv / fmaxf(Q, 1e-30f);
  const float relg = 0.5f * fminf(Q, 60.0f) * 2.0f * rel_q + 4e-7f;
  float relP;
  const float P = kf ? sharpen_ps(c0, c1, g, relg, &relP, &kf->A, &kf->br) : sharpen_ps(c0, c1, g, relg, &relP);
  if (kf) {
    kf->center = false;
    kf->clamped = -0.5f * Q < -30.0f;
    kf->g = g;
    kf->P = P;
    kf->a = a;
    kf->b = b;
    kf->r1 = r1;
    kf->delta = delta;
    kf->sh = sh;
    kf->ch = ch;
    kf->inv = inv;
    kf->lo = lo;
    kf->hi = hi;
  }
  *rel = relP + 6e-7f;
  return c1.w * P;
}

// low_pass_filter_term (core.cpp:267-273).
__device__ __forceinline__ double low_pass_filter_term(double dpw, double dph, double cos_view, double o,
                                                       double s_l) {
  const double denom = 2.0 * cos_view * cos_view * s_l * s_l;
  double e = -(dpw * dpw + dph * dph) / denom;
  if (e < kMinExponent) e = kMinExponent;
  return o * exp(e);
}

// Real SH basis (geometry.cpp:91-124), fp32.
// sh_basis (geometry.cpp:101-124) in fp64 with the reference's op order,
// explicitly rounded: the fp64 pixel path's colours are the reference's bits.
__device__ __forceinline__ void sh_basis_d(double x, double y, double z, int degree, double* out) {
  out[0] = 0.28209479177387814;
  if (degree < 1) return;
  const double k1 = 0.4886025119029199;
  out[1] = xm(-k1, y);
  out[2] = xm(k1, z);
  out[3] = xm(-k1, x);
  if (degree < 2) return;
  const double xx = xm(x, x), yy = xm(y, y), zz = xm(z, z), xy = xm(x, y), yz = xm(y, z), xz = xm(x, z);
  out[4] = xm(1.0925484305920792, xy);
  out[5] = xm(-1.0925484305920792, yz);
  out[6] = xm(0.31539156525252005, xs(xs(xm(2.0, zz), xx), yy));
  out[7] = xm(-1.0925484305920792, xz);
  out[8] = xm(0.5462742152960396, xs(xx, yy));
  if (degree < 3) return;
  out[9] = xm(xm(-0.5900435899266435, y), xs(xm(3.0, xx), yy));
  out[10] = xm(xm(2.890611442640554, xy), z);
  out[11] = xm(xm(-0.4570457994644658, y), xs(xs(xm(4.0, zz), xx), yy));
  out[12] = xm(xm(0.3731763325901154, z), xs(xs(xm(2.0, zz), xm(3.0, xx)), xm(3.0, yy)));
  out[13] = xm(xm(-0.4570457994644658, x), xs(xs(xm(4.0, zz), xx), yy));
  out[14] = xm(xm(1.445305721320277, z), xs(xx, yy));
  out[15] = xm(xm(-0.5900435899266435, x), xs(xx, xm(3.0, yy)));
}

__device__ __forceinline__ void sh_basis_f(float x, float y, float z, int degree, float* out) {
  const float kSh0 = 0.28209479177387814f, kSh1 = 0.4886025119029199f;
  out[0] = kSh0;
  if (degree < 1) return;
  out[1] = -kSh1 * y;
  out[2] = kSh1 * z;
  out[3] = -kSh1 * x;
  if (degree < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  out[4] = 1.0925484305920792f * xy;
  out[5] = -1.0925484305920792f * yz;
  out[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
  out[7] = -1.0925484305920792f * xz;
  out[8] = 0.5462742152960396f * (xx - yy);
  if (degree < 3) return;
  out[9] = -0.5900435899266435f * y * (3.f * xx - yy);
  out[10] = 2.890611442640554f * xy * z;
  out[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
  out[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
  out[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
  out[14] = 1.445305721320277f * z * (xx - yy);
  out[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
}

}  // namespace drk
