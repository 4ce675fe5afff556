// Device code shared by the fast forward (drk_raster_fast.cu) and fast backward
// (drk_raster_bwd.cu) rasterizers: staged fp32 candidate records, exact fp64
// fallbacks, fp32 alpha with error bounds (see drk_raster_fast.cu for the design).
#pragma once
#include <climits>

#include "drk_internal.h"

namespace drk {


// Per-pixel work counters of the fast kernels: compiled in where the template
// parameter STATS is true (drk_set_counters; the roofline's counts), out of
// the timed path otherwise (1.6% of the raster).
#define DRK_STAT(x) \
  do {              \
    if (STATS) ++(x); \
  } while (0)

constexpr int kRing = 512;
constexpr int kBatch = 256;
constexpr int kRecHdr = 24;
constexpr int kRecStride = kRecHdr + 8 * 8;  // K == 8

// ---------------------------------------------------------------------------
// fp32 helpers with known error
// ---------------------------------------------------------------------------
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// hi + (lo + c . dd): float-float constant plus a small linear term
__device__ __forceinline__ float lin3(float4 c, float lo, float dx, float dy, float dz) {
  return c.w + fmaf(c.x, dx, fmaf(c.y, dy, fmaf(c.z, dz, lo)));
}

// 1/x with one Newton step: relative error <= 2^-23 (one rounding of the
// refined value on top of a ~1e-14 refinement error)
__device__ __forceinline__ float rcp_nr(float x) {
  const float r = rcp_approx(x);
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}

// cos(d) for d in [0, pi] as -sin(d - pi/2) (odd minimax polynomial);
// |error| <= 1.3e-7 measured in fp32 Horner form.
__device__ __forceinline__ float cos_0pi(float d) {
  const float y = d - 1.57079637f, s = y * y;
  float r = -2.384675390e-08f;
  r = fmaf(r, s, 2.752262162e-06f);
  r = fmaf(r, s, -1.984080445e-04f);
  r = fmaf(r, s, 8.333330043e-03f);
  r = fmaf(r, s, -1.666666716e-01f);
  r = r * s;
  return -fmaf(r, y, y);
}

// atan2 in (-pi, pi]; |error| <= 2.5e-7 |result| + 1.5e-7 (minimax polynomial
// for atan on [0, 1]: relative error 8.8e-8 measured in fp32 Horner form).
__device__ __forceinline__ float atan2_fast(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float t = mx > 0.f ? __fdividef(mn, mx) : 0.f;
  const float s = t * t;
  float r = 2.920356113e-03f;
  r = fmaf(r, s, -1.636656933e-02f);
  r = fmaf(r, s, 4.320959747e-02f);
  r = fmaf(r, s, -7.552013546e-02f);
  r = fmaf(r, s, 1.066590250e-01f);
  r = fmaf(r, s, -1.421102583e-01f);
  r = fmaf(r, s, 1.999376863e-01f);
  r = fmaf(r, s, -3.333315253e-01f);
  r = r * s;
  r = fmaf(r, t, t);
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.f) r = 3.14159274f - r;
  return copysignf(r, y);
}

#ifndef DRK_PSEUDO_ANGLE
#define DRK_PSEUDO_ANGLE 1
#endif
// 1: alpha_entry loads the shape record's bracket-lookup angles and eta first
// 1: L1 prefetch of the SH coefficients once an entry passes the bracket bound
// (measured: config-1 raster 19.73 -> 20.36 ms; off)
#ifndef DRK_SH_PREFETCH
#define DRK_SH_PREFETCH 0
#endif
// 1: the bracket lookup and its loads move ahead of the radius reject
#ifndef DRK_EARLY_BRACKET
#define DRK_EARLY_BRACKET 1  // measured: config-1 raster 20.09 -> 19.72 ms, config 2 11.10 -> 11.04 ms
#endif
#ifndef DRK_EARLY_LOADS
#define DRK_EARLY_LOADS 1  // measured: config-1 raster 20.32 -> 20.22 ms, config-2 backward 41.9 -> 41.0 ms
#endif

// Pseudo-angle of (x, y): monotone in the polar angle, 0 < p <= 4 for angles in
// (0, 2 pi] (the angle 0 maps to 4, like atan2's 0 -> 2 pi; (0, 0) -> 4).
__device__ __forceinline__ float pseudo_angle(float y, float x) {
  const float s = fabsf(x) + fabsf(y);
  if (!(s > 0.f)) return 4.f;
  float p;
  if (y >= 0.f) p = x >= 0.f ? __fdividef(y, s) : 1.f - __fdividef(x, s);
  else p = x < 0.f ? 2.f - __fdividef(y, s) : 3.f + __fdividef(x, s);
  return p <= 0.f ? 4.f : p;
}
__host__ __device__ inline double pseudo_angle_d(double y, double x) {
  const double s = fabs(x) + fabs(y);
  if (!(s > 0.0)) return 4.0;
  double p;
  if (y >= 0.0) p = x >= 0.0 ? y / s : 1.0 - x / s;
  else p = x < 0.0 ? 2.0 - y / s : 3.0 + x / s;
  return p <= 0.0 ? 4.0 : p;
}

// ---------------------------------------------------------------------------
// Staging (fp64, once per (entry, tile))
// ---------------------------------------------------------------------------
struct Rec {
  float4 r0, r1, r2, r3, r4, r5;  // r5 = low parts (dz0, N_u(d0), N_v(d0)) of the float-float constants
};

// Per-tile constants shared by the CTA: reference ray d0 (tile centre), tile
// origin, bound of |dd| over the tile's pixels.
struct TileConst {
  double d0[3];
  double tx0, ty0;
  float ddmax;
};

__device__ __forceinline__ void stage_record_from(const RasterParams& P, const Geo& g, const TileConst& tc, Rec& R);
__device__ __forceinline__ void stage_record(const RasterParams& P, int id, const TileConst& tc, Rec& R) {
  stage_record_from(P, P.geo[id], tc, R);
}

// g: the primitive's Geo record (global, or a shared-memory copy staged by
// cp.async.bulk in the fast forward)
__device__ __forceinline__ void stage_record_from(const RasterParams& P, const Geo& g, const TileConst& tc, Rec& R) {
  const double d00 = tc.d0[0], d01 = tc.d0[1], d02 = tc.d0[2], tx0 = tc.tx0, ty0 = tc.ty0;
  const double ddmax = tc.ddmax;
  const double a0 = P.cam.o[0] - g.mu[0], a1 = P.cam.o[1] - g.mu[1], a2 = P.cam.o[2] - g.mu[2];
  const double au = g.rx[0] * a0 + g.rx[1] * a1 + g.rx[2] * a2;
  const double av = g.ry[0] * a0 + g.ry[1] * a1 + g.ry[2] * a2;
  const double az = -g.num;  // R_z . (o - mu) = -num exactly (same op order, negated operands)
  const double dz0 = g.rz[0] * d00 + g.rz[1] * d01 + g.rz[2] * d02;
  const double dx0 = g.rx[0] * d00 + g.rx[1] * d01 + g.rx[2] * d02;
  const double dy0 = g.ry[0] * d00 + g.ry[1] * d01 + g.ry[2] * d02;
  const double nu0 = au * dz0 - az * dx0, nv0 = av * dz0 - az * dy0;
  double gu[3], gv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gu[k] = au * g.rz[k] - az * g.rx[k];
    gv[k] = av * g.rz[k] - az * g.ry[k];
  }
  const double rz1 = fabs(g.rz[0]) + fabs(g.rz[1]) + fabs(g.rz[2]);
  const double gu1 = fabs(gu[0]) + fabs(gu[1]) + fabs(gu[2]);
  const double gv1 = fabs(gv[0]) + fabs(gv[1]) + fabs(gv[2]);
  // Absolute error bounds of the per-pixel fp32 evaluations
  // x = hi + (lo + sum_k c_k dd_k) (lin3): the constant enters as a float-float
  // pair, so only the final rounding (2^-24 of |x| <= |x0| + |c|_1 |dd|) and the
  // small linear term (fp32 c, dd and three roundings: <= 3.6e-7 |c|_1 |dd|)
  // contribute.
  const double ez = 6.5e-8 * fabs(dz0) + 4.3e-7 * rz1 * ddmax + 1e-12;
  const double g1 = fmax(gu1, gv1);
  const double eN = 6.5e-8 * fmax(fabs(nu0), fabs(nv0)) + 4.3e-7 * g1 * ddmax + 1e-30;
  const float dz0h = (float)dz0, nu0h = (float)nu0, nv0h = (float)nv0;
  R.r0 = make_float4((float)g.rz[0], (float)g.rz[1], (float)g.rz[2], dz0h);
  R.r1 = make_float4((float)gu[0], (float)gu[1], (float)gu[2], nu0h);
  R.r2 = make_float4((float)gv[0], (float)gv[1], (float)gv[2], nv0h);
  R.r5 = make_float4((float)(dz0 - (double)dz0h), (float)(nu0 - (double)nu0h), (float)(nv0 - (double)nv0h), 0.f);
  R.r3 = make_float4((float)g.num, (float)ez, (float)eN, (float)g.r2max);
  const float fvis2 = g.fvis2;
  R.r4 = g.has_proj ? make_float4((float)(g.ppx - tx0), (float)(g.ppy - ty0), (float)g.dp2max, fvis2)
                    : make_float4(0.f, 0.f, -1.f, fvis2);
}

// Exact r_t of primitive id on the ray of pixel (x, y) (geometry.cpp:40-47,
// reference op order); returns false for grazing / behind.
static __device__ __noinline__ bool exact_rt(const RasterParams& P, int id, int x, int y, double* rt) {
  double dir[3];
  pixel_dir(P.cam, x + 0.5, y + 0.5, dir);
  const Geo& g = P.geo[id];
  const double denom = xdot3(dir[0], dir[1], dir[2], g.rz[0], g.rz[1], g.rz[2]);
  if (fabs(denom) < P.opt.grazing_eps) return false;
  const double r = g.num / denom;
  *rt = r;
  return r > 0;
}

// fp64 composite_candidate values (raster.cpp:327-350) for one popped entry:
// alpha (before the skip test / clamp), low-pass flag, r_t and the normal sign.
struct Pop64 {
  double a, ak, rt;  // alpha, its kernel part o Psi(g)
  double u, v, denom, dpw, dph;  // tangent coordinates, ray-plane denominator, low-pass offsets
  KEval ev;          // kernel intermediates (backward)
  float sgn;
  bool lp, degen;
};
static __device__ __noinline__ void pop_f64(const RasterParams& P, int id, int x, int y, Pop64& o) {
  double dir[3];
  const double px = x + 0.5, py = y + 0.5;
  pixel_dir(P.cam, px, py, dir);
  const Geo& g = P.geo[id];
  const double denom = xdot3(dir[0], dir[1], dir[2], g.rz[0], g.rz[1], g.rz[2]);
  const double rt = g.num / denom;
  const double h0 = xs(xa(P.cam.o[0], xm(rt, dir[0])), g.mu[0]);
  const double h1 = xs(xa(P.cam.o[1], xm(rt, dir[1])), g.mu[1]);
  const double h2 = xs(xa(P.cam.o[2], xm(rt, dir[2])), g.mu[2]);
  const double u = xdot3(g.rx[0], g.rx[1], g.rx[2], h0, h1, h2);
  const double v = xdot3(g.ry[0], g.ry[1], g.ry[2], h0, h1, h2);
  KEval& ev = o.ev;
  eval_kernel(u, v, P.S, id, ev);
  o.degen = ev.degenerate;
  o.rt = rt;
  o.u = u;
  o.v = v;
  o.denom = denom;
  o.dpw = g.has_proj ? xs(px, g.ppx) : 0.0;
  o.dph = g.has_proj ? xs(py, g.ppy) : 0.0;
  o.sgn = denom < 0 ? 1.f : -1.f;
  o.lp = false;
  if (ev.degenerate) {
    o.a = o.ak = 0;
    return;
  }
  const double ak = P.S.o[id] * sharpen(ev.g, P.S.tau[id]);
  o.a = ak;
  o.ak = ak;
  if (g.has_proj) {
    const double f = low_pass_filter_term(o.dpw, o.dph, fabs(denom), P.S.o[id], P.opt.lowpass_radius);
    if (f > ak) {
      o.a = f;
      o.lp = true;
    }
  }
}

template <int RING = kRing>
__device__ __forceinline__ int entry_id(const RasterParams& P, const int* s_id, long long beg, int jr, int ring_lo) {
  return jr >= ring_lo ? s_id[jr & (RING - 1)] : P.lid[beg + jr];
}

// ---------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------
struct FastPixel {
  double T;
  float C0, C1, C2, D, N0, N1, N2, A, E;
  float ddx, ddy, ddz, pxr, pyr;
  int ncomp, stop;
  unsigned n_pop, n_rej1, n_rej2, n_f64, n_miss;
  bool uncertain, err;
};

// composite_candidate up to the blend (raster.cpp:327-348) for one entry:
// tangent coordinates from the staged record, cheap rejects, fp32 alpha with
// its error bound, fp64 re-evaluation of decisions inside the bound.
struct AlphaOut {
  double a;     // clamped alpha (valid unless skip / degen)
  float rel;    // relative error bound of a (0: exact fp64)
  float rt;     // depth
  float sgn;    // normal sign (raster.cpp:350-351)
  bool skip;    // below alpha_min (or rejected): not composited
  bool degen;   // DegenerateBasisError (core.cpp:191)
};

// Intermediates of one composited entry for the backward: fp32 kernel state
// (grad.cpp:16-101 differentiated on the fp32 quantities) or, when the entry
// fell back to fp64, the fp64 evaluation.
struct GradF {
  float u, v, r2, dz, dpx, dpy;
  bool lp, f64;
  KEvalF k;
};

template <bool VALIDATE, bool GRAD = false, bool STATS = true>
__device__ __forceinline__ void alpha_entry(const RasterParams& P, FastPixel& px, const Rec& R, int id, int x, int y,
                                            AlphaOut& out, GradF* gf = nullptr, Pop64* o64 = nullptr) {
  out.skip = false;
  out.degen = false;
#if DRK_EARLY_LOADS
  // the bracket-lookup angles and eta of the shape record, issued before the
  // tangent-coordinate math so that their load latency overlaps it
  const float* hd_e = P.shrec + (size_t)kRecStride * id;
  const float4 ela = __ldg(reinterpret_cast<const float4*>(hd_e) + (DRK_PSEUDO_ANGLE ? 4 : 0));
  const float4 elb = __ldg(reinterpret_cast<const float4*>(hd_e) + (DRK_PSEUDO_ANGLE ? 5 : 1));
  const float eeta = __ldg(hd_e + 16);
#endif
  const float dz = lin3(R.r0, R.r5.x, px.ddx, px.ddy, px.ddz);
  const float nu = lin3(R.r1, R.r5.y, px.ddx, px.ddy, px.ddz);
  const float nv = lin3(R.r2, R.r5.z, px.ddx, px.ddy, px.ddz);
  const float inv = rcp_nr(dz);
  const float ainv = fabsf(inv);
  const float rel_z = R.r3.y * ainv;
  const float u = nu * inv, v = nv * inv;
  float rt = R.r3.x * inv;
  float sgn = dz < 0.f ? 1.f : -1.f;
  const float amin = (float)P.opt.alpha_min;
  float at = 0.f, relt = 0.f;
  bool use64 = rel_z > 1e-3f;
  double a64 = 0;
  (void)px;
  if (!use64) {
#if DRK_EARLY_BRACKET && DRK_EARLY_LOADS
    // bracket lookup and its record loads issued before the radius test: their
    // latency overlaps the error-bound arithmetic (a wasted lookup for the ~7%
    // of pops the radius test rejects)
#if DRK_PSEUDO_ANGLE
    const float th = pseudo_angle(v, u);
    int lo;
    if (th <= ela.y) {
      lo = 7;
    } else {
      lo = (ela.z < th) + (ela.w < th) + (elb.x < th) + (elb.y < th) + (elb.z < th) + (elb.w < th);
    }
#else
    float th = atan2_fast(v, u);
    if (th <= 0.f) th += 6.28318530717958647692f;
    int lo;
    if (th <= ela.x || th > elb.w) {
      lo = 7;
    } else {
      lo = (ela.y < th) + (ela.z < th) + (ela.w < th) + (elb.x < th) + (elb.y < th) + (elb.z < th);
    }
#endif
    const float4* bp_e = reinterpret_cast<const float4*>(hd_e + kRecHdr + 8 * lo);
    const float4 e = __ldg(bp_e), f = __ldg(bp_e + 1);
#endif
    // absolute error bound of u and v (N error / |dz|, relative errors of dz,
    // 1/dz and the product)
    const float du = ainv * R.r3.z + fabsf(u) * (rel_z + 1.85e-7f);
    const float dv = ainv * R.r3.z + fabsf(v) * (rel_z + 1.85e-7f);
    const float dp = fmaxf(du, dv);
    const float r2 = fmaf(u, u, v * v);
    const float au_ = fabsf(u), av_ = fabsf(v);
    const float dr2 = 2.f * (au_ + av_) * dp + 2.f * dp * dp + 2.5e-7f * r2;
    // low-pass reach: dp^2 <= cos^2 dp2max (raster.cpp:337, core.cpp:267-273)
    bool lp_possible = false;
    float dpx = 0.f, dpy = 0.f, dpp2 = 0.f;
    if (R.r4.z >= 0.f) {
      dpx = px.pxr - R.r4.x;
      dpy = px.pyr - R.r4.y;
      dpp2 = fmaf(dpx, dpx, dpy * dpy);
      lp_possible = dpp2 <= dz * dz * R.r4.z * (1.0001f + 4.f * rel_z) + 1e-6f;
    }
    if (r2 - dr2 > R.r3.w * 1.000001f && !lp_possible) {
      DRK_STAT(px.n_rej1);
      out.skip = true;
      return;
    }
    // ---- alpha = o Psi(g(u, v)) (core.cpp:148-265) ----
    const float* hd = P.shrec + (size_t)kRecStride * id;
#if DRK_EARLY_BRACKET && DRK_EARLY_LOADS
    (void)hd;
#elif DRK_PSEUDO_ANGLE
    // bracket from the pseudo-angle (monotone in the polar angle, (0, 4] for
    // (0, 2 pi]) against the record's pseudo-angles of theta_0..theta_6
    // (theta_7 = 2 pi <-> 4); misassignment only within ~5e-7 rad of an
    // endpoint, where the kernel is continuous across brackets (as with the
    // fp32 atan2 it replaces)
#if DRK_EARLY_LOADS
    const float4 p0 = ela, p1 = elb;
#else
    const float4 p0 = __ldg(reinterpret_cast<const float4*>(hd) + 4), p1 = __ldg(reinterpret_cast<const float4*>(hd) + 5);
#endif
    const float th = pseudo_angle(v, u);
    int lo;
    if (th <= p0.y) {
      lo = 7;
    } else {
      lo = (p0.z < th) + (p0.w < th) + (p1.x < th) + (p1.y < th) + (p1.z < th) + (p1.w < th);
    }
#else
#if DRK_EARLY_LOADS
    const float4 t0 = ela, t1 = elb;
#else
    const float4 t0 = __ldg(reinterpret_cast<const float4*>(hd)), t1 = __ldg(reinterpret_cast<const float4*>(hd) + 1);
#endif
    float th = atan2_fast(v, u);
    if (th <= 0.f) th += 6.28318530717958647692f;
    int lo;
    if (th <= t0.x || th > t1.w) {
      lo = 7;
    } else {
      lo = (t0.y < th) + (t0.z < th) + (t0.w < th) + (t1.x < th) + (t1.y < th) + (t1.z < th);
    }
#endif
#if !(DRK_EARLY_BRACKET && DRK_EARLY_LOADS)
    const float4* bp = reinterpret_cast<const float4*>(hd + kRecHdr + 8 * lo);
    const float4 e = __ldg(bp), f = __ldg(bp + 1);  // (elx, ely, ehx, ehy), (1/det, pi/gap, h_lo, h_hi)
#endif
    if (isnan(f.x)) {
      out.degen = true;
      return;
    }
#if DRK_EARLY_LOADS
    const float eta = eeta;
#else
    const float eta = __ldg(hd + 16);
#endif
    const float ka = (e.w * u - e.z * v) * f.x;
    const float kb = (e.x * v - e.y * u) * f.x;
    const float r1 = fabsf(ka) + fabsf(kb);
    const float L1 = fabsf(f.x) * (fabsf(e.x) + fabsf(e.y) + fabsf(e.z) + fabsf(e.w));
    const float dr1 = L1 * (dp + 3.6e-7f * fmaxf(au_, av_));
    const float hmin = fminf(f.z, f.w);
    const float fvis2 = R.r4.w;
    {
      // in-bracket lower bound of Q: alpha_kernel < alpha_min once it exceeds f_vis^2
      const float r1l = fmaxf(r1 - dr1, 0.f);
      const float qlb = eta * r1l * r1l + (1.f - eta) * fmaxf(r2 - dr2, 0.f) * hmin;
      if (qlb > fvis2 * 1.00002f && !lp_possible) {
        DRK_STAT(px.n_rej2);
        out.skip = true;
        return;
      }
    }
#if DRK_SH_PREFETCH
    if (!GRAD) {
      // most entries past the bracket bound composite: pull their SH
      // coefficients into L1 while the kernel value is evaluated
      const char* shp = reinterpret_cast<const char*>(P.sh + (size_t)id * P.terms * 3);
      const size_t bytes = (size_t)P.terms * 12;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(shp));
      if (bytes > 64) asm volatile("prefetch.global.L1 [%0];" ::"l"(shp + bytes - 4));
      if (bytes > 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(shp + 128));
    }
#endif
    const float4 c0 = __ldg(reinterpret_cast<const float4*>(hd) + 2), c1 = __ldg(reinterpret_cast<const float4*>(hd) + 3);
    float ak, relk;
    KEvalF kf;
    if (r2 == 0.f) {
      float relP;
      ak = c1.w * sharpen_ps(c0, c1, 1.0f, 1e-6f, &relP, &kf.A, &kf.br);
      relk = relP + 2e-7f;
      if (GRAD) {
        kf.center = true;
        kf.clamped = false;
        kf.g = 1.f;
        kf.P = ak / c1.w;
      }
    } else {
      // angle from e_lo inside the bracket, delta = that * pi / gap
      const float cr = e.x * v - e.y * u, dt = e.x * u + e.y * v;
      const float dth = atan2_fast(cr, dt);
      const float delta = fmaxf(dth, 0.f) * f.y;
      const float cd = cos_0pi(fminf(delta, 3.14159274f));
      const float hs = 0.5f * (f.z + f.w), hdiff = 0.5f * (f.z - f.w);
      const float inv_s = fmaf(hdiff, cd, hs);
      const float Q = fmaf(eta * r1, r1, (1.f - eta) * r2 * inv_s);
      // error of Q: r1 and r2 from the tangent coordinates, the bracket angle
      // (atan2 + coordinate error) through the cosine blend, __cosf (<= 5e-7
      // absolute), rounding
      // (bound arithmetic: approximate reciprocals, inflated by 1e-3)
      const float dth_err = 2.5e-7f * dth + 2.5e-7f + 1.5015f * dp * rsqrtf(r2);
      const float dinv = fabsf(hdiff) * (dth_err * f.y + 2.4e-7f * delta + 2e-7f) + 2e-7f * (hs + fabsf(hdiff));
      const float dQ = eta * (2.f * r1 * dr1 + dr1 * dr1) + (1.f - eta) * (r2 * dinv + inv_s * dr2) + 3.6e-7f * Q;
      const float ex = fmaxf(-0.5f * Q, -30.0f);
      const float g = __expf(ex);
      float relP;
      const float Pv = sharpen_ps(c0, c1, g, 0.5f * dQ + 2.5e-7f + 7e-8f * fabsf(ex), &relP, &kf.A, &kf.br);
      ak = c1.w * Pv;
      relk = relP + 2e-7f;
      if (GRAD) {
        kf.center = false;
        kf.clamped = -0.5f * Q < -30.0f;
        kf.g = g;
        kf.P = Pv;
        kf.a = ka;
        kf.b = kb;
        kf.r1 = r1;
        kf.delta = delta;
        kf.ch = sqrtf(fmaxf(0.5f * (1.f + cd), 0.f));
        kf.sh = sqrtf(fmaxf(0.5f * (1.f - cd), 0.f));
        kf.inv = inv_s;
        kf.lo = lo;
        kf.hi = (lo + 1) & 7;
      }
    }
    at = ak;
    relt = relk;
    bool lp_used = false;
    if (lp_possible) {
      const float sl = (float)P.opt.lowpass_radius;
      const float den = 2.0f * dz * dz * sl * sl;
      const float exl = fmaxf(-__fdividef(dpp2, den), -30.0f);  // 2 ulp: inside relf's 1e-6 |exl|
      const float fl = c1.w * __expf(exl);
      const float ddp = 6e-8f * (fabsf(R.r4.x) + fabsf(R.r4.y) + 32.f);
      const float relf = 4e-7f + 1.2e-7f * fabsf(exl) + fabsf(exl) * (2.f * rel_z + 1e-6f) +
                         4.004f * (dpp2 > 0.f ? dpp2 * rsqrtf(dpp2) : 0.f) * __fdividef(ddp, den);
      if (fabsf(fl - ak) <= relk * ak + relf * fl) use64 = true;
      if (fl > ak) {
        at = fl;
        relt = relf;
        lp_used = true;
      }
    }
    if (GRAD) {
      gf->u = u;
      gf->v = v;
      gf->r2 = r2;
      gf->dz = dz;
      gf->dpx = dpx;
      gf->dpy = dpy;
      gf->lp = lp_used;
      gf->f64 = false;
      gf->k = kf;
    }
    if (fabsf(at - amin) <= relt * at + 1e-12f) use64 = true;
    if (at >= 0.99f && fabsf(at - 0.999999f) <= relt * at + 1e-6f) use64 = true;
    if (VALIDATE && !use64) {
      Pop64 o;
      pop_f64(P, id, x, y, o);
      // where the floor is certainly out of reach (lp_possible false) the fp32
      // path evaluates the kernel term alone: compare like with like
      const double ref = lp_possible ? o.a : o.ak;
      if (!o.degen && ref >= 1e-4) {
        const double ratio = fabs((double)at - ref) / ((double)relt * at + 1e-30);
        atomicMax(P.vstat, (unsigned long long)__double_as_longlong(ratio));
        atomicMax(P.vstat + 1, (unsigned long long)__double_as_longlong(fabs((double)at - ref)));
        if (ratio > 1.0 && atomicCAS(P.vstat + 2, 0ull, 1ull) == 0ull) {
          double* d = reinterpret_cast<double*>(P.vstat + 3);
          d[0] = x; d[1] = y; d[2] = id; d[3] = u; d[4] = v; d[5] = at; d[6] = ref; d[7] = relt;
          d[8] = lp_possible; d[9] = rel_z; d[10] = dp; d[11] = r1; d[12] = dr1; d[13] = lo;
          d[14] = th; d[15] = ak; d[16] = relk; d[17] = o.a; d[18] = o.ak; d[19] = o.lp; d[20] = dz;
        }
      }
    }
  }
  if (use64) {
    DRK_STAT(px.n_f64);
    Pop64 o_local;
    Pop64& o = GRAD ? *o64 : o_local;
    pop_f64(P, id, x, y, o);
    if (GRAD) gf->f64 = true;
    if (o.degen) {
      out.degen = true;
      return;
    }
    a64 = o.a;
    rt = (float)o.rt;
    sgn = o.sgn;
    relt = 0.f;
    if (a64 < P.opt.alpha_min) {
      out.skip = true;
      return;
    }
    a64 = dmin(a64, 1.0 - 1e-6);
  } else {
    if (at < amin) {
      out.skip = true;
      return;
    }
    a64 = dmin((double)at, 1.0 - 1e-6);
  }
  out.a = a64;
  out.rel = relt;
  out.rt = rt;
  out.sgn = sgn;
}
// blend (raster.cpp:349-361): colour from SH, accumulation, transmittance
// and its error bound; returns false once the pixel saturates.
template <int BSTRIDE = kBatch>
__device__ __forceinline__ bool blend(const RasterParams& P, FastPixel& px, const float4* s_b4, int id, double a64,
                                      float relt, float rt, float sgn, float rz0, float rz1, float rz2) {
  const float* shp = P.sh + (size_t)id * P.terms * 3;
  float c0 = 0.5f, c1 = 0.5f, c2 = 0.5f;
  const int ta = P.opt.terms_active;
  if ((P.terms & 3) == 0 && (ta & 3) == 0) {
    const float4* q = reinterpret_cast<const float4*>(shp);
#pragma unroll
    for (int t = 0; t < 16; t += 4) {
      if (t < ta) {
        const float4 a = __ldg(q + 3 * (t / 4)), b = __ldg(q + 3 * (t / 4) + 1), c = __ldg(q + 3 * (t / 4) + 2);
        const float4 bq = s_b4[(t / 4) * BSTRIDE];  // this pixel's basis, terms t..t+3
        const float b0 = bq.x, b1 = bq.y, b2 = bq.z, b3 = bq.w;
        c0 = fmaf(b0, a.x, c0);
        c1 = fmaf(b0, a.y, c1);
        c2 = fmaf(b0, a.z, c2);
        c0 = fmaf(b1, a.w, c0);
        c1 = fmaf(b1, b.x, c1);
        c2 = fmaf(b1, b.y, c2);
        c0 = fmaf(b2, b.z, c0);
        c1 = fmaf(b2, b.w, c1);
        c2 = fmaf(b2, c.x, c2);
        c0 = fmaf(b3, c.y, c0);
        c1 = fmaf(b3, c.z, c1);
        c2 = fmaf(b3, c.w, c2);
      }
    }
  } else {
    for (int t = 0; t < ta; ++t) {
      const float4 bq = s_b4[(t >> 2) * BSTRIDE];
      const int tq = t & 3;
      const float bt = tq == 0 ? bq.x : (tq == 1 ? bq.y : (tq == 2 ? bq.z : bq.w));
      c0 = fmaf(bt, __ldg(shp + 3 * t), c0);
      c1 = fmaf(bt, __ldg(shp + 3 * t + 1), c1);
      c2 = fmaf(bt, __ldg(shp + 3 * t + 2), c2);
    }
  }
  c0 = fmaxf(c0, 0.f);
  c1 = fmaxf(c1, 0.f);
  c2 = fmaxf(c2, 0.f);
  const float w = (float)(px.T * a64);
  px.C0 = fmaf(w, c0, px.C0);
  px.C1 = fmaf(w, c1, px.C1);
  px.C2 = fmaf(w, c2, px.C2);
  px.D = fmaf(w, rt, px.D);
  const float ws = w * sgn;
  px.N0 = fmaf(ws, rz0, px.N0);
  px.N1 = fmaf(ws, rz1, px.N1);
  px.N2 = fmaf(ws, rz2, px.N2);
  px.A += w;
  px.T = xm(px.T, xs(1.0, a64));
  ++px.ncomp;
  if (relt > 0.f) {
    const float af = (float)a64;
    px.E += relt * __fdividef(af, 1.0f - af) + 1e-15f;
  }
  {
    // |T - early_stop| <= T E, in fp32 with the roundings of T and the threshold covered
    const float tf = (float)px.T, thr = (float)P.opt.early_stop;
    if (fabsf(tf - thr) <= tf * (px.E * 1.001f + 2.5e-7f)) px.uncertain = true;
  }
  if (px.T < P.opt.early_stop) {
    px.stop = px.ncomp;
    return false;
  }
  return true;
}

template <bool VALIDATE, int NT = kBatch, bool STATS = true, int RINGN = 2 * NT>
__device__ __forceinline__ bool pop_eval(const RasterParams& P, FastPixel& px, const float4* s_b4, const Rec* ring,
                                         const int* s_id, const TileConst& tc, long long beg, int ring_lo, int jr,
                                         int x, int y) {
  DRK_STAT(px.n_pop);
  Rec R;
  int id;
  if (jr >= ring_lo) {
    const int slot = jr & (RINGN - 1);
    R = ring[slot];
    id = s_id[slot];
  } else {
    id = P.lid[beg + jr];
    stage_record(P, id, tc, R);
    DRK_STAT(px.n_miss);
  }
  AlphaOut o;
  alpha_entry<VALIDATE, false, STATS>(P, px, R, id, x, y, o);
  if (o.degen) {
    px.err = true;
    return false;
  }
  if (o.skip) return true;
  return blend<NT>(P, px, s_b4, id, o.a, o.rel, o.rt, o.sgn, R.r0.x, R.r0.y, R.r0.z);
}

}  // namespace drk
