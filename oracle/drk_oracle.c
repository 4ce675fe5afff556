/* CPU restatement of the reference DRK rasterizer hot path — TEST
 * INFRASTRUCTURE ONLY.  See drk_oracle.h.  Compile with -ffp-contract=off.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Reductions that Eigen performs (dot, squaredNorm,
 * matrix-vector products, cwiseProduct().sum()) are written out left to
 * right, matching oracle/shim/Eigen/Core against which the reference oracle
 * build is compiled.
 */
#define _GNU_SOURCE
#include "drk_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define TWO_PI (2.0 * M_PI)
#define THREE_SIGMA_LEVEL 1.2340980408667956e-4 /* core.cpp:14 */
#define TAU_LOW (-0.1)
#define TAU_HIGH 0.99
#define MIN_EXPONENT (-30.0)
#define NEAR_CLIP 1e-6 /* raster.cpp:12 */
#define TILE 16
#define CACHE_CAP 8

enum { ST_OK = 0, ST_GENERIC = 1, ST_NONFINITE = 2, ST_DEGEN_QUAT = 3, ST_DEGEN_BASIS = 4,
       ST_REPLAY = 5, ST_DIM = 6, ST_INVALID = 7, ST_OOM = 9 };

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int st, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return st;
}

/* ------------------------------------------------------------------ */
/* small vector helpers (left-to-right, no contraction)                */
/* ------------------------------------------------------------------ */
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
/* static_cast<int>(double) as executed on x86-64 (cvttsd2si): out-of-range and
 * NaN give INT_MIN.  The reference relies on it in raster.cpp:226-231. */
static int x86_int(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return (int)0x80000000u;
  return (int)v;
}

/* ------------------------------------------------------------------ */
/* primitives                                                          */
/* ------------------------------------------------------------------ */
typedef struct Prim {
  double mu[3];
  double R[9]; /* row-major; column c is local axis c (R_x, R_y, R_z = normal) */
  double s[16], th[16];
  double eta, tau, o;
  const double* raw; /* SoA base (for SH) */
  int idx;
} Prim;

typedef struct Scene {
  int n, k, terms;
  const double* raw;
  Prim* p;
} Scene;

static double raw_at(const Scene* sc, int s, int i) { return sc->raw[(size_t)s * sc->n + i]; }
static double sh_at(const Scene* sc, int i, int t, int c) {
  return raw_at(sc, 3 + 4 + 2 * sc->k + 3 + 3 * t + c, i);
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* core.cpp:80 */

/* geometry.cpp:21-30 */
static int quat_to_rotation(const double q[4], double R[9]) {
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (n < 1e-12) return fail(ST_DEGEN_QUAT, "quaternion norm below 1e-12");
  const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
  return ST_OK;
}

/* core.cpp:89-108 */
static void angle_activation(const double* raw, int k, double* theta) {
  const double residual = 1.0 / (k - 2);
  double total = 0;
  for (int i = 0; i < k; ++i) {
    double s = sigmoid(raw[i]);
    s = s < 1e-9 ? 1e-9 : (1.0 - 1e-9 < s ? 1.0 - 1e-9 : s);
    total += s + residual;
    theta[i] = total;
  }
  const double scale = TWO_PI / total;
  for (int i = 0; i < k; ++i) theta[i] = theta[i] * scale;
  theta[k - 1] = TWO_PI;
}

/* core.cpp:133-146 (+ RawDrkParams::all_finite, core.cpp:17-21) */
static int activate_one(const Scene* sc, int i, Prim* p) {
  const int k = sc->k, S = 3 + 4 + 2 * k + 3 + 3 * sc->terms;
  for (int s = 0; s < S; ++s)
    if (!isfinite(raw_at(sc, s, i))) return fail(ST_NONFINITE, "raw parameters contain NaN/Inf");
  if (k < 3) return fail(ST_GENERIC, "K must be at least 3");
  for (int a = 0; a < 3; ++a) p->mu[a] = raw_at(sc, a, i);
  double q[4] = {raw_at(sc, 3, i), raw_at(sc, 4, i), raw_at(sc, 5, i), raw_at(sc, 6, i)};
  int st = quat_to_rotation(q, p->R);
  if (st) return st;
  double ar[16];
  for (int j = 0; j < k; ++j) {
    p->s[j] = exp(raw_at(sc, 7 + j, i));
    ar[j] = raw_at(sc, 7 + k + j, i);
  }
  angle_activation(ar, k, p->th);
  p->eta = sigmoid(raw_at(sc, 7 + 2 * k, i));
  p->tau = TAU_LOW + (TAU_HIGH - TAU_LOW) * sigmoid(raw_at(sc, 8 + 2 * k, i));
  p->o = sigmoid(raw_at(sc, 9 + 2 * k, i));
  p->raw = sc->raw;
  p->idx = i;
  return ST_OK;
}

static int build_scene(Scene* sc, const double* raw, int n, int k, int terms) {
  sc->n = n; sc->k = k; sc->terms = terms; sc->raw = raw;
  if (k > 16 || k < 3) return fail(ST_INVALID, "K outside [3, 16]");
  sc->p = (Prim*)calloc((size_t)(n > 0 ? n : 1), sizeof(Prim));
  if (!sc->p) return fail(ST_OOM, "out of memory");
  for (int i = 0; i < n; ++i) {
    int st = activate_one(sc, i, &sc->p[i]);
    if (st) { free(sc->p); sc->p = NULL; return st; }
  }
  return ST_OK;
}

int orc_activate(const double* raw, int n, int k, int terms, double* mu, double* rot,
                 double* scales, double* angles, double* eta, double* tau, double* opacity) {
  Scene sc;
  int st = build_scene(&sc, raw, n, k, terms);
  if (st) return st;
  for (int i = 0; i < n; ++i) {
    const Prim* p = &sc.p[i];
    memcpy(mu + 3 * i, p->mu, sizeof p->mu);
    memcpy(rot + 9 * i, p->R, sizeof p->R);
    memcpy(scales + (size_t)k * i, p->s, sizeof(double) * k);
    memcpy(angles + (size_t)k * i, p->th, sizeof(double) * k);
    eta[i] = p->eta; tau[i] = p->tau; opacity[i] = p->o;
  }
  free(sc.p);
  return ST_OK;
}

/* ------------------------------------------------------------------ */
/* kernel math (core.cpp)                                              */
/* ------------------------------------------------------------------ */
/* core.cpp:239-245 */
static double sharpen_inverse(double y, double tau) {
  y = dmin(1.0, dmax(0.0, y));
  if (y < (1.0 - tau) / 4.0) return (1.0 + tau) / (1.0 - tau) * y;
  if (y < (3.0 + tau) / 4.0) return ((1.0 - tau) * y + tau) / (1.0 + tau);
  return ((1.0 + tau) * y - 2.0 * tau) / (1.0 - tau);
}
/* core.cpp:210-214 */
static int sharpen_branch(double g, double tau) {
  if (g < (1.0 + tau) / 4.0) return 0;
  if (g < (3.0 - tau) / 4.0) return 1;
  return 2;
}
/* core.cpp:216-219 */
static double sharpen_slope(int b, double tau) {
  if (b == 1) return (1.0 + tau) / (1.0 - tau);
  return (1.0 - tau) / (1.0 + tau);
}
/* core.cpp:221-227 */
static double sharpen_dtau(int b, double g, double tau) {
  if (b == 0) return -2.0 * g / ((1.0 + tau) * (1.0 + tau));
  if (b == 1) return (2.0 * g - 1.0) / ((1.0 - tau) * (1.0 - tau));
  return (2.0 - 2.0 * g) / ((1.0 + tau) * (1.0 + tau));
}
/* core.cpp:229-237 */
static double sharpen(double g, double tau) {
  g = dmin(1.0, dmax(0.0, g));
  switch (sharpen_branch(g, tau)) {
    case 0: return (1.0 - tau) / (1.0 + tau) * g;
    case 1: return ((1.0 + tau) * g - tau) / (1.0 - tau);
    default: return ((1.0 - tau) * g + 2.0 * tau) / (1.0 + tau);
  }
}

typedef struct KEval {
  double value, r2_sq, theta, delta, inv_sbar_sq, a, b, r1;
  int lo, hi, at_center, exp_clamped;
} KEval;

/* core.cpp:148-204.  Returns ST_DEGEN_BASIS on a singular endpoint pair. */
static int eval_kernel(double u, double v, const Prim* p, int k, KEval* ev) {
  memset(ev, 0, sizeof *ev);
  ev->value = 1.0;
  ev->r2_sq = u * u + v * v;
  if (ev->r2_sq == 0) { ev->at_center = 1; return ST_OK; }
  double theta = atan2(v, u);
  if (theta <= 0) theta += TWO_PI;
  ev->theta = theta;
  int lo, hi;
  double alo, ahi;
  if (theta <= p->th[0] || theta > p->th[k - 1]) {
    lo = k - 1; hi = 0;
    alo = p->th[k - 1] - TWO_PI;
    ahi = p->th[0];
    if (theta > p->th[k - 1]) theta -= TWO_PI;
  } else {
    hi = 0; /* lower_bound: first index with th[hi] >= theta */
    while (hi < k && p->th[hi] < theta) ++hi;
    lo = hi - 1;
    alo = p->th[lo];
    ahi = p->th[hi];
  }
  ev->lo = lo; ev->hi = hi;
  ev->delta = (theta - alo) * M_PI / (ahi - alo);
  const double c = cos(ev->delta);
  const double slo = p->s[lo], shi = p->s[hi];
  ev->inv_sbar_sq = (1.0 + c) / (2.0 * slo * slo) + (1.0 - c) / (2.0 * shi * shi);
  const double elx = slo * cos(p->th[lo]), ely = slo * sin(p->th[lo]);
  const double ehx = shi * cos(p->th[hi]), ehy = shi * sin(p->th[hi]);
  const double det = elx * ehy - ely * ehx;
  if (fabs(det) < 1e-12) return fail(ST_DEGEN_BASIS, "adjacent endpoints nearly collinear");
  ev->a = (ehy * u - ehx * v) / det;
  ev->b = (-ely * u + elx * v) / det;
  ev->r1 = fabs(ev->a) + fabs(ev->b);
  double e = -0.5 * (p->eta * ev->r1 * ev->r1 + (1.0 - p->eta) * ev->r2_sq * ev->inv_sbar_sq);
  if (e < MIN_EXPONENT) { e = MIN_EXPONENT; ev->exp_clamped = 1; }
  ev->value = exp(e);
  return ST_OK;
}

/* core.cpp:267-273 */
static double low_pass_filter_term(double dpw, double dph, double cos_view, double o,
                                   const orc_options* opt) {
  const double denom = 2.0 * cos_view * cos_view * opt->lowpass_radius * opt->lowpass_radius;
  double e = -(dpw * dpw + dph * dph) / denom;
  if (e < MIN_EXPONENT) e = MIN_EXPONENT;
  return o * exp(e);
}

/* core.cpp:305-318.  Returns 0 when alpha can never reach alpha_min. */
static int binning_radius_factor(double o, double tau, double amin, double* factor) {
  const double vis = amin / o;
  if (vis >= 1.0) return 0;
  const double gv = sharpen_inverse(vis, tau);
  double f = sqrt(-2.0 * log(gv));
  const double cal = THREE_SIGMA_LEVEL / o;
  if (cal < 1.0) {
    const double gc = sharpen_inverse(cal, tau);
    if (gc > 0 && gc < 1) f = dmax(f, sqrt(-log(gc)));
  }
  *factor = f;
  return 1;
}

/* ------------------------------------------------------------------ */
/* geometry (geometry.cpp)                                             */
/* ------------------------------------------------------------------ */
typedef struct Ray { double o[3], d[3]; } Ray;

/* geometry.cpp:32-38 with Camera::position (geometry.hpp:15) */
static Ray pixel_ray(const orc_camera* c, double px, double py) {
  Ray r;
  const double* R = c->R;
  const double dc[3] = {(px - c->cx) / c->fx, (py - c->cy) / c->fy, 1.0};
  for (int i = 0; i < 3; ++i) r.o[i] = (-R[0 + i]) * c->t[0] + (-R[3 + i]) * c->t[1] + (-R[6 + i]) * c->t[2];
  double v[3];
  for (int i = 0; i < 3; ++i) v[i] = R[0 + i] * dc[0] + R[3 + i] * dc[1] + R[6 + i] * dc[2];
  const double sq = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (sq > 0) {
    const double nn = sqrt(sq);
    for (int i = 0; i < 3; ++i) v[i] = v[i] / nn;
  }
  memcpy(r.d, v, sizeof v);
  return r;
}

static void prim_col(const Prim* p, int c, double out[3]) {
  out[0] = p->R[c]; out[1] = p->R[3 + c]; out[2] = p->R[6 + c];
}

enum { HIT = 0, GRAZING = 1, BEHIND = 2 };
/* geometry.cpp:40-52 */
static int classify_intersect(const Ray* ray, const Prim* p, double eps, double* rt_out,
                              double* u_out, double* v_out) {
  double rz[3], rx[3], ry[3];
  prim_col(p, 2, rz);
  const double denom = dot3(ray->d, rz);
  if (fabs(denom) < eps) return GRAZING;
  const double m[3] = {p->mu[0] - ray->o[0], p->mu[1] - ray->o[1], p->mu[2] - ray->o[2]};
  const double rt = dot3(m, rz) / denom;
  if (rt <= 0) return BEHIND;
  const double d[3] = {ray->o[0] + rt * ray->d[0] - p->mu[0], ray->o[1] + rt * ray->d[1] - p->mu[1],
                       ray->o[2] + rt * ray->d[2] - p->mu[2]};
  prim_col(p, 0, rx);
  prim_col(p, 1, ry);
  *rt_out = rt;
  *u_out = dot3(rx, d);
  *v_out = dot3(ry, d);
  return HIT;
}

static void to_camera(const orc_camera* c, const double w[3], double out[3]) {
  for (int i = 0; i < 3; ++i)
    out[i] = (c->R[3 * i] * w[0] + c->R[3 * i + 1] * w[1] + c->R[3 * i + 2] * w[2]) + c->t[i];
}

/* geometry.cpp:67-74 */
static int try_project_point(const orc_camera* c, const double w[3], double out[3]) {
  double p[3];
  to_camera(c, w, p);
  if (p[2] <= 0) return 0;
  out[0] = c->fx * p[0] / p[2] + c->cx;
  out[1] = c->fy * p[1] / p[2] + c->cy;
  out[2] = p[2];
  return 1;
}

/* geometry.cpp:82-89: J = [fx/z 0 -fx x/z^2; 0 fy/z -fy y/z^2] * R */
static void projection_jacobian(const orc_camera* c, const double w[3], double J[6]) {
  double p[3];
  to_camera(c, w, p);
  const double z = p[2];
  const double jc[6] = {c->fx / z, 0, -c->fx * p[0] / (z * z), 0, c->fy / z, -c->fy * p[1] / (z * z)};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      J[3 * i + j] = jc[3 * i] * c->R[j] + jc[3 * i + 1] * c->R[3 + j] + jc[3 * i + 2] * c->R[6 + j];
}

/* geometry.cpp:91-124 */
static const double kSh0 = 0.28209479177387814;
static const double kSh1 = 0.4886025119029199;
static const double kSh2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                               -1.0925484305920792, 0.5462742152960396};
static const double kSh3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                               0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                               -0.5900435899266435};
static void sh_basis(const double* dir, int degree, double* out) {
  const double x = dir[0], y = dir[1], z = dir[2];
  out[0] = kSh0;
  if (degree < 1) return;
  out[1] = -kSh1 * y;
  out[2] = kSh1 * z;
  out[3] = -kSh1 * x;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  const double xy = x * y, yz = y * z, xz = x * z;
  out[4] = kSh2[0] * xy;
  out[5] = kSh2[1] * yz;
  out[6] = kSh2[2] * (2 * zz - xx - yy);
  out[7] = kSh2[3] * xz;
  out[8] = kSh2[4] * (xx - yy);
  if (degree < 3) return;
  out[9] = kSh3[0] * y * (3 * xx - yy);
  out[10] = kSh3[1] * xy * z;
  out[11] = kSh3[2] * y * (4 * zz - xx - yy);
  out[12] = kSh3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  out[13] = kSh3[4] * x * (4 * zz - xx - yy);
  out[14] = kSh3[5] * z * (xx - yy);
  out[15] = kSh3[6] * x * (xx - 3 * yy);
}

static int active_terms(const Scene* sc, int degree) {
  const int t = (degree + 1) * (degree + 1);
  return t < sc->terms ? t : sc->terms;
}

/* geometry.cpp:126-138 */
static void sh_eval(const Scene* sc, int i, const double* dir, int degree, double rgb[3], int clamped[3]) {
  double basis[16];
  sh_basis(dir, degree, basis);
  const int terms = active_terms(sc, degree);
  rgb[0] = rgb[1] = rgb[2] = 0.5;
  for (int t = 0; t < terms; ++t)
    for (int c = 0; c < 3; ++c) rgb[c] += basis[t] * sh_at(sc, i, t, c);
  for (int c = 0; c < 3; ++c) {
    clamped[c] = rgb[c] < 0;
    if (clamped[c]) rgb[c] = 0;
  }
}

/* ------------------------------------------------------------------ */
/* binning (raster.cpp:12-265)                                         */
/* ------------------------------------------------------------------ */
typedef struct V3buf { double* v; int n, cap; } V3buf;
static void v3_push(V3buf* b, const double p[3]) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 256;
    b->v = (double*)realloc(b->v, sizeof(double) * 3 * b->cap);
  }
  memcpy(b->v + 3 * b->n, p, sizeof(double) * 3);
  b->n++;
}

typedef struct PolyCtx {
  const Prim* p;
  const orc_camera* cam;
  double support_c, alo, gap, slo, shi, elx, ely, ehx, ehy, det;
  V3buf* out;
} PolyCtx;

typedef struct W2 { double rho1, inv_sbar; } W2;

/* raster.cpp:158-168 */
static W2 weight_at(const PolyCtx* c, double a) {
  const double delta = (a - c->alo) * M_PI / c->gap;
  const double cd = cos(delta);
  W2 w;
  w.inv_sbar = (1.0 + cd) / (2.0 * c->slo * c->slo) + (1.0 - cd) / (2.0 * c->shi * c->shi);
  const double dx = cos(a), dy = sin(a);
  const double ca = (c->ehy * dx - c->ehx * dy) / c->det;
  const double cb = (-c->ely * dx + c->elx * dy) / c->det;
  w.rho1 = fabs(ca) + fabs(cb);
  return w;
}
/* raster.cpp:170-173 */
static double radius_true(const PolyCtx* c, W2 w) {
  const double total = c->p->eta * w.rho1 * w.rho1 + (1.0 - c->p->eta) * w.inv_sbar;
  return sqrt(c->support_c / dmax(total, 1e-12));
}
/* raster.cpp:178-198 */
static void emit(const PolyCtx* c, double a0, double a1, W2 w0, W2 w1, int depth) {
  const Prim* p = c->p;
  const double rho1_min = dmin(w0.rho1, w1.rho1);
  const double inv_min = dmin(w0.inv_sbar, w1.inv_sbar);
  const double w_lb = p->eta * rho1_min * rho1_min + (1.0 - p->eta) * inv_min;
  const double bound = sqrt(c->support_c / dmax(w_lb, 1e-12)) / cos(0.5 * (a1 - a0));
  if (depth < 9 && a1 - a0 > 2e-3 && bound > 1.25 * dmin(radius_true(c, w0), radius_true(c, w1))) {
    const double mid = 0.5 * (a0 + a1);
    const W2 wm = weight_at(c, mid);
    emit(c, a0, mid, w0, wm, depth + 1);
    emit(c, mid, a1, wm, w1, depth + 1);
    return;
  }
  const double as[2] = {a0, a1};
  double rx[3], ry[3];
  prim_col(p, 0, rx);
  prim_col(p, 1, ry);
  for (int j = 0; j < 2; ++j) {
    const double ca = cos(as[j]), sa = sin(as[j]);
    double w[3], pc[3];
    for (int i = 0; i < 3; ++i) w[i] = p->mu[i] + bound * (ca * rx[i] + sa * ry[i]);
    to_camera(c->cam, w, pc);
    v3_push(c->out, pc);
  }
}

/* raster.cpp:15-30 */
static void clip_near(const V3buf* in, V3buf* out) {
  out->n = 0;
  const int n = in->n;
  for (int i = 0; i < n; ++i) {
    const double* a = in->v + 3 * i;
    const double* b = in->v + 3 * ((i + 1) % n);
    const int a_in = a[2] >= NEAR_CLIP, b_in = b[2] >= NEAR_CLIP;
    if (a_in) v3_push(out, a);
    if (a_in != b_in) {
      const double t = (NEAR_CLIP - a[2]) / (b[2] - a[2]);
      const double q[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]), a[2] + t * (b[2] - a[2])};
      v3_push(out, q);
    }
  }
}

typedef struct P2 { double x, y; } P2;
static int cmp_p2(const void* A, const void* B) {
  const P2* a = (const P2*)A;
  const P2* b = (const P2*)B;
  if (a->x < b->x || (a->x == b->x && a->y < b->y)) return -1;
  if (b->x < a->x || (b->x == a->x && b->y < a->y)) return 1;
  return 0;
}
static double cross2(P2 o, P2 a, P2 b) { return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x); }

/* raster.cpp:33-58; hull written into h (capacity >= 2n), returns its size */
static int convex_hull(P2* pts, int n, P2* h) {
  qsort(pts, n, sizeof(P2), cmp_p2);
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || !(pts[i].x == pts[m - 1].x && pts[i].y == pts[m - 1].y)) pts[m++] = pts[i];
  n = m;
  if (n <= 2) {
    memcpy(h, pts, sizeof(P2) * n);
    return n;
  }
  int k = 0;
  for (int i = 0; i < n; ++i) {
    while (k >= 2 && cross2(h[k - 2], h[k - 1], pts[i]) <= 0) --k;
    h[k++] = pts[i];
  }
  const int lower = k + 1;
  for (int i = n - 2; i >= 0; --i) {
    while (k >= lower && cross2(h[k - 2], h[k - 1], pts[i]) <= 0) --k;
    h[k++] = pts[i];
  }
  return k - 1;
}

/* raster.cpp:63-97 */
static int hull_overlaps_rect(const P2* h, int n, double x0, double y0, double x1, double y1) {
  if (n == 0) return 0;
  double hx0 = h[0].x, hx1 = h[0].x, hy0 = h[0].y, hy1 = h[0].y;
  for (int i = 0; i < n; ++i) {
    hx0 = dmin(hx0, h[i].x); hx1 = dmax(hx1, h[i].x);
    hy0 = dmin(hy0, h[i].y); hy1 = dmax(hy1, h[i].y);
  }
  if (hx1 < x0 || hx0 > x1 || hy1 < y0 || hy0 > y1) return 0;
  if (n <= 1) return 1;
  const P2 cs[4] = {{x0, y0}, {x1, y0}, {x1, y1}, {x0, y1}};
  for (int i = 0; i < n; ++i) {
    const P2 a = h[i], b = h[(i + 1) % n];
    const double ex = b.x - a.x, ey = b.y - a.y;
    if (ex * ex + ey * ey < 1e-24) continue;
    const double ax = -ey, ay = ex;
    double pmin = ax * h[0].x + ay * h[0].y, pmax = pmin;
    for (int j = 0; j < n; ++j) {
      const double d = ax * h[j].x + ay * h[j].y;
      pmin = dmin(pmin, d); pmax = dmax(pmax, d);
    }
    double rmin = ax * cs[0].x + ay * cs[0].y, rmax = rmin;
    for (int j = 0; j < 4; ++j) {
      const double d = ax * cs[j].x + ay * cs[j].y;
      rmin = dmin(rmin, d); rmax = dmax(rmax, d);
    }
    if (pmax < rmin || pmin > rmax) return 0;
  }
  return 1;
}

/* raster.cpp:99-115 */
static double nearest_depth_key(const Prim* p, const orc_camera* cam, const orc_options* opt,
                                double x0, double y0, double x1, double y1) {
  const double xs[5] = {x0, x1, x1, x0, 0.5 * (x0 + x1)};
  const double ys[5] = {y0, y0, y1, y1, 0.5 * (y0 + y1)};
  double best = INFINITY;
  for (int i = 0; i < 5; ++i) {
    const Ray r = pixel_ray(cam, xs[i], ys[i]);
    double rt, u, v;
    if (classify_intersect(&r, p, opt->grazing_eps, &rt, &u, &v) == HIT) best = dmin(best, rt);
  }
  if (isinf(best)) {
    double pr[3];
    if (try_project_point(cam, p->mu, pr)) best = pr[2];
  }
  return best;
}

typedef struct Entry { double key; int32_t id; } Entry;
typedef struct EntryVec { Entry* v; int64_t n, cap; } EntryVec;
static void ev_push(EntryVec* b, Entry e) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 64;
    b->v = (Entry*)realloc(b->v, sizeof(Entry) * b->cap);
  }
  b->v[b->n++] = e;
}
static int cmp_entry(const void* A, const void* B) {
  const Entry* a = (const Entry*)A;
  const Entry* b = (const Entry*)B;
  if (a->key < b->key || (a->key == b->key && a->id < b->id)) return -1;
  if (b->key < a->key || (b->key == a->key && b->id < a->id)) return 1;
  return 0;
}

typedef struct Bins {
  int tiles_x, tiles_y;
  EntryVec* tiles;
} Bins;

static void free_bins(Bins* b) {
  if (!b->tiles) return;
  for (int t = 0; t < b->tiles_x * b->tiles_y; ++t) free(b->tiles[t].v);
  free(b->tiles);
  b->tiles = NULL;
}

/* raster.cpp:119-265 */
static void bin_primitives(const Scene* sc, const orc_camera* cam, const orc_options* opt, Bins* bins,
                           orc_stats* stats) {
  bins->tiles_x = (cam->width + TILE - 1) / TILE;
  bins->tiles_y = (cam->height + TILE - 1) / TILE;
  bins->tiles = (EntryVec*)calloc((size_t)bins->tiles_x * bins->tiles_y + 1, sizeof(EntryVec));
  const double lp_pad = opt->lowpass_radius * sqrt(2.0 * log(1.0 / opt->alpha_min)) + 1e-9;
  V3buf poly = {0}, clipped = {0};
  P2* pts = NULL;
  P2* hull = NULL;
  int pts_cap = 0;
  const int k = sc->k;
  for (int pid = 0; pid < sc->n; ++pid) {
    const Prim* p = &sc->p[pid];
    double factor;
    if (!binning_radius_factor(p->o, p->tau, opt->alpha_min, &factor)) continue;
    PolyCtx c;
    c.p = p;
    c.cam = cam;
    c.support_c = factor * factor;
    c.out = &poly;
    poly.n = 0;
    for (int kk = 0; kk < k; ++kk) {
      const int hi = (kk + 1) % k;
      c.alo = kk + 1 < k ? p->th[kk] : p->th[kk] - 2.0 * M_PI;
      const double ahi = kk + 1 < k ? p->th[hi] : p->th[0];
      c.gap = ahi - c.alo;
      c.slo = p->s[kk];
      c.shi = p->s[hi];
      c.elx = p->s[kk] * cos(p->th[kk]); c.ely = p->s[kk] * sin(p->th[kk]);
      c.ehx = p->s[hi] * cos(p->th[hi]); c.ehy = p->s[hi] * sin(p->th[hi]);
      c.det = c.elx * c.ehy - c.ely * c.ehx;
      const int coarse_i = (int)ceil(c.gap / (M_PI / 8.0));
      const int coarse = coarse_i > 1 ? coarse_i : 1;
      W2 prev = weight_at(&c, c.alo);
      for (int j = 0; j < coarse; ++j) {
        const double a0 = c.alo + c.gap * j / coarse;
        const double a1 = c.alo + c.gap * (j + 1) / coarse;
        const W2 next = weight_at(&c, a1);
        emit(&c, a0, a1, prev, next, 0);
        prev = next;
      }
    }
    if (stats) {
      stats->poly_vertices += poly.n;
      if (poly.n > stats->max_poly) stats->max_poly = poly.n;
    }
    clip_near(&poly, &clipped);
    if (clipped.n == 0) continue;
    if (clipped.n > pts_cap) {
      pts_cap = clipped.n;
      pts = (P2*)realloc(pts, sizeof(P2) * pts_cap);
      hull = (P2*)realloc(hull, sizeof(P2) * 2 * pts_cap + 2);
    }
    for (int i = 0; i < clipped.n; ++i) {
      const double* q = clipped.v + 3 * i;
      pts[i].x = cam->fx * q[0] / q[2] + cam->cx;
      pts[i].y = cam->fy * q[1] / q[2] + cam->cy;
    }
    const int hn = convex_hull(pts, clipped.n, hull);
    if (hn == 0) continue;
    double hx0 = hull[0].x, hx1 = hx0, hy0 = hull[0].y, hy1 = hy0;
    for (int i = 0; i < hn; ++i) {
      hx0 = dmin(hx0, hull[i].x); hx1 = dmax(hx1, hull[i].x);
      hy0 = dmin(hy0, hull[i].y); hy1 = dmax(hy1, hull[i].y);
    }
    int tx0 = x86_int(floor((hx0 - lp_pad) / TILE)); tx0 = tx0 > 0 ? tx0 : 0;
    int tx1 = x86_int(floor((hx1 + lp_pad) / TILE)); tx1 = tx1 < bins->tiles_x - 1 ? tx1 : bins->tiles_x - 1;
    int ty0 = x86_int(floor((hy0 - lp_pad) / TILE)); ty0 = ty0 > 0 ? ty0 : 0;
    int ty1 = x86_int(floor((hy1 + lp_pad) / TILE)); ty1 = ty1 < bins->tiles_y - 1 ? ty1 : bins->tiles_y - 1;
    for (int ty = ty0; ty <= ty1; ++ty) {
      for (int tx = tx0; tx <= tx1; ++tx) {
        const double x0 = tx * TILE, y0 = ty * TILE, x1 = x0 + TILE, y1 = y0 + TILE;
        if (!hull_overlaps_rect(hull, hn, x0 - lp_pad, y0 - lp_pad, x1 + lp_pad, y1 + lp_pad)) continue;
        double key = 0;
        if (opt->presort == 0) {
          key = (double)pid;
        } else if (opt->presort == 1) {
          double pr[3];
          key = try_project_point(cam, p->mu, pr) ? pr[2] : INFINITY;
        } else {
          key = nearest_depth_key(p, cam, opt, x0, y0, x1, y1);
        }
        Entry e = {key, pid};
        ev_push(&bins->tiles[ty * bins->tiles_x + tx], e);
      }
    }
  }
  for (int t = 0; t < bins->tiles_x * bins->tiles_y; ++t) {
    EntryVec* l = &bins->tiles[t];
    if (l->n > 1) qsort(l->v, l->n, sizeof(Entry), cmp_entry);
    if (stats) stats->pairs += l->n;
  }
  free(poly.v); free(clipped.v); free(pts); free(hull);
}

static Bins g_bins;

int orc_bin(const double* raw, int n, int k, int terms, const orc_camera* cam, const orc_options* opt,
            int64_t* total_pairs) {
  Scene sc;
  int st = build_scene(&sc, raw, n, k, terms);
  if (st) return st;
  free_bins(&g_bins);
  orc_stats stats = {0};
  bin_primitives(&sc, cam, opt, &g_bins, &stats);
  *total_pairs = stats.pairs;
  free(sc.p);
  return ST_OK;
}

void orc_bins_copy(int64_t* offsets, int32_t* ids, double* keys) {
  int64_t o = 0;
  offsets[0] = 0;
  for (int t = 0; t < g_bins.tiles_x * g_bins.tiles_y; ++t) {
    const EntryVec* l = &g_bins.tiles[t];
    for (int64_t j = 0; j < l->n; ++j) {
      ids[o + j] = l->v[j].id;
      keys[o + j] = l->v[j].key;
    }
    o += l->n;
    offsets[t + 1] = o;
  }
}

/* ------------------------------------------------------------------ */
/* render (raster.cpp:267-485)                                         */
/* ------------------------------------------------------------------ */
typedef struct CEntry { double depth; int id; double u, v; } CEntry;
typedef struct Cache { CEntry e[CACHE_CAP]; int size; } Cache;
enum { R_NONE = 0, R_POPPED = 1, R_FINISHED = 2 };

/* raster.cpp:267-303 */
static int cache_step(Cache* c, const CEntry* in, CEntry* popped) {
  if (c->size == 0) {
    if (!in) return R_FINISHED;
    c->e[0] = *in;
    c->size = 1;
    return R_NONE;
  }
  if (!in) {
    *popped = c->e[0];
    --c->size;
    for (int i = 0; i < c->size; ++i) c->e[i] = c->e[i + 1];
    return R_POPPED;
  }
  if (c->size == CACHE_CAP) {
    if (in->depth < c->e[0].depth) {
      *popped = *in;
      return R_POPPED;
    }
    *popped = c->e[0];
    int pos = 1;
    while (pos < CACHE_CAP && c->e[pos].depth <= in->depth) {
      c->e[pos - 1] = c->e[pos];
      ++pos;
    }
    c->e[pos - 1] = *in;
    return R_POPPED;
  }
  int pos = c->size;
  while (pos > 0 && c->e[pos - 1].depth > in->depth) {
    c->e[pos] = c->e[pos - 1];
    --pos;
  }
  c->e[pos] = *in;
  ++c->size;
  return R_NONE;
}

typedef struct Rec { int id; double u, v, depth, alpha; int lowpass; } Rec;
typedef struct RecVec { Rec* v; int64_t n, cap; } RecVec;
static void rec_push(RecVec* b, Rec r) {
  if (b->n == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 64;
    b->v = (Rec*)realloc(b->v, sizeof(Rec) * b->cap);
  }
  b->v[b->n++] = r;
}

typedef struct PixelState { double color[3], depth, normal[3], alpha, T; } PixelState;

typedef struct RCtx {
  const Scene* sc;
  const orc_camera* cam;
  const orc_options* opt;
  double* proj; /* n x 3 */
  char* has_proj;
  int err;
} RCtx;

/* raster.cpp:327-362; returns 0 once the pixel saturates */
static int composite_candidate(RCtx* cx, const Ray* ray, double px, double py, const CEntry* e,
                               PixelState* st, RecVec* rec, orc_stats* stats) {
  const Prim* p = &cx->sc->p[e->id];
  const orc_options* opt = cx->opt;
  KEval ev;
  if (eval_kernel(e->u, e->v, p, cx->sc->k, &ev)) { cx->err = ST_DEGEN_BASIS; return 0; }
  const double a_kernel = p->o * sharpen(ev.value, p->tau);
  double a = a_kernel;
  int lp = 0;
  double rz[3];
  prim_col(p, 2, rz);
  const double cos_view = fabs(dot3(ray->d, rz));
  if (cx->has_proj[e->id]) {
    const double dpw = px - cx->proj[3 * e->id], dph = py - cx->proj[3 * e->id + 1];
    const double f = low_pass_filter_term(dpw, dph, cos_view, p->o, opt);
    if (f > a_kernel) { a = f; lp = 1; }
  }
  if (stats) stats->popped++;
  if (a < opt->alpha_min) return 1;
  a = dmin(a, 1.0 - 1e-6);
  double rgb[3];
  int clamped[3];
  sh_eval(cx->sc, e->id, ray->d, opt->sh_degree, rgb, clamped);
  const double sgn = dot3(ray->d, rz) < 0 ? 1.0 : -1.0;
  const double w = st->T * a;
  for (int c = 0; c < 3; ++c) st->color[c] += w * rgb[c];
  st->depth += w * e->depth;
  for (int c = 0; c < 3; ++c) st->normal[c] += w * (sgn * rz[c]);
  st->alpha += w;
  st->T *= 1.0 - a;
  if (stats) stats->composited++;
  if (rec) {
    Rec r = {e->id, e->u, e->v, e->depth, a, lp};
    rec_push(rec, r);
  }
  return st->T >= opt->early_stop_transmittance;
}

static int cmp_depth_stable(const void* A, const void* B) {
  const CEntry* a = (const CEntry*)A;
  const CEntry* b = (const CEntry*)B;
  if (a->depth < b->depth) return -1;
  if (b->depth < a->depth) return 1;
  return 0;
}

/* std::stable_sort by depth (raster.cpp:396-399): insertion-merge via an index tiebreak */
static void stable_sort_depth(CEntry* v, int n) {
  /* simple stable insertion sort for small lists, merge sort otherwise */
  if (n < 2) return;
  CEntry* tmp = (CEntry*)malloc(sizeof(CEntry) * n);
  for (int w = 1; w < n; w *= 2) {
    for (int i = 0; i < n; i += 2 * w) {
      int a = i, am = i + w < n ? i + w : n, b = am, bm = i + 2 * w < n ? i + 2 * w : n, o = i;
      while (a < am && b < bm) tmp[o++] = (cmp_depth_stable(&v[b], &v[a]) < 0) ? v[b++] : v[a++];
      while (a < am) tmp[o++] = v[a++];
      while (b < bm) tmp[o++] = v[b++];
    }
    memcpy(v, tmp, sizeof(CEntry) * n);
  }
  free(tmp);
}

static RecVec* g_replay_px = NULL;
static int64_t g_replay_pixels = 0;
static void free_replay(void) {
  if (!g_replay_px) return;
  for (int64_t i = 0; i < g_replay_pixels; ++i) free(g_replay_px[i].v);
  free(g_replay_px);
  g_replay_px = NULL;
  g_replay_pixels = 0;
}

/* raster.cpp:364-430 */
static void render_tile(RCtx* cx, const Bins* bins, int tx, int ty, double* color, double* depth,
                        double* normal, double* alpha, RecVec* replay, orc_stats* stats) {
  const orc_camera* cam = cx->cam;
  const orc_options* opt = cx->opt;
  const EntryVec* cand = &bins->tiles[ty * bins->tiles_x + tx];
  const int x0 = tx * TILE, y0 = ty * TILE;
  const int x1 = cam->width < x0 + TILE ? cam->width : x0 + TILE;
  const int y1 = cam->height < y0 + TILE ? cam->height : y0 + TILE;
  CEntry* valid = (CEntry*)malloc(sizeof(CEntry) * (cand->n + 1));
  for (int y = y0; y < y1; ++y) {
    for (int x = x0; x < x1; ++x) {
      const double px = x + 0.5, py = y + 0.5;
      const Ray ray = pixel_ray(cam, px, py);
      int nv = 0;
      for (int64_t j = 0; j < cand->n; ++j) {
        const int id = cand->v[j].id;
        double rt, u, v;
        if (classify_intersect(&ray, &cx->sc->p[id], opt->grazing_eps, &rt, &u, &v) != HIT) continue;
        CEntry e = {rt, id, u, v};
        valid[nv++] = e;
      }
      if (stats) stats->hits += nv;
      PixelState st = {{0, 0, 0}, 0, {0, 0, 0}, 0, 1.0};
      RecVec* rp = replay ? &replay[(size_t)y * cam->width + x] : NULL;
      if (opt->exact_sort) {
        stable_sort_depth(valid, nv);
        for (int i = 0; i < nv; ++i) {
          if (stats) stats->streamed++;
          if (!composite_candidate(cx, &ray, px, py, &valid[i], &st, rp, stats)) break;
        }
      } else if (opt->use_cache) {
        Cache cache;
        cache.size = 0;
        CEntry popped;
        int saturated = 0;
        for (int i = 0; i < nv && !saturated; ++i) {
          if (stats) stats->streamed++;
          if (cache_step(&cache, &valid[i], &popped) == R_POPPED)
            saturated = !composite_candidate(cx, &ray, px, py, &popped, &st, rp, stats);
        }
        while (!saturated) {
          if (cache_step(&cache, NULL, &popped) == R_FINISHED) break;
          saturated = !composite_candidate(cx, &ray, px, py, &popped, &st, rp, stats);
        }
      } else {
        for (int i = 0; i < nv; ++i) {
          if (stats) stats->streamed++;
          if (!composite_candidate(cx, &ray, px, py, &valid[i], &st, rp, stats)) break;
        }
      }
      for (int c = 0; c < 3; ++c) st.color[c] += st.T * opt->background[c];
      const size_t pix = (size_t)y * cam->width + x;
      for (int c = 0; c < 3; ++c) {
        if (color) color[3 * pix + c] = st.color[c];
        if (normal) normal[3 * pix + c] = st.normal[c];
      }
      if (depth) depth[pix] = st.depth;
      if (alpha) alpha[pix] = st.alpha;
    }
  }
  free(valid);
}

static void project_centers(const Scene* sc, const orc_camera* cam, double* proj, char* has) {
  for (int i = 0; i < sc->n; ++i) has[i] = (char)try_project_point(cam, sc->p[i].mu, proj + 3 * i);
}

int orc_render(const double* raw, int n, int k, int terms, const orc_camera* cam, const orc_options* opt,
               double* color, double* depth, double* normal, double* alpha, int want_replay,
               int64_t* replay_records, orc_stats* stats) {
  Scene sc;
  int st = build_scene(&sc, raw, n, k, terms);
  if (st) return st;
  if (stats) memset(stats, 0, sizeof *stats);
  Bins bins = {0};
  bin_primitives(&sc, cam, opt, &bins, stats);
  RCtx cx = {&sc, cam, opt, (double*)calloc((size_t)3 * (n + 1), sizeof(double)),
             (char*)calloc((size_t)n + 1, 1), 0};
  project_centers(&sc, cam, cx.proj, cx.has_proj);
  free_replay();
  RecVec* replay = NULL;
  if (want_replay) {
    g_replay_pixels = (int64_t)cam->width * cam->height;
    g_replay_px = replay = (RecVec*)calloc((size_t)g_replay_pixels + 1, sizeof(RecVec));
  }
  for (int t = 0; t < bins.tiles_x * bins.tiles_y; ++t)
    render_tile(&cx, &bins, t % bins.tiles_x, t / bins.tiles_x, color, depth, normal, alpha, replay, stats);
  if (replay && replay_records) {
    int64_t tot = 0;
    for (int64_t i = 0; i < g_replay_pixels; ++i) tot += replay[i].n;
    *replay_records = tot;
  }
  free_bins(&bins);
  free(cx.proj);
  free(cx.has_proj);
  free(sc.p);
  if (cx.err) return fail(cx.err, "adjacent endpoints nearly collinear");
  return ST_OK;
}

void orc_replay_copy(int64_t* offsets, int32_t* ids, double* vals) {
  int64_t o = 0;
  offsets[0] = 0;
  for (int64_t p = 0; p < g_replay_pixels; ++p) {
    const RecVec* r = &g_replay_px[p];
    for (int64_t j = 0; j < r->n; ++j) {
      const Rec* q = &r->v[j];
      ids[o + j] = q->id;
      double* v = vals + 5 * (o + j);
      v[0] = q->u; v[1] = q->v; v[2] = q->depth; v[3] = q->alpha; v[4] = q->lowpass;
    }
    o += r->n;
    offsets[p + 1] = o;
  }
}

/* ------------------------------------------------------------------ */
/* backward (grad.cpp)                                                 */
/* ------------------------------------------------------------------ */
/* PrimGrads (grad.hpp:19-29) flattened: d_center[3], d_rot[9] (row-major),
 * d_scales[K], d_angles[K], d_eta, d_tau, d_opacity, d_sh[terms*3]. */
typedef struct GLayout { int k, terms, rot, sc, an, eta, tau, op, sh, size; } GLayout;
static GLayout glayout(int k, int terms) {
  GLayout L;
  L.k = k; L.terms = terms;
  L.rot = 3; L.sc = 12; L.an = 12 + k; L.eta = 12 + 2 * k; L.tau = L.eta + 1; L.op = L.eta + 2;
  L.sh = L.eta + 3; L.size = L.sh + 3 * terms;
  return L;
}

typedef struct AGrads { double ds[16], da[16], d_eta, d_tau, d_op, d_u, d_v; } AGrads;

/* grad.cpp:16-101 */
static void backward_alpha(double u, double v, const Prim* p, int k, double d_alpha, AGrads* g) {
  memset(g, 0, sizeof *g);
  KEval ev;
  eval_kernel(u, v, p, k, &ev);
  g->d_op = d_alpha * sharpen(ev.value, p->tau);
  if (ev.at_center) return;
  const int br = sharpen_branch(ev.value, p->tau);
  g->d_tau = d_alpha * p->o * sharpen_dtau(br, ev.value, p->tau);
  if (ev.exp_clamped) return;
  const double d_g = d_alpha * p->o * sharpen_slope(br, p->tau);
  const double d_q = d_g * (-0.5 * ev.value);
  const int lo = ev.lo, hi = ev.hi;
  const double slo = p->s[lo], shi = p->s[hi], eta = p->eta;
  g->d_eta = d_q * (ev.r1 * ev.r1 - ev.r2_sq * ev.inv_sbar_sq);
  const double d_r1 = d_q * eta * 2.0 * ev.r1;
  const double d_r2sq = d_q * (1.0 - eta) * ev.inv_sbar_sq;
  const double d_inv = d_q * (1.0 - eta) * ev.r2_sq;
  const double c = cos(ev.delta);
  g->ds[lo] += d_inv * (-(1.0 + c) / (slo * slo * slo));
  g->ds[hi] += d_inv * (-(1.0 - c) / (shi * shi * shi));
  const double d_c = d_inv * (0.5 / (slo * slo) - 0.5 / (shi * shi));
  const double d_delta = d_c * (-sin(ev.delta));
  double alo = p->th[lo], ahi = p->th[hi], theta = ev.theta;
  if (hi == 0) {
    alo -= TWO_PI;
    if (theta > p->th[k - 1]) theta -= TWO_PI;
  }
  const double gap = ahi - alo;
  const double d_tfd = d_delta * M_PI / gap;
  g->da[lo] += d_delta * M_PI * (theta - ahi) / (gap * gap);
  g->da[hi] += d_delta * (-M_PI) * (theta - alo) / (gap * gap);
  const double r2s = dmax(ev.r2_sq, 1e-24);
  double du = d_tfd * (-v / r2s);
  double dv = d_tfd * (u / r2s);
  du += d_r2sq * 2.0 * u;
  dv += d_r2sq * 2.0 * v;
  const double sa = ev.a > 0 ? 1 : (ev.a < 0 ? -1 : 0);
  const double sb = ev.b > 0 ? 1 : (ev.b < 0 ? -1 : 0);
  const double elx = slo * cos(p->th[lo]), ely = slo * sin(p->th[lo]);
  const double ehx = shi * cos(p->th[hi]), ehy = shi * sin(p->th[hi]);
  const double det = elx * ehy - ely * ehx;
#define MINV_X(wx, wy) ((ehy * (wx) - ehx * (wy)) / det)
#define MINV_Y(wx, wy) ((-ely * (wx) + elx * (wy)) / det)
  const double dab_du_x = MINV_X(1.0, 0.0), dab_du_y = MINV_Y(1.0, 0.0);
  const double dab_dv_x = MINV_X(0.0, 1.0), dab_dv_y = MINV_Y(0.0, 1.0);
  du += d_r1 * (sa * dab_du_x + sb * dab_du_y);
  dv += d_r1 * (sa * dab_dv_x + sb * dab_dv_y);
  const double ca = cos(p->th[lo]), sa_lo = sin(p->th[lo]);
  const double cb = cos(p->th[hi]), sb_hi = sin(p->th[hi]);
  g->ds[lo] += d_r1 * (-sa * ev.a / slo);
  g->ds[hi] += d_r1 * (-sb * ev.b / shi);
  const double tlo_wx = -slo * sa_lo, tlo_wy = slo * ca;
  const double thi_wx = -shi * sb_hi, thi_wy = shi * cb;
  const double na = -ev.a, nb = -ev.b;
  const double dtlo_x = na * MINV_X(tlo_wx, tlo_wy), dtlo_y = na * MINV_Y(tlo_wx, tlo_wy);
  const double dthi_x = nb * MINV_X(thi_wx, thi_wy), dthi_y = nb * MINV_Y(thi_wx, thi_wy);
#undef MINV_X
#undef MINV_Y
  g->da[lo] += d_r1 * (sa * dtlo_x + sb * dtlo_y);
  g->da[hi] += d_r1 * (sa * dthi_x + sb * dthi_y);
  g->d_u = du;
  g->d_v = dv;
}

typedef struct BCtx {
  const Scene* sc;
  const orc_camera* cam;
  const orc_options* opt;
  const double *dC, *dD, *dN, *dA;
  double* proj;
  GLayout L;
  double* part;   /* n x L.size, per-tile partials */
  char* in_tile;
  int* touched_list;
  int n_touched;
} BCtx;

static double* part_of(BCtx* b, int id) {
  if (!b->in_tile[id]) {
    b->in_tile[id] = 1;
    b->touched_list[b->n_touched++] = id;
    memset(b->part + (size_t)id * b->L.size, 0, sizeof(double) * b->L.size);
  }
  return b->part + (size_t)id * b->L.size;
}

/* grad.cpp:178-303 */
static void backward_pixel(BCtx* b, const RecVec* recs, int x, int y) {
  const orc_camera* cam = b->cam;
  const orc_options* opt = b->opt;
  const GLayout* L = &b->L;
  const int n = (int)recs->n;
  const size_t pix = (size_t)y * cam->width + x;
  double dC[3] = {0, 0, 0}, dN[3] = {0, 0, 0}, dD = 0, dA = 0;
  if (b->dC) for (int c = 0; c < 3; ++c) dC[c] = b->dC[3 * pix + c];
  if (b->dD) dD = b->dD[pix];
  if (b->dN) for (int c = 0; c < 3; ++c) dN[c] = b->dN[3 * pix + c];
  if (b->dA) dA = b->dA[pix];
  if (n == 0) return;
  const double px = x + 0.5, py = y + 0.5;
  const Ray ray = pixel_ray(cam, px, py);
  double* trans = (double*)malloc(sizeof(double) * (n + 1));
  double* cw = (double*)malloc(sizeof(double) * n);
  double* rgbs = (double*)malloc(sizeof(double) * 3 * n);
  int* clampeds = (int*)malloc(sizeof(int) * 3 * n);
  double* sgns = (double*)malloc(sizeof(double) * n);
  trans[0] = 1.0;
  for (int i = 0; i < n; ++i) trans[i + 1] = trans[i] * (1.0 - recs->v[i].alpha);
  double total = 0;
  for (int i = 0; i < n; ++i) {
    const Rec* r = &recs->v[i];
    const Prim* p = &b->sc->p[r->id];
    double rz[3];
    prim_col(p, 2, rz);
    sh_eval(b->sc, r->id, ray.d, opt->sh_degree, rgbs + 3 * i, clampeds + 3 * i);
    sgns[i] = dot3(ray.d, rz) < 0 ? 1.0 : -1.0;
    const double no[3] = {sgns[i] * rz[0], sgns[i] * rz[1], sgns[i] * rz[2]};
    cw[i] = dot3(dC, rgbs + 3 * i) + dD * r->depth + dot3(dN, no) + dA;
    total += trans[i] * r->alpha * cw[i];
  }
  total += trans[n] * dot3(dC, opt->background);
  double rest = total;
  double basis[16];
  sh_basis(ray.d, opt->sh_degree, basis);
  const int terms = active_terms(b->sc, opt->sh_degree);
  for (int i = 0; i < n; ++i) {
    const Rec* r = &recs->v[i];
    const Prim* p = &b->sc->p[r->id];
    const double t_i = trans[i];
    const double wb = t_i * r->alpha;
    rest -= wb * cw[i];
    const double dat = t_i * cw[i] - rest / (1.0 - r->alpha);
    double* pg = part_of(b, r->id);
    for (int ch = 0; ch < 3; ++ch) {
      if (clampeds[3 * i + ch]) continue;
      const double dc = wb * dC[ch];
      if (dc == 0) continue;
      for (int t = 0; t < terms; ++t) pg[L->sh + 3 * t + ch] += dc * basis[t];
    }
    double rx[3], ry[3], rz[3];
    prim_col(p, 0, rx); prim_col(p, 1, ry); prim_col(p, 2, rz);
    if (b->dN)
      for (int a = 0; a < 3; ++a) pg[L->rot + 3 * a + 2] += wb * sgns[i] * dN[a];
    const double rdz = dot3(ray.d, rz);
    if (dD != 0) {
      const double d_rt = wb * dD;
      for (int a = 0; a < 3; ++a) {
        const double h = ray.o[a] + r->depth * ray.d[a] - p->mu[a];
        pg[a] += d_rt * rz[a] / rdz;
        pg[L->rot + 3 * a + 2] += d_rt * (-h / rdz);
      }
    }
    const int alpha_clamped = r->alpha >= 1.0 - 1e-6 - 1e-12;
    if (alpha_clamped) {
    } else if (r->lowpass) {
      const double cv = fabs(rdz);
      const double dpw = px - b->proj[3 * r->id], dph = py - b->proj[3 * r->id + 1];
      pg[L->op] += dat * r->alpha / p->o;
      const double inv = 1.0 / (cv * cv * opt->lowpass_radius * opt->lowpass_radius);
      const double d_dpw = dat * r->alpha * (-dpw * inv);
      const double d_dph = dat * r->alpha * (-dph * inv);
      const double d_cos = dat * r->alpha * (dpw * dpw + dph * dph) * inv / cv;
      double J[6];
      projection_jacobian(cam, p->mu, J);
      for (int a = 0; a < 3; ++a) pg[a] += -(J[a] * d_dpw + J[3 + a] * d_dph);
      const double sg = rdz < 0 ? -1.0 : 1.0;
      for (int a = 0; a < 3; ++a) pg[L->rot + 3 * a + 2] += d_cos * sg * ray.d[a];
    } else {
      AGrads ag;
      backward_alpha(r->u, r->v, p, b->sc->k, dat, &ag);
      for (int j = 0; j < b->sc->k; ++j) {
        pg[L->sc + j] += ag.ds[j];
        pg[L->an + j] += ag.da[j];
      }
      pg[L->eta] += ag.d_eta;
      pg[L->tau] += ag.d_tau;
      pg[L->op] += ag.d_op;
      const double drx = dot3(ray.d, rx), dry = dot3(ray.d, ry);
      double h[3];
      for (int a = 0; a < 3; ++a) h[a] = ray.o[a] + r->depth * ray.d[a] - p->mu[a];
      for (int a = 0; a < 3; ++a) {
        const double du_dmu = rz[a] * (drx / rdz) - rx[a];
        const double dv_dmu = rz[a] * (dry / rdz) - ry[a];
        pg[a] += ag.d_u * du_dmu + ag.d_v * dv_dmu;
      }
      for (int a = 0; a < 3; ++a) pg[L->rot + 3 * a + 0] += ag.d_u * h[a];
      for (int a = 0; a < 3; ++a) pg[L->rot + 3 * a + 1] += ag.d_v * h[a];
      const double f = -(ag.d_u * drx + ag.d_v * dry) / rdz;
      for (int a = 0; a < 3; ++a) pg[L->rot + 3 * a + 2] += f * h[a];
    }
  }
  free(trans); free(cw); free(rgbs); free(clampeds); free(sgns);
}

/* grad.cpp:122-141 */
static void quat_rotation_backward(const double q[4], const double dR[9], double out[4]) {
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double qh[4] = {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
  const double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
  /* row-major matrices as in the comma initialisers of grad.cpp:129-132 */
  const double dw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
  const double dx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
  const double dy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
  const double dz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
  const double* Ms[4] = {dw, dx, dy, dz};
  double dqh[4];
  for (int m = 0; m < 4; ++m) {
    /* cwiseProduct(d_rot).sum() in column-major storage order */
    double acc = Ms[m][0] * dR[0];
    for (int idx = 1; idx < 9; ++idx) {
      const int r = idx % 3, c = idx / 3;
      acc = acc + Ms[m][3 * r + c] * dR[3 * r + c];
    }
    dqh[m] = 2.0 * acc;
  }
  const double d = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
  for (int m = 0; m < 4; ++m) out[m] = (dqh[m] - qh[m] * d) / n;
}

/* core.cpp:110-131 */
static void angle_activation_jacobian(const double* raw, int k, double* jac /* k x k row-major */) {
  const double residual = 1.0 / (k - 2);
  double dstep[16], cum[16], total = 0;
  for (int i = 0; i < k; ++i) {
    const double s = sigmoid(raw[i]);
    const int cl = s < 1e-9 || s > 1.0 - 1e-9;
    const double sc = s < 1e-9 ? 1e-9 : (1.0 - 1e-9 < s ? 1.0 - 1e-9 : s);
    dstep[i] = cl ? 0.0 : s * (1.0 - s);
    total += sc + residual;
    cum[i] = total;
  }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      const double ind = (j <= i) ? 1.0 : 0.0;
      jac[i * k + j] = TWO_PI / total * (ind - cum[i] / total) * dstep[j];
    }
  for (int j = 0; j < k; ++j) jac[(k - 1) * k + j] = 0.0;
}

/* grad.cpp:143-159; writes the raw gradient of primitive i into SoA grad_raw */
static void activation_backward(const Scene* sc, int i, const double* g, const GLayout* L, double* grad_raw) {
  const int n = sc->n, k = sc->k;
#define G(s) grad_raw[(size_t)(s) * n + i]
  for (int a = 0; a < 3; ++a) G(a) = g[a];
  double q[4] = {raw_at(sc, 3, i), raw_at(sc, 4, i), raw_at(sc, 5, i), raw_at(sc, 6, i)};
  double dq[4];
  quat_rotation_backward(q, g + L->rot, dq);
  for (int a = 0; a < 4; ++a) G(3 + a) = dq[a];
  for (int j = 0; j < k; ++j) G(7 + j) = g[L->sc + j] * exp(raw_at(sc, 7 + j, i));
  double ar[16], jac[256];
  for (int j = 0; j < k; ++j) ar[j] = raw_at(sc, 7 + k + j, i);
  angle_activation_jacobian(ar, k, jac);
  for (int c = 0; c < k; ++c) {
    double acc = jac[0 * k + c] * g[L->an + 0];
    for (int r = 1; r < k; ++r) acc = acc + jac[r * k + c] * g[L->an + r];
    G(7 + k + c) = acc;
  }
  const double eta = sigmoid(raw_at(sc, 7 + 2 * k, i));
  G(7 + 2 * k) = g[L->eta] * eta * (1.0 - eta);
  const double st = sigmoid(raw_at(sc, 8 + 2 * k, i));
  G(8 + 2 * k) = g[L->tau] * (TAU_HIGH - TAU_LOW) * st * (1.0 - st);
  const double o = sigmoid(raw_at(sc, 9 + 2 * k, i));
  G(9 + 2 * k) = g[L->op] * o * (1.0 - o);
  for (int t = 0; t < 3 * sc->terms; ++t) G(10 + 2 * k + t) = g[L->sh + t];
#undef G
}

/* grad.cpp:307-384, taking the replay from a fresh orc render */
int orc_backward(const double* raw, int n, int k, int terms, const orc_camera* cam, const orc_options* opt,
                 const double* d_color, const double* d_depth, const double* d_normal, const double* d_alpha,
                 double* grad_raw, double* d_center_world, double* screen_grad, int8_t* touched) {
  int64_t nrec = 0;
  int st = orc_render(raw, n, k, terms, cam, opt, NULL, NULL, NULL, NULL, 1, &nrec, NULL);
  if (st) return st;
  Scene sc;
  st = build_scene(&sc, raw, n, k, terms);
  if (st) return st;
  BCtx b;
  memset(&b, 0, sizeof b);
  b.sc = &sc; b.cam = cam; b.opt = opt;
  b.dC = d_color; b.dD = d_depth; b.dN = d_normal; b.dA = d_alpha;
  b.L = glayout(k, terms);
  b.proj = (double*)calloc((size_t)3 * (n + 1), sizeof(double));
  char* has_proj = (char*)calloc((size_t)n + 1, 1);
  project_centers(&sc, cam, b.proj, has_proj);
  b.part = (double*)calloc((size_t)(n + 1) * b.L.size, sizeof(double));
  b.in_tile = (char*)calloc((size_t)n + 1, 1);
  b.touched_list = (int*)calloc((size_t)n + 1, sizeof(int));
  double* reduced = (double*)calloc((size_t)(n + 1) * b.L.size, sizeof(double));
  char* tch = (char*)calloc((size_t)n + 1, 1);
  if (!b.part || !reduced) return fail(ST_OOM, "out of memory");
  const int tiles_x = (cam->width + TILE - 1) / TILE, tiles_y = (cam->height + TILE - 1) / TILE;
  for (int t = 0; t < tiles_x * tiles_y; ++t) {
    const int tx = t % tiles_x, ty = t / tiles_x;
    const int x1 = cam->width < (tx + 1) * TILE ? cam->width : (tx + 1) * TILE;
    const int y1 = cam->height < (ty + 1) * TILE ? cam->height : (ty + 1) * TILE;
    b.n_touched = 0;
    for (int y = ty * TILE; y < y1; ++y)
      for (int x = tx * TILE; x < x1; ++x) backward_pixel(&b, &g_replay_px[(size_t)y * cam->width + x], x, y);
    for (int j = 0; j < b.n_touched; ++j) {
      const int id = b.touched_list[j];
      double* dst = reduced + (size_t)id * b.L.size;
      const double* src = b.part + (size_t)id * b.L.size;
      for (int e = 0; e < b.L.size; ++e) dst[e] += src[e];
      tch[id] = 1;
      b.in_tile[id] = 0;
    }
  }
  for (int i = 0; i < n; ++i) {
    const double* g = reduced + (size_t)i * b.L.size;
    activation_backward(&sc, i, g, &b.L, grad_raw);
    for (int a = 0; a < 3; ++a) d_center_world[3 * i + a] = g[a];
    screen_grad[i] = 0.0;
    touched[i] = tch[i];
    if (tch[i] && has_proj[i]) {
      double J[6];
      projection_jacobian(cam, sc.p[i].mu, J);
      const double jx = J[0] * g[0] + J[1] * g[1] + J[2] * g[2];
      const double jy = J[3] * g[0] + J[4] * g[1] + J[5] * g[2];
      screen_grad[i] = sqrt(jx * jx + jy * jy);
    }
  }
  free(b.proj); free(has_proj); free(b.part); free(b.in_tile); free(b.touched_list);
  free(reduced); free(tch); free(sc.p);
  return ST_OK;
}

/* ------------------------------------------------------------------ */
/* loss (optimize.cpp:171-204, dssim_weight = 0) and Adam (:226-307)    */
/* ------------------------------------------------------------------ */
int orc_loss_l1(const double* r, const double* t, int w, int h, double* value, double* d_color) {
  const size_t n = (size_t)w * h * 3;
  const double inv_n = 1.0 / (double)n;
  double l1 = 0;
  for (size_t i = 0; i < n; ++i) {
    const double d = r[i] - t[i];
    l1 += fabs(d);
    d_color[i] = (1.0 - 0.0) * inv_n * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0));
  }
  l1 *= inv_n;
  *value = (1.0 - 0.0) * l1;
  return ST_OK;
}

/* lrs = {lr_drk, lr_position, lr_rotation, lr_opacity, lr_sh} */
int orc_adam_step(double* params, const double* grads, double* m, double* v, int n, int k, int terms,
                  int64_t* step, const double* lrs, int steps_total, double extent, int freeze_eta_tau,
                  int freeze_angles) {
  *step += 1;
  const double bc1 = 1.0 - pow(0.9, (double)*step);
  const double bc2 = 1.0 - pow(0.999, (double)*step);
  const double t = steps_total > 0 ? dmin(1.0, (double)*step / steps_total) : 1.0;
  const double decay = pow(1e-2, t);
  const double lr_center = lrs[1] * extent * decay, lr_quat = lrs[2], lr_drk = lrs[0] * decay;
  const double lr_op = lrs[3], lr_sh = lrs[4], lr_sh_rest = lr_sh / 20.0;
  const int S = 3 + 4 + 2 * k + 3 + 3 * terms;
  for (int s = 0; s < S; ++s) {
    double lr;
    if (s < 3) lr = lr_center;
    else if (s < 7) lr = lr_quat;
    else if (s < 7 + k) lr = lr_drk;
    else if (s < 7 + 2 * k) lr = freeze_angles ? 0 : lr_drk;
    else if (s < 9 + 2 * k) lr = freeze_eta_tau ? 0 : lr_drk;
    else if (s == 9 + 2 * k) lr = lr_op;
    else lr = (s - (10 + 2 * k)) < 3 ? lr_sh : lr_sh_rest;
    for (int i = 0; i < n; ++i) {
      const size_t j = (size_t)s * n + i;
      const double g = grads[j];
      m[j] = 0.9 * m[j] + (1.0 - 0.9) * g;
      v[j] = 0.999 * v[j] + (1.0 - 0.999) * g * g;
      const double mh = m[j] / bc1, vh = v[j] / bc2;
      params[j] -= lr * mh / (sqrt(vh) + 1e-15);
    }
  }
  return ST_OK;
}
