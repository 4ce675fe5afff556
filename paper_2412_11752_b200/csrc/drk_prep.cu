// K0 activation, K1 per-primitive preprocess (support polygon, near clip,
// projection, convex hull, tile bbox), K2 per-row tile intervals and K3 pair
// emission with NearestDepth keys.  Restates reference core.cpp:133-146
// (activate) and raster.cpp:12-265 (bin_primitives) for sm_100a.
//
// Layout: one thread per primitive for K0/K1/K2 (SoA fp64 loads), one thread
// per (primitive, tile row) for K3.  The hull of every primitive goes to a
// bump-allocated pool; rows are addressed through an exclusive scan of the
// per-primitive row counts so that pairs come out primitive-major (ascending
// prim id inside every tile), which the stable radix sort turns into the
// reference's (key, prim_id) order (raster.cpp:260-263).
#include <cfloat>

#include "drk_internal.h"

namespace drk {

// ---------------------------------------------------------------------------
// K0: activation (core.cpp:89-146, geometry.cpp:21-30)
// ---------------------------------------------------------------------------
__global__ void k_activate(const float* __restrict__ raw, int n, int K, int terms, double* mu, double* rot,
                           double* s, double* th, double* eta, double* tau, double* o, float* sh,
                           unsigned long long* counters, int i0, int i1) {
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const int S = 3 + 4 + 2 * K + 3 + 3 * terms;
  bool finite = true;
  for (int j = 0; j < S; ++j) finite &= isfinite(raw[(size_t)j * n + i]);
  if (!finite) atomicAdd(&counters[C_ERR_NONFINITE], 1ull);
#define RAW(j) ((double)raw[(size_t)(j)*n + i])
  for (int a = 0; a < 3; ++a) mu[3 * i + a] = RAW(a);
  const double q0 = RAW(3), q1 = RAW(4), q2 = RAW(5), q3 = RAW(6);
  const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  if (qn < 1e-12) atomicAdd(&counters[C_ERR_DEGEN_QUAT], 1ull);
  const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
  double* R = rot + 9 * (size_t)i;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
  double* si = s + (size_t)K * i;
  double* ti = th + (size_t)K * i;
  for (int j = 0; j < K; ++j) si[j] = exp(RAW(7 + j));
  // angle_activation (core.cpp:89-108)
  const double residual = 1.0 / (K - 2);
  double total = 0;
  for (int j = 0; j < K; ++j) {
    double sg = sigmoid(RAW(7 + K + j));
    sg = sg < 1e-9 ? 1e-9 : (1.0 - 1e-9 < sg ? 1.0 - 1e-9 : sg);
    total += sg + residual;
    ti[j] = total;
  }
  const double scale = kTwoPi / total;
  for (int j = 0; j < K; ++j) ti[j] = ti[j] * scale;
  ti[K - 1] = kTwoPi;
  eta[i] = sigmoid(RAW(7 + 2 * K));
  tau[i] = kTauLow + (kTauHigh - kTauLow) * sigmoid(RAW(8 + 2 * K));
  o[i] = sigmoid(RAW(9 + 2 * K));
  for (int j = 0; j < 3 * terms; ++j) sh[(size_t)3 * terms * i + j] = raw[(size_t)(10 + 2 * K + j) * n + i];
#undef RAW
}

// Endpoints and bracket determinants (types.hpp:93-95, core.cpp:188-190) and
// the fp32 fast-path constants of ShapeView.
__global__ void k_shape(int i0, int i1, int K, const double* s, const double* th, double* ex, double* ey, double* det,
                        float* thf, float* invdetf, float* piogf, float* hf, const double* tau, const double* o,
                        float* psif) {
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  {
    // sharpen (core.cpp:229-237) in point-slope form
    const double t = tau[i];
    const double g1 = (1.0 + t) / 4.0, g2 = (3.0 - t) / 4.0;
    const double A0 = (1.0 - t) / (1.0 + t), A1 = (1.0 + t) / (1.0 - t);
    const double P1 = A0 * g1, P2 = ((1.0 + t) * g2 - t) / (1.0 - t);
    float* q = psif + 12 * (size_t)i;
    q[0] = (float)g1;
    q[1] = (float)g2;
    q[2] = (float)A0;
    q[3] = (float)A1;
    q[4] = (float)A0;
    q[5] = (float)P1;
    q[6] = (float)P2;
    q[7] = (float)o[i];
    // q[8] = f_vis^2 = -2 ln Psi^-1(alpha_min / o) (core.cpp:309-310) depends on the
    // render options: written per view by K1 (prep_body)
    q[8] = 0.f;
    q[9] = q[10] = q[11] = 0.f;
  }
  const size_t b = (size_t)K * i;
  for (int j = 0; j < K; ++j) {
    ex[b + j] = s[b + j] * cos(th[b + j]);
    ey[b + j] = s[b + j] * sin(th[b + j]);
  }
  for (int j = 0; j < K; ++j) {
    const int h = (j + 1) % K;
    det[b + j] = ex[b + j] * ey[b + h] - ey[b + j] * ex[b + h];
    const double gap = j + 1 < K ? th[b + h] - th[b + j] : th[b] - (th[b + K - 1] - kTwoPi);
    thf[b + j] = (float)th[b + j];
    invdetf[b + j] = (float)(1.0 / det[b + j]);
    piogf[b + j] = (float)(kPi / gap);
    hf[b + j] = (float)(1.0 / (s[b + j] * s[b + j]));
  }
}

// ---------------------------------------------------------------------------
// K1: support polygon -> clip -> project -> hull -> bbox  (raster.cpp:131-231)
// ---------------------------------------------------------------------------
struct PolyParams {
  double alo, gap, slo, shi, elx, ely, ehx, ehy, det, eta, support_c;
};
struct W2 {
  double rho1, inv;
};

// raster.cpp:158-168
__device__ __forceinline__ W2 weight_at(const PolyParams& p, double a) {
  const double delta = (a - p.alo) * kPi / p.gap;
  const double c = cos(delta);
  W2 w;
  w.inv = (1.0 + c) / (2.0 * p.slo * p.slo) + (1.0 - c) / (2.0 * p.shi * p.shi);
  const double dx = cos(a), dy = sin(a);
  const double ca = (p.ehy * dx - p.ehx * dy) / p.det;
  const double cb = (-p.ely * dx + p.elx * dy) / p.det;
  w.rho1 = fabs(ca) + fabs(cb);
  return w;
}
// raster.cpp:170-173
__device__ __forceinline__ double radius_true(const PolyParams& p, W2 w) {
  const double total = p.eta * w.rho1 * w.rho1 + (1.0 - p.eta) * w.inv;
  return sqrt(p.support_c / dmax(total, 1e-12));
}

// Streaming Sutherland-Hodgman against z >= kNearClip (raster.cpp:15-30):
// emits exactly the reference's output sequence, projected to pixels
// (raster.cpp:214-215).
struct Clipper {
  double first[3], prev[3];
  int count;
  double2* out;
  int cap, n;
  const CamD* cam;
  __device__ void push(const double q[3]) {
    if (n < cap) out[n] = make_double2(cam->fx * q[0] / q[2] + cam->cx, cam->fy * q[1] / q[2] + cam->cy);
    ++n;
  }
  __device__ void edge(const double a[3], const double b[3]) {
    const bool a_in = a[2] >= kNearClip, b_in = b[2] >= kNearClip;
    if (a_in) push(a);
    if (a_in != b_in) {
      const double t = (kNearClip - a[2]) / (b[2] - a[2]);
      const double q[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]), a[2] + t * (b[2] - a[2])};
      push(q);
    }
  }
  __device__ void feed(const double b[3]) {
    if (count == 0) {
      first[0] = b[0]; first[1] = b[1]; first[2] = b[2];
    } else {
      edge(prev, b);
    }
    prev[0] = b[0]; prev[1] = b[1]; prev[2] = b[2];
    ++count;
  }
  __device__ void finish() {
    if (count > 0) edge(prev, first);
  }
};

__device__ __forceinline__ bool lessp(double2 a, double2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

__device__ void heap_sort(double2* a, int n) {
  auto sift = [&](int root, int end) {
    while (true) {
      int child = 2 * root + 1;
      if (child >= end) break;
      if (child + 1 < end && lessp(a[child], a[child + 1])) ++child;
      if (lessp(a[root], a[child])) {
        const double2 t = a[root];
        a[root] = a[child];
        a[child] = t;
        root = child;
      } else {
        break;
      }
    }
  };
  for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
  for (int end = n - 1; end > 0; --end) {
    const double2 t = a[0];
    a[0] = a[end];
    a[end] = t;
    sift(0, end);
  }
}

__device__ __forceinline__ double cross2(double2 o, double2 a, double2 b) {
  return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x);
}

// Andrew monotone chain (raster.cpp:33-58); pts sorted + deduplicated in
// place, hull written to h (capacity n + 2).  Returns the hull size.
__device__ int convex_hull(double2* pts, int n, double2* h) {
  heap_sort(pts, n);
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || !(pts[i].x == pts[m - 1].x && pts[i].y == pts[m - 1].y)) pts[m++] = pts[i];
  n = m;
  if (n <= 2) {
    for (int i = 0; i < n; ++i) h[i] = pts[i];
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

// Builds the projected support polygon of primitive i into pts (capacity cap)
// and its hull into h.  Returns the hull size, 0 when fully behind, or -1 on
// polygon overflow (caller retries with a larger buffer).
__device__ int build_hull(const Activated& A, int i, const CamD& cam, double factor, double2* pts, int cap,
                          double2* h) {
  const int K = A.K;
  const double* s = A.s + (size_t)K * i;
  const double* th = A.th + (size_t)K * i;
  const double* R = A.rot + 9 * (size_t)i;
  const double mu[3] = {A.mu[3 * i], A.mu[3 * i + 1], A.mu[3 * i + 2]};
  const double rx[3] = {R[0], R[3], R[6]}, ry[3] = {R[1], R[4], R[7]};
  Clipper clip;
  clip.count = 0;
  clip.out = pts;
  clip.cap = cap;
  clip.n = 0;
  clip.cam = &cam;
  PolyParams p;
  p.eta = A.eta[i];
  p.support_c = factor * factor;
  struct Frame {
    double a0, a1;
    W2 w0, w1;
    int depth;
  };
  Frame stack[12];
  for (int k = 0; k < K; ++k) {
    const int hi = (k + 1) % K;
    p.alo = k + 1 < K ? th[k] : th[k] - 2.0 * kPi;
    const double ahi = k + 1 < K ? th[hi] : th[0];
    p.gap = ahi - p.alo;
    p.slo = s[k];
    p.shi = s[hi];
    p.elx = A.ex[(size_t)K * i + k];
    p.ely = A.ey[(size_t)K * i + k];
    p.ehx = A.ex[(size_t)K * i + hi];
    p.ehy = A.ey[(size_t)K * i + hi];
    p.det = A.det[(size_t)K * i + k];
    const int coarse_i = (int)ceil(p.gap / (kPi / 8.0));
    const int coarse = coarse_i > 1 ? coarse_i : 1;
    W2 prev = weight_at(p, p.alo);
    for (int j = 0; j < coarse; ++j) {
      const double a0 = p.alo + p.gap * j / coarse;
      const double a1 = p.alo + p.gap * (j + 1) / coarse;
      const W2 next = weight_at(p, a1);
      // iterative depth-first emit (raster.cpp:178-198)
      int sp = 0;
      stack[sp++] = {a0, a1, prev, next, 0};
      while (sp > 0) {
        const Frame f = stack[--sp];
        const double rho1_min = dmin(f.w0.rho1, f.w1.rho1);
        const double inv_min = dmin(f.w0.inv, f.w1.inv);
        const double w_lb = p.eta * rho1_min * rho1_min + (1.0 - p.eta) * inv_min;
        const double bound = sqrt(p.support_c / dmax(w_lb, 1e-12)) / cos(0.5 * (f.a1 - f.a0));
        if (f.depth < 9 && f.a1 - f.a0 > 2e-3 &&
            bound > 1.25 * dmin(radius_true(p, f.w0), radius_true(p, f.w1))) {
          const double mid = 0.5 * (f.a0 + f.a1);
          const W2 wm = weight_at(p, mid);
          stack[sp++] = {mid, f.a1, wm, f.w1, f.depth + 1};  // right half after
          stack[sp++] = {f.a0, mid, f.w0, wm, f.depth + 1};  // left half first
          continue;
        }
        const double as[2] = {f.a0, f.a1};
        for (int e = 0; e < 2; ++e) {
          const double ca = cos(as[e]), sa = sin(as[e]);
          double w[3], pc[3];
          for (int a = 0; a < 3; ++a) w[a] = mu[a] + bound * (ca * rx[a] + sa * ry[a]);
          to_camera(cam, w, pc);
          clip.feed(pc);
        }
      }
      prev = next;
    }
  }
  clip.finish();
  if (clip.n > cap) return -1;
  if (clip.n == 0) return 0;
  return convex_hull(pts, clip.n, h);
}

constexpr int kPolyCap = 256;

// K1.  pass == 0: all primitives with local buffers; pass == 1: the overflow
// list with large per-thread global scratch.
template <int pass>
__device__ __forceinline__ void prep_body(Activated A, CamD cam, OptD opt, Geo* geo, int4* bbox, int2* hullref,
                                          double2* pool, long long pool_cap, int* rowcnt,
                                          unsigned long long* counters, const int* list, int list_n,
                                          double2* scratch, int scratch_cap, int* overflow) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int i;
  if (pass == 0) {
    if (t >= A.n) return;
    i = t;
  } else {
    if (t >= list_n) return;
    i = list[t];
  }
  const int K = A.K;
  if (pass == 0) {
    // per-view geometry record
    Geo g;
    const double* R = A.rot + 9 * (size_t)i;
    for (int a = 0; a < 3; ++a) {
      g.mu[a] = A.mu[3 * i + a];
      g.rx[a] = R[3 * a];
      g.ry[a] = R[3 * a + 1];
      g.rz[a] = R[3 * a + 2];
    }
    const double m0 = g.mu[0] - cam.o[0], m1 = g.mu[1] - cam.o[1], m2 = g.mu[2] - cam.o[2];
    g.num = m0 * g.rz[0] + m1 * g.rz[1] + m2 * g.rz[2];
    double pr[3];
    g.has_proj = try_project(cam, g.mu, pr) ? 1 : 0;
    g.ppx = g.has_proj ? pr[0] : 0.0;
    g.ppy = g.has_proj ? pr[1] : 0.0;
    g.projz = g.has_proj ? pr[2] : __longlong_as_double(0x7ff0000000000000ll);
    double f, fv;
    const double o = A.o[i];
    g.visible = binning_radius_factor(o, A.tau[i], opt.alpha_min, &f, &fv) ? 1 : 0;
    double smax = 0;
    for (int j = 0; j < K; ++j) smax = dmax(smax, A.s[(size_t)K * i + j]);
    g.r2max = g.visible ? (smax * fv) * (smax * fv) * (1.0 + 1e-9) : 0.0;
    const_cast<float*>(A.psif)[12 * (size_t)i + 8] = g.visible ? (float)(fv * fv) : __int_as_float(0x7f800000);
    g.fvis2 = A.psif[12 * (size_t)i + 8];
    g.pad_ = 0;
    g.dp2max = g.visible ? 2.0 * opt.lowpass_radius * opt.lowpass_radius * log(o / opt.alpha_min) * (1.0 + 1e-9) : 0.0;
    geo[i] = g;
    rowcnt[i] = 0;
    bbox[i] = make_int4(1, 0, 1, 0);
    hullref[i] = make_int2(0, 0);
    if (!g.visible) return;
  }
  double f, fv;
  binning_radius_factor(A.o[i], A.tau[i], opt.alpha_min, &f, &fv);
  double2 pts_local[pass == 0 ? kPolyCap : 1];
  double2 hull_local[pass == 0 ? kPolyCap + 2 : 1];
  double2* pts = pts_local;
  double2* hh = hull_local;
  int cap = kPolyCap;
  if (pass == 1) {
    pts = scratch + (size_t)t * 2 * (scratch_cap + 2);
    hh = pts + scratch_cap + 2;
    cap = scratch_cap;
  }
  const int hn = build_hull(A, i, cam, f, pts, cap, hh);
  if (hn < 0) {
    if (pass == 0) {
      const unsigned long long slot = atomicAdd(&counters[C_POLY_OVERFLOW], 1ull);
      overflow[slot] = i;
    } else {
      atomicAdd(&counters[C_POLY_FAIL], 1ull);  // polygon larger than the big scratch
    }
    return;
  }
  if (hn == 0) return;
  double hx0 = hh[0].x, hx1 = hx0, hy0 = hh[0].y, hy1 = hy0;
  for (int j = 0; j < hn; ++j) {
    hx0 = dmin(hx0, hh[j].x);
    hx1 = dmax(hx1, hh[j].x);
    hy0 = dmin(hy0, hh[j].y);
    hy1 = dmax(hy1, hh[j].y);
  }
  const double lp = opt.lp_pad;
  int tx0 = x86_int(floor((hx0 - lp) / kTile));
  tx0 = tx0 > 0 ? tx0 : 0;
  int tx1 = x86_int(floor((hx1 + lp) / kTile));
  tx1 = tx1 < cam.tiles_x - 1 ? tx1 : cam.tiles_x - 1;
  int ty0 = x86_int(floor((hy0 - lp) / kTile));
  ty0 = ty0 > 0 ? ty0 : 0;
  int ty1 = x86_int(floor((hy1 + lp) / kTile));
  ty1 = ty1 < cam.tiles_y - 1 ? ty1 : cam.tiles_y - 1;
  if (tx1 < tx0 || ty1 < ty0) return;
  const long long off = (long long)atomicAdd(&counters[C_HULL_POOL], (unsigned long long)hn);
  if (off + hn > pool_cap) return;  // host detects via the cursor and retries with a larger pool
  for (int j = 0; j < hn; ++j) pool[off + j] = hh[j];
  hullref[i] = make_int2((int)off, hn);
  bbox[i] = make_int4(tx0, tx1, ty0, ty1);
  rowcnt[i] = ty1 - ty0 + 1;
  atomicAdd(&counters[C_VISIBLE], 1ull);
}

// ---------------------------------------------------------------------------
// K1 warp-per-primitive variant (pass 0 of every primitive).  The adaptive
// wedge tree (raster.cpp:178-207) is expanded breadth-first by the 32 lanes:
// a leaf's two vertices are pure functions of its endpoint angles and
// weights, so the vertex SET is the reference's whatever the traversal
// order.  Without near clipping (every vertex at z >= 1e-6, the common case)
// the polygon order is irrelevant to the hull: the projected vertices are
// sorted (x, y) by a warp bitonic sort in shared memory and lane 0 runs the
// reference's monotone chain, so the hull is bit-identical.  Primitives that
// need the near clip (vertex order matters for Sutherland-Hodgman) or exceed
// the per-warp buffers go to the serial k_prep1 path through the overflow list.
// ---------------------------------------------------------------------------
namespace {
#ifndef DRK_PREP_WARPS
#define DRK_PREP_WARPS 4  // measured: 4 warps per CTA -3% K1 time vs 8; stack 96 best of 48..160
#endif
#ifndef DRK_PREP_STACK
#define DRK_PREP_STACK 96
#endif
constexpr int kPW = DRK_PREP_WARPS;       // warps per block
constexpr int kWStack = DRK_PREP_STACK;   // wedge work items per warp
constexpr int kWVerts = 256;    // projected vertices per warp
struct WItem {
  double a0, a1, r0, i0, r1, i1, c0, s0, c1, s1;  // endpoint angles, weights, cos / sin
  int depth, k;
};
struct BrP {
  double alo, gap, slo, shi, elx, ely, ehx, ehy, det;
  int coarse, first;
};
struct WarpScratch {
  WItem stack[kWStack];
  double2 verts[kWVerts + 8];
  BrP br[kMaxK];
};
// build mode of the vertex cache: the leaves' world-space vertices beside
struct WarpScratchB {
  WarpScratch w;
  double world[3 * kWVerts];
};
__device__ __forceinline__ PolyParams poly_params(const BrP& b, double eta, double support_c) {
  PolyParams p;
  p.alo = b.alo;
  p.gap = b.gap;
  p.slo = b.slo;
  p.shi = b.shi;
  p.elx = b.elx;
  p.ely = b.ely;
  p.ehx = b.ehx;
  p.ehy = b.ehy;
  p.det = b.det;
  p.eta = eta;
  p.support_c = support_c;
  return p;
}
__device__ __forceinline__ bool lessp2(double2 a, double2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// One monotone chain of raster.cpp:46-56 over pts in forward (dir = 1) or
// reverse order into h; the two top stack entries live in registers.
__device__ int mono_chain(const double2* pts, int n, bool reverse, double2* h) {
  int k = 0;
  double2 a = make_double2(0, 0), b = a;  // h[k-2], h[k-1]
  for (int t = 0; t < n; ++t) {
    const double2 pt = pts[reverse ? n - 1 - t : t];
    while (k >= 2 && cross2(a, b, pt) <= 0) {
      --k;
      b = a;
      if (k >= 2) a = h[k - 2];
    }
    h[k++] = pt;
    a = b;
    b = pt;
  }
  return k;
}
}  // namespace

static size_t prep_warp_smem(int mode) {
  return (size_t)kPW * (mode == 1 ? sizeof(WarpScratchB) : sizeof(WarpScratch));
}

// weight_at (raster.cpp:158-168) that also returns cos(a), sin(a) for the
// wedge vertices at a (raster.cpp:199-201 evaluates the same cos/sin).
__device__ __forceinline__ W2 weight_cs(const PolyParams& p, double a, double* ca, double* sa) {
  const double delta = (a - p.alo) * kPi / p.gap;
  const double c = cos(delta);
  W2 w;
  w.inv = (1.0 + c) / (2.0 * p.slo * p.slo) + (1.0 - c) / (2.0 * p.shi * p.shi);
  double dx, dy;
  sincos(a, &dy, &dx);
  *ca = dx;
  *sa = dy;
  const double cva = (p.ehy * dx - p.ehx * dy) / p.det;
  const double cvb = (-p.ely * dx + p.elx * dy) / p.det;
  w.rho1 = fabs(cva) + fabs(cvb);
  return w;
}

// Phase A: vertices -> sorted unique points in the point pool.  ptsref[i] =
// (offset, count) of the sorted points; the pool slot holds 3 count entries
// (points, lower chain, upper chain) for k_prep_hull.
// MODE 0: plain.  Vertex cache (camera-independent leaves of the wedge tree, for
// several views of one activation): MODE 1 builds it (the tree runs to the end
// even when a vertex is near-clipped in this view, and its world-space
// vertices go to vpool; vref[i] = (offset, count), count -1: the tree overflows
// the warp buffers, -2: not cached), MODE 2 projects the cached vertices
// instead of expanding the tree (uncached primitives expand it as in MODE 0).
// The vertex set, hence the hull, is the same bits in every mode.
template <int MODE>
__global__ void __launch_bounds__(kPW * 32) k_prep_warp(Activated A, CamD cam, OptD opt, Geo* geo, int4* bbox,
                                                         int2* hullref, double2* pts_pool, long long pts_cap,
                                                         int2* ptsref, int* rowcnt, unsigned long long* counters,
                                                         int* overflow, float4* frame32, int i0, int i1,
                                                         double* vpool, long long vcap, int2* vref,
                                                         unsigned long long* vcursor) {
  extern __shared__ double4 prep_dyn[];
  const unsigned FULL = 0xffffffffu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = i0 + blockIdx.x * kPW + warp;
  if (i >= i1) return;  // warp-uniform
  WarpScratch& W = MODE == 1 ? reinterpret_cast<WarpScratchB*>(prep_dyn)[warp].w
                             : reinterpret_cast<WarpScratch*>(prep_dyn)[warp];
  double* Wworld = MODE == 1 ? reinterpret_cast<WarpScratchB*>(prep_dyn)[warp].world : nullptr;
  const int K = A.K;
  double f = 0, fv = 0;
  const double o = A.o[i];
  const bool visible = binning_radius_factor(o, A.tau[i], opt.alpha_min, &f, &fv);
  if (lane == 0) {
    // per-view geometry record (as prep_body pass 0)
    Geo g;
    const double* R = A.rot + 9 * (size_t)i;
    for (int a = 0; a < 3; ++a) {
      g.mu[a] = A.mu[3 * i + a];
      g.rx[a] = R[3 * a];
      g.ry[a] = R[3 * a + 1];
      g.rz[a] = R[3 * a + 2];
    }
    const double m0 = g.mu[0] - cam.o[0], m1 = g.mu[1] - cam.o[1], m2 = g.mu[2] - cam.o[2];
    g.num = m0 * g.rz[0] + m1 * g.rz[1] + m2 * g.rz[2];
    double pr[3];
    g.has_proj = try_project(cam, g.mu, pr) ? 1 : 0;
    g.ppx = g.has_proj ? pr[0] : 0.0;
    g.ppy = g.has_proj ? pr[1] : 0.0;
    g.projz = g.has_proj ? pr[2] : __longlong_as_double(0x7ff0000000000000ll);
    g.visible = visible ? 1 : 0;
    double smax = 0;
    for (int j = 0; j < K; ++j) smax = dmax(smax, A.s[(size_t)K * i + j]);
    g.r2max = visible ? (smax * fv) * (smax * fv) * (1.0 + 1e-9) : 0.0;
    const_cast<float*>(A.psif)[12 * (size_t)i + 8] = visible ? (float)(fv * fv) : __int_as_float(0x7f800000);
    g.fvis2 = visible ? (float)(fv * fv) : __int_as_float(0x7f800000);
    g.pad_ = 0;
    g.dp2max = visible ? 2.0 * opt.lowpass_radius * opt.lowpass_radius * log(o / opt.alpha_min) * (1.0 + 1e-9) : 0.0;
    geo[i] = g;
    if (frame32) {
      const double a0 = cam.o[0] - g.mu[0], a1 = cam.o[1] - g.mu[1], a2 = cam.o[2] - g.mu[2];
      frame32[3 * (size_t)i] = make_float4((float)g.rx[0], (float)g.rx[1], (float)g.rx[2], (float)a0);
      frame32[3 * (size_t)i + 1] = make_float4((float)g.ry[0], (float)g.ry[1], (float)g.ry[2], (float)a1);
      frame32[3 * (size_t)i + 2] = make_float4((float)g.rz[0], (float)g.rz[1], (float)g.rz[2], (float)a2);
    }
    rowcnt[i] = 0;
    bbox[i] = make_int4(1, 0, 1, 0);
    hullref[i] = make_int2(0, 0);
    ptsref[i] = make_int2(0, 0);
    if (MODE == 1) vref[i] = make_int2(0, 0);
  }
  if (!visible) return;
  bool fail = false;
  int nv = 0;
  bool cached = false;
  if (MODE == 2) {
    const int2 vr = vref[i];
    if (vr.y == -1) {
      fail = true;
      cached = true;
    } else if (vr.y >= 0) {
      // project the cached world-space vertices (the leaves' order)
      cached = true;
      nv = vr.y;
      bool clip = false;
      for (int t = lane; t < nv; t += 32) {
        const double* wv = vpool + 3 * ((size_t)vr.x + t);
        const double w[3] = {wv[0], wv[1], wv[2]};
        double pc[3];
        to_camera(cam, w, pc);
        clip |= !(pc[2] >= kNearClip);
        W.verts[t] = make_double2(cam.fx * pc[0] / pc[2] + cam.cx, cam.fy * pc[1] / pc[2] + cam.cy);
      }
      if (__any_sync(FULL, clip)) fail = true;
      __syncwarp();
    }
  }
  if (!cached) {
    const double eta = A.eta[i];
    const double support_c = f * f;
    const double* s = A.s + (size_t)K * i;
    const double* th = A.th + (size_t)K * i;
    // bracket parameters (raster.cpp:146-153) and coarse wedge counts (:202)
    int coarse = 0;
    BrP b;
    if (lane < K) {
      const int k = lane, hi = (k + 1) % K;
      b.alo = k + 1 < K ? th[k] : th[k] - 2.0 * kPi;
      const double ahi = k + 1 < K ? th[hi] : th[0];
      b.gap = ahi - b.alo;
      b.slo = s[k];
      b.shi = s[hi];
      b.elx = A.ex[(size_t)K * i + k];
      b.ely = A.ey[(size_t)K * i + k];
      b.ehx = A.ex[(size_t)K * i + hi];
      b.ehy = A.ey[(size_t)K * i + hi];
      b.det = A.det[(size_t)K * i + k];
      const int ci = (int)ceil(b.gap / (kPi / 8.0));
      coarse = ci > 1 ? ci : 1;
      b.coarse = coarse;
    }
    int incl = coarse;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += v;
    }
    if (lane < K) {
      b.first = incl - coarse;
      W.br[lane] = b;
    }
    const int total = (int)__reduce_add_sync(FULL, (unsigned)coarse);
    __syncwarp();
    fail = total > kWStack - 16;
    // coarse wedges with their endpoint weights (and cos / sin of the endpoints)
    if (!fail) {
      for (int idx = lane; idx < total; idx += 32) {
        int k = 0;
        while (k + 1 < K && W.br[k + 1].first <= idx) ++k;
        const BrP& bk = W.br[k];
        const int j = idx - bk.first;
        const PolyParams p = poly_params(bk, eta, support_c);
        const double a0 = bk.alo + bk.gap * j / bk.coarse;
        const double a1 = bk.alo + bk.gap * (j + 1) / bk.coarse;
        WItem it;
        const W2 w0 = weight_cs(p, a0, &it.c0, &it.s0), w1 = weight_cs(p, a1, &it.c1, &it.s1);
        it.a0 = a0;
        it.a1 = a1;
        it.r0 = w0.rho1;
        it.i0 = w0.inv;
        it.r1 = w1.rho1;
        it.i1 = w1.inv;
        it.depth = 0;
        it.k = k;
        W.stack[idx] = it;
      }
    }
    __syncwarp();
    int sp = fail ? 0 : total;
    bool clip_any = false;
    const double mu[3] = {A.mu[3 * i], A.mu[3 * i + 1], A.mu[3 * i + 2]};
    const double* R = A.rot + 9 * (size_t)i;
    const double rx[3] = {R[0], R[3], R[6]}, ry[3] = {R[1], R[4], R[7]};
    while (sp > 0 && !fail) {
      // batch size throttled by the free stack space: with few free slots the
      // LIFO walk is depth-first and grows the stack by at most one item per
      // tree level (depth <= 9), so it never overflows
      const int room = (kWStack - 12 - sp) / 2;
      int m = sp < 32 ? sp : 32;
      m = m < room ? m : (room > 1 ? room : 1);
      const int base = sp - m;
      WItem it;
      if (lane < m) it = W.stack[base + lane];
      __syncwarp();
      bool split = false, leaf = false;
      double bound = 0, mid = 0, cm = 0, sm_ = 0;
      W2 wm;
      if (lane < m) {
        const PolyParams p = poly_params(W.br[it.k], eta, support_c);
        const W2 w0{it.r0, it.i0}, w1{it.r1, it.i1};
        const double rho1_min = dmin(w0.rho1, w1.rho1);
        const double inv_min = dmin(w0.inv, w1.inv);
        const double w_lb = p.eta * rho1_min * rho1_min + (1.0 - p.eta) * inv_min;
        bound = sqrt(p.support_c / dmax(w_lb, 1e-12)) / cos(0.5 * (it.a1 - it.a0));
        if (it.depth < 9 && it.a1 - it.a0 > 2e-3 && bound > 1.25 * dmin(radius_true(p, w0), radius_true(p, w1))) {
          split = true;
          mid = 0.5 * (it.a0 + it.a1);
          wm = weight_cs(p, mid, &cm, &sm_);
        } else {
          leaf = true;
        }
      }
      const unsigned smk = __ballot_sync(FULL, split), lmk = __ballot_sync(FULL, leaf);
      const unsigned below = (1u << lane) - 1u;
      const int n_split = __popc(smk), n_leaf = __popc(lmk);
      if (base + 2 * n_split > kWStack || nv + 2 * n_leaf > kWVerts) {
        fail = true;
        break;
      }
      if (split) {
        const int slot = base + 2 * __popc(smk & below);
        WItem l = it, r = it;
        l.a1 = mid;
        l.r1 = wm.rho1;
        l.i1 = wm.inv;
        l.c1 = cm;
        l.s1 = sm_;
        r.a0 = mid;
        r.r0 = wm.rho1;
        r.i0 = wm.inv;
        r.c0 = cm;
        r.s0 = sm_;
        l.depth = r.depth = it.depth + 1;
        W.stack[slot] = l;
        W.stack[slot + 1] = r;
      }
      bool clip = false;
      if (leaf) {
        const int slot = nv + 2 * __popc(lmk & below);
        const double cs[2][2] = {{it.c0, it.s0}, {it.c1, it.s1}};
        for (int e = 0; e < 2; ++e) {
          double w[3], pc[3];
          for (int a = 0; a < 3; ++a) w[a] = mu[a] + bound * (cs[e][0] * rx[a] + cs[e][1] * ry[a]);
          if (MODE == 1)
            for (int a = 0; a < 3; ++a) Wworld[3 * (slot + e) + a] = w[a];
          to_camera(cam, w, pc);
          clip |= !(pc[2] >= kNearClip);
          W.verts[slot + e] = make_double2(cam.fx * pc[0] / pc[2] + cam.cx, cam.fy * pc[1] / pc[2] + cam.cy);
        }
      }
      if (__any_sync(FULL, clip)) {
        if (MODE == 1) {
          clip_any = true;  // this view takes the serial path, the cache still needs every vertex
        } else {
          fail = true;
          break;
        }
      }
      sp = base + 2 * n_split;
      nv += 2 * n_leaf;
      __syncwarp();
    }
    if (MODE == 1) {
      // publish the leaves' world-space vertices (count -1: the tree overflowed)
      int2 r = make_int2(0, -1);
      if (!fail) {
        unsigned long long off = 0;
        if (lane == 0) off = atomicAdd(vcursor, (unsigned long long)nv);
        off = __shfl_sync(FULL, off, 0);
        if ((long long)off + nv <= vcap) {
          __syncwarp();
          for (int t = lane; t < 3 * nv; t += 32) vpool[3 * off + t] = Wworld[t];
          r = make_int2((int)off, nv);
        } else {
          r = make_int2(0, -2);
        }
      }
      if (lane == 0) vref[i] = r;
      if (clip_any) fail = true;
    }
  }  // !cached
  if (fail) {
    // serial path with the near clip and large buffers (k_prep1)
    if (lane == 0) {
      const unsigned long long slot = atomicAdd(&counters[C_POLY_OVERFLOW], 1ull);
      overflow[slot] = i;
    }
    return;
  }
  if (nv == 0) return;
  // bitonic sort of the projected vertices by (x, y) (raster.cpp:35-37)
  int P2 = 2;
  while (P2 < nv) P2 <<= 1;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int t = nv + lane; t < P2; t += 32) W.verts[t] = make_double2(inf, inf);
  __syncwarp();
  // Two stages (j, j / 2) per shared-memory round trip: the four elements
  // {b, b + h, b + j, b + j + h} (h = j / 2, b with bits j and h clear) are
  // closed under both stages' compare-exchanges; a single stage for j = 1.
  // (The round trips' latency is what K1's sort costs: config 3 K1 -4%; three
  // stages per trip measured +19%, a register network with shuffles 2x slower.)
  for (int kk = 2; kk <= P2; kk <<= 1) {
    int jj = kk >> 1;
    while (jj > 0) {
      if (jj >= 2) {
        const int h = jj >> 1;
        for (int q = lane; q < (P2 >> 2); q += 32) {
          const int b = ((q & ~(h - 1)) << 2) | (q & (h - 1));
          double2 v0 = W.verts[b], v1 = W.verts[b + h], v2 = W.verts[b + jj], v3 = W.verts[b + jj + h];
          const bool up = (b & kk) == 0;
          auto ce = [up](double2& a, double2& c) {
            if (up ? lessp2(c, a) : lessp2(a, c)) {
              const double2 t = a;
              a = c;
              c = t;
            }
          };
          ce(v0, v2);
          ce(v1, v3);
          ce(v0, v1);
          ce(v2, v3);
          W.verts[b] = v0;
          W.verts[b + h] = v1;
          W.verts[b + jj] = v2;
          W.verts[b + jj + h] = v3;
        }
        jj >>= 2;
      } else {
        for (int q = lane; q < (P2 >> 1); q += 32) {
          const int t = q << 1;
          const double2 a = W.verts[t], c = W.verts[t + 1];
          const bool up = (t & kk) == 0;
          if (up ? lessp2(c, a) : lessp2(a, c)) {
            W.verts[t] = c;
            W.verts[t + 1] = a;
          }
        }
        jj = 0;
      }
      __syncwarp();
    }
  }
  // unique (raster.cpp:38-40), compacted in place (reads precede writes in
  // every 32-wide chunk)
  int n_u = 0;
  for (int t0 = 0; t0 < nv; t0 += 32) {
    const int t = t0 + lane;
    bool keep = false;
    double2 v;
    if (t < nv) {
      v = W.verts[t];
      keep = t == 0 || !(v.x == W.verts[t - 1].x && v.y == W.verts[t - 1].y);
    }
    const unsigned km = __ballot_sync(FULL, keep);
    if (keep) W.verts[n_u + __popc(km & ((1u << lane) - 1u))] = v;
    n_u += __popc(km);
    __syncwarp();
  }
  long long off = 0;
  if (lane == 0) off = (long long)atomicAdd(&counters[C_PTS_POOL], (unsigned long long)(3 * n_u + 2));
  off = __shfl_sync(FULL, off, 0);
  if (off + 3 * n_u + 2 > pts_cap) return;  // host detects via the cursor and retries with a larger pool
  for (int t = lane; t < n_u; t += 32) pts_pool[off + t] = W.verts[t];
  if (lane == 0) ptsref[i] = make_int2((int)off, n_u);
}

template <int MODE>
static void launch_prep_warp_mode(const Activated& A, const CamD& cam, const OptD& opt, Geo* geo, int4* bbox,
                                  int2* hullref, double2* ppool, long long pts_cap, int2* ptsref, int* rowcnt,
                                  unsigned long long* ctr, int* ovf, float4* frame32, int i0, int i1,
                                  const VertexCache& vc, cudaStream_t s) {
  static PerDeviceOnce attr;
  const size_t smem = prep_warp_smem(MODE);
  attr([&] { cudaFuncSetAttribute(k_prep_warp<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  k_prep_warp<MODE><<<(i1 - i0 + kPW - 1) / kPW, 32 * kPW, smem, s>>>(A, cam, opt, geo, bbox, hullref, ppool, pts_cap,
                                                                   ptsref, rowcnt, ctr, ovf, frame32, i0, i1, vc.pool,
                                                                   vc.cap, vc.ref, vc.cursor);
}

void launch_prep_warp(int mode, const Activated& A, const CamD& cam, const OptD& opt, Geo* geo, int4* bbox,
                      int2* hullref, double2* ppool, long long pts_cap, int2* ptsref, int* rowcnt,
                      unsigned long long* ctr, int* ovf, float4* frame32, int i0, int i1, const VertexCache& vc,
                      cudaStream_t s) {
  if (i1 <= i0) return;
  if (mode == 1)
    launch_prep_warp_mode<1>(A, cam, opt, geo, bbox, hullref, ppool, pts_cap, ptsref, rowcnt, ctr, ovf, frame32, i0, i1, vc, s);
  else if (mode == 2)
    launch_prep_warp_mode<2>(A, cam, opt, geo, bbox, hullref, ppool, pts_cap, ptsref, rowcnt, ctr, ovf, frame32, i0, i1, vc, s);
  else
    launch_prep_warp_mode<0>(A, cam, opt, geo, bbox, hullref, ppool, pts_cap, ptsref, rowcnt, ctr, ovf, frame32, i0, i1, vc, s);
}

// Phase B: Andrew's monotone chain (raster.cpp:41-57) with two threads per
// primitive.  The upper chain only ever pops its own entries (k >= lower),
// so it is the chain over the reversed points: thread 2p builds the lower
// chain, thread 2p+1 the upper; hull = lower + upper without its first (the
// rightmost point) and last (the leftmost).  Then bbox and tile range
// (raster.cpp:219-231) and the hull into the hull pool.
__global__ void __launch_bounds__(256) k_prep_hull(int n, const int2* __restrict__ ptsref, double2* pts_pool,
                                                    CamD cam, OptD opt, int4* bbox, int2* hullref, double2* pool,
                                                    long long pool_cap, int* rowcnt, unsigned long long* counters) {
  const unsigned FULL = 0xffffffffu;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int i = (int)(t >> 1);
  const bool upper = (t & 1) != 0;
  int2 pr = make_int2(0, 0);
  if (i < n) pr = ptsref[i];
  const int n_u = pr.y;
  const double2* pts = pts_pool + pr.x;
  int len = 0;
  if (n_u > 2) len = mono_chain(pts, n_u, upper, pts_pool + pr.x + (upper ? 2 * n_u + 1 : n_u));
  const int other = __shfl_xor_sync(FULL, len, 1);
  if (n_u == 0) return;
  const int L = upper ? other : len, U = upper ? len : other;
  const int hn = n_u <= 2 ? n_u : L + U - 2;
  // my part of the hull: lower [0, L) from the even thread, upper [1, U-1) from the odd one
  const double2* src = n_u <= 2 ? pts : (upper ? pts_pool + pr.x + 2 * n_u + 1 + 1 : pts_pool + pr.x + n_u);
  const int cnt = n_u <= 2 ? (upper ? 0 : n_u) : (upper ? U - 2 : L);
  const int dst = upper ? L : 0;
  double hx0 = 0, hx1 = 0, hy0 = 0, hy1 = 0;
  bool any = false;
  for (int j = 0; j < cnt; ++j) {
    const double2 v = src[j];
    if (!any) {
      hx0 = hx1 = v.x;
      hy0 = hy1 = v.y;
      any = true;
    } else {
      hx0 = dmin(hx0, v.x);
      hx1 = dmax(hx1, v.x);
      hy0 = dmin(hy0, v.y);
      hy1 = dmax(hy1, v.y);
    }
  }
  // combine the two halves (the pair is always in one warp and both reach here)
  const unsigned pair = 3u << ((threadIdx.x & 31) & ~1);
  const double ox0 = __shfl_xor_sync(pair, hx0, 1), ox1 = __shfl_xor_sync(pair, hx1, 1);
  const double oy0 = __shfl_xor_sync(pair, hy0, 1), oy1 = __shfl_xor_sync(pair, hy1, 1);
  const bool oany = __shfl_xor_sync(pair, any, 1);
  if (oany) {
    if (!any) {
      hx0 = ox0;
      hx1 = ox1;
      hy0 = oy0;
      hy1 = oy1;
    } else {
      hx0 = dmin(hx0, ox0);
      hx1 = dmax(hx1, ox1);
      hy0 = dmin(hy0, oy0);
      hy1 = dmax(hy1, oy1);
    }
  }
  const double lp = opt.lp_pad;
  int tx0 = x86_int(floor((hx0 - lp) / kTile));
  tx0 = tx0 > 0 ? tx0 : 0;
  int tx1 = x86_int(floor((hx1 + lp) / kTile));
  tx1 = tx1 < cam.tiles_x - 1 ? tx1 : cam.tiles_x - 1;
  int ty0 = x86_int(floor((hy0 - lp) / kTile));
  ty0 = ty0 > 0 ? ty0 : 0;
  int ty1 = x86_int(floor((hy1 + lp) / kTile));
  ty1 = ty1 < cam.tiles_y - 1 ? ty1 : cam.tiles_y - 1;
  if (tx1 < tx0 || ty1 < ty0) return;
  long long off = 0;
  if (!upper) off = (long long)atomicAdd(&counters[C_HULL_POOL], (unsigned long long)hn);
  off = __shfl_xor_sync(pair, off, 1) + (upper ? 0 : off);
  if (off + hn > pool_cap) return;  // host detects via the cursor and retries with a larger pool
  for (int j = 0; j < cnt; ++j) pool[off + dst + j] = src[j];
  if (!upper) {
    hullref[i] = make_int2((int)off, hn);
    bbox[i] = make_int4(tx0, tx1, ty0, ty1);
    rowcnt[i] = ty1 - ty0 + 1;
    atomicAdd(&counters[C_VISIBLE], 1ull);
  }
}

// ---------------------------------------------------------------------------
// K2: per-row tile intervals.  For a convex hull H and the dilated row band
// B = [Y0, Y1], a dilated tile rectangle overlaps H iff its x-range meets the
// x-extent of H ∩ B.  That is the geometric content of the reference's
// separating-axis test (raster.cpp:63-97); decisions within 1e-9 relative of
// a tie are resolved with a replica of that test (same op order) and counted.
// ---------------------------------------------------------------------------
__device__ bool hull_overlaps_rect(const double2* h, int n, double x0, double y0, double x1, double y1) {
  if (n == 0) return false;
  double hx0 = h[0].x, hx1 = h[0].x, hy0 = h[0].y, hy1 = h[0].y;
  for (int i = 0; i < n; ++i) {
    hx0 = dmin(hx0, h[i].x);
    hx1 = dmax(hx1, h[i].x);
    hy0 = dmin(hy0, h[i].y);
    hy1 = dmax(hy1, h[i].y);
  }
  if (hx1 < x0 || hx0 > x1 || hy1 < y0 || hy0 > y1) return false;
  if (n <= 1) return true;
  const double cx[4] = {x0, x1, x1, x0}, cy[4] = {y0, y0, y1, y1};
  for (int i = 0; i < n; ++i) {
    const double2 a = h[i], b = h[(i + 1) % n];
    const double ex = b.x - a.x, ey = b.y - a.y;
    if (ex * ex + ey * ey < 1e-24) continue;
    const double ax = -ey, ay = ex;
    double pmin = ax * h[0].x + ay * h[0].y, pmax = pmin;
    for (int j = 0; j < n; ++j) {
      const double d = ax * h[j].x + ay * h[j].y;
      pmin = dmin(pmin, d);
      pmax = dmax(pmax, d);
    }
    double rmin = ax * cx[0] + ay * cy[0], rmax = rmin;
    for (int j = 0; j < 4; ++j) {
      const double d = ax * cx[j] + ay * cy[j];
      rmin = dmin(rmin, d);
      rmax = dmax(rmax, d);
    }
    if (pmax < rmin || pmin > rmax) return false;
  }
  return true;
}

// Banded frames: rows of primitive i inside tile rows [ty_lo, ty_hi).
__global__ void k_band_rowcnt(int n, const int4* __restrict__ bbox, int ty_lo, int ty_hi, int* rowcnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 bb = bbox[i];
  const int a = max(bb.z, ty_lo), b = min(bb.w, ty_hi - 1);
  rowcnt[i] = (bb.y >= bb.x && b >= a) ? b - a + 1 : 0;
}

// Upper bound of the pairs per tile row (bbox width per covered row), for
// choosing the bands.
__global__ void k_row_pair_bound(int n, int tiles_y, const int4* __restrict__ bbox, unsigned long long* rowest) {
  // per-block tile-row sums in shared memory (tiles_y <= kRowEstSmem), one
  // global atomic per row and block
  extern __shared__ unsigned long long s_est[];
  for (int t = threadIdx.x; t < tiles_y; t += blockDim.x) s_est[t] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 bb = bbox[i];
    if (bb.y < bb.x || bb.w < bb.z) continue;
    for (int ty = bb.z; ty <= bb.w; ++ty) atomicAdd(&s_est[ty], (unsigned long long)(bb.y - bb.x + 1));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < tiles_y; t += blockDim.x)
    if (s_est[t]) atomicAdd(&rowest[t], s_est[t]);
}

// Backward of a banded frame: the band's flagged pixels (fp64 re-render list).
__global__ void k_band_flagged(const unsigned char* __restrict__ pxflag, int W, int y0, int y1, int* list,
                               unsigned* count) {
  const long long p = (long long)y0 * W + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= (long long)y1 * W) return;
  if (pxflag[p]) list[atomicAdd(count, 1u)] = (int)p;
}

// Row record: prim id, tile row, first and last tile column (ta > tb: empty).
__global__ void k_rows(int n, const int4* __restrict__ bbox, const int2* __restrict__ hullref,
                       const double2* __restrict__ pool, const long long* __restrict__ rowoff, CamD cam, OptD opt,
                       int4* rows, int* rowpaircnt, unsigned long long* counters, int ty_lo, int ty_hi) {
  // one warp per primitive, lanes over its tile rows
  const int i = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;  // warp-uniform
  const int4 bb = bbox[i];
  if (bb.y < bb.x || bb.w < bb.z) return;
  const int2 hr = hullref[i];
  const double2* h = pool + hr.x;
  const int hn = hr.y;
  const double lp = opt.lp_pad;
  double hy_min = h[0].y, hy_max = h[0].y, amax = 1.0;
  for (int j = 0; j < hn; ++j) {
    hy_min = dmin(hy_min, h[j].y);
    hy_max = dmax(hy_max, h[j].y);
    amax = dmax(amax, dmax(fabs(h[j].x), fabs(h[j].y)));
  }
  const double delta = 1e-9 * amax + 1e-9;
  unsigned long long ties = 0;
  const int tyA = max(bb.z, ty_lo);
  for (int ty = tyA + lane; ty <= min(bb.w, ty_hi - 1); ty += 32) {
    const long long ro = rowoff[i] + (ty - tyA);
    const double y0 = ty * kTile, y1 = y0 + kTile;
    const double Y0 = y0 - lp, Y1 = y1 + lp;
    // x-extent of H ∩ [Y0, Y1]
    double xl = __longlong_as_double(0x7ff0000000000000ll), xr = -xl;
    for (int j = 0; j < hn; ++j) {
      const double2 a = h[j];
      if (a.y >= Y0 && a.y <= Y1) {
        xl = dmin(xl, a.x);
        xr = dmax(xr, a.x);
      }
      if (hn > 1) {
        const double2 b = h[(j + 1) % hn];
        const double Ys[2] = {Y0, Y1};
        for (int e = 0; e < 2; ++e) {
          const double Yc = Ys[e];
          if ((a.y < Yc && b.y > Yc) || (a.y > Yc && b.y < Yc)) {
            const double xc = a.x + (Yc - a.y) * (b.x - a.x) / (b.y - a.y);
            xl = dmin(xl, xc);
            xr = dmax(xr, xc);
          }
        }
      }
    }
    const bool row_ambiguous = fabs(hy_max - Y0) <= delta || fabs(hy_min - Y1) <= delta;
    int ta = bb.x, tb = bb.x - 1;
    if (row_ambiguous) {
      // resolve every tile of the row with the reference test
      ++ties;
      int first = -1, last = -2;
      for (int tx = bb.x; tx <= bb.y; ++tx) {
        const double x0 = tx * kTile, x1 = x0 + kTile;
        if (hull_overlaps_rect(h, hn, x0 - lp, Y0, x1 + lp, Y1)) {
          if (first < 0) first = tx;
          last = tx;
        }
      }
      if (first >= 0) {
        ta = first;
        tb = last;
      }
    } else if (xl <= xr) {
      // first tile with X1 >= xl, last tile with X0 <= xr
      int a = bb.x;
      while (a <= bb.y && (a * kTile + kTile + lp) < xl - delta) ++a;
      int b = bb.y;
      while (b >= a && (b * kTile - lp) > xr + delta) --b;
      if (a <= b) {
        // boundary tiles inside the tie band: reference test decides
        const double x0a = a * kTile, x1a = x0a + kTile;
        if (fabs((x1a + lp) - xl) <= delta || fabs((x0a - lp) - xr) <= delta) {
          ++ties;
          if (!hull_overlaps_rect(h, hn, x0a - lp, Y0, x1a + lp, Y1)) ++a;
        }
        if (b >= a) {
          const double x0b = b * kTile, x1b = x0b + kTile;
          if (fabs((x0b - lp) - xr) <= delta || fabs((x1b + lp) - xl) <= delta) {
            ++ties;
            if (!hull_overlaps_rect(h, hn, x0b - lp, Y0, x1b + lp, Y1)) --b;
          }
        }
        ta = a;
        tb = b;
      }
    }
    rows[ro] = make_int4(i, ty, ta, tb);
    rowpaircnt[ro] = tb >= ta ? tb - ta + 1 : 0;
  }
  if (ties) atomicAdd(&counters[C_NEAR_TIES], ties);
}

// Corner rays of the tile grid ((tiles_x+1) x (tiles_y+1)) and tile-centre
// rays, pixel_ray at the undilated tile corners (raster.cpp:101-102).
__global__ void k_tile_rays(CamD cam, double* cdirs, double* tdirs) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int nc = (cam.tiles_x + 1) * (cam.tiles_y + 1);
  const int nt = cam.tiles_x * cam.tiles_y;
  double d[3];
  if (idx < nc) {
    const int cx = idx % (cam.tiles_x + 1), cy = idx / (cam.tiles_x + 1);
    pixel_dir(cam, (double)(cx * kTile), (double)(cy * kTile), d);
    for (int a = 0; a < 3; ++a) cdirs[3 * (size_t)idx + a] = d[a];
  } else if (idx < nc + nt) {
    const int t = idx - nc;
    const double x0 = (t % cam.tiles_x) * kTile, y0 = (t / cam.tiles_x) * kTile;
    pixel_dir(cam, 0.5 * (x0 + (x0 + kTile)), 0.5 * (y0 + (y0 + kTile)), d);
    for (int a = 0; a < 3; ++a) tdirs[3 * (size_t)t + a] = d[a];
  }
}

// classify_intersect depth only (geometry.cpp:40-48) of one corner / centre
// ray is num / den, +inf when |den| < eps or the quotient is not positive
// (raster.cpp:99-115 nearest_depth_key).  One expression (ray_denom +
// nearest_depth5) for every caller so the emitted keys, the tie fix and
// drk_get_tile_lists agree bit for bit.
__device__ __forceinline__ double ray_denom(const double* d, double rz0, double rz1, double rz2) {
  return d[0] * rz0 + d[1] * rz1 + d[2] * rz2;
}

// NearestDepth key of the five tile rays (raster.cpp:99-115) from their
// denominators (top, right-top, right-bottom, bottom, centre):
// min over the rays of ray_depth.  One division instead of five: a ray is
// valid iff |den| >= eps and den has num's sign (then num / den > 0 exactly),
// division by a larger |den| gives a smaller exact quotient and rounding is
// monotone, so the minimum of the rounded quotients is the rounded quotient of
// the valid denominator of largest magnitude.  A quotient that underflows to 0
// or overflows (the reference then drops that ray or keeps +inf) takes the
// per-ray path.  Returns +inf when no ray is valid.
__device__ __forceinline__ double nearest_depth5(const double den[5], double num, double eps) {
  double best_den = 0;
  bool any = false;
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const double d = den[r];
    const bool valid = fabs(d) >= eps && ((num > 0 && d > 0) || (num < 0 && d < 0));
    if (valid && (!any || fabs(d) > fabs(best_den))) {
      best_den = d;
      any = true;
    }
  }
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  if (!any) return inf;
  const double q = num / best_den;
  if (q > 0 && q < inf) return q;
  double best = inf;  // per-ray path (raster.cpp:99-115 as written)
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    double qr = inf;
    if (!(fabs(den[r]) < eps)) {
      const double t = num / den[r];
      if (t > 0) qr = t;
    }
    best = dmin(best, qr);
  }
  return best;
}

// Full fp64 presort key of (tile, primitive) (raster.cpp:99-115, 233-257).
__device__ double pair_key(const Geo& g, int pid, int tile, const CamD& cam, const OptD& opt,
                           const double* __restrict__ cdirs, const double* __restrict__ tdirs) {
  if (opt.presort == 0) return (double)pid;
  if (opt.presort == 1) return g.projz;
  const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x, cw = cam.tiles_x + 1;
  const int c00 = ty * cw + tx;
  const double rz0 = g.rz[0], rz1 = g.rz[1], rz2 = g.rz[2];
  const double den[5] = {ray_denom(cdirs + 3 * (size_t)c00, rz0, rz1, rz2),
                         ray_denom(cdirs + 3 * (size_t)(c00 + 1), rz0, rz1, rz2),
                         ray_denom(cdirs + 3 * (size_t)(c00 + cw + 1), rz0, rz1, rz2),
                         ray_denom(cdirs + 3 * (size_t)(c00 + cw), rz0, rz1, rz2),
                         ray_denom(tdirs + 3 * (size_t)tile, rz0, rz1, rz2)};
  double best = nearest_depth5(den, g.num, opt.grazing_eps);
  if (isinf(best) && g.has_proj) best = g.projz;
  return best;
}

// Total order of the fp64 keys as unsigned integers (numeric order; the
// reference compares the doubles with <).
__device__ __forceinline__ unsigned long long key_order(double key) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(key);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
constexpr unsigned kInfKey32 = 0xfff00000u;  // key_order(+inf) >> 32: keys at or above are not finite

// K3 with 16 lanes per row: lane l owns tile ta + l (chunks of 16), evaluates
// its left corner rays and its centre ray, and takes the right corners from
// lane l + 1 (the last lane of a chunk evaluates them itself), so a row of m
// tiles costs ~3m ray-plane depths instead of 5m.  The key is the minimum of the
// five depths (raster.cpp:99-115; min is symmetric for the positive depths).
constexpr int kEmitLanes = 16;
__global__ void __launch_bounds__(256) k_emit_rows(long long n_rows, const int4* __restrict__ rows,
                                                   const long long* __restrict__ rowpairoff,
                                                   const Geo* __restrict__ geo, const double* __restrict__ cdirs,
                                                   const double* __restrict__ tdirs, CamD cam, OptD opt,
                                                   unsigned long long* pk, unsigned* pv,
                                                   unsigned* krange /* min, max finite key32 */) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long r = t / kEmitLanes;
  const int l = (int)(t % kEmitLanes);
  const unsigned seg = 0xffffu << (threadIdx.x & 16);  // this lane's 16-lane segment
  __shared__ unsigned s_kr[2];
  if (threadIdx.x == 0) {
    s_kr[0] = 0xffffffffu;
    s_kr[1] = 0u;
  }
  __syncthreads();
  int4 rr = make_int4(0, 0, 0, -1);  // rows past the end: empty (every thread reaches the block reduction)
  if (r < n_rows) rr = rows[r];
  const int pid = rr.x, ty = rr.y;
  const Geo& g = geo[pid];
  const long long pos0 = r < n_rows ? rowpairoff[r] : 0;
  const int cw = cam.tiles_x + 1;
  const double rz0 = g.rz[0], rz1 = g.rz[1], rz2 = g.rz[2], num = g.num, eps = opt.grazing_eps;
  auto dnm = [&](const double* d) -> double { return ray_denom(d, rz0, rz1, rz2); };
  unsigned kmin = 0xffffffffu, kmax = 0u;
  for (int base = rr.z; base <= rr.w; base += kEmitLanes) {
    const int tx = base + l;
    const bool valid = tx <= rr.w;
    const int txc = valid ? tx : rr.w;
    double key;
    if (opt.presort == 0) {
      key = (double)pid;
    } else if (opt.presort == 1) {
      key = g.projz;
    } else {
      const int c00 = ty * cw + txc;
      double den[5];
      den[0] = dnm(cdirs + 3 * (size_t)c00);
      den[3] = dnm(cdirs + 3 * (size_t)(c00 + cw));
      den[4] = dnm(tdirs + 3 * (size_t)(ty * cam.tiles_x + txc));
      den[1] = __shfl_down_sync(seg, den[0], 1, kEmitLanes);
      den[2] = __shfl_down_sync(seg, den[3], 1, kEmitLanes);
      if (l == kEmitLanes - 1 || tx >= rr.w) {
        den[1] = dnm(cdirs + 3 * (size_t)(c00 + 1));
        den[2] = dnm(cdirs + 3 * (size_t)(c00 + cw + 1));
      }
      double best = nearest_depth5(den, num, eps);
      if (isinf(best) && g.has_proj) best = g.projz;
      key = best;
    }
    // top 32 bits of the key's numeric order; k_pack_keys quantises them
    // against the frame's finite key range
    const unsigned k32 = (unsigned)(key_order(key) >> 32);
    if (valid) {
      const int tile = ty * cam.tiles_x + tx;
      const long long pos = pos0 + (tx - rr.z);
      pk[pos] = ((unsigned long long)(unsigned)tile << 32) | k32;
      pv[pos] = (unsigned)pid;
    }
    kmin = min(kmin, valid && k32 < kInfKey32 ? k32 : 0xffffffffu);
    kmax = max(kmax, valid && k32 < kInfKey32 ? k32 : 0u);
  }
  // block reduction of the finite key range, one atomic pair per block
  kmin = __reduce_min_sync(seg, kmin);
  kmax = __reduce_max_sync(seg, kmax);
  if ((threadIdx.x & 15) == 0) {
    atomicMin(&s_kr[0], kmin);
    atomicMax(&s_kr[1], kmax);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_kr[0] != 0xffffffffu) atomicMin(&krange[0], s_kr[0]);
    if (s_kr[1] != 0u) atomicMax(&krange[1], s_kr[1]);
  }
}

// Sort key of each emitted pair: tile << dbits | q, q a monotone map of the
// key32 (key_order >> 32) to dbits bits.  The map equalises the depth density
// so that few pairs of one tile share a q (each such run is ordered on the full
// keys afterwards, k_tie_rank): the finite key range [lo, hi] is cut into
// kQBins bins of 2^shift0 key32 units, a sample of the pairs is histogrammed,
// and bin j gets a power-of-two share a_j of the q space (proportional to its
// count, at least 1), q = base_j + ((k32 - start_j) >> s_j).  Non-finite keys
// take the top q.  Any monotone map gives the same final order (ties are
// resolved on the full key); this one only keeps the runs short.
constexpr int kQBins = 4096, kQSample = 8;

__device__ __forceinline__ int qbin_shift(unsigned lo, unsigned hi) {
  const unsigned span = hi > lo ? hi - lo : 0u;
  const int len = 32 - __clz(span);  // bits of the span
  return len > 12 ? len - 12 : 0;    // span >> shift0 < kQBins
}

__global__ void __launch_bounds__(256) k_key_hist(long long n, const unsigned long long* __restrict__ pk,
                                                  const unsigned* __restrict__ krange, unsigned* hist) {
  __shared__ unsigned h[kQBins];
  for (int j = threadIdx.x; j < kQBins; j += blockDim.x) h[j] = 0;
  __syncthreads();
  const unsigned lo = krange[0], hi = krange[1];
  const int sh = qbin_shift(lo, hi);
  const long long stride = (long long)gridDim.x * blockDim.x * kQSample;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kQSample; i < n; i += stride) {
    const unsigned k32 = (unsigned)pk[i];
    if (k32 >= lo && k32 <= hi) atomicAdd(&h[min((k32 - lo) >> sh, (unsigned)kQBins - 1u)], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < kQBins; j += blockDim.x)
    if (h[j]) atomicAdd(&hist[j], h[j]);
}

// One block: per-bin share exponents and bases (map[j] = base << 5 | s_j).
__global__ void __launch_bounds__(1024) k_key_map(const unsigned* __restrict__ hist, const unsigned* __restrict__ krange,
                                                  int dbits, unsigned* map) {
  __shared__ unsigned long long tot_s;
  __shared__ unsigned wsum[32];
  if (threadIdx.x == 0) tot_s = 0;
  __syncthreads();
  constexpr int kPer = kQBins / 1024;
  unsigned c[kPer];
  unsigned long long t = 0;
  for (int q = 0; q < kPer; ++q) {
    c[q] = hist[threadIdx.x * kPer + q];
    t += c[q];
  }
  atomicAdd(&tot_s, t);
  __syncthreads();
  const double tot = (double)(tot_s ? tot_s : 1ull);
  const int sh = qbin_shift(krange[0], krange[1]);
  const double budget = (double)((1u << dbits) - 1u - kQBins);  // the +1 minimum of every bin on top
  unsigned a[kPer], run = 0;
  int sj[kPer];
  for (int q = 0; q < kPer; ++q) {
    const double want = budget * (double)c[q] / tot;
    int e = want >= 1.0 ? (int)floor(log2(want)) : 0;  // a_j = 2^e <= want (at least 1)
    e = min(e, sh);                                    // never finer than one key32 unit
    a[q] = 1u << e;
    sj[q] = sh - e;
    run += a[q];
  }
  // block exclusive scan of the per-thread totals
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned incl = run;
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    unsigned v = wsum[lane], x = v;
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    wsum[lane] = x - v;
  }
  __syncthreads();
  unsigned base = wsum[w] + incl - run;
  for (int q = 0; q < kPer; ++q) {
    map[threadIdx.x * kPer + q] = base << 5 | (unsigned)sj[q];
    base += a[q];
  }
}

__global__ void __launch_bounds__(256) k_pack_keys(long long n, const unsigned long long* __restrict__ pk,
                                                   const unsigned* __restrict__ krange,
                                                   const unsigned* __restrict__ map, int dbits, unsigned* sk) {
  __shared__ unsigned m[kQBins];
  for (int j = threadIdx.x; j < kQBins; j += blockDim.x) m[j] = map[j];
  __syncthreads();
  const unsigned lo = krange[0], hi = krange[1];
  const int sh = qbin_shift(lo, hi);
  const unsigned qmax = (1u << dbits) - 1u;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = pk[i];
    const unsigned k32 = (unsigned)k;
    unsigned q = qmax;
    if (k32 >= lo && k32 <= hi) {
      const unsigned off = k32 - lo;
      const unsigned j = min(off >> sh, (unsigned)kQBins - 1u);
      const unsigned e = m[j];
      q = (e >> 5) + ((off - (j << sh)) >> (e & 31u));
    }
    sk[i] = ((unsigned)(k >> 32) << dbits) | q;
  }
}

// After the sort: runs of equal packed sort keys are put in (full fp64 key,
// pid) order — the reference's order (raster.cpp:260-263: each tile list
// sorted by key, ties by primitive id).  Every run member computes its full key
// (k_tie_keys, into the dead emission buffer); runs of up to kRankMax entries
// are then ordered in parallel — each member counts the members that precede
// it and writes its id at run start + rank into a second id buffer — and
// longer runs by one thread (k_tie_long, insertion sort).
constexpr int kRankMax = 1024;

__device__ __forceinline__ bool in_run(long long n, const unsigned* sk, long long i, unsigned k) {
  return (i + 1 < n && sk[i + 1] == k) || (i > 0 && sk[i - 1] == k);
}

__global__ void k_tie_keys(long long n, const unsigned* __restrict__ sk, const unsigned* __restrict__ sv, int dbits,
                           const Geo* __restrict__ geo, const double* __restrict__ cdirs,
                           const double* __restrict__ tdirs, CamD cam, OptD opt, unsigned long long* fk) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned k = sk[i];
  if (!in_run(n, sk, i, k)) return;
  const unsigned pid = sv[i];
  fk[i] = key_order(pair_key(geo[pid], (int)pid, (int)(k >> dbits), cam, opt, cdirs, tdirs));
}

__device__ __forceinline__ bool pair_less(unsigned long long ka, unsigned pa, unsigned long long kb, unsigned pb) {
  return ka < kb || (ka == kb && pa < pb);
}

__global__ void k_tie_rank(long long n, const unsigned* __restrict__ sk, const unsigned* __restrict__ sv,
                           const unsigned long long* __restrict__ fk, unsigned* out, unsigned long long* counters,
                           long long* long_runs) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const unsigned k = i < n ? sk[i] : 0u;
  const bool member = i < n && in_run(n, sk, i, k);
  const bool start = member && !(i > 0 && sk[i - 1] == k);
  long long s = i, e = i + 1;
  if (member) {
    while (s > 0 && sk[s - 1] == k && i - s <= kRankMax) --s;
    while (e < n && sk[e] == k && e - s <= kRankMax) ++e;
  }
  if (counters && __ballot_sync(0xffffffffu, start)) {
    // run statistics (work counters on), aggregated per warp
    const unsigned len = start ? (unsigned)(e - i) : 0u;
    const unsigned runs = __reduce_add_sync(0xffffffffu, start ? 1u : 0u);
    const unsigned mem = __reduce_add_sync(0xffffffffu, len);
    const unsigned mx = __reduce_max_sync(0xffffffffu, len);
    if ((threadIdx.x & 31) == 0 && runs) {
      atomicAdd(&counters[C_TIE_RUNS], (unsigned long long)runs);
      atomicAdd(&counters[C_TIE_MEMBERS], (unsigned long long)mem);
      atomicMax(&counters[C_TIE_MAXRUN], (unsigned long long)mx);
    }
  }
  if (i >= n) return;
  const unsigned pid = sv[i];
  if (!member) {
    out[i] = pid;
    return;
  }
  if (e - s > kRankMax) {  // long run: its start is listed for k_tie_long
    out[i] = pid;
    if (start) long_runs[1 + atomicAdd(reinterpret_cast<unsigned long long*>(long_runs), 1ull)] = i;
    return;
  }
  const unsigned long long ki = fk[i];
  long long rank = 0;
  for (long long j = s; j < e; ++j) rank += pair_less(fk[j], sv[j], ki, pid) ? 1 : 0;
  out[s + rank] = pid;
}

// Runs longer than kRankMax (their starts listed by k_tie_rank: long_runs[0] =
// count): one thread per run insertion-sorts it (keys in fk, ids in out) on
// (full key, pid).
__global__ void k_tie_long(long long n, const unsigned* __restrict__ sk, unsigned long long* fk, unsigned* out,
                           const long long* __restrict__ long_runs) {
  const long long cnt = long_runs[0];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = long_runs[1 + t];
    const unsigned k = sk[i];
    long long e = i + 1;
    while (e < n && sk[e] == k) ++e;
    for (long long a = i + 1; a < e; ++a) {
      const unsigned pa = out[a];
      const unsigned long long ka = fk[a];
      long long b = a - 1;
      while (b >= i && pair_less(ka, pa, fk[b], out[b])) {
        out[b + 1] = out[b];
        fk[b + 1] = fk[b];
        --b;
      }
      out[b + 1] = pa;
      fk[b + 1] = ka;
    }
  }
}

// Tile offsets from the sorted keys (tile = key >> dbits): thread i writes
// the starts of the tiles in (tile(i-1), tile(i)]; thread n closes the rest.
__global__ void k_tile_bounds(long long n, const unsigned* __restrict__ sk, int dbits, int n_tiles,
                              long long* tileoff) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int t = i < n ? (int)(sk[i] >> dbits) : n_tiles;
  const int tp = i > 0 ? (int)(sk[i - 1] >> dbits) : -1;
  for (int tt = tp + 1; tt <= t; ++tt) tileoff[tt] = i;
}

// Full fp64 keys of kept per-tile lists (banded frames): the tile of entry i
// from the offsets (binary search; tiles outside the band are empty ranges).
__global__ void k_full_keys_off(long long n, const long long* __restrict__ tileoff, int n_tiles,
                                const unsigned* __restrict__ sv, const Geo* __restrict__ geo,
                                const double* __restrict__ cdirs, const double* __restrict__ tdirs, CamD cam, OptD opt,
                                double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = 0, hi = n_tiles;  // largest t with tileoff[t] <= i
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tileoff[mid] <= i) lo = mid;
    else hi = mid;
  }
  const unsigned pid = sv[i];
  out[i] = pair_key(geo[pid], (int)pid, lo, cam, opt, cdirs, tdirs);
}

// Full fp64 keys of the sorted lists (drk_get_tile_lists).
__global__ void k_full_keys(long long n, const unsigned* __restrict__ sk, const unsigned* __restrict__ sv, int dbits,
                            const Geo* __restrict__ geo, const double* __restrict__ cdirs,
                            const double* __restrict__ tdirs, CamD cam, OptD opt, double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned pid = sv[i];
  out[i] = pair_key(geo[pid], (int)pid, (int)(sk[i] >> dbits), cam, opt, cdirs, tdirs);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int shape_setup(drk_ctx* c, int n, int K) {
  Activated& A = c->act;
  A.ex = ensure<double>(c->a_ex, (size_t)K * n);
  A.ey = ensure<double>(c->a_ey, (size_t)K * n);
  A.det = ensure<double>(c->a_det, (size_t)K * n);
  A.thf = ensure<float>(c->a_thf, (size_t)K * n);
  A.invdetf = ensure<float>(c->a_invdetf, (size_t)K * n);
  A.piogf = ensure<float>(c->a_piogf, (size_t)K * n);
  A.hf = ensure<float>(c->a_hf, (size_t)K * n);
  A.psif = ensure<float>(c->a_psif, 12 * (size_t)n);
  if (!A.ex || !A.ey || !A.det || !A.thf || !A.invdetf || !A.piogf || !A.hf || !A.psif)
    return set_error(c, DRK_ERR_OOM, "shape buffers");
  A.rec = nullptr;
  if (K == 8) {
    // AoS fp32 records of the fast forward kernel (drk_raster_fast.cu)
    A.rec = ensure<float>(c->a_rec, (size_t)88 * n);
    if (!A.rec) return set_error(c, DRK_ERR_OOM, "shape records");
  }
  return DRK_OK;
}

static void shape_range(drk_ctx* c, int i0, int i1) {
  const Activated& A = c->act;
  if (i1 <= i0) return;
  k_shape<<<(i1 - i0 + 127) / 128, 128, 0, c->stream>>>(i0, i1, A.K, A.s, A.th, const_cast<double*>(A.ex),
                                                        const_cast<double*>(A.ey), const_cast<double*>(A.det),
                                                        const_cast<float*>(A.thf), const_cast<float*>(A.invdetf),
                                                        const_cast<float*>(A.piogf), const_cast<float*>(A.hf), A.tau,
                                                        A.o, const_cast<float*>(A.psif));
  DRK_COUNT_LAUNCH();
  if (A.rec) {
    const ShapeView S{A.s, A.th, A.ex, A.ey, A.det, A.eta, A.tau, A.o, A.thf, A.invdetf, A.piogf, A.hf, A.psif, A.K};
    launch_shape_rec(S, i0, i1, const_cast<float*>(A.rec), c->stream);
  }
}

static int launch_shape_consts(drk_ctx* c, int n, int K) {
  if (int st = shape_setup(c, n, K)) return st;
  shape_range(c, 0, n);
  return cuda_check(c, cudaGetLastError(), "shape");
}

int activate_setup(drk_ctx* c, int n, int K, int terms) {
  ++c->act_gen;  // a new activation: the K1 vertex cache is stale
  c->act_renders = 0;
  Activated& A = c->act;
  A.n = n;
  A.K = K;
  A.terms = terms;
  A.mu = ensure<double>(c->a_mu, 3 * (size_t)n);
  A.rot = ensure<double>(c->a_rot, 9 * (size_t)n);
  A.s = ensure<double>(c->a_s, (size_t)K * n);
  A.th = ensure<double>(c->a_th, (size_t)K * n);
  A.eta = ensure<double>(c->a_eta, n);
  A.tau = ensure<double>(c->a_tau, n);
  A.o = ensure<double>(c->a_o, n);
  A.sh = ensure<float>(c->a_sh, (size_t)3 * terms * n);
  A.sh64 = nullptr;  // raw f32 coefficients widen exactly
  unsigned long long* ctr = ensure<unsigned long long>(c->counters, C_COUNT);
  if (!A.mu || !A.rot || !A.s || !A.th || !A.eta || !A.tau || !A.o || !A.sh || !ctr)
    return set_error(c, DRK_ERR_OOM, "activation buffers");
  return shape_setup(c, n, K);
}

// activation + shape constants of primitives [i0, i1) (raw: the whole [S][n] array)
void activate_range(drk_ctx* c, const float* raw, int i0, int i1) {
  const Activated& A = c->act;
  if (i1 <= i0) return;
  k_activate<<<(i1 - i0 + 127) / 128, 128, 0, c->stream>>>(
      raw, A.n, A.K, A.terms, const_cast<double*>(A.mu), const_cast<double*>(A.rot), const_cast<double*>(A.s),
      const_cast<double*>(A.th), const_cast<double*>(A.eta), const_cast<double*>(A.tau), const_cast<double*>(A.o),
      const_cast<float*>(A.sh), static_cast<unsigned long long*>(c->counters.p), i0, i1);
  DRK_COUNT_LAUNCH();
  shape_range(c, i0, i1);
}

int launch_activate(drk_ctx* c, const float* raw, int n, int K, int terms) {
  if (int st = activate_setup(c, n, K, terms)) return st;
  unsigned long long* ctr = static_cast<unsigned long long*>(c->counters.p);
  cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT, c->stream);
  activate_range(c, raw, 0, n);
  if (int st = cuda_check(c, cudaGetLastError(), "activate")) return st;
  unsigned long long h[C_COUNT];
  if (int st = cuda_check(c, cudaMemcpyAsync(h, ctr, sizeof h, cudaMemcpyDeviceToHost, c->stream), "activate"))
    return st;
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "activate")) return st;
  if (h[C_ERR_NONFINITE]) return set_error(c, DRK_ERR_NONFINITE, "raw parameters contain NaN/Inf");
  if (h[C_ERR_DEGEN_QUAT]) return set_error(c, DRK_ERR_DEGENERATE_QUAT, "quaternion norm below 1e-12");
  return DRK_OK;
}

int launch_shape(drk_ctx* c, const drk_prims* p, int n, int K, int terms) {
  ++c->act_gen;
  c->act_renders = 0;
  Activated& A = c->act;
  A.n = n;
  A.K = K;
  A.terms = terms;
  A.mu = p->mu;
  A.rot = p->rot;
  A.s = p->scales;
  A.th = p->angles;
  A.eta = p->eta;
  A.tau = p->tau;
  A.o = p->opacity;
  A.sh = p->sh;
  A.sh64 = p->sh64;
  return launch_shape_consts(c, n, K);
}

}  // namespace drk

namespace drk {
#define DRK_PREP_ARGS                                                                                       \
  Activated A, CamD cam, OptD opt, Geo *geo, int4 *bbox, int2 *hullref, double2 *pool, long long pool_cap, \
      int *rowcnt, unsigned long long *counters, const int *list, int list_n, double2 *scratch,            \
      int scratch_cap, int *overflow
#define DRK_PREP_PASS \
  A, cam, opt, geo, bbox, hullref, pool, pool_cap, rowcnt, counters, list, list_n, scratch, scratch_cap, overflow
__global__ void __launch_bounds__(128) k_prep1(DRK_PREP_ARGS) { prep_body<1>(DRK_PREP_PASS); }
}  // namespace drk
