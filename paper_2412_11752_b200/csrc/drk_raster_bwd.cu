// K5 fast path: backward rasterizer (reference grad.cpp:178-303, :16-101) on
// the fast forward's streaming (drk_raster_fast.cu): fp32 tile-linearised
// intersections, the interval SortCache with exact tie resolution and the same
// alpha evaluation (alpha_entry), so every discrete decision is the forward's
// (and the reference's); termination is the forward's per-pixel composite
// count (P.pxstop).  `rest` starts from the forward's accumulators:
// total = dC.C + dD D + dN.N + dA A with C including T_n bg (grad.cpp:210-222).
//
// Per composited record the activated-space gradient is formed in fp32
// (fp64 for entries whose alpha fell back to fp64) and reduced over the lanes
// of the warp that composite the same primitive in the same step:
//   - SH (48 components): d sh[t][c] = sum_l w_c(l) basis_t(pixel l), a GEMV of
//     the group's 3 weights against the per-pixel SH basis already in shared
//     memory (lane = component);
//   - the other 31 components (centre, rotation, scales and angles of all 8
//     brackets, eta, tau, opacity): lanes write their row to shared memory,
//     lane c sums column c over the group.
// One scalar red.global.add per nonzero component and group.
//
// This translation unit is compiled with --fmad=true.
// the backward keeps the atan2 bracket lookup (pseudo-angle measured +0.9% here,
// -2.6% / -4.7% in the forward on configs 1 / 2)
#ifndef DRK_PSEUDO_ANGLE
#define DRK_PSEUDO_ANGLE 0
#endif
#include "drk_fast.cuh"

#ifndef DRK_BWDF_MINB
#define DRK_BWDF_MINB 1
#endif
// half-tile CTAs (128 threads): resident CTAs per SM the register budget is set for
#ifndef DRK_BWD_MINB128
#define DRK_BWD_MINB128 3  // 168 registers, 12 warps / SM (config 2: 41.8 ms vs 43.4 ms with whole-tile CTAs)
#endif
// 1: warp-group sums read the members' rows / SH weights / basis from shared
// memory (lane = gradient component); 0: register transposes with shuffles
#ifndef DRK_BWD_THRU
#define DRK_BWD_THRU 1  // pop-through fast path (config 2 backward -1%)
#endif
// list entries per staged batch (0: one per thread); the ring holds two.
// Measured, config-2 fwd+bwd: 60.7 ms with one per thread (128), 59.3 ms with
// 64, 59.8 ms with 32 (the smaller ring leaves more L1 to the shape, SH and
// frame records)
#ifndef DRK_BWD_BATCH
#define DRK_BWD_BATCH 64
#endif
#ifndef DRK_BWD_SMEM
#define DRK_BWD_SMEM 0  // measured on config 2: 47.8 ms with 1, 47.0 ms with 0 (groups average 18 lanes)
#endif
// 1: the SH-gradient group sums on the tensor cores (mma.sync tf32, 3 products
// on hi / lo splits; parity green); 0: register transposes with shuffles.
// Measured on config 2 fwd+bwd: 63.3 ms with 1 (padded basis rows, four
// accumulator chains; 63.6 ms with one chain) vs 60.9 ms with 0 — the splits,
// fragment loads and MMA latency cost more than the 47 shuffles they replace.
#ifndef DRK_BWD_MMA
#define DRK_BWD_MMA 0
#endif
namespace drk {

namespace {
constexpr int kGCols = 31;       // non-SH gradient columns
// row stride padding of the per-pixel SH basis [16][NT + pad]: the MMA's A
// fragments read 8 terms x 4 pixels per load (pad 4: 32 distinct banks)
constexpr int kBasisPad = DRK_BWD_SMEM ? 1 : (DRK_BWD_MMA ? 4 : 0);

__device__ __forceinline__ unsigned f32_to_tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// D += A B, m16n8k8, A row-major tf32 (4 regs), B col-major tf32 (2 regs), fp32 accumulators
__device__ __forceinline__ void mma_tf32(float& d0, float& d1, float& d2, float& d3, const unsigned a[4],
                                         const unsigned b[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ int gcol_global(int c) {
  if (c < 12) return c;                   // centre 0..2, rotation 3..11 (row-major)
  if (c < 20) return kGOffSc + (c - 12);  // scales, K == 8
  if (c < 28) return kGOffAn + (c - 20);  // angles
  return c == 28 ? kGOffEta : (c == 29 ? kGOffTau : kGOffOp);
}

// SH colour before the clamp (geometry.cpp:126-138), float4 coefficient loads
template <int BSTRIDE>
__device__ __forceinline__ void sh_colour(const RasterParams& P, const float* s_basis, int id, float& c0, float& c1,
                                          float& c2) {
  const float* shp = P.sh + (size_t)id * P.terms * 3;
  c0 = c1 = c2 = 0.5f;
  const int ta = P.opt.terms_active;
  if ((P.terms & 3) == 0 && (ta & 3) == 0) {
    const float4* q = reinterpret_cast<const float4*>(shp);
#pragma unroll
    for (int t = 0; t < 16; t += 4) {
      if (t < ta) {
        const float4 a = __ldg(q + 3 * (t / 4)), b = __ldg(q + 3 * (t / 4) + 1), c = __ldg(q + 3 * (t / 4) + 2);
        const float b0 = s_basis[t * BSTRIDE], b1 = s_basis[(t + 1) * BSTRIDE], b2 = s_basis[(t + 2) * BSTRIDE],
                    b3 = s_basis[(t + 3) * BSTRIDE];
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
    return;
  }
  for (int t = 0; t < ta; ++t) {
    const float bt = s_basis[t * BSTRIDE];
    c0 = fmaf(bt, __ldg(shp + 3 * t), c0);
    c1 = fmaf(bt, __ldg(shp + 3 * t + 1), c1);
    c2 = fmaf(bt, __ldg(shp + 3 * t + 2), c2);
  }
}

struct BwdPixel {
  float dC0, dC1, dC2, dD, dN0, dN1, dN2, dA;
  double rest;
  bool has_dN;
};

// fp32 gradient of one record (grad.cpp:237-301, backward_alpha grad.cpp:16-101)
// from the fp32 evaluation; writes the 31 non-SH components to row.
__device__ __forceinline__ void record_grad_fast(const RasterParams& P, const BwdPixel& bp, int id, const Geo& g,
                                                 const GradF& gf, float rt, double a, float wbf, float datf,
                                                 float sgn, const float df[3], float* row) {
  float dcen[3] = {0, 0, 0}, drot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  float deta = 0, dtau = 0, dop = 0, ds_lo = 0, ds_hi = 0, da_lo = 0, da_hi = 0;
  int lo = 0, hi = 1;
  const float denf = gf.dz, af = (float)a;
  // reciprocals instead of IEEE divisions (2^-23 relative; the backward's
  // tolerance is 1e-3 relative L2)
  const float iden = rcp_nr(denf);
  const float4* fr = P.frame32 + 3 * (size_t)id;
  const float4 fx = __ldg(fr), fy = __ldg(fr + 1), fz = __ldg(fr + 2);
  const float rzf[3] = {fz.x, fz.y, fz.z};
  float hv[3] = {fx.w + rt * df[0], fy.w + rt * df[1], fz.w + rt * df[2]};
  if (bp.has_dN) {
    drot[2] += wbf * sgn * bp.dN0;
    drot[5] += wbf * sgn * bp.dN1;
    drot[8] += wbf * sgn * bp.dN2;
  }
  if (bp.dD != 0.f) {
    const float d_rt = wbf * bp.dD;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      dcen[q] += d_rt * rzf[q] * iden;
      drot[3 * q + 2] += d_rt * (-hv[q] * iden);
    }
  }
  if (a < 1.0 - 1e-6 - 1e-12) {  // alpha not clamped
    const float o = (float)P.S.o[id];
    if (gf.lp) {
      const float cv = fabsf(denf), sl = (float)P.opt.lowpass_radius;
      const float dpwf = gf.dpx, dphf = gf.dpy;  // pixel - projected centre
      dop += datf * af * rcp_nr(o);
      const float inv = rcp_nr(cv * cv * sl * sl);
      const float d_dpw = datf * af * (-dpwf * inv), d_dph = datf * af * (-dphf * inv);
      const float d_cos = datf * af * (dpwf * dpwf + dphf * dphf) * inv * rcp_nr(cv);
      double J[6];
      projection_jacobian(P.cam, g.mu, J);
      const float sg = denf < 0 ? -1.0f : 1.0f;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        dcen[q] += -((float)J[q] * d_dpw + (float)J[3 + q] * d_dph);
        drot[3 * q + 2] += d_cos * sg * df[q];
      }
    } else {
      const KEvalF& k = gf.k;
      const float tau = (float)P.S.tau[id];
      dop += datf * k.P;
      if (!k.center) {
        const float tp = k.br == 1 ? 1.0f - tau : 1.0f + tau;
        dtau += datf * o *
                (k.br == 0 ? -2.0f * k.g : (k.br == 1 ? 2.0f * k.g - 1.0f : 2.0f - 2.0f * k.g)) * rcp_nr(tp * tp);
        if (!k.clamped) {
          lo = k.lo;
          hi = k.hi;
          const float* br = P.shrec + (size_t)kRecStride * id + kRecHdr + 8 * lo;
          const float4 e = __ldg(reinterpret_cast<const float4*>(br));
          const float4 f = __ldg(reinterpret_cast<const float4*>(br) + 1);  // 1/det, pi/gap, h_lo, h_hi
          const float elx = e.x, ely = e.y, ehx = e.z, ehy = e.w, invd = f.x, piog = f.y, hlo = f.z, hhi = f.w;
          const float slo = rsqrtf(hlo), shi = rsqrtf(hhi);
          const float islo = hlo * slo, ishi = hhi * shi;  // 1 / s_lo, 1 / s_hi
          const float eta = __ldg(P.shrec + (size_t)kRecStride * id + 16);
          const float r2f = gf.r2;
          const float d_q = datf * o * k.A * (-0.5f * k.g);
          deta += d_q * (k.r1 * k.r1 - r2f * k.inv);
          const float d_r1 = d_q * eta * 2.0f * k.r1;
          const float d_r2sq = d_q * (1.0f - eta) * k.inv;
          const float d_inv = d_q * (1.0f - eta) * r2f;
          ds_lo = d_inv * (-2.0f * k.ch * k.ch * hlo * islo);
          ds_hi = d_inv * (-2.0f * k.sh * k.sh * hhi * ishi);
          const float d_delta = -(d_inv * 0.5f * (hlo - hhi)) * (2.0f * k.sh * k.ch);
          const float d_tfd = d_delta * piog;
          const float dl = k.delta * (float)(1.0 / kPi);
          da_lo = d_tfd * (dl - 1.0f);
          da_hi = -d_tfd * dl;
          const float uf = gf.u, vf = gf.v, ir2s = rcp_nr(fmaxf(r2f, 1e-24f));
          const float sa = k.a > 0.f ? 1.f : (k.a < 0.f ? -1.f : 0.f);
          const float sb = k.b > 0.f ? 1.f : (k.b < 0.f ? -1.f : 0.f);
          const float du = d_tfd * (-vf * ir2s) + 2.0f * d_r2sq * uf + d_r1 * (sa * ehy - sb * ely) * invd;
          const float dv = d_tfd * (uf * ir2s) + 2.0f * d_r2sq * vf + d_r1 * (sb * elx - sa * ehx) * invd;
          ds_lo += d_r1 * (-sa * k.a * islo);
          ds_hi += d_r1 * (-sb * k.b * ishi);
          const float cross = ehy * ely + ehx * elx;
          da_lo += d_r1 * invd * (sa * k.a * cross - sb * k.a * slo * slo);
          da_hi += d_r1 * invd * (sa * k.b * shi * shi - sb * k.b * cross);
          // (u, v) and r_t chain to centre and rotation columns (grad.cpp:290-300)
          const float rxf[3] = {fx.x, fx.y, fx.z};
          const float ryf[3] = {fy.x, fy.y, fy.z};
          const float drx = df[0] * rxf[0] + df[1] * rxf[1] + df[2] * rxf[2];
          const float dry = df[0] * ryf[0] + df[1] * ryf[1] + df[2] * ryf[2];
          const float fq = -(du * drx + dv * dry) * iden;
          const float drxd = drx * iden, dryd = dry * iden;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            dcen[q] += du * (rzf[q] * drxd - rxf[q]) + dv * (rzf[q] * dryd - ryf[q]);
            drot[3 * q + 0] += du * hv[q];
            drot[3 * q + 1] += dv * hv[q];
            drot[3 * q + 2] += fq * hv[q];
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) row[q] = dcen[q];
#pragma unroll
  for (int q = 0; q < 9; ++q) row[3 + q] = drot[q];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    row[12 + q] = (q == lo ? ds_lo : 0.f) + (q == hi ? ds_hi : 0.f);
    row[20 + q] = (q == lo ? da_lo : 0.f) + (q == hi ? da_hi : 0.f);
  }
  row[28] = deta;
  row[29] = dtau;
  row[30] = dop;
}

// fp64 gradient of one record whose alpha was evaluated in fp64 (reference
// formulation, grad.cpp:237-301, :16-101).
__device__ __noinline__ void record_grad_f64(const RasterParams& P, const BwdPixel& bp, int id, const Geo& g,
                                             const Pop64& o64, double a, double wb, double dat, const double* dir,
                                             float* row) {
  const int K = P.S.K;
  const double rt = o64.rt, denom = o64.denom, u = o64.u, v = o64.v;
  const KEval& ev = o64.ev;
  double dcen[3] = {0, 0, 0}, drot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double deta = 0, dtau = 0, dop = 0, ds_lo = 0, ds_hi = 0, da_lo = 0, da_hi = 0;
  int lo = 0, hi = 1;
  const double sgn = denom < 0 ? 1.0 : -1.0;
  const double rz[3] = {g.rz[0], g.rz[1], g.rz[2]};
  if (bp.has_dN) {
    drot[2] += wb * sgn * bp.dN0;
    drot[5] += wb * sgn * bp.dN1;
    drot[8] += wb * sgn * bp.dN2;
  }
  if (bp.dD != 0.f) {
    const double d_rt = wb * bp.dD;
    for (int q = 0; q < 3; ++q) {
      const double h = P.cam.o[q] + rt * dir[q] - g.mu[q];
      dcen[q] += d_rt * rz[q] / denom;
      drot[3 * q + 2] += d_rt * (-h / denom);
    }
  }
  const bool alpha_clamped = a >= 1.0 - 1e-6 - 1e-12;
  const double o = P.S.o[id];
  if (!alpha_clamped && o64.lp) {
    const double cv = fabs(denom), sl = P.opt.lowpass_radius;
    dop += dat * a / o;
    const double inv = 1.0 / (cv * cv * sl * sl);
    const double d_dpw = dat * a * (-o64.dpw * inv);
    const double d_dph = dat * a * (-o64.dph * inv);
    const double d_cos = dat * a * (o64.dpw * o64.dpw + o64.dph * o64.dph) * inv / cv;
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
  for (int q = 0; q < 3; ++q) row[q] = (float)dcen[q];
  for (int q = 0; q < 9; ++q) row[3 + q] = (float)drot[q];
  for (int q = 0; q < 8; ++q) {
    row[12 + q] = (q == lo ? (float)ds_lo : 0.f) + (q == hi ? (float)ds_hi : 0.f);
    row[20 + q] = (q == lo ? (float)da_lo : 0.f) + (q == hi ? (float)da_hi : 0.f);
  }
  row[28] = (float)deta;
  row[29] = (float)dtau;
  row[30] = (float)dop;
}
}  // namespace

// NT threads per CTA: 256 = a 16x16 tile, 128 = half a tile (8 x 16 pixels;
// long tile lists), as in the fast forward.
// DET: deterministic mode — each composited record writes its own gradient row
// (det_row) instead of the warp-group reduction and atomics.
template <int NT, bool DET>
__global__ void __launch_bounds__(NT, NT == 128 ? DRK_BWD_MINB128 : DRK_BWDF_MINB) k_raster_bwd_fast(
    const __grid_constant__ RasterParams P) {
  constexpr int BATCH = DRK_BWD_BATCH > 0 && DRK_BWD_BATCH < NT ? DRK_BWD_BATCH : NT;  // entries per staged batch
  constexpr int RING = 2 * BATCH;
  extern __shared__ float4 dyn[];
  Rec* ring = reinterpret_cast<Rec*>(dyn);
  int* s_id = reinterpret_cast<int*>(ring + RING);
  // per-pixel SH basis [16][BS]; BS = NT + 1 so that one pixel's 16 terms sit in
  // distinct banks (the shared-memory group sums read them across lanes)
  constexpr int BS = NT + kBasisPad;
  float* s_basis_all = reinterpret_cast<float*>(s_id + RING);  // [16][BS]
  float* s_w_all = s_basis_all + 16 * BS;                     // [NT][4]: SH weights per lane
  float* s_row = s_w_all + 4 * NT;                            // [NT][kGCols]: gradient rows (odd stride: no bank conflicts)
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  float* s_basis = s_basis_all + threadIdx.x;
  float* s_w = s_w_all + 4 * threadIdx.x;
  __shared__ unsigned s_ddmax;
  __shared__ TileConst tc;
  const int cta_tile = NT == 256 ? blockIdx.x : blockIdx.x >> 1;
  const int tile = P.tile_base + (P.tile_order ? P.tile_order[cta_tile] : cta_tile);
  const int tx = tile % P.cam.tiles_x, ty = tile / P.cam.tiles_x;
  const int half = NT == 256 ? ((threadIdx.x >> 5) & 1) : (int)(blockIdx.x & 1);
  const int x = tx * kTile + half * 8 + (threadIdx.x & 7),
            y = ty * kTile + (NT == 256 ? (threadIdx.x >> 6) : (threadIdx.x >> 5)) * 4 + ((threadIdx.x & 31) >> 3);  // 8 x 4 per warp
  bool active = x < P.cam.W && y < P.cam.H;
  if (active && P.pxflag && P.pxflag[(size_t)y * P.cam.W + x]) active = false;  // fp64 backward owns flagged pixels
  if (__syncthreads_count(active) == 0) return;
  const double tx0 = (double)tx * kTile, ty0 = (double)ty * kTile;
  double d0[3], dir[3];
  pixel_dir(P.cam, tx0 + 8.0, ty0 + 8.0, d0);
  pixel_dir(P.cam, x + 0.5, y + 0.5, dir);
  const float df[3] = {(float)dir[0], (float)dir[1], (float)dir[2]};
  FastPixel px;
  px.ddx = (float)(dir[0] - d0[0]);
  px.ddy = (float)(dir[1] - d0[1]);
  px.ddz = (float)(dir[2] - d0[2]);
  px.pxr = (float)(x + 0.5 - tx0);
  px.pyr = (float)(y + 0.5 - ty0);
  {
    float b[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) b[t] = 0.f;
    sh_basis_f(df[0], df[1], df[2], P.opt.sh_degree, b);
#pragma unroll
    for (int t = 0; t < 16; ++t) s_basis[t * BS] = b[t];
  }
#if !DRK_BWD_SMEM
  float bas[16];  // this pixel's SH basis, zero beyond the active terms (SH gradient columns)
  {
    const int ta = P.opt.terms_active;
#pragma unroll
    for (int t = 0; t < 16; ++t) bas[t] = t < ta ? s_basis[t * BS] : 0.f;
  }
#endif
  if (threadIdx.x == 0) {
    s_ddmax = 0u;
    tc.d0[0] = d0[0];
    tc.d0[1] = d0[1];
    tc.d0[2] = d0[2];
    tc.tx0 = tx0;
    tc.ty0 = ty0;
  }
  __syncthreads();
  {
    const float m = fmaxf(fabsf(px.ddx), fmaxf(fabsf(px.ddy), fabsf(px.ddz)));
    const unsigned wm = __reduce_max_sync(FULL, __float_as_uint(m));
    if (lane == 0) atomicMax(&s_ddmax, wm);
  }
  // upstream gradients and rest (grad.cpp:198-222)
  const size_t pix = (size_t)y * P.cam.W + x;
  BwdPixel bp;
  bp.dC0 = bp.dC1 = bp.dC2 = bp.dD = bp.dN0 = bp.dN1 = bp.dN2 = bp.dA = 0.f;
  bp.rest = 0;
  bp.has_dN = P.dN != nullptr;
  int stop = 0;
  if (active) {
    if (P.dC) {
      bp.dC0 = P.dC[3 * pix];
      bp.dC1 = P.dC[3 * pix + 1];
      bp.dC2 = P.dC[3 * pix + 2];
    }
    if (P.dD) bp.dD = P.dD[pix];
    if (P.dN) {
      bp.dN0 = P.dN[3 * pix];
      bp.dN1 = P.dN[3 * pix + 1];
      bp.dN2 = P.dN[3 * pix + 2];
    }
    if (P.dA) bp.dA = P.dA[pix];
    const double* st = P.pxstate + 8 * pix;
    bp.rest = ((double)bp.dC0 * st[0] + (double)bp.dC1 * st[1] + (double)bp.dC2 * st[2]) + (double)bp.dD * st[3] +
              ((double)bp.dN0 * st[4] + (double)bp.dN1 * st[5] + (double)bp.dN2 * st[6]) + (double)bp.dA * st[7];
    stop = P.pxstop[pix];
  }
  px.T = 1.0;
  px.ncomp = 0;
  px.n_pop = px.n_rej1 = px.n_rej2 = px.n_f64 = px.n_miss = 0;
  px.err = false;
  unsigned n_steps = 0, n_groups = 0;
  float clo[kCacheCap], chi[kCacheCap];
  int cj[kCacheCap];
#pragma unroll
  for (int q = 0; q < kCacheCap; ++q) {
    clo[q] = chi[q] = __int_as_float(0x7f800000);
    cj[q] = 0;
  }
  int csz = 0;
  bool done = !active || stop <= 0;
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  const float eps = (float)P.opt.grazing_eps;
  __syncthreads();
  if (threadIdx.x == 0) tc.ddmax = __uint_as_float(s_ddmax) * 1.0001f + 1e-30f;
  int ring_lo = 0;
  const int G = P.G;

  // One warp-cooperative pop step: lanes with want pop entry pj.
  auto pop_step = [&](bool want, int pj) {
    bool rec = false;
    int id = -1;
    float w0 = 0.f, w1 = 0.f, w2 = 0.f;
    long long det_r = -1;
    float* row = s_row + kGCols * threadIdx.x;
    if (want) {
      Rec R;
      if (pj >= ring_lo) {
        const int slot = pj & (RING - 1);
        R = ring[slot];
        id = s_id[slot];
      } else {
        id = P.lid[beg + pj];
        stage_record(P, id, tc, R);
      }
      AlphaOut o;
      GradF gf;
      Pop64 o64;  // fp64 evaluation (rare); kept apart so gf stays in registers
      alpha_entry<false, true>(P, px, R, id, x, y, o, &gf, &o64);
      if (o.degen) {
        px.err = true;
        done = true;
      } else if (!o.skip) {
        rec = true;
        const double a = o.a;
        // colour (geometry.cpp:126-138) with the clamp, upstream scalars (grad.cpp:224-233)
        float c0, c1, c2;
        sh_colour<BS>(P, s_basis, id, c0, c1, c2);
        const bool cl0 = c0 < 0.f, cl1 = c1 < 0.f, cl2 = c2 < 0.f;
        const float r0 = cl0 ? 0.f : c0, r1 = cl1 ? 0.f : c1, r2 = cl2 ? 0.f : c2;
        const double wb = px.T * a;
        const float rzx = R.r0.x, rzy = R.r0.y, rzz = R.r0.z;
        const double cw = ((double)(bp.dC0 * r0) + (double)(bp.dC1 * r1) + (double)(bp.dC2 * r2)) +
                          (double)(bp.dD * o.rt) +
                          (double)(o.sgn * (bp.dN0 * rzx + bp.dN1 * rzy + bp.dN2 * rzz)) + (double)bp.dA;
        bp.rest -= wb * cw;
        const double dat = px.T * cw - bp.rest / (1.0 - a);
        const float wbf = (float)wb;
        w0 = cl0 ? 0.f : wbf * bp.dC0;
        w1 = cl1 ? 0.f : wbf * bp.dC1;
        w2 = cl2 ? 0.f : wbf * bp.dC2;
        const Geo& g = P.geo[id];
        if (!gf.f64) {
          record_grad_fast(P, bp, id, g, gf, o.rt, a, wbf, (float)dat, o.sgn, df, row);
        } else {
          double dd[3];
          pixel_dir(P.cam, x + 0.5, y + 0.5, dd);
          record_grad_f64(P, bp, id, g, o64, a, wb, dat, dd, row);
        }
        P.touched[id] = 1;
        if (DET) det_r = det_row(P, x, y, px.ncomp, id);  // the row is written by the warp below
        px.T = xm(px.T, xs(1.0, a));
        ++px.ncomp;
        if (px.ncomp >= stop) done = true;
      }
    }
    s_w[0] = w0;
    s_w[1] = w1;
    s_w[2] = w2;
    if (DET) {
      // deterministic mode: each record's whole row (zeros included) to its slot,
      // written by the warp 32 columns per store (coalesced)
      const unsigned wm = __ballot_sync(FULL, rec && det_r >= 0);
      __syncwarp();
      const int wbase = threadIdx.x & ~31;
      const int ta = P.opt.terms_active;
      for (unsigned mm = wm; mm; mm &= mm - 1u) {
        const int m = __ffs(mm) - 1;
        const long long r = __shfl_sync(FULL, det_r, m);
        const int tm = wbase + m;
        const float* rw = s_row + kGCols * tm;
        float* dst = P.det_rec32 + (size_t)r * G;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int c = 32 * q + lane;
          if (c >= G) continue;
          float val = 0.f;
          if (c < 12) val = rw[c];
          else if (c < kGOffAn) val = c - kGOffSc < 8 ? rw[12 + c - kGOffSc] : 0.f;
          else if (c < kGOffEta) val = c - kGOffAn < 8 ? rw[20 + c - kGOffAn] : 0.f;
          else if (c < kGOffSh) val = rw[28 + c - kGOffEta];
          else {
            const int k = c - kGOffSh, t = k / 3, ch = k - 3 * t;
            if (t < ta) val = s_w_all[4 * tm + ch] * s_basis_all[t * BS + tm];
          }
          dst[c] = val;
        }
      }
      __syncwarp();
      return;
    }
    const unsigned recmask = __ballot_sync(FULL, rec);
    if (!recmask) return;
    ++n_steps;
    __syncwarp();
    unsigned remaining = recmask;
    while (remaining) {
      const int lead = __ffs(remaining) - 1;
      const int gid = __shfl_sync(FULL, id, lead);
      const unsigned gm = __ballot_sync(FULL, rec && id == gid) & remaining;
      remaining &= ~gm;
      ++n_groups;
      float* pg = P.gact + (size_t)gid * G;
#if DRK_BWD_SMEM
      {
        // lane = component: non-SH column `lane` (< 31), SH components lane and
        // 32 + lane (k = 3 t + ch: w_ch basis_t of each member pixel)
        const int wbase = threadIdx.x & ~31;
        const int ta = P.opt.terms_active;
        const int t1 = lane / 3, c1 = lane - 3 * t1, t2 = (32 + lane) / 3, c2 = 32 + lane - 3 * t2;
        const bool v1 = t1 < ta, v2 = lane < 16 && t2 < ta;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
        for (unsigned mm = gm; mm; mm &= mm - 1u) {
          const int tm = wbase + __ffs(mm) - 1;
          if (lane < kGCols) a0 += s_row[kGCols * tm + lane];
          if (v1) a1 = fmaf(s_w_all[4 * tm + c1], s_basis_all[t1 * BS + tm], a1);
          if (v2) a2 = fmaf(s_w_all[4 * tm + c2], s_basis_all[t2 * BS + tm], a2);
        }
        if (lane < kGCols && a0 != 0.f) atomicAdd(pg + gcol_global(lane), a0);
        if (v1 && a1 != 0.f) atomicAdd(pg + kGOffSh + lane, a1);
        if (v2 && a2 != 0.f) atomicAdd(pg + kGOffSh + 32 + lane, a2);
      }
#else
      // non-SH columns: transpose-reduce (5 halving steps, 31 shuffles) leaves
      // lane c with the group sum of column c
      {
        const bool in_g = (gm >> lane) & 1u;
        float xv[32];
#pragma unroll
        for (int i = 0; i < kGCols; ++i) xv[i] = in_g ? row[i] : 0.f;  // row written this step by in_g lanes
        xv[31] = 0.f;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < off; ++i) {
            const float send = up ? xv[i] : xv[i + off];
            const float keep = up ? xv[i + off] : xv[i];
            xv[i] = keep + __shfl_xor_sync(FULL, send, off);
          }
        }
        if (lane < kGCols && xv[0] != 0.f) atomicAdd(pg + gcol_global(lane), xv[0]);
      }
#if DRK_BWD_MMA
      // SH: d sh[t][c] = sum over the group's lanes k of basis_t(k) w_c(k), a
      // [16 x 32] x [32 x 3] product on the tensor cores (mma.sync m16n8k8
      // tf32, four k-chunks of 8 lanes; three products per chunk on hi / lo
      // tf32 splits for fp32-level accuracy).  A = the pixels' basis (shared
      // memory), B = the members' SH weights (s_w, zero outside the group);
      // lane (g, tig) ends with D[g (+8)][2 tig (+1)].
      {
        const int wbase = threadIdx.x & ~31;
        const int ta = P.opt.terms_active;
        const int g = lane >> 2, tig = lane & 3;
        // one accumulator set per k-chunk: four independent MMA chains of three
        float dk[4][4];
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) dk[kc][0] = dk[kc][1] = dk[kc][2] = dk[kc][3] = 0.f;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const int k0 = kc * 8 + tig, k1 = k0 + 4;
          float a[4] = {s_basis_all[g * BS + wbase + k0], s_basis_all[(g + 8) * BS + wbase + k0],
                        s_basis_all[g * BS + wbase + k1], s_basis_all[(g + 8) * BS + wbase + k1]};
          float b[2] = {g < 3 && ((gm >> k0) & 1u) ? s_w_all[4 * (wbase + k0) + g] : 0.f,
                        g < 3 && ((gm >> k1) & 1u) ? s_w_all[4 * (wbase + k1) + g] : 0.f};
          unsigned ah[4], al[4], bh[2], bl[2];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            ah[i] = f32_to_tf32(a[i]);
            al[i] = f32_to_tf32(a[i] - __uint_as_float(ah[i]));
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            bh[i] = f32_to_tf32(b[i]);
            bl[i] = f32_to_tf32(b[i] - __uint_as_float(bh[i]));
          }
          mma_tf32(dk[kc][0], dk[kc][1], dk[kc][2], dk[kc][3], al, bh);
          mma_tf32(dk[kc][0], dk[kc][1], dk[kc][2], dk[kc][3], ah, bl);
          mma_tf32(dk[kc][0], dk[kc][1], dk[kc][2], dk[kc][3], ah, bh);
        }
        const float d0 = (dk[0][0] + dk[1][0]) + (dk[2][0] + dk[3][0]);
        const float d1 = (dk[0][1] + dk[1][1]) + (dk[2][1] + dk[3][1]);
        const float d2 = (dk[0][2] + dk[1][2]) + (dk[2][2] + dk[3][2]);
        const float d3 = (dk[0][3] + dk[1][3]) + (dk[2][3] + dk[3][3]);
        float* psh = pg + kGOffSh;
        const int c0 = 2 * tig;
        if (c0 < 3) {
          if (g < ta && d0 != 0.f) atomicAdd(psh + 3 * g + c0, d0);
          if (g + 8 < ta && d2 != 0.f) atomicAdd(psh + 3 * (g + 8) + c0, d2);
        }
        if (c0 + 1 < 3) {
          if (g < ta && d1 != 0.f) atomicAdd(psh + 3 * g + c0 + 1, d1);
          if (g + 8 < ta && d3 != 0.f) atomicAdd(psh + 3 * (g + 8) + c0 + 1, d3);
        }
      }
#else
      // SH: component k = 3 t + ch (t < 16), value w_ch basis_t(pixel):
      // k = 0..31 by a 32-wide transpose, k = 32..47 by a 16-value halving
      // transpose (16 shuffles) that leaves value v in lanes 2v and 2v + 1
      {
        const bool ing = (gm >> lane) & 1u;
        const float m0 = ing ? w0 : 0.f, m1 = ing ? w1 : 0.f, m2 = ing ? w2 : 0.f;
        {
          float xv[32];
#pragma unroll
          for (int i2 = 0; i2 < 32; ++i2) {
            const int ch = i2 % 3;
            xv[i2] = (ch == 0 ? m0 : (ch == 1 ? m1 : m2)) * bas[i2 / 3];
          }
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i2 = 0; i2 < off; ++i2) {
              const float send = up ? xv[i2] : xv[i2 + off];
              const float keep = up ? xv[i2 + off] : xv[i2];
              xv[i2] = keep + __shfl_xor_sync(FULL, send, off);
            }
          }
          if (xv[0] != 0.f) atomicAdd(pg + kGOffSh + lane, xv[0]);
        }
        {
          float xv[16];
#pragma unroll
          for (int i2 = 0; i2 < 16; ++i2) {
            const int k = 32 + i2, ch = k % 3;
            xv[i2] = (ch == 0 ? m0 : (ch == 1 ? m1 : m2)) * bas[k / 3];
          }
#pragma unroll
          for (int off = 16, h = 8; off >= 2; off >>= 1, h >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i2 = 0; i2 < h; ++i2) {
              const float send = up ? xv[i2] : xv[i2 + h];
              const float keep = up ? xv[i2 + h] : xv[i2];
              xv[i2] = keep + __shfl_xor_sync(FULL, send, off);
            }
          }
          xv[0] += __shfl_xor_sync(FULL, xv[0], 1);
          if (!(lane & 1) && xv[0] != 0.f) atomicAdd(pg + kGOffSh + 32 + (lane >> 1), xv[0]);
        }
      }
#endif  // DRK_BWD_MMA
#endif
    }
    __syncwarp();
  };

  for (long long b0 = beg; b0 < end; b0 += BATCH) {
    const int jb = (int)(b0 - beg);
    __syncthreads();
    {
      const long long j = b0 + threadIdx.x;
      if ((int)threadIdx.x < BATCH && j < end) {
        const int id = P.lid[j];
        const int slot = (jb + threadIdx.x) & (RING - 1);
        stage_record(P, id, tc, ring[slot]);
        s_id[slot] = id;
      }
    }
    __syncthreads();
    ring_lo = jb >= BATCH ? jb - BATCH : 0;
    const int cnt = (int)min((long long)BATCH, end - b0);
    if (__any_sync(FULL, !done)) {
      for (int c = 0; c < cnt; ++c) {
        bool want = false;
        int pj = 0;
        if (!done) {
          const int jr = jb + c;
          const int slot = jr & (RING - 1);
          const float4 r0 = ring[slot].r0;
          const float2 r3 = *reinterpret_cast<const float2*>(&ring[slot].r3);
          const float dz = lin3(r0, ring[slot].r5.x, px.ddx, px.ddy, px.ddz);
          const float adz = fabsf(dz);
          bool hit = false;
          float lo = 0.f, hi = 0.f;
          if (!(adz < eps - r3.y)) {
            const float inv = rcp_nr(dz);
            const float rel_z = r3.y * fabsf(inv);
            if (adz > eps + r3.y && r3.x != 0.f && rel_z <= 1e-3f) {
              const float rt = r3.x * inv;
              if (rt > 0.f) {
                hit = true;
                const float er = rt * (3.3e-7f + rel_z * 1.01f);
                lo = rt - er;
                hi = rt + er;
              }
            } else {
              double rx;
              if (exact_rt(P, s_id[slot], x, y, &rx)) {
                hit = true;
                lo = __double2float_rd(rx);
                hi = __double2float_ru(rx);
              }
            }
          }
          if (hit && DRK_BWD_THRU && csz == kCacheCap && hi < clo[0]) {
            // certainly shallower than the head: pops through, cache unchanged
            want = true;
            pj = jr;
          } else if (hit) {
            bool le[kCacheCap];
            bool amb = false;
#pragma unroll
            for (int q = 0; q < kCacheCap; ++q) {
              le[q] = chi[q] <= lo;
              amb |= !le[q] && !(clo[q] > hi);
            }
            if (amb) {
              double rin = 0;
              exact_rt(P, s_id[slot], x, y, &rin);
              lo = __double2float_rd(rin);
              hi = __double2float_ru(rin);
#pragma unroll
              for (int q = 0; q < kCacheCap; ++q) {
                if (!le[q]) {
                  if (chi[q] <= lo) {
                    le[q] = true;
                  } else if (!(clo[q] > hi)) {
                    double rq = 0;
                    exact_rt(P, entry_id<RING>(P, s_id, beg, cj[q], ring_lo), x, y, &rq);
                    le[q] = rq <= rin;
                    clo[q] = __double2float_rd(rq);
                    chi[q] = __double2float_ru(rq);
                  }
                }
              }
            }
            if (csz < kCacheCap) {
#pragma unroll
              for (int q = kCacheCap - 1; q >= 0; --q) {
                const bool prev = q == 0 ? true : le[q - 1];
                if (!le[q]) {
                  clo[q] = prev ? lo : clo[q - 1];
                  chi[q] = prev ? hi : chi[q - 1];
                  cj[q] = prev ? jr : cj[q - 1];
                }
              }
              ++csz;
            } else {
              want = true;
              if (!le[0]) {
                pj = jr;
              } else {
                pj = cj[0];
#pragma unroll
                for (int q = 0; q < kCacheCap; ++q) {
                  const bool nxt = q + 1 < kCacheCap ? le[q + 1] : false;
                  if (nxt) {
                    clo[q] = clo[q + 1];
                    chi[q] = chi[q + 1];
                    cj[q] = cj[q + 1];
                  } else if (le[q]) {
                    clo[q] = lo;
                    chi[q] = hi;
                    cj[q] = jr;
                  }
                }
              }
            }
          }
        }
        if (__any_sync(FULL, want)) pop_step(want, pj);
      }
    }
    if (__syncthreads_count(!done) == 0) break;
  }
  // end marker: drain the cache head (raster.cpp:410-414), warp-uniform rounds
  for (int r = 0; r < kCacheCap; ++r) {
    const bool want = !done && csz > 0;
    if (!__any_sync(FULL, want)) break;
    int pj = 0;
    if (want) {
      pj = cj[0];
#pragma unroll
      for (int q = 0; q < kCacheCap - 1; ++q) {
        clo[q] = clo[q + 1];
        chi[q] = chi[q + 1];
        cj[q] = cj[q + 1];
      }
      --csz;
    }
    pop_step(want, pj);
  }
  if (active && px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  if (lane == 0) {
    if (n_steps) atomicAdd(&P.counters[C_BWD_WARPSTEPS], (unsigned long long)n_steps);
    if (n_groups) atomicAdd(&P.counters[C_BWD_LEAD_RECORDS], (unsigned long long)n_groups);
  }
}

size_t raster_bwd_fast_smem(int nt) {
  const int batch = DRK_BWD_BATCH > 0 && DRK_BWD_BATCH < nt ? DRK_BWD_BATCH : nt;
  return (size_t)2 * batch * (sizeof(Rec) + sizeof(int)) + (16 * (nt + kBasisPad) + (4 + kGCols) * nt) * sizeof(float);
}

template <int NT, bool DET>
static void launch_bwd_nt(const RasterParams& P, int n_tiles, cudaStream_t s) {
  const size_t smem = raster_bwd_fast_smem(NT);
  static PerDeviceOnce attr;
  attr([&] { cudaFuncSetAttribute(k_raster_bwd_fast<NT, DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  k_raster_bwd_fast<NT, DET><<<n_tiles * (256 / NT), NT, smem, s>>>(P);
}

void launch_raster_bwd_fast(const RasterParams& P, int n_tiles, cudaStream_t s) {
  if (P.fast_nt == 128) launch_bwd_nt<128, false>(P, n_tiles, s);
  else launch_bwd_nt<256, false>(P, n_tiles, s);
}

void launch_raster_bwd_fast_det(const RasterParams& P, int n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return;
  launch_counter() += 1;
  // half-tile CTAs as in the atomic backward (config 2 record raster -11%); DRK_DET_NT=256: whole tiles
  static const int det_nt = getenv("DRK_DET_NT") ? atoi(getenv("DRK_DET_NT")) : 128;
  if (det_nt == 128) launch_bwd_nt<128, true>(P, n_tiles, s);
  else launch_bwd_nt<256, true>(P, n_tiles, s);
}

}  // namespace drk
