// K4 fast path: forward rasterizer for the SortCache mode (reference
// raster.cpp:267-430) with every per-candidate quantity in fp32 and exact
// fp64 fallbacks wherever a discrete decision falls inside its error bound.
//
// One CTA per 16x16 tile (or per half tile for long lists), one thread per
// pixel.  Tile-list entries are staged DRK_BATCH256 / DRK_BATCH128 at a time
// into a two-batch shared-memory ring (the current and the previous batch) as
// a 96-byte fp32 record computed once per (entry, tile) in fp64 (stage_record):
//
//   r0 = (R_z, R_z . d0)                     ray-plane denominator at the tile ray d0
//   r1 = (G_u, N_u(d0)), r2 = (G_v, N_v(d0)) tangent-coordinate numerators
//   r3 = (num, e_z, e_N, r2max)              r_t numerator and error scales
//   r4 = (projected centre - tile origin, dp2max, f_vis^2)
//
// With a = o - mu and the primitive frame (R_x, R_y, R_z), the reference's
// r_t = num / (d . R_z) and (u, v) = R_{x,y} . (a + r_t d) (geometry.cpp:40-52)
// are u = N_u(d) / (d . R_z), v = N_v(d) / (d . R_z) with
// N_u(d) = (R_x . a)(R_z . d) - (R_z . a)(R_x . d) linear in d.  Expanding
// around the tile ray d0 (d = d0 + dd, |dd| <= ~8 px / f) leaves the
// cancellation in the fp64 staging and gives u, v, r_t with ~1e-7 relative
// error from 9 FMAs and one reciprocal per (pixel, candidate).
//
// The SortCache holds fp32 depth intervals [lo, hi] that contain the exact
// fp64 r_t; a comparison whose intervals overlap is resolved exactly
// (exact_rt: the reference's op order in fp64), so the pop sequence is the
// reference's.  The grazing / behind tests are exact the same way.  Alpha
// (core.cpp:148-265) is evaluated in fp32 with a relative error bound that
// includes the tangent-coordinate error; alpha_min / low-pass / clamp
// decisions inside the bound are re-evaluated in fp64 (pop_f64), and pixels
// whose early-stop decision falls inside the accumulated transmittance bound
// are flagged for the fp64 re-render (k_raster_pixels_warp), as in k_raster.
//
// This translation unit is compiled with --fmad=true; the exact fp64 paths use
// explicitly rounded intrinsics (__dmul_rn / __dadd_rn).
#include "drk_fast.cuh"

// 1: the next batch's Geo records are gathered into shared memory with
// cp.async.bulk (one 160-byte bulk copy per entry, completion on an mbarrier)
// while the current batch streams; 0: synchronous loads at staging time.
#ifndef DRK_TMA_STAGE
#define DRK_TMA_STAGE 1
#endif
// 1: the streaming loop takes two candidates per iteration (both intersections,
// then both cache steps): independent instructions for the scheduler
#ifndef DRK_ISECT2
#define DRK_ISECT2 0
#endif
// 1: SortCache steps whose incoming entry is certainly deeper than the whole
// (full) cache take a branch-free shift (no per-entry compares / selects)
#ifndef DRK_CACHE_FAST
#define DRK_CACHE_FAST 0
#endif
#ifndef DRK_POP_THRU
#define DRK_POP_THRU -1  // -1: half-tile CTAs only (long lists); 0: off; 1: always
#endif
// 1: a barrier at the top of every batch (0: the previous batch's closing
// __syncthreads_count already orders the ring reuse; measured +0.6% raster time)
#ifndef DRK_TOP_BARRIER
#define DRK_TOP_BARRIER 1
#endif
// list entries per staged batch (the ring holds two) of the whole-tile and the
// half-tile kernel: one per thread, or fewer for less shared memory (more L1
// for the shape and SH records) at more batch barriers.  Measured: whole-tile
// 256 -> 128 entries, config-1 raster 19.73 -> 19.60 ms (64: 20.18 ms);
// half-tile 128 -> 64 entries, config-2 raster 10.96 -> 10.82 ms, config 3
// 34.4 -> 34.0 ms (32: config 2 11.1 ms, config 3 34.7 ms).
#ifndef DRK_BATCH256
#define DRK_BATCH256 128
#endif
#ifndef DRK_BATCH128
#define DRK_BATCH128 64
#endif
#ifndef DRK_THRU_STAT
#define DRK_THRU_STAT 0
#endif


namespace drk {

// ---------------------------------------------------------------------------
// Per-primitive fp32 shape record (view independent, K == 8), AoS:
//   [0, 8)   theta_k
//   [8, 12)  sharpen point-slope constants (g1, g2, A0, A1)
//   [12, 16) (A2, Psi(g1), Psi(g2), opacity)
//   [16]     eta
//   [17, 24) pseudo-angles of theta_0..theta_6 (pseudo_angle)
//   [24 + 8k, 32 + 8k) bracket (k, k+1 mod K): e_lo (x, y), e_hi (x, y),
//            1/det (NaN when |det| < 1e-12, core.cpp:191), pi/gap, 1/s_lo^2, 1/s_hi^2
// ---------------------------------------------------------------------------
__global__ void k_shape_rec(int i0, int i1, ShapeView S, float* __restrict__ rec) {
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const int K = 8;
  float* r = rec + (size_t)kRecStride * i;
  const size_t b = (size_t)K * i;
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = (float)S.th[b + k];
  const float* q = S.psif + 12 * (size_t)i;
#pragma unroll
  for (int k = 0; k < 8; ++k) r[8 + k] = q[k];
  r[16] = (float)S.eta[i];
  // [17, 24): pseudo-angles of theta_0..theta_6 (bracket lookup, DRK_PSEUDO_ANGLE)
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const double t = S.th[b + k];
    r[17 + k] = (float)pseudo_angle_d(sin(t), cos(t));
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int h = (k + 1) & 7;
    float* br = r + kRecHdr + 8 * k;
    br[0] = (float)S.ex[b + k];
    br[1] = (float)S.ey[b + k];
    br[2] = (float)S.ex[b + h];
    br[3] = (float)S.ey[b + h];
    const double det = S.det[b + k];
    br[4] = fabs(det) < 1e-12 ? __int_as_float(0x7fc00000) : (float)(1.0 / det);
    br[5] = S.piogf[b + k];
    br[6] = S.hf[b + k];
    br[7] = S.hf[b + h];
  }
}

void launch_shape_rec(const ShapeView& S, int i0, int i1, float* rec, cudaStream_t s) {
  if (i1 > i0 && S.K == 8) {
    k_shape_rec<<<(i1 - i0 + 127) / 128, 128, 0, s>>>(i0, i1, S, rec);
    DRK_COUNT_LAUNCH();
  }
}

// --- mbarrier + 1-D bulk copy (TMA engine, sm_90+) --------------------------
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void write_pixel(const RasterParams& P, const FastPixel& px, int x, int y);

// NT threads per CTA: 256 = one 16x16 tile per CTA; 128 = half a tile (8 x 16
// pixels) per CTA with the tile list staged by both halves — finer-grained
// release of SM resources when a tile's pixels saturate unevenly (long lists).
template <bool VALIDATE, int NT, bool STATS>
__global__ void __launch_bounds__(NT, 512 / NT) k_raster_fast(const __grid_constant__ RasterParams P) {
  constexpr int BATCH = NT == 256 ? DRK_BATCH256 : DRK_BATCH128;  // list entries staged per batch
  constexpr int RING = 2 * BATCH;
  extern __shared__ float4 dyn[];
  Rec* ring = reinterpret_cast<Rec*>(dyn);
  int* s_id = reinterpret_cast<int*>(ring + RING);
  float4* s_b4 = reinterpret_cast<float4*>(s_id + RING) + threadIdx.x;  // [4][NT] float4, this thread's column
#if DRK_TMA_STAGE
  Geo* s_geo = reinterpret_cast<Geo*>(reinterpret_cast<float4*>(s_id + RING) + 4 * NT);  // [BATCH]: next batch's Geo
  __shared__ unsigned long long s_bar;
#endif
  __shared__ unsigned s_ddmax;
  __shared__ TileConst tc;
  const int cta_tile = NT == 256 ? blockIdx.x : blockIdx.x >> 1;
  const int tile = P.tile_base + (P.tile_order ? P.tile_order[cta_tile] : cta_tile);
  const int tx = tile % P.cam.tiles_x, ty = tile / P.cam.tiles_x;
  // warp w covers an 8 x 4 pixel block (spatially compact: coherent saturation
  // depth and popped primitives across the lanes)
  const int wv = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int half = NT == 256 ? (wv & 1) : (int)(blockIdx.x & 1);
  const int x = tx * kTile + half * 8 + (ln & 7), y = ty * kTile + (NT == 256 ? (wv >> 1) : wv) * 4 + (ln >> 3);
  const bool active = x < P.cam.W && y < P.cam.H;
  const double tx0 = (double)tx * kTile, ty0 = (double)ty * kTile;
  // tile reference ray d0 (centre of the tile) and this pixel's offset dd
  double d0[3], dir[3];
  pixel_dir(P.cam, tx0 + 8.0, ty0 + 8.0, d0);
  pixel_dir(P.cam, x + 0.5, y + 0.5, dir);
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
    sh_basis_f((float)dir[0], (float)dir[1], (float)dir[2], P.opt.sh_degree, b);
#pragma unroll
    for (int q = 0; q < 4; ++q) s_b4[q * NT] = make_float4(b[4 * q], b[4 * q + 1], b[4 * q + 2], b[4 * q + 3]);
  }
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
    const unsigned wm = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_ddmax, wm);
  }
  px.T = 1.0;
  px.C0 = px.C1 = px.C2 = px.D = px.N0 = px.N1 = px.N2 = px.A = px.E = 0.f;
  px.ncomp = 0;
  px.stop = INT_MAX;
  px.n_pop = px.n_rej1 = px.n_rej2 = px.n_f64 = px.n_miss = 0;
  px.uncertain = px.err = false;
  unsigned n_str = 0, n_amb = 0, n_app = 0;
  float clo[kCacheCap], chi[kCacheCap];
  int cj[kCacheCap];
#pragma unroll
  for (int q = 0; q < kCacheCap; ++q) {
    clo[q] = chi[q] = __int_as_float(0x7f800000);
    cj[q] = 0;
  }
  int csz = 0;
  float maxhi = __int_as_float(0x7f800000);  // max of chi[] (+inf while the cache has free slots)
  bool done = !active;
  const long long beg = P.tileoff[tile], end = P.tileoff[tile + 1];
  const float eps = (float)P.opt.grazing_eps;
  __syncthreads();
  if (threadIdx.x == 0) tc.ddmax = __uint_as_float(s_ddmax) * 1.0001f + 1e-30f;
  int ring_lo = 0;
  // ray-plane intersection of stream entry jr (geometry.cpp:40-47) as an fp32
  // interval [lo, hi] containing the exact fp64 r_t; false: grazing / behind
  auto isect = [&](int jr, float& lo, float& hi) -> bool {
    const int slot = jr & (RING - 1);
    const float4 r0 = ring[slot].r0;
    const float2 r3 = *reinterpret_cast<const float2*>(&ring[slot].r3);
    const float dz = lin3(r0, ring[slot].r5.x, px.ddx, px.ddy, px.ddz);
    const float adz = fabsf(dz);
    if (adz < eps - r3.y) return false;  // certainly grazing
    const float inv = rcp_nr(dz);
    const float rel_z = r3.y * fabsf(inv);
    if (adz > eps + r3.y && r3.x != 0.f && rel_z <= 1e-3f) {
      const float rt = r3.x * inv;
      if (rt <= 0.f) return false;
      // num (2^-24), 1/dz (2^-23), product (2^-24), dz (rel_z), interval ends
      const float er = rt * (3.3e-7f + rel_z * 1.01f);
      lo = rt - er;
      hi = rt + er;
      return true;
    }
    double rx;
    if (!exact_rt(P, s_id[slot], x, y, &rx)) return false;
    lo = __double2float_rd(rx);
    hi = __double2float_ru(rx);
    return true;
  };
  // SortCache::step (raster.cpp:267-303) for a hit of entry jr on intervals
  // that contain the exact depths, popping (pop_eval) when full; false once the
  // pixel saturates
  auto cache_step = [&](int jr, float lo, float hi) -> bool {
    DRK_STAT(n_str);
    // Fast path: a full cache and an incoming entry certainly shallower than the
    // head (the cache's exact minimum) -- it pops through and the cache is
    // unchanged.  Compiled into the half-tile kernel only, i.e. for long tile
    // lists: 93% of config-3 steps pop through (raster -5%), while config 1's
    // 59% leave most warps divergent (+7.5% with the fast path).
    constexpr bool kThru = DRK_POP_THRU == 1 || (DRK_POP_THRU < 0 && NT == 128);
    int pj = jr;
    const bool thru = kThru && csz == kCacheCap && hi < clo[0];
#if DRK_THRU_STAT
    if (thru) DRK_STAT(n_app);
#endif
    if (!thru) {
#if DRK_CACHE_FAST
      if (maxhi <= lo) {
        // full cache and the incoming entry certainly deeper than every cached one
        // (the common case: lists are presorted by depth): pop the head, append
        const int pj = cj[0];
#pragma unroll
        for (int q = 0; q < kCacheCap - 1; ++q) {
          clo[q] = clo[q + 1];
          chi[q] = chi[q + 1];
          cj[q] = cj[q + 1];
        }
        clo[kCacheCap - 1] = lo;
        chi[kCacheCap - 1] = hi;
        cj[kCacheCap - 1] = jr;
        maxhi = hi;
        return pop_eval<VALIDATE, NT, STATS, RING>(P, px, s_b4, ring, s_id, tc, beg, ring_lo, pj, x, y);
      }
#endif
      bool le[kCacheCap];
      bool amb = false;
#pragma unroll
      for (int q = 0; q < kCacheCap; ++q) {
        le[q] = chi[q] <= lo;
        amb |= !le[q] && !(clo[q] > hi);
      }
      if (amb) {
        // overlapping intervals: compare the exact fp64 depths
        DRK_STAT(n_amb);
        double rin = 0;
        exact_rt(P, s_id[jr & (RING - 1)], x, y, &rin);
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
      if (STATS && !DRK_THRU_STAT && csz == kCacheCap && le[kCacheCap - 1]) ++n_app;  // le is a prefix: all entries <= incoming
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
#if DRK_CACHE_FAST
        if (csz == kCacheCap) {
          maxhi = chi[0];
#pragma unroll
          for (int q = 1; q < kCacheCap; ++q) maxhi = fmaxf(maxhi, chi[q]);
        }
#endif
        return true;
      }
      if (!le[0]) {  // incoming strictly shallower than the head: pops through
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
#if DRK_CACHE_FAST
      // the cache changed (shift + insert, or intervals tightened to exact depths)
      maxhi = chi[0];
#pragma unroll
      for (int q = 1; q < kCacheCap; ++q) maxhi = fmaxf(maxhi, chi[q]);
#endif
    }
    return pop_eval<VALIDATE, NT, STATS, RING>(P, px, s_b4, ring, s_id, tc, beg, ring_lo, pj, x, y);
  };
#if DRK_TMA_STAGE
  // batch b's Geo records arrive in s_geo by bulk copies issued while batch b-1
  // streamed (thread j copies entry j of the batch); s_bar completes one phase
  // per batch
  unsigned gpar = 0;
  int my_id = 0;
  bool pending = false;
  auto prefetch = [&](long long b0n) {
    const int cntn = (int)min((long long)BATCH, end - b0n);
    if (threadIdx.x == 0) mbar_expect_tx(&s_bar, (unsigned)(cntn * sizeof(Geo)));
    fence_proxy_async();  // s_geo was last read by the generic proxy
    if ((int)threadIdx.x < cntn) {
      my_id = P.lid[b0n + threadIdx.x];
      bulk_g2s(s_geo + threadIdx.x, P.geo + my_id, (unsigned)sizeof(Geo), &s_bar);
    }
    pending = true;
  };
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (beg < end) prefetch(beg);
#endif
  long long streamed = 0;
  for (long long b0 = beg; b0 < end; b0 += BATCH) {
    const int jb = (int)(b0 - beg);
    streamed = min(end, b0 + BATCH) - beg;
#if DRK_TOP_BARRIER
    __syncthreads();
#endif
#if DRK_TMA_STAGE
    mbar_wait(&s_bar, gpar);
    gpar ^= 1u;
    pending = false;
    {
      const long long j = b0 + threadIdx.x;
      if ((int)threadIdx.x < BATCH && j < end) {
        const int slot = (jb + threadIdx.x) & (RING - 1);
        stage_record_from(P, s_geo[threadIdx.x], tc, ring[slot]);
        s_id[slot] = my_id;
      }
    }
    __syncthreads();
    if (b0 + BATCH < end) prefetch(b0 + BATCH);
#else
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
#endif
    ring_lo = jb >= BATCH ? jb - BATCH : 0;
    const int cnt = (int)min((long long)BATCH, end - b0);
    if (!done) {
#if DRK_ISECT2
      // two candidates per iteration: both ray-plane intersections first
      // (independent work for the scheduler), then the two cache steps in order
      int c = 0;
      for (; c + 1 < cnt; c += 2) {
        float lo0, hi0, lo1, hi1;
        const bool h0 = isect(jb + c, lo0, hi0);
        const bool h1 = isect(jb + c + 1, lo1, hi1);
        if (h0 && !cache_step(jb + c, lo0, hi0)) {
          done = true;
          break;
        }
        if (h1 && !cache_step(jb + c + 1, lo1, hi1)) {
          done = true;
          break;
        }
      }
      if (!done && c < cnt) {
        float lo0, hi0;
        if (isect(jb + c, lo0, hi0) && !cache_step(jb + c, lo0, hi0)) done = true;
      }
#else
      for (int c = 0; c < cnt; ++c) {
        float lo, hi;
        if (!isect(jb + c, lo, hi)) continue;
        if (!cache_step(jb + c, lo, hi)) {
          done = true;
          break;
        }
      }
#endif
    }
    if (__syncthreads_count(!done) == 0) break;
  }
#if DRK_TMA_STAGE
  if (pending) mbar_wait(&s_bar, gpar);  // no bulk copy may land after the CTA exits
#endif
  if (P.tile_cost && threadIdx.x == 0) atomicMax(P.tile_cost + tile, (unsigned)streamed);
  // end marker: drain the cache head first (raster.cpp:410-414)
  while (!done && csz > 0) {
    const int pj = cj[0];
#pragma unroll
    for (int q = 0; q < kCacheCap - 1; ++q) {
      clo[q] = clo[q + 1];
      chi[q] = chi[q + 1];
      cj[q] = cj[q + 1];
    }
    --csz;
    if (!pop_eval<VALIDATE, NT, STATS, RING>(P, px, s_b4, ring, s_id, tc, beg, ring_lo, pj, x, y))
      done = true;
  }
  // counters: one atomic per warp and counter
  {
    unsigned long long v[9] = {n_str, px.n_pop, (unsigned long long)px.ncomp, px.n_rej1, px.n_rej2, px.n_f64,
                               n_amb, px.n_miss, n_app};
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      unsigned long long s = v[k];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      v[k] = s;
    }
    if ((threadIdx.x & 31) == 0) {
      const int slots[9] = {C_STREAMED, C_POPPED, C_COMPOSITED, C_REJECT_RADIUS, C_REJECT_BRACKET, C_FP64_EVALS,
                            C_AMBIGUOUS, C_RING_MISS, C_CACHE_APPEND};
#pragma unroll
      for (int k = 0; k < 9; ++k)
        if (v[k]) atomicAdd(&P.counters[slots[k]], v[k]);
    }
  }
  if (active) write_pixel(P, px, x, y);
}

__device__ __forceinline__ void write_pixel(const RasterParams& P, const FastPixel& px, int x, int y) {
  if (px.err) atomicAdd(&P.counters[C_ERR_DEGEN_BASIS], 1ull);
  const size_t p = (size_t)y * P.cam.W + x;
  const double c0 = (double)px.C0 + px.T * P.opt.bg[0];
  const double c1 = (double)px.C1 + px.T * P.opt.bg[1];
  const double c2 = (double)px.C2 + px.T * P.opt.bg[2];
  if (P.color) {
    P.color[3 * p] = (float)c0;
    P.color[3 * p + 1] = (float)c1;
    P.color[3 * p + 2] = (float)c2;
  }
  if (P.normal) {
    P.normal[3 * p] = px.N0;
    P.normal[3 * p + 1] = px.N1;
    P.normal[3 * p + 2] = px.N2;
  }
  if (P.depth) P.depth[p] = px.D;
  if (P.alpha) P.alpha[p] = px.A;
  if (P.pxstate) {
    double* st = P.pxstate + 8 * p;
    st[0] = c0;
    st[1] = c1;
    st[2] = c2;
    st[3] = px.D;
    st[4] = px.N0;
    st[5] = px.N1;
    st[6] = px.N2;
    st[7] = px.A;
  }
  if (P.pxstop) P.pxstop[p] = px.stop;
  if (P.pxcomp) P.pxcomp[p] = px.ncomp;
  if (P.pxflag) {
    P.pxflag[p] = px.uncertain ? 1 : 0;
    if (px.uncertain) P.redo_list[atomicAdd(P.redo_count, 1u)] = (int)p;
  }
}

// Tile order of the fast forward: key = (band << 20) | (2^20 - 1 - list length),
// sorted ascending: the longest lists start first (shorter tail).  band_rows > 0
// groups tiles by bands of rows first (measured: no gain); 0 = one global order.
__global__ void k_tile_order_keys(int n, int tiles_x, int band_rows, const long long* __restrict__ tileoff,
                                  int tile_base, unsigned* key, unsigned* id) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const long long len = tileoff[tile_base + t + 1] - tileoff[tile_base + t];
  const unsigned band = band_rows > 0 ? (unsigned)((tile_base + t) / tiles_x / band_rows) : 0u;
  key[t] = (band << 20) | (0xfffffu - (unsigned)min(len, 0xfffffLL));
  id[t] = (unsigned)t;
}

// Backward dispatch order: the tiles that streamed the most list entries in
// the forward (their CTAs run longest) first.
__global__ void k_tile_cost_keys(int n, const unsigned* __restrict__ cost, unsigned* key, unsigned* id) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  key[t] = ~cost[t];
  id[t] = (unsigned)t;
}

void launch_tile_cost_keys(int n, const unsigned* cost, unsigned* key, unsigned* id, cudaStream_t s) {
  if (n > 0) k_tile_cost_keys<<<(n + 255) / 256, 256, 0, s>>>(n, cost, key, id);
}

void launch_tile_order_keys(int n, int tiles_x, int band_rows, const long long* tileoff, int tile_base, unsigned* key,
                            unsigned* id, cudaStream_t s) {
  if (n > 0) k_tile_order_keys<<<(n + 255) / 256, 256, 0, s>>>(n, tiles_x, band_rows, tileoff, tile_base, key, id);
}

size_t raster_fast_smem(int nt) {
  const int batch = nt == 256 ? DRK_BATCH256 : DRK_BATCH128;
  return (size_t)2 * batch * (sizeof(Rec) + sizeof(int)) + 16 * nt * sizeof(float) +
         (DRK_TMA_STAGE ? batch * sizeof(Geo) : 0);
}

// Half-tile CTAs pay off once tile lists are long (measured: config 2 / 3 with
// ~9.5k / 28k entries per tile -3% / -2.3% raster time, config 1 with 2.2k
// +0.6%).
int raster_fast_nt(long long pairs, int n_tiles) { return pairs > 4000LL * n_tiles ? 128 : 256; }
static_assert(sizeof(Rec) == 96, "ring record");

bool raster_fast_eligible(const RasterParams& P) {
  return P.S.K == 8 && P.shrec != nullptr && P.opt.use_cache && !P.opt.exact_sort && !P.opt.fp64_alpha &&
         P.replay_cap == 0;
}

template <int NT>
static void launch_nt(const RasterParams& P, int n_tiles, bool validate, cudaStream_t s) {
  const size_t smem = raster_fast_smem(NT);
  static PerDeviceOnce attr;
  attr([&] {
    cudaFuncSetAttribute(k_raster_fast<false, NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_raster_fast<false, NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_raster_fast<true, NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  const int ctas = n_tiles * (256 / NT);
  if (validate) k_raster_fast<true, NT, true><<<ctas, NT, smem, s>>>(P);
  else if (P.no_counters) k_raster_fast<false, NT, false><<<ctas, NT, smem, s>>>(P);
  else k_raster_fast<false, NT, true><<<ctas, NT, smem, s>>>(P);
}

// 128 registers per thread either way: 2 CTAs of 256 or 4 CTAs of 128 per SM
void launch_raster_fast(const RasterParams& P, int n_tiles, bool validate, cudaStream_t s) {
  if (P.fast_nt == 128) launch_nt<128>(P, n_tiles, validate, s);
  else launch_nt<256>(P, n_tiles, validate, s);
}

}  // namespace drk
