// Deterministic parallel backward (drk_backward(..., deterministic = 1)).
//
// The reference reduces per-primitive gradients in a fixed order: every tile
// accumulates its own partials over its pixels (row-major) and their records
// (composite order), then the partials are added tile by tile in index order
// (grad.cpp:327-368; "no unordered atomic float accumulation").
// On the GPU:
//   1. the forward left the number of composited entries of every pixel
//      (pxcomp); an exclusive scan over the pixels in (tile, row-major pixel in
//      the tile) order gives every (pixel, composite) record a fixed slot;
//   2. the backward kernels run in parallel as usual, but each composited
//      record writes its gradient row into its slot (det_row) instead of
//      adding it atomically — the fast fp32 kernel for ordinary pixels, the fp64
//      per-pixel path for the pixels the forward re-rendered in fp64 (or for
//      every pixel in the list / exact-sort / fp64-alpha modes);
//   3. a stable radix sort of the record slots by primitive id keeps, within a
//      primitive, the (tile, pixel, composite) order; the records of each
//      (primitive, tile) pair — a tile segment — are summed in order by one warp
//      (fp64, in parallel over the segments), then one warp per primitive adds
//      its tile partials in tile order to an fp64 accumulator.
// The result does not depend on scheduling: two runs are bitwise identical.
// Record rows take G floats (fast-kernel frames) or doubles (reference precision) each; frames whose records exceed the memory budget
// are processed in chunks of tile rows (in row order, so the accumulation order
// is unchanged).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "drk_internal.h"

namespace drk {

template <typename T>
int exclusive_scan(drk_ctx* c, const T* in, long long n, long long* out, long long* total);
int sort_pairs(drk_ctx* c, unsigned* k, unsigned* v, unsigned* k2, unsigned* v2, long long n);
__global__ void k_band_flagged(const unsigned char* pxflag, int W, int y0, int y1, int* list, unsigned* count);

namespace {

// records per slot: slot = tile * 256 + (y % 16) * 16 + x % 16
__global__ void k_det_slot_counts(CamD cam, const int* __restrict__ pxcomp, int* cnt) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)cam.tiles_x * cam.tiles_y * 256;
  if (s >= n) return;
  const int tile = (int)(s >> 8), l = (int)(s & 255);
  const int x = (tile % cam.tiles_x) * 16 + (l & 15), y = (tile / cam.tiles_x) * 16 + (l >> 4);
  cnt[s] = (x < cam.W && y < cam.H) ? pxcomp[(size_t)y * cam.W + x] : 0;
}

// record offsets at the tile-row boundaries
__global__ void k_det_row_offsets(const long long* __restrict__ base, const int* __restrict__ cnt, int tiles_x,
                                  int tiles_y, long long* rowoff) {
  const int ty = blockIdx.x * blockDim.x + threadIdx.x;
  if (ty > tiles_y) return;
  if (ty < tiles_y) {
    rowoff[ty] = base[(long long)ty * tiles_x * 256];
  } else {
    const long long last = (long long)tiles_y * tiles_x * 256 - 1;
    rowoff[ty] = base[last] + cnt[last];
  }
}

__global__ void k_band_all(int W, int y0, int y1, int* list, unsigned* count) {
  const long long p = (long long)y0 * W + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p == (long long)y0 * W) *count = (unsigned)((long long)(y1 - y0) * W);
  if (p >= (long long)y1 * W) return;
  list[p - (long long)y0 * W] = (int)p;
}

__global__ void k_det_keys(long long n, const int* __restrict__ id, unsigned* k, unsigned* v) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  k[i] = (unsigned)id[i];
  v[i] = (unsigned)i;
}

// [first, end) of every primitive's run of sorted records (untouched: 0, 0)
__global__ void k_det_segments(long long n, const unsigned* __restrict__ k, long long* seg) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned key = k[i];
  if (i == 0 || k[i - 1] != key) seg[2 * (size_t)key] = i;
  if (i == n - 1 || k[i + 1] != key) seg[2 * (size_t)key + 1] = i + 1;
}

// Tile segments of the sorted records: a segment = the records of one
// (primitive, tile) pair, consecutive after the stable sort by primitive.
__global__ void k_det_tseg_flags(long long n, const unsigned* __restrict__ k, const unsigned* __restrict__ rec_of,
                                 const int* __restrict__ tile_of, int* flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || k[i] != k[i - 1] || tile_of[rec_of[i]] != tile_of[rec_of[i - 1]]) ? 1 : 0;
}

__global__ void k_det_tseg_starts(long long n, const int* __restrict__ flag, const long long* __restrict__ pos,
                                  const unsigned* __restrict__ k, long long* starts, unsigned* seg_prim) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (flag[i]) {
    starts[pos[i]] = i;
    seg_prim[pos[i]] = k[i];
  }
}

// Phase 1: one warp per tile segment sums its records' rows in order (fp64)
// and stores the tile partial in the segment's first row.
template <typename RT>
__global__ void k_det_tseg_sum(long long nseg, long long nrec, int G, const long long* __restrict__ starts,
                               const unsigned* __restrict__ rec_of, RT* rows) {
  constexpr int kB = 8;
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nseg) return;
  const long long b = starts[t], e = t + 1 < nseg ? starts[t + 1] : nrec;
  double part[3] = {0.0, 0.0, 0.0};
  for (long long r0 = b; r0 < e; r0 += kB) {
    double v[kB][3];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const unsigned rec = r0 + u < e ? rec_of[r0 + u] : 0u;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int c = 32 * q + lane;
        v[u][q] = (r0 + u < e && c < G) ? (double)rows[(size_t)rec * G + c] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u)
#pragma unroll
      for (int q = 0; q < 3; ++q) part[q] += v[u][q];
  }
  const unsigned first = rec_of[b];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int c = 32 * q + lane;
    if (c < G) rows[(size_t)first * G + c] = (RT)part[q];
  }
}

// Phase 2: one warp per primitive adds its tile partials in tile order to the
// fp64 accumulator (the reference's tile-then-id reduction, grad.cpp:352-368).
template <typename RT>
__global__ void k_det_prim_sum(int n, int G, const long long* __restrict__ pseg, const long long* __restrict__ starts,
                               const unsigned* __restrict__ rec_of, const RT* __restrict__ rows, double* acc) {
  constexpr int kB = 8;
  const int p = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= n) return;
  const long long b = pseg[2 * (size_t)p], e = pseg[2 * (size_t)p + 1];
  if (e <= b) return;
  double total[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int c = 32 * q + lane;
    total[q] = c < G ? acc[(size_t)p * G + c] : 0.0;
  }
  for (long long t0 = b; t0 < e; t0 += kB) {
    double v[kB][3];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const unsigned rec = t0 + u < e ? rec_of[starts[t0 + u]] : 0u;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int c = 32 * q + lane;
        v[u][q] = (t0 + u < e && c < G) ? (double)rows[(size_t)rec * G + c] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u)
#pragma unroll
      for (int q = 0; q < 3; ++q) total[q] += v[u][q];
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int c = 32 * q + lane;
    if (c < G) acc[(size_t)p * G + c] = total[q];
  }
}

__global__ void k_det_finish(long long n, const double* __restrict__ acc, float* gact) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) gact[i] = (float)acc[i];
}

unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// P: the backward's parameters (gact, touched, frame gradients, pixel state);
// band_lists(b, Q): sets Q's tile lists for band b.  Writes P.gact (fp32) and
// leaves the fp64 sums in ctx->det_acc for the activation backward.
int run_backward_det(drk_ctx* c, const RasterParams& P, const std::vector<int>& bands,
                     int (*band_lists)(drk_ctx*, int, RasterParams&)) {
  cudaStream_t s = c->stream;
  const CamD& cd = c->camd;
  const int n = c->act.n, G = P.G;
  // DRK_HOST_TRACE=1: phase times (stream synchronised at each checkpoint) on stderr
  static const bool trace = getenv("DRK_HOST_TRACE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  std::string tline;
  auto tr = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    char b[64];
    snprintf(b, sizeof b, " %s %.2f", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    tline += b;
    t_last = now;
  };
  const long long slots = (long long)cd.tiles_x * cd.tiles_y * 256;
  if (!P.pxcomp) return set_error(c, DRK_ERR_GENERIC, "deterministic backward: no composite counts");
  int* cnt = ensure<int>(c->det_cnt, (size_t)slots + 1);
  long long* base = ensure<long long>(c->det_base, (size_t)slots + 1);
  long long* rowoff_d = ensure<long long>(c->det_rowoff, (size_t)cd.tiles_y + 2);
  double* acc = ensure<double>(c->det_acc, (size_t)n * G + 1);
  long long* seg = ensure<long long>(c->det_poff, 2 * (size_t)n + 2);
  if (!cnt || !base || !rowoff_d || !acc || !seg) return set_error(c, DRK_ERR_OOM, "deterministic backward");
  cudaMemsetAsync(acc, 0, sizeof(double) * (size_t)n * G, s);
  if (slots > 0) {
    k_det_slot_counts<<<blocks(slots, 256), 256, 0, s>>>(cd, P.pxcomp, cnt);
    DRK_COUNT_LAUNCH();
    if (int st = exclusive_scan<int>(c, cnt, slots, base, nullptr)) return st;
    k_det_row_offsets<<<blocks(cd.tiles_y + 1, 128), 128, 0, s>>>(base, cnt, cd.tiles_x, cd.tiles_y, rowoff_d);
    DRK_COUNT_LAUNCH();
  }
  tr("offsets");
  std::vector<long long> rowoff((size_t)cd.tiles_y + 1, 0);
  if (slots > 0) cudaMemcpyAsync(rowoff.data(), rowoff_d, sizeof(long long) * rowoff.size(), cudaMemcpyDeviceToHost, s);
  if (int st = cuda_check(c, cudaStreamSynchronize(s), "deterministic backward offsets")) return st;

  // records per chunk: the budget covers the row (G floats), id, tile and the
  // sort's four u32 arrays
  const bool fast = P.opt.use_cache && !P.opt.exact_sort && P.opt.raster_kernel != 1 && P.opt.raster_kernel != 5 &&
                    raster_fast_eligible(P);
  // fp32 rows where the fast fp32 kernel computes the records; fp64 rows where
  // every record comes from the fp64 per-pixel path (reference precision)
  const size_t row_bytes = fast ? sizeof(float) : sizeof(double);
  const size_t per_rec = row_bytes * G + 2 * sizeof(int) + 4 * sizeof(unsigned) + 28;  // + tile-segment scratch
  long long limit = c->det_chunk_limit;
  if (limit <= 0) {
    // at most 16 GB of record scratch (kept by the context between calls: no
    // multi-second allocation of a frame-sized buffer per backward), and at most
    // half of the free memory
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t have = c->det_rec.bytes + c->det_id.bytes + c->det_tile.bytes + c->det_sort.bytes +
                        c->det_tflag.bytes + c->det_tpos.bytes + c->det_tstart.bytes + c->det_tprim.bytes;
    limit = (long long)(std::min<size_t>((free_b + have) / 2, (size_t)16 << 30) / per_rec);
  }
  limit = std::max(1LL, std::min(limit, (long long)0x7fffffff));

  const int nb = (int)bands.size() - 1;
  for (int b = 0; b < nb; ++b) {
    RasterParams Q = P;
    if (nb > 1 && band_lists) {
      if (int st = band_lists(c, b, Q)) return st;
    }
    int ty0 = bands[b];
    while (ty0 < bands[b + 1]) {
      int ty1 = ty0 + 1;
      while (ty1 < bands[b + 1] && rowoff[ty1 + 1] - rowoff[ty0] <= limit) ++ty1;
      const long long off = rowoff[ty0], R = rowoff[ty1] - rowoff[ty0];
      const int nt = (ty1 - ty0) * cd.tiles_x;
      const int y0 = ty0 * kTile, y1 = std::min(ty1 * kTile, cd.H);
      if (R > 0) {
        void* rows = ensure_bytes(c->det_rec, row_bytes * (size_t)R * G);
        int* ids = ensure<int>(c->det_id, (size_t)R);
        int* tiles = ensure<int>(c->det_tile, (size_t)R);
        unsigned* sk = ensure<unsigned>(c->det_sort, 4 * (size_t)R + 4);
        if (!rows || !ids || !tiles || !sk) return set_error(c, DRK_ERR_OOM, "deterministic backward records");
        tr("alloc");  // no clearing: every record's writer stores its whole row
        Q.det_rec = fast ? nullptr : static_cast<double*>(rows);
        Q.det_rec32 = fast ? static_cast<float*>(rows) : nullptr;
        Q.det_id = ids;
        Q.det_tile = tiles;
        Q.det_base = base;
        Q.det_off = off;
        Q.det_cap = R;
        Q.tile_base = ty0 * cd.tiles_x;
        Q.tile_order = nullptr;
        const long long npx = (long long)(y1 - y0) * cd.W;
        if (P.opt.exact_sort) {
          launch_exact_bwd(Q, nt, s);
        } else if (fast) {
          launch_raster_bwd_fast_det(Q, nt, s);
          cudaMemsetAsync(Q.redo_count, 0, sizeof(unsigned), s);
          k_band_flagged<<<blocks(npx, 256), 256, 0, s>>>(Q.pxflag, cd.W, y0, y1, Q.redo_list, Q.redo_count);
          DRK_COUNT_LAUNCH();
          launch_pixels_bwd(Q, s);
        } else {
          k_band_all<<<blocks(npx, 256), 256, 0, s>>>(cd.W, y0, y1, Q.redo_list, Q.redo_count);
          DRK_COUNT_LAUNCH();
          launch_pixels_bwd(Q, s);
        }
        if (int st = cuda_check(c, cudaGetLastError(), "deterministic backward raster")) return st;
        tr("raster");
        // group the records by primitive, keeping their order, and reduce
        unsigned *kk = sk, *vv = sk + R + 1, *k2 = vv + R + 1, *v2 = k2 + R;
        k_det_keys<<<blocks(R, 256), 256, 0, s>>>(R, ids, kk, vv);
        DRK_COUNT_LAUNCH();
        if (int st = sort_pairs(c, kk, vv, k2, v2, R)) return st;
        tr("sort");
        // tile segments (one per (primitive, tile)): partials in parallel, then
        // each primitive's partials in tile order
        int* tflag = ensure<int>(c->det_tflag, (size_t)R + 1);
        long long* tpos = ensure<long long>(c->det_tpos, (size_t)R + 1);
        long long* tstart = ensure<long long>(c->det_tstart, (size_t)R + 1);
        unsigned* tprim = ensure<unsigned>(c->det_tprim, (size_t)R + 1);
        if (!tflag || !tpos || !tstart || !tprim) return set_error(c, DRK_ERR_OOM, "deterministic backward segments");
        k_det_tseg_flags<<<blocks(R, 256), 256, 0, s>>>(R, kk, vv, tiles, tflag);
        long long nseg = 0;
        if (int st = exclusive_scan<int>(c, tflag, R, tpos, &nseg)) return st;
        k_det_tseg_starts<<<blocks(R, 256), 256, 0, s>>>(R, tflag, tpos, kk, tstart, tprim);
        if (fast) k_det_tseg_sum<float><<<blocks(32LL * nseg, 256), 256, 0, s>>>(nseg, R, G, tstart, vv, Q.det_rec32);
        else k_det_tseg_sum<double><<<blocks(32LL * nseg, 256), 256, 0, s>>>(nseg, R, G, tstart, vv, Q.det_rec);
        cudaMemsetAsync(seg, 0, sizeof(long long) * 2 * (size_t)n, s);
        k_det_segments<<<blocks(nseg, 256), 256, 0, s>>>(nseg, tprim, seg);
        if (fast) k_det_prim_sum<float><<<blocks(32LL * n, 256), 256, 0, s>>>(n, G, seg, tstart, vv, Q.det_rec32, acc);
        else k_det_prim_sum<double><<<blocks(32LL * n, 256), 256, 0, s>>>(n, G, seg, tstart, vv, Q.det_rec, acc);
        launch_counter() += 5;
        if (int st = cuda_check(c, cudaGetLastError(), "deterministic backward reduce")) return st;
        tr("reduce");
      }
      ty0 = ty1;
    }
  }
  if (n > 0) {
    k_det_finish<<<blocks((long long)n * G, 256), 256, 0, s>>>((long long)n * G, acc, P.gact);
    DRK_COUNT_LAUNCH();
  }
  // the chunks rebuilt the fp64 pass's pixel list; restore the forward's
  // (whole-frame) list for a later non-deterministic backward of this frame
  if (nb == 1 && P.pxflag && !P.opt.fp64_alpha && !P.opt.exact_sort) {
    cudaMemsetAsync(P.redo_count, 0, sizeof(unsigned), s);
    const long long npx = (long long)cd.W * cd.H;
    if (npx > 0) {
      k_band_flagged<<<blocks(npx, 256), 256, 0, s>>>(P.pxflag, cd.W, 0, cd.H, P.redo_list, P.redo_count);
      DRK_COUNT_LAUNCH();
    }
  } else if (nb == 1 && P.opt.fp64_alpha) {
    const long long npx = (long long)cd.W * cd.H;
    if (npx > 0) {
      k_band_all<<<blocks(npx, 256), 256, 0, s>>>(cd.W, 0, cd.H, P.redo_list, P.redo_count);
      DRK_COUNT_LAUNCH();
    }
  }
  tr("release");
  if (trace) fprintf(stderr, "[drk det]%s\n", tline.c_str());
  unsigned long long ovf = 0;
  cudaMemcpyAsync(&ovf, P.counters + C_DET_OVERFLOW, sizeof ovf, cudaMemcpyDeviceToHost, s);
  if (int st = cuda_check(c, cudaStreamSynchronize(s), "deterministic backward")) return st;
  if (ovf) {
    cudaMemsetAsync(P.counters + C_DET_OVERFLOW, 0, sizeof ovf, s);
    return set_error(c, DRK_ERR_GENERIC, "deterministic backward: composite counts differ from the forward");
  }
  return DRK_OK;
}

}  // namespace drk
