// C-ABI (include/drk_b200.h) and the host-side orchestration of one view:
// activate -> K1 prep -> scan -> K2 rows -> scan -> K3 emit -> radix sort ->
// tile offsets -> K4 raster; backward: K5 raster-bwd -> K6 activation bwd.
#include <cuda.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstdio>
#include <cstring>
#include <vector>

#include "drk_internal.h"

namespace drk {

// kernels defined in the other translation units
__global__ void k_prep_hull(int n, const int2* ptsref, double2* pts_pool, CamD cam, OptD opt, int4* bbox, int2* hullref,
                            double2* pool, long long pool_cap, int* rowcnt, unsigned long long* counters);
__global__ void k_prep1(Activated A, CamD cam, OptD opt, Geo* geo, int4* bbox, int2* hullref, double2* pool,
                        long long pool_cap, int* rowcnt, unsigned long long* counters, const int* list, int list_n,
                        double2* scratch, int scratch_cap, int* overflow);
__global__ void k_rows(int n, const int4* bbox, const int2* hullref, const double2* pool, const long long* rowoff,
                       CamD cam, OptD opt, int4* rows, int* rowpaircnt, unsigned long long* counters, int ty_lo,
                       int ty_hi);
__global__ void k_band_rowcnt(int n, const int4* bbox, int ty_lo, int ty_hi, int* rowcnt);
__global__ void k_row_pair_bound(int n, int tiles_y, const int4* bbox, unsigned long long* rowest);
__global__ void k_band_flagged(const unsigned char* pxflag, int W, int y0, int y1, int* list, unsigned* count);
__global__ void k_tile_rays(CamD cam, double* cdirs, double* tdirs);
__global__ void k_emit_rows(long long n_rows, const int4* rows, const long long* rowpairoff, const Geo* geo,
                            const double* cdirs, const double* tdirs, CamD cam, OptD opt, unsigned long long* pk,
                            unsigned* pv, unsigned* krange);
__global__ void k_tile_bounds(long long n, const unsigned* sk, int dbits, int n_tiles, long long* tileoff);
__global__ void k_key_hist(long long n, const unsigned long long* pk, const unsigned* krange, unsigned* hist);
__global__ void k_key_map(const unsigned* hist, const unsigned* krange, int dbits, unsigned* map);
__global__ void k_pack_keys(long long n, const unsigned long long* pk, const unsigned* krange, const unsigned* map,
                            int dbits, unsigned* sk);
__global__ void k_tie_keys(long long n, const unsigned* sk, const unsigned* sv, int dbits, const Geo* geo,
                           const double* cdirs, const double* tdirs, CamD cam, OptD opt, unsigned long long* fk);
__global__ void k_tie_rank(long long n, const unsigned* sk, const unsigned* sv, const unsigned long long* fk,
                           unsigned* out, unsigned long long* counters, long long* long_runs);
__global__ void k_tie_long(long long n, const unsigned* sk, unsigned long long* fk, unsigned* out,
                           const long long* long_runs);
__global__ void k_full_keys(long long n, const unsigned* sk, const unsigned* sv, int dbits, const Geo* geo,
                            const double* cdirs, const double* tdirs, CamD cam, OptD opt, double* out);
__global__ void k_full_keys_off(long long n, const long long* tileoff, int n_tiles, const unsigned* sv, const Geo* geo,
                                const double* cdirs, const double* tdirs, CamD cam, OptD opt, double* out);
template <typename T>
int exclusive_scan(drk_ctx* c, const T* in, long long n, long long* out, long long* total);
int sort_pairs(drk_ctx* c, unsigned* k, unsigned* v, unsigned* k2, unsigned* v2, long long n);
void launch_tile_cost_keys(int n, const unsigned* cost, unsigned* key, unsigned* id, cudaStream_t s);
void launch_tile_order_keys(int n, int tiles_x, int band_rows, const long long* tileoff, int tile_base, unsigned* key,
                            unsigned* id, cudaStream_t s);
void launch_act_bwd(int n, int K, int terms, const float* raw, const double* gact, int G,
                    const unsigned char* touched_dev, const Geo* geo, const CamD& cam, float* grad_raw,
                    float* d_center_world, float* screen_grad, unsigned char* touched_out, int accumulate,
                    cudaStream_t s);
void launch_act_bwd(int n, int K, int terms, const float* raw, const float* gact, int G,
                    const unsigned char* touched_dev, const Geo* geo, const CamD& cam, float* grad_raw,
                    float* d_center_world, float* screen_grad, unsigned char* touched_out, int accumulate,
                    cudaStream_t s);
void launch_l1(long long n, const float* r, const float* t, double* loss, float* dcol, cudaStream_t s);
void launch_alpha_bound(const ShapeView& S, int n, long long samples, unsigned long long seed,
                        unsigned long long* out, cudaStream_t s);

void* ensure_bytes(DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return b.p;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  size_t want = bytes + bytes / 4 + 256;
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      b.p = nullptr;
      return nullptr;
    }
    want = bytes;
  }
  b.bytes = want;
  return b.p;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

int set_error(drk_ctx* c, int status, const std::string& msg) {
  if (c) c->err = msg;
  return status;
}

int cuda_check(drk_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DRK_OK;
  cudaGetLastError();
  return set_error(c, e == cudaErrorMemoryAllocation ? DRK_ERR_OOM : DRK_ERR_CUDA,
                   std::string(where) + ": " + cudaGetErrorString(e));
}

static CamD make_cam(const drk_camera* c) {
  CamD d;
  d.fx = c->fx;
  d.fy = c->fy;
  d.cx = c->cx;
  d.cy = c->cy;
  for (int i = 0; i < 9; ++i) d.R[i] = c->R[i];
  for (int i = 0; i < 3; ++i) d.t[i] = c->t[i];
  // Camera::position (geometry.hpp:15): (-R^T) t, left to right
  for (int i = 0; i < 3; ++i) {
    volatile double a = (-c->R[0 + i]) * c->t[0];
    volatile double b = (-c->R[3 + i]) * c->t[1];
    volatile double s = a + b;
    volatile double e = (-c->R[6 + i]) * c->t[2];
    d.o[i] = s + e;
  }
  d.W = c->width;
  d.H = c->height;
  d.tiles_x = (c->width + kTile - 1) / kTile;
  d.tiles_y = (c->height + kTile - 1) / kTile;
  return d;
}

static OptD make_opt(const drk_options* o, int terms) {
  OptD d;
  d.lowpass_radius = o->lowpass_radius;
  d.alpha_min = o->alpha_min;
  d.grazing_eps = o->grazing_eps;
  for (int i = 0; i < 3; ++i) d.bg[i] = o->background[i];
  d.early_stop = o->early_stop_transmittance;
  d.lp_pad = o->lowpass_radius * std::sqrt(2.0 * std::log(1.0 / o->alpha_min)) + 1e-9;
  d.sh_degree = o->sh_degree;
  d.use_cache = o->use_cache;
  d.exact_sort = o->exact_sort;
  d.presort = o->presort;
  d.record_replay = o->record_replay;
  d.fp64_alpha = o->fp64_alpha;
  d.raster_kernel = o->raster_kernel;
  const int t = (o->sh_degree + 1) * (o->sh_degree + 1);
  d.terms_active = t < terms ? t : terms;
  return d;
}

// CTA shape of the fast kernels (raster_kernel 6 / 7 force half / whole tiles)
static int choose_nt(const drk_ctx* c, long long pairs, int tiles) {
  return c->opt.raster_kernel == 6 ? 128 : c->opt.raster_kernel == 7 ? 256 : raster_fast_nt(pairs, tiles);
}

static RasterParams raster_params(drk_ctx* c) {
  RasterParams P;
  std::memset(&P, 0, sizeof P);
  P.cam = c->camd;
  P.opt = c->optd;
  P.tileoff = static_cast<const long long*>(c->tileoff.p);
  P.lid = static_cast<const int*>(c->pv.p);
  P.geo = static_cast<const Geo*>(c->geo.p);
  const Activated& A = c->act;
  P.S = ShapeView{A.s, A.th, A.ex, A.ey, A.det, A.eta, A.tau, A.o, A.thf, A.invdetf, A.piogf, A.hf, A.psif, A.K};
  P.sh = A.sh;
  P.sh64 = A.sh64;
  P.terms = A.terms;
  P.counters = static_cast<unsigned long long*>(c->counters.p);
  // pixels flagged for the fp64 re-render (list written by the fp32 pass)
  P.redo_list = static_cast<int*>(c->redo.p);
  P.redo_tmp = c->redo.p && c->redo_half > 0 ? P.redo_list + c->redo_half : nullptr;
  P.redo_hist = P.redo_tmp ? reinterpret_cast<unsigned*>(P.redo_tmp + c->redo_half) : nullptr;
  P.redo_count = reinterpret_cast<unsigned int*>(ensure<unsigned long long>(c->redo_cnt, 1));
  P.shrec = A.rec;
  P.frame32 = static_cast<const float4*>(c->frame32.p);
  P.fast_nt = 256;
  P.no_counters = c->work_counters ? 0 : 1;
  P.pxcomp = static_cast<int*>(c->pxcomp.p);
  return P;
}

static int read_counters(drk_ctx* c, unsigned long long* h) {
  cudaMemcpyAsync(h, c->counters.p, sizeof(unsigned long long) * C_COUNT, cudaMemcpyDeviceToHost, c->stream);
  return cuda_check(c, cudaStreamSynchronize(c->stream), "counters");
}

static void mark(drk_ctx* c, int i) {
  if (c->timing) cudaEventRecord(c->ev[i], c->stream);
}

static float elapsed(drk_ctx* c, int a, int b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

// Bands of tile rows: one band unless the frame's pairs (upper bound from the
// bounding boxes) would not fit in device memory; then greedy bands whose
// bound fits (SURVEY.md §7 hard part 5: banded binning for config 4).
// device bytes per (tile, primitive) pair: emitted 64-bit keys (reused as the
// sort's second buffer and for the full keys of tied entries), sorted keys and
// two id lists (8 + 4 + 4 + 4), plus row / tile scratch
constexpr double kPairBytes = 22.0;

static int plan_bands(drk_ctx* c) {
  const CamD& cd = c->camd;
  const int n = c->act.n;
  c->bands.assign({0, cd.tiles_y});
  if (n == 0 || cd.tiles_y <= 1) return DRK_OK;
  // cudaMemGetInfo is slow (tens of ms): the device size is queried once per
  // context and free memory only when a trivial bound does not fit
  if (c->device_bytes == 0) {
    size_t f0 = 0, t0 = 0;
    cudaMemGetInfo(&f0, &t0);
    c->device_bytes = t0;
  }
  if (c->band_pair_limit == 0 && (double)n * cd.tiles_x * cd.tiles_y <= 0.25 * (double)c->device_bytes / kPairBytes)
    return DRK_OK;  // every primitive in every tile would still fit in a quarter of the device
  unsigned long long* rowest = ensure<unsigned long long>(c->rowest, cd.tiles_y + 1);
  if (!rowest) return set_error(c, DRK_ERR_OOM, "row estimates");
  cudaMemsetAsync(rowest, 0, sizeof(unsigned long long) * (cd.tiles_y + 1), c->stream);
  if (cd.tiles_y > 6000) return set_error(c, DRK_ERR_UNSUPPORTED, "more than 6000 tile rows");
  k_row_pair_bound<<<std::min((n + 255) / 256, 148 * 4), 256, sizeof(unsigned long long) * cd.tiles_y, c->stream>>>(
      n, cd.tiles_y, static_cast<const int4*>(c->bbox.p), rowest);
  DRK_COUNT_LAUNCH();
  std::vector<unsigned long long> est(cd.tiles_y);
  cudaMemcpyAsync(est.data(), rowest, sizeof(unsigned long long) * cd.tiles_y, cudaMemcpyDeviceToHost, c->stream);
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "band plan")) return st;
  unsigned long long total = 0;
  for (auto e : est) total += e;
  double limit = (double)c->band_pair_limit;
  if (limit <= 0) {
    // the bound fits a quarter of the device: no free-memory query (cudaMemGetInfo
    // costs milliseconds to tens of milliseconds per call)
    if ((double)total <= 0.25 * (double)c->device_bytes / kPairBytes) return DRK_OK;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t held = c->pk.bytes + c->pv.bytes + c->sk.bytes + c->pidx.bytes + c->hist.bytes + c->sortoff.bytes;
    limit = 0.7 * (double)(free_b + held) / kPairBytes;
  }
  if ((double)total <= limit) return DRK_OK;
  c->bands.assign({0});
  unsigned long long acc = 0;
  for (int ty = 0; ty < cd.tiles_y; ++ty) {
    if (acc > 0 && (double)(acc + est[ty]) > limit) {
      c->bands.push_back(ty);
      acc = 0;
    }
    acc += est[ty];
  }
  c->bands.push_back(cd.tiles_y);
  return DRK_OK;
}

// Binning of tile rows [ty_lo, ty_hi): rows, pairs with NearestDepth keys,
// radix sort, tile offsets (tiles outside the band get empty lists).
static int bin_band(drk_ctx* c, int ty_lo, int ty_hi, long long* n_pairs_out) {
  const CamD& cd = c->camd;
  const OptD& od = c->optd;
  const int n = c->act.n;
  const int n_tiles = cd.tiles_x * cd.tiles_y;
  cudaStream_t s = c->stream;
  const int4* bbox = static_cast<const int4*>(c->bbox.p);
  int* rowcnt = static_cast<int*>(c->rowcnt.p);
  long long* rowoff = static_cast<long long*>(c->rowoff.p);
  unsigned long long* ctr = static_cast<unsigned long long*>(c->counters.p);
  const bool whole = ty_lo == 0 && ty_hi == cd.tiles_y;
  if (!whole && n > 0) {
    k_band_rowcnt<<<(n + 127) / 128, 128, 0, s>>>(n, bbox, ty_lo, ty_hi, rowcnt);
    DRK_COUNT_LAUNCH();
  }
  long long n_rows = 0;
  if (int st = exclusive_scan<int>(c, rowcnt, n, rowoff, &n_rows)) return st;
  c->n_rows = n_rows;
  int4* rows = ensure<int4>(c->rows, n_rows + 1);
  int* rowpaircnt = ensure<int>(c->rowpaircnt, n_rows + 1);
  long long* rowpairoff = ensure<long long>(c->rowpairoff, n_rows + 1);
  if (!rows || !rowpaircnt || !rowpairoff) return set_error(c, DRK_ERR_OOM, "row buffers");
  if (n > 0)
    k_rows<<<(unsigned)((32LL * n + 127) / 128), 128, 0, s>>>(n, bbox, static_cast<const int2*>(c->hullref.p),
                                           static_cast<const double2*>(c->hull.p), rowoff, cd, od, rows, rowpaircnt,
                                           ctr, ty_lo, ty_hi);
  long long n_pairs = 0;
  if (int st = exclusive_scan<int>(c, rowpaircnt, n_rows, rowpairoff, &n_pairs)) return st;
  unsigned long long* pk = ensure<unsigned long long>(c->pk, n_pairs + 1);
  unsigned* pv = ensure<unsigned>(c->pv, n_pairs + 1);
  unsigned* sk = ensure<unsigned>(c->sk, n_pairs + 1);
  unsigned* ids2 = ensure<unsigned>(c->pidx, n_pairs + 1);  // the tie ordering's output id list
  unsigned* krange = ensure<unsigned>(c->bits, 2 + 2 * 4096);  // range, sampled histogram, q map
  long long* tileoff = ensure<long long>(c->tileoff, n_tiles + 1);
  if (!pk || !pv || !sk || !ids2 || !krange || !tileoff) return set_error(c, DRK_ERR_OOM, "pair buffers");
  const unsigned kr0[2] = {0xffffffffu, 0u};
  cudaMemcpyAsync(krange, kr0, sizeof kr0, cudaMemcpyHostToDevice, s);
  if (n_rows > 0)
    k_emit_rows<<<(unsigned)((n_rows * 16 + 255) / 256), 256, 0, s>>>(
        n_rows, rows, rowpairoff, static_cast<const Geo*>(c->geo.p), static_cast<const double*>(c->cdirs.p),
        static_cast<const double*>(c->tdirs.p), cd, od, pk, pv, krange);
  launch_counter() += 2;
  mark(c, 3);
  sort_trace("start", s);
  // sort key: tile in the high bits, the quantised depth key in the rest
  int tbits = 1;
  while ((1ll << tbits) < n_tiles) ++tbits;
  c->key_dbits = std::min(26, 32 - tbits);  // k_key_map packs base << 5 in 32 bits
  if (n_pairs > 0) {
    unsigned* khist = krange + 2;
    unsigned* kmap = khist + 4096;
    cudaMemsetAsync(khist, 0, sizeof(unsigned) * 4096, s);
    const unsigned nb = (unsigned)std::min<long long>((n_pairs + 256 * 8 * 4 - 1) / (256 * 8 * 4), 148 * 8);
    k_key_hist<<<nb, 256, 0, s>>>(n_pairs, pk, krange, khist);
    k_key_map<<<1, 1024, 0, s>>>(khist, krange, c->key_dbits, kmap);
    k_pack_keys<<<(unsigned)std::min<long long>((n_pairs + 1023) / 1024, 148 * 16), 256, 0, s>>>(n_pairs, pk, krange, kmap,
                                                                                             c->key_dbits, sk);
    launch_counter() += 3;
  }
  sort_trace("pack", s);
  // the emitted 64-bit keys are dead after packing: their buffer is the sort's
  // ping-pong space (four passes end back in sk / pv)
  unsigned* tmp = reinterpret_cast<unsigned*>(pk);
  if (int st = sort_pairs(c, sk, pv, tmp, tmp + n_pairs + 1, n_pairs)) return st;
  sort_trace("radix", s);
  if (n_pairs > 0) {
    // runs of equal sort keys: full keys (into the dead emission buffer), then
    // the ids in (key, id) order into the second id buffer, which becomes the list
    const unsigned nb = (unsigned)((n_pairs + 255) / 256);
    unsigned long long* fk = pk;
    k_tie_keys<<<nb, 256, 0, s>>>(n_pairs, sk, pv, c->key_dbits, static_cast<const Geo*>(c->geo.p),
                                  static_cast<const double*>(c->cdirs.p), static_cast<const double*>(c->tdirs.p), cd,
                                  od, fk);
    // run statistics only with the work counters on (same-address atomics from
    // billions of entries would serialise on config 4)
    long long* long_runs = ensure<long long>(c->tie_long, (size_t)(n_pairs / 1024 + 2));
    if (!long_runs) return set_error(c, DRK_ERR_OOM, "tie runs");
    cudaMemsetAsync(long_runs, 0, sizeof(long long), s);
    sort_trace("tie_keys", s);
    k_tie_rank<<<nb, 256, 0, s>>>(n_pairs, sk, pv, fk, ids2,
                                  c->work_counters ? static_cast<unsigned long long*>(c->counters.p) : nullptr,
                                  long_runs);
    sort_trace("tie_rank", s);
    k_tie_long<<<64, 128, 0, s>>>(n_pairs, sk, fk, ids2, long_runs);
    sort_trace("tie_long", s);
    launch_counter() += 3;
    std::swap(c->pv, c->pidx);
  }
  k_tile_bounds<<<(unsigned)((n_pairs + 256) / 256), 256, 0, s>>>(n_pairs, sk, c->key_dbits, n_tiles, tileoff);
  DRK_COUNT_LAUNCH();
  mark(c, 4);
  sort_trace("bounds", s, true);
  *n_pairs_out = n_pairs;
  return DRK_OK;
}

// DRK_HOST_TRACE=1: host wall-clock checkpoints of run_forward on stderr
// (development aid for host-side gaps between the device stages)
struct HostTrace {
  bool on = getenv("DRK_HOST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  std::string line;
  void at(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    char b[64];
    snprintf(b, sizeof b, " %s %.2f", what, std::chrono::duration<double, std::milli>(now - last).count());
    line += b;
    last = now;
  }
  ~HostTrace() {
    if (on)
      fprintf(stderr, "[drk host] %s | total %.2f ms\n", line.c_str(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

int run_forward(drk_ctx* c, const drk_camera* cam, const drk_options* opt, float* color, float* depth,
                float* normal, float* alpha, const H2DPipe* pipe) {
  HostTrace ht;
  const Activated& A = c->act;
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0) || !(cam->fy > 0))
    return set_error(c, DRK_ERR_INVALID_ARG, "invalid camera");
  if (A.K < 3 || A.K > kMaxK) return set_error(c, DRK_ERR_UNSUPPORTED, "K must be in [3, 16]");
  cudaStream_t s = c->stream;
  mark(c, 1);
  c->cam = *cam;
  c->opt = *opt;
  c->camd = make_cam(cam);
  c->optd = make_opt(opt, A.terms);
  const CamD& cd = c->camd;
  const OptD& od = c->optd;
  const int n = A.n;
  const int n_tiles = cd.tiles_x * cd.tiles_y;
  const long long n_pix = (long long)cam->width * cam->height;
  unsigned long long* ctr = ensure<unsigned long long>(c->counters, C_COUNT);
  Geo* geo = ensure<Geo>(c->geo, n);
  if (!ensure<float4>(c->frame32, 3 * (size_t)n)) return set_error(c, DRK_ERR_OOM, "frame buffer");
  int4* bbox = ensure<int4>(c->bbox, n);
  int2* hullref = ensure<int2>(c->hullref, n);
  int* rowcnt = ensure<int>(c->rowcnt, n + 1);
  long long* rowoff = ensure<long long>(c->rowoff, n + 1);
  if (!ctr || !geo || !bbox || !hullref || !rowcnt || !rowoff) return set_error(c, DRK_ERR_OOM, "prep buffers");
  static_assert(sizeof(Geo) % 8 == 0, "Geo alignment");
  if (c->hull_cap < (long long)n * 96 + 1024) c->hull_cap = (long long)n * 96 + 1024;
  if (c->pts_cap < (long long)n * 260 + 1024) c->pts_cap = (long long)n * 260 + 1024;
  int2* ptsref = ensure<int2>(c->ptsref, n + 1);
  if (!ptsref) return set_error(c, DRK_ERR_OOM, "point refs");
  // K1 vertex cache: off for the first forward of an activation (the usual
  // single view), built on the second, used from the third (views of one
  // activation: multi-view batches, training views).  DRK_VCACHE=0: off.
  static const bool vc_on = !getenv("DRK_VCACHE") || atoi(getenv("DRK_VCACHE")) != 0;
  int k1_mode = 0;
  VertexCache vc;
  if (vc_on && n >= 4096 && !pipe) {
    const bool ready = c->vc_gen == c->act_gen && c->vc_alpha_min == opt->alpha_min && c->vc_ref.p;
    if (ready) {
      k1_mode = 2;
    } else if (c->act_renders >= 1) {
      // room for ~96 vertices per primitive, within an eighth of the free memory
      const long long cap = (long long)n * 96;
      const size_t bytes = sizeof(double) * 3 * (size_t)cap + sizeof(int2) * (size_t)n + 64;
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t have = c->vc_pool.bytes + c->vc_ref.bytes;
      if (bytes <= (free_b + have) / 8) {
        double* pool = ensure<double>(c->vc_pool, 3 * (size_t)cap);
        int2* ref = ensure<int2>(c->vc_ref, (size_t)n);
        unsigned long long* cur = ensure<unsigned long long>(c->vc_cursor, 1);
        if (pool && ref && cur) {
          k1_mode = 1;
          cudaMemsetAsync(cur, 0, sizeof(unsigned long long), s);
        }
      }
    }
    if (k1_mode) {
      vc.pool = static_cast<double*>(c->vc_pool.p);
      vc.cap = (long long)(c->vc_pool.bytes / (3 * sizeof(double)));
      vc.ref = static_cast<int2*>(c->vc_ref.p);
      vc.cursor = static_cast<unsigned long long*>(c->vc_cursor.p);
    }
  }
  // K1 with retry on hull-pool overflow
  DevBuf& ovf_buf = c->rows;  // reused as overflow list before rows are built
  for (int attempt = 0; attempt < 4; ++attempt) {
    double2* pool = ensure<double2>(c->hull, (size_t)c->hull_cap);
    double2* ppool = ensure<double2>(c->ptspool, (size_t)c->pts_cap);
    int* ovf = ensure<int>(ovf_buf, n + 1);
    if (!pool || !ovf || !ppool) return set_error(c, DRK_ERR_OOM, "hull pool");
    // the pipelined host-buffer forward zeroed the counters before its
    // activation (whose error counts they carry) on the first attempt
    const bool piped = pipe && attempt == 0;
    if (!piped) cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT, s);
    if (n > 0) {
      // warp per primitive; near-clipped / oversized polygons -> overflow list (k_prep1)
      const int mode = attempt == 0 ? k1_mode : (k1_mode ? 2 : 0);  // a retry reuses the cache built
      // pipelined: activation + K1 of each chunk of primitives as soon as its
      // parameters have crossed the link (the copies of later chunks overlap)
      const int nchunk = piped ? pipe->nchunk : 1;
      for (int q = 0; q < nchunk; ++q) {
        const int i0 = piped ? pipe->bounds[q] : 0, i1 = piped ? pipe->bounds[q + 1] : n;
        if (piped) {
          cudaStreamWaitEvent(s, pipe->ready[q], 0);
          activate_range(c, pipe->raw, i0, i1);
        }
        launch_prep_warp(mode, A, cd, od, geo, bbox, hullref, ppool, c->pts_cap, ptsref, rowcnt, ctr, ovf,
                         static_cast<float4*>(c->frame32.p), i0, i1, vc, s);
      }
      k_prep_hull<<<(unsigned)((2LL * n + 255) / 256), 256, 0, s>>>(n, ptsref, ppool, cd, od, bbox, hullref, pool,
                                                                    c->hull_cap, rowcnt, ctr);
    }
    launch_counter() += 2;
    unsigned long long h[C_COUNT];
    if (int st = read_counters(c, h)) return st;
    if (piped) {  // the activation's checks, deferred to the first read of the counters
      if (h[C_ERR_NONFINITE]) return set_error(c, DRK_ERR_NONFINITE, "raw parameters contain NaN/Inf");
      if (h[C_ERR_DEGEN_QUAT]) return set_error(c, DRK_ERR_DEGENERATE_QUAT, "quaternion norm below 1e-12");
    }
    if ((long long)h[C_PTS_POOL] > c->pts_cap) {
      c->pts_cap = (long long)h[C_PTS_POOL] + (long long)h[C_PTS_POOL] / 4 + 1024;
      if (attempt == 3) return set_error(c, DRK_ERR_OOM, "point pool retries");
      continue;
    }
    const long long n_ovf = (long long)h[C_POLY_OVERFLOW];
    if (n_ovf > 0) {
      // large-polygon path: 64k-vertex scratch per primitive, batches of 256
      const int cap = 65536;
      std::vector<int> list(n_ovf);
      cudaMemcpyAsync(list.data(), ovf, sizeof(int) * n_ovf, cudaMemcpyDeviceToHost, s);
      if (int st = cuda_check(c, cudaStreamSynchronize(s), "overflow list")) return st;
      // grow-only context buffers: a per-call cudaMalloc / cudaFree of the
      // 0.5 GB scratch stalled views with near-clipped primitives by 10-500 ms
      const int batch = 256;
      double2* scr = ensure<double2>(c->ovf_scr, (size_t)batch * 2 * (cap + 2));
      int* dl = ensure<int>(c->ovf_list, n_ovf);
      if (!scr || !dl) return set_error(c, DRK_ERR_OOM, "large polygon scratch");
      cudaMemcpyAsync(dl, list.data(), sizeof(int) * n_ovf, cudaMemcpyHostToDevice, s);
      for (long long b = 0; b < n_ovf; b += batch) {
        const int cnt = (int)std::min<long long>(batch, n_ovf - b);
        k_prep1<<<(cnt + 127) / 128, 128, 0, s>>>(A, cd, od, geo, bbox, hullref, pool, c->hull_cap, rowcnt, ctr,
                                                    dl + b, cnt, scr, cap, ovf);
      }
      if (int st = read_counters(c, h)) return st;
      if (h[C_POLY_FAIL]) return set_error(c, DRK_ERR_UNSUPPORTED, "support polygon above 65536 vertices");
    }
    if ((long long)h[C_HULL_POOL] <= c->hull_cap) {
      c->stats.poly_overflow = n_ovf;
      c->stats.primitives = (int64_t)h[C_VISIBLE];
      if (k1_mode == 1) {
        c->vc_gen = c->act_gen;
        c->vc_alpha_min = opt->alpha_min;
      }
      break;
    }
    c->hull_cap = (long long)h[C_HULL_POOL] + (long long)h[C_HULL_POOL] / 4 + 1024;
    if (attempt == 3) return set_error(c, DRK_ERR_OOM, "hull pool retries");
  }
  mark(c, 2);
  ht.at("k1");
  float prep_ms[2] = {0, 0};
  if (c->timing) {
    cudaEventSynchronize(c->ev[2]);
    prep_ms[0] = elapsed(c, 0, 1);
    prep_ms[1] = elapsed(c, 1, 2);
  }
  double* cdirs = ensure<double>(c->cdirs, 3 * (size_t)(cd.tiles_x + 1) * (cd.tiles_y + 1));
  double* tdirs = ensure<double>(c->tdirs, 3 * (size_t)n_tiles);
  if (!cdirs || !tdirs) return set_error(c, DRK_ERR_OOM, "tile rays");
  {
    const int nr = (cd.tiles_x + 1) * (cd.tiles_y + 1) + n_tiles;
    k_tile_rays<<<(nr + 127) / 128, 128, 0, s>>>(cd, cdirs, tdirs);
    DRK_COUNT_LAUNCH();
  }
  if (int st = plan_bands(c)) return st;
  ht.at("plan");
  // per-pixel state / replay
  double* pxstate = ensure<double>(c->pxstate, 8 * (size_t)n_pix);
  unsigned char* pxflag = ensure<unsigned char>(c->pxflag, (size_t)n_pix);
  int* pxstop = ensure<int>(c->pxstop, (size_t)n_pix);
  int* pxcomp = ensure<int>(c->pxcomp, (size_t)n_pix);
  int* redo = ensure<int>(c->redo, 2 * ((size_t)n_pix + 1) + 128);  // list + ordering scratch + counters
  c->redo_half = n_pix + 1;
  if (!pxstate || !pxflag || !redo || !pxstop || !pxcomp) return set_error(c, DRK_ERR_OOM, "pixel state");
  if (opt->record_replay > 0) {
    ensure<int>(c->replay_cnt, n_pix);
    ensure<int>(c->replay_ids, (size_t)n_pix * opt->record_replay);
    ensure<double>(c->replay_rec, 5 * (size_t)n_pix * opt->record_replay);
    if (!c->replay_cnt.p || !c->replay_ids.p || !c->replay_rec.p) return set_error(c, DRK_ERR_OOM, "replay buffers");
  }
  // bands of tile rows (one band unless the pairs of the frame would not fit)
  long long n_pairs_total = 0;
  float band_ms[4] = {0, 0, 0, 0};
  const int nb = (int)c->bands.size() - 1;
  // banded frames keep each band's sorted lists for the backward while free
  // memory stays above an eighth of the device (the next band's binning reuses
  // the pair buffers, so this only needs room for the ids and offsets)
  c->band_cache_valid = nb > 1 && opt->record_replay == 0;
  if (c->band_cache_valid) {
    c->band_ids.resize(nb);
    c->band_off.resize(nb);
  }
  // per-tile streamed lengths of the fast forward (the backward's dispatch order)
  unsigned* tcost = ensure<unsigned>(c->tile_cost, (size_t)n_tiles + 1);
  if (!tcost) return set_error(c, DRK_ERR_OOM, "tile costs");
  cudaMemsetAsync(tcost, 0, sizeof(unsigned) * n_tiles, s);
  c->tile_cost_valid = false;
  for (int b = 0; b < nb; ++b) {
    const int ty_lo = c->bands[b], ty_hi = c->bands[b + 1];
    mark(c, 2);
    long long n_pairs = 0;
    if (int st = bin_band(c, ty_lo, ty_hi, &n_pairs)) return st;
    ht.at("bin");
    n_pairs_total += n_pairs;
    if (c->band_cache_valid) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t need = sizeof(int) * (size_t)(n_pairs + 1) + sizeof(long long) * (size_t)(n_tiles + 1);
      const size_t have = c->band_ids[b].bytes + c->band_off[b].bytes;
      int* ids = nullptr;
      long long* offs = nullptr;
      if (free_b + have > need + total_b / 8) {
        ids = ensure<int>(c->band_ids[b], (size_t)n_pairs + 1);
        offs = ensure<long long>(c->band_off[b], (size_t)n_tiles + 1);
      }
      if (ids && offs) {
        cudaMemcpyAsync(ids, c->pv.p, sizeof(int) * (size_t)n_pairs, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(offs, c->tileoff.p, sizeof(long long) * (size_t)(n_tiles + 1), cudaMemcpyDeviceToDevice, s);
      } else {
        c->band_cache_valid = false;
        for (auto& d : c->band_ids) release(d);
        for (auto& d : c->band_off) release(d);
      }
    }
    RasterParams P = raster_params(c);
    P.pxflag = pxflag;
    P.pxstop = pxstop;
    if (c->validate_fast) {
      P.vstat = ensure<unsigned long long>(c->vstat, 32);
      if (!P.vstat) return set_error(c, DRK_ERR_OOM, "validation buffer");
    }
    P.color = color;
    P.depth = depth;
    P.normal = normal;
    P.alpha = alpha;
    P.pxstate = pxstate;
    if (opt->record_replay > 0) {
      P.replay_cap = opt->record_replay;
      P.replay_cnt = static_cast<int*>(c->replay_cnt.p);
      P.replay_ids = static_cast<int*>(c->replay_ids.p);
      P.replay_rec = static_cast<double*>(c->replay_rec.p);
    }
    P.tile_base = ty_lo * cd.tiles_x;
    P.tile_cost = tcost;
    c->tile_cost_valid = nb == 1 && raster_fast_eligible(P) && P.opt.raster_kernel != 1;
    P.fast_nt = choose_nt(c, n_pairs, (ty_hi - ty_lo) * cd.tiles_x);
    // Longest tile lists first (a shorter tail: config 1 -1.9%, config 2 -4% raster
    // time).  DRK_TILE_ORDER=0 forces row-major.
    static const int tile_order_mode = getenv("DRK_TILE_ORDER") ? atoi(getenv("DRK_TILE_ORDER")) : 1;
    if (tile_order_mode > 0 && raster_fast_eligible(P) && P.opt.raster_kernel != 1) {
      const int nt = (ty_hi - ty_lo) * cd.tiles_x;
      unsigned* tk = ensure<unsigned>(c->tord, 4 * (size_t)nt + 4);
      if (!tk) return set_error(c, DRK_ERR_OOM, "tile order");
      unsigned *tv = tk + nt + 1, *tk2 = tv + nt + 1, *tv2 = tk2 + nt + 1;
      launch_tile_order_keys(nt, cd.tiles_x, 0, P.tileoff, P.tile_base, tk, tv, s);
      launch_counter() += 1;
      if (int st = sort_pairs(c, tk, tv, tk2, tv2, nt)) return st;
      P.tile_order = reinterpret_cast<const int*>(tv);
    }
    launch_raster(P, (ty_hi - ty_lo) * cd.tiles_x, false, s, c->timing ? c->ev[5] : nullptr);
    mark(c, 6);
    if (int st = cuda_check(c, cudaGetLastError(), "raster")) return st;
    if (c->timing) {
      cudaEventSynchronize(c->ev[6]);
      for (int k = 0; k < 4; ++k) band_ms[k] += elapsed(c, 2 + k, 3 + k);
    }
  }
  c->n_pairs = n_pairs_total;
  ht.at("launch");
  unsigned long long h[C_COUNT];
  if (int st = read_counters(c, h)) return st;
  ht.at("raster");
  if (c->timing) {
    for (int i = 0; i < 2; ++i) c->stats.stage_ms[i] = prep_ms[i];
    for (int k = 0; k < 4; ++k) c->stats.stage_ms[2 + k] = band_ms[k];
  }
  c->stats.launches = launch_counter() - c->launch_base;
  c->stats.pairs = n_pairs_total;
  c->stats.streamed = (int64_t)h[C_STREAMED];
  c->stats.popped = (int64_t)h[C_POPPED];
  c->stats.composited = (int64_t)h[C_COMPOSITED];
  c->stats.near_ties = (int64_t)h[C_NEAR_TIES];
  c->stats.replay_overflow = (int64_t)h[C_REPLAY_OVERFLOW];
  c->stats.fp64_pixels = (int64_t)h[C_REDO_PIXELS];
  c->stats.reject_radius = (int64_t)h[C_REJECT_RADIUS];
  c->stats.reject_bracket = (int64_t)h[C_REJECT_BRACKET];
  c->stats.fp64_evals = (int64_t)h[C_FP64_EVALS];
  c->stats.ambiguous = (int64_t)h[C_AMBIGUOUS];
  c->stats.ring_miss = (int64_t)h[C_RING_MISS];
  c->stats.tie_runs = (int64_t)h[C_TIE_RUNS];
  c->stats.tie_members = (int64_t)h[C_TIE_MEMBERS];
  c->stats.tie_max_run = (int64_t)h[C_TIE_MAXRUN];
  c->stats.cache_appends = (int64_t)h[C_CACHE_APPEND];
  if (h[C_ERR_DEGEN_BASIS]) return set_error(c, DRK_ERR_DEGENERATE_BASIS, "adjacent endpoints nearly collinear");
  c->has_fwd = true;
  ++c->act_renders;
  return DRK_OK;
}

int run_backward_det(drk_ctx* c, const RasterParams& P, const std::vector<int>& bands,
                     int (*band_lists)(drk_ctx*, int, RasterParams&));

// Tile lists of band b of a banded frame for the deterministic backward: the
// forward's kept lists, or the band binned again.
static int det_band_lists(drk_ctx* c, int b, RasterParams& Q) {
  const int nb = (int)c->bands.size() - 1;
  if (c->band_cache_valid && (int)c->band_ids.size() == nb) {
    Q.lid = static_cast<const int*>(c->band_ids[b].p);
    Q.tileoff = static_cast<const long long*>(c->band_off[b].p);
    return DRK_OK;
  }
  long long np = 0;
  if (int st = bin_band(c, c->bands[b], c->bands[b + 1], &np)) return st;
  Q.lid = static_cast<const int*>(c->pv.p);
  Q.tileoff = static_cast<const long long*>(c->tileoff.p);
  Q.geo = static_cast<const Geo*>(c->geo.p);
  return DRK_OK;
}

int run_backward(drk_ctx* c, const float* raw, const drk_frame_grad* fg, float* grad_raw, float* d_center_world,
                 float* screen_grad, uint8_t* touched, int accumulate, int deterministic) {
  if (!c->has_fwd) return set_error(c, DRK_ERR_REPLAY_MISMATCH, "backward without a forward on this context");
  const Activated& A = c->act;
  const int n = A.n, K = A.K;
  // activated-space gradient rows, padded to a multiple of 4 floats so that
  // the warp-reduced sums go out as 16-byte vector atomics
  const int G = grad_row_stride(A.terms);
  cudaStream_t s = c->stream;
  float* gact = ensure<float>(c->gact, (size_t)G * n + 4);
  unsigned char* tch = ensure<unsigned char>(c->touched, n + 1);
  if (!gact || !tch) return set_error(c, DRK_ERR_OOM, "gradient buffers");
  cudaMemsetAsync(gact, 0, sizeof(float) * G * (size_t)n, s);
  cudaMemsetAsync(tch, 0, n + 1, s);
  RasterParams P = raster_params(c);
  P.pxstate = static_cast<double*>(c->pxstate.p);
  P.pxflag = static_cast<unsigned char*>(c->pxflag.p);
  P.pxstop = static_cast<int*>(c->pxstop.p);
  if (fg) {
    P.dC = fg->d_color;
    P.dD = fg->d_depth;
    P.dN = fg->d_normal;
    P.dA = fg->d_alpha;
  }
  P.gact = gact;
  P.G = G;
  P.touched = tch;
  const int n_tiles = c->camd.tiles_x * c->camd.tiles_y;
  // half-tile CTAs of 128 threads at 3 per SM (168 registers): 12 warps / SM
  // instead of 8 (config 2 backward 41.8 ms vs 43.4 ms); raster_kernel 7 or
  // DRK_BWD_NT=256 keep whole tiles
  static const int bwd_nt = getenv("DRK_BWD_NT") ? atoi(getenv("DRK_BWD_NT")) : 128;
  P.fast_nt = (c->opt.raster_kernel == 7 || (bwd_nt == 256 && c->opt.raster_kernel != 6)) ? 256 : 128;
  mark(c, 7);
  const int nb = (int)c->bands.size() - 1;
  if (deterministic) {
    // parallel, fixed accumulation order (drk_det.cu)
    std::vector<int> bands = c->bands.size() >= 2 ? c->bands : std::vector<int>{0, c->camd.tiles_y};
    if (int st = run_backward_det(c, P, bands, det_band_lists)) return st;
  } else if (nb <= 1) {
    // longest tile lists first, as in the forward
    static const int tile_order_mode = getenv("DRK_TILE_ORDER") ? atoi(getenv("DRK_TILE_ORDER")) : 1;
    if (tile_order_mode > 0 && n_tiles > 0) {
      unsigned* tk = ensure<unsigned>(c->tord, 4 * (size_t)n_tiles + 4);
      if (!tk) return set_error(c, DRK_ERR_OOM, "tile order");
      unsigned *tv = tk + n_tiles + 1, *tk2 = tv + n_tiles + 1, *tv2 = tk2 + n_tiles + 1;
      static const bool by_cost = !getenv("DRK_BWD_ORDER") || atoi(getenv("DRK_BWD_ORDER")) != 0;
      if (by_cost && c->tile_cost_valid && c->tile_cost.p)
        launch_tile_cost_keys(n_tiles, static_cast<const unsigned*>(c->tile_cost.p), tk, tv, s);
      else
        launch_tile_order_keys(n_tiles, c->camd.tiles_x, 0, P.tileoff, 0, tk, tv, s);
      launch_counter() += 1;
      if (int st = sort_pairs(c, tk, tv, tk2, tv2, n_tiles)) return st;
      P.tile_order = reinterpret_cast<const int*>(tv);
    }
    launch_raster(P, n_tiles, true, s);
  } else {
    // banded frame: re-bin each band, then its backward raster and the fp64
    // backward of its flagged pixels
    for (int b = 0; b < nb; ++b) {
      const int ty_lo = c->bands[b], ty_hi = c->bands[b + 1];
      long long np = 0;
      const bool cached = c->band_cache_valid && (int)c->band_ids.size() == nb;
      if (!cached) {
        if (int st = bin_band(c, ty_lo, ty_hi, &np)) return st;
      }
      RasterParams Q = raster_params(c);
      if (cached) {  // the forward's sorted lists of this band
        Q.lid = static_cast<const int*>(c->band_ids[b].p);
        Q.tileoff = static_cast<const long long*>(c->band_off[b].p);
      }
      Q.pxstate = P.pxstate;
      Q.pxflag = P.pxflag;
      Q.pxstop = P.pxstop;
      Q.dC = P.dC;
      Q.dD = P.dD;
      Q.dN = P.dN;
      Q.dA = P.dA;
      Q.gact = P.gact;
      Q.G = P.G;
      Q.touched = P.touched;
      Q.tile_base = ty_lo * c->camd.tiles_x;
      Q.fast_nt = P.fast_nt;
      const int y0 = ty_lo * kTile, y1 = std::min(ty_hi * kTile, c->camd.H);
      cudaMemsetAsync(Q.redo_count, 0, sizeof(unsigned), s);
      const long long npx = (long long)(y1 - y0) * c->camd.W;
      if (npx > 0)
        k_band_flagged<<<(unsigned)((npx + 255) / 256), 256, 0, s>>>(Q.pxflag, c->camd.W, y0, y1, Q.redo_list,
                                                                     Q.redo_count);
      launch_raster(Q, (ty_hi - ty_lo) * c->camd.tiles_x, true, s);
    }
  }
  mark(c, 8);
  if (int st = cuda_check(c, cudaGetLastError(), "raster bwd")) return st;
  if (deterministic)  // the fp64 sums of the fixed-order reduction
    launch_act_bwd(n, K, A.terms, raw, static_cast<const double*>(c->det_acc.p), G, tch,
                   static_cast<const Geo*>(c->geo.p), c->camd, grad_raw, d_center_world, screen_grad, touched,
                   accumulate, s);
  else
    launch_act_bwd(n, K, A.terms, raw, gact, G, tch, static_cast<const Geo*>(c->geo.p), c->camd, grad_raw,
                   d_center_world, screen_grad, touched, accumulate, s);
  DRK_COUNT_LAUNCH();
  mark(c, 9);
  if (int st = cuda_check(c, cudaGetLastError(), "activation bwd")) return st;
  if (int st = cuda_check(c, cudaStreamSynchronize(s), "backward")) return st;
  {
    unsigned long long h[C_COUNT];
    if (int st = read_counters(c, h)) return st;
    c->stats.bwd_warp_steps = (int64_t)h[C_BWD_WARPSTEPS];
    c->stats.bwd_lead_records = (int64_t)h[C_BWD_LEAD_RECORDS];
    cudaMemsetAsync(static_cast<unsigned long long*>(c->counters.p) + C_BWD_WARPSTEPS, 0,
                    2 * sizeof(unsigned long long), s);
  }
  if (c->timing) {
    c->stats.stage_ms[6] = elapsed(c, 7, 8);
    c->stats.stage_ms[7] = elapsed(c, 8, 9);
  }
  c->stats.launches = launch_counter() - c->launch_base;
  return DRK_OK;
}

int run_l1_loss(drk_ctx* c, const float* r, const float* t, int w, int h, double* loss, float* dcol) {
  launch_l1((long long)w * h * 3, r, t, loss, dcol, c->stream);
  return cuda_check(c, cudaGetLastError(), "l1 loss");
}

}  // namespace drk

using namespace drk;

extern "C" {

int drk_abi_version(void) { return DRK_ABI_VERSION; }
int drk_scalar_count(int k, int sh_terms) { return 3 + 4 + 2 * k + 3 + 3 * sh_terms; }

void drk_default_options(drk_options* o) {
  o->lowpass_radius = 0.5;
  o->alpha_min = 1.0 / 255.0;
  o->grazing_eps = 1e-6;
  o->background[0] = o->background[1] = o->background[2] = 1.0;
  o->early_stop_transmittance = 1e-4;
  o->sh_degree = 3;
  o->use_cache = 1;
  o->exact_sort = 0;
  o->presort = 2;
  o->threads = 1;
  o->record_replay = 0;
  o->fp64_alpha = 0;
  o->raster_kernel = 0;
}

const char* drk_status_string(int s) {
  switch (s) {
    case DRK_OK: return "ok";
    case DRK_ERR_GENERIC: return "error";
    case DRK_ERR_NONFINITE: return "non-finite parameters";
    case DRK_ERR_DEGENERATE_QUAT: return "degenerate quaternion";
    case DRK_ERR_DEGENERATE_BASIS: return "degenerate basis";
    case DRK_ERR_REPLAY_MISMATCH: return "replay mismatch";
    case DRK_ERR_DIMENSION: return "dimension mismatch";
    case DRK_ERR_INVALID_ARG: return "invalid argument";
    case DRK_ERR_CUDA: return "CUDA error";
    case DRK_ERR_OOM: return "out of device memory";
    case DRK_ERR_UNSUPPORTED: return "unsupported";
    case DRK_ERR_IO: return "i/o error";
    case DRK_ERR_CORRUPT_FILE: return "corrupt file";
    case DRK_ERR_VERSION: return "version mismatch";
    case DRK_ERR_DEGENERATE_FACE: return "degenerate face";
    case DRK_ERR_TOO_MANY_VERTICES: return "too many vertices";
    case DRK_ERR_PARSE: return "parse error";
    case DRK_ERR_EMPTY_MESH: return "empty mesh";
    case DRK_ERR_COMM: return "communication error";
  }
  return "unknown status";
}

int drk_ctx_create(int device, drk_ctx** out) {
  if (!out) return DRK_ERR_INVALID_ARG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return DRK_ERR_CUDA;
  }
  drk_ctx* c = new drk_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return DRK_ERR_CUDA;
  }
  c->own_stream = true;
  for (cudaEvent_t& e : c->ev) cudaEventCreate(&e);
  *out = c;
  return DRK_OK;
}

int drk_set_timing(drk_ctx* c, int enabled) {
  if (!c) return DRK_ERR_INVALID_ARG;
  c->timing = enabled != 0;
  return DRK_OK;
}

int drk_set_validation(drk_ctx* c, int enabled) {
  if (!c) return DRK_ERR_INVALID_ARG;
  c->validate_fast = enabled != 0;
  if (c->validate_fast) {
    cudaSetDevice(c->device);
    unsigned long long* v = ensure<unsigned long long>(c->vstat, 32);
    if (!v) return set_error(c, DRK_ERR_OOM, "validation buffer");
    cudaMemsetAsync(v, 0, 32 * sizeof(unsigned long long), c->stream);
  }
  return cuda_check(c, cudaGetLastError(), "validation");
}

int drk_get_validation(drk_ctx* c, double* out) {
  if (!c || !out) return DRK_ERR_INVALID_ARG;
  out[0] = out[1] = 0;
  if (!c->vstat.p) return DRK_OK;
  unsigned long long h[32];
  cudaMemcpyAsync(h, c->vstat.p, sizeof h, cudaMemcpyDeviceToHost, c->stream);
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "validation")) return st;
  std::memcpy(&out[0], &h[0], 8);
  std::memcpy(&out[1], &h[1], 8);
  return DRK_OK;
}

int drk_get_validation_detail(drk_ctx* c, double* out) {
  if (!c || !out) return DRK_ERR_INVALID_ARG;
  for (int i = 0; i < 22; ++i) out[i] = 0;
  if (!c->vstat.p) return DRK_OK;
  unsigned long long h[32];
  cudaMemcpyAsync(h, c->vstat.p, sizeof h, cudaMemcpyDeviceToHost, c->stream);
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "validation")) return st;
  std::memcpy(out, &h[2], 8 * 22);
  return DRK_OK;
}

int drk_measure_fp32_peak(drk_ctx* c, double* tflops) {
  if (!c || !tflops) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  *tflops = measure_fp32_peak(c->stream);
  return cuda_check(c, cudaGetLastError(), "fp32 peak");
}

void drk_ctx_destroy(drk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->h2d_stream) {
    cudaStreamSynchronize(c->h2d_stream);
    cudaStreamDestroy(c->h2d_stream);
  }
  for (cudaEvent_t e : c->h2d_ev)
    if (e) cudaEventDestroy(e);
  DevBuf* bufs[] = {&c->a_mu, &c->a_rot, &c->a_s, &c->a_th, &c->a_eta, &c->a_tau, &c->a_o, &c->a_sh,
                    &c->a_ex, &c->a_ey, &c->a_det, &c->a_thf, &c->a_invdetf, &c->a_piogf, &c->a_hf,
                    &c->a_psif, &c->a_rec, &c->pxflag, &c->pxstop, &c->vstat, &c->redo, &c->redo_cnt, &c->tile_cost, &c->planes64, &c->vc_pool, &c->vc_ref, &c->vc_cursor, &c->geo, &c->frame32, &c->bbox, &c->hullref, &c->hull, &c->ptspool, &c->ptsref, &c->rowcnt,
                    &c->rowoff, &c->rows, &c->rowpaircnt, &c->rowpairoff, &c->pk, &c->pv, &c->sk,
                    &c->hist, &c->sortoff, &c->tileoff, &c->cdirs, &c->tdirs, &c->bits,
                    &c->pxstate, &c->replay_cnt, &c->replay_rec, &c->replay_ids, &c->gact, &c->touched,
                    &c->counters, &c->scan_tmp, &c->loss_tmp, &c->scene_aos,
                    &c->loss_part, &c->ssim_f, &c->dens_code, &c->dens_pos,
                    &c->eval_scr, &c->eval_px, &c->eval_off, &c->ovf_scr, &c->ovf_list, &c->tord,
                    &c->rowest, &c->host_raw, &c->host_img, &c->pxcomp, &c->det_cnt, &c->det_base,
                    &c->det_rec, &c->det_id, &c->det_tile, &c->det_sort, &c->det_poff, &c->det_acc, &c->det_rowoff,
                    &c->comm_buf, &c->scan_tmp2, &c->replay_cid, &c->replay_cval, &c->pidx, &c->tie_long,
                    &c->det_tflag, &c->det_tpos, &c->det_tstart, &c->det_tprim};
  for (DevBuf* b : bufs) release(*b);
  for (DevBuf& b : c->band_ids) release(b);
  for (DevBuf& b : c->band_off) release(b);
  for (cudaEvent_t e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* drk_last_error(const drk_ctx* c) { return c ? c->err.c_str() : "null context"; }

int drk_set_stream(drk_ctx* c, void* stream) {
  if (!c) return DRK_ERR_INVALID_ARG;
  if (c->own_stream) cudaStreamDestroy(c->stream);
  c->stream = static_cast<cudaStream_t>(stream);
  c->own_stream = false;
  return DRK_OK;
}

int drk_get_stats(const drk_ctx* c, drk_stats* out) {
  if (!c || !out) return DRK_ERR_INVALID_ARG;
  *out = c->stats;
  return DRK_OK;
}

int drk_activate(drk_ctx* c, const float* raw, int n, int k, int sh_terms, drk_prims* out) {
  if (!c || n < 0 || (n > 0 && !raw)) return DRK_ERR_INVALID_ARG;
  if (k < 3 || k > kMaxK) return set_error(c, DRK_ERR_GENERIC, "K must be at least 3 (and at most 16 here)");
  cudaSetDevice(c->device);
  c->has_act = false;
  c->has_fwd = false;
  if (int st = launch_activate(c, raw, n, k, sh_terms)) return st;
  c->has_act = true;  // drk_forward_again now renders this set
  if (out) {
    const Activated& A = c->act;
    *out = drk_prims{A.mu, A.rot, A.s, A.th, A.eta, A.tau, A.o, A.sh, nullptr};
  }
  return DRK_OK;
}

int drk_forward(drk_ctx* c, const float* raw, int n, int k, int sh_terms, const drk_camera* cam,
                const drk_options* opt, float* color, float* depth, float* normal, float* alpha) {
  if (!c || !cam || !opt || n < 0 || (n > 0 && !raw)) return DRK_ERR_INVALID_ARG;
  if (k < 3 || k > kMaxK) return set_error(c, DRK_ERR_GENERIC, "K must be at least 3 (and at most 16 here)");
  cudaSetDevice(c->device);
  c->has_fwd = false;
  c->launch_base = launch_counter();
  mark(c, 0);
  c->has_act = false;
  if (int st = launch_activate(c, raw, n, k, sh_terms)) return st;
  c->has_act = true;
  return run_forward(c, cam, opt, color, depth, normal, alpha);
}

int drk_forward_again(drk_ctx* c, const drk_camera* cam, const drk_options* opt, float* color, float* depth,
                      float* normal, float* alpha) {
  if (!c || !cam || !opt) return DRK_ERR_INVALID_ARG;
  if (!c->has_act) return set_error(c, DRK_ERR_INVALID_ARG, "no activated primitives on this context");
  cudaSetDevice(c->device);
  c->has_fwd = false;
  c->launch_base = launch_counter();
  mark(c, 0);
  return run_forward(c, cam, opt, color, depth, normal, alpha);
}

int drk_forward_prims(drk_ctx* c, const drk_prims* prims, int n, int k, int sh_terms, const drk_camera* cam,
                      const drk_options* opt, float* color, float* depth, float* normal, float* alpha) {
  if (!c || !prims || !cam || !opt || n < 0) return DRK_ERR_INVALID_ARG;
  if (k < 3 || k > kMaxK) return set_error(c, DRK_ERR_GENERIC, "K must be at least 3 (and at most 16 here)");
  cudaSetDevice(c->device);
  c->has_fwd = false;
  c->launch_base = launch_counter();
  mark(c, 0);
  c->has_act = false;
  if (int st = launch_shape(c, prims, n, k, sh_terms)) return st;
  c->has_act = true;
  return run_forward(c, cam, opt, color, depth, normal, alpha);
}

// Device address of a page-locked host buffer (mapped under unified
// addressing), or null: the kernels then write the framebuffer straight into
// host memory (zero-copy) as tiles finish.
static float* mapped(float* p, bool* ok) {
  if (!p) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
    cudaGetLastError();
    *ok = false;
    return nullptr;
  }
  return static_cast<float*>(a.devicePointer);
}

int drk_forward_host(drk_ctx* c, const float* raw_host, int n, int k, int sh_terms, const drk_camera* cam,
                     const drk_options* opt, float* color_host, float* depth_host, float* normal_host,
                     float* alpha_host) {
  if (!c || !cam || !opt || n < 0) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  const size_t S = (size_t)drk_scalar_count(k, sh_terms);
  const size_t npix = (size_t)cam->width * cam->height;
  float* r = ensure<float>(c->host_raw, S * n + 1);
  float* img = ensure<float>(c->host_img, 8 * npix + 1);
  if (!r || !img) return set_error(c, DRK_ERR_OOM, "host staging");
  // Page-locked parameters of a large scene: copied in chunks of primitives on
  // a second stream, each chunk's activation and K1 (per-primitive polygons,
  // the longest prep stage) launched as soon as it has landed, so the copy
  // overlaps them (config 1: the 29.6 MB upload hides behind K1).
  // DRK_H2D_CHUNKS=1 turns the pipeline off.
  static const int env_chunks = getenv("DRK_H2D_CHUNKS") ? atoi(getenv("DRK_H2D_CHUNKS")) : 4;
  const int nchunk = std::max(1, std::min(8, n >= 65536 ? env_chunks : 1));
  bool piped = nchunk > 1 && k >= 3 && k <= kMaxK;
  if (piped) {
    cudaPointerAttributes pa;
    piped = cudaPointerGetAttributes(&pa, raw_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
  }
  if (piped && !c->h2d_stream) {
    bool ok = cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking) == cudaSuccess;
    for (int q = 0; q < 9 && ok; ++q) ok = cudaEventCreateWithFlags(&c->h2d_ev[q], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      piped = false;
    }
  }
  H2DPipe pipe;
  if (piped) {
    pipe.raw = r;
    pipe.nchunk = nchunk;
    // the copies may start once the context's stream is past earlier work on r
    cudaEventRecord(c->h2d_ev[8], c->stream);
    cudaStreamWaitEvent(c->h2d_stream, c->h2d_ev[8], 0);
    for (int q = 0; q <= nchunk; ++q) pipe.bounds[q] = (int)((long long)n * q / nchunk);
    for (int q = 0; q < nchunk; ++q) {
      const size_t i0 = pipe.bounds[q], w = pipe.bounds[q + 1] - pipe.bounds[q];
      cudaMemcpy2DAsync(r + i0, sizeof(float) * n, raw_host + i0, sizeof(float) * n, sizeof(float) * w, S,
                        cudaMemcpyHostToDevice, c->h2d_stream);
      cudaEventRecord(c->h2d_ev[q], c->h2d_stream);
      pipe.ready[q] = c->h2d_ev[q];
    }
  } else {
    cudaMemcpyAsync(r, raw_host, sizeof(float) * S * n, cudaMemcpyHostToDevice, c->stream);
  }
  // forward on device parameters: the whole activation up front, or (piped)
  // the counters zeroed here and the activation issued chunk by chunk from K1
  auto forward = [&](float* col, float* dep, float* nor, float* alp) -> int {
    if (!piped) return drk_forward(c, r, n, k, sh_terms, cam, opt, col, dep, nor, alp);
    if (!c || !cam || !opt || n < 0) return DRK_ERR_INVALID_ARG;
    c->has_fwd = false;
    c->launch_base = launch_counter();
    mark(c, 0);
    c->has_act = false;
    int st = activate_setup(c, n, k, sh_terms);
    if (!st) {
      cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned long long) * C_COUNT, c->stream);
      c->has_act = true;
      st = run_forward(c, cam, opt, col, dep, nor, alp, &pipe);
    }
    if (st) {
      // an early error may leave chunk copies in flight: none may outlive the call
      c->has_act = false;
      cudaStreamSynchronize(c->h2d_stream);
    }
    return st;
  };
  // Page-locked outputs: the raster kernels store the pixels straight into
  // them as tiles finish (zero-copy; config 1 e2e 25.9 ms vs 26.8 ms with a
  // band-wise staging copy).  DRK_HOST_OUT=copy forces device framebuffers.
  static const bool zero_copy = !getenv("DRK_HOST_OUT") || std::string(getenv("DRK_HOST_OUT")) != "copy";
  if (zero_copy) {
    bool ok = true;
    float* mc = mapped(color_host, &ok);
    float* md = mapped(depth_host, &ok);
    float* mn = mapped(normal_host, &ok);
    float* ma = mapped(alpha_host, &ok);
    if (ok) {
      const int st = forward(mc, md, mn, ma);
      if (st) return st;
      return cuda_check(c, cudaStreamSynchronize(c->stream), "forward_host");
    }
  }
  // not page-locked (or not mapped): device framebuffers, copied out afterwards
  float* dcol = color_host ? img : nullptr;
  float* ddep = depth_host ? img + 3 * npix : nullptr;
  float* dnor = normal_host ? img + 4 * npix : nullptr;
  float* dalp = alpha_host ? img + 7 * npix : nullptr;
  if (int st = forward(dcol, ddep, dnor, dalp)) return st;
  if (color_host) cudaMemcpyAsync(color_host, dcol, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost, c->stream);
  if (depth_host) cudaMemcpyAsync(depth_host, ddep, sizeof(float) * npix, cudaMemcpyDeviceToHost, c->stream);
  if (normal_host) cudaMemcpyAsync(normal_host, dnor, sizeof(float) * 3 * npix, cudaMemcpyDeviceToHost, c->stream);
  if (alpha_host) cudaMemcpyAsync(alpha_host, dalp, sizeof(float) * npix, cudaMemcpyDeviceToHost, c->stream);
  return cuda_check(c, cudaStreamSynchronize(c->stream), "forward_host");
}

int drk_set_counters(drk_ctx* c, int enabled) {
  if (!c) return DRK_ERR_INVALID_ARG;
  c->work_counters = enabled != 0;
  return DRK_OK;
}

int drk_set_det_chunk_limit(drk_ctx* c, int64_t records) {
  if (!c || records < 0) return DRK_ERR_INVALID_ARG;
  c->det_chunk_limit = records;
  return DRK_OK;
}

int drk_set_band_limit(drk_ctx* c, int64_t pairs) {
  if (!c || pairs < 0) return DRK_ERR_INVALID_ARG;
  c->band_pair_limit = pairs;
  return DRK_OK;
}

int drk_get_bands(const drk_ctx* c, int32_t* n_bands) {
  if (!c || !n_bands) return DRK_ERR_INVALID_ARG;
  *n_bands = c->bands.empty() ? 0 : (int32_t)c->bands.size() - 1;
  return DRK_OK;
}

int drk_eval_sorting(drk_ctx* c, double* out4) {
  if (!c || !out4) return DRK_ERR_INVALID_ARG;
  if (!c->has_fwd) return set_error(c, DRK_ERR_INVALID_ARG, "no forward on this context");
  if (c->bands.size() > 2) return set_error(c, DRK_ERR_UNSUPPORTED, "tile lists of a banded frame are not kept");
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  const int n_tiles = c->camd.tiles_x * c->camd.tiles_y;
  std::vector<long long> off(n_tiles + 1);
  cudaMemcpyAsync(off.data(), c->tileoff.p, sizeof(long long) * (n_tiles + 1), cudaMemcpyDeviceToHost, s);
  if (int st = cuda_check(c, cudaStreamSynchronize(s), "eval_sorting offsets")) return st;
  const size_t n_pix = (size_t)c->cam.width * c->cam.height;
  double* tau = ensure<double>(c->eval_px, 2 * n_pix + n_pix / 8 + 8);
  if (!tau) return set_error(c, DRK_ERR_OOM, "eval_sorting pixel buffers");
  double* mae = tau + n_pix;
  unsigned char* flag = reinterpret_cast<unsigned char*>(mae + n_pix);
  cudaMemsetAsync(flag, 0, n_pix, s);
  // tile chunks whose scratch (256 pixels x 3 L doubles per tile) fits the budget
  const long long budget = 1LL << 27;  // doubles (1 GiB)
  long long maxL = 0;
  for (int t = 0; t < n_tiles; ++t) maxL = std::max(maxL, off[t + 1] - off[t]);
  double* scr = ensure<double>(c->eval_scr, (size_t)std::max(budget, 768 * maxL));
  long long* doff = ensure<long long>(c->eval_off, (size_t)n_tiles + 1);
  if (!scr || !doff) return set_error(c, DRK_ERR_OOM, "eval_sorting scratch");
  RasterParams P = raster_params(c);
  std::vector<long long> chunk_off;
  int t0 = 0;
  while (t0 < n_tiles) {
    chunk_off.clear();
    long long used = 0;
    int t1 = t0;
    while (t1 < n_tiles) {
      const long long need = 768 * (off[t1 + 1] - off[t1]);
      if (t1 > t0 && used + need > std::max(budget, 768 * maxL)) break;
      chunk_off.push_back(used);
      used += need;
      ++t1;
    }
    cudaMemcpyAsync(doff, chunk_off.data(), sizeof(long long) * chunk_off.size(), cudaMemcpyHostToDevice, s);
    launch_eval_sorting(P, t0, t1, doff, scr, c->opt.use_cache, tau, mae, flag, s);
    DRK_COUNT_LAUNCH();
    if (int st = cuda_check(c, cudaStreamSynchronize(s), "eval_sorting")) return st;  // chunk_off reused
    t0 = t1;
  }
  double* dout = reinterpret_cast<double*>(doff);
  launch_eval_sorting_reduce(c->camd, static_cast<const long long*>(c->tileoff.p), tau, mae, flag, dout, s);
  DRK_COUNT_LAUNCH();
  cudaMemcpyAsync(out4, dout, sizeof(double) * 4, cudaMemcpyDeviceToHost, s);
  return cuda_check(c, cudaStreamSynchronize(s), "eval_sorting");
}

// Banded frame: the per-band lists the forward kept (ids + per-tile offsets;
// bands are tile-row ranges in order, so concatenating them keeps tile order),
// keys recomputed per band.
static int banded_tile_lists(drk_ctx* c, int64_t* total, int64_t* offsets, int32_t* ids, double* keys) {
  const int nb = (int)c->bands.size() - 1;
  if (!(c->band_cache_valid && (int)c->band_ids.size() == nb))
    return set_error(c, DRK_ERR_UNSUPPORTED, "tile lists of this banded frame were not kept (device memory)");
  const int n_tiles = c->camd.tiles_x * c->camd.tiles_y;
  std::vector<int64_t> off_b((size_t)n_tiles + 1);
  int64_t base = 0;
  if (offsets) offsets[0] = 0;
  for (int b = 0; b < nb; ++b) {
    cudaMemcpyAsync(off_b.data(), c->band_off[b].p, sizeof(int64_t) * (n_tiles + 1), cudaMemcpyDeviceToHost,
                    c->stream);
    if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "band offsets")) return st;
    const long long np = off_b[n_tiles];
    const int t0 = c->bands[b] * c->camd.tiles_x, t1 = c->bands[b + 1] * c->camd.tiles_x;
    if (offsets)
      for (int t = t0; t < t1; ++t) offsets[t + 1] = base + off_b[t + 1];
    if (ids && np > 0) {
      std::vector<unsigned> v((size_t)np);
      cudaMemcpyAsync(v.data(), c->band_ids[b].p, sizeof(unsigned) * np, cudaMemcpyDeviceToHost, c->stream);
      if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "band ids")) return st;
      for (long long i = 0; i < np; ++i) ids[base + i] = (int32_t)v[i];
    }
    if (keys && np > 0) {
      DevBuf tmp;
      double* kd = ensure<double>(tmp, (size_t)np);
      if (!kd) return set_error(c, DRK_ERR_OOM, "key buffer");
      k_full_keys_off<<<(unsigned)((np + 255) / 256), 256, 0, c->stream>>>(
          np, static_cast<const long long*>(c->band_off[b].p), n_tiles, static_cast<const unsigned*>(c->band_ids[b].p),
          static_cast<const Geo*>(c->geo.p), static_cast<const double*>(c->cdirs.p),
          static_cast<const double*>(c->tdirs.p), c->camd, c->optd, kd);
      cudaMemcpyAsync(keys + base, kd, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream);
      const int st = cuda_check(c, cudaStreamSynchronize(c->stream), "band keys");
      release(tmp);
      if (st) return st;
    }
    base += np;
  }
  if (total) *total = base;
  return DRK_OK;
}

int drk_get_tile_lists(drk_ctx* c, int64_t* total, int64_t* offsets, int32_t* ids, double* keys) {
  if (!c || !c->has_fwd) return c ? set_error(c, DRK_ERR_INVALID_ARG, "no forward on this context") : DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (c->bands.size() > 2) return banded_tile_lists(c, total, offsets, ids, keys);
  if (total) *total = c->n_pairs;
  const int n_tiles = c->camd.tiles_x * c->camd.tiles_y;
  if (offsets)
    cudaMemcpyAsync(offsets, c->tileoff.p, sizeof(int64_t) * (n_tiles + 1), cudaMemcpyDeviceToHost, c->stream);
  std::vector<unsigned> v;
  if (ids) {
    v.resize(c->n_pairs);
    cudaMemcpyAsync(v.data(), c->pv.p, sizeof(unsigned) * c->n_pairs, cudaMemcpyDeviceToHost, c->stream);
  }
  if (keys && c->n_pairs > 0) {
    // the sort carries truncated keys; the full fp64 keys are recomputed
    DevBuf tmp;
    double* kd = ensure<double>(tmp, c->n_pairs);
    if (!kd) return set_error(c, DRK_ERR_OOM, "key buffer");
    k_full_keys<<<(unsigned)((c->n_pairs + 255) / 256), 256, 0, c->stream>>>(
        c->n_pairs, static_cast<const unsigned*>(c->sk.p), static_cast<const unsigned*>(c->pv.p), c->key_dbits,
        static_cast<const Geo*>(c->geo.p), static_cast<const double*>(c->cdirs.p),
        static_cast<const double*>(c->tdirs.p), c->camd, c->optd, kd);
    cudaMemcpyAsync(keys, kd, sizeof(double) * c->n_pairs, cudaMemcpyDeviceToHost, c->stream);
    const int st = cuda_check(c, cudaStreamSynchronize(c->stream), "tile keys");
    release(tmp);
    if (st) return st;
  }
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "tile lists")) return st;
  for (int64_t i = 0; ids && i < c->n_pairs; ++i) ids[i] = (int32_t)v[i];
  return DRK_OK;
}

// pixel state (8 doubles per pixel) -> colour, depth, normal, alpha planes
__global__ void k_split_state(long long npix, const double* __restrict__ st, double* color, double* depth,
                              double* normal, double* alpha) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const double* q = st + 8 * p;
  for (int k = 0; k < 3; ++k) {
    color[3 * p + k] = q[k];
    normal[3 * p + k] = q[4 + k];
  }
  depth[p] = q[3];
  alpha[p] = q[7];
}

int drk_get_framebuffers_f64(drk_ctx* c, double* color, double* depth, double* normal, double* alpha) {
  if (!c || !c->has_fwd) return c ? set_error(c, DRK_ERR_INVALID_ARG, "no forward on this context") : DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  const size_t npix = (size_t)c->cam.width * c->cam.height;
  if (npix == 0) return DRK_OK;
  double* d = ensure<double>(c->planes64, 8 * npix);
  if (!d) return set_error(c, DRK_ERR_OOM, "framebuffer planes");
  k_split_state<<<(unsigned)((npix + 255) / 256), 256, 0, c->stream>>>((long long)npix,
                                                                       static_cast<const double*>(c->pxstate.p), d,
                                                                       d + 3 * npix, d + 4 * npix, d + 7 * npix);
  DRK_COUNT_LAUNCH();
  if (color) cudaMemcpyAsync(color, d, sizeof(double) * 3 * npix, cudaMemcpyDeviceToHost, c->stream);
  if (depth) cudaMemcpyAsync(depth, d + 3 * npix, sizeof(double) * npix, cudaMemcpyDeviceToHost, c->stream);
  if (normal) cudaMemcpyAsync(normal, d + 4 * npix, sizeof(double) * 3 * npix, cudaMemcpyDeviceToHost, c->stream);
  if (alpha) cudaMemcpyAsync(alpha, d + 7 * npix, sizeof(double) * npix, cudaMemcpyDeviceToHost, c->stream);
  return cuda_check(c, cudaStreamSynchronize(c->stream), "framebuffers");
}

__global__ void k_replay_compact(long long npix, int cap, const int* __restrict__ cnt, const long long* __restrict__ off,
                                 const int* __restrict__ ids, const double* __restrict__ rec, int* cid, double* cval) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const int n = min(cnt[p], cap);
  const long long o = off[p];
  for (int j = 0; j < n; ++j) {
    cid[o + j] = ids[p * cap + j];
    for (int q = 0; q < 5; ++q) cval[5 * (o + j) + q] = rec[5 * (p * cap + j) + q];
  }
}

int drk_get_replay(drk_ctx* c, int64_t* total, int64_t* offsets, int32_t* ids, double* vals) {
  if (!c || !c->has_fwd || c->opt.record_replay <= 0)
    return c ? set_error(c, DRK_ERR_INVALID_ARG, "no replay recorded") : DRK_ERR_INVALID_ARG;
  if (c->stats.replay_overflow) return set_error(c, DRK_ERR_UNSUPPORTED, "replay capacity exceeded");
  cudaSetDevice(c->device);
  const size_t npix = (size_t)c->cam.width * c->cam.height;
  const int cap = c->opt.record_replay;
  std::vector<int> cnt(npix);
  cudaMemcpyAsync(cnt.data(), c->replay_cnt.p, sizeof(int) * npix, cudaMemcpyDeviceToHost, c->stream);
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "replay")) return st;
  int64_t tot = 0;
  for (size_t p = 0; p < npix; ++p) tot += cnt[p];
  if (total) *total = tot;
  if (offsets) {
    offsets[0] = 0;
    for (size_t p = 0; p < npix; ++p) offsets[p + 1] = offsets[p] + cnt[p];
  }
  if ((!ids && !vals) || tot == 0) return DRK_OK;
  // compact the per-pixel slots (npix x cap) on the device; copy only the records
  long long* off_d = ensure<long long>(c->scan_tmp2, npix + 1);
  int* cid = ensure<int>(c->replay_cid, (size_t)tot);
  double* cval = ensure<double>(c->replay_cval, 5 * (size_t)tot);
  if (!off_d || !cid || !cval) return set_error(c, DRK_ERR_OOM, "replay compaction");
  if (int st = exclusive_scan<int>(c, static_cast<const int*>(c->replay_cnt.p), (long long)npix, off_d, nullptr))
    return st;
  k_replay_compact<<<(unsigned)((npix + 255) / 256), 256, 0, c->stream>>>(
      (long long)npix, cap, static_cast<const int*>(c->replay_cnt.p), off_d, static_cast<const int*>(c->replay_ids.p),
      static_cast<const double*>(c->replay_rec.p), cid, cval);
  if (ids) cudaMemcpyAsync(ids, cid, sizeof(int) * tot, cudaMemcpyDeviceToHost, c->stream);
  if (vals) cudaMemcpyAsync(vals, cval, sizeof(double) * 5 * tot, cudaMemcpyDeviceToHost, c->stream);
  return cuda_check(c, cudaStreamSynchronize(c->stream), "replay");
}

int drk_backward(drk_ctx* c, const float* raw, const drk_frame_grad* fg, float* grad_raw, float* d_center_world,
                 float* screen_grad, uint8_t* touched, int accumulate, int deterministic) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (grad_raw && !raw) return set_error(c, DRK_ERR_INVALID_ARG, "grad_raw needs the raw parameters");
  return run_backward(c, raw, fg, grad_raw, d_center_world, screen_grad, touched, accumulate, deterministic);
}

int drk_get_prim_grads(drk_ctx* c, const float** grads, int* stride) {
  if (!c || !grads || !stride) return DRK_ERR_INVALID_ARG;
  *grads = static_cast<const float*>(c->gact.p);
  *stride = (3 + 9 + 2 * c->act.K + 3 + 3 * c->act.terms + 3) & ~3;
  return DRK_OK;
}

int drk_debug_alpha_bound(drk_ctx* c, int64_t samples, uint64_t seed, double* max_ratio, double* max_abs) {
  if (!c || !max_ratio || !max_abs || c->act.n <= 0) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  unsigned long long* out = ensure<unsigned long long>(c->bits, 4);
  if (!out) return set_error(c, DRK_ERR_OOM, "alpha bound");
  RasterParams P = raster_params(c);
  launch_alpha_bound(P.S, c->act.n, samples, seed, out, c->stream);
  unsigned long long h[2];
  cudaMemcpyAsync(h, out, sizeof h, cudaMemcpyDeviceToHost, c->stream);
  if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "alpha bound")) return st;
  std::memcpy(max_ratio, &h[0], sizeof(double));
  std::memcpy(max_abs, &h[1], sizeof(double));
  return DRK_OK;
}

int drk_l1_loss(drk_ctx* c, const float* rendered, const float* target, int width, int height, double* loss_out,
                float* d_color) {
  if (!c || !rendered || !target || !loss_out || width < 0 || height < 0) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_l1_loss(c, rendered, target, width, height, loss_out, d_color);
}

int drk_adam_step(drk_ctx* c, float* params, const float* grads, float* m, float* v, int n, int k, int sh_terms,
                  int64_t* step, const drk_adam_config* cfg) {
  if (!c || !params || !grads || !m || !v || !step || !cfg || n < 0) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  *step += 1;
  return run_adam(c, params, grads, m, v, n, k, sh_terms, *step, cfg);
}

}  // extern "C"
