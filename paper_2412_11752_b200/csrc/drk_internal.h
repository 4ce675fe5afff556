// Host-side internals shared by the kernel launchers and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "drk_b200.h"
#include "drk_device.cuh"

namespace drk {

// DRK_SORT_TRACE=1: device-time checkpoints of the binning sort on stderr
// (development aid: per-phase CUDA events, printed when the phase list closes)
inline bool sort_trace_on() {
  static const bool on = getenv("DRK_SORT_TRACE") != nullptr;
  return on;
}
inline void sort_trace(const char* what, cudaStream_t s, bool flush = false) {
  if (!sort_trace_on()) return;
  static std::vector<std::pair<std::string, cudaEvent_t>> evs;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  evs.emplace_back(what, e);
  if (!flush) return;
  cudaEventSynchronize(e);
  std::string line;
  for (size_t i = 1; i < evs.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, evs[i - 1].second, evs[i].second);
    char b[96];
    snprintf(b, sizeof b, " %s %.3f", evs[i].first.c_str(), ms);
    line += b;
  }
  fprintf(stderr, "[drk sort]%s\n", line.c_str());
  for (auto& x : evs) cudaEventDestroy(x.second);
  evs.clear();
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// Process-wide count of kernels this library has launched (drk_stats.launches).
// Atomic: MultiViewRenderer drives several contexts from concurrent host threads.
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}

// Runs a function once per (call site, device), thread-safe.  Function attributes
// such as cudaFuncAttributeMaxDynamicSharedMemorySize are per device, so a
// process-wide flag would leave a second GPU without them.
struct PerDeviceOnce {
  static constexpr int kMaxDevices = 64;
  std::once_flag flags[kMaxDevices];
  template <class F>
  void operator()(F&& f) {
    int d = 0;
    cudaGetDevice(&d);
    std::call_once(flags[d & (kMaxDevices - 1)], std::forward<F>(f));
  }
};
#define DRK_COUNT_LAUNCH() (++::drk::launch_counter())

// Grow-only device allocation; returns nullptr on OOM.
void* ensure_bytes(DevBuf& b, size_t bytes);
template <class T>
T* ensure(DevBuf& b, size_t count) {
  return static_cast<T*>(ensure_bytes(b, (count ? count : 1) * sizeof(T)));
}
void release(DevBuf& b);

// Per-primitive, per-view record (fp64).  num = (mu - o) . R_z with the op
// order of classify_intersect (geometry.cpp:40-52); proj = projected centre.
struct Geo {
  double num;
  double rz[3];
  double rx[3];
  double ry[3];
  double mu[3];
  double ppx, ppy, projz;  // projected centre (valid iff has_proj); projz = +inf if not
  double r2max;            // (s_max f_vis)^2 (1+1e-9): beyond it alpha_kernel < alpha_min
  double dp2max;           // 2 s_l^2 ln(o / alpha_min) (1+1e-9): low-pass floor bound / cos^2
  int has_proj;
  int visible;
  float fvis2;             // f_vis^2 (fp32, as ShapeView psif[12 i + 8])
  int pad_;                // 160 bytes: a multiple of 16 (cp.async.bulk staging of the fast forward)
};
static_assert(sizeof(Geo) == 160, "Geo record size");

struct Activated {
  const double *mu, *rot, *s, *th, *eta, *tau, *o;
  const float* sh;  // n x terms x 3 (AoS)
  const double* sh64;  // optional fp64 copy (drk_prims.sh64) for the fp64 pixel path, or nullptr
  const double *ex, *ey, *det;
  const float *thf, *invdetf, *piogf, *hf, *psif;
  const float* rec;  // fast-kernel shape records (K == 8), else nullptr
  int n, K, terms;
};

struct RasterParams {
  CamD cam;
  OptD opt;
  const long long* tileoff;
  const int* lid;  // sorted tile lists: primitive ids (offsets in tileoff)
  const Geo* geo;
  ShapeView S;
  const float* sh;
  const double* sh64;  // optional fp64 SH (fp64 pixel path colours), or nullptr
  int terms;  // stored SH rows per primitive
  float *color, *depth, *normal, *alpha;
  double* pxstate;  // 8 doubles per pixel: C(3, incl. background), D, N(3), A
  int* replay_cnt;
  double* replay_rec;  // 5 doubles per record
  int* replay_ids;
  int replay_cap;
  // backward
  const float *dC, *dD, *dN, *dA;
  float* gact;  // activated-space gradients, fp32, row stride G (multiple of 4)
  int G;
  unsigned char* touched;
  unsigned long long* counters;
  unsigned char* pxflag;  // 1 = pixel needs the fp64 re-render (uncertain termination)
  int* redo_list;         // flagged pixel indices (forward fp32 pass appends)
  int* redo_tmp;          // scratch of the same size (order_redo_list), or null
  unsigned* redo_hist;    // 128 counters of order_redo_list
  unsigned* tile_cost;    // fast forward: list entries each tile streamed before its pixels saturated (backward tile order), or null
  unsigned int* redo_count;
  const float4* frame32;  // per prim: (R_x, a_x), (R_y, a_y), (R_z, a_z) with a = o - mu, fp32 (backward)
  int tile_base;          // first tile of this launch (banded frames: tile rows processed band by band)
  const float* shrec;     // fast kernel: per-primitive fp32 shape records (K == 8)
  int* pxstop;            // composites until saturation per pixel (INT_MAX: never), written by the forward
  int fast_nt;            // fast forward: threads per CTA (256: tile, 128: half tile), raster_fast_nt
  int no_counters;        // fast forward: work counters compiled out (drk_set_counters(ctx, 0))
  const int* tile_order;  // fast forward: band-local tile of each CTA (longest lists first), or null = row-major
  unsigned long long* vstat;  // fast kernel validation: max |a32 - a64| / bound, max |a32 - a64| (double bits)
  int* pxcomp;                // forward: composited entries per pixel (the deterministic backward's record counts)
  // deterministic backward (drk_backward(..., deterministic = 1)): every composited
  // record writes its gradient row to det_rec[det_base[slot] + k - det_off] (slot =
  // tile * 256 + row-major pixel in the tile, k = composite index in the pixel)
  // instead of adding it atomically; records are reduced per primitive afterwards
  // in (tile, pixel, composite) order (reference grad.cpp:327-368)
  double* det_rec;   // fp64 rows (reference-precision frames), or
  float* det_rec32;  // fp32 rows (fast-kernel frames: their gradients are fp32 already; half the bytes)
  int* det_id;
  int* det_tile;
  const long long* det_base;
  long long det_off, det_cap;
};

// Record index of a composited (pixel, k) in the deterministic backward, or -1
// (counted in C_DET_OVERFLOW) when the backward composites more entries than
// the forward counted.
__device__ __forceinline__ long long det_row(const RasterParams& P, int x, int y, int k, int id) {
  const int tile = (y >> 4) * P.cam.tiles_x + (x >> 4);
  const long long slot = (long long)tile * 256 + (y & 15) * 16 + (x & 15);
  const long long r = P.det_base[slot] + k - P.det_off;
  if (k >= P.pxcomp[(size_t)y * P.cam.W + x] || r < 0 || r >= P.det_cap) {
    atomicAdd(&P.counters[C_DET_OVERFLOW], 1ull);
    return -1;
  }
  P.det_id[r] = id;
  P.det_tile[r] = tile;
  return r;
}

void launch_raster(const RasterParams& P, int n_tiles, bool bwd, cudaStream_t s, cudaEvent_t mid = nullptr);
bool raster_fast_eligible(const RasterParams& P);
void launch_raster_fast(const RasterParams& P, int n_tiles, bool validate, cudaStream_t s);
int raster_fast_nt(long long pairs, int n_tiles);
void launch_raster_bwd_fast(const RasterParams& P, int n_tiles, cudaStream_t s);
void launch_shape_rec(const ShapeView& S, int i0, int i1, float* rec, cudaStream_t s);
// Activation split for the host-buffer pipeline (drk_forward_host): buffers and
// the Activated view first, then kernels over primitive ranges as their
// parameters arrive.
int activate_setup(drk_ctx* c, int n, int K, int terms);
// K1 vertex cache (several views of one activation): world-space vertices of
// the wedge-tree leaves, vref[i] = (offset, count) (drk_prep.cu k_prep_warp)
struct VertexCache {
  double* pool = nullptr;
  long long cap = 0;  // vertices
  int2* ref = nullptr;
  unsigned long long* cursor = nullptr;
};
// mode 0: plain K1; 1: build the cache; 2: use it
void launch_prep_warp(int mode, const Activated& A, const CamD& cam, const OptD& opt, Geo* geo, int4* bbox,
                      int2* hullref, double2* ppool, long long pts_cap, int2* ptsref, int* rowcnt,
                      unsigned long long* ctr, int* ovf, float4* frame32, int i0, int i1, const VertexCache& vc,
                      cudaStream_t s);
void activate_range(drk_ctx* c, const float* raw, int i0, int i1);
double measure_fp32_peak(cudaStream_t s);
void launch_raster_bwd_fast_det(const RasterParams& P, int n_tiles, cudaStream_t s);
void launch_pixels_bwd(const RasterParams& P, cudaStream_t s);  // k_raster_pixels_warp<MODE, true> over P.redo_list
void launch_exact_bwd(const RasterParams& P, int n_tiles, cudaStream_t s);
void launch_eval_sorting(const RasterParams& P, int tile0, int tile1, const long long* scr_off, double* scratch,
                         int use_cache, double* tau, double* mae, unsigned char* flag, cudaStream_t s);
void launch_eval_sorting_reduce(const CamD& cam, const long long* tileoff, const double* tau, const double* mae,
                                const unsigned char* flag, double* out, cudaStream_t s);

}  // namespace drk

struct drk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // drk_forward_host pipeline: parameter chunks copied on h2d_stream, h2d_ev[q] = chunk q landed
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t h2d_ev[9] = {};
  bool own_stream = false;
  std::string err;

  // activated primitives owned by the context (raw path)
  drk::DevBuf a_mu, a_rot, a_s, a_th, a_eta, a_tau, a_o, a_sh, a_ex, a_ey, a_det;
  drk::DevBuf a_thf, a_invdetf, a_piogf, a_hf, a_psif, a_rec, pxflag, pxstop, redo, redo_cnt, vstat;
  drk::Activated act{};

  // per view
  drk::DevBuf geo, frame32, bbox, hullref, hull, ptspool, ptsref, rowcnt, rowoff, rows, rowpaircnt, rowpairoff;
  drk::DevBuf pk, pv, sk, hist, sortoff, tileoff, cdirs, tdirs, bits;
  drk::DevBuf pidx;      // second sorted-id list (tie ordering output; swapped with pv)
  drk::DevBuf tie_long;  // starts of tied runs longer than kRankMax (count first)
  int key_dbits = 19;  // depth bits of the packed 32-bit sort keys (32 - tile bits)
  drk::DevBuf pxstate, replay_cnt, replay_rec, replay_ids;
  drk::DevBuf gact, touched;
  drk::DevBuf counters, scan_tmp, loss_tmp;
  drk::DevBuf scene_aos;                  // record-major staging of scene files (drk_scene_load / drk_scene_save)
  drk::DevBuf loss_part, ssim_f;          // drk_loss / drk_ssim / drk_psnr: partial sums, SSIM adjoint fields
  drk::DevBuf dens_code, dens_pos;        // drk_densify_and_prune / drk_mesh_convert: per-item code / count, scanned positions
  drk::DevBuf eval_scr, eval_px, eval_off;  // drk_eval_sorting: sequence scratch, per-pixel metrics, chunk offsets
  drk::DevBuf ovf_scr, ovf_list;
  drk::DevBuf tord;                       // fast forward tile order: keys / ids and their sort ping-pong
  drk::DevBuf host_raw, host_img;         // drk_forward_host: device staging of the host params / framebuffers
  drk::DevBuf pxcomp;                     // composited entries per pixel (forward)
  // deterministic backward: slot counts / record offsets, record rows, ids, tiles,
  // sort buffers, per-primitive offsets, fp64 accumulator
  drk::DevBuf det_cnt, det_base, det_rec, det_id, det_tile, det_sort, det_poff, det_acc, det_rowoff;
  drk::DevBuf det_tflag, det_tpos, det_tstart, det_tprim;  // tile segments of the sorted records
  long long det_chunk_limit = 0;          // test hook: records per chunk (0 = memory-based)
  drk::DevBuf comm_buf;                   // drk_allreduce_adam: padded gradient / parameter exchange buffers
  drk::DevBuf scan_tmp2, replay_cid, replay_cval;  // drk_get_replay: per-pixel offsets, compacted records
  int64_t hull_cap = 0;
  drk::DevBuf rowest;
  std::vector<int> bands;         // tile-row band boundaries of the last forward
  // banded frames: each band's sorted tile lists (ids + tile offsets) kept from
  // the forward so the backward need not re-bin (when device memory allows)
  std::vector<drk::DevBuf> band_ids, band_off;
  bool band_cache_valid = false;
  long long band_pair_limit = 0;  // test hook: force bands above this many pairs (0 = memory-based)
  size_t device_bytes = 0;        // cudaMemGetInfo total, queried once
  int64_t pts_cap = 0;
  drk::DevBuf planes64;  // drk_get_framebuffers_f64 staging
  drk::DevBuf tile_cost;       // per tile: entries the fast forward streamed (the backward's dispatch order)
  bool tile_cost_valid = false;
  // K1 vertex cache: built on the second forward of one activation, used from the third
  drk::DevBuf vc_pool, vc_ref, vc_cursor;
  uint64_t act_gen = 0;       // bumped by every new activation
  int act_renders = 0;        // forwards of the current activation
  uint64_t vc_gen = ~0ull;    // activation the cache holds
  double vc_alpha_min = -1;   // ... and the alpha_min its support radii used
  long long redo_half = 0;  // offset of the redo list's ordering scratch (pixels of the last forward + 1)

  // stage timing
  bool timing = false;
  bool validate_fast = false;  // fast kernel: check every fp32 alpha against fp64 (drk_validate_fast)
  cudaEvent_t ev[10] = {};
  long long launch_base = 0;

  // last forward
  bool has_fwd = false;
  bool has_act = false;  // activated primitives + shape constants of the last drk_forward / drk_forward_prims / drk_activate
  bool work_counters = false;  // fast forward work counters (streamed / popped / rejects); off by default
  drk_camera cam{};
  drk_options opt{};
  drk::CamD camd{};
  drk::OptD optd{};
  int64_t n_pairs = 0;
  int64_t n_rows = 0;
  drk_stats stats{};
};

namespace drk {

// Launchers (drk_kernels.cu).  All return a drk_status.
int launch_activate(drk_ctx* c, const float* raw, int n, int K, int terms);
int launch_shape(drk_ctx* c, const drk_prims* p, int n, int K, int terms);
// Host-buffer pipeline (drk_forward_host): the raw parameters arrive in nchunk
// primitive ranges [bounds[q], bounds[q+1]), chunk q complete when ready[q] fires.
struct H2DPipe {
  const float* raw = nullptr;  // device copy of the [S][n] parameters
  int nchunk = 0;
  int bounds[9] = {};
  cudaEvent_t ready[8] = {};
};
int run_forward(drk_ctx* c, const drk_camera* cam, const drk_options* opt, float* color, float* depth,
                float* normal, float* alpha,
                const H2DPipe* pipe = nullptr);
int run_backward(drk_ctx* c, const float* raw, const drk_frame_grad* fg, float* grad_raw,
                 float* d_center_world, float* screen_grad, uint8_t* touched, int accumulate,
                 int deterministic);
int run_l1_loss(drk_ctx* c, const float* r, const float* t, int w, int h, double* loss, float* dcol);
int run_adam(drk_ctx* c, float* params, const float* grads, float* m, float* v, int n, int K, int terms,
             int64_t step, const drk_adam_config* cfg);
// Adam on scalars [e0, e1) of the SoA parameters; gradient of scalar e at grads[e - g0]
int run_adam_range(drk_ctx* c, float* params, const float* grads, long long g0, float* m, float* v, int n, int K,
                   long long e0, long long e1, int64_t step, const drk_adam_config* cfg);
int set_error(drk_ctx* c, int status, const std::string& msg);
int cuda_check(drk_ctx* c, cudaError_t e, const char* where);

}  // namespace drk
