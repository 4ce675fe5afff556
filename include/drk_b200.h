/* drk_b200.h — C-ABI of the B200-native DRK splatting rasterizer.
 *
 * This is the drop-in boundary for the reference's render / backward_render
 * path.  The reference exposes a C++ API only; each entry
 * point below cites the reference interface it replaces.  No C++ types, no
 * exceptions: every call returns a drk_status whose non-zero values map 1:1
 * onto the reference's drk::Error subclasses (reference include/drk/errors.hpp)
 * plus CUDA / allocation / argument failures.
 *
 * Data layout at the boundary
 *   raw parameters  float32, scalar-major SoA: raw[s * n + i] is scalar s of
 *                   primitive i, s in drk::for_each_scalar order
 *                   (reference types.hpp:48-72): center(3), quat(4, w first),
 *                   scale_raw(K), angle_raw(K), eta_raw, tau_raw, opacity_raw,
 *                   sh_raw(terms x 3, coefficient-major then RGB).
 *                   S = drk_scalar_count(K, terms) = 3 + 4 + 2K + 3 + 3*terms.
 *   activated       drk_prims (below): fp64 centre/rotation/shape, f32 SH.
 *   images          float32, row-major, interleaved channels, H x W x C
 *                   (same shapes as drk::FrameBuffers, reference raster.hpp:57-63).
 *   gradients       same layout as the raw parameters (drk::ParamGrads::raw,
 *                   reference grad.hpp:48-53).
 * Device pointers unless a function name ends in _host.  Calls are ordered on
 * the given CUDA stream (NULL = the context's stream).
 */
#ifndef DRK_B200_H
#define DRK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DRK_ABI_VERSION 2

typedef enum drk_status {
  DRK_OK = 0,
  DRK_ERR_GENERIC = 1,            /* drk::Error */
  DRK_ERR_NONFINITE = 2,          /* drk::NonFiniteError (core.cpp:134) */
  DRK_ERR_DEGENERATE_QUAT = 3,    /* drk::DegenerateQuaternionError (geometry.cpp:23) */
  DRK_ERR_DEGENERATE_BASIS = 4,   /* drk::DegenerateBasisError (core.cpp:191) */
  DRK_ERR_REPLAY_MISMATCH = 5,    /* drk::ReplayMismatchError (grad.cpp:311-314) */
  DRK_ERR_DIMENSION = 6,          /* drk::DimensionMismatchError */
  DRK_ERR_INVALID_ARG = 7,
  DRK_ERR_CUDA = 8,
  DRK_ERR_OOM = 9,
  DRK_ERR_UNSUPPORTED = 10,
  DRK_ERR_IO = 11,                /* drk::IoError (io.cpp:51,60) */
  DRK_ERR_CORRUPT_FILE = 12,      /* drk::CorruptFileError (io.cpp:63,68,72,80) */
  DRK_ERR_VERSION = 13,           /* drk::VersionMismatchError (io.cpp:70,74) */
  DRK_ERR_DEGENERATE_FACE = 14,   /* drk::DegenerateFaceError (mesh.cpp:222-258) */
  DRK_ERR_TOO_MANY_VERTICES = 15, /* drk::TooManyVerticesError (mesh.cpp:223-225) */
  DRK_ERR_PARSE = 16,             /* drk::ParseError (mesh.cpp:153-185) */
  DRK_ERR_EMPTY_MESH = 17,        /* drk::EmptyMeshError (mesh.cpp:197) */
  DRK_ERR_COMM = 18               /* NCCL failure (ncclCommGetAsyncError / call status); the communicator is aborted */
} drk_status;

/* drk::Camera (reference geometry.hpp:9-19). */
typedef struct drk_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9]; /* world->camera rotation, row-major */
  double t[3]; /* world->camera translation */
} drk_camera;

/* drk::RenderOptions + drk::KernelConfig (reference raster.hpp:81-90,
 * types.hpp:100-105).  presort: 0 None, 1 CenterDepth, 2 NearestDepth.
 * `threads` is accepted for API parity and ignored (the GPU path is
 * deterministic by construction).  record_replay > 0 keeps up to that many
 * blend records per pixel for drk_get_replay (the ReplayBuffer* argument of
 * drk::render; small images only). */
typedef struct drk_options {
  double lowpass_radius;            /* s_l, pixels (default 0.5) */
  double alpha_min;                 /* default 1/255 */
  double grazing_eps;               /* default 1e-6 */
  double background[3];             /* default (1,1,1) */
  double early_stop_transmittance;  /* default 1e-4 */
  int32_t sh_degree;                /* default 3 */
  int32_t use_cache;                /* default 1 */
  int32_t exact_sort;               /* default 0 */
  int32_t presort;                  /* default 2 */
  int32_t threads;                  /* ignored */
  int32_t record_replay;            /* default 0 */
  int32_t fp64_alpha;               /* default 0; 1 = every alpha in fp64 (reference-precision mode:
                                       identical arithmetic across cache / list / exact-sort modes) */
  int32_t raster_kernel;            /* 0 = auto (fp32 interval forward and backward where eligible),
                                       1 = legacy fp64-depth forward and backward, 5 = legacy backward only,
                                       6 / 7 = auto with the fast forward forced to half-tile / tile CTAs */
} drk_options;

/* Activated primitives (drk::DrkPrimitive, reference types.hpp:77-98), all
 * device pointers, primitive-major.  rot is row-major per primitive; its
 * columns are the local axes R_x, R_y, R_z.  sh may be NULL (then terms=0). */
typedef struct drk_prims {
  const double* mu;       /* n x 3 */
  const double* rot;      /* n x 9 */
  const double* scales;  /* n x K */
  const double* angles;  /* n x K, strictly increasing, angles[K-1] == 2 pi */
  const double* eta;     /* n */
  const double* tau;     /* n */
  const double* opacity; /* n */
  const float* sh;       /* n x terms x 3 */
  const double* sh64;    /* optional (may be NULL): the same coefficients in fp64.  When given, the
                          * fp64 pixel path (reference precision, fp64 re-render) evaluates colours from
                          * them bit-exactly like the reference (geometry.cpp:101-138) */
} drk_prims;

/* Frame gradients (drk::FrameGrad, reference grad.hpp:40-45); NULL = empty. */
typedef struct drk_frame_grad {
  const float* d_color;  /* H x W x 3 */
  const float* d_depth;  /* H x W */
  const float* d_normal; /* H x W x 3 */
  const float* d_alpha;  /* H x W */
} drk_frame_grad;

/* Work counters of the last forward (algorithmic-work accounting). */
typedef struct drk_stats {
  int64_t primitives;      /* primitives binned (visible at alpha_min) */
  int64_t pairs;           /* tile-list entries */
  int64_t streamed;        /* (pixel, candidate) intersections until saturation */
  int64_t popped;          /* cache pops (alpha evaluations, incl. cheap rejects) */
  int64_t composited;      /* blended entries */
  int64_t near_ties;       /* binning decisions within 1e-9 relative of a tie */
  int64_t poly_overflow;   /* primitives that needed the large-polygon path */
  int64_t replay_overflow; /* pixels whose replay exceeded record_replay */
  int64_t fp64_pixels;     /* pixels re-rendered in fp64 (termination within the fp32 error bound) */
  int64_t launches;        /* kernels launched by the last forward + backward */
  /* CUDA-event stage times of the last forward / backward, ms (when
   * drk_set_timing(ctx, 1)): activate, preprocess, rows+emit, sort, raster,
   * raster_fp64, backward_raster, activation_backward */
  double stage_ms[8];
  int64_t bwd_warp_steps;    /* warp-cooperative backward steps with >= 1 composited record */
  int64_t bwd_lead_records;  /* primitive groups reduced in the warp-cooperative backward */
  int64_t reject_radius;     /* pops rejected by the isotropic alpha_min support radius */
  int64_t reject_bracket;    /* pops rejected by the in-bracket lower bound of the exponent */
  int64_t fp64_evals;        /* pops re-evaluated in fp64 (decision inside the fp32 error bound) */
  int64_t ambiguous;         /* cache steps whose fp32 depth intervals overlapped (resolved in fp64) */
  int64_t ring_miss;         /* pops of entries older than the shared-memory ring (re-staged from HBM) */
  int64_t tie_runs;          /* sort: runs of equal packed 32-bit keys (ordered on the fp64 key afterwards) */
  int64_t tie_members;       /* sort: entries in those runs */
  int64_t tie_max_run;       /* sort: longest run */
  int64_t cache_appends;     /* fast forward: full-cache steps whose incoming entry is certainly deeper than
                              * every cached one (work counters on) */
} drk_stats;

typedef struct drk_ctx drk_ctx;

/* --- context ------------------------------------------------------------ */
int drk_ctx_create(int device, drk_ctx** out);
void drk_ctx_destroy(drk_ctx* ctx);
const char* drk_status_string(int status);
const char* drk_last_error(const drk_ctx* ctx);
int drk_abi_version(void);
int drk_scalar_count(int k, int sh_terms);
void drk_default_options(drk_options* opt);
int drk_get_stats(const drk_ctx* ctx, drk_stats* out);
int drk_set_stream(drk_ctx* ctx, void* cuda_stream);
/* Enables per-stage CUDA-event timing (drk_stats.stage_ms). */
int drk_set_timing(drk_ctx* ctx, int enabled);
/* Banded binning (frames whose tile-pair lists exceed device memory are binned,
 * sorted and rasterized one band of tile rows at a time; automatic).  Test hook:
 * force bands above `pairs` pairs per band (0 = memory-based). */
int drk_set_band_limit(drk_ctx* ctx, int64_t pairs);
/* Deterministic backward: records per chunk of tile rows (test hook; 0 = memory-based). */
int drk_set_det_chunk_limit(drk_ctx* ctx, int64_t records);
/* Work counters of the fast forward (drk_stats streamed / popped / reject
 * counts): off by default (the counter-free kernel is launched, those fields
 * stay 0); on launches the counting instantiation (about 1.6% slower). */
int drk_set_counters(drk_ctx* ctx, int enabled);
int drk_get_bands(const drk_ctx* ctx, int32_t* n_bands);
/* Validation of the fast forward kernel: while enabled, every fp32 alpha is
 * also evaluated in fp64; drk_get_validation returns max |a32 - a64| / bound
 * (must stay below 1) and max |a32 - a64| since validation was enabled. */
int drk_set_validation(drk_ctx* ctx, int enabled);
int drk_get_validation(drk_ctx* ctx, double* out2);
/* First pop whose error exceeded its bound (flag, then 21 diagnostic values). */
int drk_get_validation_detail(drk_ctx* ctx, double* out22);
/* Measured FP32 FFMA throughput of this device (TFLOP/s), for rooflines. */
int drk_measure_fp32_peak(drk_ctx* ctx, double* tflops);

/* --- activation (reference core.cpp:133-146 activate) -------------------- */
/* raw (f32 SoA) -> activated fp64 arrays owned by the context; the pointers
 * stay valid until the next call that activates.  Throws the reference's
 * NonFinite / DegenerateQuaternion errors as status codes. */
int drk_activate(drk_ctx* ctx, const float* raw, int n, int k, int sh_terms, drk_prims* out);

/* --- forward (reference raster.hpp:92-93 render; raster.hpp:30-31
 * bin_primitives) ---------------------------------------------------------- */
/* From raw parameters (activation on device).  Outputs may be NULL. */
int drk_forward(drk_ctx* ctx, const float* raw, int n, int k, int sh_terms,
                const drk_camera* cam, const drk_options* opt, float* color, float* depth,
                float* normal, float* alpha);
/* Renders the primitives of the last drk_forward / drk_forward_prims /
 * drk_activate on this context (activation and shape constants kept) from another camera / options:
 * a multi-view batch activates once.  The caller's parameters must not have
 * changed since (call drk_forward again after an update). */
int drk_forward_again(drk_ctx* ctx, const drk_camera* cam, const drk_options* opt, float* color, float* depth,
                      float* normal, float* alpha);
/* From activated primitives (the reference's std::vector<DrkPrimitive> input). */
int drk_forward_prims(drk_ctx* ctx, const drk_prims* prims, int n, int k, int sh_terms,
                      const drk_camera* cam, const drk_options* opt, float* color,
                      float* depth, float* normal, float* alpha);
/* Host-buffer variant of drk_forward: copies raw in and renders; page-locked
 * outputs (mapped under unified addressing) are written in place by the
 * kernels as tiles finish (zero-copy), other outputs are copied out after the
 * forward.  Any output may be NULL; synchronous. */
int drk_forward_host(drk_ctx* ctx, const float* raw_host, int n, int k, int sh_terms,
                     const drk_camera* cam, const drk_options* opt, float* color_host,
                     float* depth_host, float* normal_host, float* alpha_host);

/* Tile lists of the last forward (drk::TileBinning): per-tile offsets
 * (tiles_x*tiles_y + 1), primitive ids and f64 presort keys, in the
 * reference's per-tile (key, prim_id) order.  Host pointers; pass NULL to
 * query sizes only. */
int drk_get_tile_lists(drk_ctx* ctx, int64_t* total_pairs, int64_t* offsets_host,
                       int32_t* ids_host, double* keys_host);
/* fp64 framebuffers of the last forward (the rasterizer's per-pixel fp64
 * accumulators; colour includes the background term), host pointers, any may
 * be NULL.  drk::FrameBuffers holds doubles; the drop-in adapter returns
 * these. */
int drk_get_framebuffers_f64(drk_ctx* ctx, double* color_host, double* depth_host, double* normal_host,
                             double* alpha_host);
/* Replay of the last forward with record_replay > 0 (drk::ReplayBuffer):
 * per-pixel offsets (H*W + 1), prim ids and 5 doubles per record
 * (u, v, depth, alpha, lowpass_active).  Host pointers; NULL to query. */
int drk_get_replay(drk_ctx* ctx, int64_t* total_records, int64_t* offsets_host,
                   int32_t* ids_host, double* vals_host);

/* --- backward (reference grad.hpp:58-61 backward_render) ----------------- */
/* Uses the state of the last drk_forward / drk_forward_prims call on this
 * context (its binning and per-pixel accumulators stand in for the
 * ReplayBuffer).  Camera dimensions / n must match it, else
 * DRK_ERR_REPLAY_MISMATCH.  grad_raw (SoA, like raw) receives the raw-space
 * gradient; with accumulate != 0 it is added to instead of overwritten
 * (multi-view batches).  d_center_world (n x 3), screen_grad (n), touched (n)
 * may be NULL.  deterministic != 0 selects the fixed-order reduction: every
 * composited record writes its gradient row to its own slot and the rows are
 * reduced per primitive in (tile, pixel, composite) order, tile partials in fp64
 * (reference grad.cpp:327-368) — parallel, and bitwise reproducible. */
int drk_backward(drk_ctx* ctx, const float* raw, const drk_frame_grad* fg, float* grad_raw,
                 float* d_center_world, float* screen_grad, uint8_t* touched, int accumulate,
                 int deterministic);
/* Activated-space gradients (drk::PrimGrads, reference grad.hpp:19-29) of the
 * last backward, fp32, n rows of *stride floats in a K-independent layout:
 * d_center [0,3), d_rot [3,12) (row-major), d_scales [12,28), d_angles
 * [28,44) (first K used), d_eta 44, d_tau 45, d_opacity 46, d_sh from 47
 * (RGB per term); rows padded to a multiple of 4.  Device pointer owned by
 * the context. */
int drk_get_prim_grads(drk_ctx* ctx, const float** grads, int* stride);

/* --- loss and optimizer (reference optimize.cpp:171-204, :226-307) -------- */
/* L1 branch of drk::loss (dssim_weight = 0): loss_out (device, 1 double)
 * receives mean |r - t|, d_color = sign(r - t) / (3 W H). */
int drk_l1_loss(drk_ctx* ctx, const float* rendered, const float* target, int width, int height,
                double* loss_out, float* d_color);

/* drk::loss (optimize.cpp:171-204), channels-interleaved f32 images
 * (H x W x channels, device): value = (1-w) mean|r-t| + w (1 - mean SSIM),
 * w = dssim_weight when > 0 and both sides >= 11 (else 0).  out3 (device,
 * 3 doubles) = {value, L1, mean SSIM}; d_color (device, may be NULL) = dvalue/dr.
 * SSIM: 11-tap Gaussian (sigma 1.5), valid region, C1 = 1e-4, C2 = 9e-4. */
int drk_loss(drk_ctx* ctx, const float* rendered, const float* target, int width, int height, int channels,
             double dssim_weight, double* out3, float* d_color);
/* drk::ssim (optimize.cpp:157-166): out1 (device) = mean over channels of the
 * valid-region SSIM; DRK_ERR_DIMENSION if a side is < 11. */
int drk_ssim(drk_ctx* ctx, const float* a, const float* b, int width, int height, int channels, double* out1);
/* drk::psnr (optimize.cpp:145-155): out2 (device) = {psnr (100 if mse < 1e-10), mse}. */
int drk_psnr(drk_ctx* ctx, const float* a, const float* b, int width, int height, int channels, double* out2);
/* The same three on double images (drk::Image, the drop-in adapter's types). */
int drk_loss_f64(drk_ctx* ctx, const double* rendered, const double* target, int width, int height, int channels,
                 double dssim_weight, double* out3, double* d_color);
int drk_ssim_f64(drk_ctx* ctx, const double* a, const double* b, int width, int height, int channels, double* out1);
int drk_psnr_f64(drk_ctx* ctx, const double* a, const double* b, int width, int height, int channels, double* out2);
/* psnr(quantize_8bit(a), b) (image.cpp:7-14; train's evaluation, optimize.cpp:432,460). */
int drk_psnr_quantized(drk_ctx* ctx, const float* a, const float* b, int width, int height, int channels,
                       double* out2);

/* drk::TrainConfig learning-rate fields used by adam_step. */
typedef struct drk_adam_config {
  double lr_drk, lr_position, lr_rotation, lr_opacity, lr_sh;
  int32_t steps;             /* schedule length (TrainConfig::steps) */
  int32_t freeze_eta_tau, freeze_angles;
  int32_t pad_;
  double scene_extent;
  double grad_scale;         /* gradients are multiplied by this first (1/views) */
} drk_adam_config;
/* drk::adam_step on SoA f32 params / grads / moments.  *step is
 * OptState::step (host value, incremented). */
int drk_adam_step(drk_ctx* ctx, float* params, const float* grads, float* m, float* v, int n,
                  int k, int sh_terms, int64_t* step, const drk_adam_config* cfg);

/* --- multi-GPU gradient exchange (BASELINE.json config 4) --
 * The reference has no distributed path: the multi-view gradient is the mean
 * over views of per-view backward_render.  One process per
 * GPU; NCCL is loaded at drk_comm_init (dlopen of libnccl.so.2: the copy a
 * host framework already loaded, else the system's), so the library has no
 * link-time NCCL dependency.  Calls are ordered on the context's stream; NCCL
 * failures are detected with ncclCommGetAsyncError while waiting and abort
 * the communicator (DRK_ERR_COMM). */
typedef struct drk_comm drk_comm;
/* 128-byte NCCL unique id, created by rank 0 and shared by the caller. */
int drk_comm_unique_id(uint8_t id_out[128]);
int drk_comm_init(drk_ctx* ctx, const uint8_t id[128], int nranks, int rank, drk_comm** out);
void drk_comm_destroy(drk_comm* comm);
/* In-place sum over the ranks of `count` floats (device). */
int drk_allreduce_sum(drk_ctx* ctx, drk_comm* comm, float* buf, int64_t count);
/* One training-step exchange + update: the raw-gradient buffers (SoA f32,
 * like drk_adam_step) are reduce-scattered (sum) across the ranks, each rank
 * applies drk::adam_step (reference optimize.cpp:259-307, gradients scaled by
 * cfg->grad_scale, normally 1 / total views) to its contiguous shard of the
 * scalars, and the updated parameters are all-gathered: every rank ends with
 * the same parameters, 1/N of the Adam work each.  m and v are full-size but
 * a rank only ever reads and writes its own shard of them. */
int drk_allreduce_adam(drk_ctx* ctx, drk_comm* comm, float* params, float* grads, float* m, float* v, int n, int k,
                       int sh_terms, int64_t* step, const drk_adam_config* cfg);

/* drk::eval_sorting (raster.cpp:487-560) of the last forward on this context
 * (its camera, presort and use_cache): out4 (host) = {accuracy, kendall_tau,
 * mae, pixels}.  Per-pixel values are the reference's exactly and are summed
 * in its order.  DRK_ERR_UNSUPPORTED for banded frames. */
int drk_eval_sorting(drk_ctx* ctx, double* out4);

/* --- density control (reference optimize.cpp:309-383) ----------------------- */
/* TrainConfig fields used by densify_and_prune (optimize.hpp:30-61). */
typedef struct drk_densify_config {
  double densify_grad_threshold;  /* default 5e-4 */
  double prune_opacity_threshold; /* default 5e-2 */
  double percent_dense;           /* default 0.01 */
} drk_densify_config;
/* DensifyStats::accumulate (optimize.cpp:309-318): for touched primitives,
 * accum[i] += screen_grad[i], count[i] += 1 (device buffers; screen_grad and
 * touched as written by drk_backward). */
int drk_densify_accumulate(drk_ctx* ctx, const float* screen_grad, const uint8_t* touched, int n, double* accum,
                           int32_t* count);
/* densify_and_prune (optimize.cpp:320-373) on raw parameters and Adam moments
 * f32 [S][n] (device): prune sigmoid(opacity_raw) < prune threshold; primitives
 * whose mean screen gradient exceeds the threshold are cloned (largest scale
 * <= percent_dense * extent; the copy gets zero moments) or split in two
 * (scales / 2, centres +- 0.25 s_max along the longest basis, zero moments).
 * Output f32 [S][cap] in source order; *n_out = new count (raw_out may be NULL
 * to query it). */
int drk_densify_and_prune(drk_ctx* ctx, const float* raw, const float* m, const float* v, int n, int k, int sh_terms,
                          const double* accum, const int32_t* count, const drk_densify_config* cfg, double extent,
                          float* raw_out, float* m_out, float* v_out, int64_t cap, int64_t* n_out);
/* scene_extent (optimize.cpp:375-383): out (device) = max(1e-6, |hi - lo| / 2)
 * of the raw centres. */
int drk_scene_extent(drk_ctx* ctx, const float* raw, int n, double* out);

/* --- scene files (DRKSCENE v1, reference io.hpp:20-25, io.cpp:40-97) ------ */
typedef struct drk_scene_header {
  int32_t version;      /* 1 */
  int32_t basis_count;  /* K */
  int32_t sh_degree;    /* 0..3 */
  int32_t scalar_count; /* scalar_count(K, (sh_degree+1)^2): floats per primitive */
  int64_t count;        /* primitives */
} drk_scene_header;
/* Header checks of drk::load_scene (io.cpp:58-80): DRK_ERR_IO (cannot open),
 * DRK_ERR_CORRUPT_FILE (missing / malformed / implausible header, payload size
 * not count records), DRK_ERR_VERSION (version != 1, K != expected_basis_count
 * when that is > 0).  No device work. */
int drk_scene_read_header(const char* path, int expected_basis_count, drk_scene_header* out);
/* drk::load_scene (io.cpp:58-97) straight to the device: raw_dev (device,
 * capacity primitives) receives the scene in the C-ABI raw layout, f32
 * [scalar_count][count] (record-major file -> scalar-major device, bit-exact). */
int drk_scene_load(drk_ctx* ctx, const char* path, int expected_basis_count, float* raw_dev, int64_t capacity,
                   drk_scene_header* out);
/* drk::save_scene (io.cpp:40-56) from device raw parameters f32 [S][n]. */
int drk_scene_save(drk_ctx* ctx, const char* path, const float* raw_dev, int n, int k, int sh_degree);

/* --- Mesh2DRK (reference mesh.hpp, mesh.cpp) ------------------------------- */
typedef struct drk_mesh drk_mesh;
/* load_mesh (mesh.cpp:134-217): OBJ subset (v, f, usemtl / mtllib diffuse
 * colour); non-planar or concave polygons fan-triangulated.  Host only.  *out
 * is always set (free it with drk_mesh_free; drk_mesh_error has the message);
 * DRK_ERR_IO / DRK_ERR_PARSE / DRK_ERR_EMPTY_MESH like the reference. */
int drk_mesh_load(const char* path, drk_mesh** out);
int drk_mesh_info(const drk_mesh* mesh, int64_t* n_vertices, int64_t* n_faces, int64_t* n_indices,
                  int32_t* n_warnings);
const char* drk_mesh_error(const drk_mesh* mesh);
/* Host arrays: vertices [nv][3], face_offsets [nf+1] (CSR), indices, colors [nf][3]. */
int drk_mesh_arrays(const drk_mesh* mesh, double* vertices, int32_t* face_offsets, int32_t* indices, double* colors);
void drk_mesh_free(drk_mesh* mesh);
/* convert (mesh.cpp:326-343) on the device: one DRK per face (face_to_drk_raw,
 * mesh.cpp:219-319), degenerate faces skipped in order (*n_skipped), a face
 * with more than k vertices -> DRK_ERR_TOO_MANY_VERTICES.  Inputs are device
 * arrays as drk_mesh_arrays lays them out; raw_out (device, may be NULL to
 * query *n_out) = f32 [scalar_count(k, 1)][cap], SH degree 0. */
int drk_mesh_convert(drk_ctx* ctx, const double* vertices, int64_t n_vertices, const int32_t* face_offsets,
                     const int32_t* indices, const double* colors, int n_faces, int k, float* raw_out, int64_t cap,
                     int64_t* n_out, int64_t* n_skipped);
/* shade_lambert (mesh.cpp:345-357) in place on device raw f32 [S][n]. */
int drk_shade_lambert(drk_ctx* ctx, float* raw, int n, int k, const double* light_dir, double ambient);

/* --- validation hook ----------------------------------------------------- */
/* Samples the fp32 alpha fast path against the fp64 path on the activated
 * primitives of this context: max |a32 - a64| / (bound * a32) and
 * max |a32 - a64|.  Used by the parity tests to check the error bound that
 * gates the fp64 fallback. */
int drk_debug_alpha_bound(drk_ctx* ctx, int64_t samples, uint64_t seed, double* max_ratio, double* max_abs);

#ifdef __cplusplus
}
#endif
#endif /* DRK_B200_H */
