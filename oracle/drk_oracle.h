/* CPU restatement of the reference DRK rasterizer hot path — TEST
 * INFRASTRUCTURE ONLY (the checker for the CUDA path; never shipped).
 *
 * Plain C11, double precision, op order copied from the reference sources
 * (cited per function in drk_oracle.c) and from the Eigen shim's documented
 * left-to-right reductions.  Pinned against the unmodified reference build
 * (oracle/_ref/libdrk_refcapi.so) by tests/test_oracle.py.
 *
 * Layouts are the product ABI's (include/drk_b200.h): raw parameters are
 * scalar-major SoA raw[s*n + i] in drk::for_each_scalar order; images are
 * row-major interleaved.
 */
#ifndef DRK_ORACLE_H
#define DRK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9]; /* world->camera, row-major */
  double t[3];
} orc_camera;

typedef struct orc_options {
  double lowpass_radius, alpha_min, grazing_eps;
  double background[3];
  double early_stop_transmittance;
  int32_t sh_degree, use_cache, exact_sort, presort, threads, pad_;
} orc_options;

/* Work counters of one render (per-frame totals), used for the roofline's
 * algorithmic flop count. */
typedef struct orc_stats {
  int64_t pairs;           /* tile-list entries */
  int64_t hits;            /* valid ray-plane hits over all (pixel, candidate) */
  int64_t streamed;        /* candidates streamed until saturation */
  int64_t popped;          /* cache pops (alpha evaluations) */
  int64_t composited;      /* blended entries */
  int64_t poly_vertices;   /* support-polygon vertices before clipping */
  int64_t max_poly;        /* largest support polygon */
} orc_stats;

/* Status codes mirror drk_status in include/drk_b200.h. */
int orc_activate(const double* raw, int n, int k, int terms, double* mu, double* rot,
                 double* scales, double* angles, double* eta, double* tau, double* opacity);
int orc_bin(const double* raw, int n, int k, int terms, const orc_camera* cam,
            const orc_options* opt, int64_t* total_pairs);
void orc_bins_copy(int64_t* offsets, int32_t* ids, double* keys);
int orc_render(const double* raw, int n, int k, int terms, const orc_camera* cam,
               const orc_options* opt, double* color, double* depth, double* normal,
               double* alpha, int want_replay, int64_t* replay_records, orc_stats* stats);
void orc_replay_copy(int64_t* offsets, int32_t* ids, double* vals);
int orc_backward(const double* raw, int n, int k, int terms, const orc_camera* cam,
                 const orc_options* opt, const double* d_color, const double* d_depth,
                 const double* d_normal, const double* d_alpha, double* grad_raw,
                 double* d_center_world, double* screen_grad, int8_t* touched);
int orc_loss_l1(const double* rendered, const double* target, int w, int h, double* value,
                double* d_color);
int orc_adam_step(double* params, const double* grads, double* m, double* v, int n, int k,
                  int terms, int64_t* step, const double* lrs, int steps_total, double extent,
                  int freeze_eta_tau, int freeze_angles);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
