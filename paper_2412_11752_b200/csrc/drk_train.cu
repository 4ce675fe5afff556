// Density control and helpers of the training loop on the device (reference
// optimize.cpp:309-383): DensifyStats::accumulate, densify_and_prune (prune
// by opacity, clone small / split large primitives above the mean screen-space
// gradient threshold, optimizer rows following the primitive set) and
// scene_extent.  Parameters and Adam moments stay in the C-ABI raw layout,
// f32 [S][n] scalar-major, so the new set is a stable stream compaction:
// per-primitive output counts (0 prune, 1 keep, 2 clone or split) -> exclusive
// scan -> one thread per source primitive writes its rows at the scanned
// position, in source order like the reference's push_backs.  The split
// offset (optimize.cpp:356-366) is formed in fp64 from the activated angle and
// rotation (same expressions as k_activate) and rounded once to f32.
// Compiled with --fmad=false (the reference's x86-64 build does not contract).
#include "drk_internal.h"

namespace drk {

int set_error(drk_ctx* c, int status, const std::string& msg);
int cuda_check(drk_ctx* c, cudaError_t e, const char* where);
template <typename T>
int exclusive_scan(drk_ctx* c, const T* in, long long n, long long* out, long long* total);

namespace {

enum : int { kPrune = 0, kKeep = 1, kClone = 2, kSplit = 3 };

__device__ __forceinline__ double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }  // core.cpp:80

// DensifyStats::accumulate (optimize.cpp:309-318)
__global__ void k_densify_accumulate(int n, const float* __restrict__ sg, const unsigned char* __restrict__ touched,
                                     double* accum, int* count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !touched[i]) return;
  accum[i] += (double)sg[i];
  count[i] += 1;
}

// per-primitive decision of densify_and_prune (optimize.cpp:338-352)
__global__ void k_densify_decide(int n, int K, const float* __restrict__ raw, const double* __restrict__ accum,
                                 const int* __restrict__ count, double grad_thr, double prune_thr, double dense_size,
                                 int* code, int* outcnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double opacity = sigm((double)raw[(size_t)(9 + 2 * K) * n + i]);
  int c;
  if (opacity < prune_thr) {
    c = kPrune;
  } else {
    const double mean_grad = count[i] > 0 ? accum[i] / count[i] : 0.0;
    if (mean_grad <= grad_thr) {
      c = kKeep;
    } else {
      double smax = exp((double)raw[(size_t)7 * n + i]);  // largest activated scale (optimize.cpp:344-348)
      for (int k = 1; k < K; ++k) {
        const double s = exp((double)raw[(size_t)(7 + k) * n + i]);
        if (s > smax) smax = s;
      }
      c = smax <= dense_size ? kClone : kSplit;
    }
  }
  code[i] = c;
  outcnt[i] = c == kPrune ? 0 : (c == kKeep ? 1 : 2);
}

__global__ void k_densify_emit(int n, int K, int S, const float* __restrict__ raw, const float* __restrict__ m,
                               const float* __restrict__ v, const int* __restrict__ code,
                               const long long* __restrict__ pos, long long cap, float* raw_out, float* m_out,
                               float* v_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = code[i];
  if (c == kPrune) return;
  const long long p = pos[i];
  if (c == kKeep || c == kClone) {
    for (int s = 0; s < S; ++s) {
      raw_out[(size_t)s * cap + p] = raw[(size_t)s * n + i];
      m_out[(size_t)s * cap + p] = m[(size_t)s * n + i];
      v_out[(size_t)s * cap + p] = v[(size_t)s * n + i];
    }
    if (c == kClone)  // the copy starts with fresh moments (optimize.cpp:332-336, 352-355)
      for (int s = 0; s < S; ++s) {
        raw_out[(size_t)s * cap + p + 1] = raw[(size_t)s * n + i];
        m_out[(size_t)s * cap + p + 1] = 0.f;
        v_out[(size_t)s * cap + p + 1] = 0.f;
      }
    return;
  }
  // split (optimize.cpp:356-366): activate -> angle of the longest basis, axes
#define RAW(j) ((double)raw[(size_t)(j)*n + i])
  int longest = 0;
  double smax = exp(RAW(7));
  for (int k = 1; k < K; ++k) {
    const double s = exp(RAW(7 + k));
    if (s > smax) {
      smax = s;
      longest = k;
    }
  }
  // angle_activation (core.cpp:89-108), as in k_activate
  const double residual = 1.0 / (K - 2);
  double total = 0, th_long = 0;
  for (int j = 0; j < K; ++j) {
    double sg = sigm(RAW(7 + K + j));
    sg = sg < 1e-9 ? 1e-9 : (1.0 - 1e-9 < sg ? 1.0 - 1e-9 : sg);
    total += sg + residual;
    if (j == longest) th_long = total;
  }
  const double a = longest == K - 1 ? kTwoPi : th_long * (kTwoPi / total);
  // quat_to_rotation (geometry.cpp:21-30): columns R_x, R_y
  const double q0 = RAW(3), q1 = RAW(4), q2 = RAW(5), q3 = RAW(6);
  const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
  const double ax[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};
  const double ay[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};
  const double ca = cos(a), sa = sin(a);
  double dir[3];
  for (int j = 0; j < 3; ++j) dir[j] = ca * ax[j] + sa * ay[j];
  const double ln2 = log(2.0);
  for (int child = 0; child < 2; ++child) {
    const long long q = p + child;
    const double f = (child == 0 ? 1.0 : -1.0) * 0.25 * smax;
    for (int s = 0; s < S; ++s) {
      double val = RAW(s);
      if (s < 3) val = val + f * dir[s];
      else if (s >= 7 && s < 7 + K) val = val - ln2;
      raw_out[(size_t)s * cap + q] = (float)val;
      m_out[(size_t)s * cap + q] = 0.f;
      v_out[(size_t)s * cap + q] = 0.f;
    }
  }
#undef RAW
}

// scene_extent (optimize.cpp:375-383): one block, fixed-order min / max
__global__ void k_scene_extent(int n, const float* __restrict__ raw, double* out) {
  __shared__ double lo[3][256], hi[3][256];
  double l[3], h[3];
  for (int j = 0; j < 3; ++j) {
    l[j] = n > 0 ? (double)raw[(size_t)j * n] : 0.0;
    h[j] = l[j];
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int j = 0; j < 3; ++j) {
      const double x = raw[(size_t)j * n + i];
      l[j] = x < l[j] ? x : l[j];
      h[j] = h[j] < x ? x : h[j];
    }
  for (int j = 0; j < 3; ++j) {
    lo[j][threadIdx.x] = l[j];
    hi[j][threadIdx.x] = h[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (n == 0) {
      out[0] = 1.0;
      return;
    }
    for (int t = 1; t < blockDim.x; ++t)
      for (int j = 0; j < 3; ++j) {
        l[j] = lo[j][t] < l[j] ? lo[j][t] : l[j];
        h[j] = h[j] < hi[j][t] ? hi[j][t] : h[j];
      }
    const double d0 = h[0] - l[0], d1 = h[1] - l[1], d2 = h[2] - l[2];
    const double e = 0.5 * sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    out[0] = e < 1e-6 ? 1e-6 : e;
  }
}

}  // namespace
}  // namespace drk

using namespace drk;

extern "C" int drk_densify_accumulate(drk_ctx* c, const float* screen_grad, const uint8_t* touched, int n,
                                      double* accum, int32_t* count) {
  if (!c || n < 0 || (n > 0 && (!screen_grad || !touched || !accum || !count))) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (n > 0) {
    k_densify_accumulate<<<(n + 255) / 256, 256, 0, c->stream>>>(n, screen_grad, touched, accum, count);
    DRK_COUNT_LAUNCH();
  }
  return cuda_check(c, cudaGetLastError(), "densify accumulate");
}

extern "C" int drk_scene_extent(drk_ctx* c, const float* raw, int n, double* out) {
  if (!c || n < 0 || !out || (n > 0 && !raw)) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  k_scene_extent<<<1, 256, 0, c->stream>>>(n, raw, out);
  DRK_COUNT_LAUNCH();
  return cuda_check(c, cudaGetLastError(), "scene extent");
}

extern "C" int drk_densify_and_prune(drk_ctx* c, const float* raw, const float* m, const float* v, int n, int k,
                                     int sh_terms, const double* accum, const int32_t* count,
                                     const drk_densify_config* cfg, double extent, float* raw_out, float* m_out,
                                     float* v_out, int64_t cap, int64_t* n_out) {
  if (!c || !cfg || !n_out || n < 0 || k < 3 || k > 16 || sh_terms < 0) return DRK_ERR_INVALID_ARG;
  if (n > 0 && (!raw || !m || !v || !accum || !count)) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  const int S = 3 + 4 + 2 * k + 3 + 3 * sh_terms;
  *n_out = 0;
  if (n == 0) return DRK_OK;
  int* code = ensure<int>(c->dens_code, 2 * (size_t)n);
  long long* pos = ensure<long long>(c->dens_pos, (size_t)n + 1);
  if (!code || !pos) return set_error(c, DRK_ERR_OOM, "densify scratch");
  int* cnt = code + n;
  cudaStream_t s = c->stream;
  k_densify_decide<<<(n + 255) / 256, 256, 0, s>>>(n, k, raw, accum, count, cfg->densify_grad_threshold,
                                                    cfg->prune_opacity_threshold, cfg->percent_dense * extent, code,
                                                    cnt);
  DRK_COUNT_LAUNCH();
  long long total = 0;
  if (int st = exclusive_scan<int>(c, cnt, n, pos, &total)) return st;
  *n_out = total;
  if (total > cap || !raw_out || !m_out || !v_out)
    return raw_out ? set_error(c, DRK_ERR_INVALID_ARG, "output capacity below the densified count") : DRK_OK;
  k_densify_emit<<<(n + 255) / 256, 256, 0, s>>>(n, k, S, raw, m, v, code, pos, cap, raw_out, m_out, v_out);
  DRK_COUNT_LAUNCH();
  return cuda_check(c, cudaGetLastError(), "densify");
}
