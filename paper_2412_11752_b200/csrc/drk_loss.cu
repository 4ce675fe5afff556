// Image losses and metrics of the training step on the device: the full
// drk::loss (reference optimize.cpp:171-204: (1 - w) L1 + w (1 - mean SSIM)
// with its gradient), drk::ssim (:157-166) and drk::psnr (:145-155).
//
// SSIM follows ssim_channel (optimize.cpp:97-143): 11-tap Gaussian (sigma 1.5)
// separable correlation over the valid region of x, y, x^2, y^2, xy; per valid
// pixel the SSIM map s and the three adjoint fields
//   f1 = ds/dmu_x (all paths), f2 = ds/dvar_x, f3 = ds/dcov_xy;
// the gradient w.r.t. the rendered channel is
//   d_x = inv_n (S1 + 2 x S2 + y S3),  S_k = scatter_full(f_k)   (:129-141)
// where scatter_full is the adjoint (full-size, zero-padded) correlation.
//
// Two tiled kernels per call, every channel of a 32 x 16 tile in one CTA:
//   k_ssim_map   (valid-region tile + 10-pixel halo in shared memory)
//                horizontal then vertical taps -> s, f1..f3 (fp64 planes),
//                per-CTA partial sums of s (deterministic final reduction);
//   k_ssim_grad  (image tile + halo of f1..f3) -> adjoint taps -> d_color,
//                the L1 sign term added first as in loss().
// Taps are summed in the reference's order (correlation: i ascending;
// adjoint: contributions in ascending source index) in fp64 with this
// translation unit compiled --fmad=false, and the Gaussian weights come from
// the host's libm exp like the reference's, so s, f_k and d_x are the
// reference's values bit for bit; only the mean reductions are reordered.
#include <cmath>

#include "drk_internal.h"

namespace drk {

int set_error(drk_ctx* c, int status, const std::string& msg);
int cuda_check(drk_ctx* c, cudaError_t e, const char* where);

namespace {

constexpr int kWin = 11, kHalo = kWin - 1;     // optimize.cpp:14
constexpr int kTW = 32, kTH = 16;              // output tile
constexpr int kIW = kTW + kHalo, kIH = kTH + kHalo;  // input tile with halo
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;  // optimize.cpp:16-17
constexpr int kThreads = 256;

struct Gauss {
  double g[kWin];
};

// ssim_kernel (optimize.cpp:23-33), host libm
Gauss ssim_gauss() {
  Gauss G;
  double sum = 0;
  for (int i = 0; i < kWin; ++i) {
    const double d = i - (kWin - 1) / 2.0;
    G.g[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += G.g[i];
  }
  for (double& v : G.g) v /= sum;
  return G;
}

// block-wide sum in a fixed order (warp xor tree, then warps in order)
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

// Valid-region SSIM map of one tile, all channels.  f (GRAD): 3 planes per
// channel, [c][k][vh][vw].  part: per-CTA sums of s, [c][nblocks].
template <bool GRAD, typename T>
__global__ void __launch_bounds__(kThreads) k_ssim_map(const T* __restrict__ xr, const T* __restrict__ yr,
                                                       int W, int H, int C, const Gauss G, double* f,
                                                       double* part) {
  extern __shared__ double sm[];
  double* xs = sm;                  // [kIH][kIW]
  double* ys = xs + kIH * kIW;      // [kIH][kIW]
  double* hp = ys + kIH * kIW;      // [5][kIH][kTW]
  __shared__ double red[kThreads / 32];
  const int vw = W - kHalo, vh = H - kHalo;
  const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
  const int nblk = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  const size_t plane = (size_t)vw * vh;
  for (int c = 0; c < C; ++c) {
    __syncthreads();
    for (int e = threadIdx.x; e < kIH * kIW; e += kThreads) {
      const int r = e / kIW, q = e - r * kIW;
      const int X = x0 + q, Y = y0 + r;
      const bool in = X < W && Y < H;
      xs[e] = in ? (double)xr[((size_t)Y * W + X) * C + c] : 0.0;
      ys[e] = in ? (double)yr[((size_t)Y * W + X) * C + c] : 0.0;
    }
    __syncthreads();
    // horizontal taps (correlate_valid, optimize.cpp:47-53), i ascending
    for (int e = threadIdx.x; e < kIH * kTW; e += kThreads) {
      const int r = e / kTW, j = e - r * kTW;
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
      for (int i = 0; i < kWin; ++i) {
        const double xv = xs[r * kIW + j + i], yv = ys[r * kIW + j + i];
        const double g = G.g[i];
        s0 += g * xv;
        s1 += g * yv;
        s2 += g * (xv * xv);
        s3 += g * (yv * yv);
        s4 += g * (xv * yv);
      }
      hp[(0 * kIH + r) * kTW + j] = s0;
      hp[(1 * kIH + r) * kTW + j] = s1;
      hp[(2 * kIH + r) * kTW + j] = s2;
      hp[(3 * kIH + r) * kTW + j] = s3;
      hp[(4 * kIH + r) * kTW + j] = s4;
    }
    __syncthreads();
    double acc = 0;
    for (int e = threadIdx.x; e < kTH * kTW; e += kThreads) {
      const int r = e / kTW, j = e - r * kTW;
      const int X = x0 + j, Y = y0 + r;
      if (X >= vw || Y >= vh) continue;
      double m[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        double s = 0;
#pragma unroll
        for (int i = 0; i < kWin; ++i) s += G.g[i] * hp[(k * kIH + r + i) * kTW + j];
        m[k] = s;
      }
      // optimize.cpp:111-128, same expression order
      const double ux = m[0], uy = m[1];
      const double vx = m[2] - ux * ux;
      const double vy = m[3] - uy * uy;
      const double vxy = m[4] - ux * uy;
      const double a1 = 2 * ux * uy + kC1, a2 = 2 * vxy + kC2;
      const double b1 = ux * ux + uy * uy + kC1, b2 = vx + vy + kC2;
      const double s = (a1 * a2) / (b1 * b2);
      acc += s;
      if (GRAD) {
        const double ds_dvx = -s / b2;
        const double ds_dvxy = 2 * a1 / (b1 * b2);
        const double ds_dux = 2 * uy * a2 / (b1 * b2) - 2 * ux * s / b1 - 2 * ux * ds_dvx - uy * ds_dvxy;
        const size_t p = (size_t)Y * vw + X;
        double* fc = f + (size_t)c * 3 * plane;
        fc[p] = ds_dux;
        fc[plane + p] = ds_dvx;
        fc[2 * plane + p] = ds_dvxy;
      }
    }
    const double bs = block_sum(acc, red);
    if (threadIdx.x == 0) part[(size_t)c * nblk + bid] = bs;
  }
}

// d_color of loss() (optimize.cpp:184-200) for one image tile, all channels:
// L1 sign term, then + (-w / C) d_x with d_x from the adjoint taps of f1..f3.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_ssim_grad(const T* __restrict__ xr, const T* __restrict__ yr,
                                                        int W, int H, int C, const Gauss G, const double* __restrict__ f,
                                                        double w, double inv_n_img, double inv_n_ssim,
                                                        T* __restrict__ dcol) {
  extern __shared__ double sm[];
  double* fs = sm;                 // [3][kIH][kIW]: f rows y0-10.., cols x0-10..
  double* hp = fs + 3 * kIH * kIW; // [3][kIH][kTW]
  const int vw = W - kHalo, vh = H - kHalo;
  const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
  const size_t plane = (size_t)vw * vh;
  const double scale = -w / C;
  for (int c = 0; c < C; ++c) {
    __syncthreads();
    const double* fc = f + (size_t)c * 3 * plane;
    for (int e = threadIdx.x; e < 3 * kIH * kIW; e += kThreads) {
      const int k = e / (kIH * kIW), rq = e - k * kIH * kIW, r = rq / kIW, q = rq - r * kIW;
      const int X = x0 - kHalo + q, Y = y0 - kHalo + r;
      fs[e] = (X >= 0 && X < vw && Y >= 0 && Y < vh) ? fc[k * plane + (size_t)Y * vw + X] : 0.0;
    }
    __syncthreads();
    // horizontal adjoint (scatter_full, optimize.cpp:69-75): tmp(X) receives
    // g[i] f(X - i) in ascending source index X - i, i.e. i descending
    for (int e = threadIdx.x; e < 3 * kIH * kTW; e += kThreads) {
      const int k = e / (kIH * kTW), rj = e - k * kIH * kTW, r = rj / kTW, j = rj - r * kTW;
      double s = 0;
#pragma unroll
      for (int i = kWin - 1; i >= 0; --i) {
        const double v = fs[(k * kIH + r) * kIW + j + kHalo - i];
        if (v != 0) s += G.g[i] * v;
      }
      hp[(k * kIH + r) * kTW + j] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kTH * kTW; e += kThreads) {
      const int r = e / kTW, j = e - r * kTW;
      const int X = x0 + j, Y = y0 + r;
      if (X >= W || Y >= H) continue;
      double S[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double s = 0;
#pragma unroll
        for (int i = kWin - 1; i >= 0; --i) {
          const double v = hp[(k * kIH + r + kHalo - i) * kTW + j];
          if (v != 0) s += G.g[i] * v;
        }
        S[k] = s;
      }
      const size_t p = ((size_t)Y * W + X) * C + c;
      const double x = xr[p], y = yr[p];
      const double dx = inv_n_ssim * (S[0] + 2.0 * x * S[1] + y * S[2]);  // optimize.cpp:139-140
      const double d = x - y;
      double g = (1.0 - w) * inv_n_img * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0));  // optimize.cpp:184
      g += scale * dx;                                                         // optimize.cpp:196
      dcol[p] = (T)g;
    }
  }
}

// L1 part of loss() (optimize.cpp:180-186): per-CTA sums of |r - t|; the sign
// gradient is written when SSIM is off (otherwise k_ssim_grad writes d_color).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_loss_l1(long long n, const T* __restrict__ r,
                                                      const T* __restrict__ t, double gscale, T* dcol,
                                                      double* part) {
  __shared__ double red[kThreads / 32];
  double acc = 0;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
    const double d = (double)r[i] - (double)t[i];
    acc += fabs(d);
    if (dcol) dcol[i] = (T)(gscale * (d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0)));
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// sum of squared differences (psnr, optimize.cpp:147-151); QUANT: the first
// image through quantize_8bit first (image.cpp:7-14, train's eval metric)
template <bool QUANT, typename T>
__global__ void __launch_bounds__(kThreads) k_sq_diff(long long n, const T* __restrict__ a,
                                                      const T* __restrict__ b, double* part) {
  __shared__ double red[kThreads / 32];
  double acc = 0;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
    double av = (double)a[i];
    if (QUANT) av = round(dmin(1.0, dmax(0.0, av)) * 255.0) / 255.0;
    const double d = av - (double)b[i];
    acc += d * d;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// One thread: fixed-order sums of the partials and the scalar results.
//   mode 0 (loss):  out = {value, l1, mean_ssim}
//   mode 1 (ssim):  out = {mean_ssim}
//   mode 2 (psnr):  out = {psnr, mse}
__global__ void k_loss_final(int mode, const double* l1p, int nl1, const double* sp, int nblk, int C, double inv_n_img,
                             double inv_n_ssim, double w, bool use_ssim, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double l1 = 0;
  for (int b = 0; b < nl1; ++b) l1 += l1p[b];
  if (mode >= 2) {
    const double mse = l1 * inv_n_img;
    out[0] = mse < 1e-10 ? 100.0 : -10.0 * log10(mse);
    out[1] = mse;
    return;
  }
  double mean_ssim = 0;
  if (use_ssim) {
    for (int c = 0; c < C; ++c) {
      double s = 0;
      for (int b = 0; b < nblk; ++b) s += sp[(size_t)c * nblk + b];
      mean_ssim += s * inv_n_ssim;
    }
    mean_ssim /= C;
  }
  if (mode == 1) {
    out[0] = mean_ssim;
    return;
  }
  l1 *= inv_n_img;
  double value = (1.0 - w) * l1;
  if (use_ssim) value += w * (1.0 - mean_ssim);
  out[0] = value;
  out[1] = l1;
  out[2] = mean_ssim;
}

size_t map_smem() { return sizeof(double) * (2 * kIH * kIW + 5 * kIH * kTW); }
size_t grad_smem() { return sizeof(double) * (3 * kIH * kIW + 3 * kIH * kTW); }

template <typename T>
void set_smem_attrs() {
  static drk::PerDeviceOnce once;
  once([] {
    cudaFuncSetAttribute(k_ssim_map<true, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)map_smem());
    cudaFuncSetAttribute(k_ssim_map<false, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)map_smem());
    cudaFuncSetAttribute(k_ssim_grad<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grad_smem());
  });
}

}  // namespace

// mode 0: loss, 1: ssim, 2: psnr, 3: psnr of quantize_8bit(first image)
// T = float (framebuffers of this library) or double (the reference's Image,
// drop-in adapter)
template <typename T>
int run_image_loss(drk_ctx* c, int mode, const T* r, const T* t, int W, int H, int C, double dssim_weight,
                   double* out, T* dcol) {
  if (W < 0 || H < 0 || C <= 0 || !r || !t || !out) return set_error(c, DRK_ERR_INVALID_ARG, "loss arguments");
  const bool window_fits = W >= kWin && H >= kWin;
  if (mode == 1 && !window_fits) return set_error(c, DRK_ERR_DIMENSION, "image smaller than the SSIM window");
  const bool use_ssim = mode == 1 || (mode == 0 && dssim_weight > 0 && window_fits);  // optimize.cpp:173-175
  const double w = (mode == 0 && use_ssim) ? dssim_weight : 0.0;
  cudaStream_t s = c->stream;
  set_smem_attrs<T>();
  const long long n = (long long)W * H * C;
  const double inv_n_img = n > 0 ? 1.0 / (double)n : 0.0;
  const int vw = W - kHalo, vh = H - kHalo;
  const double inv_n_ssim = use_ssim ? 1.0 / ((double)vw * vh) : 0.0;
  const int nl1 = (int)std::max<long long>(1, std::min<long long>((n + kThreads - 1) / kThreads, 148 * 4));
  const dim3 grid(use_ssim ? (vw + kTW - 1) / kTW : 1, use_ssim ? (vh + kTH - 1) / kTH : 1);
  const int nblk = (int)(grid.x * grid.y);
  double* l1p = ensure<double>(c->loss_part, (size_t)nl1 + (size_t)C * nblk);
  double* sp = l1p + nl1;
  double* f = nullptr;
  if (use_ssim && mode == 0) {
    f = ensure<double>(c->ssim_f, (size_t)C * 3 * vw * vh);
    if (!f) return set_error(c, DRK_ERR_OOM, "ssim fields");
  }
  if (!l1p) return set_error(c, DRK_ERR_OOM, "loss partials");
  cudaMemsetAsync(l1p, 0, sizeof(double) * nl1, s);
  const Gauss G = ssim_gauss();
  if (mode >= 2) {
    if (n > 0 && mode == 2) k_sq_diff<false, T><<<nl1, kThreads, 0, s>>>(n, r, t, l1p);
    if (n > 0 && mode == 3) k_sq_diff<true, T><<<nl1, kThreads, 0, s>>>(n, r, t, l1p);
  } else if (mode == 0 && n > 0) {
    k_loss_l1<T><<<nl1, kThreads, 0, s>>>(n, r, t, (1.0 - w) * inv_n_img, use_ssim ? nullptr : dcol, l1p);
  }
  if (use_ssim) {
    if (f) k_ssim_map<true, T><<<grid, kThreads, map_smem(), s>>>(r, t, W, H, C, G, f, sp);
    else k_ssim_map<false, T><<<grid, kThreads, map_smem(), s>>>(r, t, W, H, C, G, nullptr, sp);
    if (f && dcol) {
      const dim3 ig((W + kTW - 1) / kTW, (H + kTH - 1) / kTH);
      k_ssim_grad<T><<<ig, kThreads, grad_smem(), s>>>(r, t, W, H, C, G, f, w, inv_n_img, inv_n_ssim, dcol);
    }
  }
  k_loss_final<<<1, 32, 0, s>>>(mode, l1p, nl1, sp, nblk, C, inv_n_img, inv_n_ssim, w, use_ssim, out);
  launch_counter() += 4;
  return cuda_check(c, cudaGetLastError(), "image loss");
}

}  // namespace drk

using namespace drk;

extern "C" int drk_loss(drk_ctx* c, const float* rendered, const float* target, int width, int height, int channels,
                        double dssim_weight, double* out3, float* d_color) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<float>(c, 0, rendered, target, width, height, channels, dssim_weight, out3, d_color);
}

extern "C" int drk_ssim(drk_ctx* c, const float* a, const float* b, int width, int height, int channels,
                        double* out1) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<float>(c, 1, a, b, width, height, channels, 0.0, out1, nullptr);
}

extern "C" int drk_psnr(drk_ctx* c, const float* a, const float* b, int width, int height, int channels,
                        double* out2) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<float>(c, 2, a, b, width, height, channels, 0.0, out2, nullptr);
}

extern "C" int drk_psnr_quantized(drk_ctx* c, const float* a, const float* b, int width, int height, int channels,
                                  double* out2) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<float>(c, 3, a, b, width, height, channels, 0.0, out2, nullptr);
}

// double-image variants (drk::Image of the reference; the drop-in adapter)
extern "C" int drk_loss_f64(drk_ctx* c, const double* rendered, const double* target, int width, int height,
                            int channels, double dssim_weight, double* out3, double* d_color) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<double>(c, 0, rendered, target, width, height, channels, dssim_weight, out3, d_color);
}

extern "C" int drk_ssim_f64(drk_ctx* c, const double* a, const double* b, int width, int height, int channels,
                            double* out1) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<double>(c, 1, a, b, width, height, channels, 0.0, out1, nullptr);
}

extern "C" int drk_psnr_f64(drk_ctx* c, const double* a, const double* b, int width, int height, int channels,
                            double* out2) {
  if (!c) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  return run_image_loss<double>(c, 2, a, b, width, height, channels, 0.0, out2, nullptr);
}
