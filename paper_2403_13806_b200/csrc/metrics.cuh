// metrics.cuh -- image metrics on the device (reference
// metrics.py:34-117): MSE / PSNR and the windowed SSIM with its gradient (the
// training loss and the benchmark / prune-sweep quality numbers).
//
// float64 throughout, the reference's formulas term by term: SSIM per channel
// over 'valid' windows (correlate2d with the normalised win x win Gaussian the
// host builds exactly as gaussian_window does), s = (a1 a2) / (b1 b2) with
// C1 = 0.01^2, C2 = 0.03^2; the gradient as metrics.py:94-109: per window
// g_mu, g_vx, g_vxy, then 'full' convolutions back to the pixels. Sums are
// fp64 atomics (order-dependent only in the last bits).
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kMaxSsimWin = 31;

__global__ void __launch_bounds__(256) sq_diff_sum_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t n, double* __restrict__ out) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = __dsub_rn(a[i], b[i]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// one thread per (valid window, channel): local means / variances / covariance -> s
// (atomically summed) and, with grad maps, the window's g_mu, g_vx, g_vxy
__global__ void __launch_bounds__(256) ssim_window_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                          int H, int W, int C, int win,
                                                          const double* __restrict__ kern, double* __restrict__ sum,
                                                          double* __restrict__ gmaps) {
  const int Ho = H - win + 1, Wo = W - win + 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)Ho * Wo * C;
  double s = 0.0;
  if (idx < total) {
    const int ch = (int)(idx % C);
    const int64_t pix = idx / C;
    const int i = (int)(pix / Wo), j = (int)(pix % Wo);
    double mx = 0.0, my = 0.0, xx = 0.0, yy = 0.0, xy = 0.0;
    for (int u = 0; u < win; ++u)
      for (int v = 0; v < win; ++v) {
        const double k = kern[u * win + v];
        const int64_t p = ((int64_t)(i + u) * W + (j + v)) * C + ch;
        const double a = x[p], b = y[p];
        mx += a * k;
        my += b * k;
        xx += (a * a) * k;
        yy += (b * b) * k;
        xy += (a * b) * k;
      }
    const double vx = xx - mx * mx, vy = yy - my * my, vxy = xy - mx * my;
    const double a1 = 2.0 * mx * my + 1e-4, a2 = 2.0 * vxy + 9e-4;
    const double b1 = mx * mx + my * my + 1e-4, b2 = vx + vy + 9e-4;
    s = (a1 * a2) / (b1 * b2);
    if (gmaps) {
      const double d = b1 * b2;
      const double ds_da1 = a2 / d, ds_da2 = a1 / d, ds_db1 = -s / b1, ds_db2 = -s / b2;
      const double g_mu = ds_da1 * 2.0 * my + ds_db1 * 2.0 * mx + ds_db2 * (-2.0 * mx) + ds_da2 * 2.0 * (-my);
      const int64_t q = ((int64_t)ch * Ho + i) * Wo + j;  // channel-major window maps
      const int64_t plane = (int64_t)Ho * Wo * C;
      gmaps[q] = g_mu;
      gmaps[plane + q] = ds_db2;
      gmaps[2 * plane + q] = ds_da2 * 2.0;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(sum, s);
}

// dSSIM/dx per pixel: 'full' convolutions of the window maps (metrics.py:106-109), / n_windows
__global__ void __launch_bounds__(256) ssim_grad_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                        int H, int W, int C, int win,
                                                        const double* __restrict__ kern,
                                                        const double* __restrict__ gmaps, double inv_n,
                                                        double* __restrict__ grad) {
  const int Ho = H - win + 1, Wo = W - win + 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)H * W * C) return;
  const int ch = (int)(idx % C);
  const int64_t pix = idx / C;
  const int r = (int)(pix / W), c = (int)(pix % W);
  const int64_t plane = (int64_t)Ho * Wo * C;
  double cm = 0.0, cv = 0.0, cxy = 0.0;
  for (int u = 0; u < win; ++u) {
    const int i = r - u;
    if (i < 0 || i >= Ho) continue;
    for (int v = 0; v < win; ++v) {
      const int j = c - v;
      if (j < 0 || j >= Wo) continue;
      const double k = kern[u * win + v];
      const int64_t q = ((int64_t)ch * Ho + i) * Wo + j;
      cm += gmaps[q] * k;
      cv += gmaps[plane + q] * k;
      cxy += gmaps[2 * plane + q] * k;
    }
  }
  grad[idx] = (cm + 2.0 * x[idx] * cv + y[idx] * cxy) * inv_n;
}

// Nearest cluster centre of each camera position (visibility.py:80-83):
// Euclidean distance as np.linalg.norm computes it (sqrt(((dx^2 + dy^2) + dz^2)),
// float64), argmin with the lowest index on ties; one thread per position.
__global__ void __launch_bounds__(256) nearest_cluster_kernel(const double* __restrict__ centers, int k,
                                                              const double* __restrict__ pos, int64_t m,
                                                              int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
  double best = 0.0;
  int arg = 0;
  for (int j = 0; j < k; ++j) {
    const double dx = __dsub_rn(centers[3 * j], px), dy = __dsub_rn(centers[3 * j + 1], py),
                 dz = __dsub_rn(centers[3 * j + 2], pz);
    const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    if (j == 0 || d < best) {  // strict: the first minimum wins (np.argmin)
      best = d;
      arg = j;
    }
  }
  out[i] = arg;
}

}  // namespace rs
