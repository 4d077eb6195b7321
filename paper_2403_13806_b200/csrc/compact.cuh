// compact.cuh -- visible-index lists and small utilities.
//
// compact_kernel turns a per-Gaussian indicator (visibility.py:204, one byte
// per Gaussian) or an LSB-first bitset (the RVIS on-disk form, io.py:205-206)
// into the ascending index list np.nonzero would give, in one pass: each
// thread owns 32 consecutive flags (one 32-bit mask), the CTA scans the
// popcounts, a decoupled look-back over earlier CTAs (logical order from an
// atomic ticket) supplies the global offset, and threads write their indices.
// rs_render then projects only the listed Gaussians (the reference projects
// all N and filters the order afterwards, render.py:241-244).
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kCompactThreads = 256;
constexpr int kCompactPerBlock = kCompactThreads * 32;

template <bool BITS>
__global__ void __launch_bounds__(kCompactThreads) compact_kernel(const uint8_t* __restrict__ flags, int64_t n,
                                                                  int32_t* __restrict__ out_idx,
                                                                  uint32_t* __restrict__ out_count,
                                                                  unsigned long long* __restrict__ status,
                                                                  uint32_t* __restrict__ ticket) {
  __shared__ uint32_t s_block;
  __shared__ uint32_t s_wsum[8];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_block = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t b = s_block;
  const int64_t start = (int64_t)b * kCompactPerBlock + (int64_t)tid * 32;
  uint32_t mask = 0;
  if (start < n) {
    const int64_t lim = n - start;  // flags available from start
    if (BITS) {
      const uint8_t* p = flags + start / 8;
      const int nbytes = lim >= 32 ? 4 : (int)((lim + 7) / 8);
      for (int k = 0; k < nbytes; ++k) mask |= (uint32_t)__ldg(p + k) << (8 * k);
    } else {
      const uint8_t* p = flags + start;
      if (lim >= 32 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
        const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(p));
        const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if ((w[q] >> (8 * k)) & 0xffu) mask |= 1u << (4 * q + k);
      } else {
        const int m = lim >= 32 ? 32 : (int)lim;
        for (int k = 0; k < m; ++k)
          if (__ldg(p + k)) mask |= 1u << k;
      }
    }
    if (lim < 32) mask &= (1u << lim) - 1u;
  }
  const uint32_t cnt = (uint32_t)__popc(mask);
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t off = 0, total = 0;
  for (int w = 0; w < 8; ++w) {
    if (w < warp) off += s_wsum[w];
    total += s_wsum[w];
  }
  const uint32_t excl = off + x - cnt;
  if (tid == 0) {
    volatile unsigned long long* st = status;
    constexpr unsigned long long AGG = 1ull << 62, INC = 2ull << 62, MASK = (1ull << 62) - 1;
    unsigned long long pre = 0;
    if (b == 0) {
      st[0] = INC | total;
    } else {
      st[b] = AGG | total;
      int j = (int)b - 1;
      while (j >= 0) {
        const unsigned long long s = st[j];
        if ((s & ~MASK) == 0) continue;
        pre += s & MASK;
        if (s & INC) break;
        --j;
      }
      st[b] = INC | (pre + total);
    }
    s_base = pre;
    if ((int64_t)(b + 1) * kCompactPerBlock >= n) *out_count = (uint32_t)(pre + total);
  }
  __syncthreads();
  uint32_t pos = (uint32_t)s_base + excl;
  while (mask) {
    const int k = __ffs(mask) - 1;
    mask &= mask - 1;
    out_idx[pos++] = (int32_t)(start + k);
  }
}

// number of non-finite values over the 11 planes and the SH rows (core.py:522-525)
template <typename T>
__global__ void finite_kernel(const T* __restrict__ planes, const T* __restrict__ sh, int64_t n,
                              int64_t stride, uint32_t* __restrict__ bad) {
  uint32_t local = 0;
  const int64_t total = n * 11 + n * 48;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    T v;
    if (k < n * 11) {
      const int64_t plane = k / n, i = k - plane * n;
      v = __ldg(planes + plane * stride + i);
    } else {
      v = __ldg(sh + (k - n * 11));
    }
    if (!isfinite(v)) ++local;
  }
  local = __reduce_add_sync(0xffffffffu, local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}

__global__ void max_merge_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = max(dst[i], __ldg(src + i));
}

}  // namespace rs
