// bsort.cuh -- the depth sort of small frames (at most kBsortMaxItems projected items: the
// visibility-filtered index lists of configs[3], configs[0]) in ONE CTA's shared memory.
//
// Same result as dsort_kernel / the onesweep path (np.lexsort((idx, depth)) of
// render.py:218-222 over the binned items: stable LSD radix sort of the 32-bit depth keys,
// 8-bit digits, 4 passes, values = item index). The grid-wide sorts pay a fixed latency per
// pass (grid barrier, digit tables through L2, key loads from L2) that dominates at a few
// thousand keys; here every pass is a few __syncthreads over shared memory:
//   the binned keys are compacted in item order into shared memory (block scan of the
//   valid flags), then per pass: warp w ranks its contiguous slice of the keys 32 at a time
//   (warp multisplit, per-warp digit counters), one block pass turns the 32 x 256 counters
//   into each warp's digit starts (digit-major: digit, then warp, then rank -- stable), and
//   the keys and values move to the other buffer. The last pass writes kA / vA.
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kBsortThreads = 1024;
constexpr int kBsortWarps = kBsortThreads / 32;
constexpr uint32_t kBsortMaxItems = 8192;

struct BsortSmem {
  uint32_t keys[2][kBsortMaxItems];
  uint32_t vals[2][kBsortMaxItems];
  uint32_t whist[kBsortWarps][256];  // per-warp digit counts, then per-warp digit starts
  uint32_t wsum[kBsortWarps];
  uint32_t n;
};

template <bool LAST_KEYS>
__global__ void __launch_bounds__(kBsortThreads, 1) bsort_kernel(const uint32_t* __restrict__ keys_all,
                                                                 uint32_t n_items, uint32_t* __restrict__ kA,
                                                                 uint32_t* __restrict__ vA,
                                                                 Counters* __restrict__ ctr) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char bsort_smem[];
  BsortSmem& S = *reinterpret_cast<BsortSmem*>(bsort_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  // compaction: thread t owns items [8t, 8t + 8) (n_items <= 8192)
  constexpr int kPer = kBsortMaxItems / kBsortThreads;
  uint32_t k8[kPer], cnt = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const uint32_t i = tid * kPer + q;
    k8[q] = i < n_items ? __ldcg(keys_all + i) : kInvalidKey;
    cnt += k8[q] != kInvalidKey ? 1u : 0u;
  }
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) S.wsum[warp] = x;
  __syncthreads();
  uint32_t run = x - cnt, all = 0;
  for (int w = 0; w < kBsortWarps; ++w) {
    const uint32_t v = S.wsum[w];
    run += w < warp ? v : 0u;
    all += v;
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q)
    if (k8[q] != kInvalidKey) {
      S.keys[0][run] = k8[q];
      S.vals[0][run] = tid * kPer + q;
      ++run;
    }
  const uint32_t n = all;
  const uint32_t slice = (n + kBsortWarps - 1) / kBsortWarps;  // warp w: positions [w slice, (w+1) slice)
  const uint32_t lo = min(warp * slice, n), hi = min(lo + slice, n);
  int cur = 0;
  for (int p = 0; p < 4; ++p) {
    const int shift = 8 * p;
    for (int i = tid; i < kBsortWarps * 256; i += kBsortThreads) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    // per-warp digit counts of its slice
    for (uint32_t j = lo + lane; j < hi; j += 32) atomicAdd(&S.whist[warp][(S.keys[cur][j] >> shift) & 0xffu], 1u);
    __syncthreads();
    // digit-major exclusive scan over (digit, warp): digit starts (thread d < 256, a block scan
    // over the digit totals), then each warp's start inside its digit's run
    uint32_t c = 0;
    if (tid < 256) {
      for (int w = 0; w < kBsortWarps; ++w) c += S.whist[w][tid];
      x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) S.wsum[warp] = x;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t st = x - c;
      for (int w = 0; w < warp; ++w) st += S.wsum[w];
      for (int w = 0; w < kBsortWarps; ++w) {
        const uint32_t v = S.whist[w][tid];
        S.whist[w][tid] = st;
        st += v;
      }
    }
    __syncthreads();
    // stable scatter: each warp walks its slice in order, 32 keys at a time
    const int nxt = cur ^ 1;
    for (uint32_t base = lo; base < hi; base += 32) {
      const uint32_t j = base + lane;
      const bool ok = j < hi;
      const uint32_t k = ok ? S.keys[cur][j] : 0u, v = ok ? S.vals[cur][j] : 0u;
      const uint32_t d = (k >> shift) & 0xffu;
      uint32_t peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int bt = 0; bt < 8; ++bt) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> bt) & 1u);
        peers &= ((d >> bt) & 1u) ? bal : ~bal;
      }
      uint32_t r0 = 0;
      if (ok) r0 = S.whist[warp][d];
      __syncwarp();
      if (ok && (31 - __clz(peers)) == lane) S.whist[warp][d] = r0 + __popc(peers);
      __syncwarp();
      if (ok) {
        const uint32_t pos = r0 + __popc(peers & lt);
        if (p < 3) {
          S.keys[nxt][pos] = k;
          S.vals[nxt][pos] = v;
        } else {
          if (LAST_KEYS) kA[pos] = k;
          vA[pos] = v;
        }
      }
    }
    __syncthreads();
    cur = nxt;
  }
  if (tid == 0) ctr->n_visible = n;
}

}  // namespace rs
