// sort.cuh -- hand-written stable LSD radix sort (onesweep, 8-bit digits).
//
// Replaces np.lexsort (render.py:218-222) twice per frame:
//   * depth sort: 32-bit depth keys of all n items (culled = 0xffffffff, last),
//     values = item index (implicit on the first pass), 4 passes;
//   * tile sort:  16-bit tile ids of the P Gaussian-tile pairs emitted in
//     (depth, index) order, values = item id, ceil(tile_bits/8) passes.
// Stability makes the per-tile order exactly the reference's (depth, index)
// order restricted to the tile.
//
// Per sort: one histogram kernel reads the keys once and builds every pass's
// 256-bin histogram (warp-aggregated shared atomics), then one onesweep
// kernel per pass: a persistent grid takes 4096-key chunks in order from an
// atomic ticket, ranks keys inside the chunk with warp match_any multisplit,
// obtains the chunk's global digit offsets by decoupled look-back over
// earlier chunks, and scatters through shared memory so that global writes
// are contiguous runs per digit. Each key and value is read once and written
// once per pass. All sizes are read from device memory, so a frame contains
// no host synchronization and can be graph-captured.
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kChunk = kSortThreads * kSortItems;  // 4096 keys per chunk
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Histograms of all passes; also zeroes the pass-0 look-back region and
// resets the chunk tickets. hist must be zero on entry.
template <typename K>
__global__ void __launch_bounds__(256) radix_hist_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ n_ptr,
                                                         uint32_t n_static, int passes, int begin_bit,
                                                         uint32_t* __restrict__ hist, uint32_t* __restrict__ lookback0,
                                                         uint32_t* __restrict__ tickets) {
  __shared__ uint32_t sh[4][256];
  const uint32_t n = n_ptr ? *n_ptr : n_static;
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint32_t i = base + threadIdx.x;
    const bool ok = i < n;
    const uint32_t k = ok ? (uint32_t)keys[i] : 0u;
    for (int p = 0; p < passes; ++p) {
      const uint32_t d = (k >> (begin_bit + 8 * p)) & 0xffu;
      const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + lane);
      if (ok && (31 - __clz(peers)) == (int)lane) atomicAdd(&sh[p][d], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
  // zero the first pass's look-back status words and the tickets
  const uint32_t chunks = (n + kChunk - 1) / kChunk;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < chunks * 256u; i += stride) lookback0[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < passes) tickets[threadIdx.x] = 0;
}

template <typename K>
struct OnesweepSmem {
  K keys[kChunk];
  uint32_t vals[kChunk];
  uint32_t whist[8][256];   // per-warp digit counts, then per-warp exclusive offsets
  uint32_t gbase[256];      // global exclusive digit offsets of this pass
  uint32_t lstart[256];     // chunk-local exclusive digit starts
  uint32_t gout[256];       // global position of local slot 0 for each digit
  uint32_t chunk;
};

template <typename K>
__global__ void __launch_bounds__(kSortThreads) onesweep_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ n_ptr, uint32_t n_static,
    const uint32_t* __restrict__ pass_hist, uint32_t* __restrict__ lookback, uint32_t* __restrict__ lookback_next,
    uint32_t* __restrict__ ticket, int shift, int write_keys) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem<K>& S = *reinterpret_cast<OnesweepSmem<K>*>(smem_raw);
  const uint32_t n = n_ptr ? *n_ptr : n_static;
  const uint32_t chunks = (n + kChunk - 1) / kChunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // exclusive scan of this pass's digit histogram (one warp per 32 digits)
  {
    const uint32_t v = pass_hist[tid];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) S.whist[0][warp] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += S.whist[0][w];
    S.gbase[tid] = off + x - v;
    __syncthreads();
  }
  // zero the next pass's look-back region (this pass owns `lookback`)
  if (lookback_next)
    for (uint32_t i = blockIdx.x * blockDim.x + tid; i < chunks * 256u; i += gridDim.x * blockDim.x)
      lookback_next[i] = 0;

  for (;;) {
    if (tid == 0) S.chunk = atomicAdd(ticket, 1u);
    for (int w = 0; w < 8; ++w) S.whist[w][tid] = 0;
    __syncthreads();
    const uint32_t c = S.chunk;
    if (c >= chunks) break;
    const uint32_t cbase = c * kChunk;
    const uint32_t wbase = cbase + warp * 32 * kSortItems;
    uint32_t kk[kSortItems], vv[kSortItems], rk[kSortItems];
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
      const uint32_t i = wbase + it * 32 + lane;
      const bool ok = i < n;
      kk[it] = ok ? (uint32_t)keys_in[i] : 0u;
      vv[it] = ok ? (vals_in ? vals_in[i] : i) : 0u;
    }
    // warp multisplit ranking, in key order (item-major, lane-minor)
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
      const uint32_t i = wbase + it * 32 + lane;
      const bool ok = i < n;
      const uint32_t d = (kk[it] >> shift) & 0xffu;
      const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + lane);
      uint32_t base = 0;
      if (ok) base = S.whist[warp][d];
      __syncwarp();
      if (ok && (31 - __clz(peers)) == lane) S.whist[warp][d] = base + __popc(peers);
      __syncwarp();
      rk[it] = base + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    // per digit: chunk count, per-warp exclusive offsets
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = S.whist[w][tid];
      S.whist[w][tid] = cnt;
      cnt += t;
    }
    // publish the aggregate, then look back for the exclusive prefix
    volatile uint32_t* lb = lookback;
    if (c == 0) {
      lb[tid] = kFlagInc | cnt;
    } else {
      lb[c * 256 + tid] = kFlagAgg | cnt;
    }
    uint32_t excl = 0;
    if (c > 0) {
      int j = (int)c - 1;
      for (;;) {
        const uint32_t s = lb[j * 256 + tid];
        if ((s & ~kValMask) == 0) continue;  // predecessor not published yet
        excl += s & kValMask;
        if (s & kFlagInc) break;
        --j;
      }
      lb[c * 256 + tid] = kFlagInc | (excl + cnt);
    }
    // chunk-local digit starts (block exclusive scan of cnt)
    {
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      __shared__ uint32_t wsum[8];
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      uint32_t off = 0;
      for (int w = 0; w < warp; ++w) off += wsum[w];
      const uint32_t ls = off + x - cnt;
      S.lstart[tid] = ls;
      S.gout[tid] = S.gbase[tid] + excl - ls;
    }
    __syncthreads();
    // scatter into shared memory in chunk-sorted order
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
      const uint32_t i = wbase + it * 32 + lane;
      if (i < n) {
        const uint32_t d = (kk[it] >> shift) & 0xffu;
        const uint32_t pos = S.lstart[d] + S.whist[warp][d] + rk[it];
        S.keys[pos] = (K)kk[it];
        S.vals[pos] = vv[it];
      }
    }
    __syncthreads();
    const uint32_t m = min((uint32_t)kChunk, n - cbase);
    for (uint32_t p = tid; p < m; p += kSortThreads) {
      const K k = S.keys[p];
      const uint32_t d = ((uint32_t)k >> shift) & 0xffu;
      const uint32_t g = S.gout[d] + p;
      if (write_keys) keys_out[g] = k;
      vals_out[g] = S.vals[p];
    }
    __syncthreads();
  }
}

}  // namespace rs
