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
// Digit histograms of every pass come from the key producer (radix_hist_kernel
// for depth keys, emit_kernel for tile ids), so each pass is ONE kernel: CTAs
// take chunks of 256*ITEMS keys in launch order from an atomic ticket, rank
// keys inside the chunk with a warp multisplit built from one ballot per digit
// bit (no match instructions: a fixed, fully pipelined ALU sequence), publish
// the chunk's digit counts, get the chunk's global digit offsets by decoupled
// look-back over earlier chunks (4 predecessors per load round), and scatter
// through shared memory so global writes are contiguous runs per digit.
// Keys and values are read once and written once per pass; sizes come from
// device memory, so a frame has no host synchronization.
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr int kSortThreads = 256;
constexpr int kMinChunk = kSortThreads * 8;  // smallest chunk used (look-back region sizing)
enum : uint32_t { kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1 };

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Digit histograms of all passes of a 32-bit key sort (per-warp shared
// sub-histograms), plus zeroing of the first pass's look-back words.
// hist must be zero on entry.
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint32_t* __restrict__ keys, uint32_t n, int passes,
                                                         uint32_t chunk, uint32_t* __restrict__ hist,
                                                         uint32_t* __restrict__ lookback0) {
  __shared__ uint32_t sh[8][4][256];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 4 * 256; i += blockDim.x) (&sh[0][0][0])[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[warp][p][(k >> (8 * p)) & 0xffu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += (&sh[w][0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
  const uint32_t words = (n + chunk - 1) / chunk * 256u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) lookback0[i] = 0;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <typename K, int ITEMS>
struct OnesweepSmem {
  K keys[kSortThreads * ITEMS];
  uint32_t vals[kSortThreads * ITEMS];
  uint32_t vstage[kSortThreads * ITEMS];  // this chunk's values in input order (cp.async prefetch)
  uint32_t whist[8][256];   // per-warp digit counts, then per-warp exclusive offsets
  uint32_t gbase[256];      // global exclusive digit offsets of this pass
  uint32_t lstart[256];     // chunk-local exclusive digit starts
  uint32_t gout[256];       // global position of local slot 0 for each digit
  uint32_t wsum[8];
  uint32_t chunk;
};

// One pass over bits [shift, shift + NBITS), NBITS <= 8 (compile-time: the
// per-bit ballots unroll into a straight SHF/VOTE/LOP3 sequence).
template <typename K, int ITEMS, int NBITS>
__global__ void __launch_bounds__(kSortThreads, 4) onesweep_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ n_ptr, uint32_t n_static,
    const uint32_t* __restrict__ pass_hist, uint32_t* __restrict__ lookback, uint32_t* __restrict__ lookback_next,
    uint32_t* __restrict__ ticket, int shift, int write_keys) {
  constexpr uint32_t CHUNK = kSortThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem<K, ITEMS>& S = *reinterpret_cast<OnesweepSmem<K, ITEMS>*>(smem_raw);
  const uint32_t n = n_ptr ? *n_ptr : n_static;
  const uint32_t chunks = (n + CHUNK - 1) / CHUNK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t dmask = (1u << NBITS) - 1u;

  if (tid == 0) S.chunk = atomicAdd(ticket, 1u);
#pragma unroll
  for (int w = 0; w < 8; ++w) S.whist[w][tid] = 0;
  if (lookback_next)  // zero the next pass's look-back words (this pass owns `lookback`)
    for (uint32_t i = blockIdx.x * blockDim.x + tid; i < chunks * 256u; i += gridDim.x * blockDim.x)
      lookback_next[i] = 0;
  __syncthreads();
  const uint32_t c = S.chunk;
  if (c >= chunks) return;

  {  // exclusive scan of this pass's digit histogram
    const uint32_t v = pass_hist[tid];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += S.wsum[w];
    S.gbase[tid] = off + x - v;
  }

  const uint32_t cbase = c * CHUNK;
  const uint32_t wbase = cbase + warp * 32 * ITEMS;
  const uint32_t lt = lanemask_lt();
  const uint32_t m = min(CHUNK, n - cbase);
  if (vals_in) {  // prefetch the chunk's values (16-byte cp.async, zero-filled tail) behind the ranking
    for (uint32_t q = tid; q < CHUNK / 4; q += kSortThreads) {
      const uint32_t e = 4 * q;
      const uint32_t bytes = e < m ? min(16u, 4 * (m - e)) : 0u;
      cp_async16(&S.vstage[e], vals_in + cbase + (bytes ? e : 0), bytes);
    }
  }
  uint32_t kk[ITEMS], rk[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    kk[it] = i < n ? (uint32_t)keys_in[i] : 0u;
  }
  // warp multisplit ranking in key order (item-major, lane-minor)
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const uint32_t i = wbase + it * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = (kk[it] >> shift) & dmask;
    uint32_t peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
    for (int b = 0; b < NBITS; ++b) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    uint32_t base = 0;
    if (ok) base = S.whist[warp][d];
    __syncwarp();
    if (ok && (31 - __clz(peers)) == lane) S.whist[warp][d] = base + __popc(peers);
    __syncwarp();
    rk[it] = base + __popc(peers & lt);
  }
  __syncthreads();
  uint32_t cnt = 0;  // per digit: chunk count, per-warp exclusive offsets
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t t = S.whist[w][tid];
    S.whist[w][tid] = cnt;
    cnt += t;
  }
  // publish the aggregate, then look back for the exclusive prefix: each digit thread
  // reads LB predecessors per round trip (independent loads), then folds them in order
  volatile uint32_t* lb = lookback;
  lb[c * 256 + tid] = (c == 0 ? (uint32_t)kFlagInc : (uint32_t)kFlagAgg) | cnt;
  uint32_t excl = 0;
  if (c > 0) {
    constexpr int LB = 4;
    int j = (int)c - 1;
    for (;;) {
      uint32_t s[LB];
#pragma unroll
      for (int q = 0; q < LB; ++q) s[q] = j - q >= 0 ? lb[(j - q) * 256 + tid] : (uint32_t)kFlagInc;
      int q = 0;
      bool fin = false;
#pragma unroll
      for (int qq = 0; qq < LB; ++qq) {
        if (!fin && q == qq) {
          if ((s[qq] & ~(uint32_t)kValMask) == 0) {
            q = -1 - qq;  // not published yet: resume from here
          } else {
            excl += s[qq] & kValMask;
            if (s[qq] & kFlagInc) fin = true; else q = qq + 1;
          }
        }
      }
      if (fin) break;
      j -= q >= 0 ? q : (-1 - q);
    }
    lb[c * 256 + tid] = kFlagInc | (excl + cnt);
  }
  {  // chunk-local digit starts (block exclusive scan of cnt)
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncthreads();  // wsum reuse
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += S.wsum[w];
    const uint32_t ls = off + x - cnt;
    S.lstart[tid] = ls;
    S.gout[tid] = S.gbase[tid] + excl - ls;
  }
  if (vals_in) cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {  // scatter into shared memory in chunk-sorted order
    const uint32_t i = wbase + it * 32 + lane;
    if (i < n) {
      const uint32_t d = (kk[it] >> shift) & dmask;
      const uint32_t pos = S.lstart[d] + S.whist[warp][d] + rk[it];
      S.keys[pos] = (K)kk[it];
      S.vals[pos] = vals_in ? S.vstage[i - cbase] : i;
    }
  }
  __syncthreads();
  for (uint32_t p = tid; p < m; p += kSortThreads) {
    const K k = S.keys[p];
    const uint32_t g = S.gout[((uint32_t)k >> shift) & dmask] + p;
    if (write_keys) keys_out[g] = k;
    vals_out[g] = S.vals[p];
  }
}

}  // namespace rs
