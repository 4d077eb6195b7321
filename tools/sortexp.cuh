#pragma once
#include "../paper_2403_13806_b200/csrc/sort.cuh"
namespace rs {
// One pass over bits [shift, shift + NBITS), NBITS <= 8 (compile-time: the
// per-bit ballots unroll into a straight SHF/VOTE/LOP3 sequence).
template <typename K, int ITEMS, int NBITS, int MODE>
__global__ void __launch_bounds__(kSortThreads, 4) exp_kernel(
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
  S.ccnt[tid] = 0;
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
  // early digit counts of the chunk (unordered shared atomics), published at once so that
  // successors' look-back never waits for this chunk's ranking
#pragma unroll
  for (int it = 0; it < ITEMS; ++it)
    if (wbase + it * 32 + lane < n) atomicAdd(&S.ccnt[(kk[it] >> shift) & dmask], 1u);
  __syncthreads();
  const uint32_t cnt = S.ccnt[tid];
  volatile uint32_t* lb = lookback;
  lb[c * 256 + tid] = (c == 0 ? (uint32_t)kFlagInc : (uint32_t)kFlagAgg) | cnt;
  // decoupled look-back for the exclusive prefix (LB predecessors per round trip)
  uint32_t excl = 0;
  if (c > 0 && !(MODE & 1)) {
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
  // warp multisplit ranking in key order (item-major, lane-minor)
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    if (MODE & 2) { rk[it] = it * 32 + lane; continue; }
    const uint32_t i = wbase + it * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = (kk[it] >> shift) & dmask;
    uint32_t peers;
    if (MODE & 8) {
      peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + lane);
    } else {
      peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int b = 0; b < NBITS; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
    }
    if (MODE & 16) {
      const int leader = 31 - __clz(peers);
      uint32_t base = 0;
      if (ok && leader == lane) base = atomicAdd(&S.whist[warp][d], (uint32_t)__popc(peers));
      rk[it] = __popc(peers & lt) + (ok ? 0u : 0u);
      kk[it] |= 0;  // keep
      // broadcast deferred: store leader in rk high bits? use separate pass below
      rk[it] = (rk[it] & 0xffffu) | ((uint32_t)leader << 16);
      S.vals[it * 256 + tid] = base;  // temp: leader's base (vals array reused before scatter)
    } else {
    uint32_t base = 0;
    if (ok) base = S.whist[warp][d];
    __syncwarp();
    if (ok && (31 - __clz(peers)) == lane) S.whist[warp][d] = base + __popc(peers);
    __syncwarp();
    rk[it] = base + __popc(peers & lt);
    }
  }
  if (MODE & 16) {
    __syncwarp();
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const uint32_t leader = rk[it] >> 16;
      const uint32_t base = S.vals[it * 256 + warp * 32 + leader];
      rk[it] = (rk[it] & 0xffffu) + base;
    }
  }
  __syncthreads();
  {  // per digit: per-warp exclusive offsets
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t t = S.whist[w][tid];
      S.whist[w][tid] = run;
      run += t;
    }
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
    if (MODE & 4) { if (g == 0xffffffffu) vals_out[0] = k; continue; }
    if (write_keys) keys_out[g] = k;
    vals_out[g] = S.vals[p];
  }
}

}
