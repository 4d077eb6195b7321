// sort.cuh -- hand-written stable LSD radix sort (onesweep, 8-bit digits).
//
// Replaces np.lexsort (render.py:218-222): the depth sort of the frame -- 32-bit
// depth keys of the n_visible binned items, values = item index (compacted in
// item order by compact_hist_kernel), 4 passes. Stability keeps equal depths in
// index order; the per-tile lists are then placed in this order without a
// second sort (segbin.cuh), so each tile's list is exactly the reference's
// (depth, index) order restricted to the tile.
//
// Digit histograms of every pass come from the key producer (compact_hist_kernel),
// so each pass is ONE kernel: CTAs take chunks of 256*ITEMS keys in launch order from an atomic ticket, rank
// keys inside the chunk with a warp multisplit (match_any for narrow digits,
// per-bit ballots for 7-8 bit digits, whichever measured faster), publish
// the chunk's digit counts right after loading (before ranking, so successors
// never wait on it), get the chunk's global digit offsets by decoupled
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

// Order-preserving compaction of the binned items' depth keys (culled items carry
// kInvalidKey) into (key, item) arrays for the depth sort, plus the digit histograms of
// all 4 passes over the compacted keys and zeroing of the first pass's look-back words.
// CTAs take chunks of kCompactKeys items from a ticket and find their output offset by
// decoupled look-back; the last chunk publishes n_visible. hist must be zero on entry.
constexpr int kCompactKeys = 256 * 16;

__global__ void __launch_bounds__(256) compact_hist_kernel(const uint32_t* __restrict__ keys_all, uint32_t n,
                                                           uint32_t* __restrict__ keys_out,
                                                           uint32_t* __restrict__ vals_out,
                                                           unsigned long long* __restrict__ status,
                                                           Counters* __restrict__ ctr, uint32_t chunk,
                                                           uint32_t* __restrict__ hist,
                                                           uint32_t* __restrict__ lookback0) {
  pdl_wait();
  pdl_trigger();
  constexpr int IT = kCompactKeys / 256;
  __shared__ uint32_t sh[4][4][256];  // 4 warp pairs x 4 digits
  __shared__ uint32_t s_wcnt[8], s_blk;
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(&ctr->proj_ticket, 1u);
  for (int i = tid; i < 4 * 4 * 256; i += 256) (&sh[0][0][0])[i] = 0;
  __syncthreads();
  const uint32_t b = s_blk, nb = (n + kCompactKeys - 1) / kCompactKeys;
  const uint32_t base = b * kCompactKeys + warp * 32 * IT;  // warp-contiguous items, lane-minor
  uint32_t k[IT];
  uint32_t cnt = 0;
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const uint32_t i = base + it * 32 + lane;
    k[it] = i < n ? keys_all[i] : kInvalidKey;
    cnt += k[it] != kInvalidKey;
  }
  // warp count (in item order within the warp: item-major, lane-minor)
  uint32_t wc = cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wc += __shfl_xor_sync(0xffffffffu, wc, o);
  if (lane == 0) s_wcnt[warp] = wc;
  __syncthreads();
  if (warp == 0) {
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) total += s_wcnt[w];
    volatile unsigned long long* st = status;
    if (lane == 0) st[b] = (b == 0 ? kLbInc : kLbAgg) | total;
    const unsigned long long excl = b == 0 ? 0ull : warp_lookback(st, b, lane);
    if (lane == 0) {
      if (b) st[b] = kLbInc | (excl + total);
      s_base = excl;
      if (b == nb - 1) ctr->n_visible = (uint32_t)(excl + total);
    }
  }
  __syncthreads();
  uint32_t pos = (uint32_t)s_base;
  for (int w = 0; w < warp; ++w) pos += s_wcnt[w];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const bool v = k[it] != kInvalidKey;
    const unsigned bal = __ballot_sync(0xffffffffu, v);
    if (v) {
      const uint32_t at = pos + (uint32_t)__popc(bal & ((1u << lane) - 1u));
      keys_out[at] = k[it];
      vals_out[at] = base + it * 32 + lane;
#pragma unroll
      for (int p = 0; p < 4; ++p) atomicAdd(&sh[warp >> 1][p][(k[it] >> (8 * p)) & 0xffu], 1u);
    }
    pos += (uint32_t)__popc(bal);
  }
  __syncthreads();
  for (int i = tid; i < 4 * 256; i += 256) {
    const uint32_t v = sh[0][0][i] + sh[1][0][i] + sh[2][0][i] + sh[3][0][i];
    if (v) atomicAdd(&hist[i], v);
  }
  // the first depth pass's look-back words: sized for every item (n_visible is not known yet)
  const uint32_t words = (n + chunk - 1) / chunk * 256u;
  for (uint32_t i = b * 256 + tid; i < words; i += nb * 256) lookback0[i] = 0;
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
  uint32_t ccnt[256];       // this chunk's digit counts
  uint32_t wsum[8];
  uint32_t chunk;
};

// One pass over bits [shift, shift + NBITS), NBITS <= 8.
template <typename K, int ITEMS, int NBITS>
__global__ void __launch_bounds__(kSortThreads, 4) onesweep_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ n_ptr, uint32_t n_static,
    const uint32_t* __restrict__ pass_hist, uint32_t* __restrict__ lookback, uint32_t* __restrict__ lookback_next,
    uint32_t* __restrict__ ticket, int shift, int write_keys) {
  pdl_wait();
  pdl_trigger();
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
  if (c > 0) {
#ifndef RS_SORT_LB
#define RS_SORT_LB 4  // measured 4 / 8 / 16 / 32: configs[2] 1557 / 1555 / 1537 / 1496 views/s
#endif
    constexpr int LB = RS_SORT_LB;
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
    const uint32_t i = wbase + it * 32 + lane;
    const bool ok = i < n;
    const uint32_t d = (kk[it] >> shift) & dmask;
    uint32_t peers;
    if (NBITS <= 6) {  // few distinct digits per warp: one MATCH is cheapest
      peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + lane);
    } else {           // many distinct digits: MATCH serialises, per-bit ballots do not
      peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int b = 0; b < NBITS; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
    }
    uint32_t base = 0;
    if (ok) base = S.whist[warp][d];
    __syncwarp();
    if (ok && (31 - __clz(peers)) == lane) S.whist[warp][d] = base + __popc(peers);
    __syncwarp();
    rk[it] = base + __popc(peers & lt);
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
    if (write_keys) keys_out[g] = k;
    vals_out[g] = S.vals[p];
  }
}

// RS_F64 frames: the depth keys are the fp32 roundings of the fp64 depths (monotone, so
// the radix order is the fp64 order except inside runs of equal keys). Each run is
// re-ordered by (fp64 depth, item) -- the reference's exact lexsort((idx, depth))
// (render.py:218-222): the run's first position sorts it by insertion (runs are short:
// a few items share an fp32 depth; equal fp64 depths keep item order, so an already
// ordered run costs one pass).
__global__ void __launch_bounds__(256) tiefix_kernel(const uint32_t* __restrict__ keys, uint32_t* __restrict__ items,
                                                     const uint32_t* __restrict__ n_ptr,
                                                     const Rec64* __restrict__ recs64) {
  pdl_wait();
  pdl_trigger();
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (keys[i + 1] != k || (i > 0 && keys[i - 1] == k)) continue;  // not the start of a run
    uint32_t e = i + 2;
    while (e < n && keys[e] == k) ++e;
    for (uint32_t a = i + 1; a < e; ++a) {
      const uint32_t it = items[a];
      const double d = recs64[it].depth;
      uint32_t b = a;
      while (b > i) {
        const uint32_t pv = items[b - 1];
        const double pd = recs64[pv].depth;
        if (pd < d || (pd == d && pv < it)) break;
        items[b] = pv;
        --b;
      }
      items[b] = it;
    }
  }
}

}  // namespace rs
