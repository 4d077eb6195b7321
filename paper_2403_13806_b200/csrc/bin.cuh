// bin.cuh -- tile binning: pair emission and per-tile ranges.
//
// The reference composites in one global (depth, index) order with a
// per-Gaussian pixel bbox gate (render.py:218-222, :250-281); there are no
// tiles. Here the bbox [x0,x1)x[y0,y1) of render.py:133-137 is mapped to the
// 16x16 tiles it touches, tx in [x0/16, (x1-1)/16], ty likewise, and one pair
// (tile, item) is emitted per overlap in depth-rank order. A stable sort by
// tile (sort.cuh) then yields each tile's list in exactly the reference's
// (depth, index) order restricted to that tile; ranges_kernel reads the tile
// boundaries off the sorted ids.
//
// Two kernels, so that work is balanced over PAIRS, not Gaussians (near
// Gaussians are both first in depth order and the largest on screen):
//   count_kernel  one thread per depth rank: tile count, block scan, decoupled
//                 look-back (logical block ids from an atomic ticket) ->
//                 exclusive pair offset per rank; total P.
//   emit_kernel   one CTA per 2048 consecutive pairs: the owning ranks of the
//                 CTA's pair range are found by one binary search, their
//                 offsets and rectangles staged in shared memory, and each
//                 thread writes (tile, item) for its pairs -- coalesced stores.
//                 The CTA also accumulates both 8-bit digit histograms of the
//                 tile ids for the tile sort (no separate histogram pass).
#pragma once
#include "rs_common.cuh"

namespace rs {

enum : unsigned long long { kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = (1ull << 62) - 1 };
constexpr int kEmitPairs = 2048;  // pairs per emit CTA

// Decoupled look-back over 64-bit status words (flag in the top 2 bits);
// one warp reads 32 predecessors per step.
__device__ __forceinline__ unsigned long long warp_lookback(volatile unsigned long long* st, uint32_t b, int lane) {
  unsigned long long excl = 0;
  int j = (int)b - 1;
  while (j >= 0) {
    const int k = j - lane;
    unsigned long long s = k >= 0 ? st[k] : kLbInc;  // before block 0: an inclusive zero
    const unsigned ready = __ballot_sync(0xffffffffu, (s & ~kLbMask) != 0);
    if (ready != 0xffffffffu) continue;  // wait until the 32-wide window is published
    const unsigned inc = __ballot_sync(0xffffffffu, (s & kLbInc) != 0);
    const int first = __ffs(inc) - 1;  // nearest inclusive predecessor in the window (lane order = j, j-1, ...)
    unsigned long long v = (inc && lane <= first) || !inc ? (s & kLbMask) : 0ull;
    if (k < 0) v = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    j -= 32;
  }
  return excl;
}

__global__ void __launch_bounds__(256) count_kernel(const uint32_t* __restrict__ items_sorted,
                                                    const Rec* __restrict__ recs, Counters* __restrict__ ctr, int TW,
                                                    uint32_t pair_cap, uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ chunk_owner,
                                                    unsigned long long* __restrict__ status) {
  __shared__ uint32_t s_block;
  __shared__ uint32_t s_wsum[8];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_block = atomicAdd(&ctr->emit_ctr, 1u);
  __syncthreads();
  const uint32_t b = s_block;
  const uint32_t nvis = ctr->n_visible;
  const uint32_t r = b * 256 + tid;
  uint32_t nt = 0;
  if (r < nvis) {
    const int4 d = cullbox_of(recs[items_sorted[r]].d);
    const int tx0 = d.x / kTile, tx1 = (d.y - 1) / kTile, ty0 = d.z / kTile, ty1 = (d.w - 1) / kTile;
    nt = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
  }
  uint32_t x = nt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t off = 0, total = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    off += w < warp ? s_wsum[w] : 0u;
    total += s_wsum[w];
  }
  if (warp == 0) {
    volatile unsigned long long* st = status;
    if (lane == 0) st[b] = (b == 0 ? kLbInc : kLbAgg) | total;
    const unsigned long long excl = b == 0 ? 0ull : warp_lookback(st, b, lane);
    if (lane == 0) {
      if (b) st[b] = kLbInc | (excl + total);
      s_base = excl;
      if (nvis > 0 && b == (nvis - 1) / 256) {
        const unsigned long long end = excl + total;
        ctr->pairs_needed = end;
        ctr->n_pairs = (uint32_t)(end < pair_cap ? end : pair_cap);
        ctr->overflow = end > pair_cap ? 1u : 0u;
      }
    }
  }
  __syncthreads();
  if (r < nvis) {
    const unsigned long long o = s_base + off + x - nt;
    offsets[r] = (uint32_t)(o < 0xffffffffull ? o : 0xffffffffull);
    // this rank owns the first pair of every emit chunk that starts inside [o, o + nt)
    const unsigned long long e = o + nt;
    for (unsigned long long c = (o + kEmitPairs - 1) / kEmitPairs; c * kEmitPairs < e && c * kEmitPairs < pair_cap; ++c)
      chunk_owner[c] = r;
  }
}

__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ items_sorted,
                                                   const Rec* __restrict__ recs, const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ chunk_owner,
                                                   const Counters* __restrict__ ctr, int TW,
                                                   uint16_t* __restrict__ pair_tiles, uint32_t* __restrict__ pair_items,
                                                   uint32_t* __restrict__ tile_hist /* 2 x 256 */,
                                                   uint32_t* __restrict__ lookback0, uint32_t sort_chunk) {
  __shared__ uint32_t s_off[kEmitPairs + 1];
  __shared__ uint16_t s_tx0[kEmitPairs], s_ty0[kEmitPairs], s_tw[kEmitPairs];
  __shared__ uint32_t s_item[kEmitPairs];
  __shared__ uint16_t s_tile_out[kEmitPairs];
  __shared__ uint32_t s_item_out[kEmitPairs];
  __shared__ uint32_t s_hist[2][256];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t P = ctr->n_pairs, nvis = ctr->n_visible;
  // zero the tile sort's first-pass look-back words
  const uint32_t lb_words = (P + sort_chunk - 1) / sort_chunk * 256u;
  for (uint32_t k = blockIdx.x * blockDim.x + tid; k < lb_words; k += gridDim.x * blockDim.x) lookback0[k] = 0;
  const uint32_t k0 = blockIdx.x * kEmitPairs;
  if (k0 >= P) return;
  const uint32_t k1 = min(P, k0 + kEmitPairs);
  for (int i = tid; i < 512; i += 256) (&s_hist[0][0])[i] = 0;
  const uint32_t r0 = chunk_owner[blockIdx.x];
  // owners of [k0, k1): ranks r0 .. owner(k1 - 1) <= chunk_owner[next chunk]; at most k1 - k0 of them
  const uint32_t rlast = k1 < P ? chunk_owner[blockIdx.x + 1] : nvis - 1;
  const uint32_t nown = min((uint32_t)kEmitPairs, rlast - r0 + 1);
  for (uint32_t i = tid; i < nown; i += 256) {
    const uint32_t o = offsets[r0 + i];
    s_off[i] = o;
    if (o < k1) {
      const uint32_t it = items_sorted[r0 + i];
      const int4 d = cullbox_of(recs[it].d);
      const int tx0 = d.x / kTile, tx1 = (d.y - 1) / kTile;
      s_tx0[i] = (uint16_t)tx0; s_ty0[i] = (uint16_t)(d.z / kTile); s_tw[i] = (uint16_t)(tx1 - tx0 + 1);
      s_item[i] = it;
    }
  }
  if (tid == 0) s_off[nown] = 0xffffffffu;
  __syncthreads();
  // each thread emits 8 consecutive pairs into shared memory: one binary search, then a forward walk
  const uint32_t q0 = k0 + 8 * tid;
  if (q0 < k1) {
    uint32_t lo = 0, hi = nown - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= q0) lo = mid; else hi = mid - 1;
    }
    uint32_t j = lo;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t k = q0 + q;
      if (k >= k1) break;
      while (s_off[j + 1] <= k) ++j;
      const uint32_t local = k - s_off[j];
      const uint32_t tw = s_tw[j];
      const uint32_t row = local / tw;
      s_tile_out[8 * tid + q] = (uint16_t)((s_ty0[j] + row) * TW + s_tx0[j] + (local - row * tw));
      s_item_out[8 * tid + q] = s_item[j];
    }
  }
  __syncthreads();
  // coalesced copy-out + digit histograms of the tile sort (uniform trip count: full-warp votes)
  const uint32_t npair = k1 - k0;
  for (uint32_t p0 = 0; p0 < npair; p0 += 256) {
    const uint32_t p = p0 + tid;
    const bool ok = p < npair;
    const uint32_t tile = ok ? (uint32_t)s_tile_out[p] : 0u;
    if (ok) {
      pair_tiles[k0 + p] = (uint16_t)tile;
      pair_items[k0 + p] = s_item_out[p];
      atomicAdd(&s_hist[0][tile & 255], 1u);
    }
    // high digit: consecutive pairs mostly share it -> one shared atomic per run of equal digits
    const uint32_t hi8 = ok ? tile >> 8 : 0xffffffffu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, hi8, 1);
    const uint32_t next = __shfl_down_sync(0xffffffffu, hi8, 1);
    const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || prev != hi8);
    if (ok && (lane == 31 || next != hi8)) {
      const int run_start = 31 - __clz(starts & ((2u << lane) - 1u));
      atomicAdd(&s_hist[1][hi8], (uint32_t)(lane - run_start + 1));
    }
  }
  __syncthreads();
  for (int i = tid; i < 512; i += 256) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(&tile_hist[i], v);
  }
}

// Per-tile [start, end) from the tile-sorted keys: a pair starts (ends) its
// tile's range when its predecessor (successor) has another tile id. Ranges
// of empty tiles stay at the zero the frame memset wrote.
__global__ void __launch_bounds__(256) ranges_kernel(const uint16_t* __restrict__ tiles, const Counters* __restrict__ ctr,
                                                     uint2* __restrict__ ranges) {
  const uint32_t P = ctr->n_pairs;
  const uint32_t k0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8u;  // 8 consecutive pairs per thread
  if (k0 >= P) return;
  uint32_t t[8];
  if (k0 + 8 <= P) {
    const uint4 v = *reinterpret_cast<const uint4*>(tiles + k0);  // k0 is a multiple of 8: 16-B aligned
    t[0] = v.x & 0xffffu; t[1] = v.x >> 16; t[2] = v.y & 0xffffu; t[3] = v.y >> 16;
    t[4] = v.z & 0xffffu; t[5] = v.z >> 16; t[6] = v.w & 0xffffu; t[7] = v.w >> 16;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = k0 + q < P ? tiles[k0 + q] : 0xffffffffu;
  }
  const uint32_t prev = k0 ? tiles[k0 - 1] : 0xffffffffu;
  const uint32_t next = k0 + 8 < P ? tiles[k0 + 8] : 0xffffffffu;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t k = k0 + q;
    if (k >= P) break;
    if ((q ? t[q - 1] : prev) != t[q]) ranges[t[q]].x = k;
    if ((q < 7 ? t[q + 1] : next) != t[q]) ranges[t[q]].y = k + 1;
  }
}

}  // namespace rs
