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
//   count_kernel  one thread per depth rank (1024-rank CTAs): tile count, block scan, decoupled
//                 look-back (logical block ids from an atomic ticket) ->
//                 exclusive pair offset per rank; total P.
//   emit_kernel   one CTA per 2048 consecutive pairs: the owning ranks of the
//                 CTA's pair range come from the count kernel's chunk owners;
//                 a warp per owner computes its tile-row spans and marks the
//                 row segments inside the window; a block max-scan maps every
//                 pair slot to its segment and each thread writes (tile, item)
//                 for its 8 pairs -- coalesced stores.
//                 The CTA also accumulates both 8-bit digit histograms of the
//                 tile ids for the tile sort (no separate histogram pass).
#pragma once
#include "rows.cuh"
#include "rs_common.cuh"

namespace rs {

enum : unsigned long long { kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = (1ull << 62) - 1 };
constexpr int kEmitPairs = 2048;  // pairs per emit CTA
constexpr int kCountThreads = 1024;  // ranks per count CTA (few CTAs: short look-back chains)

// Decoupled look-back over 64-bit status words (flag in the top 2 bits);
// one warp reads 32 predecessors per step.
__device__ __forceinline__ unsigned long long warp_lookback(volatile unsigned long long* st, uint32_t b, int lane) {
  unsigned long long excl = 0;
  int j = (int)b - 1;
  while (j >= 0) {
    const int k = j - lane;  // lane 0 = nearest predecessor
    const unsigned long long s = k >= 0 ? st[k] : (unsigned long long)kLbInc;  // before block 0: inclusive zero
    const unsigned ready = __ballot_sync(0xffffffffu, (s & ~(unsigned long long)kLbMask) != 0);
    const unsigned inc = __ballot_sync(0xffffffffu, (s & (unsigned long long)kLbInc) != 0) & ready;
    const unsigned notready = ~ready;
    // use the window up to (and including) the nearest inclusive entry, or up to the first
    // unpublished entry, whichever comes first
    const int first_inc = inc ? __ffs(inc) - 1 : 32;
    const int first_nr = notready ? __ffs(notready) - 1 : 32;
    const int take = first_inc < first_nr ? first_inc + 1 : first_nr;  // lanes [0, take)
    unsigned long long v = (lane < take && k >= 0) ? (s & (unsigned long long)kLbMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (first_inc < first_nr) break;
    j -= take;
  }
  return excl;
}

__global__ void __launch_bounds__(kCountThreads) count_kernel(const uint32_t* __restrict__ items_sorted,
                                                    const uint32_t* __restrict__ tcount, Counters* __restrict__ ctr,
                                                    uint32_t pair_cap, uint32_t* __restrict__ offsets,
                                                    uint32_t* __restrict__ chunk_owner,
                                                    unsigned long long* __restrict__ status,
                                                    Sticky* __restrict__ sticky) {
  __shared__ uint32_t s_block;
  __shared__ uint32_t s_wsum[kCountThreads / 32];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_block = atomicAdd(&ctr->emit_ctr, 1u);
  __syncthreads();
  const uint32_t b = s_block;
  const uint32_t nvis = ctr->n_visible;
  if (b * kCountThreads >= nvis && b > 0) return;  // no ranks here, and no later block needs this status
  const uint32_t r = b * kCountThreads + tid;
  const uint32_t nt = r < nvis ? tcount[items_sorted[r]] : 0u;  // row-span pair count (project_kernel)
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
  for (int w = 0; w < kCountThreads / 32; ++w) {
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
      if (nvis > 0 && b == (nvis - 1) / kCountThreads) {
        const unsigned long long end = excl + total;
        ctr->pairs_needed = end;
        ctr->n_pairs = (uint32_t)(end < pair_cap ? end : pair_cap);
        ctr->overflow = end > pair_cap ? 1u : 0u;
        if (end > pair_cap) {  // survives the next frame's counter reset (checked once per batch)
          atomicOr(&sticky->overflowed, 1u);
          atomicMax(&sticky->pairs_needed_max, end);
        }
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

constexpr int kEmitOwners = 256;  // owners staged per batch (one per thread)

__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ items_sorted,
                                                   const Rec* __restrict__ recs, const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ chunk_owner,
                                                   const Counters* __restrict__ ctr, int TW,
                                                   uint16_t* __restrict__ pair_tiles, uint32_t* __restrict__ pair_items,
                                                   uint32_t* __restrict__ tile_hist /* 2 x 256 */,
                                                   uint32_t* __restrict__ lookback0, uint32_t sort_chunk) {
  // A "segment" is one tile row of one Gaussian: consecutive pairs with consecutive tile ids.
  // Segment data is keyed by the CTA-local slot of its first pair inside this window.
  __shared__ __align__(16) uint16_t s_seg_tile[kEmitPairs];
  __shared__ uint32_t s_seg_item[kEmitPairs];
  __shared__ __align__(16) uint16_t s_tile_out[kEmitPairs];
  // s_start (segment start marks) and s_item_out share storage (a barrier separates the
  // last mark read from the first item write)
  __shared__ __align__(16) int s_start_item[kEmitPairs];
  int* const s_start = s_start_item;
  uint32_t* const s_item_out = reinterpret_cast<uint32_t*>(s_start_item);
  __shared__ uint32_t s_hist[2][256];
  __shared__ int s_wmax[8];
  // owner batch: row geometry, record boxes, item and the exclusive prefix of their row counts
  __shared__ RowGeom s_g[kEmitOwners];
  __shared__ int4 s_cb[kEmitOwners];
  __shared__ uint32_t s_oitem[kEmitOwners];
  __shared__ int s_rpre[kEmitOwners + 1];
  __shared__ uint32_t s_wsum[8];
  __shared__ uint32_t s_o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t P = ctr->n_pairs, nvis = ctr->n_visible;
  // zero the tile sort's first-pass look-back words
  const uint32_t lb_words = (P + sort_chunk - 1) / sort_chunk * 256u;
  for (uint32_t k = blockIdx.x * blockDim.x + tid; k < lb_words; k += gridDim.x * blockDim.x) lookback0[k] = 0;
  const uint32_t k0 = blockIdx.x * kEmitPairs;
  if (k0 >= P) return;
  const uint32_t k1 = min(P, k0 + kEmitPairs);
  for (int i = tid; i < 512; i += 256) (&s_hist[0][0])[i] = 0;
  for (int i = tid; i < kEmitPairs; i += 256) s_start[i] = -1;
  // owners of [k0, k1): ranks r0 .. owner(k1 - 1) <= chunk_owner[next chunk] (ranks without
  // pairs may lie in between), staged 256 at a time. Their tile rows are flattened across the
  // CTA (8 consecutive rows per thread); a block scan of the rows' span widths gives every
  // row segment's pair position -- consecutive ranks own consecutive pair ranges, so the
  // position is the batch's first offset plus the prefix -- and each segment overlapping the
  // window leaves a start mark.
  const uint32_t r0 = chunk_owner[blockIdx.x];
  const uint32_t rlast = k1 < P ? chunk_owner[blockIdx.x + 1] : nvis - 1;
  for (uint32_t rb = r0; rb <= rlast; rb += kEmitOwners) {
    __syncthreads();  // previous batch's staging fully consumed
    const uint32_t r = rb + tid;
    int nrows = 0;
    if (r <= rlast) {
      const uint32_t o = offsets[r];
      if (o < k1) {
        const uint32_t it = items_sorted[r];
        const Rec* R = recs + it;
        const int4 d = __ldg(&R->d);
        const int4 cb = cullbox_of(d);
        if (cullbox_ell(d)) s_g[tid] = row_geom(__ldg(&R->a), __ldg(&R->b));  // else: full rows
        s_cb[tid] = d;
        s_oitem[tid] = it;
        nrows = (cb.w - 1) / kTile - cb.z / kTile + 1;
      }
      if (tid == 0) s_o0 = o;
    }
    // exclusive prefix of the row counts (owners past the window count 0 rows)
    int x = nrows;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = (uint32_t)x;
    __syncthreads();
    int wbase = 0, total_rows = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      wbase += w < warp ? (int)s_wsum[w] : 0;
      total_rows += (int)s_wsum[w];
    }
    s_rpre[tid] = wbase + x - nrows;
    if (tid == 0) s_rpre[kEmitOwners] = total_rows;
    const uint32_t o0 = s_o0;
    __syncthreads();
    if (o0 >= k1) break;  // uniform: this batch starts past the window
    uint32_t carry = 0;   // pairs of the rows of earlier chunks
    for (int c0 = 0; c0 < total_rows && o0 + carry < k1; c0 += 8 * 256) {
      const int j0 = c0 + 8 * tid;
      int own = 0;
      uint32_t w[8];
      int t0[8], ty[8];
      if (j0 < total_rows) {  // owner of row j0: last owner whose first row is <= j0
        int lo = 0, hi = kEmitOwners - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_rpre[mid] <= j0) lo = mid; else hi = mid - 1;
        }
        own = lo;
      }
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = j0 + q;
        w[q] = 0;
        t0[q] = 0;
        ty[q] = 0;
        if (j < total_rows) {
          while (s_rpre[own + 1] <= j) ++own;  // skips owners with no rows
          const int4 d = s_cb[own];
          const int4 cb = cullbox_of(d);
          ty[q] = cb.z / kTile + (j - s_rpre[own]);
          int a, b;
          if (row_span(s_g[own], cb, cullbox_ell(d), ty[q], a, b)) {
            w[q] = (uint32_t)(b - a + 1);
            t0[q] = a;
          }
          t0[q] |= own << 16;
        }
        sum += w[q];
      }
      // block exclusive scan of the per-thread sums
      uint32_t xs = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
        if (lane >= o) xs += y;
      }
      __syncthreads();  // s_wsum reuse
      if (lane == 31) s_wsum[warp] = xs;
      __syncthreads();
      uint32_t base = 0, ctot = 0;
#pragma unroll
      for (int w8 = 0; w8 < 8; ++w8) {
        base += w8 < warp ? s_wsum[w8] : 0u;
        ctot += s_wsum[w8];
      }
      uint32_t pos = o0 + carry + base + xs - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t s0 = pos, s1 = pos + w[q];
        if (w[q] && s1 > k0 && s0 < k1) {
          const uint32_t first = max(s0, k0);
          const int ls = (int)(first - k0);
          const int ow = t0[q] >> 16;
          s_seg_tile[ls] = (uint16_t)(ty[q] * TW + (t0[q] & 0xffff) + (int)(first - s0));
          s_seg_item[ls] = s_oitem[ow];
          s_start[ls] = ls;
        }
        pos = s1;
      }
      carry += ctot;
    }
  }
  __syncthreads();
  // segment of every pair slot without a search: a block-wide running max carries the
  // last start mark forward (slot 0 always holds one: the segment containing pair k0)
  const uint32_t q0 = 8 * tid;  // this thread's 8 consecutive pair slots
  int own[8];
  {  // two 128-bit shared loads per thread (no bank conflicts at an 8-word stride)
    const int4 m0 = reinterpret_cast<const int4*>(s_start)[2 * tid];
    const int4 m1 = reinterpret_cast<const int4*>(s_start)[2 * tid + 1];
    own[0] = m0.x; own[1] = m0.y; own[2] = m0.z; own[3] = m0.w;
    own[4] = m1.x; own[5] = m1.y; own[6] = m1.z; own[7] = m1.w;
  }
  int run = -1;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    run = max(run, own[q]);
    own[q] = run;
  }
  // exclusive max-scan of the per-thread last mark across the block
  int x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) x = max(x, __shfl_up_sync(0xffffffffu, x, o));
  if (lane == 31) s_wmax[warp] = x;
  __syncthreads();
  int carry = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) carry = -1;
  for (int w = 0; w < warp; ++w) carry = max(carry, s_wmax[w]);
  uint32_t tl[8], itm[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t k = k0 + q0 + q;
    tl[q] = 0;
    itm[q] = 0;
    if (k < k1) {
      const int j = max(own[q], carry);
      tl[q] = (uint32_t)s_seg_tile[j] + (q0 + q - (uint32_t)j);
      itm[q] = s_seg_item[j];
    }
  }
  __syncthreads();  // all marks read before the aliased item slots are written
  reinterpret_cast<uint4*>(s_tile_out)[tid] =
      make_uint4(tl[0] | (tl[1] << 16), tl[2] | (tl[3] << 16), tl[4] | (tl[5] << 16), tl[6] | (tl[7] << 16));
  reinterpret_cast<uint4*>(s_item_out)[2 * tid] = make_uint4(itm[0], itm[1], itm[2], itm[3]);
  reinterpret_cast<uint4*>(s_item_out)[2 * tid + 1] = make_uint4(itm[4], itm[5], itm[6], itm[7]);
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
