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

constexpr int kEmitPairs = 2048;  // pairs per emit CTA
constexpr int kCountThreads = 1024;  // ranks per count CTA (few CTAs: short look-back chains)

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

// Two emitters, chosen on the device per frame (both are launched; one returns at once):
// the pair-balanced emit_kernel wins when Gaussians cover many tiles (configs[1]: 33 pairs
// per visible Gaussian, configs[4]: ~300), the rank-balanced emitw_kernel when they are
// small (configs[2]: 17) -- measured on B200.
constexpr uint32_t kEmitPairBalancedMean = 24;
__device__ __forceinline__ bool emit_pair_balanced(uint32_t P, uint32_t nvis) {
  return (unsigned long long)P >= (unsigned long long)kEmitPairBalancedMean * nvis;
}

__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ items_sorted,
                                                   const Rec* __restrict__ recs, const uint4* __restrict__ rowtab,
                                                   const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ chunk_owner,
                                                   const Counters* __restrict__ ctr, int TW,
                                                   uint16_t* __restrict__ pair_tiles, uint32_t* __restrict__ pair_items,
                                                   uint32_t* __restrict__ tile_hist /* 2 x 256 */,
                                                   uint32_t* __restrict__ lookback0, uint32_t sort_chunk) {
  // A "segment" is one tile row of one Gaussian: consecutive pairs with consecutive tile ids.
  // Segment data is keyed by the CTA-local slot of its first pair inside this window.
  __shared__ __align__(16) uint16_t s_seg_tile[kEmitPairs];
  __shared__ uint32_t s_seg_item[kEmitPairs];
  // s_tile_out reuses s_seg_tile and s_item_out reuses s_start (segment start marks): a
  // barrier separates the last segment/mark read from the first output write
  uint16_t* const s_tile_out = s_seg_tile;
  __shared__ __align__(16) int s_start_item[kEmitPairs];
  int* const s_start = s_start_item;
  uint32_t* const s_item_out = reinterpret_cast<uint32_t*>(s_start_item);
  __shared__ uint32_t s_hist[2][256];
  __shared__ int s_wmax[8];
  // owner batch: row geometry, record boxes, item and the exclusive prefix of their row counts
  union __align__(16) OwnerRows {  // row table (<= kRowTab rows) or the geometry to evaluate rows from
    RowGeom g;
    uint32_t tab[kRowTab];
  };
  __shared__ OwnerRows s_g[kEmitOwners];
  __shared__ int4 s_cb[kEmitOwners];
  __shared__ uint32_t s_oitem[kEmitOwners];
  __shared__ int s_rpre[kEmitOwners + 1];
  __shared__ uint32_t s_wsum[8];
  __shared__ uint32_t s_o0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t P = ctr->n_pairs, nvis = ctr->n_visible;
  if (!emit_pair_balanced(P, nvis)) return;  // emitw_kernel emits this frame
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
    if (tid < kEmitOwners && r <= rlast) {
      const uint32_t o = offsets[r];
      if (o < k1) {
        const uint32_t it = items_sorted[r];
        const Rec* R = recs + it;
        const int4 d = __ldg(&R->d);
        const int4 cb = cullbox_of(d);
        nrows = (cb.w - 1) / kTile - cb.z / kTile + 1;
        if (cullbox_ell(d)) {  // else: full rows
          if (nrows <= kRowTab) {
            uint4* t = reinterpret_cast<uint4*>(s_g[tid].tab);
#pragma unroll
            for (int v = 0; v < kRowTab / 4; ++v) t[v] = __ldg(rowtab + (kRowTab / 4) * (size_t)it + v);
          } else {
            s_g[tid].g = row_geom(__ldg(&R->a), __ldg(&R->b));
          }
        }
        s_cb[tid] = d;
        s_oitem[tid] = it;
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
    if (tid < kEmitOwners) s_rpre[tid] = wbase + x - nrows;
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
          const int k = j - s_rpre[own];
          ty[q] = cb.z / kTile + k;
          int a = cb.x / kTile, b = (cb.y - 1) / kTile;  // rectangle row
          bool ok = true;
          if (cullbox_ell(d)) {
            if ((cb.w - 1) / kTile - cb.z / kTile < kRowTab) {  // tabulated by the projection
              const uint32_t e = s_g[own].tab[k];
              a = (int)(e & 0xffffu);
              b = a + (int)(e >> 16) - 1;
              ok = e != 0u;
            } else {
              ok = row_span(s_g[own].g, cb, ty[q], a, b);
            }
          }
          if (ok) {
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

// Rank-balanced emitter: one warp per 32 consecutive depth ranks. The warp walks the
// contiguous pair range of its ranks 32 pairs at a time (coalesced stores): each lane finds
// its pair's rank (binary search over the ranks' offsets, shuffles) and tile row (binary
// search over the rank's row-table prefix in shared memory; rectangle rows by division).
// Ranks with more than kRowTab ellipse rows are emitted afterwards, one at a time by the
// whole warp: rows evaluated 32 at a time (row_span), a warp scan, then their pairs. Warps are
// independent (no block barriers in the main loop), so the imbalance between near (large)
// and far (small) Gaussians is absorbed by the other warps of the SM.
constexpr int kEmitWarps = 8;

__global__ void __launch_bounds__(32 * kEmitWarps) emitw_kernel(
    const uint32_t* __restrict__ items_sorted, const Rec* __restrict__ recs, const uint4* __restrict__ rowtab,
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ tcount, Counters* __restrict__ ctr,
    int TW, uint16_t* __restrict__ pair_tiles, uint32_t* __restrict__ pair_items,
    uint32_t* __restrict__ tile_hist /* 2 x 256 */, uint32_t* __restrict__ lookback0, uint32_t sort_chunk) {
  __shared__ uint32_t s_hist[2][256];
  __shared__ uint16_t s_tx[kEmitWarps][32][kRowTab];   // first tile column of each tabulated row
  __shared__ uint16_t s_pre[kEmitWarps][32][kRowTab];  // exclusive prefix of the row widths
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t P = ctr->n_pairs, nvis = ctr->n_visible;
  if (emit_pair_balanced(P, nvis)) return;  // emit_kernel emits this frame
  const uint32_t lb_words = (P + sort_chunk - 1) / sort_chunk * 256u;
  for (uint32_t k = blockIdx.x * blockDim.x + tid; k < lb_words; k += gridDim.x * blockDim.x) lookback0[k] = 0;
  for (int i = tid; i < 512; i += 32 * kEmitWarps) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  // persistent warps: chunks of 32 ranks from a work counter, so the SM slots of a finished
  // warp are refilled at once (no block barrier waits on the slowest warp until the end)
  for (;;) {
    uint32_t chunk = 0;
    if (lane == 0) chunk = atomicAdd(&ctr->emit_work, 1u);
    const uint32_t r0 = __shfl_sync(0xffffffffu, chunk, 0) * 32u;
    if (r0 >= nvis) break;
    const uint32_t r = r0 + lane;
    const bool has = r < nvis;
    uint32_t o = 0, cnt = 0, it = 0;
    int kind = 0, ty0 = 0, tx0 = 0, tw = 1, nrows = 0;  // kind 0 rectangle, 1 table, 2 evaluated rows
    int4 cb = make_int4(0, 0, 0, 0);
    if (has) {
      o = offsets[r];
      it = items_sorted[r];
      cnt = tcount[it];
      const int4 d = __ldg(&recs[it].d);
      cb = cullbox_of(d);
      ty0 = cb.z / kTile;
      nrows = (cb.w - 1) / kTile - ty0 + 1;
      tx0 = cb.x / kTile;
      tw = (cb.y - 1) / kTile - tx0 + 1;
      if (cullbox_ell(d)) {
        if (nrows <= kRowTab) {
          kind = 1;
          uint32_t acc = 0;
#pragma unroll
          for (int v = 0; v < kRowTab / 4; ++v) {
            const uint4 q = __ldg(rowtab + (kRowTab / 4) * (size_t)it + v);
            const uint32_t t[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int k = 4 * v + u;
              s_tx[warp][lane][k] = (uint16_t)(t[u] & 0xffffu);
              s_pre[warp][lane][k] = (uint16_t)acc;
              acc += k < nrows ? t[u] >> 16 : 0u;
            }
          }
        } else {
          kind = 2;
        }
      }
    }
    __syncwarp();
    const uint32_t o_first = __shfl_sync(0xffffffffu, o, 0);
    const uint32_t rel = o - o_first;
    const int last = min(31, (int)(nvis - 1 - r0));
    const uint32_t T = __shfl_sync(0xffffffffu, rel + cnt, last);  // pairs of the warp's ranks
    for (uint32_t p0 = 0; p0 < T; p0 += 32) {
      const uint32_t p = p0 + lane;
      // owner lane: the last one whose first pair is <= p (ranks without pairs share the
      // next rank's offset, so the last such lane owns pairs)
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, rel, lo + step);
        if (lo + step <= last && v <= p) lo += step;
      }
      const int okind = __shfl_sync(0xffffffffu, kind, lo);
      const uint32_t L = p - __shfl_sync(0xffffffffu, rel, lo);
      const uint32_t oitem = __shfl_sync(0xffffffffu, it, lo);
      const int oty0 = __shfl_sync(0xffffffffu, ty0, lo);
      const int otx0 = __shfl_sync(0xffffffffu, tx0, lo);
      const int otw = __shfl_sync(0xffffffffu, tw, lo);
      const uint32_t k = o_first + p;
      const bool ok = p < T && okind != 2 && k < P;
      uint32_t tile = 0;
      if (ok) {
        if (okind == 1) {
          int rk = 0;
#pragma unroll
          for (int step = kRowTab / 2; step > 0; step >>= 1)
            if (s_pre[warp][lo][rk + step] <= L) rk += step;
          tile = (uint32_t)((oty0 + rk) * TW + s_tx[warp][lo][rk]) + (L - s_pre[warp][lo][rk]);
        } else {
          const uint32_t row = L / (uint32_t)otw;
          tile = (uint32_t)((oty0 + (int)row) * TW + otx0) + (L - row * (uint32_t)otw);
        }
        pair_tiles[k] = (uint16_t)tile;
        pair_items[k] = oitem;
        atomicAdd(&s_hist[0][tile & 255u], 1u);
      }
      // high digit: consecutive pairs mostly share it -> one shared atomic per run
      const uint32_t hi8 = ok ? tile >> 8 : 0xffffffffu;
      const uint32_t prev = __shfl_up_sync(0xffffffffu, hi8, 1);
      const uint32_t next = __shfl_down_sync(0xffffffffu, hi8, 1);
      const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || prev != hi8);
      if (ok && (lane == 31 || next != hi8)) {
        const int run_start = 31 - __clz(starts & ((2u << lane) - 1u));
        atomicAdd(&s_hist[1][hi8], (uint32_t)(lane - run_start + 1));
      }
    }
    // ranks whose ellipse rows were not tabulated: one at a time, the whole warp
    unsigned big = __ballot_sync(0xffffffffu, kind == 2);
    while (big) {
      const int b = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t bitem = __shfl_sync(0xffffffffu, it, b);
      const int4 bcb = make_int4(__shfl_sync(0xffffffffu, cb.x, b), __shfl_sync(0xffffffffu, cb.y, b),
                                 __shfl_sync(0xffffffffu, cb.z, b), __shfl_sync(0xffffffffu, cb.w, b));
      const int bty0 = __shfl_sync(0xffffffffu, ty0, b), bn = __shfl_sync(0xffffffffu, nrows, b);
      uint32_t pos = __shfl_sync(0xffffffffu, o, b);
      const RowGeom g = row_geom(__ldg(&recs[bitem].a), __ldg(&recs[bitem].b));
      for (int rc = 0; rc < bn; rc += 32) {
        const int rowk = rc + lane;
        int a0 = 0, a1 = -1;
        const uint32_t w = rowk < bn && row_span(g, bcb, bty0 + rowk, a0, a1) ? (uint32_t)(a1 - a0 + 1) : 0u;
        uint32_t incl = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        const uint32_t excl = incl - w;
        const uint32_t ct = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t q0 = 0; q0 < ct; q0 += 32) {
          const uint32_t q = q0 + lane;
          int lo = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, excl, lo + step);
            if (v <= q) lo += step;
          }
          const uint32_t rx = q - __shfl_sync(0xffffffffu, excl, lo);
          const int ra0 = __shfl_sync(0xffffffffu, a0, lo);
          const uint32_t k = pos + q;
          const bool ok = q < ct && k < P;
          uint32_t tile = 0;
          if (ok) {
            tile = (uint32_t)((bty0 + rc + lo) * TW + ra0) + rx;
            pair_tiles[k] = (uint16_t)tile;
            pair_items[k] = bitem;
            atomicAdd(&s_hist[0][tile & 255u], 1u);
          }
          const uint32_t hi8 = ok ? tile >> 8 : 0xffffffffu;
          const uint32_t prev = __shfl_up_sync(0xffffffffu, hi8, 1);
          const uint32_t next = __shfl_down_sync(0xffffffffu, hi8, 1);
          const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || prev != hi8);
          if (ok && (lane == 31 || next != hi8)) {
            const int run_start = 31 - __clz(starts & ((2u << lane) - 1u));
            atomicAdd(&s_hist[1][hi8], (uint32_t)(lane - run_start + 1));
          }
        }
        pos += ct;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < 512; i += 32 * kEmitWarps) {
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
