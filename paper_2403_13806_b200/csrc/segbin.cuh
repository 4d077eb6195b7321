// segbin.cuh -- tile binning through row segments.
//
// The per-tile lists are the reference's global (depth, index) order
// (render.py:218-222) restricted to each tile, over the tiles a Gaussian is
// binned to (rows.cuh: per tile row of its culling box, a contiguous span of
// tile columns). Instead of emitting one (tile, Gaussian) pair per overlap and
// sorting all pairs by tile, the binning works on ROW SEGMENTS -- one per
// (Gaussian, tile row), ~5x fewer than pairs:
//
//   segcount_kernel  per depth rank: its segment count (tile rows of its
//                    culling box), block scan + decoupled look-back ->
//                    exclusive segment offset per rank; S.
//   segemit_kernel   one warp per 32 ranks, rows flattened over the lanes:
//                    each segment's span (row_span), written in depth-rank
//                    order as (row key, item, span); per-row segment counts
//                    (= the sort's digit histogram).
//   onesweep (1 pass over the row key, sort.cuh) -> every row's segments in
//                    depth order (stable).
//   row_scan_kernel  per-row segment starts; rows cut into chunks of 1024.
//   chunk_count_kernel  one CTA per chunk: per tile column the number of the
//                    chunk's segments covering it (shared-memory counters).
//   tile_chunks_kernel / tile_scan_kernel  per tile: prefix over its row's
//                    chunks and its total; exclusive scan over the tiles ->
//                    ranges [start, end), P, overflow.
//   expand_kernel<true>  the same walk again, appending each covering
//                    segment's item to the column's tile list at its rank.
// The pair lists and ranges are the same as a stable sort of all pairs by
// tile would produce (the parity tests compare them with the oracle).
#pragma once
#include "rows.cuh"
#include "rs_common.cuh"

namespace rs {

constexpr int kSegCountThreads = 1024;
constexpr uint32_t kEmptySpan = 0x00000001u;  // t0 = 1 > t1 = 0: the row lists no tile
constexpr int kExpandCols = 32;                // tile columns per expand CTA (8 warps x 4)
constexpr int kMaxTileRows = 2048;             // image height <= 32767 px
constexpr int kMaxTileCols = 2048;             // image width <= 32767 px

constexpr int kSegCountItems = 4;  // ranks per thread (fewer, longer CTAs: a short look-back chain)

__global__ void __launch_bounds__(kSegCountThreads) segcount_kernel(const uint32_t* __restrict__ items_sorted,
                                                                    const uint32_t* __restrict__ nrows,
                                                                    Counters* __restrict__ ctr, uint32_t seg_cap,
                                                                    uint32_t* __restrict__ offsets,
                                                                    unsigned long long* __restrict__ status,
                                                                    Sticky* __restrict__ sticky) {
  constexpr uint32_t kPer = kSegCountThreads * kSegCountItems;
  __shared__ uint32_t s_block;
  __shared__ uint32_t s_wsum[kSegCountThreads / 32];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_block = atomicAdd(&ctr->emit_ctr, 1u);
  __syncthreads();
  const uint32_t b = s_block;
  const uint32_t nvis = ctr->n_visible;
  if (b * kPer >= nvis && b > 0) return;
  // this thread's kSegCountItems consecutive ranks
  const uint32_t r0 = b * kPer + tid * kSegCountItems;
  uint32_t nt[kSegCountItems], tsum = 0;
#pragma unroll
  for (int q = 0; q < kSegCountItems; ++q) {
    nt[q] = r0 + q < nvis ? nrows[items_sorted[r0 + q]] : 0u;
    tsum += nt[q];
  }
  uint32_t x = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t off = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kSegCountThreads / 32; ++w) {
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
      if (nvis > 0 && b == (nvis - 1) / kPer) {
        const unsigned long long end = excl + total;
        ctr->n_segs = (uint32_t)(end < seg_cap ? end : seg_cap);
        if (end > seg_cap) {  // too many segments: the frame is re-run with a larger workspace
          ctr->overflow = 1u;
          atomicOr(&sticky->overflowed, 1u);
          // pair capacity that certainly holds this frame's segments (segments <= pairs + 2 n)
          const unsigned long long need = end;
          if (need > ctr->pairs_needed) ctr->pairs_needed = need;
          atomicMax(&sticky->pairs_needed_max, need);
        }
      }
    }
  }
  __syncthreads();
  uint32_t o = (uint32_t)s_base + off + x - tsum;
#pragma unroll
  for (int q = 0; q < kSegCountItems; ++q) {
    if (r0 + q < nvis) offsets[r0 + q] = o;
    o += nt[q];
  }
}

// One warp per 32 consecutive ranks (persistent warps take rank chunks from a counter).
__global__ void __launch_bounds__(256) segemit_kernel(const uint32_t* __restrict__ items_sorted,
                                                      const Rec* __restrict__ recs,
                                                      const uint32_t* __restrict__ offsets,
                                                      Counters* __restrict__ ctr, int TW,
                                                      uint16_t* __restrict__ seg_key, uint32_t* __restrict__ seg_item,
                                                      uint32_t* __restrict__ seg_span,
                                                      int TH, uint32_t* __restrict__ row_count,
                                                      uint32_t* __restrict__ key_hist /* 2 x 256 */,
                                                      uint32_t* __restrict__ lookback0, uint32_t sort_chunk) {
  __shared__ RowGeom s_g[8][32];
  __shared__ int4 s_cb[8][32];
  __shared__ int s_pre[8][33];
  __shared__ int s_rows[kMaxTileRows + 1];  // per-row difference array of this CTA's segments
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nvis = ctr->n_visible;
  const uint32_t S = ctr->n_segs;
  const bool over = ctr->overflow != 0u;
  const uint32_t lb_words = (S + sort_chunk - 1) / sort_chunk * 256u;
  for (uint32_t k = blockIdx.x * blockDim.x + tid; k < lb_words; k += gridDim.x * blockDim.x) lookback0[k] = 0;
  for (int i = tid; i <= TH; i += 256) s_rows[i] = 0;
  __syncthreads();
  if (!over) {
    for (;;) {
      uint32_t chunk = 0;
      if (lane == 0) chunk = atomicAdd(&ctr->emit_work, 1u);
      const uint32_t r0 = __shfl_sync(0xffffffffu, chunk, 0) * 32u;
      if (r0 >= nvis) break;
      const uint32_t r = r0 + lane;
      int nr = 0;
      uint32_t o = 0, it = 0;
      if (r < nvis) {
        o = offsets[r];
        it = items_sorted[r];
        const Rec* R = recs + it;
        const int4 d = __ldg(&R->d);
        const int4 cb = cullbox_of(d);
        nr = (cb.w - 1) / kTile - cb.z / kTile + 1;
        s_cb[warp][lane] = make_int4(cb.x, cb.y, cb.z, cb.w | (cullbox_ell(d) ? (int)0x80000000 : 0));
        if (cullbox_ell(d)) s_g[warp][lane] = row_geom(__ldg(&R->a), __ldg(&R->b));
        atomicAdd(&s_rows[cb.z / kTile], 1);  // one segment in each of its rows
        atomicAdd(&s_rows[cb.z / kTile + nr], -1);
      }
      int x = nr;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      s_pre[warp][lane] = x - nr;
      if (lane == 31) s_pre[warp][32] = x;
      __syncwarp();
      const int total = s_pre[warp][32];
      for (int base = 0; base < total; base += 32) {
        const int j = base + lane;
        int lo = 0;
        if (j < total) {
          int hi = 31;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pre[warp][mid] <= j) lo = mid; else hi = mid - 1;
          }
        }
        const uint32_t so = __shfl_sync(0xffffffffu, o, lo);
        const uint32_t sitem = __shfl_sync(0xffffffffu, it, lo);
        if (j < total) {
          const int k = j - s_pre[warp][lo];
          const int4 c4 = s_cb[warp][lo];
          const bool ell = c4.w < 0;
          const int4 cb = make_int4(c4.x, c4.y, c4.z, c4.w & 0x7fffffff);
          const int ty = cb.z / kTile + k;
          int t0 = cb.x / kTile, t1 = (cb.y - 1) / kTile;
          const bool ok = ell ? row_span(s_g[warp][lo], cb, ty, t0, t1) : true;
          const uint32_t s = so + (uint32_t)k;
          seg_key[s] = (uint16_t)ty;
          seg_item[s] = sitem;
          seg_span[s] = ok ? ((uint32_t)t0 | ((uint32_t)t1 << 16)) : kEmptySpan;

        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (tid == 0) {  // difference array -> per-row segment counts (TH <= 2048, one pass)
    int run = 0;
    for (int i = 0; i < TH; ++i) {
      run += s_rows[i];
      s_rows[i] = run;
    }
  }
  __syncthreads();
  for (int i = tid; i < TH; i += 256) {
    const uint32_t v = (uint32_t)s_rows[i];
    if (v) {
      atomicAdd(&row_count[i], v);
      atomicAdd(&key_hist[i & 255], v);
      if (TH > 256) atomicAdd(&key_hist[256 + (i >> 8)], v);
    }
  }
}

// One CTA: per-row segment starts and chunk starts (chunks of kExpandChunk segments).
constexpr int kExpandChunk = 1024;
__global__ void __launch_bounds__(256) row_scan_kernel(const uint32_t* __restrict__ row_count, int TH,
                                                       uint32_t* __restrict__ row_start,
                                                       uint32_t* __restrict__ chunk_start) {
  if (threadIdx.x != 0) return;
  uint32_t acc = 0, ch = 0;
  for (int ty = 0; ty < TH; ++ty) {
    row_start[ty] = acc;
    chunk_start[ty] = ch;
    acc += row_count[ty];
    ch += (row_count[ty] + kExpandChunk - 1) / kExpandChunk;
  }
  row_start[TH] = acc;
  chunk_start[TH] = ch;
}

// (chunk, 32 columns) of a row: which row / which of its chunks (binary search over chunk starts)
__device__ __forceinline__ bool chunk_of(const uint32_t* __restrict__ chunk_start, int TH, uint32_t gc, int& ty,
                                         uint32_t& lc) {
  if (gc >= chunk_start[TH]) return false;
  int lo = 0, hi = TH - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (chunk_start[mid] <= gc) lo = mid; else hi = mid - 1;
  }
  ty = lo;
  lc = gc - chunk_start[lo];
  return true;
}

// Pass 2: the chunk's covering segments appended to each column's tile list after all
// earlier chunks of the row (ranges + chunk prefix): warp w owns 4 columns, 32 segments per
// ballot (their order = depth order), segments staged 256 at a time. (WRITE = false: the
// same walk only counting -- kept for reference; chunk_count_kernel is the pass 1 used.)
template <bool WRITE>
__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ sorted_seg,
                                                     const uint32_t* __restrict__ seg_item,
                                                     const uint32_t* __restrict__ seg_span,
                                                     const uint32_t* __restrict__ row_start,
                                                     const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                     uint32_t* __restrict__ chunk_count /* [chunk][TW] */,
                                                     const uint2* __restrict__ ranges,
                                                     const Counters* __restrict__ ctr,
                                                     uint32_t* __restrict__ pair_items) {
  __shared__ uint32_t s_item[256], s_span[256];
  __shared__ int s_wk[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (WRITE && ctr->overflow) return;
  const int c0 = blockIdx.y * kExpandCols + warp * 4;  // this warp's 4 tile columns
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t gc = blockIdx.x;; gc += gridDim.x) {  // chunks of all rows, grid-strided
    int ty;
    uint32_t lc;
    if (!chunk_of(chunk_start, TH, gc, ty, lc)) break;
    const uint32_t s0 = row_start[ty] + lc * kExpandChunk, s1 = min(row_start[ty + 1], s0 + kExpandChunk);
    uint32_t pos[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      pos[q] = 0;
      if (WRITE && c0 + q < TW) pos[q] = ranges[ty * TW + c0 + q].x + chunk_count[(size_t)gc * TW + c0 + q];
    }
    const int g0 = blockIdx.y * kExpandCols, g1 = g0 + kExpandCols - 1;  // this CTA's columns
    for (uint32_t base = s0; base < s1; base += 256) {
      const uint32_t nb = min(256u, s1 - base);
      __syncthreads();
      // stage only the segments that reach this CTA's 32 columns, in order (block compaction):
      // the warps then walk ~45% of the chunk instead of all of it
      uint32_t sp = kEmptySpan, sit = 0;
      if (tid < nb) {
        const uint32_t sid = sorted_seg[base + tid];
        sp = seg_span[sid];
        if (WRITE) sit = seg_item[sid];
      }
      const int a0 = (int)(sp & 0xffffu), a1 = (int)(sp >> 16);
      const bool keep = a0 <= a1 && a0 <= g1 && a1 >= g0;
      const unsigned kb = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s_wk[warp] = __popc(kb);
      __syncthreads();
      int koff = 0, n2 = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        koff += w < warp ? s_wk[w] : 0;
        n2 += s_wk[w];
      }
      if (keep) {
        const int at = koff + __popc(kb & lt);
        s_span[at] = sp;
        if (WRITE) s_item[at] = sit;
      }
      __syncthreads();
      const uint32_t n = (uint32_t)n2;
      if (c0 >= TW) continue;
      for (uint32_t sub = 0; sub < n; sub += 32) {
        const uint32_t e = sub + lane;
        const uint32_t sp = e < n ? s_span[e] : kEmptySpan;
        const int t0 = (int)(sp & 0xffffu), t1 = (int)(sp >> 16);
        const bool near = t0 <= t1 && t0 <= c0 + 3 && t1 >= c0;
        if (!__any_sync(0xffffffffu, near)) continue;
        const uint32_t item = (WRITE && near) ? s_item[e] : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q;
          const bool cov = near && t0 <= c && c <= t1;
          const unsigned bal = __ballot_sync(0xffffffffu, cov);
          if (WRITE && cov) pair_items[pos[q] + __popc(bal & lt)] = item;
          pos[q] += __popc(bal);
        }
      }
    }
    if (!WRITE && lane == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + q < TW) chunk_count[(size_t)gc * TW + c0 + q] = pos[q];
    }
  }
}

// Pass 1 (order-free): per (chunk, tile column) the number of the chunk's segments covering
// the column -- shared-memory counters over all the row's columns, one CTA per chunk.
__global__ void __launch_bounds__(256) chunk_count_kernel(const uint32_t* __restrict__ sorted_seg,
                                                          const uint32_t* __restrict__ seg_span,
                                                          const uint32_t* __restrict__ row_start,
                                                          const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                          uint32_t* __restrict__ chunk_count) {
  __shared__ uint32_t s_cnt[kMaxTileCols];
  const int tid = threadIdx.x;
  for (uint32_t gc = blockIdx.x;; gc += gridDim.x) {
    int ty;
    uint32_t lc;
    if (!chunk_of(chunk_start, TH, gc, ty, lc)) break;
    __syncthreads();
    for (int c = tid; c < TW; c += 256) s_cnt[c] = 0;
    __syncthreads();
    const uint32_t s0 = row_start[ty] + lc * kExpandChunk, s1 = min(row_start[ty + 1], s0 + kExpandChunk);
    for (uint32_t sidx = s0 + tid; sidx < s1; sidx += 256) {
      const uint32_t sp = seg_span[sorted_seg[sidx]];
      const int t0 = (int)(sp & 0xffffu), t1 = (int)(sp >> 16);
      for (int c = t0; c <= t1; ++c) atomicAdd(&s_cnt[c], 1u);
    }
    __syncthreads();
    for (int c = tid; c < TW; c += 256) chunk_count[(size_t)gc * TW + c] = s_cnt[c];
  }
}

// Per tile: its chunks' counts -> exclusive prefix over the row's chunks (in place) and the
// tile's total (one warp per tile, 32 chunks per scan step).
__global__ void __launch_bounds__(256) tile_chunks_kernel(const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                          uint32_t* __restrict__ chunk_count,
                                                          uint32_t* __restrict__ tile_count) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= TW * TH) return;
  const int ty = t / TW, tx = t - ty * TW;
  const uint32_t c0 = chunk_start[ty], c1 = chunk_start[ty + 1];
  uint32_t carry = 0;
  for (uint32_t cb = c0; cb < c1; cb += 32) {
    const uint32_t c = cb + lane;
    const uint32_t v = c < c1 ? chunk_count[(size_t)c * TW + tx] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (c < c1) chunk_count[(size_t)c * TW + tx] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) tile_count[t] = carry;
}

// One CTA: exclusive scan of the tile counts (row-major tile ids) -> ranges (empty tiles
// [0, 0)), P and the overflow verdict.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ tile_count, int T,
                                                         Counters* __restrict__ ctr, uint32_t pair_cap,
                                                         uint2* __restrict__ ranges, Sticky* __restrict__ sticky) {
  __shared__ unsigned long long s_wsum[32];
  __shared__ unsigned long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int t0 = 0; t0 < T; t0 += 1024) {
    const int t = t0 + tid;
    const unsigned long long v = t < T ? (unsigned long long)tile_count[t] : 0ull;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    unsigned long long off = s_carry;
    for (int w = 0; w < warp; ++w) off += s_wsum[w];
    const unsigned long long st = off + x - v;
    if (t < T)
      ranges[t] = v ? make_uint2((uint32_t)min(st, (unsigned long long)pair_cap),
                                 (uint32_t)min(st + v, (unsigned long long)pair_cap))
                    : make_uint2(0u, 0u);
    __syncthreads();
    if (tid == 1023) s_carry = off + x;
    __syncthreads();
  }
  if (tid == 0) {
    const unsigned long long P = s_carry;
    ctr->n_pairs = (uint32_t)(P < pair_cap ? P : pair_cap);
    if (P > ctr->pairs_needed) ctr->pairs_needed = P;
    if (P > pair_cap) {
      ctr->overflow = 1u;
      atomicOr(&sticky->overflowed, 1u);
      atomicMax(&sticky->pairs_needed_max, P);
    }
  }
}

}  // namespace rs
