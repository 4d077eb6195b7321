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
//                    (= the sort's digit histogram). The last CTA scans the
//                    counts: per-row segment starts, rows cut into chunks of
//                    1024.
//   onesweep (1 pass over the row key, sort.cuh) -> every row's segments in
//                    depth order (stable).
//   chunk_count_kernel  one CTA per chunk: per tile column the number of the
//                    chunk's segments covering it (shared-memory counters);
//                    the chunk's {first segment, row, count, dense} record and
//                    the list of dense chunks (>= 8 tiles per segment).
//   tile_chunks_kernel / tile_scan_kernel  per tile: prefix over its row's
//                    chunks and its total; exclusive scan over the tiles ->
//                    ranges [start, end), P, overflow.
//   expand_kernel    sparse chunks x 32-column groups: per warp 32 segments'
//                    column masks, transposed (lane = column), each column's
//                    covering items appended at its rank.
//   expand_dense_kernel  dense chunks (second stream, concurrently): warp =
//                    4 columns, one ballot per column per 32 segments.
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

constexpr int kExpandChunk = 1024;  // segments per expansion chunk (rows cut into chunks)

// Per-row segment starts and chunk starts (chunks of kExpandChunk segments) of TH <= 2048 rows:
// a 256-thread block scan, 8 rows per thread (row counts read from L2).
__device__ __forceinline__ void row_scan_block(const uint32_t* row_count, int TH, uint32_t* s_rs, uint32_t* s_cs,
                                               uint32_t* s_w /* 16, shared */) {
  constexpr int kPer = (kMaxTileRows + 255) / 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t rc[kPer], rs = 0, cs = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int ty = tid * kPer + q;
    rc[q] = ty < TH ? __ldcg(row_count + ty) : 0u;
    rs += rc[q];
    cs += (rc[q] + kExpandChunk - 1) / kExpandChunk;
  }
  uint32_t xr = rs, xc = cs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yr = __shfl_up_sync(0xffffffffu, xr, o), yc = __shfl_up_sync(0xffffffffu, xc, o);
    if (lane >= o) {
      xr += yr;
      xc += yc;
    }
  }
  if (lane == 31) {
    s_w[warp] = xr;
    s_w[8 + warp] = xc;
  }
  __syncthreads();
  uint32_t r = xr - rs, ch = xc - cs;
#pragma unroll
  for (int w = 0; w < 8; ++w)
    if (w < warp) {
      r += s_w[w];
      ch += s_w[8 + w];
    }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int ty = tid * kPer + q;
    if (ty <= TH) {
      s_rs[ty] = r;
      s_cs[ty] = ch;
    }
    r += rc[q];
    ch += (rc[q] + kExpandChunk - 1) / kExpandChunk;
  }
  if (tid == 255) {  // the totals (TH = 2048 has no thread for index TH above)
    s_rs[TH] = r;
    s_cs[TH] = ch;
  }
  __syncthreads();
}

// One warp per 32 consecutive ranks (persistent warps take rank chunks from a counter).
__global__ void __launch_bounds__(256) segemit_kernel(const uint32_t* __restrict__ items_sorted,
                                                      const Rec* __restrict__ recs,
                                                      const uint32_t* __restrict__ offsets,
                                                      Counters* __restrict__ ctr, int TW,
                                                      uint16_t* __restrict__ seg_key, uint32_t* __restrict__ seg_item,
                                                      uint32_t* __restrict__ seg_span, float4* __restrict__ geom,
                                                      int TH, uint32_t* __restrict__ row_count,
                                                      uint32_t* __restrict__ key_hist /* 2 x 256 */,
                                                      uint32_t* __restrict__ lookback0, uint32_t sort_chunk,
                                                      uint32_t* __restrict__ row_start,
                                                      uint32_t* __restrict__ chunk_start) {
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
        if (cullbox_ell(d)) {
          s_g[warp][lane] = row_geom(__ldg(&R->a), __ldg(&R->b));
          store_row_geom(geom + 2 * (size_t)it, s_g[warp][lane]);  // blend2_kernel's quarter masks
        }
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
  // the last CTA to finish: row segment starts and chunk starts for the expansion passes
  __shared__ uint32_t s_last, s_w[16];
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&ctr->emit_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    row_scan_block(row_count, TH, row_start, chunk_start, s_w);
  }
}

// (chunk, 32 columns) of a row: which row / which of its chunks (binary search over chunk starts)
__device__ __forceinline__ bool chunk_of(const uint32_t* chunk_start, int TH, uint32_t gc, int& ty, uint32_t& lc) {
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
// earlier chunks of the row (ranges + chunk prefix). A CTA owns 32 tile columns and takes the
// chunk 256 segments at a time, warp w the w-th 32 of them: each lane turns its segment's span
// into a 32-bit mask over the CTA's columns, a 32x32 bit transpose (5 shuffle stages) gives
// lane c the mask of the warp's segments covering column c, and lane c appends those items in
// segment (= depth) order after the earlier warps' counts (one shared-memory exchange).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  constexpr uint32_t kM[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t m = kM[s];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// Dense chunks (long spans: most of the CTA's columns covered by most segments): warp w owns
// 4 columns and walks all the chunk's segments that reach the CTA's columns (staged 256 at a
// time, block-compacted in order), one ballot per column per 32 segments -- every store
// instruction writes one column's run contiguously.
__device__ __forceinline__ void expand_dense_chunk(const uint32_t* __restrict__ sorted_seg,
                                                   const uint32_t* __restrict__ seg_item,
                                                   const uint32_t* __restrict__ seg_span, uint32_t s0, uint32_t cnt,
                                                   int ty, uint32_t gc, int g0, int TW,
                                                   const uint32_t* __restrict__ chunk_count,
                                                   const uint2* __restrict__ ranges,
                                                   uint32_t* __restrict__ pair_items, uint32_t* s_item,
                                                   uint32_t* s_span, int* s_wk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int c0 = g0 + warp * 4;  // this warp's 4 tile columns
  const int g1 = g0 + kExpandCols - 1;
  uint32_t pos[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) pos[q] = c0 + q < TW ? ranges[ty * TW + c0 + q].x + chunk_count[(size_t)gc * TW + c0 + q] : 0u;
  for (uint32_t base = 0; base < cnt; base += 256) {
    const uint32_t nb = min(256u, cnt - base);
    uint32_t sp = kEmptySpan, sit = 0;
    if (tid < nb) {
      const uint32_t sid = sorted_seg[s0 + base + tid];
      sp = seg_span[sid];
      sit = seg_item[sid];
    }
    const int a0 = (int)(sp & 0xffffu), a1 = (int)(sp >> 16);
    const bool keep = a0 <= a1 && a0 <= g1 && a1 >= g0;
    const unsigned kb = __ballot_sync(0xffffffffu, keep);
    __syncthreads();  // the previous batch's readers are done
    if (lane == 0) s_wk[warp] = __popc(kb);
    __syncthreads();
    int koff = 0, n = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      koff += w < warp ? s_wk[w] : 0;
      n += s_wk[w];
    }
    if (keep) {
      const int at = koff + __popc(kb & lt);
      s_span[at] = sp;
      s_item[at] = sit;
    }
    __syncthreads();
    if (c0 >= TW) continue;
    for (int sub = 0; sub < n; sub += 32) {
      const int e = sub + lane;
      const uint32_t sq = e < n ? s_span[e] : kEmptySpan;
      const int t0 = (int)(sq & 0xffffu), t1 = (int)(sq >> 16);
      const bool near = t0 <= t1 && t0 <= c0 + 3 && t1 >= c0;
      if (!__any_sync(0xffffffffu, near)) continue;
      const uint32_t item = near ? s_item[e] : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + q;
        const bool cov = near && t0 <= c && c <= t1;
        const unsigned bal = __ballot_sync(0xffffffffu, cov);
        if (cov) pair_items[pos[q] + __popc(bal & lt)] = item;
        pos[q] += __popc(bal);
      }
    }
  }
}

constexpr int kExpandSub = kExpandChunk / 256;  // 32-segment sub-steps per warp per chunk

__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ sorted_seg,
                                                     const uint32_t* __restrict__ seg_item,
                                                     const uint32_t* __restrict__ seg_span,
                                                     const uint2* __restrict__ chunk_info,
                                                     const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                     const uint32_t* __restrict__ chunk_count /* [chunk][TW] */,
                                                     const uint2* __restrict__ ranges,
                                                     const Counters* __restrict__ ctr,
                                                     uint32_t* __restrict__ pair_items, int major_thresh) {
  __shared__ uint32_t s_cnt[2][8][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ctr->overflow) return;
  const uint32_t lt = (1u << lane) - 1u;
  // column group fastest in the grid: a chunk's CTAs run together and share its segments in L2
  const int g0 = blockIdx.x * kExpandCols;  // this CTA's first tile column
  const int c = g0 + lane;                  // lane's column (every warp)
  const uint32_t n_chunks = chunk_start[TH];
  int flip = 0;
  for (uint32_t gc = blockIdx.y; gc < n_chunks; gc += gridDim.y) {  // chunks of all rows, grid-strided
    const uint2 info = chunk_info[gc];  // {first segment, row | count << 16 | dense << 31}
    if (info.y >> 31) continue;         // dense: expand_dense_kernel (concurrently, on a second stream)
    const int ty = (int)(info.y & 0xffffu);
    const uint32_t cnt = (info.y >> 16) & 0x7fffu;
    const uint32_t pos = c < TW ? ranges[ty * TW + c].x + chunk_count[(size_t)gc * TW + c] : 0u;
    // warp w: the chunk's segments [128 w, 128 w + 128), 32 per sub-step, all loads issued up front
    uint32_t sid[kExpandSub], m[kExpandSub], item[kExpandSub], cm[kExpandSub];
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const uint32_t e = (uint32_t)(warp * 32 * kExpandSub + k * 32 + lane);
      sid[k] = e < cnt ? sorted_seg[info.x + e] : 0xffffffffu;
    }
    uint32_t sp[kExpandSub];
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) sp[k] = seg_span[sid[k] != 0xffffffffu ? sid[k] : 0u];  // all in flight
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const int a = max((int)(sp[k] & 0xffffu) - g0, 0), b = min((int)(sp[k] >> 16) - g0, kExpandCols - 1);
      m[k] = sid[k] != 0xffffffffu && a <= b ? (0xffffffffu >> (31 - b)) & (0xffffffffu << a) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) item[k] = m[k] ? seg_item[sid[k]] : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      cm[k] = __any_sync(0xffffffffu, m[k] != 0u) ? transpose32(m[k], lane) : 0u;
      mine += __popc(cm[k]);
    }
    s_cnt[flip][warp][lane] = mine;
    __syncthreads();
    uint32_t p = pos;  // after the earlier warps' segments
#pragma unroll
    for (int w = 0; w < 8; ++w) p += w < warp ? s_cnt[flip][w][lane] : 0u;
    flip ^= 1;  // double-buffered counts: one barrier per chunk
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      uint32_t x = cm[k];
      const uint32_t cols = __ballot_sync(0xffffffffu, x != 0u);
      if (!cols) continue;
      const int deep = __reduce_max_sync(0xffffffffu, (unsigned)__popc(x));
      if (__popc(cols) * major_thresh <= deep * 8) {
        // few, deep columns: one column at a time, the covering lanes store contiguously
        for (uint32_t cs = cols; cs; cs &= cs - 1u) {
          const int col = __ffs(cs) - 1;
          const uint32_t xc = __shfl_sync(0xffffffffu, x, col);
          const uint32_t pc = __shfl_sync(0xffffffffu, p, col);
          if ((xc >> lane) & 1u) pair_items[pc + __popc(xc & lt)] = item[k];
        }
        p += __popc(x);
      } else {
        // many shallow columns: lane = column, appending its covering segments in order
        while (__any_sync(0xffffffffu, x != 0u)) {
          const int src = x ? __ffs(x) - 1 : 0;
          const uint32_t it = __shfl_sync(0xffffffffu, item[k], src);
          if (x) {
            pair_items[p++] = it;
            x &= x - 1u;
          }
        }
      }
    }
  }
}

// The dense chunks (listed by chunk_count_kernel, any order: chunks are independent).
__global__ void __launch_bounds__(256) expand_dense_kernel(const uint32_t* __restrict__ sorted_seg,
                                                           const uint32_t* __restrict__ seg_item,
                                                           const uint32_t* __restrict__ seg_span,
                                                           const uint2* __restrict__ chunk_info,
                                                           const uint32_t* __restrict__ dense_list, int TW,
                                                           const uint32_t* __restrict__ chunk_count,
                                                           const uint2* __restrict__ ranges,
                                                           Counters* __restrict__ ctr,
                                                           uint32_t* __restrict__ pair_items) {
  __shared__ uint32_t s_item[256], s_span[256];
  __shared__ int s_wk[8];
  __shared__ uint32_t s_tk[2];
  if (ctr->overflow) return;
  const uint32_t groups = (uint32_t)(TW + kExpandCols - 1) / kExpandCols;
  const uint32_t total = ctr->n_dense * groups;
  if (threadIdx.x == 0) s_tk[0] = atomicAdd(&ctr->dense_work, 1u);
  __syncthreads();
  int flip = 0;
  // persistent CTAs take (dense chunk, column group) tickets, the next one fetched while this one
  // runs (every chunk walk has a barrier); a chunk's column groups are consecutive tickets
  for (;;) {
    const uint32_t t = s_tk[flip];
    if (t >= total) break;
    if (threadIdx.x == 0) s_tk[flip ^ 1] = atomicAdd(&ctr->dense_work, 1u);
    const uint32_t gc = dense_list[t / groups];
    const uint2 info = chunk_info[gc];
    expand_dense_chunk(sorted_seg, seg_item, seg_span, info.x, (info.y >> 16) & 0x7fffu, (int)(info.y & 0xffffu), gc,
                       (int)(t % groups) * kExpandCols, TW, chunk_count, ranges, pair_items, s_item, s_span, s_wk);
    flip ^= 1;
  }
}

// Pass 1 (order-free): per (chunk, tile column) the number of the chunk's segments covering
// the column -- shared-memory counters over all the row's columns, one CTA per chunk.
__global__ void __launch_bounds__(256) chunk_count_kernel(const uint32_t* __restrict__ sorted_seg,
                                                          const uint32_t* __restrict__ seg_span,
                                                          const uint32_t* __restrict__ row_start,
                                                          const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                          uint32_t* __restrict__ chunk_count,
                                                          uint2* __restrict__ chunk_info, int dense_span,
                                                          Counters* __restrict__ ctr,
                                                          uint32_t* __restrict__ dense_list) {
  __shared__ uint32_t s_cnt[kMaxTileCols];
  __shared__ uint32_t s_tiles;
  const int tid = threadIdx.x;
  for (uint32_t gc = blockIdx.x;; gc += gridDim.x) {
    int ty;
    uint32_t lc;
    if (!chunk_of(chunk_start, TH, gc, ty, lc)) break;
    __syncthreads();
    for (int c = tid; c < TW; c += 256) s_cnt[c] = 0;
    if (tid == 0) s_tiles = 0;
    __syncthreads();
    const uint32_t s0 = row_start[ty] + lc * kExpandChunk, s1 = min(row_start[ty + 1], s0 + kExpandChunk);
    int tiles = 0;
    for (uint32_t sidx = s0 + tid; sidx < s1; sidx += 256) {
      const uint32_t sp = seg_span[sorted_seg[sidx]];
      const int t0 = (int)(sp & 0xffffu), t1 = (int)(sp >> 16);
      for (int c = t0; c <= t1; ++c) atomicAdd(&s_cnt[c], 1u);
      tiles += max(t1 - t0 + 1, 0);
    }
    tiles = __reduce_add_sync(0xffffffffu, tiles);
    if ((tid & 31) == 0) atomicAdd(&s_tiles, (uint32_t)tiles);
    __syncthreads();
    // dense: the segments average >= dense_span tiles (expand_kernel's ballot walk)
    if (tid == 0) {
      const bool dense = s_tiles >= (uint32_t)dense_span * (s1 - s0);
      chunk_info[gc] = make_uint2(s0, (uint32_t)ty | ((s1 - s0) << 16) | (dense ? 0x80000000u : 0u));
      if (dense) dense_list[atomicAdd(&ctr->n_dense, 1u)] = gc;
    }
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
// [0, 0)), P and the overflow verdict. Thread t owns ceil(T / 1024) consecutive tiles.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ tile_count, int T,
                                                         Counters* __restrict__ ctr, uint32_t pair_cap,
                                                         uint2* __restrict__ ranges, Sticky* __restrict__ sticky) {
  __shared__ unsigned long long s_w[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (T + 1023) / 1024;
  const int t0 = min(tid * per, T), t1 = min(t0 + per, T);
  unsigned long long sum = 0;
  for (int t = t0; t < t1; ++t) sum += tile_count[t];
  unsigned long long x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long v = s_w[lane];
    unsigned long long z = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    s_w[lane] = z - v;  // exclusive warp offsets
    if (lane == 31) {   // P and the overflow verdict
      const unsigned long long P = z;
      ctr->n_pairs = (uint32_t)(P < pair_cap ? P : pair_cap);
      if (P > ctr->pairs_needed) ctr->pairs_needed = P;
      if (P > pair_cap) {
        ctr->overflow = 1u;
        atomicOr(&sticky->overflowed, 1u);
        atomicMax(&sticky->pairs_needed_max, P);
      }
    }
  }
  __syncthreads();
  unsigned long long st = s_w[warp] + x - sum;
  for (int t = t0; t < t1; ++t) {
    const unsigned long long v = tile_count[t];
    ranges[t] = v ? make_uint2((uint32_t)min(st, (unsigned long long)pair_cap),
                               (uint32_t)min(st + v, (unsigned long long)pair_cap))
                  : make_uint2(0u, 0u);
    st += v;
  }
}

}  // namespace rs
