// segbin.cuh -- tile binning through row segments.
//
// The per-tile lists are the reference's global (depth, index) order
// (render.py:218-222) restricted to each tile, over the tiles a Gaussian is
// binned to (rows.cuh: per tile row of its culling box, a contiguous span of
// tile columns). Instead of emitting one (tile, Gaussian) pair per overlap and
// sorting all pairs by tile, the binning works on ROW SEGMENTS -- one per
// (Gaussian, tile row), ~5x fewer than pairs:
//
//   segrows_kernel   per chunk of 256 depth ranks: its Gaussians per tile row
//                    (a difference array over the rows of their culling boxes).
//   segscan_kernel   per row: exclusive prefix over the chunks and the row's
//                    total; the last CTA: per-row segment starts, rows cut into
//                    expansion chunks of 1024, S.
//   segplace_kernel  per rank chunk: each segment's span (row_span) written
//                    straight to its row-major, depth-stable place (row start +
//                    earlier chunks + earlier warps + a per-row ballot), rows
//                    flattened over the lanes. No sort of the segments.
//   chunk_count_kernel  one CTA per chunk: per tile column the number of the
//                    chunk's segments covering it (shared-memory counters);
//                    the chunk's {first segment, row, count, dense} record and
//                    the list of dense chunks (>= 8 tiles per segment).
//   tile_chunks_kernel  per tile (one warp): prefix over its row's chunks and
//                    its total; per 64-tile block the sum and list-length class
//                    counts (atomics).
//   tile_scan_kernel one CTA per 64-tile block: exclusive scan over the tiles
//                    -> ranges [start, end), P, overflow, the blend order.
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

constexpr uint32_t kEmptySpan = 0x00000001u;  // t0 = 1 > t1 = 0: the row lists no tile
constexpr int kExpandCols = 32;                // tile columns per expand CTA (8 warps x 4)
constexpr int kMaxTileRows = 2048;             // image height <= 32767 px
constexpr int kMaxTileCols = 2048;             // image width <= 32767 px
constexpr int kRankChunk = 256;                // depth ranks per placement chunk (one CTA)
#ifndef RS_EXPAND_CHUNK
#define RS_EXPAND_CHUNK 1024  // measured 512 / 1024 / 2048: render 3375 / 3380 / 3316 fps, score
#endif                          // 1492 / 1558 / 1564 views/s, configs[4] 859 / 900 / 913 fps
constexpr int kExpandChunk = RS_EXPAND_CHUNK;  // segments per expansion chunk (rows cut into chunks)

// Tile rows [r0, r1] of a binned record's culling box.
__device__ __forceinline__ void box_rows(const int4 cb, int& r0, int& r1) {
  r0 = cb.z / kTile;
  r1 = (cb.w - 1) / kTile;
}

// Pass 1: per rank chunk (256 consecutive depth ranks) the number of its Gaussians in each tile
// row (a per-CTA difference array over the rows), stored row-major: row_tab[ty][chunk].
__device__ __forceinline__ void segrows_block(uint32_t c, const uint32_t* items_sorted,
                                              const uint32_t* item_rows, uint32_t nvis, int TH,
                                              uint32_t tab_stride, uint32_t* row_tab) {
  __shared__ int s_d[kMaxTileRows + 1];
  __shared__ uint32_t s_w[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (c * kRankChunk >= nvis) return;
  for (int i = tid; i <= TH; i += 256) s_d[i] = 0;
  __syncthreads();
  const uint32_t r = c * kRankChunk + tid;
  if (r < nvis) {
    int r0, r1;
    const uint32_t rr = __ldg(item_rows + __ldg(items_sorted + r));  // the projection's r0 | r1 << 16
    r0 = (int)(rr & 0xffffu);
    r1 = (int)(rr >> 16);
    atomicAdd(&s_d[r0], 1);
    atomicAdd(&s_d[r1 + 1], -1);
  }
  __syncthreads();
  // prefix over the rows (8 per thread) -> the chunk's Gaussians per row
  constexpr int kPer = (kMaxTileRows + 255) / 256;
  int v[kPer], sum = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int ty = tid * kPer + q;
    v[q] = ty < TH ? s_d[ty] : 0;
    sum += v[q];
  }
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = (uint32_t)x;
  __syncthreads();
  int run = x - sum;
#pragma unroll
  for (int w = 0; w < 8; ++w) run += w < warp ? (int)s_w[w] : 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int ty = tid * kPer + q;
    run += v[q];
    if (ty < TH) row_tab[(size_t)ty * tab_stride + c] = (uint32_t)run;
  }
}

__global__ void __launch_bounds__(256) segrows_kernel(const uint32_t* __restrict__ items_sorted,
                                                      const uint32_t* __restrict__ item_rows,
                                                      const Counters* __restrict__ ctr, int TH, uint32_t tab_stride,
                                                      uint32_t* __restrict__ row_tab) {
  pdl_wait();
  pdl_trigger();
  segrows_block(blockIdx.x, items_sorted, item_rows, ctr->n_visible, TH, tab_stride, row_tab);
}

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

// Pass 2, one CTA per tile row: exclusive prefix of the row's chunk counts (in place) and the
// row's total. The last CTA: per-row segment starts, expansion chunk starts, S and the
// segment-capacity verdict.
__device__ __forceinline__ void segscan_row(uint32_t ty, uint32_t* row_tab, uint32_t tab_stride,
                                            uint32_t nvis, uint32_t* row_total) {
  __shared__ uint32_t s_w[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nc = (nvis + kRankChunk - 1) / kRankChunk;
  uint32_t* tab = row_tab + (size_t)ty * tab_stride;
  uint32_t carry = 0;
  constexpr int kPer = 4;
  for (uint32_t base = 0; base < nc; base += 256 * kPer) {
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t i = base + tid * kPer + q;
      v[q] = i < nc ? tab[i] : 0u;
      sum += v[q];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncthreads();  // s_w reuse
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t run = carry + x - sum, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      run += w < warp ? s_w[w] : 0u;
      tot += s_w[w];
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t i = base + tid * kPer + q;
      if (i < nc) tab[i] = run;
      run += v[q];
    }
    carry += tot;
  }
  if (tid == 0) row_total[ty] = carry;
  __syncthreads();
}

// The row totals -> per-row segment starts, expansion chunk starts, S and the
// segment-capacity verdict (one CTA, after every row's total is written).
__device__ __forceinline__ void segscan_tail(Counters* ctr, int TH, uint32_t seg_cap,
                                             const uint32_t* row_total, uint32_t* row_start,
                                             uint32_t* chunk_start, Sticky* sticky) {
  __shared__ uint32_t s_w[16];
  const int tid = threadIdx.x;
  row_scan_block(row_total, TH, row_start, chunk_start, s_w);
  const uint32_t S = __ldcg(row_start + TH);
  if (S > seg_cap)  // nothing is placed: no chunks for the later passes either
    for (int ty = tid; ty <= TH; ty += 256) {
      row_start[ty] = 0;
      chunk_start[ty] = 0;
    }
  if (tid == 0) {
    ctr->n_segs = S < seg_cap ? S : seg_cap;
    if (S > seg_cap) {  // too many segments: the frame is re-run with a larger workspace
      ctr->overflow = 1u;
      atomicOr(&sticky->overflowed, 1u);
      // pair capacity that certainly holds this frame's segments (segments <= pairs + 2 n)
      if (S > ctr->pairs_needed) ctr->pairs_needed = S;
      atomicMax(&sticky->pairs_needed_max, (unsigned long long)S);
    }
  }
  __syncthreads();
}

// Pass 2, one CTA per tile row: exclusive prefix of the row's chunk counts (in place) and the
// row's total. The last CTA: per-row segment starts, expansion chunk starts, S and the
// segment-capacity verdict.
__global__ void __launch_bounds__(256) segscan_kernel(uint32_t* __restrict__ row_tab, uint32_t tab_stride,
                                                      Counters* __restrict__ ctr, int TH, uint32_t seg_cap,
                                                      uint32_t* __restrict__ row_total,
                                                      uint32_t* __restrict__ row_start,
                                                      uint32_t* __restrict__ chunk_start,
                                                      Sticky* __restrict__ sticky) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_last;
  segscan_row(blockIdx.x, row_tab, tab_stride, ctr->n_visible, row_total);
  __threadfence();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctr->emit_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  segscan_tail(ctr, TH, seg_cap, row_total, row_start, chunk_start, sticky);
}

// Pass 3, one CTA per rank chunk: every segment written straight to its place in row-major,
// depth-stable order -- row start + the earlier chunks' Gaussians in the row (pass 2) + the
// earlier warps' (a per-row ballot per warp) + the earlier lanes'. The rows of the warp's
// Gaussians are flattened over the lanes for the span computation (row_span, rows.cuh).
// Dynamic shared memory: per warp and row the ballot and the offset (2 x 8 x TH words).
__device__ __forceinline__ void segplace_block(uint32_t c, const uint32_t* items_sorted,
                                               const Rec* recs, uint32_t nvis, int TH,
                                               const uint32_t* row_tab, uint32_t tab_stride,
                                               const uint32_t* row_start,
                                               uint32_t* seg_item, uint32_t* seg_span,
                                               float4* geom) {
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_bal = s_dyn;           // [8][TH]
  uint32_t* s_off = s_dyn + 8 * TH;  // [8][TH]
  __shared__ RowGeom s_g[8][32];
  __shared__ int4 s_cb[8][32];
  __shared__ int s_pre[8][33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (c * kRankChunk >= nvis) return;
  const uint32_t r = c * kRankChunk + tid;
  int r0 = 0x7fffffff, r1 = -1, nr = 0;
  uint32_t it = 0;
  if (r < nvis) {
    it = __ldg(items_sorted + r);
    const Rec* R = recs + it;
    const int4 d = __ldg(&R->d);
    const int4 cb = cullbox_of(d);
    box_rows(cb, r0, r1);
    nr = r1 - r0 + 1;
    s_cb[warp][lane] = make_int4(cb.x, cb.y, cb.z, cb.w | (cullbox_ell(d) ? (int)0x80000000 : 0));
    if (cullbox_ell(d)) {
      s_g[warp][lane] = row_geom(__ldg(&R->a), __ldg(&R->b));
      store_row_geom(geom + 2 * (size_t)it, s_g[warp][lane]);  // blend2_kernel's quarter masks
    }
  }
  for (int i = lane; i < TH; i += 32) s_off[warp * TH + i] = 0u;
  __syncwarp();
  const int lo = __reduce_min_sync(0xffffffffu, r0), hi = __reduce_max_sync(0xffffffffu, r1);
  const uint32_t span = (uint32_t)(r1 - r0);
  for (int t0 = lo; t0 <= hi; t0 += 32) {  // per row: which of the warp's Gaussians lie in it
    uint32_t mine = 0;                      // row t0 + lane's ballot
    const int m = min(32, hi - t0 + 1);
    for (int q = 0; q < m; ++q) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (uint32_t)(t0 + q - r0) <= span);
      mine = lane == q ? bal : mine;
    }
    if (lane < m) {
      s_bal[warp * TH + t0 + lane] = mine;
      s_off[warp * TH + t0 + lane] = (uint32_t)__popc(mine);
    }
  }
  __syncthreads();
  for (int ty = tid; ty < TH; ty += 256) {  // per row: start of each warp's run
    uint32_t run = __ldg(row_start + ty) + __ldg(row_tab + (size_t)ty * tab_stride + c);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t v = s_off[w * TH + ty];
      s_off[w * TH + ty] = run;
      run += v;
    }
  }
  __syncthreads();
  // the warp's segments flattened over the lanes
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
  const int pre = x - nr;
  int carry = 0;  // owners started before the window (the valid lanes are 0..m-1, nr >= 1)
  for (int base = 0; base < total; base += 32) {
    const int j = base + lane;
    const int rel = pre - base;
    const uint32_t starts = __reduce_or_sync(0xffffffffu, nr > 0 && rel >= 0 && rel < 32 ? 1u << rel : 0u);
    const int own = j < total ? carry + __popc(starts & ((2u << lane) - 1u)) - 1 : 0;
    carry += __popc(starts);
    const uint32_t sitem = __shfl_sync(0xffffffffu, it, own);
    if (j < total) {
      const int k = j - s_pre[warp][own];
      const int4 c4 = s_cb[warp][own];
      const bool ell = c4.w < 0;
      const int4 cb = make_int4(c4.x, c4.y, c4.z, c4.w & 0x7fffffff);
      const int ty = cb.z / kTile + k;
      int t0 = cb.x / kTile, t1 = (cb.y - 1) / kTile;
      const bool ok = ell ? row_span(s_g[warp][own], cb, ty, t0, t1) : true;
      const uint32_t pos = s_off[warp * TH + ty] + (uint32_t)__popc(s_bal[warp * TH + ty] & ((1u << own) - 1u));
      seg_item[pos] = sitem;
      seg_span[pos] = ok ? ((uint32_t)t0 | ((uint32_t)t1 << 16)) : kEmptySpan;
    }
  }
  __syncthreads();  // shared memory reuse by the caller's next block
}

__global__ void __launch_bounds__(256) segplace_kernel(const uint32_t* __restrict__ items_sorted,
                                                       const Rec* __restrict__ recs, const Counters* __restrict__ ctr,
                                                       int TH, const uint32_t* __restrict__ row_tab,
                                                       uint32_t tab_stride, const uint32_t* __restrict__ row_start,
                                                       uint32_t* __restrict__ seg_item,
                                                       uint32_t* __restrict__ seg_span, float4* __restrict__ geom) {
  pdl_wait();
  pdl_trigger();
  if (ctr->overflow) return;
  segplace_block(blockIdx.x, items_sorted, recs, ctr->n_visible, TH, row_tab, tab_stride, row_start, seg_item,
                 seg_span, geom);
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

// Expansion: a chunk's covering segments appended to each column's tile list after all earlier
// chunks of the row (ranges + chunk prefix). A sparse-chunk CTA owns 32 tile columns; warp w
// takes 128 of the chunk's segments (all loads issued up front), compacts the ones reaching
// the CTA's columns, turns each span into a 32-bit column mask, and a 32x32 bit transpose (5
// shuffle stages) gives lane c the mask of the warp's segments covering column c; lane c then
// appends those items in segment (= depth) order after the earlier warps' counts (one
// shared-memory exchange per chunk).
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
__device__ __forceinline__ void expand_dense_chunk(const uint32_t* __restrict__ seg_item,
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
      sp = seg_span[s0 + base + tid];
      sit = seg_item[s0 + base + tid];
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
#ifndef RS_EXPAND_GROUPS
#define RS_EXPAND_GROUPS 4  // column groups per sparse-expansion CTA (measured 1 / 2 / 4: score
#endif                      // 1545 / 1554 / 1563 views/s, render 3381 / 3390 / 3380 fps)

__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ seg_item,
                                                     const uint32_t* __restrict__ seg_span,
                                                     const uint2* __restrict__ chunk_info,
                                                     const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                     const uint32_t* __restrict__ chunk_count /* [chunk][TW] */,
                                                     const uint2* __restrict__ ranges,
                                                     const Counters* __restrict__ ctr,
                                                     uint32_t* __restrict__ pair_items, int major_thresh) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_cnt[2][8][32];
  __shared__ uint32_t s_cm[8][kExpandSub * 32], s_ci[8][kExpandSub * 32];  // per-warp compaction
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ctr->overflow) return;
  const uint32_t lt = (1u << lane) - 1u;
  // column group fastest in the grid: a chunk's CTAs run together and share its segments in L2
  // (RS_EXPAND_GROUPS > 1: each CTA walks that many column groups of a chunk, the chunk's spans
  // and items loaded once)
  const uint32_t n_chunks = chunk_start[TH];
  int flip = 0;
  for (uint32_t gc = blockIdx.y; gc < n_chunks; gc += gridDim.y) {  // chunks of all rows, grid-strided
    const uint2 info = chunk_info[gc];  // {first segment, row | count << 16 | dense << 31}
    if (info.y >> 31) continue;         // dense: expand_dense_kernel (concurrently, on a second stream)
    const int ty = (int)(info.y & 0xffffu);
    const uint32_t cnt = (info.y >> 16) & 0x7fffu;
    // warp w: the chunk's segments [128 w, 128 w + 128), 32 per sub-step, all loads issued up front
    uint32_t sid[kExpandSub], m[kExpandSub], item[kExpandSub], cm[kExpandSub];
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const uint32_t e = (uint32_t)(warp * 32 * kExpandSub + k * 32 + lane);
      sid[k] = e < cnt ? info.x + e : 0xffffffffu;
    }
    uint32_t sp[kExpandSub];
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) sp[k] = seg_span[sid[k] != 0xffffffffu ? sid[k] : 0u];  // all in flight
#if RS_EXPAND_GROUPS > 1
    uint32_t it_all[kExpandSub];
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) it_all[k] = sid[k] != 0xffffffffu ? seg_item[sid[k]] : 0u;
#endif
    for (int g0 = blockIdx.x * kExpandCols; g0 < TW; g0 += gridDim.x * kExpandCols) {
    const int c = g0 + lane;  // lane's column (every warp)
    const uint32_t pos = c < TW ? ranges[ty * TW + c].x + chunk_count[(size_t)gc * TW + c] : 0u;
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const int a = max((int)(sp[k] & 0xffffu) - g0, 0), b = min((int)(sp[k] >> 16) - g0, kExpandCols - 1);
      m[k] = sid[k] != 0xffffffffu && a <= b ? (0xffffffffu >> (31 - b)) & (0xffffffffu << a) : 0u;
    }
#pragma unroll
#if RS_EXPAND_GROUPS > 1
    for (int k = 0; k < kExpandSub; ++k) item[k] = m[k] ? it_all[k] : 0u;
#else
    for (int k = 0; k < kExpandSub; ++k) item[k] = m[k] ? seg_item[sid[k]] : 0u;
#endif
    // the warp's segments that reach the CTA's columns, compacted in order (fewer transposes)
    uint32_t nrel = 0;
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const uint32_t bal = __ballot_sync(0xffffffffu, m[k] != 0u);
      if (m[k]) {
        const uint32_t at = nrel + __popc(bal & lt);
        s_cm[warp][at] = m[k];
        s_ci[warp][at] = item[k];
      }
      nrel += __popc(bal);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      const uint32_t e = k * 32 + lane;
      m[k] = e < nrel ? s_cm[warp][e] : 0u;
      item[k] = e < nrel ? s_ci[warp][e] : 0u;
    }
    __syncwarp();
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < kExpandSub; ++k) {
      cm[k] = k * 32 < (int)nrel ? transpose32(m[k], lane) : 0u;
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
    }  // column groups
  }
}

// The dense chunks (listed by chunk_count_kernel, any order: chunks are independent).
__global__ void __launch_bounds__(256) expand_dense_kernel(const uint32_t* __restrict__ seg_item,
                                                           const uint32_t* __restrict__ seg_span,
                                                           const uint2* __restrict__ chunk_info,
                                                           const uint32_t* __restrict__ dense_list, int TW,
                                                           const uint32_t* __restrict__ chunk_count,
                                                           const uint2* __restrict__ ranges,
                                                           Counters* __restrict__ ctr,
                                                           uint32_t* __restrict__ pair_items) {
  pdl_wait();
  pdl_trigger();
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
    expand_dense_chunk(seg_item, seg_span, info.x, (info.y >> 16) & 0x7fffu, (int)(info.y & 0xffffu), gc,
                       (int)(t % groups) * kExpandCols, TW, chunk_count, ranges, pair_items, s_item, s_span, s_wk);
    flip ^= 1;
  }
}

// Expansion counts (order-free): per (chunk, tile column) the number of the chunk's segments
// covering the column -- a shared-memory difference array over the row's columns (two
// atomics per segment) and its prefix, one CTA per chunk.
__device__ __forceinline__ void chunk_count_loop(uint32_t first, uint32_t stride,
                                                 const uint32_t* seg_span,
                                                 const uint32_t* row_start,
                                                 const uint32_t* chunk_start, int TH, int TW,
                                                 uint32_t* chunk_count,
                                                 uint2* chunk_info, int dense_span,
                                                 Counters* ctr, uint32_t* dense_list) {
  __shared__ uint32_t s_cnt[kMaxTileCols + 1];
  __shared__ uint32_t s_tiles, s_w[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t gc = first;; gc += stride) {
    int ty;
    uint32_t lc;
    if (!chunk_of(chunk_start, TH, gc, ty, lc)) break;
    __syncthreads();
    for (int c = tid; c <= TW; c += 256) s_cnt[c] = 0;
    if (tid == 0) s_tiles = 0;
    __syncthreads();
    const uint32_t s0 = row_start[ty] + lc * kExpandChunk, s1 = min(row_start[ty + 1], s0 + kExpandChunk);
    int tiles = 0;
    for (uint32_t sidx = s0 + tid; sidx < s1; sidx += 256) {  // a difference array over the columns
      const uint32_t sp = seg_span[sidx];
      const int t0 = (int)(sp & 0xffffu), t1 = (int)(sp >> 16);
      if (t0 <= t1) {
        atomicAdd(&s_cnt[t0], 1u);
        atomicAdd(&s_cnt[t1 + 1], 0xffffffffu);
      }
      tiles += max(t1 - t0 + 1, 0);
    }
    tiles = __reduce_add_sync(0xffffffffu, tiles);
    if (lane == 0) atomicAdd(&s_tiles, (uint32_t)tiles);
    __syncthreads();
    {  // inclusive prefix over the columns: thread t owns columns [8t, 8t + 8)
      constexpr int kPer = kMaxTileCols / 256;
      uint32_t v[kPer], sum = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int c = tid * kPer + q;
        v[q] = c < TW ? s_cnt[c] : 0u;
        sum += v[q];
      }
      uint32_t x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_w[warp] = x;
      __syncthreads();
      uint32_t run = x - sum;
#pragma unroll
      for (int w = 0; w < 8; ++w) run += w < warp ? s_w[w] : 0u;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int c = tid * kPer + q;
        run += v[q];
        if (c < TW) s_cnt[c] = run;
      }
    }
    __syncthreads();
    // dense: the segments average >= dense_span tiles (expand_kernel's ballot walk)
    if (tid == 0) {
      const bool dense = s_tiles >= (uint32_t)dense_span * (s1 - s0);
      chunk_info[gc] = make_uint2(s0, (uint32_t)ty | ((s1 - s0) << 16) | (dense ? 0x80000000u : 0u));
      if (dense) dense_list[atomicAdd(&ctr->n_dense, 1u)] = gc;
    }
    for (int c = tid; c < TW; c += 256) chunk_count[(size_t)gc * TW + c] = s_cnt[c];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) chunk_count_kernel(const uint32_t* __restrict__ seg_span,
                                                          const uint32_t* __restrict__ row_start,
                                                          const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                          uint32_t* __restrict__ chunk_count,
                                                          uint2* __restrict__ chunk_info, int dense_span,
                                                          Counters* __restrict__ ctr,
                                                          uint32_t* __restrict__ dense_list) {
  pdl_wait();
  pdl_trigger();
  chunk_count_loop(blockIdx.x, gridDim.x, seg_span, row_start, chunk_start, TH, TW, chunk_count, chunk_info,
                   dense_span, ctr, dense_list);
}

// Per tile: its chunks' counts -> exclusive prefix over the row's chunks (in place) and the
// tile's total (one warp per tile, 32 chunks per scan step).
__device__ __forceinline__ uint32_t tile_chunks_block(uint32_t vb, const uint32_t* chunk_start, int TH,
                                                      int TW, uint32_t* chunk_count,
                                                      uint32_t* tile_count) {
  const int lane = threadIdx.x & 31;
  const int t = (int)vb * 8 + (threadIdx.x >> 5);
  if (t >= TW * TH) return 0;
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
  return carry;
}

// Class of a tile's list length for the blend order: floor(log2 v) and the next two bits.
__device__ __forceinline__ int len_class(uint32_t v) {
  if (v < 4) return (int)v;
  const int e = 31 - __clz(v);
  return 4 * (e - 1) + (int)((v >> (e - 2)) & 3u);
}

constexpr int kScanTiles = 64;            // tiles per tile-scan block (8 tile_chunks CTAs)
constexpr int kScanClasses = 33 * 4;      // list-length classes (len_class)

// One warp per tile (tile_chunks_block), then per CTA (8 consecutive tiles, inside one
// 64-tile scan block): the block's pair-count sum and the class counts of the blend order,
// accumulated in the per-frame zeroed scan_part / scan_cls.
__global__ void __launch_bounds__(256) tile_chunks_kernel(const uint32_t* __restrict__ chunk_start, int TH, int TW,
                                                          uint32_t* __restrict__ chunk_count,
                                                          uint32_t* __restrict__ tile_count,
                                                          unsigned long long* __restrict__ scan_part,
                                                          uint32_t* __restrict__ scan_cls) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_v[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t v = tile_chunks_block(blockIdx.x, chunk_start, TH, TW, chunk_count, tile_count);
  if ((tid & 31) == 0) s_v[warp] = v;
  __syncthreads();
  const int t0 = (int)blockIdx.x * 8, T = TW * TH;
  if (tid < 8 && t0 + tid < T && s_v[tid]) atomicAdd(&scan_cls[len_class(s_v[tid])], 1u);
  if (tid == 0) {
    unsigned long long sum = 0;
    uint32_t empties = 0;
    for (int w = 0; w < 8; ++w) {
      sum += s_v[w];
      empties += (t0 + w < T && s_v[w] == 0) ? 1u : 0u;
    }
    if (sum) atomicAdd(&scan_part[t0 / kScanTiles], sum);
    if (empties) atomicAdd(&scan_cls[0], empties);
  }
}

// A frame without items (no tile scan): every range is empty (the frame memset) and the blend
// order is the identity.
__global__ void tile_order_identity_kernel(uint32_t* __restrict__ tile_order, int T) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) tile_order[t] = (uint32_t)t;
}

// One CTA (64 threads) per 64-tile scan block: the block's exclusive start from the earlier
// blocks' sums, each tile's range [start, end) (empty tiles [0, 0)), P and the pair-capacity
// verdict (block 0), and the blend order: tiles by list-length class, longest first (class
// starts from the frame's class counts, global cursors within a class).
__global__ void __launch_bounds__(64) tile_scan_kernel(const uint32_t* __restrict__ tile_count, int T,
                                                       Counters* __restrict__ ctr, uint32_t pair_cap,
                                                       uint2* __restrict__ ranges, Sticky* __restrict__ sticky,
                                                       uint32_t* __restrict__ tile_order,
                                                       const unsigned long long* __restrict__ scan_part,
                                                       uint32_t* __restrict__ scan_cls) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t s_cstart[kScanClasses];
  __shared__ unsigned long long s_w[2][2];
  __shared__ uint32_t s_x0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t k = blockIdx.x, nsb = gridDim.x;
  if (warp == 0) {  // class starts, classes descending
    constexpr int kPer = (kScanClasses + 31) / 32;
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = kScanClasses - 1 - (lane * kPer + q);
      v[q] = c >= 0 ? scan_cls[c] : 0u;
      sum += v[q];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t run = x - sum;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = kScanClasses - 1 - (lane * kPer + q);
      if (c >= 0) s_cstart[c] = run;
      run += v[q];
    }
  }
  unsigned long long pre = 0, all = 0;
  for (uint32_t j = tid; j < nsb; j += 64) {
    const unsigned long long p = scan_part[j];
    all += p;
    pre += j < k ? p : 0ull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pre += __shfl_xor_sync(0xffffffffu, pre, o);
    all += __shfl_xor_sync(0xffffffffu, all, o);
  }
  const int t = (int)k * kScanTiles + tid;
  const bool in = t < T;
  const uint32_t v = in ? tile_count[t] : 0u;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 0) {
    s_w[warp][0] = pre;
    s_w[warp][1] = all;
  }
  if (lane == 31 && warp == 0) s_x0 = x;
  __syncthreads();
  pre = s_w[0][0] + s_w[1][0];
  all = s_w[0][1] + s_w[1][1];
  if (k == 0 && tid == 0) {  // P and the overflow verdict
    ctr->n_pairs = (uint32_t)(all < pair_cap ? all : pair_cap);
    if (all > ctr->pairs_needed) ctr->pairs_needed = all;
    if (all > pair_cap) {
      ctr->overflow = 1u;
      atomicOr(&sticky->overflowed, 1u);
      atomicMax(&sticky->pairs_needed_max, all);
    }
  }
  const unsigned long long st = pre + (warp ? s_x0 : 0u) + x - v;
  if (in)
    ranges[t] = v ? make_uint2((uint32_t)min(st, (unsigned long long)pair_cap),
                               (uint32_t)min(st + v, (unsigned long long)pair_cap))
                  : make_uint2(0u, 0u);
  // empty tiles (most of a sparse frame: one class) take one cursor atomic per warp
  const uint32_t empties = __ballot_sync(0xffffffffu, in && v == 0);
  uint32_t base = 0;
  if (lane == 0 && empties) base = atomicAdd(&scan_cls[kScanClasses], (uint32_t)__popc(empties));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (in) {
    const int c = v ? len_class(v) : 0;
    tile_order[s_cstart[c] + (v ? atomicAdd(&scan_cls[kScanClasses + c], 1u)
                                : base + __popc(empties & ((1u << lane) - 1u)))] = (uint32_t)t;
  }
}

}  // namespace rs
