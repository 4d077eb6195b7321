// bin.cuh -- tile binning: pair emission and per-tile ranges.
//
// The reference composites in one global (depth, index) order with a
// per-Gaussian pixel bbox gate (render.py:218-222, :250-281); there are no
// tiles. Here the bbox [x0,x1)x[y0,y1) of render.py:133-137 is mapped to the
// 16x16 tiles it touches, tx in [x0/16, (x1-1)/16], ty likewise, and one pair
// (tile, item) is emitted per overlap in depth-rank order. A stable sort by
// tile (sort.cuh) then yields each tile's list in exactly the reference's
// (depth, index) order restricted to that tile.
//
// emit_kernel: one CTA per 256 depth ranks. Tile counts are block-scanned, the
// block's global pair offset comes from a decoupled look-back over earlier
// CTAs (logical ids taken from an atomic ticket, so it cannot deadlock), and
// the CTA then writes its pairs cooperatively: pair k of the block is owned by
// the rank found by binary search over the inclusive scan, so a Gaussian
// covering thousands of tiles is spread over all 256 threads and every global
// store is coalesced. The same CTA adds the rank's tile rectangle to a 2D
// difference array (4 atomics per Gaussian) from which ranges_kernel derives
// every tile's pair count without touching the pairs.
#pragma once
#include "rs_common.cuh"

namespace rs {

constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbInc = 2ull << 62;
constexpr unsigned long long kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long lookback_u64(volatile unsigned long long* st, uint32_t b) {
  unsigned long long excl = 0;
  int j = (int)b - 1;
  while (j >= 0) {
    const unsigned long long s = st[j];
    if ((s & ~kLbMask) == 0) continue;
    excl += s & kLbMask;
    if (s & kLbInc) break;
    --j;
  }
  return excl;
}

__global__ void __launch_bounds__(256) emit_kernel(const uint32_t* __restrict__ items_sorted,
                                                   const Rec* __restrict__ recs, Counters* __restrict__ ctr,
                                                   int TW, uint32_t pair_cap, uint16_t* __restrict__ pair_tiles,
                                                   uint32_t* __restrict__ pair_items, int32_t* __restrict__ diff,
                                                   unsigned long long* __restrict__ status) {
  __shared__ uint32_t s_block;
  __shared__ uint32_t s_incl[256];
  __shared__ int s_tx0[256], s_ty0[256], s_tw[256];
  __shared__ uint32_t s_item[256];
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
    const uint32_t it = items_sorted[r];
    const int4 d = recs[it].d;
    const int tx0 = d.x / kTile, tx1 = (d.y - 1) / kTile, ty0 = d.z / kTile, ty1 = (d.w - 1) / kTile;
    const int tw = tx1 - tx0 + 1;
    nt = (uint32_t)(tw * (ty1 - ty0 + 1));
    s_tx0[tid] = tx0; s_ty0[tid] = ty0; s_tw[tid] = tw; s_item[tid] = it;
    const int DW = TW + 1;
    atomicAdd(&diff[ty0 * DW + tx0], 1);
    atomicAdd(&diff[ty0 * DW + tx1 + 1], -1);
    atomicAdd(&diff[(ty1 + 1) * DW + tx0], -1);
    atomicAdd(&diff[(ty1 + 1) * DW + tx1 + 1], 1);
  }
  // block inclusive scan of tile counts
  uint32_t x = nt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp; ++w) off += s_wsum[w];
  s_incl[tid] = off + x;
  __syncthreads();
  const uint32_t total = s_incl[255];
  if (tid == 0) {
    volatile unsigned long long* st = status;
    if (b == 0) {
      st[0] = kLbInc | total;
      s_base = 0;
    } else {
      st[b] = kLbAgg | total;
      const unsigned long long excl = lookback_u64(st, b);
      st[b] = kLbInc | (excl + total);
      s_base = excl;
    }
    const unsigned long long end = s_base + total;
    if (nvis > 0 && b == (nvis - 1) / 256) {
      ctr->pairs_needed = end;
      ctr->n_pairs = (uint32_t)(end < pair_cap ? end : pair_cap);
      ctr->overflow = end > pair_cap ? 1u : 0u;
    }
  }
  __syncthreads();
  const unsigned long long base = s_base;
  for (uint32_t k = tid; k < total; k += 256) {
    const unsigned long long pos = base + k;
    if (pos >= pair_cap) break;
    // owner: first j with s_incl[j] > k
    int lo = 0, hi = 255;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_incl[mid] > k) hi = mid; else lo = mid + 1;
    }
    const uint32_t local = k - (lo ? s_incl[lo - 1] : 0u);
    const int tw = s_tw[lo];
    const int tile = (s_ty0[lo] + (int)(local / tw)) * TW + s_tx0[lo] + (int)(local % tw);
    pair_tiles[pos] = (uint16_t)tile;
    pair_items[pos] = s_item[lo];
  }
}

// One CTA: 2D prefix sums of the difference array in shared memory give every
// tile's pair count; an exclusive scan over tiles gives [start, end).
__global__ void __launch_bounds__(1024) ranges_kernel(const int32_t* __restrict__ diff, int TW, int TH,
                                                      uint2* __restrict__ ranges) {
  extern __shared__ int32_t sD[];  // (TH+1) x (TW+1)
  const int DW = TW + 1, DH = TH + 1, nd = DW * DH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < nd; i += blockDim.x) sD[i] = diff[i];
  __syncthreads();
  // prefix along x: one warp per row
  for (int y = warp; y < TH; y += nw) {
    int carry = 0;
    for (int x0 = 0; x0 < TW; x0 += 32) {
      const int x = x0 + lane;
      int v = x < TW ? sD[y * DW + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (x < TW) sD[y * DW + x] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // prefix along y: one warp per column
  for (int x = warp; x < TW; x += nw) {
    int carry = 0;
    for (int y0 = 0; y0 < TH; y0 += 32) {
      const int y = y0 + lane;
      int v = y < TH ? sD[y * DW + x] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (y < TH) sD[y * DW + x] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  // exclusive scan of counts in tile order t = y*TW + x; thread owns a contiguous segment
  const int T = TW * TH;
  const int per = (T + blockDim.x - 1) / blockDim.x;
  const int t0 = tid * per, t1 = min(T, t0 + per);
  uint32_t sum = 0;
  for (int t = t0; t < t1; ++t) sum += (uint32_t)sD[(t / TW) * DW + (t % TW)];
  __shared__ uint32_t s_w[32];
  uint32_t xs = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, xs, o);
    if (lane >= o) xs += u;
  }
  if (lane == 31) s_w[warp] = xs;
  __syncthreads();
  uint32_t off = 0;
  for (int w = 0; w < warp; ++w) off += s_w[w];
  uint32_t run = off + xs - sum;
  for (int t = t0; t < t1; ++t) {
    const uint32_t c = (uint32_t)sD[(t / TW) * DW + (t % TW)];
    ranges[t] = make_uint2(run, run + c);
    run += c;
  }
}

}  // namespace rs
