// dsort.cuh -- the frame's depth sort as ONE cooperative kernel (replaces the
// compaction kernel + four onesweep launches of sort.cuh on the frame path).
//
// np.lexsort((idx, depth)) of render.py:218-222 over the binned items: a stable
// LSD radix sort of their 32-bit depth keys (8-bit digits, 4 passes), values =
// item index. One CTA per SM stays resident for the whole sort; passes are
// separated by grid barriers instead of kernel boundaries, and a CTA's digit
// offsets come from the published per-CTA histograms (every CTA reads the
// G x 256 table after a barrier) instead of a decoupled look-back chain:
//
//   pass 0 reads the projection's per-item keys directly (culled items carry
//   kInvalidKey and drop out: the compaction is fused into the first pass),
//   CTA b taking items [b ci, (b+1) ci); passes 1-3 read the previous pass's
//   output, CTA b taking sorted positions [b cs, (b+1) cs), cs = ceil(n_vis/G).
//   Per pass: barrier; column prefix of the pass's [G][256] histogram table
//   over the rows < b and the digit totals; the keys ranked stably within
//   4096-key sub-chunks (warp multisplit, per-warp digit runs) and scattered to
//   their global positions, each key also counted for the next pass in the row
//   of the CTA that will own its new position (global atomics) -- so one grid
//   barrier per pass. n_visible = the pass-0 total. Passes alternate B, A, B, A: the
//   sorted keys / items end in kA / vA. Data written by other CTAs is read
//   through L2 (ld.cg): an SM's L1 may hold the buffer from two passes earlier.
//
// Same result as the onesweep path bit for bit (the parity tests compare the
// sorted order with the oracle's).
#pragma once
#include "rs_common.cuh"

namespace rs {

#ifdef RS_DSORT_PROBE  // tools/dsort_probe.cu: per-CTA globaltimer stamps at the phase boundaries
__device__ unsigned long long* g_dsort_probe;
#define DSORT_MARK(k)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0) {                                                             \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      g_dsort_probe[blockIdx.x * 32 + (k)] = t_;                                        \
    }                                                                                   \
  } while (0)
#else
#define DSORT_MARK(k) \
  do {                \
  } while (0)
#endif

constexpr int kDsortThreads = 1024;                           // one CTA of 32 warps per SM
constexpr int kDsortWarps = kDsortThreads / 32;
constexpr int kDsortItems = 4;                                // keys per thread per sub-chunk
constexpr int kDsortChunk = kDsortThreads * kDsortItems;      // 4096
// Up to kDsortRedMax visible keys (dsort_kernel's red_max; RS_DSORT_RED_MAX overrides it), the next pass's per-CTA histograms are accumulated with global
// atomics during the scatter (one grid barrier per pass); above it, each CTA histograms its own
// range after the scatter's barrier and publishes it behind a second barrier -- the per-key
// atomics cost more than a barrier there (tools/dsort_probe.cu, 9-bit digits: 200k keys 43.3
// vs 45.1 us, 275k 46.5 vs 47.2, 350k 50.3 vs 49.2, 500k 62.8 vs 58.3 us).
constexpr uint32_t kDsortRedMax = 300000;

// Grid barrier over the co-resident CTAs of a cooperative launch: arrive on a counter that
// only grows (zeroed before the launch by the frame's counter memset), spin until it reaches
// the barrier's multiple of the grid size.
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // the arrival counter only grows: this barrier is complete when it reaches the next
    // multiple of nblocks (no reset, no second word -- the last arrival releases everyone).
    // Arrival is a release RMW (the CTA's writes, ordered before it by the bar.sync above,
    // become visible with it), the polling an acquire load.
    uint32_t arrived;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    const uint32_t target = (arrived / nblocks + 1) * nblocks;
    uint32_t seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while ((int)(seen - target) < 0);
  }
  __syncthreads();
}

constexpr int kDsortMaxBins = 512;  // 9-bit digits (3 passes) when the keys' range allows

struct DsortSmem {
  uint32_t hist[kDsortMaxBins];                 // running global offset of each digit for this CTA's keys
  uint32_t whist[kDsortWarps][kDsortMaxBins];   // per-warp digit counts of a sub-chunk, then per-warp starts
  uint32_t part[kDsortWarps][kDsortMaxBins];    // column-prefix partial sums: [row slice][digit]
  uint32_t nexth[kDsortMaxBins];                // this CTA's keys per next-pass digit (the digit totals)
  uint32_t wsum[16];
};

// Column prefix of a pass's [G][NB] digit histogram table (16-bit counts, two per word):
// pre = sum over rows < b for digit tid < NB. CTAs in the first half sum the rows before
// them, the others the rows from b on and subtract from the pass's digit totals `gtot`
// (accumulated separately) -- no CTA reads more than G/2 rows, and the table traffic of the
// phase (every CTA reading it at once right after the barrier) is a quarter of a full
// 32-bit read. Thread (slice w, digit group g) sums up to kRows rows of digits [8 g, 8 g + 8)
// (one 16-byte load per row, all in flight); the slices are combined in shared memory.
template <int NB>
__device__ __forceinline__ void column_prefix(const uint32_t* __restrict__ table, const uint32_t* __restrict__ gtot,
                                              uint32_t G, uint32_t b, DsortSmem& S, uint32_t& pre,
                                              uint32_t& tot) {
  constexpr int kGroups = NB / 8, kSlices = kDsortThreads / kGroups;  // 32 x 32 (NB 256), 64 x 16 (NB 512)
  constexpr int kRows = (80 + kSlices - 1) / kSlices;                  // slices x rows >= G / 2 (G <= 160)
  constexpr int kQ = kDsortThreads / NB, kPerQ = kSlices / kQ;         // slice reducers per digit
  const int tid = threadIdx.x, g = tid % kGroups, w = tid / kGroups;
  const bool low = 2 * b <= G;
  const uint32_t ra = low ? 0u : b, rb = low ? b : G;  // rows summed: [ra, rb), rb - ra <= G / 2
  const uint32_t r0 = min(ra + w * kRows, rb);
  uint4 xs[kRows];
#pragma unroll
  for (int k = 0; k < kRows; ++k) {  // every load issued before any is used
    const uint32_t r = r0 + k;
    xs[k] = r < rb ? __ldcg(reinterpret_cast<const uint4*>(table + (size_t)r * (NB / 2)) + g)
                   : make_uint4(0, 0, 0, 0);
  }
  uint32_t sp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kRows; ++k) {
    const uint32_t v[4] = {xs[k].x, xs[k].y, xs[k].z, xs[k].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sp[2 * q] += v[q] & 0xffffu;
      sp[2 * q + 1] += v[q] >> 16;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) S.part[w][8 * g + k] = sp[k];
  __syncthreads();
  {  // the slices of digit d summed by kQ threads (kPerQ slices each), then combined
    const int d = tid % NB, q = tid / NB;
    uint32_t a = 0;
#pragma unroll
    for (int k = 0; k < kPerQ; ++k) a += S.part[kPerQ * q + k][d];
    S.whist[q][d] = a;  // whist is free until the rank phase
  }
  __syncthreads();
  pre = 0;
  tot = 0;
  if (tid < NB) {
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) sum += S.whist[q][tid];
    tot = __ldcg(gtot + tid);
    pre = low ? sum : tot - sum;
  }
}

// dtab layout (words; zero on entry, the frame memset): the pass-0 table [G][256] of raw
// 9-bit digit counts (16-bit, two per word), the tables of passes 1.. ([G][NB / 2] each), the
// digit totals [4][512] and each CTA's {smallest, largest} binned key [G][2].
__host__ __device__ constexpr size_t dsort_tab_words(uint32_t G) { return (size_t)3 * G * 256 + 4 * 512 + 2 * G; }

// The sort proper for NB-bin digits, after the kernel's pass-0 histogram and first barrier:
// NB = 256 -> 4 passes of 8 bits over the raw keys; NB = 512 -> 3 passes of 9 bits over
// key - kbase (the frame's keys span < 2^27). Pass 0's table holds raw 9-bit digit counts:
// digit (key - kbase) & 511 is a rotation of key & 511 by kbase (NB 512), digit key & 255 a
// fold of it (NB 256), applied to the column prefix. Pass p + 1's table is accumulated by
// pass p's scatter (global atomics into the row of the CTA that will own each key's new
// position; above red_max visible keys each CTA histograms its own range behind a second
// barrier instead). Passes write A / B alternately so that the last one writes kA / vA.
template <int NB, bool LAST_KEYS>
__device__ __forceinline__ void dsort_body(uint32_t n_items, uint32_t* __restrict__ kA, uint32_t* __restrict__ vA,
                                           uint32_t* __restrict__ kB, uint32_t* __restrict__ vB,
                                           uint32_t* __restrict__ tables, Counters* __restrict__ ctr,
                                           uint32_t red_max, uint32_t kbase, DsortSmem& S,
                                           const uint32_t* __restrict__ keys_all, uint32_t (&kk)[kDsortItems],
                                           bool one) {
  constexpr int DB = NB == 512 ? 9 : 8;
  constexpr int P = NB == 512 ? 3 : 4;
  constexpr uint32_t M = NB - 1;
  constexpr int NW = NB / 2;  // table words per row (passes >= 1)
  uint32_t* bar = ctr->gbar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t ci = (n_items + G - 1) / G;
  uint32_t nvis = 0, cs = 1;
  const uint32_t* kin = keys_all;
  const uint32_t* vin = nullptr;  // pass 0: value = item index
  uint32_t* kout = (P % 2 == 1) ? kA : kB;
  uint32_t* vout = (P % 2 == 1) ? vA : vB;
  bool red = true;  // next pass's histograms by atomics during the scatter (set after pass 0's prefix)
  uint32_t* gtot = tables + (size_t)3 * G * 256;  // [4][512] digit totals
  const uint32_t rot = kbase & 511u;
  auto table_of = [&](int p) { return p == 0 ? tables : tables + (size_t)G * 256 + (size_t)(p - 1) * G * NW; };
  for (int p = 0; p < P; ++p) {
    const int shift = DB * p;
    if (p > 0) grid_barrier(bar, G);
    if (p > 0 && !red) {  // this pass's histogram of the CTA's own range (written by the last scatter)
      const uint32_t lo = min(b * cs, nvis), hi = min(lo + cs, nvis);
      one = hi - lo <= (uint32_t)kDsortChunk;
      for (int i = tid; i < NB; i += kDsortThreads) S.hist[i] = 0;
      __syncthreads();
      for (uint32_t base = lo; base < hi; base += kDsortChunk) {
        const uint32_t wbase = base + warp * 32 * kDsortItems;
#pragma unroll
        for (int it = 0; it < kDsortItems; ++it) {
          const uint32_t i = wbase + it * 32 + lane;
          kk[it] = i < hi ? __ldcg(kin + i) : kInvalidKey;
          if (i < hi) atomicAdd(&S.hist[((kk[it] - kbase) >> shift) & M], 1u);
        }
      }
      __syncthreads();
      uint32_t* tp = table_of(p);
      if (tid < NW) tp[(size_t)b * NW + tid] = S.hist[2 * tid] | (S.hist[2 * tid + 1] << 16);
      if (tid < NB && S.hist[tid]) atomicAdd(gtot + p * 512 + tid, S.hist[tid]);
      grid_barrier(bar, G);
    }
    DSORT_MARK(2 + 4 * p);
    uint32_t pre, tot;
    if (p == 0) {  // raw 9-bit counts -> this pass's digits (rotation by kbase / fold to 8 bits)
      uint32_t pr, tr;
      column_prefix<512>(tables, gtot, G, b, S, pr, tr);
      if (tid < 512) {
        S.part[0][tid] = pr;
        S.part[1][tid] = tr;
      }
      __syncthreads();
      pre = tot = 0;
      if (tid < NB) {
        if (NB == 512) {
          pre = S.part[0][(tid + rot) & 511u];
          tot = S.part[1][(tid + rot) & 511u];
        } else {
          pre = S.part[0][tid] + S.part[0][tid + 256];
          tot = S.part[1][tid] + S.part[1][tid + 256];
        }
      }
      __syncthreads();
    } else {
      column_prefix<NB>(table_of(p), gtot + p * 512, G, b, S, pre, tot);
    }
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31 && warp < NB / 32) S.wsum[warp] = x;
    __syncthreads();
    uint32_t dstart = x - tot, all = 0;
#pragma unroll
    for (int w = 0; w < NB / 32; ++w) {
      dstart += w < warp ? S.wsum[w] : 0u;
      all += S.wsum[w];
    }
    if (p == 0) {
      nvis = all;
      cs = max((nvis + G - 1) / G, 1u);
      red = nvis <= red_max;
    }
    if (tid < NB) S.hist[tid] = dstart + pre;  // where this CTA's first key of digit tid goes
    uint32_t lo, hi;
    if (p == 0) {
      lo = min(b * ci, n_items);
      hi = min(lo + ci, n_items);
    } else {
      lo = min(b * cs, nvis);
      hi = min(lo + cs, nvis);
      one = hi - lo <= (uint32_t)kDsortChunk;
    }
    uint32_t* next = p < P - 1 && red ? table_of(p + 1) : nullptr;
    __syncthreads();
    DSORT_MARK(3 + 4 * p);
    // stable rank + scatter, sub-chunk by sub-chunk (warp-contiguous, item-major, lane-minor)
    for (uint32_t base = lo; base < hi; base += kDsortChunk) {
      const uint32_t wbase = base + warp * 32 * kDsortItems;
      uint32_t rk[kDsortItems], vv[kDsortItems];
      bool ok[kDsortItems];
#pragma unroll
      for (int it = 0; it < kDsortItems; ++it) {
        const uint32_t i = wbase + it * 32 + lane;
        if (!one || (p > 0 && red)) kk[it] = i < hi ? __ldcg(kin + i) : kInvalidKey;
        vv[it] = vin ? (i < hi ? __ldcg(vin + i) : 0u) : i;  // values loaded with the keys
        ok[it] = i < hi && (p > 0 || kk[it] != kInvalidKey);
      }
      for (int i = tid; i < kDsortWarps * NB; i += kDsortThreads) S.whist[i / NB][i % NB] = 0;
      __syncthreads();
      DSORT_MARK(20 + 3 * p);
#pragma unroll
      for (int it = 0; it < kDsortItems; ++it) {
        const uint32_t d = ((kk[it] - kbase) >> shift) & M;
        uint32_t peers = __ballot_sync(0xffffffffu, ok[it]);
#pragma unroll
        for (int bt = 0; bt < DB; ++bt) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (d >> bt) & 1u);
          peers &= ((d >> bt) & 1u) ? bal : ~bal;
        }
        uint32_t r0 = 0;
        if (ok[it]) r0 = S.whist[warp][d];
        __syncwarp();
        if (ok[it] && (31 - __clz(peers)) == lane) S.whist[warp][d] = r0 + __popc(peers);
        __syncwarp();
        rk[it] = r0 + __popc(peers & lt);
      }
      __syncthreads();
      DSORT_MARK(21 + 3 * p);
      // per digit: start of each warp's run = running offset + earlier warps; 4 threads per
      // digit (8 warps each), their totals combined through part, 256 digits at a time
#pragma unroll
      for (int dh = 0; dh < NB; dh += 256) {
        const int d = dh + (tid & 255), qq = tid >> 8;
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          c[w] = S.whist[8 * qq + w][d];
          sum += c[w];
        }
        S.part[qq][d] = sum;
        __syncthreads();
        uint32_t run = S.hist[d];
#pragma unroll
        for (int q = 0; q < 3; ++q) run += q < qq ? S.part[q][d] : 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          S.whist[8 * qq + w][d] = run;
          run += c[w];
        }
        __syncthreads();
        if (qq == 3) S.hist[d] = run;
      }
      __syncthreads();
      DSORT_MARK(22 + 3 * p);
#pragma unroll
      for (int it = 0; it < kDsortItems; ++it) {
        if (!ok[it]) continue;
        const uint32_t d = ((kk[it] - kbase) >> shift) & M;
        const uint32_t pos = S.whist[warp][d] + rk[it];
        if (p < P - 1 || LAST_KEYS) kout[pos] = kk[it];
        vout[pos] = vv[it];
        // next pass: this key belongs to the CTA that owns position pos
        if (next) {
          const uint32_t dn = ((kk[it] - kbase) >> (shift + DB)) & M;
          atomicAdd(next + (size_t)(pos / cs) * NW + (dn >> 1), 1u << (16 * (dn & 1u)));
          atomicAdd(&S.nexth[dn], 1u);
        }
      }
      __syncthreads();
    }
    if (next) {  // the next pass's digit totals
      for (int i = tid; i < NB; i += kDsortThreads) {
        if (S.nexth[i]) atomicAdd(gtot + (p + 1) * 512 + i, S.nexth[i]);
        S.nexth[i] = 0;
      }
    }
    DSORT_MARK(4 + 4 * p);
    kin = kout;
    vin = vout;
    kout = (kout == kB) ? kA : kB;
    vout = (vout == vB) ? vA : vB;
  }
  if (b == 0 && tid == 0) ctr->n_visible = nvis;
}

// Pass 0's histogram (raw 9-bit digits) and each CTA's smallest / largest binned key, one grid
// barrier, then the digit width: keys spanning fewer than 2^27 values -- depths within a
// factor of ~2^16 of each other -- are sorted in 3 passes of 9-bit digits over key - smallest,
// others in 4 passes of 8 bits (uniform over the grid: every CTA reduces the same [G][2]).
template <bool LAST_KEYS>
__global__ void __launch_bounds__(kDsortThreads, 1) dsort_kernel(
    const uint32_t* __restrict__ keys_all, uint32_t n_items, uint32_t* __restrict__ kA, uint32_t* __restrict__ vA,
    uint32_t* __restrict__ kB, uint32_t* __restrict__ vB, uint32_t* __restrict__ tables,
    Counters* __restrict__ ctr, uint32_t red_max, int force_bins) {
  extern __shared__ __align__(16) unsigned char dsort_smem[];
  DsortSmem& S = *reinterpret_cast<DsortSmem*>(dsort_smem);
  __shared__ uint32_t s_lo[kDsortWarps], s_hi[kDsortWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t ci = (n_items + G - 1) / G;
  uint32_t* gtot = tables + (size_t)3 * G * 256;
  uint32_t* mm = gtot + 4 * 512;
  uint32_t kk[kDsortItems];
  bool one;
  DSORT_MARK(0);
  {  // pass 0's histogram of this CTA's item range (valid keys, raw 9-bit digits) and key range
    const uint32_t lo = min(b * ci, n_items), hi = min(lo + ci, n_items);
    one = hi - lo <= (uint32_t)kDsortChunk;
    for (int i = tid; i < 512; i += kDsortThreads) {
      S.hist[i] = 0;
      S.nexth[i] = 0;
    }
    __syncthreads();
    uint32_t klo = 0xffffffffu, khi = 0;
    for (uint32_t base = lo; base < hi; base += kDsortChunk) {
      const uint32_t wbase = base + warp * 32 * kDsortItems;
#pragma unroll
      for (int it = 0; it < kDsortItems; ++it) {
        const uint32_t i = wbase + it * 32 + lane;
        kk[it] = i < hi ? __ldcg(keys_all + i) : kInvalidKey;
      }
#pragma unroll
      for (int it = 0; it < kDsortItems; ++it)
        if (kk[it] != kInvalidKey) {
          atomicAdd(&S.hist[kk[it] & 511u], 1u);
          klo = min(klo, kk[it]);
          khi = max(khi, kk[it]);
        }
    }
    klo = __reduce_min_sync(0xffffffffu, klo);
    khi = __reduce_max_sync(0xffffffffu, khi);
    if (lane == 0) {
      s_lo[warp] = klo;
      s_hi[warp] = khi;
    }
    __syncthreads();
    if (tid < 256) tables[(size_t)b * 256 + tid] = S.hist[2 * tid] | (S.hist[2 * tid + 1] << 16);
    if (tid < 512 && S.hist[tid]) atomicAdd(gtot + tid, S.hist[tid]);
    if (warp == 0) {
      const uint32_t l = __reduce_min_sync(0xffffffffu, s_lo[lane]), h = __reduce_max_sync(0xffffffffu, s_hi[lane]);
      if (lane == 0) {
        mm[2 * b] = l;
        mm[2 * b + 1] = h;
      }
    }
  }
  DSORT_MARK(1);
  grid_barrier(ctr->gbar, G);
  {  // the frame's key range: every CTA reduces the G pairs
    uint32_t l = 0xffffffffu, h = 0;
    for (uint32_t r = tid; r < G; r += kDsortThreads) {
      l = min(l, __ldcg(mm + 2 * r));
      h = max(h, __ldcg(mm + 2 * r + 1));
    }
    l = __reduce_min_sync(0xffffffffu, l);
    h = __reduce_max_sync(0xffffffffu, h);
    __syncthreads();  // s_lo / s_hi reuse
    if (lane == 0) {
      s_lo[warp] = l;
      s_hi[warp] = h;
    }
    __syncthreads();
  }
  uint32_t klo = 0xffffffffu, khi = 0;
#pragma unroll 8
  for (int w = 0; w < kDsortWarps; ++w) {
    klo = min(klo, s_lo[w]);
    khi = max(khi, s_hi[w]);
  }
  const bool nine = force_bins != 256 && (khi < klo || khi - klo < (1u << 27));
  if (nine)
    dsort_body<512, LAST_KEYS>(n_items, kA, vA, kB, vB, tables, ctr, red_max, khi >= klo ? klo : 0u, S, keys_all,
                               kk, one);
  else
    dsort_body<256, LAST_KEYS>(n_items, kA, vA, kB, vB, tables, ctr, red_max, 0u, S, keys_all, kk, one);
}

}  // namespace rs
