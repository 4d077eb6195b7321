// blend.cuh -- per-tile front-to-back compositing (replaces render.py:246-283)
// and its importance-scoring variant (render.py:267, :273-275 + pruning.py:86-92).
//
// One 256-thread CTA per 16x16 tile, one thread per pixel; warp w owns the 8x4
// sub-rectangle (w%2, w/2). The tile's (depth, index)-ordered list is consumed
// in batches of 256 records: each thread stages one 64-byte record into shared
// memory with four 128-bit loads and tags it with the 8-bit set of warps whose
// sub-rectangle its bbox touches; each warp then compacts (ballot + popc) its
// own ordered entry list and walks only that, reading records as shared-memory
// broadcasts and stopping as soon as all 32 of its pixels have terminated. The
// per-pixel bbox gate (oracles.py:36-38) is still applied exactly.
//
// Per pixel and Gaussian (Tier-A contract, bit-identical to oracle/cpu_ref.cpp):
//   p2    = fma(na*dx, dx, fma(nb*dy, dx, (nc*dy)*dy))     (= -0.5*log2(e)*q)
//   alpha = min(o * 2^min(p2, 127), alpha_max)
//   if alpha >= alpha_cut and tau >= tau_stop:   (render.py:261)
//       w = alpha*tau; rgb += c*w; depth += z*w; count++; tau *= 1 - alpha
// Pixels leave the loop once tau < tau_stop (nothing can composite after
// that, render.py:261); the CTA stops when all 256 have (__syncthreads_and).
// p2 < cut2 (a conservative per-Gaussian bound) proves alpha < alpha_cut
// without evaluating 2^p2 -- the skip changes no result, only work.
//
// Importance: w is reduced across the warp with one REDUX.MAX on its fp32 bit
// pattern (w >= 0, so the unsigned order is the float order), lane 0 folds it
// into a per-batch shared slot, and each slot reaches the global score vector
// with one atomicMax per (tile, Gaussian) -- max-merge is order independent
// (render.py:71-76), so the result is deterministic.
#pragma once
#include "f32x2.cuh"
#include "rows.cuh"
#include "rs_common.cuh"
#include "rs_math.cuh"

namespace rs {

// FAST: the host guarantees alpha_cut >= 1e-30, so every evaluated p2 is >=
// cut2 >= -126 (projection clamps it) and, after the contract's clamp at 127,
// inside exp2_core's exact range: the range-checked exp2_contract is not needed.
template <bool COLOR, bool CONTRIB, bool STATS, bool FAST>
__global__ void __launch_bounds__(kBlendThreads) blend_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_items, const Rec* __restrict__ recs,
    Counters* __restrict__ ctr, int W, int H, int TW, Opt32 o, const Out32 out,
    uint32_t* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
  __shared__ Rec s_rec[kBlendThreads];  // one 64-byte record per entry: one base address per iteration
  __shared__ uint32_t s_w[CONTRIB ? kBlendThreads : 1];
  __shared__ uint8_t s_mask[kBlendThreads];             // which warps' 8x4 sub-rectangles the entry touches
  __shared__ uint8_t s_list[kBlendThreads / 32][kBlendThreads];  // per-warp compacted entry lists

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int tx = tile % TW, ty = tile / TW;
  const int ox = tx * kTile, oy = ty * kTile;
  const int px = ox + (warp & 1) * 8 + (lane & 7);
  const int py = oy + (warp >> 1) * 4 + (lane >> 3);
  const bool inside = px < W && py < H;
  const float xs = __fadd_rn((float)px, 0.5f), ys = __fadd_rn((float)py, 0.5f);
  if (ctr->overflow) return;  // pair list incomplete: the host re-runs with a larger capacity
  const uint2 rg = ranges[tile];
  const uint32_t npairs = ctr->n_pairs;
  const uint32_t end = rg.y < npairs ? rg.y : npairs;  // memory safety on overflow
  const uint32_t lt = (1u << lane) - 1u;

  float tau = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, cd = 0.0f;
  int cnt = 0;
  unsigned long long evals = 0;
  bool done = !inside || !(1.0f >= o.tau_stop);

  for (uint32_t base = rg.x; base < end; base += kBlendThreads) {
    if (__syncthreads_and(done)) break;
    const uint32_t idx = base + tid;
    uint32_t gid = 0;
    if (idx < end) {
      const Rec* R = recs + __ldg(pair_items + idx);
      s_rec[tid].a = __ldg(&R->a);
      s_rec[tid].b = __ldg(&R->b);
      const float4 c = __ldg(&R->c);
      if (COLOR || CONTRIB) s_rec[tid].c = c;
      gid = (uint32_t)__float_as_int(c.w);
      // gate with the culling box: inside the bbox, and only pixels that can reach alpha_cut
      // (skipping the per-pixel test for "tight" boxes measured slower: the test is cheap ALU)
      const int4 d = cullbox_of(__ldg(&R->d));
      s_rec[tid].d = d;
      // bbox x sub-rectangle overlap: 2 column halves x 4 row quarters -> bit w = (w%2, w/2)
      const unsigned col = (d.x < ox + 8 && d.y > ox ? 1u : 0u) | (d.x < ox + 16 && d.y > ox + 8 ? 2u : 0u);
      unsigned m = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (d.z < oy + 4 * r + 4 && d.w > oy + 4 * r) m |= col << (2 * r);
      s_mask[tid] = (uint8_t)m;
    }
    if (CONTRIB) s_w[tid] = 0u;
    __syncthreads();
    const int n = (int)min((uint32_t)kBlendThreads, end - base);
    if (!__all_sync(0xffffffffu, done)) {
      // this warp's entries, in list order
      int cntw = 0;
      for (int c0 = 0; c0 < n; c0 += 32) {
        const int e = c0 + lane;
        const bool has = e < n && ((s_mask[e] >> warp) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (has) s_list[warp][cntw + __popc(bal & lt)] = (uint8_t)e;
        cntw += __popc(bal);
      }
      __syncwarp();
      for (int q = 0; q < cntw; ++q) {
        const Rec& E = s_rec[s_list[warp][q]];
        const int4 bb = E.d;
        const bool in = !done && px >= bb.x && px < bb.y && py >= bb.z && py < bb.w;
        float w = 0.0f;
        if (in) {
          if (STATS) ++evals;
          const float4 ga = E.a;
          const float4 gb = E.b;
          const float dx = __fsub_rn(xs, ga.x), dy = __fsub_rn(ys, ga.y);
          const float p2 =
              __fmaf_rn(__fmul_rn(ga.z, dx), dx, __fmaf_rn(__fmul_rn(ga.w, dy), dx, __fmul_rn(__fmul_rn(gb.x, dy), dy)));
          if (p2 >= gb.z) {
            const float pc = fminf(p2, 127.0f);  // contract: exp2 argument clamped at 127 (oracle does the same)
            const float e = FAST ? exp2_core(pc) : exp2_contract(pc);
            const float alpha = fminf(__fmul_rn(gb.y, e), o.alpha_max);
            if (alpha >= o.alpha_cut) {
              w = __fmul_rn(alpha, tau);
              if (COLOR) {
                const float4 gc = E.c;
                cr = __fmaf_rn(gc.x, w, cr);
                cg = __fmaf_rn(gc.y, w, cg);
                cb = __fmaf_rn(gc.z, w, cb);
                cd = __fmaf_rn(gb.w, w, cd);
              }
              ++cnt;
              tau = __fmul_rn(tau, __fsub_rn(1.0f, alpha));
              done = tau < o.tau_stop;
            }
          }
        }
        if (CONTRIB) {
          const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(w));
          if (lane == 0 && wm) atomicMax(&s_w[s_list[warp][q]], wm);
        }
        if (__all_sync(0xffffffffu, done)) break;  // every pixel of the warp terminated
      }
    }
    __syncthreads();
    if (CONTRIB && idx < end) {
      const uint32_t v = s_w[tid];
      if (v) atomicMax(scores + gid, v);
    }
  }

  if (COLOR) {
    if (inside && out.rgb) {
      const size_t p = (size_t)py * W + px;
      out.rgb[3 * p] = cr;
      out.rgb[3 * p + 1] = cg;
      out.rgb[3 * p + 2] = cb;
      out.alpha[p] = __fsub_rn(1.0f, tau);
      out.count[p] = cnt;
    }
    if (inside && out.depth) out.depth[(size_t)py * W + px] = cd;
    if (out.rgb64) {
      // reference-typed images (float64 colour/alpha, int64 count; render.py:236-239, :283),
      // usually straight into mapped pinned host memory: stage the tile in shared memory
      // (the record slots are free after the loop) and write whole tile rows, so each warp
      // store is one contiguous run -- the host-link writes overlap the other tiles' blending
      __syncthreads();
      double* s_o = reinterpret_cast<double*>(s_rec);  // [0,768) rgb, [768,1024) alpha, [1024,1280) count
      const int lp = ((warp >> 1) * 4 + (lane >> 3)) * kTile + (warp & 1) * 8 + (lane & 7);
      s_o[3 * lp] = (double)cr;
      s_o[3 * lp + 1] = (double)cg;
      s_o[3 * lp + 2] = (double)cb;
      s_o[768 + lp] = (double)__fsub_rn(1.0f, tau);
      reinterpret_cast<long long*>(s_o)[1024 + lp] = (long long)cnt;
      __syncthreads();
      const int cols = min(kTile, W - ox);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int i = tid + k * kBlendThreads;  // 16 rows x 48 values
        const int row = i / (3 * kTile), c = i - row * (3 * kTile);
        if (oy + row < H && c < 3 * cols) out.rgb64[((size_t)(oy + row) * W + ox) * 3 + c] = s_o[i];
      }
      const int row = tid / kTile, c = tid % kTile;
      if (oy + row < H && c < cols) {
        const size_t p = (size_t)(oy + row) * W + ox + c;
        out.alpha64[p] = s_o[768 + tid];
        out.count64[p] = reinterpret_cast<const long long*>(s_o)[1024 + tid];
      }
    }
  }
  if (STATS) {
    unsigned long long c = (unsigned long long)cnt;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      evals += __shfl_down_sync(0xffffffffu, evals, off);
      c += __shfl_down_sync(0xffffffffu, c, off);
    }
    if (lane == 0) {
      atomicAdd(&ctr->evals, evals);
      atomicAdd(&ctr->composites, c);
    }
  }
}

// ---------------------------------------------------------------------------
// Two pixels per thread: 128-thread CTA per 16x16 tile, warp w owns the 8x8
// sub-rectangle (w%2, w/2), lane l the pixels (l%8, l/8) and (l%8, l/8 + 4) of
// it. Each entry of a warp's list is read from shared memory once and
// evaluated for both pixels (two independent dependency chains per thread),
// halving the per-entry overhead (list walk, record loads, vote, loop).
// Per-pixel arithmetic and decisions are exactly those of blend_kernel.
// ---------------------------------------------------------------------------
constexpr int kBlend2Threads = 128;
#ifndef RS_BLEND_UNROLL
#define RS_BLEND_UNROLL 6
#endif
constexpr int kBlendUnroll = RS_BLEND_UNROLL;  // list entries per inner iteration (measured: 2 -> 4 -> 6: -2..-6%, -1.5%)
// score-only frames (no colour state): 8 entries per iteration at >= 6 CTAs per SM (<= 80
// registers): configs[2] score blend 216.6 -> 208.0 us (colour frames: 156.7 -> 157.4, kept at 6 / 1)
#ifndef RS_BLEND_UNROLL_S
#define RS_BLEND_UNROLL_S 8
#endif
#ifndef RS_BLEND_MINB_S
#define RS_BLEND_MINB_S 6
#endif

// Record staging of blend2 (RS_BLEND_CPASYNC, colour frames): the {mx,my,na,nb} /
// {nc,o,cut2,depth} / colour quads go global -> shared with 16-byte cp.async (LDGSTS, no
// register round trip); only the box quad (and the row geometry for the quarter masks) is
// loaded into registers.
#ifndef RS_BLEND_CPASYNC
#define RS_BLEND_CPASYNC 1
#endif
__device__ __forceinline__ void stage16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <bool COLOR, bool STATS, bool FAST>
__device__ __forceinline__ float blend_px(const float4 ga, const float4 gb, const float4 gc, float xs, float ys,
                                          const Opt32& o, float& tau, float& cr, float& cg, float& cb,
                                          float& cd, int& cnt, bool& done, unsigned long long& evals) {
  if (STATS) ++evals;
  const float dx = __fsub_rn(xs, ga.x), dy = __fsub_rn(ys, ga.y);
  const float p2 =
      __fmaf_rn(__fmul_rn(ga.z, dx), dx, __fmaf_rn(__fmul_rn(ga.w, dy), dx, __fmul_rn(__fmul_rn(gb.x, dy), dy)));
  float w = 0.0f;
  if (p2 >= gb.z) {
    const float pc = fminf(p2, 127.0f);
    const float e = FAST ? exp2_core(pc) : exp2_contract(pc);
    const float alpha = fminf(__fmul_rn(gb.y, e), o.alpha_max);
    if (alpha >= o.alpha_cut) {
      w = __fmul_rn(alpha, tau);
      if (COLOR) {
        cr = __fmaf_rn(gc.x, w, cr);
        cg = __fmaf_rn(gc.y, w, cg);
        cb = __fmaf_rn(gc.z, w, cb);
        cd = __fmaf_rn(gb.w, w, cd);
      }
      ++cnt;
      tau = __fmul_rn(tau, __fsub_rn(1.0f, alpha));
      done = tau < o.tau_stop;
    }
  }
  return w;
}

// TRAIN: also record each pixel's final transmittance and last composited pair index
// (rs_outputs tau / last) for rs_backward.
template <bool COLOR, bool CONTRIB, bool STATS, bool FAST, bool TRAIN = false>
#ifndef RS_BLEND_MINB
#define RS_BLEND_MINB 1
#endif
__global__ void __launch_bounds__(kBlend2Threads, COLOR ? RS_BLEND_MINB : RS_BLEND_MINB_S) blend2_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_items, const Rec* __restrict__ recs,
    const float4* __restrict__ geom, const uint32_t* __restrict__ tile_order, Counters* __restrict__ ctr, int W,
    int H, int TW, Opt32 o, const Out32 out, uint32_t* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
#ifndef RS_BLEND_BATCH
#define RS_BLEND_BATCH 256
#endif
  constexpr int kBatch = RS_BLEND_BATCH;  // entries staged per batch
  constexpr int kPerThread = kBatch / kBlend2Threads;
  constexpr int U = COLOR ? kBlendUnroll : RS_BLEND_UNROLL_S;
  // cp.async record staging for colour frames (configs[1] blend 169.8 -> 168.9 us); score-only
  // frames keep the register path (1557 vs 1555 views/s with cp.async)
  constexpr bool kCp = RS_BLEND_CPASYNC && COLOR;
  // slot kBatch: an empty-box sentinel that pads every warp list to a multiple of U entries
  __shared__ Rec s_rec[kBatch + 1 > 160 ? kBatch + 1 : 160];  // >= 10 KB: the float64 epilogue's staging
  __shared__ uint32_t s_w[CONTRIB ? kBatch + 1 : 1];
  __shared__ uint8_t s_mask[kBatch];             // which warps' 8x8 sub-rectangles the entry touches
  // per entry and quarter: which of the quarter's 8 columns (bits 0-7) and 8 rows (8-15) lie in
  // the box -- a lane's box test is one AND against its own column and row bits
  __shared__ uint16_t s_boxm[kBatch + 1][4];
  __shared__ uint16_t s_list[4][kBatch + U];     // per-warp compacted entry lists (+ sentinel pad)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = (int)__ldg(tile_order + blockIdx.x);  // longest tile lists first
  const int tx = tile % TW, ty = tile / TW;
  const int ox = tx * kTile, oy = ty * kTile;
  const int px = ox + (warp & 1) * 8 + (lane & 7);
  const int py0 = oy + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
  const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
  const float xs = __fadd_rn((float)px, 0.5f);
  if (ctr->overflow) return;  // pair list incomplete: the host re-runs with a larger capacity
  const uint2 rg = ranges[tile];
  const uint32_t npairs = ctr->n_pairs;
  const uint32_t end = rg.y < npairs ? rg.y : npairs;  // memory safety on overflow
  const uint32_t lt = (1u << lane) - 1u;

  // per-pixel state of the thread's two pixels as packed pairs {py0, py1}
  f2 tau = f2_splat(1.0f), rgb[3] = {f2_splat(0.0f), f2_splat(0.0f), f2_splat(0.0f)}, dep = f2_splat(0.0f);
  const f2 ys2 = f2_pack(__fadd_rn((float)py0, 0.5f), __fadd_rn((float)py1, 0.5f));
  // this lane's column bit and row bits in s_boxm (pixel rows lane / 8 and lane / 8 + 4)
  const uint32_t sel0 = (1u << (lane & 7)) | (1u << (8 + (lane >> 3)));
  const uint32_t sel1 = (1u << (lane & 7)) | (1u << (12 + (lane >> 3)));
  int cnt0 = 0, cnt1 = 0;
  int last0 = -1, last1 = -1;  // pair index of each pixel's last composite (training outputs)
  unsigned long long evals = 0;
  if (tid == 0) {
    s_rec[kBatch].a = make_float4(0.f, 0.f, 0.f, 0.f);
    s_rec[kBatch].b = make_float4(0.f, 0.f, 0.f, 0.f);
    s_rec[kBatch].c = make_float4(0.f, 0.f, 0.f, 0.f);
    s_rec[kBatch].d = make_int4(0, 0, 0, 0);  // empty box: never evaluated
#pragma unroll
    for (int w = 0; w < 4; ++w) s_boxm[kBatch][w] = 0;
    if (CONTRIB) s_w[kBatch] = 0u;
  }
  const bool start = 1.0f >= o.tau_stop;
  bool done0 = !in0 || !start, done1 = !in1 || !start;

  for (uint32_t base = rg.x; base < end; base += kBatch) {
    if (__syncthreads_and(done0 && done1)) break;
    uint32_t gid[kPerThread];
#pragma unroll
    for (int h = 0; h < kPerThread; ++h) {
      gid[h] = 0u;
      const int slot = tid + h * kBlend2Threads;
      const uint32_t idx = base + slot;
      if (idx < end) {
        const uint32_t it = __ldg(pair_items + idx);
        const Rec* R = recs + it;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (kCp) {
          stage16(&s_rec[slot].a, &R->a);
          stage16(&s_rec[slot].b, &R->b);
          stage16(&s_rec[slot].c, &R->c);
        } else {
          a = __ldg(&R->a);
          s_rec[slot].a = a;
          s_rec[slot].b = __ldg(&R->b);
          const float4 c = __ldg(&R->c);
          if (COLOR || CONTRIB) s_rec[slot].c = c;
          gid[h] = (uint32_t)__float_as_int(c.w);
        }
        const int4 dr = __ldg(&R->d);
        const int4 d = cullbox_of(dr);  // only as the s_boxm bits below (the walk never reads E.d)
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int qx = ox + (w & 1) * 8, qy = oy + (w >> 1) * 8;
          const int c0 = min(max(d.x - qx, 0), 8), c1 = min(max(d.y - qx, 0), 8);
          const int r0 = min(max(d.z - qy, 0), 8), r1 = min(max(d.w - qy, 0), 8);
          const uint32_t cm = ((1u << c1) - 1u) & ~((1u << c0) - 1u);
          const uint32_t rm = ((1u << r1) - 1u) & ~((1u << r0) - 1u);
          s_boxm[slot][w] = (uint16_t)(cm | (rm << 8));
        }
        // box x sub-rectangle overlap: 2 column halves x 2 row halves -> bit w = (w%2, w/2)
        const unsigned col = (d.x < ox + 8 && d.y > ox ? 1u : 0u) | (d.x < ox + 16 && d.y > ox + 8 ? 2u : 0u);
        unsigned m = 0;
        if (d.z < oy + 8 && d.w > oy) m |= col;
        if (d.z < oy + 16 && d.w > oy + 8) m |= col << 2;
        if (!STATS && cullbox_ell(dr) && (m & (m - 1u))) {
          // a box over several quarters: the ones the ellipse strips of the tile's two half-rows
          // reach -- a warp whose quarter no pixel of the entry can composite in never walks it
          // (STATS keeps the box quarters: every in-box pixel is evaluated, the oracle's E count)
          RowGeom g = load_row_geom(geom + 2 * (size_t)it, a.x, a.y);
          if constexpr (kCp) {
            stage_wait();  // this thread's own copies: mx, my readable from its slot
            g.mx = s_rec[slot].a.x;
            g.my = s_rec[slot].a.y;
          }
          m = quarter_mask(g, d, ox, oy);
        }
        s_mask[slot] = (uint8_t)m;
      }
      if (CONTRIB) s_w[slot] = 0u;
    }
    if constexpr (kCp) stage_wait();
    __syncthreads();
    if constexpr (kCp && CONTRIB) {
#pragma unroll
      for (int h = 0; h < kPerThread; ++h) {
        const int slot = tid + h * kBlend2Threads;
        gid[h] = base + slot < end ? (uint32_t)__float_as_int(s_rec[slot].c.w) : 0u;
      }
    }
    const int n = (int)min((uint32_t)kBatch, end - base);
    if (!__all_sync(0xffffffffu, done0 && done1)) {
      int cntw = 0;
      for (int c0 = 0; c0 < n; c0 += 32) {
        const int e = c0 + lane;
        const bool has = e < n && ((s_mask[e] >> warp) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (has) s_list[warp][cntw + __popc(bal & lt)] = (uint16_t)e;
        cntw += __popc(bal);
      }
      if (lane < U) s_list[warp][cntw + lane] = (uint16_t)kBatch;
      __syncwarp();
      // kBlendUnroll entries per iteration: all their coverage and alpha math (independent of
      // the transmittance) first, then the composites in list order -- independent dependency
      // chains per thread and one termination vote per group of entries. Values
      // computed for a pixel that is not composited are discarded by the selects, so the
      // decisions and results are exactly those of blend_px (the FAST exp2 is exact on
      // [-126, 127] and only p2 >= cut2 >= -126 is ever used).
      for (int q = 0; q < cntw; q += U) {
        int ent[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ent[u] = s_list[warp][q + u];
        // the two pixels (rows py0, py1) in packed fp32 pairs: every FADD2/FMUL2/FFMA2 below is
        // the scalar contract's operation on both pixels at once (f32x2.cuh)
        f2 al[U];
        bool ok[U][2], box[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Rec& E = s_rec[ent[u]];
          const float4 ga = E.a, gb = E.b;
          const uint32_t bm = s_boxm[ent[u]][warp];
          box[u][0] = (bm & sel0) == sel0;
          box[u][1] = (bm & sel1) == sel1;
          const float dx = __fsub_rn(xs, ga.x);
          const float ax = __fmul_rn(ga.z, dx);
          const f2 dy = f2_sub(ys2, f2_splat(ga.y));
          // p2 = fma(ax, dx, fma(nb*dy, dx, (nc*dy)*dy))
          const f2 t3 = f2_mul(f2_mul(f2_splat(gb.x), dy), dy);
          const f2 p2 = f2_fma(f2_splat(ax), f2_splat(dx), f2_fma(f2_mul(f2_splat(ga.w), dy), f2_splat(dx), t3));
          const float p20 = f2_lo(p2), p21 = f2_hi(p2);
          // exp2_core(min(p2, 127)) (rs_math.cuh) on the pair
          f2 ex;
          if (FAST) {
            const f2 x = f2_pack(fminf(p20, 127.0f), fminf(p21, 127.0f));
            const f2 t = f2_add(x, f2_splat(kMagic));
            const f2 r = f2_sub(x, f2_sub(t, f2_splat(kMagic)));
            const f2 sc = f2_exp2_scale(t);
            f2 pp = f2_fma(f2_splat(fbits(0x3920e999u)), r, f2_splat(fbits(0x3aafa2b5u)));
            pp = f2_fma(pp, r, f2_splat(fbits(0x3c1d96deu)));
            pp = f2_fma(pp, r, f2_splat(fbits(0x3d63576au)));
            pp = f2_fma(pp, r, f2_splat(fbits(0x3e75fdedu)));
            pp = f2_fma(pp, r, f2_splat(fbits(0x3f317218u)));
            pp = f2_fma(pp, r, f2_splat(1.0f));
            ex = f2_mul(pp, sc);
          } else {
            ex = f2_pack(exp2_contract(fminf(p20, 127.0f)), exp2_contract(fminf(p21, 127.0f)));
          }
          const f2 av = f2_mul(f2_splat(gb.y), ex);
          const float a0 = fminf(f2_lo(av), o.alpha_max), a1 = fminf(f2_hi(av), o.alpha_max);
          al[u] = f2_pack(a0, a1);
          ok[u][0] = box[u][0] && p20 >= gb.z && a0 >= o.alpha_cut;
          ok[u][1] = box[u][1] && p21 >= gb.z && a1 >= o.alpha_cut;
        }
        float wmax[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Rec& E = s_rec[ent[u]];
          // a pixel composites iff tau_before >= tau_stop (render.py:261); out-of-image pixels
          // never pass the box test. Colour frames take a non-compositing pixel's alpha as 0
          // (w = 0 * tau = +0, tau * (1 - 0) = tau: exactly the skipped composite, fewer
          // selects); score-only frames select the products instead (a shorter dependency
          // chain through tau, which their lighter loop cannot hide)
          const bool live0 = COLOR ? f2_lo(tau) >= o.tau_stop : !done0;
          const bool live1 = COLOR ? f2_hi(tau) >= o.tau_stop : !done1;
          if (STATS) evals += (unsigned)(box[u][0] && live0 && in0) + (unsigned)(box[u][1] && live1 && in1);
          const bool c0 = ok[u][0] && live0, c1 = ok[u][1] && live1;
          f2 wt;
          if (COLOR) {
            const f2 ae = f2_pack(c0 ? f2_lo(al[u]) : 0.0f, c1 ? f2_hi(al[u]) : 0.0f);
            wt = f2_mul(ae, tau);
            const float4 gc = E.c;
            rgb[0] = f2_fma(f2_splat(gc.x), wt, rgb[0]);
            rgb[1] = f2_fma(f2_splat(gc.y), wt, rgb[1]);
            rgb[2] = f2_fma(f2_splat(gc.z), wt, rgb[2]);
            dep = f2_fma(f2_splat(E.b.w), wt, dep);
            tau = f2_mul(tau, f2_sub(f2_splat(1.0f), ae));
          } else {
            const f2 wp = f2_mul(al[u], tau);
            wt = f2_pack(c0 ? f2_lo(wp) : 0.0f, c1 ? f2_hi(wp) : 0.0f);
            const f2 tn = f2_mul(tau, f2_sub(f2_splat(1.0f), al[u]));
            tau = f2_pack(c0 ? f2_lo(tn) : f2_lo(tau), c1 ? f2_hi(tn) : f2_hi(tau));
            done0 = done0 || f2_lo(tau) < o.tau_stop;
            done1 = done1 || f2_hi(tau) < o.tau_stop;
          }
          const float w0 = f2_lo(wt), w1 = f2_hi(wt);
          cnt0 += c0 ? 1 : 0;
          cnt1 += c1 ? 1 : 0;
          if (TRAIN) {
            const int k = (int)base + ent[u];
            last0 = c0 ? k : last0;
            last1 = c1 ? k : last1;
          }
          wmax[u] = fmaxf(w0, w1);
        }
        if (CONTRIB) {
          // the group's U warp maxima, lane u folding entry u's into the batch slot: one
          // shared atomic instruction per group instead of U
          uint32_t mine = 0;
          int slot = 0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(wmax[u]));
            mine = lane == u ? wm : mine;
            slot = lane == u ? ent[u] : slot;
          }
          if (mine) atomicMax(&s_w[slot], mine);
        }
        if (COLOR) {
          done0 = !in0 || f2_lo(tau) < o.tau_stop;
          done1 = !in1 || f2_hi(tau) < o.tau_stop;
        }
        if (__all_sync(0xffffffffu, done0 && done1)) break;  // all 64 pixels of the warp terminated
      }
    }
    // the batch's score slots are complete once every warp has walked it; without scores the
    // next batch's __syncthreads_and is the barrier before the slots are restaged
    if (CONTRIB) __syncthreads();
    if (CONTRIB) {
#pragma unroll
      for (int h = 0; h < kPerThread; ++h) {
        const int slot = tid + h * kBlend2Threads;
        if (base + slot < end) {
          const uint32_t v = s_w[slot];
          if (v) atomicMax(scores + gid[h], v);
        }
      }
    }
  }

  const float tau0 = f2_lo(tau), tau1 = f2_hi(tau);
  const float r0 = f2_lo(rgb[0]), g0 = f2_lo(rgb[1]), b0 = f2_lo(rgb[2]), d0 = f2_lo(dep);
  const float r1 = f2_hi(rgb[0]), g1 = f2_hi(rgb[1]), b1 = f2_hi(rgb[2]), d1 = f2_hi(dep);
  if (COLOR) {
    if (out.rgb) {
      if (in0) {
        const size_t p = (size_t)py0 * W + px;
        out.rgb[3 * p] = r0; out.rgb[3 * p + 1] = g0; out.rgb[3 * p + 2] = b0;
        out.alpha[p] = __fsub_rn(1.0f, tau0);
        out.count[p] = cnt0;
      }
      if (in1) {
        const size_t p = (size_t)py1 * W + px;
        out.rgb[3 * p] = r1; out.rgb[3 * p + 1] = g1; out.rgb[3 * p + 2] = b1;
        out.alpha[p] = __fsub_rn(1.0f, tau1);
        out.count[p] = cnt1;
      }
    }
    if (out.depth) {
      if (in0) out.depth[(size_t)py0 * W + px] = d0;
      if (in1) out.depth[(size_t)py1 * W + px] = d1;
    }
    if (TRAIN) {
      if (in0) { out.tau[(size_t)py0 * W + px] = tau0; out.last[(size_t)py0 * W + px] = last0; }
      if (in1) { out.tau[(size_t)py1 * W + px] = tau1; out.last[(size_t)py1 * W + px] = last1; }
    }
    if (out.rgb64) {
      // reference-typed images written straight to (mapped host) memory in whole tile rows,
      // staged through the free record slots (see blend_kernel)
      __syncthreads();
      double* s_o = reinterpret_cast<double*>(s_rec);  // [0,768) rgb, [768,1024) alpha, [1024,1280) count
      const int lx = (warp & 1) * 8 + (lane & 7);
      const int l0 = ((warp >> 1) * 8 + (lane >> 3)) * kTile + lx, l1 = l0 + 4 * kTile;
      s_o[3 * l0] = (double)r0; s_o[3 * l0 + 1] = (double)g0; s_o[3 * l0 + 2] = (double)b0;
      s_o[3 * l1] = (double)r1; s_o[3 * l1 + 1] = (double)g1; s_o[3 * l1 + 2] = (double)b1;
      s_o[768 + l0] = (double)__fsub_rn(1.0f, tau0);
      s_o[768 + l1] = (double)__fsub_rn(1.0f, tau1);
      reinterpret_cast<long long*>(s_o)[1024 + l0] = (long long)cnt0;
      reinterpret_cast<long long*>(s_o)[1024 + l1] = (long long)cnt1;
      __syncthreads();
      const int cols = min(kTile, W - ox);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int i = tid + k * kBlend2Threads;  // 16 rows x 48 values
        const int row = i / (3 * kTile), c = i - row * (3 * kTile);
        if (oy + row < H && c < 3 * cols) out.rgb64[((size_t)(oy + row) * W + ox) * 3 + c] = s_o[i];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = tid + k * kBlend2Threads;
        const int row = i / kTile, c = i % kTile;
        if (oy + row < H && c < cols) {
          const size_t p = (size_t)(oy + row) * W + ox + c;
          out.alpha64[p] = s_o[768 + i];
          out.count64[p] = reinterpret_cast<const long long*>(s_o)[1024 + i];
        }
      }
    }
  }
  if (STATS) {
    unsigned long long c = (unsigned long long)(cnt0 + cnt1);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      evals += __shfl_down_sync(0xffffffffu, evals, off);
      c += __shfl_down_sync(0xffffffffu, c, off);
    }
    if (lane == 0) {
      atomicAdd(&ctr->evals, evals);
      atomicAdd(&ctr->composites, c);
    }
  }
}

}  // namespace rs
