// blend64.cuh -- RS_F64 frames: per-tile front-to-back compositing in double,
// the reference's own expressions (render.py:250-281) and the importance max
// (render.py:273-275), bit-identical to the oracle's fp64 contract tier.
//
// Same tile / warp structure as blend2_kernel (blend.cuh): a 128-thread CTA per
// 16x16 tile in the blend order, warp w = 8x8 quarter (w%2, w/2), lane l = the
// pixels (l%8, l/8) and (l%8, l/8 + 4) -- one column, so the two pixels share
// dx and (ia dx) dx. Batches of 256 records (96-B Rec64) staged in shared
// memory, per-warp entry lists from the box x quarter overlap and the ellipse
// quarter masks (the binning's conservative fp32 region, which contains the
// fp64 region alpha >= alpha_cut), the per-pixel culling-box gate as one AND
// against the lane's column / row bits.
//
// Per pixel and Gaussian (render.py:254-281, with fused roundings):
//   x     = fma(nc dy, dy, fma(nb dy, dx, (na dx) dx))   (= -q/2; (na,nb,nc) = -(ia/2, ib, ic/2))
//   alpha = min(o exp(min(x, 709)), alpha_max)          (exp64_tab, rs_math.cuh: 1024-entry table)
//   if alpha >= alpha_cut and tau >= tau_stop:
//       w = alpha tau; rgb = fma(c, w, rgb); depth = fma(z, w, depth); count++;
//       tau = fma(-alpha, tau, tau)
// x < lnc (a conservative per-Gaussian bound) proves alpha < alpha_cut. A pixel
// that does not composite takes alpha = 0 (w = +0, fma(c, 0, rgb) = rgb, tau
// unchanged: exactly the skipped composite), so the loop has no branches. With
// FAST (alpha_cut >= 1e-300, alpha_max and tau_stop >= 0, lowpass >= 0) the threshold tests are
// integer compares of the fp64 bit patterns (the thresholds are non-negative, so
// the signed order of the bits is the value order) -- the FP64 pipe is the
// kernel's bound. Importance: the warp maximum of w's fp64 bits (two REDUX
// steps: high words, then low words among the lanes holding the maximal high
// word; w >= 0, so the unsigned order is the value order), one shared 64-bit
// atomicMax per (entry, group), one global atomicMax per (tile, Gaussian).
#pragma once
#include "rows.cuh"
#include "rs_common.cuh"
#include "rs_math.cuh"

namespace rs {

constexpr int kBlend64Threads = 128;

// a >= b / a > b for doubles with b >= 0 (not NaN): the signed order of the bit patterns
__device__ __forceinline__ bool ge_nn(double a, double b) { return __double_as_longlong(a) >= __double_as_longlong(b); }
__device__ __forceinline__ bool gt_nn(double a, double b) { return __double_as_longlong(a) > __double_as_longlong(b); }

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

#ifndef RS_BLEND64_MINB
#define RS_BLEND64_MINB 4  // 4 CTAs / SM: <= 128 registers (shared memory allows 4 as well)
#endif
template <bool COLOR, bool CONTRIB, bool STATS, bool FAST>
__global__ void __launch_bounds__(kBlend64Threads, RS_BLEND64_MINB) blend64_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_items, const Rec* __restrict__ recs,
    const Rec64* __restrict__ recs64, const float4* __restrict__ geom, const uint32_t* __restrict__ tile_order,
    Counters* __restrict__ ctr, int W, int H, int TW, Opt64 o, const Out64 out,
    unsigned long long* __restrict__ scores, const double* __restrict__ exp_table) {
  pdl_wait();
  pdl_trigger();
  constexpr int kBatch = 256;
  constexpr int kPerThread = kBatch / kBlend64Threads;
#ifndef RS_BLEND64_UNROLL_C
#define RS_BLEND64_UNROLL_C 2  // colour frames (measured 2: 303 us < 4: 332 < 6: 340 at configs[1])
#endif
#ifndef RS_BLEND64_UNROLL_S
#define RS_BLEND64_UNROLL_S 8  // score-only frames (measured 8: 426 us < 6: 435 < 4: 451 < 2: 495)
#endif
  constexpr int U = COLOR ? RS_BLEND64_UNROLL_C : RS_BLEND64_UNROLL_S;  // list entries per inner iteration
  __shared__ Rec64 s_rec[kBatch + 1];  // slot kBatch: empty-box sentinel padding the warp lists
  __shared__ unsigned long long s_w[CONTRIB ? kBatch + 1 : 1];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint16_t s_boxm[kBatch + 1][4];
  __shared__ uint16_t s_list[4][kBatch + U];
  __shared__ double s_exp[kExpTab];  // exp64_tab's 2^(j/1024) table

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = (int)__ldg(tile_order + blockIdx.x);
  const int tx = tile % TW, ty = tile / TW;
  const int ox = tx * kTile, oy = ty * kTile;
  const int px = ox + (warp & 1) * 8 + (lane & 7);
  const int py0 = oy + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
  const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
  const double xs = (double)px + 0.5, ys0 = (double)py0 + 0.5, ys1 = (double)py1 + 0.5;
  if (ctr->overflow) return;
  const uint2 rg = ranges[tile];
  const uint32_t npairs = ctr->n_pairs;
  const uint32_t end = rg.y < npairs ? rg.y : npairs;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t sel0 = (1u << (lane & 7)) | (1u << (8 + (lane >> 3)));
  const uint32_t sel1 = (1u << (lane & 7)) | (1u << (12 + (lane >> 3)));

  double tau0 = 1.0, tau1 = 1.0;
  double r0 = 0.0, g0 = 0.0, b0 = 0.0, d0 = 0.0, r1 = 0.0, g1 = 0.0, b1 = 0.0, d1 = 0.0;
  int cnt0 = 0, cnt1 = 0;
  unsigned long long evals = 0;
  for (int j = tid; j < kExpTab; j += kBlend64Threads) s_exp[j] = __ldg(exp_table + j);
  if (tid == 0) {
    Rec64 z{};
    s_rec[kBatch] = z;
#pragma unroll
    for (int w = 0; w < 4; ++w) s_boxm[kBatch][w] = 0;
    if (CONTRIB) s_w[kBatch] = 0ull;
  }
  const bool start = 1.0 >= o.tau_stop;
  bool done0 = !in0 || !start, done1 = !in1 || !start;

  for (uint32_t base = rg.x; base < end; base += kBatch) {
    if (__syncthreads_and(done0 && done1)) break;
    uint32_t gid[kPerThread];
#pragma unroll
    for (int h = 0; h < kPerThread; ++h) {
      gid[h] = 0u;
      const int slot = tid + h * kBlend64Threads;
      const uint32_t idx = base + slot;
      if (idx < end) {
        const uint32_t it = __ldg(pair_items + idx);
        const float4* R = reinterpret_cast<const float4*>(recs64 + it);
        float4* D = reinterpret_cast<float4*>(s_rec + slot);
        float4 v[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = __ldg(R + k);
#pragma unroll
        for (int k = 0; k < 6; ++k) D[k] = v[k];
        gid[h] = __float_as_uint(v[5].z);
        const float4 a = __ldg(&recs[it].a);
        const int4 dr = __ldg(&recs[it].d);
        const int4 d = cullbox_of(dr);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int qx = ox + (w & 1) * 8, qy = oy + (w >> 1) * 8;
          const int c0 = min(max(d.x - qx, 0), 8), c1 = min(max(d.y - qx, 0), 8);
          const int q0 = min(max(d.z - qy, 0), 8), q1 = min(max(d.w - qy, 0), 8);
          const uint32_t cm = ((1u << c1) - 1u) & ~((1u << c0) - 1u);
          const uint32_t rm = ((1u << q1) - 1u) & ~((1u << q0) - 1u);
          s_boxm[slot][w] = (uint16_t)(cm | (rm << 8));
        }
        const unsigned col = (d.x < ox + 8 && d.y > ox ? 1u : 0u) | (d.x < ox + 16 && d.y > ox + 8 ? 2u : 0u);
        unsigned m = 0;
        if (d.z < oy + 8 && d.w > oy) m |= col;
        if (d.z < oy + 16 && d.w > oy + 8) m |= col << 2;
        if (!STATS && cullbox_ell(dr) && (m & (m - 1u)))
          m = quarter_mask(load_row_geom(geom + 2 * (size_t)it, a.x, a.y), d, ox, oy);
        s_mask[slot] = (uint8_t)m;
      }
      if (CONTRIB) s_w[slot] = 0ull;
    }
    __syncthreads();
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
      for (int q = 0; q < cntw; q += U) {
        int ent[U];
#pragma unroll
        for (int u = 0; u < U; ++u) ent[u] = s_list[warp][q + u];
        // alpha of the U entries for both pixels (independent of tau)
        double al0[U], al1[U];
        bool ok0[U], ok1[U], bx0[U], bx1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Rec64& E = s_rec[ent[u]];
          const uint32_t bm = s_boxm[ent[u]][warp];
          bx0[u] = (bm & sel0) == sel0;
          bx1[u] = (bm & sel1) == sel1;
          const double dx = xs - E.mx;
          const double qa = (E.na * dx) * dx;
          const double dy0 = ys0 - E.my, dy1 = ys1 - E.my;
          const double x0 = __fma_rn(E.nc * dy0, dy0, __fma_rn(E.nb * dy0, dx, qa));
          const double x1 = __fma_rn(E.nc * dy1, dy1, __fma_rn(E.nb * dy1, dx, qa));
          const bool e0 = bx0[u] && x0 >= E.lnc, e1 = bx1[u] && x1 >= E.lnc;
          // evaluated for every lane (the values of skipped pixels are discarded)
          // the contract clamps the exp argument at 709; with FAST (lowpass >= 0: the conic is
          // positive definite, -q/2 <= 0 up to rounding) the clamp never binds
          const double xc0 = FAST ? x0 : (x0 > 709.0 ? 709.0 : x0), xc1 = FAST ? x1 : (x1 > 709.0 ? 709.0 : x1);
          const double raw0 = E.o * exp64_tab<FAST>(xc0, s_exp), raw1 = E.o * exp64_tab<FAST>(xc1, s_exp);
          double a0, a1;
          if (FAST) {
            a0 = gt_nn(raw0, o.alpha_max) ? o.alpha_max : raw0;
            a1 = gt_nn(raw1, o.alpha_max) ? o.alpha_max : raw1;
            ok0[u] = e0 && ge_nn(a0, o.alpha_cut);
            ok1[u] = e1 && ge_nn(a1, o.alpha_cut);
          } else {
            a0 = raw0 > o.alpha_max ? o.alpha_max : raw0;
            a1 = raw1 > o.alpha_max ? o.alpha_max : raw1;
            ok0[u] = e0 && a0 >= o.alpha_cut;
            ok1[u] = e1 && a1 >= o.alpha_cut;
          }
          al0[u] = a0;
          al1[u] = a1;
        }
        unsigned long long wmax[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Rec64& E = s_rec[ent[u]];
          const bool live0 = FAST ? ge_nn(tau0, o.tau_stop) : tau0 >= o.tau_stop;
          const bool live1 = FAST ? ge_nn(tau1, o.tau_stop) : tau1 >= o.tau_stop;
          if (STATS) evals += (unsigned)(bx0[u] && live0 && in0) + (unsigned)(bx1[u] && live1 && in1);
          const bool c0 = ok0[u] && live0, c1 = ok1[u] && live1;
          const double ae0 = c0 ? al0[u] : 0.0, ae1 = c1 ? al1[u] : 0.0;
          const double w0 = ae0 * tau0, w1 = ae1 * tau1;
          if (COLOR) {
            r0 = __fma_rn(E.r, w0, r0);
            g0 = __fma_rn(E.g, w0, g0);
            b0 = __fma_rn(E.b, w0, b0);
            d0 = __fma_rn(E.depth, w0, d0);
            r1 = __fma_rn(E.r, w1, r1);
            g1 = __fma_rn(E.g, w1, g1);
            b1 = __fma_rn(E.b, w1, b1);
            d1 = __fma_rn(E.depth, w1, d1);
          }
          tau0 = __fma_rn(-ae0, tau0, tau0);
          tau1 = __fma_rn(-ae1, tau1, tau1);
          cnt0 += c0 ? 1 : 0;
          cnt1 += c1 ? 1 : 0;
          wmax[u] = (unsigned long long)__double_as_longlong(w0 > w1 ? w0 : w1);
        }
        if (CONTRIB) {
          unsigned long long mine = 0;
          int slot = 0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const unsigned long long wm = warp_max_u64(wmax[u]);
            mine = lane == u ? wm : mine;
            slot = lane == u ? ent[u] : slot;
          }
          if (mine) atomicMax(&s_w[slot], mine);
        }
        done0 = !in0 || !(FAST ? ge_nn(tau0, o.tau_stop) : tau0 >= o.tau_stop);
        done1 = !in1 || !(FAST ? ge_nn(tau1, o.tau_stop) : tau1 >= o.tau_stop);
        if (__all_sync(0xffffffffu, done0 && done1)) break;
      }
    }
    __syncthreads();
    if (CONTRIB) {
#pragma unroll
      for (int h = 0; h < kPerThread; ++h) {
        const int slot = tid + h * kBlend64Threads;
        if (base + slot < end) {
          const unsigned long long v = s_w[slot];
          if (v) atomicMax(scores + gid[h], v);
        }
      }
    }
  }

  if (COLOR) {
    if (out.rgb) {
      if (in0) {
        const size_t p = (size_t)py0 * W + px;
        out.rgb[3 * p] = r0; out.rgb[3 * p + 1] = g0; out.rgb[3 * p + 2] = b0;
        out.alpha[p] = 1.0 - tau0;
        out.count[p] = cnt0;
      }
      if (in1) {
        const size_t p = (size_t)py1 * W + px;
        out.rgb[3 * p] = r1; out.rgb[3 * p + 1] = g1; out.rgb[3 * p + 2] = b1;
        out.alpha[p] = 1.0 - tau1;
        out.count[p] = cnt1;
      }
    }
    if (out.depth) {
      if (in0) out.depth[(size_t)py0 * W + px] = d0;
      if (in1) out.depth[(size_t)py1 * W + px] = d1;
    }
    if (out.rgb64) {
      // reference-typed images written straight to (mapped host) memory in whole tile rows,
      // staged through the free record slots (see blend2_kernel)
      __syncthreads();
      double* s_o = reinterpret_cast<double*>(s_rec);  // [0,768) rgb, [768,1024) alpha, [1024,1280) count
      const int lx = (warp & 1) * 8 + (lane & 7);
      const int l0 = ((warp >> 1) * 8 + (lane >> 3)) * kTile + lx, l1 = l0 + 4 * kTile;
      s_o[3 * l0] = r0; s_o[3 * l0 + 1] = g0; s_o[3 * l0 + 2] = b0;
      s_o[3 * l1] = r1; s_o[3 * l1 + 1] = g1; s_o[3 * l1 + 2] = b1;
      s_o[768 + l0] = 1.0 - tau0;
      s_o[768 + l1] = 1.0 - tau1;
      reinterpret_cast<long long*>(s_o)[1024 + l0] = (long long)cnt0;
      reinterpret_cast<long long*>(s_o)[1024 + l1] = (long long)cnt1;
      __syncthreads();
      const int cols = min(kTile, W - ox);
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int i = tid + k * kBlend64Threads;
        const int row = i / (3 * kTile), c = i - row * (3 * kTile);
        if (oy + row < H && c < 3 * cols) out.rgb64[((size_t)(oy + row) * W + ox) * 3 + c] = s_o[i];
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = tid + k * kBlend64Threads;
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

// exp64_tab's table, built once per workspace (rs_workspace_create)
__global__ void exp_table_kernel(double* __restrict__ t) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < kExpTab) t[j] = exp64_tab_entry(j);
}

}  // namespace rs
