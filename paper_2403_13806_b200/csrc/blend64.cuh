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
// Per pixel and Gaussian (render.py:254-281):
//   q     = (ia dx) dx + ((2 ib) dy) dx + (ic dy) dy
//   alpha = min(o exp(-q/2), alpha_max)            (exp64_contract, arg <= 709)
//   if alpha >= alpha_cut and tau >= tau_stop:
//       w = alpha tau; rgb = rgb + c w; depth = depth + z w; count++; tau = tau (1 - alpha)
// -q/2 < lnc (a conservative per-Gaussian bound) proves alpha < alpha_cut
// without the exp. Importance: the warp maximum of w's fp64 bits (two REDUX
// steps: high words, then low words among the lanes holding the maximal high
// word; w >= 0, so the unsigned order is the value order), one shared 64-bit
// atomicMax per (entry, group), one global atomicMax per (tile, Gaussian).
#pragma once
#include "rows.cuh"
#include "rs_common.cuh"
#include "rs_math.cuh"

namespace rs {

constexpr int kBlend64Threads = 128;

// e^x for x <= 709 (hot-loop form of exp64_contract): FAST = the caller
// guarantees x >= lnc >= ln(1e-300) - 1e-6, so the result is normal
template <bool FAST>
__device__ __forceinline__ double exp64_hot(double x) {
  if (!FAST) return exp64_contract(x);
  const double t = __fma_rn(x, kLog2e64, kMagic64);
  const double n = __dsub_rn(t, kMagic64);
  double r = __fma_rn(n, -kLn2Hi, x);
  r = __fma_rn(n, -kLn2Lo, r);
  return __dmul_rn(exp64_poly(r), pow2i64(__double2loint(t)));
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

template <bool COLOR, bool CONTRIB, bool STATS, bool FAST>
__global__ void __launch_bounds__(kBlend64Threads, 1) blend64_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_items, const Rec* __restrict__ recs,
    const Rec64* __restrict__ recs64, const float4* __restrict__ geom, const uint32_t* __restrict__ tile_order,
    Counters* __restrict__ ctr, int W, int H, int TW, Opt64 o, const Out64 out,
    unsigned long long* __restrict__ scores) {
  pdl_wait();
  pdl_trigger();
  constexpr int kBatch = 256;
  constexpr int kPerThread = kBatch / kBlend64Threads;
  constexpr int U = 4;  // list entries per inner iteration
  __shared__ Rec64 s_rec[kBatch + 1];  // slot kBatch: empty-box sentinel padding the warp lists
  __shared__ unsigned long long s_w[CONTRIB ? kBatch + 1 : 1];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint16_t s_boxm[kBatch + 1][4];
  __shared__ uint16_t s_list[4][kBatch + U];

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
          const double qa = (E.ia * dx) * dx;
          const double dy0 = ys0 - E.my, dy1 = ys1 - E.my;
          const double q0 = (qa + (E.ib2 * dy0) * dx) + (E.ic * dy0) * dy0;
          const double q1 = (qa + (E.ib2 * dy1) * dx) + (E.ic * dy1) * dy1;
          const double x0 = -0.5 * q0, x1 = -0.5 * q1;
          const bool e0 = bx0[u] && x0 >= E.lnc, e1 = bx1[u] && x1 >= E.lnc;
          double a0 = 0.0, a1 = 0.0;
          if (e0) {
            const double raw = E.o * exp64_hot<FAST>(fmin(x0, 709.0));
            a0 = raw > o.alpha_max ? o.alpha_max : raw;
          }
          if (e1) {
            const double raw = E.o * exp64_hot<FAST>(fmin(x1, 709.0));
            a1 = raw > o.alpha_max ? o.alpha_max : raw;
          }
          al0[u] = a0;
          al1[u] = a1;
          ok0[u] = e0 && a0 >= o.alpha_cut;
          ok1[u] = e1 && a1 >= o.alpha_cut;
        }
        unsigned long long wmax[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const Rec64& E = s_rec[ent[u]];
          const bool live0 = tau0 >= o.tau_stop, live1 = tau1 >= o.tau_stop;
          if (STATS) evals += (unsigned)(bx0[u] && live0 && in0) + (unsigned)(bx1[u] && live1 && in1);
          const bool c0 = ok0[u] && live0, c1 = ok1[u] && live1;
          double w0 = 0.0, w1 = 0.0;
          if (c0) {
            w0 = al0[u] * tau0;
            if (COLOR) {
              r0 = r0 + E.r * w0;
              g0 = g0 + E.g * w0;
              b0 = b0 + E.b * w0;
              d0 = d0 + E.depth * w0;
            }
            tau0 = tau0 * (1.0 - al0[u]);
            ++cnt0;
          }
          if (c1) {
            w1 = al1[u] * tau1;
            if (COLOR) {
              r1 = r1 + E.r * w1;
              g1 = g1 + E.g * w1;
              b1 = b1 + E.b * w1;
              d1 = d1 + E.depth * w1;
            }
            tau1 = tau1 * (1.0 - al1[u]);
            ++cnt1;
          }
          wmax[u] = (unsigned long long)__double_as_longlong(fmax(w0, w1));
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
        done0 = !in0 || tau0 < o.tau_stop;
        done1 = !in1 || tau1 < o.tau_stop;
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

}  // namespace rs
