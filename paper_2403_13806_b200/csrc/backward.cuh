// backward.cuh -- analytic gradients through the rendered image (SURVEY §8f
// next #1; replaces render.py:328-394 rasterize_backward and :397-487
// _chain_to_parameters).
//
// Training forward (rs_render_ex with rs_outputs tau / last) leaves, per pixel,
// the final transmittance and the pair index of its last composite. Then:
//   backward2_kernel  one 128-thread CTA per tile, two pixels per thread, walks
//       the tile's list BACK to front (batches of 256 staged in shared memory,
//       per-warp entry lists by ellipse quarters as in blend2_kernel; FAST =
//       alpha_cut >= 1e-30: the exact-range exp2 core). For each entry the pixel
//       composited in the forward pass (index <= last, inside the box, alpha >=
//       alpha_cut -- the same fp32 alpha), tau_before = tau / (1 - alpha) and,
//       as render.py:366-391: weight = alpha tau_before, g_color += weight g,
//       d_alpha = tau_before (c.g) - suffix / (1 - alpha) (0 when alpha was
//       clamped), dq = -0.5 alpha d_alpha, suffix += weight (c.g). Per entry the
//       warp reduces its lanes' nine partial sums (both pixels added first) (g_color, sum d_alpha alpha,
//       sum dq dx, sum dq dy, sum dq dx^2, sum dq 2 dx dy, sum dq dy^2) and lane 0
//       adds them to the item's screen-space gradient (atomicAdd).
//   chain_kernel  one thread per item: recomputes the projection intermediates
//       from the scene parameters and chains the screen-space gradient to
//       positions, SH, log-scales, quaternions (through the normalization) and
//       opacity logits exactly as render.py:397-487, plus |dL/dmean2d| and the
//       touched flag.
// fp32 throughout; the per-Gaussian sums are atomics (order-dependent rounding),
// so parity with the fp64 reference is a tolerance, not bit equality.
#pragma once
#include "f32x2.cuh"
#include "rows.cuh"
#include "rs_common.cuh"
#include "rs_math.cuh"

namespace rs {

constexpr int kSGrad = 9;  // screen-space gradient words per item

// Two pixels per thread (rows py0, py0 + 4 of the warp's 8x8 quarter, as blend2_kernel),
// 128-thread CTA per tile, batches of 256 records walked back to front. The forward's
// composite decision (p2, alpha) is recomputed with blend2_kernel's packed contract ops, so
// it is the forward's bit for bit; the gradient arithmetic after it is fp32 (tolerance).
// Per entry the two pixels' nine partial sums are added before one warp reduce-scatter.
constexpr int kBwd2Threads = 128;
template <bool FAST>
__global__ void __launch_bounds__(kBwd2Threads) backward2_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ pair_items, const Rec* __restrict__ recs,
    const float4* __restrict__ geom, const uint32_t* __restrict__ tile_order, const Counters* __restrict__ ctr,
    int W, int H, int TW, Opt32 o, const float* __restrict__ grad_image, const float* __restrict__ tau_final, const int32_t* __restrict__ last,
    float* __restrict__ sgrad, uint8_t* __restrict__ touched) {
  pdl_wait();
  pdl_trigger();
  constexpr int kBatch = 256;
  __shared__ Rec s_rec[kBatch];
  __shared__ uint32_t s_item[kBatch];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint16_t s_boxm[kBatch][4];  // per quarter: box columns (bits 0-7) and rows (8-15)
  __shared__ uint8_t s_list[4][kBatch];
  __shared__ int s_maxlast[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = (int)__ldg(tile_order + blockIdx.x);  // longest tile lists first
  const int tx = tile % TW, ty = tile / TW;
  const int ox = tx * kTile, oy = ty * kTile;
  const int px = ox + (warp & 1) * 8 + (lane & 7);
  const int py0 = oy + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
  const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
  const float xs = __fadd_rn((float)px, 0.5f);
  const f2 ys2 = f2_pack(__fadd_rn((float)py0, 0.5f), __fadd_rn((float)py1, 0.5f));
  const uint32_t sel0 = (1u << (lane & 7)) | (1u << (8 + (lane >> 3)));
  const uint32_t sel1 = (1u << (lane & 7)) | (1u << (12 + (lane >> 3)));
  if (ctr->overflow) return;
  const uint2 rg = ranges[tile];
  const uint32_t end = min(rg.y, ctr->n_pairs);
  const uint32_t lt = (1u << lane) - 1u;
  float tau[2] = {1.0f, 1.0f}, gcol[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
  int lastk[2] = {-1, -1};
  const bool inside[2] = {in0, in1};
  const int pyv[2] = {py0, py1};
#pragma unroll
  for (int j = 0; j < 2; ++j)
    if (inside[j]) {
      const size_t p = (size_t)pyv[j] * W + px;
      tau[j] = tau_final[p];
      lastk[j] = last[p];
      gcol[j][0] = grad_image[3 * p];
      gcol[j][1] = grad_image[3 * p + 1];
      gcol[j][2] = grad_image[3 * p + 2];
    }
  // the two pixels' state as packed pairs {py0, py1}
  f2 tau2 = f2_pack(tau[0], tau[1]), suffix2 = f2_splat(0.0f);
  const f2 gcol2[3] = {f2_pack(gcol[0][0], gcol[1][0]), f2_pack(gcol[0][1], gcol[1][1]),
                       f2_pack(gcol[0][2], gcol[1][2])};
  // entries after every pixel's last composite are skipped wholesale
  int maxlast = max(lastk[0], lastk[1]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) maxlast = max(maxlast, __shfl_xor_sync(0xffffffffu, maxlast, off));
  if (lane == 0) s_maxlast[warp] = maxlast;
  __syncthreads();
  const int cta_last = max(max(s_maxlast[0], s_maxlast[1]), max(s_maxlast[2], s_maxlast[3]));
  const uint32_t stop = cta_last < 0 ? rg.x : min(end, (uint32_t)cta_last + 1u);

  for (uint32_t top = stop; top > rg.x;) {
    const uint32_t base = top - min((uint32_t)kBatch, top - rg.x);
    const int n = (int)(top - base);
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int slot = tid + h * kBwd2Threads;
      if (slot < n) {
        const uint32_t it = __ldg(pair_items + base + slot);
        const Rec* R = recs + it;
        const float4 a = __ldg(&R->a);
        s_rec[slot].a = a;
        s_rec[slot].b = __ldg(&R->b);
        s_rec[slot].c = __ldg(&R->c);
        const int4 dr = __ldg(&R->d);
        const int4 d = cullbox_of(dr);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int qx = ox + (w & 1) * 8, qy = oy + (w >> 1) * 8;
          const int c0 = min(max(d.x - qx, 0), 8), c1 = min(max(d.y - qx, 0), 8);
          const int r0 = min(max(d.z - qy, 0), 8), r1 = min(max(d.w - qy, 0), 8);
          const uint32_t cm = ((1u << c1) - 1u) & ~((1u << c0) - 1u);
          const uint32_t rm = ((1u << r1) - 1u) & ~((1u << r0) - 1u);
          s_boxm[slot][w] = (uint16_t)(cm | (rm << 8));
        }
        s_item[slot] = it;
        // the 8x8 quarters the entry can composite in (blend2_kernel's warp lists)
        unsigned m;
        if (cullbox_ell(dr)) {
          m = quarter_mask(load_row_geom(geom + 2 * (size_t)it, a.x, a.y), d, ox, oy);
        } else {
          const unsigned col = (d.x < ox + 8 && d.y > ox ? 1u : 0u) | (d.x < ox + 16 && d.y > ox + 8 ? 2u : 0u);
          m = 0;
          if (d.z < oy + 8 && d.w > oy) m |= col;
          if (d.z < oy + 16 && d.w > oy + 8) m |= col << 2;
        }
        s_mask[slot] = (uint8_t)m;
      }
    }
    __syncthreads();
    int cntw = 0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int e = c0 + lane;
      const bool has = e < n && ((s_mask[e] >> warp) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, has);
      if (has) s_list[warp][cntw + __popc(bal & lt)] = (uint8_t)e;
      cntw += __popc(bal);
    }
    __syncwarp();
    for (int q = cntw - 1; q >= 0; --q) {
      const int e = s_list[warp][q];
      const Rec& E = s_rec[e];
      const float4 ga = E.a, gb4 = E.b;
      const int k = (int)base + e;
      const uint32_t bm = s_boxm[e][warp];
      const bool cand0 = k <= lastk[0] && (bm & sel0) == sel0;  // (out-of-image pixels: lastk -1)
      const bool cand1 = k <= lastk[1] && (bm & sel1) == sel1;
      if (!__any_sync(0xffffffffu, cand0 || cand1)) continue;
      // the forward's p2 / alpha (blend2_kernel's operations)
      const float dx = __fsub_rn(xs, ga.x);
      const float ax = __fmul_rn(ga.z, dx);
      const f2 dy2 = f2_sub(ys2, f2_splat(ga.y));
      const f2 t3 = f2_mul(f2_mul(f2_splat(gb4.x), dy2), dy2);
      const f2 p2 = f2_fma(f2_splat(ax), f2_splat(dx), f2_fma(f2_mul(f2_splat(ga.w), dy2), f2_splat(dx), t3));
      const float p20 = f2_lo(p2), p21 = f2_hi(p2);
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
      const f2 raw2 = f2_mul(f2_splat(gb4.y), ex);
      const float a0 = fminf(f2_lo(raw2), o.alpha_max), a1 = fminf(f2_hi(raw2), o.alpha_max);
      // composited in the forward pass (same decisions as blend2_kernel)
      const bool c0 = cand0 && p20 >= gb4.z && a0 >= o.alpha_cut;
      const bool c1 = cand1 && p21 >= gb4.z && a1 >= o.alpha_cut;
      const bool comp = c0 || c1;
      float v[kSGrad];
      if (__any_sync(0xffffffffu, comp)) {
        // both pixels' gradient terms as packed pairs (tolerance path: fp32, any association)
        // a pixel that did not composite gets alpha 0 (its p2 may lie outside the exp2 core's
        // exact range: garbage there must not reach the sums)
        const f2 al = f2_pack(c0 ? a0 : 0.0f, c1 ? a1 : 0.0f);
        const f2 om = f2_sub(f2_splat(1.0f), al);
        float r0, r1;  // 1 / (1 - alpha), alpha <= alpha_max < 1: the hardware reciprocal
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(f2_lo(om)));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(f2_hi(om)));
        const f2 rom = f2_pack(r0, r1);
        const f2 tb = f2_mul(tau2, rom);
        const f2 w = f2_mul(al, tb);
        const float4 gc = E.c;
        const f2 cdot = f2_fma(f2_splat(gc.z), gcol2[2], f2_fma(f2_splat(gc.y), gcol2[1], f2_mul(f2_splat(gc.x), gcol2[0])));
        const f2 wg0 = f2_mul(w, gcol2[0]), wg1 = f2_mul(w, gcol2[1]), wg2 = f2_mul(w, gcol2[2]);
        v[0] = f2_lo(wg0) + f2_hi(wg0);
        v[1] = f2_lo(wg1) + f2_hi(wg1);
        v[2] = f2_lo(wg2) + f2_hi(wg2);
        const f2 dar = f2_sub(f2_mul(tb, cdot), f2_mul(suffix2, rom));
        // d_alpha (0 where alpha was clamped at alpha_max, or no composite)
        const f2 da = f2_pack(c0 && f2_lo(raw2) <= o.alpha_max ? f2_lo(dar) : 0.0f,
                              c1 && f2_hi(raw2) <= o.alpha_max ? f2_hi(dar) : 0.0f);
        const f2 daa = f2_mul(da, al);
        v[3] = f2_lo(daa) + f2_hi(daa);
        const f2 dq = f2_mul(f2_mul(f2_splat(-0.5f), al), da);
        const f2 dqy = f2_mul(dq, dy2), dqyy = f2_mul(dqy, dy2);
        const float sdq = f2_lo(dq) + f2_hi(dq), sdqy = f2_lo(dqy) + f2_hi(dqy);
        v[4] = sdq * dx;
        v[5] = sdqy;
        v[6] = sdq * (dx * dx);
        v[7] = 2.0f * dx * sdqy;
        v[8] = f2_lo(dqyy) + f2_hi(dqyy);
        suffix2 = f2_fma(w, cdot, suffix2);
        tau2 = f2_pack(c0 ? f2_lo(tb) : f2_lo(tau2), c1 ? f2_hi(tb) : f2_hi(tau2));
        // reduce-scatter of v[0..7] (4 + 2 + 1 + 1 + 1 shuffles), v[8] by a butterfly
        const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
        float w4[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float r = __shfl_xor_sync(0xffffffffu, b4 ? v[kk] : v[4 + kk], 16);
          w4[kk] = (b4 ? v[4 + kk] : v[kk]) + r;
        }
        float w2[2];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const float r = __shfl_xor_sync(0xffffffffu, b3 ? w4[kk] : w4[2 + kk], 8);
          w2[kk] = (b3 ? w4[2 + kk] : w4[kk]) + r;
        }
        float w1 = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], 4);
        w1 += __shfl_xor_sync(0xffffffffu, w1, 2);
        w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
        float v8 = v[8];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v8 += __shfl_xor_sync(0xffffffffu, v8, off);
        const uint32_t it = s_item[e];
        float* g = sgrad + (size_t)kSGrad * it;
        if ((lane & 3) == 0) atomicAdd(g + (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0), w1);
        if (lane == 0) {
          atomicAdd(g + 8, v8);
          touched[it] = 1;
        }
      }
    }
    top = base;
  }
}

// dL/dR -> dL/dq for a unit quaternion (core.py:142-163)
__device__ __forceinline__ void quat_rotmat_backward(const float q[4], const float g[9], float out[4]) {
  const float w = q[0], x = q[1], y = q[2], z = q[3];
  out[0] = 2.0f * (-z * g[1] + y * g[2] + z * g[3] - x * g[5] - y * g[6] + x * g[7]);
  out[1] = 2.0f * (y * g[1] + z * g[2] + y * g[3] - 2.0f * x * g[4] - w * g[5] + z * g[6] + w * g[7] - 2.0f * x * g[8]);
  out[2] = 2.0f * (-2.0f * y * g[0] + x * g[1] + w * g[2] + x * g[3] + z * g[5] - w * g[6] + z * g[7] - 2.0f * y * g[8]);
  out[3] = 2.0f * (-2.0f * z * g[0] - w * g[1] + x * g[2] + w * g[3] - 2.0f * z * g[4] + y * g[5] + x * g[6] + y * g[7]);
}

__global__ void __launch_bounds__(128) chain_kernel(
    const float* __restrict__ planes, const float* __restrict__ sh, int64_t stride, int deg,
    const int32_t* __restrict__ active_idx, uint32_t n_items, const Cam32* __restrict__ camp, Opt32 o,
    const float* __restrict__ sgrad, const uint8_t* __restrict__ touched, float* __restrict__ g_pos,
    float* __restrict__ g_sh, float* __restrict__ g_ls, float* __restrict__ g_quat, float* __restrict__ g_logit,
    float* __restrict__ g_mean2d, uint8_t* __restrict__ touched_out) {
  pdl_wait();
  pdl_trigger();
  const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n_items) return;
  const int64_t i = active_idx ? (int64_t)active_idx[item] : (int64_t)item;
  if (!touched[item]) {
    if (!active_idx) {  // every item covered here: its zero gradients too (no memset pass)
      for (int k = 0; k < 3; ++k) g_pos[3 * i + k] = 0.0f;
      if ((reinterpret_cast<uintptr_t>(g_sh) & 15) == 0) {
        float4* gs = reinterpret_cast<float4*>(g_sh + 48 * i);
        for (int k = 0; k < 12; ++k) gs[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        for (int k = 0; k < 48; ++k) g_sh[48 * i + k] = 0.0f;
      }
      for (int k = 0; k < 3; ++k) g_ls[3 * i + k] = 0.0f;
      for (int k = 0; k < 4; ++k) g_quat[4 * i + k] = 0.0f;
      g_logit[i] = 0.0f;
      g_mean2d[i] = 0.0f;
      touched_out[i] = 0;
    }
    return;
  }
  const Cam32 cam = *camp;
  const float* P = planes + i;
  const float* S = sgrad + (size_t)kSGrad * item;
  const float p[3] = {P[0], P[stride], P[2 * stride]};
  float t[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    t[k] = cam.R[3 * k] * p[0] + cam.R[3 * k + 1] * p[1] + cam.R[3 * k + 2] * p[2] + cam.t[k];
  const float tz = t[2], tz2 = tz * tz, tz3 = tz2 * tz;
  // opacity (core.py:419-421) and its logit
  const float lg = P[3 * stride];
  const float op = lg >= 0.0f ? 1.0f / (1.0f + exp_contract(-lg)) : exp_contract(lg) / (1.0f + exp_contract(lg));
  const float g_opacity = S[3] / op;
  g_logit[i] = g_opacity * op * (1.0f - op);
  // unit quaternion, rotation, scales, 3D covariance
  float q[4] = {P[7 * stride], P[8 * stride], P[9 * stride], P[10 * stride]};
  const float qraw_n = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  float qu[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) qu[k] = q[k] / qraw_n;
  const float w = qu[0], x = qu[1], y = qu[2], z = qu[3];
  const float Rq[9] = {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y - w * z), 2.0f * (x * z + w * y),
                       2.0f * (x * y + w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z - w * x),
                       2.0f * (x * z - w * y), 2.0f * (y * z + w * x), 1.0f - 2.0f * (x * x + y * y)};
  float sc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) sc[k] = exp_contract(P[(4 + k) * stride]);
  float C3[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float acc = 0.0f;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += Rq[3 * r + k] * sc[k] * sc[k] * Rq[3 * c + k];
      C3[3 * r + c] = acc;
    }
  // J, A = J R (render.py:114-119), 2D covariance and its inverse
  const float j00 = cam.fx / tz, j02 = -cam.fx * t[0] / tz2, j11 = cam.fy / tz, j12 = -cam.fy * t[1] / tz2;
  float A[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A[k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
    A[3 + k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
  }
  float AC[6];  // A C3
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) AC[3 * r + c] = A[3 * r] * C3[c] + A[3 * r + 1] * C3[3 + c] + A[3 * r + 2] * C3[6 + c];
  const float a = AC[0] * A[0] + AC[1] * A[1] + AC[2] * A[2] + o.lowpass;
  const float b = AC[0] * A[3] + AC[1] * A[4] + AC[2] * A[5];
  const float c = AC[3] * A[3] + AC[4] * A[4] + AC[5] * A[5] + o.lowpass;
  const float det = a * c - b * b;
  const float ia = c / det, ib = -b / det, ic = a / det;
  // inverse covariance -> 2D covariance: g_cov2d = -inv G inv (render.py:425-435)
  const float G00 = S[6], G01 = 0.5f * S[7], G11 = S[8];
  const float IG00 = ia * G00 + ib * G01, IG01 = ia * G01 + ib * G11;
  const float IG10 = ib * G00 + ic * G01, IG11 = ib * G01 + ic * G11;
  const float gc00 = -(IG00 * ia + IG01 * ib), gc01 = -(IG00 * ib + IG01 * ic);
  const float gc10 = -(IG10 * ia + IG11 * ib), gc11 = -(IG10 * ib + IG11 * ic);
  // 2D covariance -> A and 3D covariance (render.py:438-441)
  float GA[6];  // g_cov2d A
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    GA[k] = gc00 * A[k] + gc01 * A[3 + k];
    GA[3 + k] = gc10 * A[k] + gc11 * A[3 + k];
  }
  float gA[6];  // 2 g_cov2d A C3
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      gA[3 * r + cc] = 2.0f * (GA[3 * r] * C3[cc] + GA[3 * r + 1] * C3[3 + cc] + GA[3 * r + 2] * C3[6 + cc]);
  float gC3[9];  // A^T g_cov2d A
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) gC3[3 * r + cc] = A[r] * GA[cc] + A[3 + r] * GA[3 + cc];
  // A = J R -> J -> camera-space position (render.py:443-452)
  float gJ[6];  // g_amat R^T
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      gJ[3 * r + cc] = gA[3 * r] * cam.R[3 * cc] + gA[3 * r + 1] * cam.R[3 * cc + 1] + gA[3 * r + 2] * cam.R[3 * cc + 2];
  float gt[3] = {0.0f, 0.0f, 0.0f};
  gt[0] += gJ[2] * (-cam.fx / tz2);
  gt[1] += gJ[5] * (-cam.fy / tz2);
  gt[2] += gJ[0] * (-cam.fx / tz2) + gJ[4] * (-cam.fy / tz2) + gJ[2] * (2.0f * cam.fx * t[0] / tz3) +
           gJ[5] * (2.0f * cam.fy * t[1] / tz3);
  // screen mean (render.py:454-458): dL/dmean = -(2 inv (sum dq d))
  const float gmx = -2.0f * (ia * S[4] + ib * S[5]), gmy = -2.0f * (ib * S[4] + ic * S[5]);
  gt[0] += gmx * cam.fx / tz;
  gt[1] += gmy * cam.fy / tz;
  gt[2] += -(gmx * cam.fx * t[0] + gmy * cam.fy * t[1]) / tz2;
  float gp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) gp[k] = gt[0] * cam.R[k] + gt[1] * cam.R[3 + k] + gt[2] * cam.R[6 + k];
  // 3D covariance -> log-scales and quaternion (render.py:462-469)
  float gRm[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      float acc = 0.0f;  // (g_cov3d Rq)[r][cc]
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += gC3[3 * r + k] * Rq[3 * k + cc];
      gRm[3 * r + cc] = 2.0f * acc * sc[cc] * sc[cc];
    }
#pragma unroll
  for (int j = 0; j < 3; ++j) {  // diag(Rq^T g_cov3d Rq)
    float acc = 0.0f;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) acc += Rq[3 * r + j] * gC3[3 * r + cc] * Rq[3 * cc + j];
    g_ls[3 * i + j] = 2.0f * sc[j] * sc[j] * acc;
  }
  float gqu[4];
  quat_rotmat_backward(qu, gRm, gqu);
  const float dot = qu[0] * gqu[0] + qu[1] * gqu[1] + qu[2] * gqu[2] + qu[3] * gqu[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) g_quat[4 * i + k] = (gqu[k] - qu[k] * dot) / qraw_n;
  // colour -> SH coefficients and view direction (render.py:471-487)
  const float v3[3] = {p[0] - cam.center[0], p[1] - cam.center[1], p[2] - cam.center[2]};
  float vn = sqrtf(v3[0] * v3[0] + v3[1] * v3[1] + v3[2] * v3[2]);
  if (!(vn > 0.0f)) vn = 1.0f;
  const float dx = v3[0] / vn, dy = v3[1] / vn, dz = v3[2] / vn;
  const float C1 = 0.4886025119029199f;
  const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f, -1.0925484305920792f,
                       0.5462742152960396f};
  const float C3c[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                        -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
  const float xx = dx * dx, yy = dy * dy, zz = dz * dz;
  float Y[16], dY[16][3];
#pragma unroll
  for (int bnd = 0; bnd < 16; ++bnd) { dY[bnd][0] = dY[bnd][1] = dY[bnd][2] = 0.0f; }
  Y[0] = 0.28209479177387814f;
  Y[1] = -C1 * dy; Y[2] = C1 * dz; Y[3] = -C1 * dx;
  dY[1][1] = -C1; dY[2][2] = C1; dY[3][0] = -C1;
  Y[4] = C2[0] * dx * dy; Y[5] = C2[1] * dy * dz; Y[6] = C2[2] * (2.0f * zz - xx - yy); Y[7] = C2[3] * dx * dz;
  Y[8] = C2[4] * (xx - yy);
  dY[4][0] = C2[0] * dy; dY[4][1] = C2[0] * dx; dY[5][1] = C2[1] * dz; dY[5][2] = C2[1] * dy;
  dY[6][0] = C2[2] * (-2.0f * dx); dY[6][1] = C2[2] * (-2.0f * dy); dY[6][2] = C2[2] * (4.0f * dz);
  dY[7][0] = C2[3] * dz; dY[7][2] = C2[3] * dx; dY[8][0] = C2[4] * (2.0f * dx); dY[8][1] = C2[4] * (-2.0f * dy);
  Y[9] = C3c[0] * dy * (3.0f * xx - yy); Y[10] = C3c[1] * dx * dy * dz; Y[11] = C3c[2] * dy * (4.0f * zz - xx - yy);
  Y[12] = C3c[3] * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy); Y[13] = C3c[4] * dx * (4.0f * zz - xx - yy);
  Y[14] = C3c[5] * dz * (xx - yy); Y[15] = C3c[6] * dx * (xx - 3.0f * yy);
  dY[9][0] = C3c[0] * 6.0f * dx * dy; dY[9][1] = C3c[0] * (3.0f * xx - 3.0f * yy);
  dY[10][0] = C3c[1] * dy * dz; dY[10][1] = C3c[1] * dx * dz; dY[10][2] = C3c[1] * dx * dy;
  dY[11][0] = C3c[2] * (-2.0f * dx * dy); dY[11][1] = C3c[2] * (4.0f * zz - xx - 3.0f * yy);
  dY[11][2] = C3c[2] * (8.0f * dy * dz);
  dY[12][0] = C3c[3] * (-6.0f * dx * dz); dY[12][1] = C3c[3] * (-6.0f * dy * dz);
  dY[12][2] = C3c[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy);
  dY[13][0] = C3c[4] * (4.0f * zz - 3.0f * xx - yy); dY[13][1] = C3c[4] * (-2.0f * dx * dy);
  dY[13][2] = C3c[4] * (8.0f * dx * dz);
  dY[14][0] = C3c[5] * (2.0f * dx * dz); dY[14][1] = C3c[5] * (-2.0f * dy * dz); dY[14][2] = C3c[5] * (xx - yy);
  dY[15][0] = C3c[6] * (3.0f * xx - 3.0f * yy); dY[15][1] = C3c[6] * (-6.0f * dx * dy);
  const int nb = deg == 0 ? 1 : deg == 1 ? 4 : deg == 2 ? 9 : 16;
  const float* shr = sh + 48 * i;
  float gval[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float pre = 0.5f;
#pragma unroll
    for (int bnd = 0; bnd < 16; ++bnd)
      if (bnd < nb) pre += shr[16 * ch + bnd] * Y[bnd];
    gval[ch] = (pre > 0.0f && pre < 1.0f) ? S[ch] : 0.0f;
#pragma unroll
    for (int bnd = 0; bnd < 16; ++bnd) g_sh[48 * i + 16 * ch + bnd] = bnd < nb ? gval[ch] * Y[bnd] : 0.0f;
  }
  if (deg > 0) {
    float gd[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int bnd = 1; bnd < 16; ++bnd) {
      if (bnd >= nb) break;
      const float coeff = gval[0] * shr[bnd] + gval[1] * shr[16 + bnd] + gval[2] * shr[32 + bnd];
#pragma unroll
      for (int k = 0; k < 3; ++k) gd[k] += coeff * dY[bnd][k];
    }
    const float dd = dx * gd[0] + dy * gd[1] + dz * gd[2];
    gp[0] += (gd[0] - dx * dd) / vn;
    gp[1] += (gd[1] - dy * dd) / vn;
    gp[2] += (gd[2] - dz * dd) / vn;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) g_pos[3 * i + k] = gp[k];
  g_mean2d[i] = sqrtf(gmx * gmx + gmy * gmy);
  touched_out[i] = 1;
}

}  // namespace rs
