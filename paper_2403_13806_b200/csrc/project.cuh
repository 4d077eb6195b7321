// project.cuh -- per-Gaussian projection (replaces render.py:95-158).
//
// One thread per item. Reads the 11 geometry planes with coalesced 4-byte loads
// (all issued before any arithmetic: one memory round trip) and, for visible
// Gaussians of colour frames, the 192-byte SH row with twelve 128-bit loads
// issued together; evaluates the Tier-A fp32 contract of
// oracle/cpu_ref.cpp:project_one() in the same operation order (compiled with
// -fmad=false; explicit __fmaf_rn only where the contract fuses), and writes
//   * a 64-byte Rec and its tile-row range (u32 r0 | r1 << 16) for binned items (culled
//     items write nothing else), and
//   * every item's 32-bit depth key (kInvalidKey when not binned), which
//     compact_hist_kernel (sort.cuh) compacts for the depth sort.
#pragma once
#include "rs_common.cuh"
#include "rs_math.cuh"

namespace rs {

__device__ __forceinline__ int floor_clip(float v, int hi) {
  if (v != v) return 0;
  const float f = floorf(v);
  if (f <= 0.0f) return 0;
  if (f >= (float)hi) return hi;
  return (int)f;
}

__device__ __forceinline__ int ceil1_clip(float v, int hi) {
  if (v != v) return 0;
  const float f = ceilf(v);
  if (f <= -1.0f) return 0;
  if (f >= (float)hi) return hi;
  const int r = (int)f + 1;
  return r > hi ? hi : r;
}

// Culling box (oracle: cull_box) from a record's fp32 ellipse terms {p2 >= cut2} and its
// half-open bbox [x0,x1)x[y0,y1): pixels outside the ellipse widened by 1% + 0.5 px cannot
// reach alpha_cut even with the fp32 rounding of p2 (bounded for condition number <= 1e4;
// worse-conditioned Gaussians keep the full bbox). The tile binning uses this box; double
// precision, IEEE ops only (reproducible on the CPU). Returns {cx0, cx1 | tight << 31, cy0,
// cy1 | ell << 31}: tight = the ellipse box binds every side (no pixel outside it can
// composite, bbox gate included); ell = the ellipse bounds the box (tile rows by row_span).
__device__ __forceinline__ int4 cull_box(const Rec& rec, int x0, int x1, int y0, int y1, int width, int height) {
  int cx0 = x0, cx1 = x1, cy0 = y0, cy1 = y1;
  bool tight = false, ell = false;
  const double Na = rec.a.z, Nb = rec.a.w, Nc = rec.b.x;
  const double C2 = rec.b.z;
  const double D = __dsub_rn(__dmul_rn(__dmul_rn(4.0, Na), Nc), __dmul_rn(Nb, Nb));
  const double tr = __dadd_rn(Na, Nc);
  const double sq = __dsqrt_rn(__dadd_rn(__dmul_rn(__dsub_rn(Na, Nc), __dsub_rn(Na, Nc)), __dmul_rn(Nb, Nb)));
  const double l1 = __dmul_rn(0.5, __dsub_rn(tr, sq)), l2 = __dmul_rn(0.5, __dadd_rn(tr, sq));
  if (!(C2 < 0.0)) {
    cx1 = cx0;
    cy1 = cy0;
  } else if (C2 > -1e30 && D > 0.0 && l2 < 0.0 && l1 >= __dmul_rn(1e4, l2)) {
    const double hx = __dadd_rn(__dmul_rn(__dsqrt_rn(__ddiv_rn(__dmul_rn(__dmul_rn(C2, 4.0), Nc), D)), 1.01), 0.5);
    const double hy = __dadd_rn(__dmul_rn(__dsqrt_rn(__ddiv_rn(__dmul_rn(__dmul_rn(C2, 4.0), Na), D)), 1.01), 0.5);
    const double dmx = rec.a.x, dmy = rec.a.y;
    const int ex0 = (int)fmax(floor(__dsub_rn(__dsub_rn(dmx, hx), 0.5)), -1.0);
    const int ex1 = (int)fmin(__dadd_rn(floor(__dsub_rn(__dadd_rn(dmx, hx), 0.5)), 1.0), 65535.0);
    const int ey0 = (int)fmax(floor(__dsub_rn(__dsub_rn(dmy, hy), 0.5)), -1.0);
    const int ey1 = (int)fmin(__dadd_rn(floor(__dsub_rn(__dadd_rn(dmy, hy), 0.5)), 1.0), 65535.0);
    cx0 = max(x0, ex0);
    cx1 = min(x1, ex1);
    cy0 = max(y0, ey0);
    cy1 = min(y1, ey1);
    ell = true;
    tight = (ex0 >= x0 || x0 == 0) && (ex1 <= x1 || x1 == width) && (ey0 >= y0 || y0 == 0) &&
            (ey1 <= y1 || y1 == height);
    if (cx1 < cx0) cx1 = cx0;
    if (cy1 < cy0) cy1 = cy0;
  }
  return make_int4(cx0, cx1 | (tight ? (int)0x80000000 : 0), cy0, cy1 | (ell ? (int)0x80000000 : 0));
}

// FULL additionally writes, for every item (culled ones included), the
// ProjectedGaussian fields of render.py:49-59 as 16 floats
// {mx, my, a, b, c, ia, ib, ic, radius, depth, r, g, b, opacity, valid, 0}
// and the int4 bbox: the per-primitive API project_gaussian/project_scene.
// COLOR = false skips the SH colour (score-only frames never read it: 192 B per
// visible Gaussian less traffic, SURVEY §8d "44 B without SH in score mode").
// Scene values of either storage type as T (a double scene in an fp32 frame is
// rounded once, = numpy astype(float32); a float scene in an fp64 frame widens exactly).
template <typename T, typename TS>
__device__ __forceinline__ T ld_as(const TS* p) { return (T)__ldg(p); }

// the Gaussian's 48 SH coefficients as T (bands >= nb read as 0): 128-bit loads issued together
template <typename T, typename TS>
__device__ __forceinline__ void load_sh_row(const TS* __restrict__ sh, int64_t i, int nb, T* c) {
  if (sizeof(TS) == 4) {
    const float4* shr = reinterpret_cast<const float4*>(sh) + 12 * i;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (4 * v < nb) q = __ldg(shr + 4 * ch + v);
        c[16 * ch + 4 * v] = (T)q.x; c[16 * ch + 4 * v + 1] = (T)q.y;
        c[16 * ch + 4 * v + 2] = (T)q.z; c[16 * ch + 4 * v + 3] = (T)q.w;
      }
  } else {
    const double2* shr = reinterpret_cast<const double2*>(sh) + 24 * i;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        double2 q = make_double2(0.0, 0.0);
        if (2 * v < nb) q = __ldg(shr + 8 * ch + v);
        c[16 * ch + 2 * v] = (T)q.x; c[16 * ch + 2 * v + 1] = (T)q.y;
      }
  }
}

// active_idx entry -> scene index, or -1 (out of range: flagged, the item is culled)
__device__ __forceinline__ int64_t item_index(const int32_t* __restrict__ active_idx, uint32_t item,
                                              int64_t n_scene, Counters* ctr, Sticky* sticky) {
  if (!active_idx) return (int64_t)item;
  const int64_t i = (int64_t)__ldg(active_idx + item);
  if (i < 0 || i >= n_scene) {
    ctr->bad_index = 1u;
    sticky->bad_index = 1u;
    return -1;
  }
  return i;
}

template <bool FULL, bool COLOR, typename TS>
#ifdef RS_PROJ_MINB  // measurement: CTAs per SM the register allocation must allow
#define RS_PROJ_BOUNDS __launch_bounds__(128, RS_PROJ_MINB)
#else
#define RS_PROJ_BOUNDS __launch_bounds__(128)
#endif
__global__ void RS_PROJ_BOUNDS project_kernel(const TS* __restrict__ planes,
                                                      const TS* __restrict__ sh, int64_t stride, int deg,
                                                      const int32_t* __restrict__ active_idx, uint32_t n_items,
                                                      int64_t n_scene,
                                                      const Cam32* __restrict__ camp, Opt32 o,
                                                      Rec* __restrict__ recs,
                                                      uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
                                                      Counters* __restrict__ ctr, Sticky* __restrict__ sticky,
                                                      float* __restrict__ full, int4* __restrict__ full_bbox) {
  pdl_wait();
  pdl_trigger();
  const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item == 0) ctr->n_items = n_items;
  // the camera lives in device memory (uploaded by a stream-ordered copy), so a captured
  // CUDA graph of the frame replays with a new camera without re-instantiation
  const Cam32 cam = *camp;
  bool valid = false, binned = false;
  float depth_b = 0.0f;  // depth of a binned record (its sort key)
  const int64_t i = item < n_items ? item_index(active_idx, item, n_scene, ctr, sticky) : -1;
  if (i >= 0) {
    const TS* P = planes + i;
    // all eleven plane loads issued together (one memory round trip per thread)
    const float px = ld_as<float>(P), py = ld_as<float>(P + stride), pz = ld_as<float>(P + 2 * stride);
    const float lg = ld_as<float>(P + 3 * stride);
    const float ls0 = ld_as<float>(P + 4 * stride), ls1 = ld_as<float>(P + 5 * stride),
                ls2 = ld_as<float>(P + 6 * stride);
    float qw = ld_as<float>(P + 7 * stride), qx = ld_as<float>(P + 8 * stride), qy = ld_as<float>(P + 9 * stride),
          qz = ld_as<float>(P + 10 * stride);
    // t = R p + T (render.py:100)
    float t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      t[k] = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(cam.R[3 * k], px), __fmul_rn(cam.R[3 * k + 1], py)),
                                 __fmul_rn(cam.R[3 * k + 2], pz)),
                       cam.t[k]);
    const bool valid0 = t[2] > o.near_limit;
    const float tz = valid0 ? t[2] : 1.0f;
    const float mx = __fadd_rn(__fdiv_rn(__fmul_rn(cam.fx, t[0]), tz), cam.cx);  // render.py:104-105
    const float my = __fadd_rn(__fdiv_rn(__fmul_rn(cam.fy, t[1]), tz), cam.cy);
    const float depth = __fadd_rn(t[2], 0.0f);
    // quaternion -> rotation (core.py:111-139)
    const float qn = __fsqrt_rn(
        __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(qw, qw), __fmul_rn(qx, qx)), __fmul_rn(qy, qy)), __fmul_rn(qz, qz)));
    qw = __fdiv_rn(qw, qn); qx = __fdiv_rn(qx, qn); qy = __fdiv_rn(qy, qn); qz = __fdiv_rn(qz, qn);
    float Rq[9];
    Rq[0] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qy, qy), __fmul_rn(qz, qz))));
    Rq[1] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qx, qy), __fmul_rn(qw, qz)));
    Rq[2] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qz), __fmul_rn(qw, qy)));
    Rq[3] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qy), __fmul_rn(qw, qz)));
    Rq[4] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qz, qz))));
    Rq[5] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qy, qz), __fmul_rn(qw, qx)));
    Rq[6] = __fmul_rn(2.0f, __fsub_rn(__fmul_rn(qx, qz), __fmul_rn(qw, qy)));
    Rq[7] = __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qy, qz), __fmul_rn(qw, qx)));
    Rq[8] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(__fmul_rn(qx, qx), __fmul_rn(qy, qy))));
    // Sigma = L L^T, L = Rq diag(exp(log_s)) (render.py:108-111)
    float sc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) sc[j] = exp_contract(j == 0 ? ls0 : j == 1 ? ls1 : ls2);
    float L[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) L[3 * r + j] = __fmul_rn(Rq[3 * r + j], sc[j]);
    float S[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        S[3 * r + k] = __fadd_rn(__fadd_rn(__fmul_rn(L[3 * r], L[3 * k]), __fmul_rn(L[3 * r + 1], L[3 * k + 1])),
                                 __fmul_rn(L[3 * r + 2], L[3 * k + 2]));
    // J and A = J R_cam (render.py:114-119)
    const float tz2 = __fmul_rn(tz, tz);
    const float j00 = __fdiv_rn(cam.fx, tz), j02 = __fdiv_rn(__fmul_rn(-cam.fx, t[0]), tz2);
    const float j11 = __fdiv_rn(cam.fy, tz), j12 = __fdiv_rn(__fmul_rn(-cam.fy, t[1]), tz2);
    float A[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      A[k] = __fadd_rn(__fmul_rn(j00, cam.R[k]), __fmul_rn(j02, cam.R[6 + k]));
      A[3 + k] = __fadd_rn(__fmul_rn(j11, cam.R[3 + k]), __fmul_rn(j12, cam.R[6 + k]));
    }
    float MS[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        MS[3 * r + k] = __fadd_rn(__fadd_rn(__fmul_rn(A[3 * r], S[k]), __fmul_rn(A[3 * r + 1], S[3 + k])),
                                  __fmul_rn(A[3 * r + 2], S[6 + k]));
    const float c00 = __fadd_rn(__fadd_rn(__fmul_rn(MS[0], A[0]), __fmul_rn(MS[1], A[1])), __fmul_rn(MS[2], A[2]));
    const float c01 = __fadd_rn(__fadd_rn(__fmul_rn(MS[0], A[3]), __fmul_rn(MS[1], A[4])), __fmul_rn(MS[2], A[5]));
    const float c11 = __fadd_rn(__fadd_rn(__fmul_rn(MS[3], A[3]), __fmul_rn(MS[4], A[4])), __fmul_rn(MS[5], A[5]));
    const float a = __fadd_rn(c00, o.lowpass), b = c01, c = __fadd_rn(c11, o.lowpass);  // render.py:121-123
    const float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));                       // render.py:125-128
    const float ia = __fdiv_rn(c, det), ib = __fdiv_rn(-b, det), ic = __fdiv_rn(a, det);
    const float amc = __fsub_rn(a, c);  // render.py:130-131
    const float disc = __fadd_rn(__fmul_rn(0.25f, __fmul_rn(amc, amc)), __fmul_rn(b, b));
    const float lam = __fadd_rn(__fmul_rn(0.5f, __fadd_rn(a, c)), __fsqrt_rn(disc > 0.0f ? disc : 0.0f));
    const float radius = __fmul_rn(o.sigma_bound, __fsqrt_rn(lam > 0.0f ? lam : 0.0f));
    const int x0 = floor_clip(__fsub_rn(mx, radius), cam.width);  // render.py:133-137
    const int x1 = ceil1_clip(__fadd_rn(mx, radius), cam.width);
    const int y0 = floor_clip(__fsub_rn(my, radius), cam.height);
    const int y1 = ceil1_clip(__fadd_rn(my, radius), cam.height);
    valid = valid0 && x1 > x0 && y1 > y0;
    if (valid || FULL) {
      float col[3] = {0.0f, 0.0f, 0.0f};
      if (COLOR || FULL) {
      // view-direction SH colour (render.py:139-149, core.py:207-239)
      const float vx = __fsub_rn(px, cam.center[0]), vy = __fsub_rn(py, cam.center[1]),
                  vz = __fsub_rn(pz, cam.center[2]);
      float vn = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(vx, vx), __fmul_rn(vy, vy)), __fmul_rn(vz, vz)));
      if (!(vn > 0.0f)) vn = 1.0f;
      const float x = __fdiv_rn(vx, vn), y = __fdiv_rn(vy, vn), z = __fdiv_rn(vz, vn);
      float Y[16];
      Y[0] = (float)0.28209479177387814;
      const float C1 = (float)0.4886025119029199;
      Y[1] = __fmul_rn(-C1, y); Y[2] = __fmul_rn(C1, z); Y[3] = __fmul_rn(-C1, x);
      const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
      const float xy = __fmul_rn(x, y), yz = __fmul_rn(y, z), xz = __fmul_rn(x, z);
      Y[4] = __fmul_rn((float)1.0925484305920792, xy);
      Y[5] = __fmul_rn((float)-1.0925484305920792, yz);
      Y[6] = __fmul_rn((float)0.31539156525252005, __fsub_rn(__fsub_rn(__fmul_rn(2.0f, zz), xx), yy));
      Y[7] = __fmul_rn((float)-1.0925484305920792, xz);
      Y[8] = __fmul_rn((float)0.5462742152960396, __fsub_rn(xx, yy));
      Y[9] = __fmul_rn(__fmul_rn((float)-0.5900435899266435, y), __fsub_rn(__fmul_rn(3.0f, xx), yy));
      Y[10] = __fmul_rn(__fmul_rn((float)2.890611442640554, xy), z);
      Y[11] = __fmul_rn(__fmul_rn((float)-0.4570457994644658, y), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
      Y[12] = __fmul_rn(__fmul_rn((float)0.3731763325901154, z),
                        __fsub_rn(__fsub_rn(__fmul_rn(2.0f, zz), __fmul_rn(3.0f, xx)), __fmul_rn(3.0f, yy)));
      Y[13] = __fmul_rn(__fmul_rn((float)-0.4570457994644658, x), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
      Y[14] = __fmul_rn(__fmul_rn((float)1.445305721320277, z), __fsub_rn(xx, yy));
      Y[15] = __fmul_rn(__fmul_rn((float)-0.5900435899266435, x), __fsub_rn(xx, __fmul_rn(3.0f, yy)));
      const int nb = deg == 0 ? 1 : deg == 1 ? 4 : deg == 2 ? 9 : 16;
      // the Gaussian's SH row: 128-bit loads, issued together (one round trip)
      float c[48];
      load_sh_row<float>(sh, i, nb, c);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        float acc = __fmul_rn(c[16 * ch], Y[0]);
#pragma unroll
        for (int bnd = 1; bnd < 16; ++bnd)
          if (bnd < nb) acc = __fadd_rn(acc, __fmul_rn(c[16 * ch + bnd], Y[bnd]));
        const float pre = __fadd_rn(0.5f, acc);
        col[ch] = pre < 0.0f ? 0.0f : (pre > 1.0f ? 1.0f : pre);
      }
      }  // COLOR
      // opacity = sigmoid(logit) (core.py:419-421)
      float op;
      if (lg >= 0.0f) {
        op = __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_contract(-lg)));
      } else {
        const float e = exp_contract(lg);
        op = __fdiv_rn(e, __fadd_rn(1.0f, e));
      }
      const float K = fbits(0xbf38aa3bu);  // -0.5*log2(e)
      // conservative skip threshold: p2 < cut2 => alpha < alpha_cut; clamped at
      // -126 (p2 < -126 gives alpha < 2^-126 < alpha_cut whenever alpha_cut >= 1e-30)
      float cut2 = o.alpha_cut > 0.0f ? __fsub_rn(log2_contract(__fdiv_rn(o.alpha_cut, op)), 1e-3f) : -INFINITY;
      if (o.alpha_cut >= 1e-30f && cut2 < -126.0f) cut2 = -126.0f;
      Rec rec;
      rec.a = make_float4(mx, my, __fmul_rn(K, ia), __fmul_rn(__fmul_rn(2.0f, K), ib));
      rec.b = make_float4(__fmul_rn(K, ic), op, cut2, depth);
      rec.c = make_float4(col[0], col[1], col[2], __int_as_float((int)i));
      int4 cb;
      if (valid) cb = cull_box(rec, x0, x1, y0, y1, cam.width, cam.height);
      else cb = make_int4(x0, x1, y0, y1);
      const int cx0 = cb.x, cx1 = cb.y & 0x7fffffff, cy0 = cb.z, cy1 = cb.w & 0x7fffffff;
      binned = valid && cx1 > cx0 && cy1 > cy0;
      rec.d = make_int4(x0 | (x1 << 16), y0 | (y1 << 16), cx0 | (cx1 << 16) | (cb.y & (int)0x80000000),
                        cy0 | (cy1 << 16) | (cb.w & (int)0x80000000));
      if (binned) {
        recs[item] = rec;
        rows[item] = (uint32_t)(cy0 / kTile) | ((uint32_t)((cy1 - 1) / kTile) << 16);  // segrows_kernel
        depth_b = depth;
      }
      if (FULL) {
        float4* f = reinterpret_cast<float4*>(full + 16 * (size_t)item);
        f[0] = make_float4(mx, my, a, b);
        f[1] = make_float4(c, ia, ib, ic);
        f[2] = make_float4(radius, depth, col[0], col[1]);
        f[3] = make_float4(col[2], op, valid ? 1.0f : 0.0f, cut2);
        full_bbox[item] = make_int4(x0, x1, y0, y1);
      }
    }
  }
  if (item < n_items) keys[item] = binned ? depth_key(depth_b) : kInvalidKey;
}

}  // namespace rs

namespace rs {

// ---------------------------------------------------------------------------
// RS_F64 frames: the reference's projection in double (render.py:95-158), in
// the operation order of the oracle's fp64 tiers (oracle/cpu_ref.cpp
// project_one<double>; -fmad=false: no contraction) with the contract exp
// (rs_math.cuh exp64_contract) for the scales and the sigmoid. Writes per binned
// item the fp64 Rec64 the blend evaluates and the fp32 Rec the binning uses
// (boxes, ellipse terms, depth key = the fp32 rounding of the fp64 depth, which
// is monotone, so the radix order is the fp64 order up to fp32 ties -- those
// are resolved by tiefix_kernel, sort.cuh).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int floor_clip64(double v, int hi) {
  if (v != v) return 0;
  const double f = floor(v);
  if (f <= 0.0) return 0;
  if (f >= (double)hi) return hi;
  return (int)f;
}

__device__ __forceinline__ int ceil1_clip64(double v, int hi) {
  if (v != v) return 0;
  const double f = ceil(v);
  if (f <= -1.0) return 0;
  if (f >= (double)hi) return hi;
  const int r = (int)f + 1;
  return r > hi ? hi : r;
}

template <bool FULL, bool COLOR, typename TS>
__global__ void __launch_bounds__(128) project64_kernel(const TS* __restrict__ planes,
                                                        const TS* __restrict__ sh, int64_t stride, int deg,
                                                        const int32_t* __restrict__ active_idx, uint32_t n_items,
                                                        int64_t n_scene, const rs_camera* __restrict__ camp,
                                                        Opt64 o, Rec* __restrict__ recs, Rec64* __restrict__ recs64,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ rows,
                                                        Counters* __restrict__ ctr, Sticky* __restrict__ sticky,
                                                        double* __restrict__ full, int4* __restrict__ full_bbox) {
  pdl_wait();
  pdl_trigger();
  const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item == 0) ctr->n_items = n_items;
  const rs_camera& cam = *camp;
  bool binned = false;
  float depth_b = 0.0f;
  const int64_t i = item < n_items ? item_index(active_idx, item, n_scene, ctr, sticky) : -1;
  if (i >= 0) {
    const TS* P = planes + i;
    const double px = ld_as<double>(P), py = ld_as<double>(P + stride), pz = ld_as<double>(P + 2 * stride);
    const double lg = ld_as<double>(P + 3 * stride);
    const double ls0 = ld_as<double>(P + 4 * stride), ls1 = ld_as<double>(P + 5 * stride),
                 ls2 = ld_as<double>(P + 6 * stride);
    double qw = ld_as<double>(P + 7 * stride), qx = ld_as<double>(P + 8 * stride),
           qy = ld_as<double>(P + 9 * stride), qz = ld_as<double>(P + 10 * stride);
    // t = R p + T (render.py:100)
    double t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = ((cam.R[3 * k] * px + cam.R[3 * k + 1] * py) + cam.R[3 * k + 2] * pz) + cam.t[k];
    const bool valid0 = t[2] > o.near_limit;
    const double tz = valid0 ? t[2] : 1.0;
    const double mx = (cam.fx * t[0]) / tz + cam.cx;  // render.py:104-105
    const double my = (cam.fy * t[1]) / tz + cam.cy;
    const double depth = t[2] + 0.0;
    // quaternion -> rotation (core.py:111-139)
    const double qn = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
    qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn;
    double Rq[9];
    Rq[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
    Rq[1] = 2.0 * (qx * qy - qw * qz);
    Rq[2] = 2.0 * (qx * qz + qw * qy);
    Rq[3] = 2.0 * (qx * qy + qw * qz);
    Rq[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
    Rq[5] = 2.0 * (qy * qz - qw * qx);
    Rq[6] = 2.0 * (qx * qz - qw * qy);
    Rq[7] = 2.0 * (qy * qz + qw * qx);
    Rq[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
    // Sigma = L L^T, L = Rq diag(exp(log_s)) (render.py:108-111)
    const double sc[3] = {exp64_contract(ls0), exp64_contract(ls1), exp64_contract(ls2)};
    double L[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) L[3 * r + j] = Rq[3 * r + j] * sc[j];
    double S[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        S[3 * r + k] = (L[3 * r] * L[3 * k] + L[3 * r + 1] * L[3 * k + 1]) + L[3 * r + 2] * L[3 * k + 2];
    // J and A = J R_cam (render.py:114-119)
    const double j00 = cam.fx / tz, j02 = (-cam.fx * t[0]) / (tz * tz);
    const double j11 = cam.fy / tz, j12 = (-cam.fy * t[1]) / (tz * tz);
    double A[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      A[k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
      A[3 + k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
    }
    double MS[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        MS[3 * r + k] = (A[3 * r] * S[k] + A[3 * r + 1] * S[3 + k]) + A[3 * r + 2] * S[6 + k];
    const double c00 = (MS[0] * A[0] + MS[1] * A[1]) + MS[2] * A[2];
    const double c01 = (MS[0] * A[3] + MS[1] * A[4]) + MS[2] * A[5];
    const double c11 = (MS[3] * A[3] + MS[4] * A[4]) + MS[5] * A[5];
    const double a = c00 + o.lowpass, b = c01, c = c11 + o.lowpass;  // render.py:121-123
    const double det = a * c - b * b;                                  // render.py:125-128
    const double ia = c / det, ib = -b / det, ic = a / det;
    const double amc = a - c;  // render.py:130-131
    const double disc = 0.25 * (amc * amc) + b * b;
    const double lam = 0.5 * (a + c) + sqrt(disc > 0.0 ? disc : 0.0);
    const double radius = o.sigma_bound * sqrt(lam > 0.0 ? lam : 0.0);
    const int x0 = floor_clip64(mx - radius, cam.width);  // render.py:133-137
    const int x1 = ceil1_clip64(mx + radius, cam.width);
    const int y0 = floor_clip64(my - radius, cam.height);
    const int y1 = ceil1_clip64(my + radius, cam.height);
    const bool valid = valid0 && x1 > x0 && y1 > y0;
    if (valid || FULL) {
      double col[3] = {0.0, 0.0, 0.0};
      if (COLOR || FULL) {
        // view-direction SH colour (render.py:139-149, core.py:207-239)
        const double vx = px - cam.center[0], vy = py - cam.center[1], vz = pz - cam.center[2];
        double vn = sqrt((vx * vx + vy * vy) + vz * vz);
        if (!(vn > 0.0)) vn = 1.0;
        const double x = vx / vn, y = vy / vn, z = vz / vn;
        double Y[16];
        Y[0] = 0.28209479177387814;
        const double C1 = 0.4886025119029199;
        Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
        const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        Y[4] = 1.0925484305920792 * xy;
        Y[5] = -1.0925484305920792 * yz;
        Y[6] = 0.31539156525252005 * ((2.0 * zz - xx) - yy);
        Y[7] = -1.0925484305920792 * xz;
        Y[8] = 0.5462742152960396 * (xx - yy);
        Y[9] = (-0.5900435899266435 * y) * (3.0 * xx - yy);
        Y[10] = (2.890611442640554 * xy) * z;
        Y[11] = (-0.4570457994644658 * y) * ((4.0 * zz - xx) - yy);
        Y[12] = (0.3731763325901154 * z) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy);
        Y[13] = (-0.4570457994644658 * x) * ((4.0 * zz - xx) - yy);
        Y[14] = (1.445305721320277 * z) * (xx - yy);
        Y[15] = (-0.5900435899266435 * x) * (xx - 3.0 * yy);
        const int nb = deg == 0 ? 1 : deg == 1 ? 4 : deg == 2 ? 9 : 16;
        double cf[48];
        load_sh_row<double>(sh, i, nb, cf);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          double acc = cf[16 * ch] * Y[0];
#pragma unroll
          for (int bnd = 1; bnd < 16; ++bnd)
            if (bnd < nb) acc = acc + cf[16 * ch + bnd] * Y[bnd];
          const double pre = 0.5 + acc;
          col[ch] = pre < 0.0 ? 0.0 : (pre > 1.0 ? 1.0 : pre);
        }
      }
      // opacity = sigmoid(logit) (core.py:419-421)
      double op;
      if (lg >= 0.0) {
        op = 1.0 / (1.0 + exp64_contract(-lg));
      } else {
        const double e = exp64_contract(lg);
        op = e / (1.0 + e);
      }
      // the fp32 record of the binning (oracle: project_one's fp32 terms + cull_box)
      const float K = fbits(0xbf38aa3bu);  // -0.5*log2(e)
      const float opf = (float)op, acf = (float)o.alpha_cut;
      float cut2 = acf > 0.0f ? __fsub_rn(log2_contract(__fdiv_rn(acf, opf)), 1e-3f) : -INFINITY;
      if (acf >= 1e-30f && cut2 < -126.0f) cut2 = -126.0f;
      Rec rec;
      rec.a = make_float4((float)mx, (float)my, __fmul_rn(K, (float)ia), __fmul_rn(__fmul_rn(2.0f, K), (float)ib));
      rec.b = make_float4(__fmul_rn(K, (float)ic), opf, cut2, (float)depth);
      rec.c = make_float4((float)col[0], (float)col[1], (float)col[2], __int_as_float((int)i));
      int4 cb;
      if (valid) cb = cull_box(rec, x0, x1, y0, y1, cam.width, cam.height);
      else cb = make_int4(x0, x1, y0, y1);
      const int cx0 = cb.x, cx1 = cb.y & 0x7fffffff, cy0 = cb.z, cy1 = cb.w & 0x7fffffff;
      binned = valid && cx1 > cx0 && cy1 > cy0;
      rec.d = make_int4(x0 | (x1 << 16), y0 | (y1 << 16), cx0 | (cx1 << 16) | (cb.y & (int)0x80000000),
                        cy0 | (cy1 << 16) | (cb.w & (int)0x80000000));
      if (binned) {
        recs[item] = rec;
        Rec64 r64;
        r64.mx = mx; r64.my = my;
        r64.na = -0.5 * ia; r64.nb = -ib; r64.nc = -0.5 * ic;
        r64.o = op; r64.depth = depth;
        // conservative exp skip (a margin far above the exp / log rounding): -q/2 < lnc
        // implies o * exp(-q/2) < alpha_cut; never changes a result
        r64.lnc = log(o.alpha_cut / op) - 1e-6;
        r64.r = col[0]; r64.g = col[1]; r64.b = col[2];
        r64.gid = (uint32_t)i; r64.pad = 0u;
        recs64[item] = r64;
        rows[item] = (uint32_t)(cy0 / kTile) | ((uint32_t)((cy1 - 1) / kTile) << 16);
        depth_b = (float)depth;
      }
      if (FULL) {
        double* f = full + 16 * (size_t)item;
        f[0] = mx; f[1] = my; f[2] = a; f[3] = b;
        f[4] = c; f[5] = ia; f[6] = ib; f[7] = ic;
        f[8] = radius; f[9] = depth; f[10] = col[0]; f[11] = col[1];
        f[12] = col[2]; f[13] = op; f[14] = valid ? 1.0 : 0.0; f[15] = (double)cut2;
        full_bbox[item] = make_int4(x0, x1, y0, y1);
      }
    }
  }
  if (item < n_items) keys[item] = binned ? depth_key(depth_b) : kInvalidKey;
}

}  // namespace rs
