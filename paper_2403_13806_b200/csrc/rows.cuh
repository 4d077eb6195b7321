// rows.cuh -- which tiles of its culling box a Gaussian is binned to.
//
// Tile row ty of the culling box lists tile columns [tx0, tx1]: for an
// ellipse-derived culling box (Rec.d bit 31) the x-extent, over the strip of
// the row's pixel centres dilated by 0.5 px, of the ellipse {p2 >= cut2}
// scaled by 1.01 (q = -p2 <= 1.0201 K) and dilated by 0.5 px -- the same
// conservative region whose bounding box is the culling box (project.cuh), so
// no dropped tile holds a pixel that can reach alpha_cut. The x-extent of an
// ellipse over a strip is attained at the strip point nearest the ellipse's
// rightmost (leftmost) point, since the boundary x(dy) is concave (convex).
// Otherwise the full culling-box row.
//
// Float arithmetic (D = 4 A Cc - B^2 formed in double: it cancels for elongated
// ellipses) with explicit slack for the rounding (oracle/cpu_ref.cpp:row_geom);
// IEEE operations in the oracle's fixed order, so the binning is bit-exact.
// On configs[1] this lists 19% fewer (tile, Gaussian) pairs than the
// rectangles, 44% fewer on the anisotropic configs[4]. Used by segplace_kernel.
#pragma once
#include "rs_common.cuh"

namespace rs {

struct RowGeom {
  float mx, my, hy, dyr, ak4, d, bi, i2a, del, sd;  // sd = edge_s at dyr
};

// sqrt(max(4AK - D u^2, 0) + del): the boundary term at dy = u (even in u, so one value
// serves the rightmost point dyr and the leftmost point -dyr)
__device__ __forceinline__ float row_s(const RowGeom& g, float u) {
  return __fsqrt_rn(__fadd_rn(fmaxf(__fsub_rn(g.ak4, __fmul_rn(__fmul_rn(g.d, u), u)), 0.0f), g.del));
}
// the term at a row edge u = ys - my, clamped to the ellipse's [-hy, hy]: adjacent rows share
// their common edge, and for a non-empty row this is exactly row_s at its clamped lo / hi
__device__ __forceinline__ float edge_s(const RowGeom& g, float u) { return row_s(g, fminf(fmaxf(u, -g.hy), g.hy)); }

__device__ __forceinline__ RowGeom row_geom(const float4 a, const float4 b) {
  // D = 4 A Cc - B^2 cancels for elongated ellipses: formed in double, then rounded once
  const double Nad = a.z, Nbd = a.w, Ncd = b.x;
  const float D = (float)__dsub_rn(__dmul_rn(__dmul_rn(4.0, Nad), Ncd), __dmul_rn(Nbd, Nbd));
  const float A = -a.z, B = -a.w, Cc = -b.x;  // q = A dx^2 + B dx dy + Cc dy^2 = -p2
  const float K = __fmul_rn(b.z, -1.0201f);
  const float AK4 = __fmul_rn(__fmul_rn(4.0f, A), K);
  RowGeom g;
  g.mx = a.x;
  g.my = a.y;
  g.hy = __fmul_rn(__fsqrt_rn(__fdiv_rn(AK4, D)), 1.00001f);
  const float hx = __fsqrt_rn(__fdiv_rn(__fmul_rn(__fmul_rn(4.0f, Cc), K), D));
  g.dyr = __fdiv_rn(__fmul_rn(-B, hx), __fmul_rn(2.0f, Cc));  // dy of the rightmost point
  g.ak4 = AK4;
  g.d = D;
  g.i2a = __fdiv_rn(1.0f, __fmul_rn(2.0f, A));
  g.bi = __fmul_rn(-B, g.i2a);  // x(dy) = bi dy +- sqrt(4AK - D dy^2) / (2A)
  g.del = __fmul_rn(AK4, 4e-6f);
  g.sd = row_s(g, g.dyr);
  return g;
}

// Edge offsets of tile row ty: [ys, ye) = the row's pixel rows inside the culling box,
// ulo = ys - my, uhi = ye - my (floats; adjacent rows share an edge value).
__device__ __forceinline__ float row_edge(const RowGeom& g, int y) { return __fsub_rn((float)y, g.my); }

// Pixel columns [px0, px1) of an ellipse strip from its edge offsets and edge terms
// (slo = edge_s(ulo), shi = edge_s(uhi)); identical to oracle row_span: the clamped dyr /
// -dyr is one of lo, hi, +-dyr and the boundary term there is slo, shi or sd. Holds for any
// strip of pixel rows (the blend also takes the two 8-row halves of a tile row).
__device__ __forceinline__ bool row_px_e(const RowGeom& g, const int4 cb, float ulo, float uhi, float slo, float shi,
                                         int& px0, int& px1) {
  const float lo = fmaxf(ulo, -g.hy), hi = fminf(uhi, g.hy);
  if (!(lo <= hi)) return false;
  float ur, sr, ul, sl;
  if (g.dyr < lo) { ur = lo; sr = slo; } else if (g.dyr > hi) { ur = hi; sr = shi; } else { ur = g.dyr; sr = g.sd; }
  const float nd = -g.dyr;
  if (nd < lo) { ul = lo; sl = slo; } else if (nd > hi) { ul = hi; sl = shi; } else { ul = nd; sl = g.sd; }
  const float right = __fadd_rn(__fadd_rn(g.mx, __fadd_rn(__fmul_rn(g.bi, ur), __fmul_rn(sr, g.i2a))), 0.52f);
  const float left = __fsub_rn(__fadd_rn(g.mx, __fsub_rn(__fmul_rn(g.bi, ul), __fmul_rn(sl, g.i2a))), 0.52f);
  px0 = (int)fmaxf(floorf(__fsub_rn(left, 0.5f)), (float)cb.x);
  px1 = (int)fminf(__fadd_rn(floorf(__fsub_rn(right, 0.5f)), 1.0f), (float)cb.y);
  return px1 > px0;
}

// The same as tile columns [tx0, tx1].
__device__ __forceinline__ bool row_span_e(const RowGeom& g, const int4 cb, float ulo, float uhi, float slo, float shi,
                                           int& tx0, int& tx1) {
  int px0, px1;
  if (!row_px_e(g, cb, ulo, uhi, slo, shi, px0, px1)) return false;
  tx0 = px0 / kTile;
  tx1 = (px1 - 1) / kTile;
  return true;
}

// Span of ellipse row ty (both edge terms evaluated here).
__device__ __forceinline__ bool row_span(const RowGeom& g, const int4 cb, int ty, int& tx0, int& tx1) {
  const float ulo = row_edge(g, max(ty * kTile, cb.z)), uhi = row_edge(g, min(ty * kTile + kTile, cb.w));
  return row_span_e(g, cb, ulo, uhi, edge_s(g, ulo), edge_s(g, uhi), tx0, tx1);
}

// RowGeom without the mean, as two float4 per Gaussian (segplace_kernel -> blend2_kernel, backward2_kernel).
__device__ __forceinline__ void store_row_geom(float4* dst, const RowGeom& g) {
  dst[0] = make_float4(g.hy, g.dyr, g.ak4, g.d);
  dst[1] = make_float4(g.bi, g.i2a, g.del, g.sd);
}
__device__ __forceinline__ RowGeom load_row_geom(const float4* src, float mx, float my) {
  const float4 u = __ldg(src), v = __ldg(src + 1);
  RowGeom g;
  g.mx = mx;
  g.my = my;
  g.hy = u.x;
  g.dyr = u.y;
  g.ak4 = u.z;
  g.d = u.w;
  g.bi = v.x;
  g.i2a = v.y;
  g.del = v.z;
  g.sd = v.w;
  return g;
}

// The 8x8 quarters of the tile at (ox, oy) that the ellipse strips of its two 8-row halves
// reach (within culling box cb, whose rows meet the tile's): bit 1 top-left, 2 top-right,
// 4 bottom-left, 8 bottom-right (blend2_kernel's warp w = (w % 2, w / 2)). Each half is
// the strip of its own pixel rows, as conservative as the binning's row strips.
__device__ __forceinline__ uint32_t quarter_mask(const RowGeom& g, const int4 cb, int ox, int oy) {
  const int ys = max(oy, cb.z), ye = min(oy + kTile, cb.w), ym = oy + 8;
  const float ulo = row_edge(g, ys), uhi = row_edge(g, ye);
  const float slo = edge_s(g, ulo), shi = edge_s(g, uhi);
  int a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  if (ys < ym && ye > ym) {
    const float umid = row_edge(g, ym), smid = edge_s(g, umid);
    if (!row_px_e(g, cb, ulo, umid, slo, smid, a0, a1)) a1 = a0;
    if (!row_px_e(g, cb, umid, uhi, smid, shi, b0, b1)) b1 = b0;
  } else if (ys < ym) {
    if (!row_px_e(g, cb, ulo, uhi, slo, shi, a0, a1)) a1 = a0;
  } else {
    if (!row_px_e(g, cb, ulo, uhi, slo, shi, b0, b1)) b1 = b0;
  }
  return (a0 < ox + 8 && a1 > ox && a1 > a0 ? 1u : 0u) | (a0 < ox + 16 && a1 > ox + 8 && a1 > a0 ? 2u : 0u) |
         (b0 < ox + 8 && b1 > ox && b1 > b0 ? 4u : 0u) | (b0 < ox + 16 && b1 > ox + 8 && b1 > b0 ? 8u : 0u);
}

}  // namespace rs
