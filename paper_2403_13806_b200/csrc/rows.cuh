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
// rectangles, 44% fewer on the anisotropic configs[4]. Used by segemit_kernel.
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

// Span of an ellipse row from its edge offsets and edge terms (slo = edge_s(ulo),
// shi = edge_s(uhi)); identical to oracle row_span: the clamped dyr / -dyr is one of
// lo, hi, +-dyr and the boundary term there is slo, shi or sd.
__device__ __forceinline__ bool row_span_e(const RowGeom& g, const int4 cb, float ulo, float uhi, float slo, float shi,
                                           int& tx0, int& tx1) {
  const float lo = fmaxf(ulo, -g.hy), hi = fminf(uhi, g.hy);
  if (!(lo <= hi)) return false;
  float ur, sr, ul, sl;
  if (g.dyr < lo) { ur = lo; sr = slo; } else if (g.dyr > hi) { ur = hi; sr = shi; } else { ur = g.dyr; sr = g.sd; }
  const float nd = -g.dyr;
  if (nd < lo) { ul = lo; sl = slo; } else if (nd > hi) { ul = hi; sl = shi; } else { ul = nd; sl = g.sd; }
  const float right = __fadd_rn(__fadd_rn(g.mx, __fadd_rn(__fmul_rn(g.bi, ur), __fmul_rn(sr, g.i2a))), 0.52f);
  const float left = __fsub_rn(__fadd_rn(g.mx, __fsub_rn(__fmul_rn(g.bi, ul), __fmul_rn(sl, g.i2a))), 0.52f);
  const int px0 = (int)fmaxf(floorf(__fsub_rn(left, 0.5f)), (float)cb.x);
  const int px1 = (int)fminf(__fadd_rn(floorf(__fsub_rn(right, 0.5f)), 1.0f), (float)cb.y);
  if (px1 <= px0) return false;
  tx0 = px0 / kTile;
  tx1 = (px1 - 1) / kTile;
  return true;
}

// Span of ellipse row ty (both edge terms evaluated here).
__device__ __forceinline__ bool row_span(const RowGeom& g, const int4 cb, int ty, int& tx0, int& tx1) {
  const float ulo = row_edge(g, max(ty * kTile, cb.z)), uhi = row_edge(g, min(ty * kTile + kTile, cb.w));
  return row_span_e(g, cb, ulo, uhi, edge_s(g, ulo), edge_s(g, uhi), tx0, tx1);
}

}  // namespace rs
