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
// rectangles, 44% fewer on the anisotropic configs[4].
#pragma once
#include "rs_common.cuh"

namespace rs {

struct RowGeom {
  float mx, my, hy, dyr, ak4, d, bi, i2a, del;
};

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
  return g;
}

// cb = culling box (cx0, cx1, cy0, cy1); false = the row lists no tile.
__device__ __forceinline__ bool row_span(const RowGeom& g, const int4 cb, bool ell, int ty, int& tx0, int& tx1) {
  if (!ell) {
    tx0 = cb.x / kTile;
    tx1 = (cb.y - 1) / kTile;
    return true;
  }
  const int ys = max(ty * kTile, cb.z), ye = min(ty * kTile + kTile, cb.w);
  const float lo = fmaxf(__fsub_rn((float)ys, g.my), -g.hy), hi = fminf(__fsub_rn((float)ye, g.my), g.hy);
  if (!(lo <= hi)) return false;
  const float ur = fminf(fmaxf(g.dyr, lo), hi), ul = fminf(fmaxf(-g.dyr, lo), hi);
  const float sr = __fsqrt_rn(__fadd_rn(fmaxf(__fsub_rn(g.ak4, __fmul_rn(__fmul_rn(g.d, ur), ur)), 0.0f), g.del));
  const float sl = __fsqrt_rn(__fadd_rn(fmaxf(__fsub_rn(g.ak4, __fmul_rn(__fmul_rn(g.d, ul), ul)), 0.0f), g.del));
  const float right = __fadd_rn(__fadd_rn(g.mx, __fadd_rn(__fmul_rn(g.bi, ur), __fmul_rn(sr, g.i2a))), 0.52f);
  const float left = __fsub_rn(__fadd_rn(g.mx, __fsub_rn(__fmul_rn(g.bi, ul), __fmul_rn(sl, g.i2a))), 0.52f);
  const int px0 = (int)fmaxf(floorf(__fsub_rn(left, 0.5f)), (float)cb.x);
  const int px1 = (int)fminf(__fadd_rn(floorf(__fsub_rn(right, 0.5f)), 1.0f), (float)cb.y);
  if (px1 <= px0) return false;
  tx0 = px0 / kTile;
  tx1 = (px1 - 1) / kTile;
  return true;
}

// Pairs a binned record emits: the sum of its rows' spans.
__device__ __forceinline__ uint32_t record_tiles(const float4 a, const float4 b, const int4 d) {
  const int4 cb = cullbox_of(d);
  const bool ell = cullbox_ell(d);
  if (!ell) return (uint32_t)(((cb.y - 1) / kTile - cb.x / kTile + 1) * ((cb.w - 1) / kTile - cb.z / kTile + 1));
  const RowGeom g = row_geom(a, b);
  uint32_t n = 0;
  for (int ty = cb.z / kTile; ty <= (cb.w - 1) / kTile; ++ty) {
    int t0, t1;
    if (row_span(g, cb, true, ty, t0, t1)) n += (uint32_t)(t1 - t0 + 1);
  }
  return n;
}

}  // namespace rs
