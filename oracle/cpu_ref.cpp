// cpu_ref.cpp -- CPU ORACLE for the render-and-prune hot path.
//
// TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2403_13806_b200/)
// links, loads or calls this file; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg use it, as the checker and
// as the CPU baseline.
//
// A scalar restatement of the reference NumPy rasterizer, instantiated three times:
//   * T = double  ("Tier B"): the reference's expressions in the reference's
//     order with std::exp, pinned against golden vectors produced by the
//     reference itself (tests/golden/make_golden.py).
//   * T = double, CT ("Tier C", the parity contract of the CUDA path's RS_F64
//     frames): Tier B's projection with exp64_contract (an exp from IEEE double
//     add/mul/fma only; device twin in csrc/rs_math.cuh) instead of std::exp;
//     the composite with fused roundings -- x = -q/2 as two fmas, a table exp
//     (exp64_tab: 1024-entry table + degree-3 polynomial) with its argument
//     clamped at 709 (an overflow guard),
//     rgb/depth += c w and tau (1 - alpha) as fmas -- and the pixel gate of the
//     fp32 tier's culling box (which drops only pixels with alpha < alpha_cut).
//     Tier C vs Tier B (and the reference): a few ulp (tests: <= 1e-12).
//   * T = float   ("Tier A", the parity contract for the CUDA path): the same
//     algorithm in fp32 with every operation and its order written out, no
//     FMA contraction except the explicit fmaf() calls (-ffp-contract=off),
//     IEEE division/sqrt, and an exp/exp2 built only from IEEE add/mul/fma so
//     the GPU reproduces it bit for bit (csrc/rs_math.cuh holds the device
//     twin of exp_contract/exp2_contract; they are kept identical on purpose).
//
// Reference lines followed (paths under /root/reference/pkg/src/fieldsplat):
//   projection          render.py:95-158  (+ core.py:111-139 quaternion,
//                       core.py:207-239 SH basis, core.py:288 colour offset,
//                       core.py:419-421 sigmoid, core.py:351-354 centre)
//   composite order     render.py:218-222 (lexsort (depth, index))
//   compositing         render.py:246-283 (threshold order :259-261, weight :267,
//                       contribution max :273-275, tau update :281)
//   per-pixel oracle    pkg/tests/oracles.py:15-61 (bbox gate :36-38)
//   filtered render     render.py:241-244
//   importance merge    render.py:84-88, pruning.py:75-95
// The tile binning (64-bit (tile, depth) keys, stable sort, per-tile ranges)
// has no reference counterpart; it is derived from the bbox of render.py:133-137
// and the order of render.py:218-222.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

constexpr int TILE = 16;

inline float fbits(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }
inline uint32_t ubits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }

// ---------------------------------------------------------------------------
// fp32 exponentials of the contract (device twin: csrc/rs_math.cuh)
// ---------------------------------------------------------------------------
const float MAGIC = 12582912.0f;  // 1.5 * 2^23: x + MAGIC rounds x to an integer (ties to even)

inline float pow2i(int n) { return fbits((uint32_t)(n + 127) << 23); }  // n in [-126, 127]

inline float scale2(float p, int n) {
  if (n >= -126 && n <= 127) return p * pow2i(n);
  int h = n / 2;  // both halves normal; the second product rounds once
  return (p * pow2i(h)) * pow2i(n - h);
}

// 2^x, |rel err| < 1.4 * 2^-24 on the reduced range; polynomial fitted offline.
inline float exp2_contract(float x) {
  if (x != x) return x;
  if (x >= 128.0f) return INFINITY;
  if (x < -150.0f) return 0.0f;
  float t = x + MAGIC;
  float n = t - MAGIC;
  float r = x - n;  // exact, |r| <= 0.5
  float p = fbits(0x3920e999u);
  p = std::fma(p, r, fbits(0x3aafa2b5u));
  p = std::fma(p, r, fbits(0x3c1d96deu));
  p = std::fma(p, r, fbits(0x3d63576au));
  p = std::fma(p, r, fbits(0x3e75fdedu));
  p = std::fma(p, r, fbits(0x3f317218u));
  p = std::fma(p, r, 1.0f);
  return scale2(p, (int)n);
}

// e^x with Cody-Waite reduction; used for exp(log_scale) and the sigmoid.
inline float exp_contract(float x) {
  if (x != x) return x;
  if (x >= 89.0f) return INFINITY;
  if (x < -104.0f) return 0.0f;
  float t = std::fma(x, fbits(0x3fb8aa3bu), MAGIC);  // rint(x * log2 e)
  float n = t - MAGIC;
  float r = std::fma(n, -fbits(0x3f317200u), x);  // ln2 hi
  r = std::fma(n, -fbits(0x35bfbe8eu), r);        // ln2 lo
  float p = fbits(0x3ab55cb8u);
  p = std::fma(p, r, fbits(0x3c09368du));
  p = std::fma(p, r, fbits(0x3d2aac4du));
  p = std::fma(p, r, fbits(0x3e2aaa05u));
  p = std::fma(p, r, fbits(0x3efffffdu));
  p = std::fma(p, r, 1.0f);
  p = std::fma(p, r, 1.0f);
  return scale2(p, (int)n);
}

// log2(x) for normal x > 0 (~1e-7 relative); used only for the conservative
// skip threshold cut2, but it also fixes the culling box that the tile binning
// uses, so it must be reproducible: add/mul/div/fma only (device twin in rs_math.cuh).
inline float log2_contract(float x) {
  if (x != x) return x;
  if (x <= 0.0f) return -INFINITY;
  if (x == INFINITY) return INFINITY;
  if (x < 1.17549435e-38f) return -150.0f;  // subnormal: a lower bound is enough (conservative)
  const uint32_t u = ubits(x);
  int e = (int)((u >> 23) & 0xffu) - 127;
  float m = fbits((u & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) { m = m * 0.5f; e += 1; }
  const float t = (m - 1.0f) / (m + 1.0f);
  const float t2 = t * t;
  float p = std::fma(t2, 0.111111112f, 0.142857149f);
  p = std::fma(p, t2, 0.200000003f);
  p = std::fma(p, t2, 0.333333343f);
  p = std::fma(p, t2, 1.0f);
  return std::fma(t * p, 2.88539004f, (float)e);
}

// e^x in double (device twin: exp64_contract in csrc/rs_math.cuh): n = rint(x log2 e)
// by the magic-number add, Cody-Waite r = x - n ln2, degree-12 Taylor in Horner form
// (|r| <= 0.347), times 2^n through the exponent field.
inline double pow2i64(int n) {  // n in [-1022, 1023]
  const uint64_t u = (uint64_t)(n + 1023) << 52;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
inline double exp64_contract(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.2) return 0.0;
  const double t = std::fma(x, 1.4426950408889634, 6755399441055744.0);
  const double n = t - 6755399441055744.0;
  double r = std::fma(n, -0.6931471803691238, x);
  r = std::fma(n, -1.9082149292705877e-10, r);
  double p = 1.0 / 479001600.0;
  p = std::fma(p, r, 1.0 / 39916800.0);
  p = std::fma(p, r, 1.0 / 3628800.0);
  p = std::fma(p, r, 1.0 / 362880.0);
  p = std::fma(p, r, 1.0 / 40320.0);
  p = std::fma(p, r, 1.0 / 5040.0);
  p = std::fma(p, r, 1.0 / 720.0);
  p = std::fma(p, r, 1.0 / 120.0);
  p = std::fma(p, r, 1.0 / 24.0);
  p = std::fma(p, r, 1.0 / 6.0);
  p = std::fma(p, r, 0.5);
  p = std::fma(p, r, 1.0);
  p = std::fma(p, r, 1.0);
  uint64_t tb;
  std::memcpy(&tb, &t, 8);
  const int ni = (int)(int32_t)(uint32_t)tb;  // n in the low word of t
  if (ni > 1023) return (p * pow2i64(1023)) * 2.0;
  if (ni >= -1022) return p * pow2i64(ni);
  return (p * pow2i64(ni + 600)) * pow2i64(-600);
}

// e^x of the fp64 contract's blend (device twin: exp64_tab in csrc/rs_math.cuh):
// k = rint(x 1024 / ln 2), r = x - k ln2/1024 (Cody-Waite), degree-3 Taylor, times
// T[k mod 1024] = exp64_contract(j ln2/1024) scaled by 2^(k div 1024) in the exponent field.
struct Exp64Tab {
  double T[1024];
  Exp64Tab() {
    for (int j = 0; j < 1024; ++j) T[j] = exp64_contract((double)j * (0.6931471805599453 / 1024.0));
  }
};
inline double with_exp(double t, int add) {  // t * 2^add by the exponent field (t normal, result normal)
  uint64_t u;
  std::memcpy(&u, &t, 8);
  u += (uint64_t)(int64_t)add << 52;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
inline double exp64_tab(double x) {
  static const Exp64Tab tab;
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.2) return 0.0;
  const double t = std::fma(x, 1477.3197218702985, 6755399441055744.0);
  const double kd = t - 6755399441055744.0;
  double r = std::fma(kd, -(0.6931471803691238 / 1024.0), x);
  r = std::fma(kd, -(1.9082149292705877e-10 / 1024.0), r);
  double p = std::fma(1.0 / 6.0, r, 0.5);
  p = std::fma(p, r, 1.0);
  p = std::fma(p, r, 1.0);
  uint64_t tb;
  std::memcpy(&tb, &t, 8);
  const int k = (int)(int32_t)(uint32_t)tb;
  const int n = k >> 10;
  const double tj = tab.T[k & 1023];
  if (n >= -1022) return p * with_exp(tj, n);
  return (p * with_exp(tj, n + 600)) * pow2i64(-600);
}

template <typename T> struct M;
template <> struct M<double> {
  static double exp(double x) { return std::exp(x); }
};
template <> struct M<float> {
  static float exp(float x) { return exp_contract(x); }
};
// the exp of a tier: CT = the fp64 contract (Tier C)
template <typename T, bool CT> inline T texp(T x) {
  if constexpr (CT) return (T)exp64_contract((double)x);
  else return M<T>::exp(x);
}

// order-preserving map of the fp32 depth to 32 key bits (-0 folded into +0)
inline uint32_t depth_key(float d) {
  uint32_t u = ubits(d + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <typename T> struct Cam {
  int W, H;
  T fx, fy, cx, cy, R[9], t[3], C[3];
  explicit Cam(const T* p) {
    W = (int)p[0]; H = (int)p[1];
    fx = p[2]; fy = p[3]; cx = p[4]; cy = p[5];
    for (int i = 0; i < 9; ++i) R[i] = p[6 + i];
    for (int i = 0; i < 3; ++i) { t[i] = p[15 + i]; C[i] = p[18 + i]; }
  }
};

template <typename T> struct Opts {
  T alpha_max, alpha_cut, tau_stop, near_limit, lowpass, sigma_bound;
  explicit Opts(const T* p)
      : alpha_max(p[0]), alpha_cut(p[1]), tau_stop(p[2]), near_limit(p[3]), lowpass(p[4]), sigma_bound(p[5]) {}
};

template <typename T> struct Scene {
  const T *pos, *logit, *sh, *ls, *quat;  // (n,3) (n) (n,3,16) (n,3) (n,4)
  int64_t n;
  int deg;
};

// one projected Gaussian (render.py:95-158 / ProjectedGaussian render.py:49-59)
template <typename T> struct PG {
  uint8_t valid;
  T mx, my, a, b, c, ia, ib, ic, radius, depth, color[3], opacity;
  int32_t x0, x1, y0, y1;
  float na, nb, nc;  // fp32 contract: -0.5*log2(e) * (ia, 2*ib, ic)
  float cut2;        // fp32 contract: p2 < cut2 => alpha < alpha_cut
  int32_t cx0, cx1, cy0, cy1;  // culling box (fp32 contract); == bbox for T = double
  uint8_t bin;       // binned: valid and the culling box is non-empty
  uint8_t ell;       // the culling box came from the ellipse (then tile rows use row_span)
  float rg_hy, rg_dyr, rg_ak4, rg_d, rg_bi, rg_i2a, rg_del;  // row_geom terms (ell only)
};

template <typename T> inline int64_t floor_clip(T v, int hi) {
  // np.clip(np.floor(v).astype(int64), 0, hi); NaN -> INT64_MIN -> 0
  if (v != v) return 0;
  T f = std::floor(v);
  if (f <= 0) return 0;
  if (f >= (T)hi) return hi;
  return (int64_t)f;
}
template <typename T> inline int64_t ceil1_clip(T v, int hi) {
  // np.clip(np.ceil(v).astype(int64) + 1, 0, hi)
  if (v != v) return 0;
  T f = std::ceil(v);
  if (f <= (T)-1) return 0;
  if (f >= (T)hi) return hi;
  return (int64_t)f + 1 > hi ? hi : (int64_t)f + 1;
}

template <typename T> inline void row_geom(PG<T>& g);

// Culling box of the fp32 contract (device twin: project.cuh). cut2 is a
// conservative bound (p2 < cut2 => o*2^p2 < alpha_cut); outside the ellipse
// {p2 >= cut2} widened by 1% + 0.5 px no pixel can reach alpha_cut even with
// the fp32 rounding of p2 (condition number <= 1e4; else the full bbox). The
// tile binning uses this box; Gaussians with an empty box are not binned.
template <typename T> inline void cull_box(PG<T>& g, float alpha_cut) {
  const float op = (float)g.opacity;
  float cut2 = alpha_cut > 0.0f ? log2_contract(alpha_cut / op) - 1e-3f : -INFINITY;
  if (alpha_cut >= 1e-30f && cut2 < -126.0f) cut2 = -126.0f;
  g.cut2 = cut2;
  const double Na = g.na, Nb = g.nb, Nc = g.nc, C2 = cut2;
  const double D = 4.0 * Na * Nc - Nb * Nb;
  const double tr = Na + Nc, sq = std::sqrt((Na - Nc) * (Na - Nc) + Nb * Nb);
  const double l1 = 0.5 * (tr - sq), l2 = 0.5 * (tr + sq);
  if (!(C2 < 0.0)) {
    g.cx1 = g.cx0;
    g.cy1 = g.cy0;
  } else if (C2 > -1e30 && D > 0.0 && l2 < 0.0 && l1 >= 1e4 * l2) {
    const double hx = std::sqrt(C2 * 4.0 * Nc / D) * 1.01 + 0.5, hy = std::sqrt(C2 * 4.0 * Na / D) * 1.01 + 0.5;
    const double mx = (float)g.mx, my = (float)g.my;
    g.cx0 = std::max(g.x0, (int32_t)std::fmax(std::floor(mx - hx - 0.5), -1.0));
    g.cx1 = std::min(g.x1, (int32_t)std::fmin(std::floor(mx + hx - 0.5) + 1.0, 65535.0));
    g.cy0 = std::max(g.y0, (int32_t)std::fmax(std::floor(my - hy - 0.5), -1.0));
    g.cy1 = std::min(g.y1, (int32_t)std::fmin(std::floor(my + hy - 0.5) + 1.0, 65535.0));
    if (g.cx1 < g.cx0) g.cx1 = g.cx0;
    if (g.cy1 < g.cy0) g.cy1 = g.cy0;
    g.ell = 1;
    row_geom(g);
  }
  g.bin = g.valid && g.cx1 > g.cx0 && g.cy1 > g.cy0;
}

// Tile columns [tx0, tx1] of tile row ty that a binned Gaussian is listed in
// (device twin: rows.cuh). For an ellipse-derived culling box this is the
// x-extent, over the strip of the row's pixel centres dilated by 0.5 px, of
// the ellipse {p2 >= cut2} scaled by 1.01 (q = -p2 <= 1.0201 K) and dilated
// by 0.5 px -- the conservative region whose bounding box is the culling box
// -- so no dropped tile holds a pixel that can reach alpha_cut. The x-extent
// of an ellipse over a strip is attained at the strip point nearest the
// ellipse's rightmost (leftmost) point: the boundary x(dy) is concave
// (convex). Float arithmetic (D = 4 A Cc - B^2 is formed in double: it
// cancels for elongated ellipses) with explicit slack for the rounding: +1e-5
// relative on the half-height, +4e-6 * 4AK under the square roots (the
// argument's rounding error is a few ulp of 4AK: dy is a correctly rounded
// difference and every factor carries a few ulp), +0.02 px on each side. Otherwise (degenerate / ill-conditioned ellipse) the full row.
template <typename T> inline void row_geom(PG<T>& g) {
  // D = 4 A Cc - B^2 cancels for elongated ellipses: formed in double, then rounded once
  const double Nad = g.na, Nbd = g.nb, Ncd = g.nc;
  const float D = (float)(4.0 * Nad * Ncd - Nbd * Nbd);
  const float A = -g.na, B = -g.nb, Cc = -g.nc;  // q = A dx^2 + B dx dy + Cc dy^2 = -p2
  const float K = g.cut2 * -1.0201f;
  const float AK4 = 4.0f * A * K;
  g.rg_hy = std::sqrt(AK4 / D) * 1.00001f;
  const float hx = std::sqrt(4.0f * Cc * K / D);
  g.rg_dyr = -B * hx / (2.0f * Cc);  // dy of the rightmost point; the leftmost is at -dyr
  g.rg_ak4 = AK4;
  g.rg_d = D;
  g.rg_i2a = 1.0f / (2.0f * A);
  g.rg_bi = -B * g.rg_i2a;  // x(dy) = bi dy +- sqrt(4AK - D dy^2) / (2A)
  g.rg_del = AK4 * 4e-6f;
}

template <typename T> inline bool row_span(const PG<T>& g, int ty, int* tx0, int* tx1) {
  if (!g.ell) {
    *tx0 = g.cx0 / TILE;
    *tx1 = (g.cx1 - 1) / TILE;
    return true;
  }
  const float mx = (float)g.mx, my = (float)g.my;
  const int ys = std::max(ty * TILE, g.cy0), ye = std::min(ty * TILE + TILE, g.cy1);
  const float lo = std::fmax((float)ys - my, -g.rg_hy), hi = std::fmin((float)ye - my, g.rg_hy);
  if (!(lo <= hi)) return false;
  const float ur = std::fmin(std::fmax(g.rg_dyr, lo), hi), ul = std::fmin(std::fmax(-g.rg_dyr, lo), hi);
  const float sr = std::sqrt(std::fmax(g.rg_ak4 - g.rg_d * ur * ur, 0.0f) + g.rg_del);
  const float sl = std::sqrt(std::fmax(g.rg_ak4 - g.rg_d * ul * ul, 0.0f) + g.rg_del);
  const float right = mx + (g.rg_bi * ur + sr * g.rg_i2a) + 0.52f;
  const float left = mx + (g.rg_bi * ul - sl * g.rg_i2a) - 0.52f;
  const int px0 = (int)std::fmax(std::floor(left - 0.5f), (float)g.cx0);
  const int px1 = (int)std::fmin(std::floor(right - 0.5f) + 1.0f, (float)g.cx1);
  if (px1 <= px0) return false;
  *tx0 = px0 / TILE;
  *tx1 = (px1 - 1) / TILE;
  return true;
}

template <typename T, bool CT = false>
PG<T> project_one(const Scene<T>& s, int64_t i, const Cam<T>& cam, const Opts<T>& o) {
  PG<T> g;
  const T px = s.pos[3 * i], py = s.pos[3 * i + 1], pz = s.pos[3 * i + 2];
  // t = R p + T  (render.py:100)
  T t[3];
  for (int k = 0; k < 3; ++k) t[k] = ((cam.R[3 * k] * px + cam.R[3 * k + 1] * py) + cam.R[3 * k + 2] * pz) + cam.t[k];
  const bool valid0 = t[2] > o.near_limit;
  const T tz = valid0 ? t[2] : (T)1;
  g.mx = (cam.fx * t[0]) / tz + cam.cx;  // render.py:104-105
  g.my = (cam.fy * t[1]) / tz + cam.cy;
  g.depth = t[2] + (T)0;
  // quaternion -> rotation (core.py:111-139)
  T qw = s.quat[4 * i], qx = s.quat[4 * i + 1], qy = s.quat[4 * i + 2], qz = s.quat[4 * i + 3];
  const T qn = std::sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
  qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn;
  T Rq[9];
  Rq[0] = (T)1 - (T)2 * (qy * qy + qz * qz);
  Rq[1] = (T)2 * (qx * qy - qw * qz);
  Rq[2] = (T)2 * (qx * qz + qw * qy);
  Rq[3] = (T)2 * (qx * qy + qw * qz);
  Rq[4] = (T)1 - (T)2 * (qx * qx + qz * qz);
  Rq[5] = (T)2 * (qy * qz - qw * qx);
  Rq[6] = (T)2 * (qx * qz - qw * qy);
  Rq[7] = (T)2 * (qy * qz + qw * qx);
  Rq[8] = (T)1 - (T)2 * (qx * qx + qy * qy);
  // Sigma = L L^T, L = Rq diag(exp(log_s))  (render.py:108-111)
  T sc[3];
  for (int j = 0; j < 3; ++j) sc[j] = texp<T, CT>(s.ls[3 * i + j]);
  T L[9];
  for (int r = 0; r < 3; ++r)
    for (int j = 0; j < 3; ++j) L[3 * r + j] = Rq[3 * r + j] * sc[j];
  T S[9];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) S[3 * r + k] = (L[3 * r] * L[3 * k] + L[3 * r + 1] * L[3 * k + 1]) + L[3 * r + 2] * L[3 * k + 2];
  // Jacobian and A = J R_cam  (render.py:114-119); J01 = J10 = 0 exactly
  const T j00 = cam.fx / tz, j02 = (-cam.fx * t[0]) / (tz * tz);
  const T j11 = cam.fy / tz, j12 = (-cam.fy * t[1]) / (tz * tz);
  T A[6];
  for (int k = 0; k < 3; ++k) {
    A[k] = j00 * cam.R[k] + j02 * cam.R[6 + k];
    A[3 + k] = j11 * cam.R[3 + k] + j12 * cam.R[6 + k];
  }
  // cov2d = (A Sigma) A^T  (render.py:120)
  T MS[6];
  for (int r = 0; r < 2; ++r)
    for (int k = 0; k < 3; ++k) MS[3 * r + k] = (A[3 * r] * S[k] + A[3 * r + 1] * S[3 + k]) + A[3 * r + 2] * S[6 + k];
  const T c00 = (MS[0] * A[0] + MS[1] * A[1]) + MS[2] * A[2];
  const T c01 = (MS[0] * A[3] + MS[1] * A[4]) + MS[2] * A[5];
  const T c11 = (MS[3] * A[3] + MS[4] * A[4]) + MS[5] * A[5];
  g.a = c00 + o.lowpass;  // render.py:121-123
  g.b = c01;
  g.c = c11 + o.lowpass;
  const T det = g.a * g.c - g.b * g.b;  // render.py:125-128
  g.ia = g.c / det;
  g.ib = -g.b / det;
  g.ic = g.a / det;
  const T amc = g.a - g.c;  // render.py:130-131
  const T disc = (T)0.25 * (amc * amc) + g.b * g.b;
  const T lam = (T)0.5 * (g.a + g.c) + std::sqrt(disc > (T)0 ? disc : (T)0);
  g.radius = o.sigma_bound * std::sqrt(lam > (T)0 ? lam : (T)0);
  g.x0 = (int32_t)floor_clip(g.mx - g.radius, cam.W);  // render.py:133-137
  g.x1 = (int32_t)ceil1_clip(g.mx + g.radius, cam.W);
  g.y0 = (int32_t)floor_clip(g.my - g.radius, cam.H);
  g.y1 = (int32_t)ceil1_clip(g.my + g.radius, cam.H);
  g.valid = valid0 && g.x1 > g.x0 && g.y1 > g.y0;
  // view-direction SH colour (render.py:139-149, core.py:207-239)
  const T vx = px - cam.C[0], vy = py - cam.C[1], vz = pz - cam.C[2];
  T vn = std::sqrt((vx * vx + vy * vy) + vz * vz);
  if (!(vn > (T)0)) vn = (T)1;
  const T x = vx / vn, y = vy / vn, z = vz / vn;
  T Y[16];
  Y[0] = (T)0.28209479177387814;
  if (s.deg >= 1) {
    const T C1 = (T)0.4886025119029199;
    Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
  }
  const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  if (s.deg >= 2) {
    Y[4] = (T)1.0925484305920792 * xy;
    Y[5] = (T)-1.0925484305920792 * yz;
    Y[6] = (T)0.31539156525252005 * (((T)2 * zz - xx) - yy);
    Y[7] = (T)-1.0925484305920792 * xz;
    Y[8] = (T)0.5462742152960396 * (xx - yy);
  }
  if (s.deg >= 3) {
    Y[9] = ((T)-0.5900435899266435 * y) * ((T)3 * xx - yy);
    Y[10] = ((T)2.890611442640554 * xy) * z;
    Y[11] = ((T)-0.4570457994644658 * y) * (((T)4 * zz - xx) - yy);
    Y[12] = ((T)0.3731763325901154 * z) * (((T)2 * zz - (T)3 * xx) - (T)3 * yy);
    Y[13] = ((T)-0.4570457994644658 * x) * (((T)4 * zz - xx) - yy);
    Y[14] = ((T)1.445305721320277 * z) * (xx - yy);
    Y[15] = ((T)-0.5900435899266435 * x) * (xx - (T)3 * yy);
  }
  const int nb = (s.deg == 0) ? 1 : (s.deg == 1) ? 4 : (s.deg == 2) ? 9 : 16;
  for (int ch = 0; ch < 3; ++ch) {
    const T* shc = s.sh + 48 * i + 16 * ch;
    T acc = shc[0] * Y[0];
    for (int b = 1; b < nb; ++b) acc = acc + shc[b] * Y[b];
    const T pre = (T)0.5 + acc;
    g.color[ch] = pre < (T)0 ? (T)0 : (pre > (T)1 ? (T)1 : pre);
  }
  // opacity = sigmoid(logit) (core.py:419-421)
  const T lg = s.logit[i];
  if (lg >= (T)0) {
    g.opacity = (T)1 / ((T)1 + texp<T, CT>(-lg));
  } else {
    const T e = texp<T, CT>(lg);
    g.opacity = e / ((T)1 + e);
  }
  const float K = fbits(0xbf38aa3bu);  // -0.5 * log2(e)
  g.na = K * (float)g.ia;
  g.nb = (2.0f * K) * (float)g.ib;
  g.nc = K * (float)g.ic;
  g.cx0 = g.x0; g.cx1 = g.x1; g.cy0 = g.y0; g.cy1 = g.y1;
  g.cut2 = -INFINITY;
  g.bin = g.valid;
  g.ell = 0;
  if ((sizeof(T) == 4 || CT) && g.valid) cull_box(g, (float)o.alpha_cut);
  return g;
}

template <typename T, bool CT = false>
std::vector<PG<T>> project_all(const Scene<T>& s, const Cam<T>& cam, const Opts<T>& o) {
  std::vector<PG<T>> v((size_t)s.n);
  for (int64_t i = 0; i < s.n; ++i) v[(size_t)i] = project_one<T, CT>(s, i, cam, o);
  return v;
}

// (depth, index) order over valid (and active) Gaussians (render.py:218-222, :243-244)
template <typename T>
std::vector<int64_t> composite_order(const std::vector<PG<T>>& pg, const uint8_t* active) {
  std::vector<int64_t> idx;
  for (size_t i = 0; i < pg.size(); ++i)
    if (pg[i].bin && (!active || active[i])) idx.push_back((int64_t)i);
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return pg[a].depth < pg[b].depth; });
  return idx;
}

struct Counters { int64_t E = 0, C = 0; };

// max-merge that is safe when several threads composite different tiles
template <typename T> inline void atomic_max(T* p, T v) {
  std::atomic_ref<T> a(*p);
  T cur = a.load(std::memory_order_relaxed);
  while (v > cur && !a.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
  }
}

// Per-pixel evaluation of one Gaussian: returns alpha (render.py:255-259).
template <typename T, bool CT = false> inline T pixel_alpha(const PG<T>& g, T xs, T ys, T alpha_max);
template <> inline double pixel_alpha<double, true>(const PG<double>& g, double xs, double ys, double alpha_max) {
  // Tier C: -q/2 of render.py:254-256 with fused roundings, (na, nb, nc) = -(ia/2, ib, ic/2)
  // (exact scalings), the table exp, argument clamped at 709
  const double na = -0.5 * g.ia, nb = -g.ib, nc = -0.5 * g.ic;
  const double dx = xs - g.mx, dy = ys - g.my;
  const double x = std::fma(nc * dy, dy, std::fma(nb * dy, dx, (na * dx) * dx));
  const double raw = g.opacity * exp64_tab(x > 709.0 ? 709.0 : x);
  return (raw != raw || raw < alpha_max) ? raw : alpha_max;
}
template <> inline double pixel_alpha<double, false>(const PG<double>& g, double xs, double ys, double alpha_max) {
  const double dx = xs - g.mx, dy = ys - g.my;
  const double q = (g.ia * dx * dx) + (2.0 * g.ib) * dy * dx + (g.ic * dy * dy);
  const double raw = g.opacity * std::exp(-0.5 * q);
  return (raw != raw || raw < alpha_max) ? raw : alpha_max;  // np.minimum propagates NaN
}
template <> inline float pixel_alpha<float, false>(const PG<float>& g, float xs, float ys, float alpha_max) {
  const float dx = xs - g.mx, dy = ys - g.my;
  const float p2 = std::fma(g.na * dx, dx, std::fma(g.nb * dy, dx, (g.nc * dy) * dy));
  // 2^min(p2, 127): an overflow guard (o * 2^127 saturates alpha_max for any o >= 5.8e-39)
  const float raw = g.opacity * exp2_contract(p2 < 127.0f || p2 != p2 ? p2 : 127.0f);
  return (raw != raw || raw < alpha_max) ? raw : alpha_max;  // np.minimum propagates NaN
}

template <typename T> inline T mac(T c, T w, T acc);
template <> inline double mac<double>(double c, double w, double acc) { return acc + c * w; }
template <> inline float mac<float>(float c, float w, float acc) { return std::fma(c, w, acc); }

struct Out {
  void* img;      // (H,W,3) T or null
  void* alpha;    // (H,W) T or null
  void* depth;    // (H,W) T or null
  int32_t* count; // (H,W) or null
  void* contrib;  // (n) T, max-merged in place, or null
};

// Composite one pixel over a front-to-back list (oracles.py:32-59 semantics).
template <typename T, bool CT = false>
inline void composite_pixel(const std::vector<PG<T>>& pg, const int64_t* list, size_t len, int x, int y,
                            const Opts<T>& o, T* rgbd, T& tau_out, int32_t& cnt, T* contrib, Counters& k) {
  const T xs = (T)x + (T)0.5, ys = (T)y + (T)0.5;
  T tau = 1, r = 0, gg = 0, b = 0, d = 0;
  int32_t c = 0;
  for (size_t j = 0; j < len; ++j) {
    if (tau < o.tau_stop) break;  // nothing composites once tau < tau_stop (render.py:261)
    const PG<T>& g = pg[(size_t)list[j]];
    // bbox gate (oracles.py:36-38); the culling box lies inside the bbox and only drops
    // pixels that cannot reach alpha_cut, so gating with it changes no result
    if (!(g.cx0 <= x && x < g.cx1 && g.cy0 <= y && y < g.cy1)) continue;
    ++k.E;
    const T alpha = pixel_alpha<T, CT>(g, xs, ys, o.alpha_max);
    if (alpha >= o.alpha_cut && tau >= o.tau_stop) {
      const T w = alpha * tau;  // render.py:267
      if constexpr (CT) {  // Tier C: fused accumulation and transmittance update
        r = std::fma(g.color[0], w, r);
        gg = std::fma(g.color[1], w, gg);
        b = std::fma(g.color[2], w, b);
        d = std::fma(g.depth, w, d);
      } else {
        r = mac<T>(g.color[0], w, r);
        gg = mac<T>(g.color[1], w, gg);
        b = mac<T>(g.color[2], w, b);
        d = mac<T>(g.depth, w, d);
      }
      if (contrib) atomic_max(contrib + list[j], w);  // render.py:273-275
      ++c;
      ++k.C;
      if constexpr (CT) tau = std::fma(-alpha, tau, tau);
      else tau = tau * ((T)1 - alpha);  // render.py:281
    }
  }
  rgbd[0] = r; rgbd[1] = gg; rgbd[2] = b; rgbd[3] = d;
  tau_out = tau;
  cnt = c;
}

// Tile binning: 64-bit keys (tile << 32 | depth_key), emitted in index order,
// stable-sorted (fp64 tiers: by tile, then the fp64 depth -- the fp32 depth key
// can tie where the fp64 depths differ); ranges[t] = [start, end). Returns the
// pair count.
template <typename T>
int64_t bin_tiles(const std::vector<PG<T>>& pg, const uint8_t* active, int W, int H, std::vector<uint64_t>* keys,
                  std::vector<uint32_t>* vals, std::vector<uint32_t>* ranges) {
  const int TW = (W + TILE - 1) / TILE, TH = (H + TILE - 1) / TILE;
  std::vector<std::pair<uint64_t, uint32_t>> pairs;
  for (size_t i = 0; i < pg.size(); ++i) {
    const PG<T>& g = pg[i];
    if (!g.bin || (active && !active[i])) continue;
    const uint64_t dk = depth_key((float)g.depth);
    int a, b;
    for (int ty = g.cy0 / TILE; ty <= (g.cy1 - 1) / TILE; ++ty)
      if (row_span(g, ty, &a, &b))
        for (int tx = a; tx <= b; ++tx) pairs.emplace_back(((uint64_t)(ty * TW + tx) << 32) | dk, (uint32_t)i);
  }
  if constexpr (sizeof(T) == 4) {
    std::stable_sort(pairs.begin(), pairs.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  } else {  // fp64 tiers: (tile, fp64 depth), index order on ties -- the reference's order per tile
    std::stable_sort(pairs.begin(), pairs.end(), [&](const auto& a, const auto& b) {
      const uint64_t ta = a.first >> 32, tb = b.first >> 32;
      return ta != tb ? ta < tb : pg[a.second].depth < pg[b.second].depth;
    });
  }
  keys->resize(pairs.size());
  vals->resize(pairs.size());
  ranges->assign(2 * (size_t)TW * TH, 0);
  for (size_t p = 0; p < pairs.size(); ++p) {
    (*keys)[p] = pairs[p].first;
    (*vals)[p] = pairs[p].second;
  }
  for (size_t p = 0; p < pairs.size(); ++p) {
    const uint32_t t = (uint32_t)(pairs[p].first >> 32);
    if (p == 0 || (uint32_t)(pairs[p - 1].first >> 32) != t) (*ranges)[2 * t] = (uint32_t)p;
    (*ranges)[2 * t + 1] = (uint32_t)p + 1;
  }
  return (int64_t)pairs.size();
}

// Run fn(worker) on `threads` workers (worker 0 is the caller).
template <typename F> void parallel(int threads, F fn) {
  if (threads <= 1) { fn(0); return; }
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(fn, t);
  fn(0);
  for (auto& th : pool) th.join();
}

template <typename T, bool CT = false>
std::vector<PG<T>> project_par(const Scene<T>& s, const Cam<T>& cam, const Opts<T>& o, int threads) {
  std::vector<PG<T>> v((size_t)s.n);
  const int64_t per = (s.n + threads - 1) / std::max(threads, 1);
  parallel(threads, [&](int t) {
    const int64_t lo = t * per, hi = std::min<int64_t>(s.n, lo + per);
    for (int64_t i = lo; i < hi; ++i) v[(size_t)i] = project_one<T, CT>(s, i, cam, o);
  });
  return v;
}

// Full render of one view. method 0 = per-tile lists (the global (depth, index)
// order restricted to each tile: identical per-pixel walk), 1 = the global
// list per pixel (oracles.py literal). `threads` splits projection, tile-list
// construction (bands of tile rows) and compositing (tiles); contributions
// merge by an atomic max, which is order independent (render.py:71-76).
template <typename T, bool CT = false>
void render(const Scene<T>& s, const T* camp, const T* optp, const uint8_t* active, int method, Out out,
            Counters* kc, int threads = 1) {
  const Cam<T> cam(camp);
  const Opts<T> o(optp);
  threads = std::max(threads, 1);
  const std::vector<PG<T>> pg = project_par<T, CT>(s, cam, o, threads);
  T* contrib = (T*)out.contrib;
  const int W = cam.W, H = cam.H;
  auto store = [&](int x, int y, const T* rgbd, T tau, int32_t c) {
    const size_t p = (size_t)y * W + x;
    if (out.img) { T* im = (T*)out.img; im[3 * p] = rgbd[0]; im[3 * p + 1] = rgbd[1]; im[3 * p + 2] = rgbd[2]; }
    if (out.alpha) ((T*)out.alpha)[p] = (T)1 - tau;
    if (out.depth) ((T*)out.depth)[p] = rgbd[3];
    if (out.count) out.count[p] = c;
  };
  const std::vector<int64_t> order = composite_order(pg, active);
  std::vector<Counters> kk(threads);
  if (method == 1) {
    std::atomic<int> next(0);
    parallel(threads, [&](int t) {
      T rgbd[4], tau;
      int32_t c;
      for (int y; (y = next.fetch_add(1)) < H;)
        for (int x = 0; x < W; ++x) {
          composite_pixel<T, CT>(pg, order.data(), order.size(), x, y, o, rgbd, tau, c, contrib, kk[t]);
          store(x, y, rgbd, tau, c);
        }
    });
  } else {
    const int TW = (W + TILE - 1) / TILE, TH = (H + TILE - 1) / TILE;
    std::vector<std::vector<int64_t>> lists((size_t)TW * TH);
    const int rows_per = (TH + threads - 1) / threads;
    parallel(threads, [&](int t) {
      const int r0 = t * rows_per, r1 = std::min(TH, r0 + rows_per);
      if (r0 >= r1) return;
      for (const int64_t g : order) {
        const PG<T>& q = pg[(size_t)g];
        const int ty0 = std::max(q.cy0 / TILE, r0), ty1 = std::min((q.cy1 - 1) / TILE, r1 - 1);
        int a, b;
        for (int ty = ty0; ty <= ty1; ++ty)
          if (row_span(q, ty, &a, &b))
            for (int tx = a; tx <= b; ++tx) lists[(size_t)ty * TW + tx].push_back(g);
      }
    });
    std::atomic<int> next(0);
    parallel(threads, [&](int t) {
      T rgbd[4], tau;
      int32_t c;
      for (int tile; (tile = next.fetch_add(1)) < TW * TH;) {
        const std::vector<int64_t>& list = lists[(size_t)tile];
        const int tx = tile % TW, ty = tile / TW;
        for (int y = ty * TILE; y < std::min(H, ty * TILE + TILE); ++y)
          for (int x = tx * TILE; x < std::min(W, tx * TILE + TILE); ++x) {
            composite_pixel<T, CT>(pg, list.data(), list.size(), x, y, o, rgbd, tau, c, contrib, kk[t]);
            store(x, y, rgbd, tau, c);
          }
      }
    });
  }
  if (kc)
    for (const Counters& k : kk) { kc->E += k.E; kc->C += k.C; }
}

template <typename T> Scene<T> mkscene(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat, int64_t n, int deg) {
  Scene<T> s; s.pos = pos; s.logit = logit; s.sh = sh; s.ls = ls; s.quat = quat; s.n = n; s.deg = deg;
  return s;
}

// CPU-baseline driver: views one after another, each rendered by all threads
// (so a bounded sample of a few views still uses every core); scores merge by
// max across views (pruning.py:80-82).
template <typename T, bool CT = false>
void views(const Scene<T>& s, const T* cams, int64_t n_views, const T* optp, int threads, int want_images,
           T* contrib, T* img_last, int64_t* counters) {
  Counters kc;
  std::vector<T> img;
  for (int64_t v = 0; v < n_views; ++v) {
    const T* cp = cams + 21 * v;
    const int W = (int)cp[0], H = (int)cp[1];
    Out out{};
    if (want_images) {
      img.assign((size_t)W * H * 3, (T)0);
      out.img = img.data();
    }
    out.contrib = contrib;
    render<T, CT>(s, cp, optp, nullptr, 0, out, &kc, threads);
    if (img_last && v == n_views - 1) std::memcpy(img_last, img.data(), img.size() * sizeof(T));
  }
  if (counters) { counters[0] += kc.E; counters[1] += kc.C; }
}

// flat projection export for the tests (ctypes)
struct ProjOut {
  uint8_t* valid; void *mx, *my, *a, *b, *c, *ia, *ib, *ic, *radius, *depth, *color, *opacity;
  int32_t *x0, *x1, *y0, *y1;
  float *na, *nb, *nc, *cut2;
  int32_t *cx0, *cx1, *cy0, *cy1;
  uint8_t* bin;
  uint8_t* ell;
};

template <typename T>
void export_proj(const std::vector<PG<T>>& pg, ProjOut* po) {
  for (size_t i = 0; i < pg.size(); ++i) {
    const PG<T>& g = pg[i];
    po->valid[i] = g.valid;
    ((T*)po->mx)[i] = g.mx; ((T*)po->my)[i] = g.my;
    ((T*)po->a)[i] = g.a; ((T*)po->b)[i] = g.b; ((T*)po->c)[i] = g.c;
    ((T*)po->ia)[i] = g.ia; ((T*)po->ib)[i] = g.ib; ((T*)po->ic)[i] = g.ic;
    ((T*)po->radius)[i] = g.radius; ((T*)po->depth)[i] = g.depth;
    for (int c = 0; c < 3; ++c) ((T*)po->color)[3 * i + c] = g.color[c];
    ((T*)po->opacity)[i] = g.opacity;
    po->x0[i] = g.x0; po->x1[i] = g.x1; po->y0[i] = g.y0; po->y1[i] = g.y1;
    po->na[i] = g.na; po->nb[i] = g.nb; po->nc[i] = g.nc; po->cut2[i] = g.cut2;
    po->cx0[i] = g.cx0; po->cx1[i] = g.cx1; po->cy0[i] = g.cy0; po->cy1[i] = g.cy1; po->bin[i] = g.bin;
    po->ell[i] = g.ell;
  }
}

}  // namespace

#define ORC_DEFINE(SUF, T, CT)                                                                                       \
  extern "C" void orc_project_##SUF(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat,       \
                                    int64_t n, int deg, const T* cam, const T* opts, ProjOut* po) {              \
    export_proj(project_all<T, CT>(mkscene(pos, logit, sh, ls, quat, n, deg), Cam<T>(cam), Opts<T>(opts)), po); \
  }                                                                                                              \
  extern "C" int64_t orc_order_##SUF(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat,     \
                                     int64_t n, int deg, const T* cam, const T* opts, const uint8_t* active,     \
                                     int64_t* order) {                                                           \
    auto pg = project_all<T, CT>(mkscene(pos, logit, sh, ls, quat, n, deg), Cam<T>(cam), Opts<T>(opts));       \
    auto v = composite_order(pg, active);                                                                        \
    std::copy(v.begin(), v.end(), order);                                                                        \
    return (int64_t)v.size();                                                                                    \
  }                                                                                                              \
  extern "C" int64_t orc_bin_##SUF(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat,       \
                                   int64_t n, int deg, const T* cam, const T* opts, const uint8_t* active,       \
                                   uint64_t* keys, uint32_t* vals, uint32_t* ranges, int64_t cap) {              \
    const Cam<T> c(cam);                                                                                         \
    auto pg = project_all<T, CT>(mkscene(pos, logit, sh, ls, quat, n, deg), c, Opts<T>(opts));                 \
    std::vector<uint64_t> k; std::vector<uint32_t> v, r;                                                         \
    const int64_t P = bin_tiles(pg, active, c.W, c.H, &k, &v, &r);                                               \
    if (P <= cap) { std::copy(k.begin(), k.end(), keys); std::copy(v.begin(), v.end(), vals); }                  \
    std::copy(r.begin(), r.end(), ranges);                                                                       \
    return P;                                                                                                    \
  }                                                                                                              \
  extern "C" void orc_render_##SUF(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat,       \
                                   int64_t n, int deg, const T* cam, const T* opts, const uint8_t* active,       \
                                   int method, T* img, T* alpha, T* depth, int32_t* count, T* contrib,           \
                                   int64_t* counters) {                                                          \
    Out o{img, alpha, depth, count, contrib};                                                                    \
    Counters k;                                                                                                  \
    render<T, CT>(mkscene(pos, logit, sh, ls, quat, n, deg), cam, opts, active, method, o, &k);                  \
    if (counters) { counters[0] = k.E; counters[1] = k.C; }                                                      \
  }                                                                                                              \
  extern "C" void orc_views_##SUF(const T* pos, const T* logit, const T* sh, const T* ls, const T* quat,        \
                                  int64_t n, int deg, const T* cams, int64_t n_views, const T* opts,             \
                                  int threads, int want_images, T* contrib, T* img_last, int64_t* counters) {    \
    views<T, CT>(mkscene(pos, logit, sh, ls, quat, n, deg), cams, n_views, opts, threads, want_images, contrib,   \
             img_last, counters);                                                                                \
  }

ORC_DEFINE(f32, float, false)
ORC_DEFINE(f64, double, false)
ORC_DEFINE(c64, double, true)

// scalar access to the contract exponentials (device bit-compare tests)
extern "C" void orc_exp2_contract(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp2_contract(x[i]);
}
extern "C" void orc_exp64_contract(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp64_contract(x[i]);
}
extern "C" void orc_exp_contract(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp_contract(x[i]);
}
extern "C" uint32_t orc_depth_key(float d) { return depth_key(d); }
extern "C" void orc_log2_contract(const float* x, float* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = log2_contract(x[i]);
}
