// rs_math.cuh -- fp32 arithmetic of the parity contract, device side.
//
// Every function here is the device twin of the same-named function in
// oracle/cpu_ref.cpp and must stay operation-for-operation identical: only
// IEEE-rounded add/mul/div/sqrt and explicit fused multiply-adds, so the GPU
// result equals the CPU oracle bit for bit. The library is compiled with
// -fmad=false so the compiler cannot contract a*b+c behind our back; every
// intended fusion is an explicit __fmaf_rn.
#pragma once
#include <cstdint>

namespace rs {

__device__ __forceinline__ float fbits(uint32_t u) { return __uint_as_float(u); }

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23

__device__ __forceinline__ float pow2i(int n) { return __int_as_float((n + 127) << 23); }

__device__ __forceinline__ float scale2(float p, int n) {
  if (n >= -126 && n <= 127) return __fmul_rn(p, pow2i(n));
  const int h = n / 2;
  return __fmul_rn(__fmul_rn(p, pow2i(h)), pow2i(n - h));
}

__device__ __forceinline__ float exp2_poly(float r) {
  float p = fbits(0x3920e999u);
  p = __fmaf_rn(p, r, fbits(0x3aafa2b5u));
  p = __fmaf_rn(p, r, fbits(0x3c1d96deu));
  p = __fmaf_rn(p, r, fbits(0x3d63576au));
  p = __fmaf_rn(p, r, fbits(0x3e75fdedu));
  p = __fmaf_rn(p, r, fbits(0x3f317218u));
  p = __fmaf_rn(p, r, 1.0f);
  return p;
}

// 2^x (oracle: exp2_contract)
__device__ __forceinline__ float exp2_contract(float x) {
  if (x != x) return x;
  if (x >= 128.0f) return __int_as_float(0x7f800000);
  if (x < -150.0f) return 0.0f;
  const float t = __fadd_rn(x, kMagic);
  const float n = __fsub_rn(t, kMagic);
  const float r = __fsub_rn(x, n);
  return scale2(exp2_poly(r), (int)n);
}

// Hot-loop form, valid (and identical to exp2_contract) for x in [-126, 127]:
// the integer part is read straight out of t's mantissa, 2^n built with one
// shift+add, no conversion-pipe instructions.
__device__ __forceinline__ float exp2_core(float x) {
  const float t = __fadd_rn(x, kMagic);
  const float n = __fsub_rn(t, kMagic);
  const float r = __fsub_rn(x, n);
  const float s = __int_as_float((__float_as_int(t) << 23) + 0x3f800000);
  return __fmul_rn(exp2_poly(r), s);
}

// e^x (oracle: exp_contract)
__device__ __forceinline__ float exp_contract(float x) {
  if (x != x) return x;
  if (x >= 89.0f) return __int_as_float(0x7f800000);
  if (x < -104.0f) return 0.0f;
  const float t = __fmaf_rn(x, fbits(0x3fb8aa3bu), kMagic);
  const float n = __fsub_rn(t, kMagic);
  float r = __fmaf_rn(n, -fbits(0x3f317200u), x);
  r = __fmaf_rn(n, -fbits(0x35bfbe8eu), r);
  float p = fbits(0x3ab55cb8u);
  p = __fmaf_rn(p, r, fbits(0x3c09368du));
  p = __fmaf_rn(p, r, fbits(0x3d2aac4du));
  p = __fmaf_rn(p, r, fbits(0x3e2aaa05u));
  p = __fmaf_rn(p, r, fbits(0x3efffffdu));
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  return scale2(p, (int)n);
}

// log2(x) (oracle: log2_contract): fixes cut2, which fixes the culling box
// that the tile binning uses -- hence reproducible add/mul/div/fma only.
__device__ __forceinline__ float log2_contract(float x) {
  if (x != x) return x;
  if (x <= 0.0f) return -INFINITY;
  if (x == INFINITY) return INFINITY;
  if (x < 1.17549435e-38f) return -150.0f;
  const uint32_t u = __float_as_uint(x);
  int e = (int)((u >> 23) & 0xffu) - 127;
  float m = __uint_as_float((u & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) { m = __fmul_rn(m, 0.5f); e += 1; }
  const float t = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
  const float t2 = __fmul_rn(t, t);
  float p = __fmaf_rn(t2, 0.111111112f, 0.142857149f);
  p = __fmaf_rn(p, t2, 0.200000003f);
  p = __fmaf_rn(p, t2, 0.333333343f);
  p = __fmaf_rn(p, t2, 1.0f);
  return __fmaf_rn(__fmul_rn(t, p), 2.88539004f, (float)e);
}

// ---------------------------------------------------------------------------
// fp64 contract (RS_F64 frames; oracle: exp64_contract in oracle/cpu_ref.cpp).
// e^x: n = rint(x log2 e) by the magic-number add, r = x - n ln2 (Cody-Waite,
// two fused steps), e^r by its degree-12 Taylor polynomial in Horner form
// (|r| <= 0.347: truncation < 2e-16 relative), times 2^n built in the exponent
// field. Only IEEE double add/mul/fma: the CPU oracle computes the same bits.
// ---------------------------------------------------------------------------
constexpr double kMagic64 = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kLog2e64 = 1.4426950408889634;
constexpr double kLn2Hi = 0.6931471803691238;      // 0x3fe62e42fee00000: n * kLn2Hi exact for |n| < 2^11
constexpr double kLn2Lo = 1.9082149292705877e-10;  // ln 2 - kLn2Hi

__device__ __forceinline__ double exp64_poly(double r) {
  double p = 1.0 / 479001600.0;  // 1/12!
  p = __fma_rn(p, r, 1.0 / 39916800.0);
  p = __fma_rn(p, r, 1.0 / 3628800.0);
  p = __fma_rn(p, r, 1.0 / 362880.0);
  p = __fma_rn(p, r, 1.0 / 40320.0);
  p = __fma_rn(p, r, 1.0 / 5040.0);
  p = __fma_rn(p, r, 1.0 / 720.0);
  p = __fma_rn(p, r, 1.0 / 120.0);
  p = __fma_rn(p, r, 1.0 / 24.0);
  p = __fma_rn(p, r, 1.0 / 6.0);
  p = __fma_rn(p, r, 0.5);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  return p;
}

__device__ __forceinline__ double pow2i64(int n) { return __hiloint2double((n + 1023) << 20, 0); }  // n in [-1022, 1023]

__device__ __forceinline__ double exp64_contract(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000ll);  // overflow: inf
  if (x < -745.2) return 0.0;
  const double t = __fma_rn(x, kLog2e64, kMagic64);
  const double n = __dsub_rn(t, kMagic64);
  double r = __fma_rn(n, -kLn2Hi, x);
  r = __fma_rn(n, -kLn2Lo, r);
  const double p = exp64_poly(r);
  const int ni = __double2loint(t);  // n in the low word of t (two's complement)
  if (ni > 1023) return __dmul_rn(__dmul_rn(p, pow2i64(1023)), 2.0);
  if (ni >= -1022) return __dmul_rn(p, pow2i64(ni));
  return __dmul_rn(__dmul_rn(p, pow2i64(ni + 600)), pow2i64(-600));  // subnormal range
}

// e^x for the fp64 blend (oracle: exp64_tab): k = rint(x 1024 / ln 2), r = x - k ln2/1024
// (Cody-Waite, |r| <= ln2/2048), e^r by its degree-3 Taylor polynomial (truncation
// < 6e-16), times T[k mod 1024] 2^(k div 1024) -- T[j] = exp64_contract(j ln2/1024), a
// table built once per workspace and staged in shared memory; the power of two is
// added to T's exponent field. FAST: the caller guarantees a normal result (x in [-708, 709]).
constexpr int kExpTabBits = 10;
constexpr int kExpTab = 1 << kExpTabBits;
constexpr double kInvLn2xT = 1477.3197218702985;              // 1024 / ln 2
constexpr double kLn2oTHi = 0.6931471803691238 / 1024.0;       // kLn2Hi / 1024 (exact)
constexpr double kLn2oTLo = 1.9082149292705877e-10 / 1024.0;   // kLn2Lo / 1024 (exact)
constexpr double kLn2oT = 0.6931471805599453 / 1024.0;         // table argument step

__device__ __forceinline__ double exp64_tab_entry(int j) { return exp64_contract((double)j * kLn2oT); }

template <bool FAST>
__device__ __forceinline__ double exp64_tab(double x, const double* __restrict__ T) {
  if (!FAST) {
    if (x != x) return x;
    if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000ll);
    if (x < -745.2) return 0.0;
  }
  const double t = __fma_rn(x, kInvLn2xT, kMagic64);
  const double kd = __dsub_rn(t, kMagic64);
  double r = __fma_rn(kd, -kLn2oTHi, x);
  r = __fma_rn(kd, -kLn2oTLo, r);
  double p = __fma_rn(1.0 / 6.0, r, 0.5);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  const int k = __double2loint(t);
  const int n = k >> kExpTabBits;  // floor(k / 1024)
  const double tj = T[k & (kExpTab - 1)];
  if (FAST || n >= -1022)
    return __dmul_rn(p, __hiloint2double(__double2hiint(tj) + (n << 20), __double2loint(tj)));
  return __dmul_rn(__dmul_rn(p, __hiloint2double(__double2hiint(tj) + ((n + 600) << 20), __double2loint(tj))),
                   pow2i64(-600));
}

// order-preserving 32-bit key of an fp32 depth (-0 folded into +0)
__device__ __forceinline__ uint32_t depth_key(float d) {
  const uint32_t u = __float_as_uint(__fadd_rn(d, 0.0f));
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

}  // namespace rs
