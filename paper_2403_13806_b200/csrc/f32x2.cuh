// f32x2.cuh -- packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): two pixels' identical
// IEEE operation sequences in one instruction each, bit-identical to the scalar ops.
//
// ptxas contraction hazard (measured, CUDA 12.9): a mul.rn.f32x2 whose result only feeds an
// add.rn.f32x2 / sub.rn.f32x2 is fused into one FFMA2 despite the explicit rounding mode and
// -fmad=false (scalar mul.rn/add.rn are left alone). Callers never feed f2_mul into
// f2_add / f2_sub; products go into f2_fma operands, other products or selects only.
#pragma once
#include <cstdint>

namespace rs {

typedef unsigned long long f2;  // {lo, hi} = {first pixel, second pixel}

__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2 f2_splat(float v) { return f2_pack(v, v); }
__device__ __forceinline__ float f2_lo(f2 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(f2 v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
  f2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// {2^n_lo, 2^n_hi} from the round-to-integer magic sums t = x + 1.5 * 2^23 of an exp2
// reduction: (bits(t) << 23) + bits(1.0f) per half -- as two 32-bit shift-adds (one LEA each;
// written on the 64-bit pair in C, ptxas folds the high half into a funnel shift + mask + add)
__device__ __forceinline__ f2 f2_exp2_scale(f2 t) {
  f2 r;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tshl.b32 lo, lo, 23;\n\tshl.b32 hi, hi, 23;\n\t"
      "add.u32 lo, lo, 0x3f800000;\n\tadd.u32 hi, hi, 0x3f800000;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "l"(t));
  return r;
}

}  // namespace rs
