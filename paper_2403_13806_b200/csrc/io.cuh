// io.cuh -- scene / visibility wire formats straight to and from HBM
// (reference io.py:128-243).
//
// RSPL payload (io.py:128-191): after a 17-byte header, five contiguous
// little-endian fp32 arrays -- positions (n,3), log-scales (n,3),
// quaternions w-x-y-z (n,4), opacity logits (n), SH (n,48) -- 59 floats per
// Gaussian. The host reads the payload into page-locked memory and makes ONE
// host-to-device copy; rspl_unpack_kernel scatters it into the device scene
// layout (11 planes + SH rows), normalizing quaternions exactly as the
// reference's GaussianScene constructor does on load (core.py:111-117,
// :494-495: fp64 q / |q|, |q| = sqrt(((q0^2 + q1^2) + q2^2) + q3^2), then
// rounded to fp32 like any scene upload). rspl_pack_kernel is the inverse
// (device scene -> payload; the scene's quaternions are already unit).
//
// RVIS bitsets (io.py:198-243): per cluster an LSB-first packed indicator
// (np.packbits(bitorder="little")); pack_bits_kernel builds it with one warp
// ballot per 32 flags (bit i of the little-endian word = flag i), and
// rs_compact_bits turns a bitset straight into the cluster's index list.
#pragma once
#include "rs_common.cuh"

namespace rs {

__global__ void __launch_bounds__(256) rspl_unpack_kernel(const float* __restrict__ payload, int64_t n,
                                                          float* __restrict__ planes, int64_t stride,
                                                          float* __restrict__ sh, uint32_t* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* pos = payload;
  const float* ls = payload + 3 * n;
  const float* q = payload + 6 * n;
  const float* logit = payload + 10 * n;
  const float* shp = payload + 11 * n;
  planes[i] = pos[3 * i];
  planes[stride + i] = pos[3 * i + 1];
  planes[2 * stride + i] = pos[3 * i + 2];
  planes[3 * stride + i] = logit[i];
#pragma unroll
  for (int k = 0; k < 3; ++k) planes[(4 + k) * stride + i] = ls[3 * i + k];
  double qd[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) qd[k] = (double)q[4 * i + k];
  const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(qd[0], qd[0]), __dmul_rn(qd[1], qd[1])),
                                                    __dmul_rn(qd[2], qd[2])),
                                          __dmul_rn(qd[3], qd[3])));
  if (!(nrm >= 1e-12)) atomicAdd(bad, 1u);  // zero quaternion (core.py:115-116)
#pragma unroll
  for (int k = 0; k < 4; ++k) planes[(7 + k) * stride + i] = (float)__ddiv_rn(qd[k], nrm);
  // the SH section starts 44 n bytes into the payload: 4-byte source loads, 16-byte row stores
  const float* src = shp + 48 * i;
  float4* dst = reinterpret_cast<float4*>(sh + 48 * i);
#pragma unroll
  for (int v = 0; v < 12; ++v) dst[v] = make_float4(src[4 * v], src[4 * v + 1], src[4 * v + 2], src[4 * v + 3]);
}

__global__ void __launch_bounds__(256) rspl_pack_kernel(const float* __restrict__ planes, int64_t stride,
                                                        const float* __restrict__ sh, int64_t n,
                                                        float* __restrict__ payload) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float* pos = payload;
  float* ls = payload + 3 * n;
  float* q = payload + 6 * n;
  float* logit = payload + 10 * n;
  float* shp = payload + 11 * n;
#pragma unroll
  for (int k = 0; k < 3; ++k) pos[3 * i + k] = planes[k * stride + i];
  logit[i] = planes[3 * stride + i];
#pragma unroll
  for (int k = 0; k < 3; ++k) ls[3 * i + k] = planes[(4 + k) * stride + i];
#pragma unroll
  for (int k = 0; k < 4; ++k) q[4 * i + k] = planes[(7 + k) * stride + i];
  const float4* src = reinterpret_cast<const float4*>(sh + 48 * i);
  float* dst = shp + 48 * i;  // 4-byte aligned only (the section starts 44 n bytes in)
#pragma unroll
  for (int v = 0; v < 12; ++v) {
    const float4 x = src[v];
    dst[4 * v] = x.x; dst[4 * v + 1] = x.y; dst[4 * v + 2] = x.z; dst[4 * v + 3] = x.w;
  }
}

// flags (n bytes, nonzero = set) -> LSB-first bitset of ceil(n/8) bytes (padding bits zero)
__global__ void __launch_bounds__(256) pack_bits_kernel(const uint8_t* __restrict__ flags, int64_t n,
                                                        uint8_t* __restrict__ bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool f = i < n && flags[i] != 0;
  const uint32_t w = __ballot_sync(0xffffffffu, f);
  const int64_t w0 = i - (threadIdx.x & 31);  // first flag of this warp's word
  if ((threadIdx.x & 31) == 0 && w0 < n) {
    const int64_t nbytes = (n + 7) / 8, b0 = w0 / 8;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (b0 + k < nbytes) bits[b0 + k] = (uint8_t)(w >> (8 * k));
  }
}

}  // namespace rs
