// FP32 / FP64 FMA issue peaks of this GPU (the blend / blend64 roofline denominators):
// independent FMA chains per thread, every SM full, CUDA-event timed.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fma_peak.cu -o tools/_bin/fma_peak
#include <cstdio>

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == (T)12345) out[0] = s;  // keep the chains alive
}

template <typename T>
double run(int sms) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int threads = 256, blocks = sms * 8, iters = 1 << 14;
  fma_loop<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return 2.0 * 8 * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"fp32_fma_tflops\": %.2f, \"fp64_fma_tflops\": %.2f, \"clock_mhz_attr\": %d}\n", sms,
         run<float>(sms), run<double>(sms), khz / 1000);
  return 0;
}
