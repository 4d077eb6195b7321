// sortbench.cu -- micro-benchmark of one onesweep pass (tools only, not product).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include tools/sortbench.cu -o sortbench
//   ./sortbench N
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sortexp.cuh"

using namespace rs;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

template <int ITEMS, int NB, int MODE = 0>
float run(uint32_t n, const uint16_t* kin, const uint32_t* vin, uint16_t* kout, uint32_t* vout, uint32_t* hist,
          uint32_t* lb, uint32_t* lb2, uint32_t* ticket, int shift, int reps) {
  const int smem = sizeof(OnesweepSmem<uint16_t, ITEMS>);
  CK(cudaFuncSetAttribute(exp_kernel<uint16_t, ITEMS, NB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = (n + 256 * ITEMS - 1) / (256 * ITEMS);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemset(lb, 0, (size_t)grid * 256 * 4));
    CK(cudaMemset(ticket, 0, 4));
    cudaEventRecord(a);
    exp_kernel<uint16_t, ITEMS, NB, MODE><<<grid, 256, smem>>>(kin, vin, kout, vout, nullptr, n, hist, lb, nullptr,
                                                              ticket, shift, 1);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best * 1000.0f;
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 10000000;
  std::vector<uint16_t> hk(n);
  std::vector<uint32_t> hh(256, 0);
  srand(1);
  for (uint32_t i = 0; i < n; ++i) {  // tile-like keys: runs of consecutive tiles
    hk[i] = (uint16_t)((i / 7 + (rand() % 3)) % 4108);
    hh[hk[i] & 255]++;
  }
  uint16_t *kin, *kout;
  uint32_t *vin, *vout, *hist, *lb, *lb2, *ticket;
  CK(cudaMalloc(&kin, n * 2));
  CK(cudaMalloc(&kout, n * 2));
  CK(cudaMalloc(&vin, n * 4));
  CK(cudaMalloc(&vout, n * 4));
  CK(cudaMalloc(&hist, 256 * 4));
  CK(cudaMalloc(&lb, (n / 2048 + 2) * 256 * 4));
  CK(cudaMalloc(&lb2, (n / 2048 + 2) * 256 * 4));
  CK(cudaMalloc(&ticket, 4));
  CK(cudaMemcpy(kin, hk.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(vin, 0, n * 4));
  CK(cudaMemcpy(hist, hh.data(), 256 * 4, cudaMemcpyHostToDevice));
  const double bytes = (double)n * 12;
  float t;
  t = run<16, 8>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("ITEMS=16 NB=8: %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<8, 8>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("ITEMS=8  NB=8: %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 5>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 8, 5);
  printf("ITEMS=16 NB=5 (hi): %8.1f us  %6.0f GB/s  (hist wrong: timing only)\n", t, bytes / t / 1e3);
  t = run<16, 8, 1>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("no lookback:   %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 2>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("no ranking:    %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 4>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("no gmem write: %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 8>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("match_any:     %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 9>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("match, no lb:  %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 24>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("match+atomics: %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  t = run<16, 8, 7>(n, kin, vin, kout, vout, hist, lb, lb2, ticket, 0, 5);
  printf("none of them:  %8.1f us  %6.0f GB/s\n", t, bytes / t / 1e3);
  return 0;
}
