// Phase timing of dsort_kernel (globaltimer stamps per CTA) on configs[1]-like keys:
// 500k items, ~40% visible, fp32 depth keys in [0.5, 8], the rest kInvalidKey.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DRS_DSORT_PROBE \
//        -I paper_2403_13806_b200/csrc tools/dsort_probe.cu -o tools/_bin/dsort_probe
//   ./tools/_bin/dsort_probe [n_items] [visible_frac] [ctas]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "dsort.cuh"

using namespace rs;

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 500000;
  const double vf = argc > 2 ? atof(argv[2]) : 0.4;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int G = argc > 3 ? atoi(argv[3]) : std::min(sms, 160);
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> dep(0.5f, 8.0f), u(0.f, 1.f);
  std::vector<uint32_t> keys(n);
  for (auto& k : keys) {
    const float d = dep(rng);
    k = u(rng) < vf ? *reinterpret_cast<const uint32_t*>(&d) : kInvalidKey;
  }
  uint32_t *dk, *kA, *vA, *kB, *vB, *tab;
  Counters* ctr;
  unsigned long long* probe;
  cudaMalloc(&dk, n * 4);
  cudaMalloc(&kA, n * 4);
  cudaMalloc(&vA, n * 4);
  cudaMalloc(&kB, n * 4);
  cudaMalloc(&vB, n * 4);
  cudaMalloc(&tab, dsort_tab_words(160) * 4);
  cudaMalloc(&ctr, sizeof(Counters));
  cudaMalloc(&probe, 160 * 32 * 8);
  cudaMemcpyToSymbol(g_dsort_probe, &probe, sizeof(probe));
  cudaMemcpy(dk, keys.data(), n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(dsort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(DsortSmem));
  std::vector<unsigned long long> h(160 * 32);
  std::vector<double> acc(32, 0.0);
  const int reps = 20;
  float ms_tot = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < reps + 3; ++r) {
    cudaMemset(tab, 0, dsort_tab_words(160) * 4);
    cudaMemset(ctr, 0, sizeof(Counters));
    cudaMemset(probe, 0, 160 * 32 * 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = G;
    cfg.blockDim = kDsortThreads;
    cfg.dynamicSmemBytes = sizeof(DsortSmem);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, dsort_kernel<false>, (const uint32_t*)dk, n, kA, vA, kB, vB, tab, ctr,
                                       (uint32_t)(getenv("RS_DSORT_RED_MAX") ? atoi(getenv("RS_DSORT_RED_MAX")) : kDsortRedMax),
                                       getenv("RS_DSORT_BINS") ? atoi(getenv("RS_DSORT_BINS")) : 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("launch failed: %s\n", cudaGetErrorString(e));
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h.data(), probe, h.size() * 8, cudaMemcpyDeviceToHost);
    if (r < 3) continue;
    ms_tot += ms;
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < G; ++b) t0 = std::min(t0, h[b * 32]);
    for (int k = 0; k < 32; ++k) {
      unsigned long long mx = 0;
      for (int b = 0; b < G; ++b) mx = std::max(mx, h[b * 32 + k]);
      acc[k] += (double)(mx - t0);
    }
  }
  // check against a host stable sort
  std::vector<uint32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0u);
  std::vector<uint32_t> vis;
  for (uint32_t i = 0; i < n; ++i)
    if (keys[i] != kInvalidKey) vis.push_back(i);
  std::stable_sort(vis.begin(), vis.end(), [&](uint32_t a, uint32_t b) { return keys[a] < keys[b]; });
  std::vector<uint32_t> got(vis.size());
  cudaMemcpy(got.data(), vA, vis.size() * 4, cudaMemcpyDeviceToHost);
  printf("n=%u visible=%zu G=%d  kernel %.1f us  %s\n", n, vis.size(), G, 1e3 * ms_tot / reps,
         got == vis ? "sorted OK" : "MISMATCH");
  printf("phase ends (max over CTAs, us from the first CTA start):\n  hist0 %.1f\n", acc[1] / reps / 1e3);
  for (int p = 0; p < 4; ++p)
    printf("  pass %d: barrier %.1f  prefix %.1f  loads %.1f  rank %.1f  offsets %.1f  scatter %.1f\n", p,
           acc[2 + 4 * p] / reps / 1e3, acc[3 + 4 * p] / reps / 1e3, acc[20 + 3 * p] / reps / 1e3,
           acc[21 + 3 * p] / reps / 1e3, acc[22 + 3 * p] / reps / 1e3, acc[4 + 4 * p] / reps / 1e3);
  return 0;
}
