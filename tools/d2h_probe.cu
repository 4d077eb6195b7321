// Host-link write bandwidth on the box (what bounds the e2e render): copy-engine D2H of one
// 1256x828 reference-typed frame (40 B/px) as one copy and as B band copies, versus
// zero-copy stores into mapped pinned memory from a linear streaming kernel of G CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/d2h_probe tools/d2h_probe.cu && /tmp/d2h_probe
#include <cuda_runtime.h>
#include <cstdio>

__global__ void stream_out(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void busy(float* p, int iters) {
  float x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = x * 1.0000001f + 0.5f;
  p[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  const size_t bytes = 1256ull * 828 * 40;
  void *dev, *host;
  cudaMalloc(&dev, bytes);
  cudaMemset(dev, 1, bytes);
  cudaHostAlloc(&host, bytes, cudaHostAllocMapped);
  cudaStream_t s[8];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn, int reps) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, s[0]);
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(b, s[0]);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
  };
  float ms = timeit([&] { cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s[0]); }, 20);
  printf("copy engine, one copy:        %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
  for (int B : {4, 8, 16, 32}) {
    ms = timeit([&] {
      for (int k = 0; k < B; ++k)
        cudaMemcpyAsync((char*)host + bytes / B * k, (char*)dev + bytes / B * k, bytes / B, cudaMemcpyDeviceToHost,
                        s[0]);
    }, 20);
    printf("copy engine, %2d band copies:  %.3f ms  %.1f GB/s\n", B, ms, bytes / ms / 1e6);
  }
  // two streams alternating bands (two copy engines?)
  ms = timeit([&] {
    cudaEventRecord(a, s[0]);
    cudaStreamWaitEvent(s[1], a, 0);
    for (int k = 0; k < 8; ++k)
      cudaMemcpyAsync((char*)host + bytes / 8 * k, (char*)dev + bytes / 8 * k, bytes / 8, cudaMemcpyDeviceToHost,
                      s[k & 1]);
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, s[1]);
    cudaStreamWaitEvent(s[0], e, 0);
    cudaEventDestroy(e);
  }, 20);
  printf("copy engine, 8 bands on 2 streams: %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
  // three copies per frame in the rgb / alpha / count split (24 / 8 / 8 B per px), B bands
  for (int B : {1, 2, 4, 8}) {
    const size_t np = bytes / 40;
    ms = timeit([&] {
      for (int k = 0; k < B; ++k) {
        const size_t p0 = np * k / B, p1 = np * (k + 1) / B;
        cudaMemcpyAsync((char*)host + p0 * 24, (char*)dev + p0 * 24, (p1 - p0) * 24, cudaMemcpyDeviceToHost, s[0]);
        cudaMemcpyAsync((char*)host + np * 24 + p0 * 8, (char*)dev + np * 24 + p0 * 8, (p1 - p0) * 8,
                        cudaMemcpyDeviceToHost, s[0]);
        cudaMemcpyAsync((char*)host + np * 32 + p0 * 8, (char*)dev + np * 32 + p0 * 8, (p1 - p0) * 8,
                        cudaMemcpyDeviceToHost, s[0]);
      }
    }, 20);
    printf("copy engine, 3 arrays x %d bands: %.3f ms  %.1f GB/s\n", B, ms, bytes / ms / 1e6);
  }
  // one copy while a compute kernel keeps every SM busy on another stream
  {
    void* scratch;
    cudaMalloc(&scratch, 256 << 20);
    ms = timeit([&] {
      busy<<<148 * 4, 256, 0, s[1]>>>((float*)scratch, 4000);
      cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s[0]);
    }, 10);
    printf("copy engine under a busy kernel (timed on the copy stream): %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
    cudaDeviceSynchronize();
  }
  double2* hd;
  cudaHostGetDevicePointer((void**)&hd, host, 0);
  for (int G : {8, 16, 32, 64, 148, 296, 592}) {
    ms = timeit([&] { stream_out<<<G, 256, 0, s[0]>>>((const double2*)dev, hd, bytes / 16); }, 20);
    printf("zero-copy stream kernel, %3d CTAs: %.3f ms  %.1f GB/s\n", G, ms, bytes / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
