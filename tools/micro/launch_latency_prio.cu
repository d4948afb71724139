// Launch latency of back-to-back tiny kernels while a CE copy runs, with the
// compute stream at default vs highest priority.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(float* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0f; }
int main() {
  float* x; cudaMalloc(&x, 4);
  const size_t bytes = 512ull << 20;
  void *h, *d; cudaMallocHost(&h, bytes); cudaMalloc(&d, bytes);
  int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s1; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  const int n = 8; cudaEvent_t ev[n + 1]; for (auto& e : ev) cudaEventCreate(&e);
  for (int pr = 0; pr < 2; ++pr) {
    cudaStream_t sc; cudaStreamCreateWithPriority(&sc, cudaStreamNonBlocking, pr ? hi : lo);
    for (int mode = 0; mode < 3; ++mode) {
      cudaDeviceSynchronize();
      if (mode == 1) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1);
      if (mode == 2) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1);
      cudaEventRecord(ev[0], sc);
      for (int i = 0; i < n; ++i) { tiny<<<1, 32, 0, sc>>>(x); cudaEventRecord(ev[i + 1], sc); }
      cudaDeviceSynchronize();
      printf("prio %s %-4s:", pr ? "high" : "low ", mode == 0 ? "none" : mode == 1 ? "h2d" : "d2h");
      for (int i = 1; i < n; ++i) { float ms; cudaEventElapsedTime(&ms, ev[i], ev[i + 1]); printf(" %5.1f", ms * 1000); }
      printf(" us\n");
    }
  }
  return 0;
}
