// Per-kernel time (event to event, kernels enqueued back to back) of a tiny
// kernel and of a 1-wave compute kernel, with and without a concurrent pinned
// H2D or D2H copy on another stream.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tiny(float* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0f; }
__global__ void work(float* x, int iters) {
  float a = threadIdx.x;
  for (int i = 0; i < iters; ++i) a = a * 0.999f + 0.5f;
  if (a == -1.0f) x[0] = a;
}

int main() {
  float* x;
  cudaMalloc(&x, 4);
  const size_t bytes = 512ull << 20;
  void *h, *d;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&d, bytes);
  cudaStream_t sc, s1;
  cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  const int n = 8;
  cudaEvent_t ev[n + 1];
  for (auto& e : ev) cudaEventCreate(&e);
  for (int which = 0; which < 2; ++which)
    for (int mode = 0; mode < 3; ++mode) {
      cudaDeviceSynchronize();
      if (mode == 1) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1);
      if (mode == 2) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1);
      cudaEventRecord(ev[0], sc);
      for (int i = 0; i < n; ++i) {
        if (which == 0) tiny<<<1, 32, 0, sc>>>(x);
        else work<<<148 * 4, 256, 0, sc>>>(x, 20000);
        cudaEventRecord(ev[i + 1], sc);
      }
      cudaDeviceSynchronize();
      printf("%s %-4s:", which ? "work" : "tiny", mode == 0 ? "none" : mode == 1 ? "h2d" : "d2h");
      for (int i = 0; i < n; ++i) {
        float ms;
        cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        printf(" %6.1f", ms * 1000);
      }
      printf(" us\n");
    }
  return 0;
}
