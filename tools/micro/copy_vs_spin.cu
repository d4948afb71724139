// H2D copy-engine time while (a) nothing, (b) a grid of CTAs polls a device
// flag with nanosleep, (c) a grid runs FP64 math, runs on the GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(volatile unsigned* flag, int sleep_ns) {
  if (threadIdx.x == 0)
    while (*flag == 0u) __nanosleep(sleep_ns);
  __syncthreads();
}
__global__ void math(volatile unsigned* flag, double* out) {
  double a = threadIdx.x;
  while (*flag == 0u)
    for (int i = 0; i < 1000; ++i) a = fma(a, 0.999, 0.5);
  if (a == -1) out[0] = a;
}

int main() {
  const size_t bytes = 21914496;
  void *h, *d, *h2, *d2;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&d, bytes);
  cudaMallocHost(&h2, bytes);
  cudaMalloc(&d2, bytes);
  unsigned* flag;
  cudaMalloc(&flag, 4);
  double* out;
  cudaMalloc(&out, 8);
  unsigned* one;
  cudaMallocHost(&one, 4);
  *one = 1;
  cudaStream_t sk, sc, sd;
  cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flag, 0, 4);
      cudaDeviceSynchronize();
      if (mode == 1) spin<<<444, 128, 0, sk>>>(flag, 256);
      if (mode == 2) spin<<<444, 128, 0, sk>>>(flag, 2000);
      if (mode == 3) math<<<444, 128, 0, sk>>>(flag, out);
      cudaEventRecord(e0, sc);
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, sc);
      cudaEventRecord(e1, sc);
      if (mode >= 4) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, sd);  // both directions
      if (mode == 5) spin<<<444, 128, 0, sk>>>(flag, 2000);
      cudaEventSynchronize(e1);
      cudaMemcpyAsync(flag, one, 4, cudaMemcpyHostToDevice, sc);
      cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("mode %d (%s): H2D %.3f ms\n", mode,
               mode == 0 ? "alone" : mode == 1 ? "spin 256ns" : mode == 2 ? "spin 2us" : mode == 3 ? "fp64 math"
               : mode == 4 ? "with D2H" : "with D2H + spin launched after",
               ms);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
