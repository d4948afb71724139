// SM-driven PCIe bandwidth: kernels that read pinned host memory (mapped,
// zero-copy) into device memory and write device memory out to pinned host
// memory, with a given number of CTAs, vs the copy engines.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void h2d_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}
__global__ void d2h_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  const size_t bytes = 21914496;  // cfg1 fp64 vector
  const size_t n = bytes / 16;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  void *hp1, *hp2;
  cudaHostGetDevicePointer(&hp1, h1, 0);
  cudaHostGetDevicePointer(&hp2, h2, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy engine h2d: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(e0);
    cudaMemcpyAsync(h2, d1, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy engine d2h: %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
  }
  for (int ctas : {8, 16, 32, 64, 148, 296}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      h2d_kernel<<<ctas, 256>>>((const double2*)hp1, (double2*)d1, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("SM h2d %3d CTAs: %.3f ms %.1f GB/s\n", ctas, ms, bytes / ms / 1e6);
      cudaEventRecord(e0);
      d2h_kernel<<<ctas, 256>>>((const double2*)d1, (double2*)hp2, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("SM d2h %3d CTAs: %.3f ms %.1f GB/s\n", ctas, ms, bytes / ms / 1e6);
    }
  }
  // both directions at once with SM kernels on two streams
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int rep = 0; rep < 2; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(s1, e0, 0);
    cudaStreamWaitEvent(s2, e0, 0);
    h2d_kernel<<<64, 256, 0, s1>>>((const double2*)hp1, (double2*)d1, n);
    d2h_kernel<<<64, 256, 0, s2>>>((const double2*)d2, (double2*)hp2, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s1);
    cudaEventRecord(b, s2);
    cudaStreamWaitEvent(0, a, 0);
    cudaStreamWaitEvent(0, b, 0);
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("SM both 64+64 CTAs: %.3f ms\n", ms);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
