// Full-duplex options for 21.9 MB each way: CE H2D + CE D2H, SM zero-copy
// read (H2D) + CE D2H, CE H2D + SM zero-copy write (D2H).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_read(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}
__global__ void zc_write(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  const size_t bytes = 21914496, n = bytes / 16;
  void *hx, *hy, *dx, *dy;
  cudaMallocHost(&hx, bytes);
  cudaMallocHost(&hy, bytes);
  cudaMalloc(&dx, bytes);
  cudaMalloc(&dy, bytes);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, ea, eb;
  cudaEventCreate(&e0);
  cudaEventCreate(&ea);
  cudaEventCreate(&eb);
  for (int mode = 0; mode < 3; ++mode)
    for (int ctas : {16, 32, 64}) {
      if (mode == 0 && ctas != 16) continue;
      for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        cudaStreamWaitEvent(a, e0, 0);
        cudaStreamWaitEvent(b, e0, 0);
        if (mode == 0) cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, a);
        if (mode == 1) zc_read<<<ctas, 256, 0, a>>>((const double2*)hx, (double2*)dx, n);
        if (mode == 2) cudaMemcpyAsync(dx, hx, bytes, cudaMemcpyHostToDevice, a);
        if (mode == 2) zc_write<<<ctas, 256, 0, b>>>((const double2*)dy, (double2*)hy, n);
        else cudaMemcpyAsync(hy, dy, bytes, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(ea, a);
        cudaEventRecord(eb, b);
        cudaDeviceSynchronize();
        float ta, tb;
        cudaEventElapsedTime(&ta, e0, ea);
        cudaEventElapsedTime(&tb, e0, eb);
        if (rep == 2)
          printf("%-26s ctas %2d: h2d done %.3f  d2h done %.3f ms\n",
                 mode == 0 ? "CE h2d + CE d2h" : mode == 1 ? "SM-read h2d + CE d2h" : "CE h2d + SM-write d2h", ctas,
                 ta, tb);
      }
    }
  return 0;
}
