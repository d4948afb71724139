// FMA-pipe peak microbenchmark (roofline denominator for the FP64/FP32
// CUDA-core-bound strategies; MEASURED_PEAKS.json only carries HBM and bf16
// tensor peaks).  8 independent FMA chains per thread, one full wave of
// 148 SMs x 8 CTAs x 256 threads.
#include "internal.h"

namespace {
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = T(threadIdx.x + c) * T(1e-3);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = x[c] * a + b;
  }
  T s = T(0);
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == T(-1.2345)) out[0] = s;  // keep the chains alive
}

template <typename T>
double run(double seconds) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* out = nullptr;
  cudaMalloc(&out, sizeof(T));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_peak_kernel<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));  // warm-up
  cudaDeviceSynchronize();
  double best = 0.0, total = 0.0;
  while (total < seconds) {
    cudaEventRecord(e0);
    fma_peak_kernel<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    total += ms * 1e-3;
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}
}  // namespace

emfgpu_status emfgpu_bench_fma_peak(int precision, double seconds, double* tflops) {
  if (!tflops) return EMFGPU_ERR_INVALID;
  *tflops = precision == 64 ? run<double>(seconds) : run<float>(seconds);
  return cudaGetLastError() == cudaSuccess ? EMFGPU_OK : EMFGPU_ERR_CUDA;
}
