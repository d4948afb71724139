// Microbenchmark: FP64 tensor-core (mma.sync m8n8k4 f64) throughput vs the
// FP64 FMA pipe on this GPU, alone and concurrently (separate warps of the
// same CTA), to decide whether sum-factorisation sweeps should move to DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA
__global__ void bench(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool use_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = i * 1e-3;
  if (use_mma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)  // 16 DFMA per thread ~ 1 DMMA's worth per 8 threads... count below
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, iters = 4000;
  for (int bps : {1, 2, 4}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int grid = sms * bps;
      bench<<<grid, threads>>>(out, 10, mode);
      cudaEventRecord(e0);
      bench<<<grid, threads>>>(out, iters, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)grid * threads / 32;
      // flops: DMMA warp-instr = 8*8*4*2 = 512 flops; DFMA thread = 2 flops
      double mma_w = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0);
      double fma_w = mode == 1 ? warps : (mode == 2 ? warps / 2 : 0);
      const double fl = mma_w * iters * 8 * 512.0 + fma_w * 32 * iters * 256 * 2.0;
      printf("blocks/SM %d mode %d: %.3f ms  %.1f TFLOP/s (mma part %.1f, fma part %.1f)\n", bps, mode, ms,
             fl / ms / 1e9, mma_w * iters * 8 * 512.0 / ms / 1e9, fma_w * 32 * iters * 256 * 2.0 / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
