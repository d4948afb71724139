// Is the slowdown under an active copy per kernel or per event?  8 tiny
// kernels back to back timed by 2 events, vs 8 events back to back.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tiny(float* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0f; }
int main() {
  float* x; cudaMalloc(&x, 4);
  const size_t bytes = 512ull << 20;
  void *h, *d; cudaMallocHost(&h, bytes); cudaMalloc(&d, bytes);
  cudaStream_t s1, sc; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ev[16]; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int mode = 0; mode < 3; ++mode) {
    for (int what = 0; what < 3; ++what) {
      cudaDeviceSynchronize();
      if (mode == 1) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1);
      if (mode == 2) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1);
      cudaEventRecord(e0, sc);
      for (int i = 0; i < 8; ++i) {
        if (what == 0) tiny<<<1, 32, 0, sc>>>(x);
        else if (what == 1) cudaEventRecord(ev[i], sc);
        else { tiny<<<1, 32, 0, sc>>>(x); cudaEventRecord(ev[i], sc); cudaStreamWaitEvent(sc, ev[i], 0); }
      }
      cudaEventRecord(e1, sc);
      cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-4s %-22s: %6.1f us per item\n", mode == 0 ? "none" : mode == 1 ? "h2d" : "d2h",
             what == 0 ? "8 kernels" : what == 1 ? "8 event records" : "8 kernel+record+wait", ms * 1000 / 8);
    }
  }
  return 0;
}
