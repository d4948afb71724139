// H2D of a 21.9 MB vector as 1 copy, as 8 chunk copies, and as 8 chunk copies
// each followed by a 4-byte flag copy (pinned -> device), same stream.
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = 21914496, chunk = bytes / 8;
  char *h, *d;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&d, bytes);
  unsigned *one, *flag;
  cudaMallocHost(&one, 4);
  cudaMalloc(&flag, 64);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s);
      if (mode == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
      for (int i = 0; mode > 0 && i < 8; ++i) {
        cudaMemcpyAsync(d + i * chunk, h + i * chunk, chunk, cudaMemcpyHostToDevice, s);
        if (mode == 2) cudaMemcpyAsync(flag + i, one, 4, cudaMemcpyHostToDevice, s);
        if (mode == 3) cudaMemsetAsync(flag + i, 1, 4, s);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%s: %.3f ms\n", mode == 0 ? "1 copy" : mode == 1 ? "8 chunks" : mode == 2 ? "8 chunks + 4B flag copies"
                                                                                  : "8 chunks + memset flags",
               ms);
    }
  return 0;
}
