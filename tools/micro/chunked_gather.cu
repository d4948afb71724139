// Node-phase cost if element contributions were stored per node, contiguous
// in colour order (cnt = cx*cy*cz slots of 3 values): one thread per node
// sums its chunk.  cfg1 lattice (97^3 nodes, Q3, 32^3 elements), fp64.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void chunk_sum(const double* __restrict__ c, const long long* __restrict__ off,
                          const unsigned char* __restrict__ cnt, double* __restrict__ y, long long nn) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const double* p = c + off[n];
  const int k = cnt[n];
  double s0 = 0, s1 = 0, s2 = 0;
  for (int t = 0; t < k; ++t) {
    s0 += p[3 * t];
    s1 += p[3 * t + 1];
    s2 += p[3 * t + 2];
  }
  y[3 * n] = s0;
  y[3 * n + 1] = s1;
  y[3 * n + 2] = s2;
}

int main() {
  const int P = 3, ne = 32, m = ne * P + 1;
  const long long nn = (long long)m * m * m;
  std::vector<long long> off(nn);
  std::vector<unsigned char> cnt(nn);
  auto ax = [&](int a) { return (a % P == 0 && a > 0 && a < m - 1) ? 2 : 1; };
  long long o = 0;
  for (int c = 0; c < m; ++c)
    for (int b = 0; b < m; ++b)
      for (int a = 0; a < m; ++a) {
        const long long n = ((long long)c * m + b) * m + a;
        off[n] = o;
        cnt[n] = (unsigned char)(ax(a) * ax(b) * ax(c));
        o += 3 * cnt[n];
      }
  printf("chunk doubles %lld (%.1f MB)\n", o, o * 8e-6);
  double *dc, *dy;
  long long* doff;
  unsigned char* dcnt;
  cudaMalloc(&dc, o * 8);
  cudaMalloc(&dy, nn * 3 * 8);
  cudaMalloc(&doff, nn * 8);
  cudaMalloc(&dcnt, nn);
  cudaMemset(dc, 0, o * 8);
  cudaMemcpy(doff, off.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dcnt, cnt.data(), nn, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(dc, 0, o * 8);  // chunks L2-warm like after the element phase
    cudaEventRecord(e0);
    chunk_sum<<<(unsigned)((nn + 255) / 256), 256>>>(dc, doff, dcnt, dy, nn);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("chunked node phase %.4f ms\n", ms);
  }
  return 0;
}
