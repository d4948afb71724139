// Dense coarse-grid solve of the hp-multigrid hierarchy (CoarseSolver dense
// path, solver.hpp:49-91 and 369-401): below coarse_direct_limit DoFs the
// reference assembles the coarse tangent column by column (one apply per DoF)
// and factors it with partially pivoted LU in double.
//
// B200 version:
//  * assembly by probing: unit vectors on nodes 2p+1 apart in every axis have
//    disjoint element supports, so one apply yields (2p+1)^-3 of all columns
//    exactly (each element sees at most one nonzero input) -> 3 (2p+1)^3
//    applies instead of n;
//  * inversion by Gauss-Jordan with partial pivoting (same pivot rule as
//    DenseLU::factor: first row of maximal |a|) in ONE cooperative kernel:
//    every CTA of a one-wave grid walks the pivots, separated by grid syncs;
//  * the per-V-cycle coarse solve is then one warp-per-row double GEMV
//    (fixed reduction order, deterministic) instead of a sequential
//    triangular solve.
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.h"

namespace cg = cooperative_groups;

namespace emfgpu {

// x = sum over probed nodes (a%s==ca, b%s==cb, c%s==cc) of e_{3 node + comp}
template <typename T>
__global__ void probe_fill_kernel(T* x, int mx, int my, int mz, int s, int ca, int cb, int cc, int comp) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nn = (int64_t)mx * my * mz;
  if (node >= nn) return;
  const int a = (int)(node % mx), b = (int)((node / mx) % my), c = (int)(node / ((int64_t)mx * my));
  const bool on = a % s == ca && b % s == cb && c % s == cc;
#pragma unroll
  for (int k = 0; k < 3; ++k) x[3 * node + k] = (on && k == comp) ? T(1) : T(0);
}

// A[i][3 node_j + comp] = y_i, node_j the probed node within +-p of row i's node
template <typename T>
__global__ void probe_extract_kernel(const T* y, double* A, int64_t n, int mx, int my, int mz, int p, int s, int ca,
                                     int cb, int cc, int comp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t node = i / 3;
  const int a = (int)(node % mx), b = (int)((node / mx) % my), c = (int)(node / ((int64_t)mx * my));
  auto cand = [&](int v, int r) {  // smallest w >= v - p with w % s == r
    const int lo = v - p;
    return lo + (((r - lo) % s) + s) % s;
  };
  const int aj = cand(a, ca), bj = cand(b, cb), cj = cand(c, cc);
  if (aj < 0 || aj >= mx || bj < 0 || bj >= my || cj < 0 || cj >= mz) return;
  const int64_t j = 3 * (((int64_t)cj * my + bj) * mx + aj) + comp;
  A[i * n + j] = (double)y[i];
}

// [A | I] -> [I | A^-1] in place on M (n x 2n, row-major), partial pivoting.
__global__ void gauss_jordan_kernel(double* M, int n, int* singular) {
  cg::grid_group grid = cg::this_grid();
  const int w = 2 * n;
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_piv;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  for (int c = 0; c < n; ++c) {
    // (a) scale the previous pivot row, search the pivot of column c
    if (c > 0) {
      const int pc = c - 1;
      const double inv = 1.0 / M[(int64_t)pc * w + pc];
      for (int64_t k = pc + 1 + gtid; k < w; k += gthreads) M[(int64_t)pc * w + k] *= inv;
    }
    double best = -1.0;
    int bi = n;
    for (int r = c + threadIdx.x; r < n; r += blockDim.x) {
      const double v = fabs(M[(int64_t)r * w + c]);
      if (v > best) {  // strictly greater: first row of maximal |a| (DenseLU::factor)
        best = v;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      s_val[threadIdx.x >> 5] = best;
      s_idx[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b2 = s_val[0];
      int i2 = s_idx[0];
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
        if (s_val[q] > b2 || (s_val[q] == b2 && s_idx[q] < i2)) {
          b2 = s_val[q];
          i2 = s_idx[q];
        }
      s_piv = i2;
      if (!(b2 >= 1e-250) && blockIdx.x == 0) atomicExch(singular, 1);
    }
    __syncthreads();
    const int pr = s_piv;
    grid.sync();  // every CTA has read column c before the swap
    if (pr != c)
      for (int64_t k = gtid; k < w; k += gthreads) {
        const double t = M[(int64_t)pr * w + k];
        M[(int64_t)pr * w + k] = M[(int64_t)c * w + k];
        M[(int64_t)c * w + k] = t;
      }
    grid.sync();
    // (b) eliminate column c from every other row (pivot row read unscaled)
    const double inv = 1.0 / M[(int64_t)c * w + c];
    const int64_t cols = w - c - 1;
    const int64_t total = (int64_t)n * cols;
    for (int64_t t = gtid; t < total; t += gthreads) {
      const int r = (int)(t / cols);
      if (r == c) continue;
      const int64_t k = c + 1 + t % cols;
      const double f = M[(int64_t)r * w + c] * inv;
      M[(int64_t)r * w + k] -= f * M[(int64_t)c * w + k];
    }
    grid.sync();
  }
  const int pc = n - 1;
  const double inv = 1.0 / M[(int64_t)pc * w + pc];
  for (int64_t k = pc + 1 + gtid; k < w; k += gthreads) M[(int64_t)pc * w + k] *= inv;
}

// x = T(Ainv * double(b)); Ainv is the right half of M (row stride 2n).
template <typename T>
__global__ void coarse_gemv_kernel(const double* M, const T* b, T* x, int n) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = M + (int64_t)row * 2 * n + n;
  double acc = 0.0;
  for (int j = lane; j < n; j += 32) acc += a[j] * (double)b[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) x[row] = T(acc);
}

__global__ void identity_right_kernel(double* M, int n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * n) return;
  const int64_t r = t / n, k = t % n;
  M[r * 2 * n + n + k] = r == k ? 1.0 : 0.0;
}

__global__ void copy_left_kernel(const double* A, double* M, int n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * n) return;
  const int64_t r = t / n, k = t % n;
  M[r * 2 * n + k] = A[t];
}

template <typename T>
void launch_probe_fill(T* x, int mx, int my, int mz, int s, int ca, int cb, int cc, int comp, cudaStream_t st) {
  const int64_t nn = (int64_t)mx * my * mz;
  probe_fill_kernel<T><<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(x, mx, my, mz, s, ca, cb, cc, comp);
}

template <typename T>
void launch_probe_extract(const T* y, double* A, int64_t n, int mx, int my, int mz, int p, int s, int ca, int cb,
                          int cc, int comp, cudaStream_t st) {
  probe_extract_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, A, n, mx, my, mz, p, s, ca, cb, cc, comp);
}

void launch_dense_invert(const double* A, double* M, int n, int* d_singular, cudaStream_t st) {
  const int64_t nn = (int64_t)n * n;
  const unsigned b = (unsigned)((nn + 255) / 256);
  copy_left_kernel<<<b, 256, 0, st>>>(A, M, n);
  identity_right_kernel<<<b, 256, 0, st>>>(M, n);
  static std::atomic<int> shape[64];
  const int threads = 512;
  int sms = 0, per = 0;
  per_device_shape(shape, sms, per, [&](int& p) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, gauss_jordan_kernel, threads, 0);
  });
  const int grid = sms;  // one CTA per SM: grid syncs stay cheap
  void* args[] = {(void*)&M, (void*)&n, (void*)&d_singular};
  cudaLaunchCooperativeKernel((const void*)gauss_jordan_kernel, dim3(grid), dim3(threads), args, 0, st);
}

template <typename T>
void launch_coarse_gemv(const double* M, const T* b, T* x, int n, cudaStream_t st) {
  coarse_gemv_kernel<T><<<(unsigned)((n + 7) / 8), 256, 0, st>>>(M, b, x, n);
}

template void launch_probe_fill<float>(float*, int, int, int, int, int, int, int, int, cudaStream_t);
template void launch_probe_fill<double>(double*, int, int, int, int, int, int, int, int, cudaStream_t);
template void launch_probe_extract<float>(const float*, double*, int64_t, int, int, int, int, int, int, int, int, int,
                                          cudaStream_t);
template void launch_probe_extract<double>(const double*, double*, int64_t, int, int, int, int, int, int, int, int,
                                           int, cudaStream_t);
template void launch_coarse_gemv<float>(const double*, const float*, float*, int, cudaStream_t);
template void launch_coarse_gemv<double>(const double*, const double*, double*, int, cudaStream_t);

}  // namespace emfgpu
