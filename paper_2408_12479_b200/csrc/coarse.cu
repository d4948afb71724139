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

// [A | I] -> A^-1 on M (n x 2n, row-major), partial pivoting with DenseLU's
// rule (the first row of maximal |a| among the remaining ones, solver.hpp:55-63).
// One grid synchronisation per column: the row interchanges are logical (every
// CTA keeps the same position -> row permutation in shared memory and finds
// the pivot redundantly), and the scaling of the previous pivot row is folded
// into the elimination pass that first reads it.  The arithmetic per entry is
// that of the three-pass form (interchange, scale, eliminate).  The inverse's
// rows end in the left halves of M in their logical order.
__global__ void gauss_jordan_kernel(double* M, int n, int* singular) {
  cg::grid_group grid = cg::this_grid();
  const int w = 2 * n;
  extern __shared__ int s_perm[];  // logical position -> physical row
  __shared__ double s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_piv;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  for (int p = threadIdx.x; p < n; p += blockDim.x) s_perm[p] = p;
  __syncthreads();
  int prev = -1;          // physical row of the previous pivot (still unscaled in memory)
  double inv_prev = 0.0;  // 1 / its pivot
  for (int c = 0; c < n; ++c) {
    // pivot of column c among the logical positions c..n-1
    double best = -1.0;
    int bi = n;
    for (int p = c + threadIdx.x; p < n; p += blockDim.x) {
      const double v = fabs(M[(int64_t)s_perm[p] * w + c]);
      if (v > best) {  // strictly greater: first position of maximal |a|
        best = v;
        bi = p;
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
      if (!(b2 >= 1e-250)) {
        if (blockIdx.x == 0) atomicExch(singular, 1);
        i2 = c;  // keep going on a defined row; the caller reports the singular matrix
      }
      const int t = s_perm[c];  // the interchange of positions c and i2
      s_perm[c] = s_perm[i2];
      s_perm[i2] = t;
      s_piv = s_perm[c];
    }
    __syncthreads();
    const int prow = s_piv;
    // eliminate column c from every other row (pivot row read unscaled); the
    // previous pivot row is scaled by its 1 / pivot as it is read
    // (a warp per row with lanes over the columns measured slower, 22.7 vs 17.0 ms:
    // only n of the grid's warps work, each in a long dependent loop)
    const double inv = 1.0 / M[(int64_t)prow * w + c];
    const unsigned cols = (unsigned)(w - c - 1);
    const unsigned total = (unsigned)n * cols;  // n <= coarse_direct_limit: fits 32 bits
    const double* const prw = M + (int64_t)prow * w + c + 1;
    for (unsigned t = (unsigned)gtid; t < total; t += (unsigned)gthreads) {
      const unsigned r = t / cols, k = t - r * cols;
      if ((int)r == prow) continue;
      double* const row = M + (int64_t)r * w + c;
      const double sc = (int)r == prev ? inv_prev : 1.0;  // x * 1.0 is exact
      const double f = (row[0] * sc) * inv;
      row[1 + k] = fma(-f, prw[k], row[1 + k] * sc);
    }
    prev = prow;
    inv_prev = inv;
    grid.sync();
  }
  // the last pivot row's scaling, then the rows into logical order (left halves)
  for (int64_t k = n + gtid; k < w; k += gthreads) M[(int64_t)prev * w + k] *= inv_prev;
  grid.sync();
  for (int64_t t = gtid; t < (int64_t)n * n; t += gthreads) {
    const int p = (int)(t / n);
    const int64_t k = t % n;
    M[(int64_t)p * w + k] = M[(int64_t)s_perm[p] * w + n + k];
  }
}

// x = T(Ainv * double(b)); Ainv is the left half of M (row stride 2n).
template <typename T>
__global__ void coarse_gemv_kernel(const double* M, const T* b, T* x, int n) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = M + (int64_t)row * 2 * n;
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, gauss_jordan_kernel, threads, sizeof(int) * 2048);
  });
  const int grid = sms;  // one CTA per SM: grid syncs stay cheap
  void* args[] = {(void*)&M, (void*)&n, (void*)&d_singular};
  cudaLaunchCooperativeKernel((const void*)gauss_jordan_kernel, dim3(grid), dim3(threads), args, sizeof(int) * n, st);
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
