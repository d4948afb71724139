// hp-multigrid ingredients on the device (fp32 or fp64 levels):
//   lattice transfers          TransferOp / lattice_sweep, mesh.hpp:190-289
//   Chebyshev-Jacobi updates   ChebyshevSmoother::smooth, solver.hpp:330-361
//   deterministic dot          dot_d, solver.hpp:95-100 (fixed-order tree)
#include "internal.h"

namespace emfgpu {

// One axis of a separable lattice transfer on an interleaved 3-component
// vector.  Forward (prolongate / interpolate_down): out[d] = sum_s w[d,s]
// in[src_elem[d]*p_src + s].  Transposed (restrict): each source-lattice
// index t gathers w[d,s] in[d] over the destinations d that touch it, in
// ascending d — the order in which the reference's scatter adds them
// (mesh.hpp:228-236) — through a CSR built on the host.
template <typename T>
__global__ void lattice_sweep_kernel(const T* __restrict__ in, T* __restrict__ out, const int* __restrict__ src_elem,
                                     const double* __restrict__ w, const int* __restrict__ t_ptr,
                                     const int* __restrict__ t_d, const int* __restrict__ t_s, int stencil,
                                     int p_src, int transpose, int axis, int in0, int in1, int in2, int out_na) {
  const int o0 = axis == 0 ? out_na : in0, o1 = axis == 1 ? out_na : in1, o2 = axis == 2 ? out_na : in2;
  const int64_t total = (int64_t)o0 * o1 * o2 * 3;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int comp = (int)(idx % 3);
  const int64_t node = idx / 3;
  const int a = (int)(node % o0), b = (int)((node / o0) % o1), c = (int)(node / ((int64_t)o0 * o1));
  const int pos = axis == 0 ? a : (axis == 1 ? b : c);
  auto in_at = [&](int t) -> T {
    const int aa = axis == 0 ? t : a, bb = axis == 1 ? t : b, cc = axis == 2 ? t : c;
    return in[(((int64_t)cc * in1 + bb) * in0 + aa) * 3 + comp];
  };
  T acc = T(0);
  if (!transpose) {
    const int base = src_elem[pos] * p_src;
    for (int s = 0; s < stencil; ++s) acc += T(w[pos * stencil + s]) * in_at(base + s);
  } else {
    for (int r = t_ptr[pos]; r < t_ptr[pos + 1]; ++r) acc += T(w[t_d[r] * stencil + t_s[r]]) * in_at(t_d[r]);
  }
  out[idx] = acc;
}

template <typename T>
void launch_transfer_axis(const T* in, T* out, const int* src_elem, const double* w, const int* t_ptr,
                          const int* t_d, const int* t_s, int stencil, int p_src, int transpose, int axis, int in0,
                          int in1, int in2, int out_na, cudaStream_t s) {
  const int o0 = axis == 0 ? out_na : in0, o1 = axis == 1 ? out_na : in1, o2 = axis == 2 ? out_na : in2;
  const int64_t total = (int64_t)o0 * o1 * o2 * 3;
  lattice_sweep_kernel<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      in, out, src_elem, w, t_ptr, t_d, t_s, stencil, p_src, transpose, axis, in0, in1, in2, out_na);
}
template void launch_transfer_axis<double>(const double*, double*, const int*, const double*, const int*, const int*,
                                           const int*, int, int, int, int, int, int, int, int, cudaStream_t);
template void launch_transfer_axis<float>(const float*, float*, const int*, const double*, const int*, const int*,
                                          const int*, int, int, int, int, int, int, int, int, cudaStream_t);

// ---- Chebyshev (solver.hpp:330-361) ------------------------------------------
template <typename T>
__global__ void cheb_first_kernel(T* __restrict__ x, T* __restrict__ r, T* __restrict__ d, const T* __restrict__ b,
                                  const T* __restrict__ inv_diag, T inv_theta, int zero_start, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // zero start: r = b, x = 0; else r holds A x on entry
  const T ri = b[i] - (zero_start ? T(0) : r[i]);
  const T di = (inv_theta * inv_diag[i]) * ri;
  const T xi = (zero_start ? T(0) : x[i]) + di;
  r[i] = ri;
  d[i] = di;
  x[i] = xi;
}

template <typename T>
__global__ void cheb_step_kernel(T* __restrict__ x, T* __restrict__ r, T* __restrict__ d, const T* __restrict__ ad,
                                 const T* __restrict__ inv_diag, T f1, T f2, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T ri = r[i] - ad[i];
  const T di = fma(f1, d[i], (f2 * inv_diag[i]) * ri);
  const T xi = x[i] + di;
  r[i] = ri;
  d[i] = di;
  x[i] = xi;
}

template <typename T>
__global__ void inv_kernel(const T* __restrict__ d, T* __restrict__ inv, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[i] = T(1) / d[i];
}

template <typename T>
void launch_cheb_first(T* x, T* r, T* d, const T* b, const T* inv_diag, double inv_theta, int zero_start, int64_t n,
                       cudaStream_t s) {
  cheb_first_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, r, d, b, inv_diag, T(inv_theta), zero_start, n);
}
template <typename T>
void launch_cheb_step(T* x, T* r, T* d, const T* ad, const T* inv_diag, double f1, double f2, int64_t n,
                      cudaStream_t s) {
  cheb_step_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, r, d, ad, inv_diag, T(f1), T(f2), n);
}
template <typename T>
void launch_inv(const T* d, T* inv, int64_t n, cudaStream_t s) {
  inv_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, inv, n);
}
template void launch_cheb_first<double>(double*, double*, double*, const double*, const double*, double, int, int64_t,
                                        cudaStream_t);
template void launch_cheb_first<float>(float*, float*, float*, const float*, const float*, double, int, int64_t,
                                       cudaStream_t);
template void launch_cheb_step<double>(double*, double*, double*, const double*, const double*, double, double,
                                       int64_t, cudaStream_t);
template void launch_cheb_step<float>(float*, float*, float*, const float*, const float*, double, double, int64_t,
                                      cudaStream_t);
template void launch_inv<double>(const double*, double*, int64_t, cudaStream_t);
template void launch_inv<float>(const float*, float*, int64_t, cudaStream_t);

// ---- deterministic dot: fixed grid, fixed per-thread ranges, tree in smem ----
constexpr int kDotBlocks = 592, kDotThreads = 256;

template <typename T>
__global__ void dot_partial_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t n, double* partial) {
  __shared__ double sm[kDotThreads];
  const int64_t gt = (int64_t)blockIdx.x * kDotThreads + threadIdx.x;
  const int64_t stride = (int64_t)kDotBlocks * kDotThreads;
  double s = 0.0;
  for (int64_t i = gt; i < n; i += stride) s += double(a[i]) * double(b[i]);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sm[0];
}

__global__ void dot_final_kernel(const double* partial, double* out) {
  __shared__ double sm[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += 1024) s += partial[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

template <typename T>
void launch_dot(const T* a, const T* b, int64_t n, double* partial, double* out, cudaStream_t s) {
  dot_partial_kernel<T><<<kDotBlocks, kDotThreads, 0, s>>>(a, b, n, partial);
  dot_final_kernel<<<1, 1024, 0, s>>>(partial, out);
}
template void launch_dot<double>(const double*, const double*, int64_t, double*, double*, cudaStream_t);

// ---- node-plane-chunked deterministic dot --------------------------------------
// Partials of whole lattice node planes (kPlaneSplit fixed sub-ranges per plane,
// each a fixed-order block reduction), then one ordered sum over all partials.
// A z-slab computes the partials of its owned planes only; since every
// partial is a function of its plane alone, the slab partials all-reduced
// (exact: one nonzero per slot) and summed give bitwise the single-GPU dot
// (csrc/slab_solver.cu).
constexpr int kPlaneSplit = 4, kPlaneThreads = 256;

template <typename T>
__global__ void dot_planes_kernel(const T* __restrict__ a, const T* __restrict__ b, int64_t plane_len, int first_plane,
                                  double* partial) {
  __shared__ double sm[kPlaneThreads];
  const int plane = blockIdx.x / kPlaneSplit, part = blockIdx.x % kPlaneSplit;
  const int64_t chunk = (plane_len + kPlaneSplit - 1) / kPlaneSplit;
  const int64_t i0 = (int64_t)plane * plane_len + part * chunk;
  const int64_t i1 = (int64_t)plane * plane_len + min(plane_len, (int64_t)(part + 1) * chunk);
  double s = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kPlaneThreads) s = fma(double(a[i]), double(b[i]), s);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = kPlaneThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)(first_plane + plane) * kPlaneSplit + part] = sm[0];
}

// The same partials for k vectors b_v = basis + v * stride against one a (the
// Lanczos reorthogonalisation): a is read once per group of kDotGroup vectors;
// per vector the summation order is dot_planes_kernel's, so partial[v] is
// bitwise what k separate launches give.
constexpr int kDotGroup = 4;
__global__ void multi_dot_planes_kernel(const double* __restrict__ a, const double* __restrict__ basis, int64_t stride,
                                        int k, int64_t plane_len, int64_t pstride, double* partial) {
  __shared__ double sm[kDotGroup][kPlaneThreads];
  const int plane = blockIdx.x / kPlaneSplit, part = blockIdx.x % kPlaneSplit;
  const int64_t chunk = (plane_len + kPlaneSplit - 1) / kPlaneSplit;
  const int64_t i0 = (int64_t)plane * plane_len + part * chunk;
  const int64_t i1 = (int64_t)plane * plane_len + min(plane_len, (int64_t)(part + 1) * chunk);
  for (int v0 = 0; v0 < k; v0 += kDotGroup) {
    double s[kDotGroup];
#pragma unroll
    for (int g = 0; g < kDotGroup; ++g) s[g] = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += kPlaneThreads) {
      const double ai = a[i];
#pragma unroll
      for (int g = 0; g < kDotGroup; ++g)
        if (v0 + g < k) s[g] = fma(ai, basis[(int64_t)(v0 + g) * stride + i], s[g]);
    }
#pragma unroll
    for (int g = 0; g < kDotGroup; ++g) sm[g][threadIdx.x] = s[g];
    __syncthreads();
    for (int w = kPlaneThreads / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
#pragma unroll
        for (int g = 0; g < kDotGroup; ++g) sm[g][threadIdx.x] += sm[g][threadIdx.x + w];
      }
      __syncthreads();
    }
    if (threadIdx.x < kDotGroup && v0 + threadIdx.x < k)
      partial[(int64_t)(v0 + threadIdx.x) * pstride + (int64_t)plane * kPlaneSplit + part] = sm[threadIdx.x][0];
    __syncthreads();
  }
}
// out[v] = ordered sum of partial[v * pstride .. + m): sum_ordered_kernel per vector
__global__ void multi_sum_ordered_kernel(const double* partial, int64_t pstride, int64_t m, double* out) {
  __shared__ double sm[1024];
  const double* p = partial + (int64_t)blockIdx.x * pstride;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 1024) s += p[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}
// y -= c[0] x_0, then c[1] x_1, ... in this order (k axpy_dev_kernel launches in one)
__global__ void multi_axpy_dev_kernel(const double* __restrict__ c, const double* __restrict__ basis, int64_t stride,
                                      int k, double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double yi = y[i];
  for (int v = 0; v < k; ++v) yi = fma(-c[v], basis[(int64_t)v * stride + i], yi);
  y[i] = yi;
}
void launch_multi_dot_planes(const double* a, const double* basis, int64_t stride, int k, int64_t plane_len,
                             int nplanes, double* partial, int64_t pstride, double* out, cudaStream_t s) {
  if (k <= 0 || nplanes <= 0) return;
  multi_dot_planes_kernel<<<(unsigned)(nplanes * kPlaneSplit), kPlaneThreads, 0, s>>>(a, basis, stride, k, plane_len,
                                                                                    pstride, partial);
  multi_sum_ordered_kernel<<<(unsigned)k, 1024, 0, s>>>(partial, pstride, (int64_t)nplanes * kPlaneSplit, out);
}
void launch_multi_axpy_dev(const double* c, const double* basis, int64_t stride, int k, double* y, int64_t n,
                           cudaStream_t s) {
  if (k > 0) multi_axpy_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c, basis, stride, k, y, n);
}

__global__ void sum_ordered_kernel(const double* partial, int64_t m, double* out) {
  __shared__ double sm[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 1024) s += partial[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

template <typename T>
void launch_dot_plane_partials(const T* a, const T* b, int64_t plane_len, int nplanes, int first_plane,
                               double* partial, cudaStream_t s) {
  if (nplanes > 0)
    dot_planes_kernel<T><<<(unsigned)(nplanes * kPlaneSplit), kPlaneThreads, 0, s>>>(a, b, plane_len, first_plane,
                                                                                     partial);
}
void launch_sum_ordered(const double* partial, int64_t m, double* out, cudaStream_t s) {
  sum_ordered_kernel<<<1, 1024, 0, s>>>(partial, m, out);
}
int dot_plane_split() { return kPlaneSplit; }
template <typename T>
void launch_dot_planes(const T* a, const T* b, int64_t plane_len, int nplanes, double* partial, double* out,
                       cudaStream_t s) {
  launch_dot_plane_partials<T>(a, b, plane_len, nplanes, 0, partial, s);
  launch_sum_ordered(partial, (int64_t)nplanes * kPlaneSplit, out, s);
}
template void launch_dot_plane_partials<double>(const double*, const double*, int64_t, int, int, double*,
                                                cudaStream_t);
template void launch_dot_plane_partials<float>(const float*, const float*, int64_t, int, int, double*, cudaStream_t);
template void launch_dot_planes<double>(const double*, const double*, int64_t, int, double*, double*, cudaStream_t);
template void launch_dot_planes<float>(const float*, const float*, int64_t, int, double*, double*, cudaStream_t);
template void launch_dot<float>(const float*, const float*, int64_t, double*, double*, cudaStream_t);
int dot_partial_count() { return kDotBlocks; }

// ---- Lanczos vector kernels (solver.hpp:271-300) -------------------------------
template <typename T>
__global__ void scale_to_T_kernel(const double* __restrict__ s, const double* __restrict__ v, T* __restrict__ t,
                                  int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) t[i] = T(s[i] * v[i]);
}
template <typename T>
__global__ void scale_from_T_kernel(const double* __restrict__ s, const T* __restrict__ at, double* __restrict__ w,
                                    int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = s[i] * double(at[i]);
}
template <typename T>
__global__ void dinv_sqrt_kernel(const T* __restrict__ d, double* __restrict__ s, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) s[i] = 1.0 / sqrt(fmax(1e-300, double(d[i])));
}
__global__ void axpy_d_kernel(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] -= a * x[i];
}
__global__ void scal_d_kernel(const double* __restrict__ x, double inv, double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / inv;
}

// Lanczos start vector (solver.hpp:274-277): element i of the sequential
// splitmix64 stream is mix(seed + (i+1) gamma), so it is generated in parallel.
__global__ void lanczos_start_kernel(double* __restrict__ v, int64_t n, unsigned long long seed, int64_t offset) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // element (offset + i) of the reference's sequential splitmix64 stream
  unsigned long long z = seed + (unsigned long long)(offset + i + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  v[i] = (double)(z >> 11) * 0x1.0p-53 - 0.5;
}
// y -= c[0] x with the coefficient read from device memory (no host round trip)
__global__ void axpy_dev_kernel(const double* __restrict__ c, const double* __restrict__ x, double* __restrict__ y,
                                int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fma(-c[0], x[i], y[i]);
}
// y = x / sqrt(d[0])
__global__ void div_sqrt_dev_kernel(const double* __restrict__ d, const double* __restrict__ x,
                                    double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / sqrt(d[0]);
}
void launch_lanczos_start(double* v, int64_t n, unsigned long long seed, cudaStream_t st, int64_t offset) {
  lanczos_start_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, n, seed, offset);
}
void launch_axpy_dev(const double* c, const double* x, double* y, int64_t n, cudaStream_t st) {
  axpy_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(c, x, y, n);
}
void launch_div_sqrt_dev(const double* d, const double* x, double* y, int64_t n, cudaStream_t st) {
  div_sqrt_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d, x, y, n);
}

template <typename T>
void launch_scale_to_T(const double* s, const double* v, T* t, int64_t n, cudaStream_t st) {
  scale_to_T_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, v, t, n);
}
template <typename T>
void launch_scale_from_T(const double* s, const T* at, double* w, int64_t n, cudaStream_t st) {
  scale_from_T_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, at, w, n);
}
template <typename T>
void launch_dinv_sqrt(const T* d, double* s, int64_t n, cudaStream_t st) {
  dinv_sqrt_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d, s, n);
}
void launch_axpy_minus(double a, const double* x, double* y, int64_t n, cudaStream_t st) {
  axpy_d_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, x, y, n);
}
void launch_div(const double* x, double b, double* y, int64_t n, cudaStream_t st) {
  scal_d_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, b, y, n);
}
template void launch_scale_to_T<double>(const double*, const double*, double*, int64_t, cudaStream_t);
template void launch_scale_to_T<float>(const double*, const double*, float*, int64_t, cudaStream_t);
template void launch_scale_from_T<double>(const double*, const double*, double*, int64_t, cudaStream_t);
template void launch_scale_from_T<float>(const double*, const float*, double*, int64_t, cudaStream_t);
template void launch_dinv_sqrt<double>(const double*, double*, int64_t, cudaStream_t);
template void launch_dinv_sqrt<float>(const float*, double*, int64_t, cudaStream_t);

}  // namespace emfgpu

// ---- multigrid / Krylov vector kernels ----------------------------------------
namespace emfgpu {

// v = 0 on Dirichlet DoFs (FeLevel::dirichlet_set_zero, mesh.hpp:115-119)
template <typename T>
__global__ void mask_zero_kernel(T* v, int64_t nnodes, int mx, int my, int mz, int faces) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  const int a = (int)(i % mx), b = (int)((i / mx) % my), c = (int)(i / ((int64_t)mx * my));
  if (node_constrained(a, b, c, mx, my, mz, faces)) v[3 * i] = v[3 * i + 1] = v[3 * i + 2] = T(0);
}
template <typename T>
void launch_mask_zero(T* v, int64_t nnodes, int mx, int my, int mz, int faces, cudaStream_t s) {
  if (faces) mask_zero_kernel<T><<<(unsigned)((nnodes + 255) / 256), 256, 0, s>>>(v, nnodes, mx, my, mz, faces);
}
template void launch_mask_zero<double>(double*, int64_t, int, int, int, int, cudaStream_t);
template void launch_mask_zero<float>(float*, int64_t, int, int, int, int, cudaStream_t);

template <typename Ti, typename To>
__global__ void cast_kernel(const Ti* __restrict__ in, To* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = To(in[i]);
}
template <typename Ti, typename To>
void launch_cast(const Ti* in, To* out, int64_t n, cudaStream_t s) {
  cast_kernel<Ti, To><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n);
}
template void launch_cast<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_cast<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_cast<double, double>(const double*, double*, int64_t, cudaStream_t);

// t = b - t (residual from t = A x)
template <typename T>
__global__ void bminus_kernel(const T* __restrict__ b, T* __restrict__ t, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) t[i] = b[i] - t[i];
}
template <typename T>
void launch_bminus(const T* b, T* t, int64_t n, cudaStream_t s) {
  bminus_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(b, t, n);
}
template void launch_bminus<double>(const double*, double*, int64_t, cudaStream_t);
template void launch_bminus<float>(const float*, float*, int64_t, cudaStream_t);

// y += x
template <typename T>
__global__ void add_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += x[i];
}
template <typename T>
void launch_add(const T* x, T* y, int64_t n, cudaStream_t s) {
  add_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, y, n);
}
template void launch_add<double>(const double*, double*, int64_t, cudaStream_t);
template void launch_add<float>(const float*, float*, int64_t, cudaStream_t);

// CG update: x += T(alpha) p ; r -= T(alpha) ap  (solver.hpp:410-413)
template <typename T>
__global__ void cg_xr_kernel(T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                             const T* __restrict__ ap, T alpha, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] += alpha * p[i];
  r[i] -= alpha * ap[i];
}
template <typename T>
void launch_cg_xr(T* x, T* r, const T* p, const T* ap, double alpha, int64_t n, cudaStream_t s) {
  cg_xr_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, r, p, ap, T(alpha), n);
}
template void launch_cg_xr<double>(double*, double*, const double*, const double*, double, int64_t, cudaStream_t);
template void launch_cg_xr<float>(float*, float*, const float*, const float*, double, int64_t, cudaStream_t);

// p = z + T(beta) p
template <typename T>
__global__ void cg_p_kernel(T* __restrict__ p, const T* __restrict__ z, T beta, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = z[i] + beta * p[i];
}
template <typename T>
void launch_cg_p(T* p, const T* z, double beta, int64_t n, cudaStream_t s) {
  cg_p_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, z, T(beta), n);
}
template void launch_cg_p<double>(double*, const double*, double, int64_t, cudaStream_t);
template void launch_cg_p<float>(float*, const float*, double, int64_t, cudaStream_t);

// ---- device-resident PCG (capi.cu emfgpu_pcg_solve) -------------------------
// Scalars live on the device: sc = {rz, p.Ap, r.r, rz_new, ||b||}, ic = {it, done}.
// The arithmetic is the host loop's, in the same order (alpha = rz / pAp,
// rel = sqrt(rr) / ||b||, beta = rz_new / rz), so iterates are identical.
__global__ void pcg_xr_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                              const double* __restrict__ ap, const double* __restrict__ sc, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double alpha = sc[0] / sc[1];
  x[i] += alpha * p[i];
  r[i] -= alpha * ap[i];
}
__global__ void pcg_p_kernel(double* __restrict__ p, const double* __restrict__ z, const double* __restrict__ sc,
                             int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double beta = sc[3] / sc[0];
  p[i] = z[i] + beta * p[i];
}
__global__ void pcg_shift_kernel(double* sc) { sc[0] = sc[3]; }
__global__ void pcg_sqrt_kernel(double* v) { *v = sqrt(*v); }
__global__ void pcg_check_kernel(const double* __restrict__ sc, int* ic, double* hist, double rtol, int maxit,
                                 cudaGraphConditionalHandle h, int use_h) {
  const double rel = sqrt(sc[2]) / sc[4];
  const int it = ic[0] + 1;
  hist[it] = rel;
  ic[0] = it;
  // pAp <= 0: the operator is not positive definite on p (CG breakdown)
  const int breakdown = !(sc[1] > 0.0);
  if (breakdown) ic[2] = 1;
  const int stop = (rel <= rtol) || it >= maxit || breakdown;
  ic[1] = stop;
  if (use_h) cudaGraphSetConditional(h, stop ? 0u : 1u);
}
void launch_pcg_xr(double* x, double* r, const double* p, const double* ap, const double* sc, int64_t n,
                   cudaStream_t s) {
  pcg_xr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, r, p, ap, sc, n);
}
void launch_pcg_p(double* p, const double* z, const double* sc, int64_t n, cudaStream_t s) {
  pcg_p_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, z, sc, n);
}
void launch_pcg_shift(double* sc, cudaStream_t s) { pcg_shift_kernel<<<1, 1, 0, s>>>(sc); }
void launch_pcg_sqrt(double* v, cudaStream_t s) { pcg_sqrt_kernel<<<1, 1, 0, s>>>(v); }
void launch_pcg_check(const double* sc, int* ic, double* hist, double rtol, int maxit, cudaGraphConditionalHandle h,
                      int use_h, cudaStream_t s) {
  pcg_check_kernel<<<1, 1, 0, s>>>(sc, ic, hist, rtol, maxit, h, use_h);
}

// z = inv * r (Jacobi)
template <typename T>
__global__ void jacobi_kernel(const T* __restrict__ inv, const T* __restrict__ r, T* __restrict__ z, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = inv[i] * r[i];
}
template <typename T>
void launch_jacobi(const T* inv, const T* r, T* z, int64_t n, cudaStream_t s) {
  jacobi_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(inv, r, z, n);
}
template void launch_jacobi<double>(const double*, const double*, double*, int64_t, cudaStream_t);
template void launch_jacobi<float>(const float*, const float*, float*, int64_t, cudaStream_t);

}  // namespace emfgpu

namespace emfgpu {
// evaluate_residual tail (operator.hpp:638-640): r -= scale * load; Dirichlet rows = 0
template <typename T>
__global__ void sub_load_mask_kernel(T* r, const T* load, T scale, int64_t nnodes, int mx, int my, int mz,
                                     int faces) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnodes) return;
  const int a = (int)(i % mx), b = (int)((i / mx) % my), c = (int)(i / ((int64_t)mx * my));
  const bool fixed = node_constrained(a, b, c, mx, my, mz, faces);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    T v = r[3 * i + d];
    if (load) v -= scale * load[3 * i + d];
    r[3 * i + d] = fixed ? T(0) : v;
  }
}
template <typename T>
void launch_sub_load_mask(T* r, const T* load, double scale, int64_t nnodes, int mx, int my, int mz, int faces,
                          cudaStream_t s) {
  sub_load_mask_kernel<T><<<(unsigned)((nnodes + 255) / 256), 256, 0, s>>>(r, load, T(scale), nnodes, mx, my, mz,
                                                                            faces);
}
template void launch_sub_load_mask<double>(double*, const double*, double, int64_t, int, int, int, int, cudaStream_t);
template void launch_sub_load_mask<float>(float*, const float*, double, int64_t, int, int, int, int, cudaStream_t);
}  // namespace emfgpu
