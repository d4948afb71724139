// Node phase of the tangent apply: deterministic assembly of element-local
// results onto the lattice, one thread per node, in the reference's colour
// order.  The reference adds element results colour by colour
// (colour = (i&1) + 2(j&1) + 4(k&1), operator.hpp:145-153, 439), so every
// DoF accumulates its <=8 contributions sorted by (k parity, j parity,
// i parity); summing in exactly that order here reproduces the reference's
// association of the scatter sums, with no atomics and no colour passes.
// Dirichlet rows return the input (operator.hpp:617-620).
#include "internal.h"

namespace emfgpu {

// Candidate elements along one axis for lattice coordinate a (element size p,
// n elements, lattice size m), sorted even-index first. Local node index in
// the element along that axis is returned in loc[].  lo/hi ghost layers are
// allowed along z (index -1 and n).
__device__ __forceinline__ int axis_candidates(int a, int p, int n, int gpar, bool ghosts, int* el, int* loc,
                                               bool periodic = false) {
  const int e1 = a / p;
  if (periodic && a == 0) {  // seam of a periodic lattice: elements n-1 (local p) and 0 (local 0)
    const bool odd_last = ((n - 1) & 1) != 0;
    el[0] = odd_last ? 0 : n - 1;
    loc[0] = odd_last ? 0 : p;
    el[1] = odd_last ? n - 1 : 0;
    loc[1] = odd_last ? p : 0;
    return 2;
  }
  if (a % p == 0) {
    const bool has_lo = a > 0 || ghosts;
    const bool has_hi = a < n * p || ghosts;
    int cnt = 0;
    int c_el[2], c_loc[2];
    if (has_lo) {
      c_el[cnt] = e1 - 1;
      c_loc[cnt] = p;
      ++cnt;
    }
    if (has_hi) {
      c_el[cnt] = e1;
      c_loc[cnt] = 0;
      ++cnt;
    }
    if (cnt == 2 && (((c_el[0] + gpar) & 1) != 0)) {  // odd first -> swap so even (global) goes first
      el[0] = c_el[1];
      loc[0] = c_loc[1];
      el[1] = c_el[0];
      loc[1] = c_loc[0];
    } else {
      for (int t = 0; t < cnt; ++t) {
        el[t] = c_el[t];
        loc[t] = c_loc[t];
      }
    }
    return cnt;
  }
  el[0] = e1;
  loc[0] = a - e1 * p;
  return 1;
}

// One thread per lattice node; 3-D grid (x: 32 nodes along a, y: 8 along b,
// z: node planes) so no index division is needed.  Per axis a node has two
// candidate-element slots ordered even index first (a non-shared node uses
// only the first); the 2x2x2 slot product is visited z-major, which is the
// reference's colour order, with predicated loads and a running sum that
// starts at 0 exactly like y = 0; y += ... in operator.hpp:606, 439.
struct AxisSlots {
  int e[2], l[2];
  bool v[2];
};

template <int P>
__device__ __forceinline__ AxisSlots axis_slots(int a, int n, int par, bool lo_ok, bool hi_ok, bool periodic) {
  AxisSlots s;
  const int q = a / P, r = a - q * P;
  if (r != 0) {
    s.e[0] = q;
    s.l[0] = r;
    s.v[0] = true;
    s.e[1] = q;
    s.l[1] = 0;
    s.v[1] = false;
    return s;
  }
  int elo = q - 1, ehi = q;
  bool vlo = q > 0 || lo_ok, vhi = q < n || hi_ok;
  if (periodic && q == 0) {
    elo = n - 1;
    vlo = true;
  }
  // the even (global) element index first
  const bool swap = ((elo + par) & 1) != 0;
  s.e[0] = swap ? ehi : elo;
  s.l[0] = swap ? 0 : P;
  s.v[0] = swap ? vhi : vlo;
  s.e[1] = swap ? elo : ehi;
  s.l[1] = swap ? P : 0;
  s.v[1] = swap ? vlo : vhi;
  return s;
}

template <typename T, int P>
__global__ void __launch_bounds__(256) node_gather_kernel(const T* __restrict__ loc, const T* __restrict__ ghost_lo,
                                                          const T* __restrict__ ghost_hi, const T* x, T* y, int nx,
                                                          int ny, int nz, int faces, int kpar, int c0,
                                                          int periodic_y) {
  constexpr int N = P + 1, N3 = N * N * N, N2 = N * N;
  const int mx = nx * P + 1, my = ny * P + (periodic_y ? 0 : 1), mz = nz * P + 1;
  const int a = blockIdx.x * 32 + threadIdx.x;
  const int b = blockIdx.y * 8 + threadIdx.y;
  const int c = blockIdx.z + c0;
  if (a >= mx || b >= my) return;
  const int64_t idx = ((int64_t)c * my + b) * mx + a;
  if (node_constrained(a, b, c, mx, my, mz, faces)) {
    y[3 * idx] = x[3 * idx];
    y[3 * idx + 1] = x[3 * idx + 1];
    y[3 * idx + 2] = x[3 * idx + 2];
    return;
  }
  const AxisSlots sx = axis_slots<P>(a, nx, 0, false, false, false);
  const AxisSlots sy = axis_slots<P>(b, ny, 0, false, false, periodic_y != 0);
  const AxisSlots sz = axis_slots<P>(c, nz, kpar, ghost_lo != nullptr, ghost_hi != nullptr, false);
  T s0 = T(0), s1 = T(0), s2 = T(0);
#pragma unroll
  for (int tk = 0; tk < 2; ++tk)
#pragma unroll
    for (int tj = 0; tj < 2; ++tj)
#pragma unroll
      for (int ti = 0; ti < 2; ++ti) {
        if (!(sz.v[tk] && sy.v[tj] && sx.v[ti])) continue;
        const int k = sz.e[tk];
        T v0, v1, v2;
        if (k < 0 || k >= nz) {
          const T* src = k < 0 ? ghost_lo : ghost_hi;
          const int64_t off = ((((int64_t)sy.e[tj] * nx + sx.e[ti]) * N2) + sy.l[tj] * N + sx.l[ti]) * 3;
          v0 = src[off];
          v1 = src[off + 1];
          v2 = src[off + 2];
        } else {  // element-local results, component-major loc[(e*3 + c)*N3 + m]
          const int64_t e = ((int64_t)k * ny + sy.e[tj]) * nx + sx.e[ti];
          const int64_t off = e * 3 * N3 + (sz.l[tk] * N + sy.l[tj]) * N + sx.l[ti];
          v0 = loc[off];
          v1 = loc[off + N3];
          v2 = loc[off + 2 * N3];
        }
        s0 += v0;
        s1 += v1;
        s2 += v2;
      }
  y[3 * idx] = s0;
  y[3 * idx + 1] = s1;
  y[3 * idx + 2] = s2;
}

template <typename T>
void launch_node_gather(const T* loc, const T* ghost_lo, const T* ghost_hi, const T* x, T* y, int nx, int ny, int nz,
                        int p, int faces, int kpar, int c0, int c1, int periodic_y, cudaStream_t s) {
  if (c1 < c0) return;
  const int mx = nx * p + 1, my = ny * p + (periodic_y ? 0 : 1);
  const dim3 grid((mx + 31) / 32, (my + 7) / 8, c1 - c0 + 1), block(32, 8);
  switch (p) {
#define EMF_G(PP)                                                                                             \
  case PP:                                                                                                    \
    node_gather_kernel<T, PP><<<grid, block, 0, s>>>(loc, ghost_lo, ghost_hi, x, y, nx, ny, nz, faces, kpar, c0, periodic_y); \
    break;
    EMF_G(1)
    EMF_G(2)
    EMF_G(3)
    EMF_G(4)
#undef EMF_G
  }
}

// Face of element layer k: lower (side 0, local c=0) or upper (side 1, c=p)
// node plane of each element's local results (read from the component-major
// loc[(e*3 + c)*N3 + m]), packed as ((j*nx+i)*N2 + b*N + a)*3 + comp.
template <typename T>
__global__ void pack_face_kernel(const T* __restrict__ loc, T* __restrict__ face, int nx, int ny, int p, int k,
                                 int side) {
  const int N = p + 1, N2 = N * N, N3 = N2 * N;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)nx * ny * N2 * 3;
  if (idx >= total) return;
  const int comp = (int)(idx % 3);
  const int64_t fn = idx / 3;
  const int m2 = (int)(fn % N2);
  const int64_t ij = fn / N2;
  const int64_t e = (int64_t)k * nx * ny + ij;
  const int lc = side ? p : 0;
  face[idx] = loc[(e * 3 + comp) * N3 + lc * N2 + m2];
}

template <typename T>
void launch_pack_face(const T* loc, T* face, int nx, int ny, int p, int k, int side, cudaStream_t s) {
  const int64_t total = (int64_t)nx * ny * (p + 1) * (p + 1) * 3;
  pack_face_kernel<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(loc, face, nx, ny, p, k, side);
}

// Diagonal epilogue: constrained rows -> 1, count free rows with d <= 0
// (operator.hpp:869-877).
template <typename T>
__global__ void diag_finish_kernel(T* d, int64_t nnodes, int mx, int my, int mz, int faces,
                                   unsigned long long* nbad) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nnodes) return;
  const int a = (int)(idx % mx), b = (int)((idx / mx) % my), c = (int)(idx / ((int64_t)mx * my));
  if (node_constrained(a, b, c, mx, my, mz, faces)) {
    d[3 * idx] = d[3 * idx + 1] = d[3 * idx + 2] = T(1);
    return;
  }
  int bad = 0;
  for (int comp = 0; comp < 3; ++comp) bad += !(d[3 * idx + comp] > T(0));
  if (bad) atomicAdd(nbad, (unsigned long long)bad);
}

template <typename T>
void launch_diag_finish(T* d, int64_t nnodes, int mx, int my, int mz, int faces, unsigned long long* nbad,
                        cudaStream_t s) {
  diag_finish_kernel<T><<<(unsigned)((nnodes + 255) / 256), 256, 0, s>>>(d, nnodes, mx, my, mz, faces, nbad);
}

template void launch_node_gather<double>(const double*, const double*, const double*, const double*, double*, int,
                                         int, int, int, int, int, int, int, int, cudaStream_t);
template void launch_node_gather<float>(const float*, const float*, const float*, const float*, float*, int, int,
                                        int, int, int, int, int, int, int, cudaStream_t);
template void launch_pack_face<double>(const double*, double*, int, int, int, int, int, cudaStream_t);
template void launch_pack_face<float>(const float*, float*, int, int, int, int, int, cudaStream_t);
template void launch_diag_finish<double>(double*, int64_t, int, int, int, int, unsigned long long*, cudaStream_t);
template void launch_diag_finish<float>(float*, int64_t, int, int, int, int, unsigned long long*, cudaStream_t);

}  // namespace emfgpu
