// Node-phase assembly of one lattice node (shared by the node-gather kernel
// and the fused host-vector apply).  See gather.cu for the ordering argument.
#pragma once
#include "kernels.cuh"

namespace emfgpu {

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

// y(node) = sum of the node's element contributions in colour order (or x on
// Dirichlet rows).  CG = true reads the element results through L2 only
// (written by other CTAs of the same launch).
template <typename T, int P, bool CG = false, bool GHOSTS = true>
__device__ __forceinline__ void assemble_node(const T* __restrict__ loc, const T* __restrict__ ghost_lo,
                                              const T* __restrict__ ghost_hi, const T* x, T* y, int a, int b, int c,
                                              int nx, int ny, int nz, int faces, int kpar, int periodic_y) {
  constexpr int N = P + 1, N2 = N * N;
  const int mx = nx * P + 1, my = ny * P + (periodic_y ? 0 : 1), mz = nz * P + 1;
  const int64_t idx = ((int64_t)c * my + b) * mx + a;
  if (node_constrained(a, b, c, mx, my, mz, faces)) {
    y[3 * idx] = x[3 * idx];
    y[3 * idx + 1] = x[3 * idx + 1];
    y[3 * idx + 2] = x[3 * idx + 2];
    return;
  }
  auto ld = [](const T* p) { return CG ? __ldcg(p) : *p; };
  const AxisSlots sx = axis_slots<P>(a, nx, 0, false, false, false);
  const AxisSlots sy = axis_slots<P>(b, ny, 0, false, false, periodic_y != 0);
  const AxisSlots sz = axis_slots<P>(c, nz, kpar, GHOSTS && ghost_lo != nullptr, GHOSTS && ghost_hi != nullptr, false);
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
        if (GHOSTS && (k < 0 || k >= nz)) {
          const T* src = k < 0 ? ghost_lo : ghost_hi;
          const int64_t off = ((((int64_t)sy.e[tj] * nx + sx.e[ti]) * N2) + sy.l[tj] * N + sx.l[ti]) * 3;
          v0 = src[off];
          v1 = src[off + 1];
          v2 = src[off + 2];
        } else {  // element-local results (loc_index, kernels.cuh)
          const int64_t off = loc_index<N>((int64_t)k * ny + sy.e[tj], sx.e[ti], nx, sz.l[tk], sy.l[tj], sx.l[ti], 0);
          const int64_t cs = loc_cstride<N>(nx);
          v0 = ld(loc + off);
          v1 = ld(loc + off + cs);
          v2 = ld(loc + off + 2 * cs);
        }
        s0 += v0;
        s1 += v1;
        s2 += v2;
      }
  y[3 * idx] = s0;
  y[3 * idx + 1] = s1;
  y[3 * idx + 2] = s2;
}

}  // namespace emfgpu
