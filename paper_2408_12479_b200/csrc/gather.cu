// Node phase of the tangent apply: deterministic assembly of element-local
// results onto the lattice, one thread per node, in the reference's colour
// order.  The reference adds element results colour by colour
// (colour = (i&1) + 2(j&1) + 4(k&1), operator.hpp:145-153, 439), so every
// DoF accumulates its <=8 contributions sorted by (k parity, j parity,
// i parity); summing in exactly that order here reproduces the reference's
// association of the scatter sums, with no atomics and no colour passes.
// Dirichlet rows return the input (operator.hpp:617-620).
#include <cstdlib>


#include "gather.cuh"
#include "internal.h"

namespace emfgpu {

// Same assembly with the nodes of a plane flattened (a + mx b): every lane
// of a warp owns a node, where the (32, 8) tiling of an mx = 3n+1 row leaves
// a quarter of the warps almost empty (the kernel is issue-bound).
// 8 CTAs/SM (<= 32 registers): the kernel is latency-bound on its loc loads
// (long-scoreboard stalls), and at 39 registers only 6 CTAs fit (cfg2 fp64:
// 286 us for 1.18 GB of compulsory DRAM traffic, 4.1 TB/s).
#ifndef EMF_NODE_MINB
#define EMF_NODE_MINB 8
#endif
template <typename T, int P, bool GHOSTS>
__global__ void __launch_bounds__(256, EMF_NODE_MINB) node_gather_flat_kernel(const T* __restrict__ loc, const T* __restrict__ ghost_lo,
                                                               const T* __restrict__ ghost_hi, const T* x, T* y, int nx,
                                                               int ny, int nz, int faces, int kpar, int c0,
                                                               int periodic_y, FastDiv fd_mx) {
  const int mx = nx * P + 1, my = ny * P + (periodic_y ? 0 : 1);
  const int idx = blockIdx.x * 256 + threadIdx.x;
  const int c = blockIdx.y + c0;
  // launched as a programmatic dependent of the element kernel: wait for that
  // grid and its memory here, after the launch itself overlapped its tail
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (idx >= mx * my) return;
  const int b = (int)fd_mx.div((uint32_t)idx);
  const int a = idx - b * mx;
  assemble_node<T, P, false, GHOSTS>(loc, ghost_lo, ghost_hi, x, y, a, b, c, nx, ny, nz, faces, kpar, periodic_y);
}

// Programmatic dependent launch of the node phase (EMFGPU_PDL=0 disables).
static bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("EMFGPU_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

template <typename T>
void launch_node_gather(const T* loc, const T* ghost_lo, const T* ghost_hi, const T* x, T* y, int nx, int ny, int nz,
                        int p, int faces, int kpar, int c0, int c1, int periodic_y, cudaStream_t s, bool pdl) {
  if (c1 < c0) return;
  const int mx = nx * p + 1, my = ny * p + (periodic_y ? 0 : 1);
  {
    const dim3 gridf((unsigned)(((int64_t)mx * my + 255) / 256), c1 - c0 + 1);
    const FastDiv fd = FastDiv::make((uint32_t)mx);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gridf;
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_enabled()) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    switch (p) {
#define EMF_F(PP)                                                                                           \
  case PP:                                                                                                  \
    if (ghost_lo || ghost_hi)                                                                               \
      cudaLaunchKernelEx(&cfg, node_gather_flat_kernel<T, PP, true>, loc, ghost_lo, ghost_hi, x, y, nx, ny, nz, \
                         faces, kpar, c0, periodic_y, fd);                                                  \
    else                                                                                                    \
      cudaLaunchKernelEx(&cfg, node_gather_flat_kernel<T, PP, false>, loc, (const T*)nullptr,              \
                         (const T*)nullptr, x, y, nx, ny, nz, faces, kpar, c0, periodic_y, fd);             \
    break;
      EMF_F(1)
      EMF_F(2)
      EMF_F(3)
      EMF_F(4)
#undef EMF_F
    }
  }
}

// Face of element layer k: lower (side 0, local c=0) or upper (side 1, c=p)
// node plane of each element's local results (read from the component-major
// element-local results, loc_index), packed as ((j*nx+i)*N2 + b*N + a)*3 + comp.
template <typename T, int P>
__global__ void pack_face_kernel(const T* __restrict__ loc, T* __restrict__ face, int nx, int ny, int k, int side) {
  constexpr int N = P + 1, N2 = N * N;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)nx * ny * N2 * 3;
  if (idx >= total) return;
  const int comp = (int)(idx % 3);
  const int64_t fn = idx / 3;
  const int m2 = (int)(fn % N2);
  const int64_t ij = fn / N2;
  const int64_t j = ij / nx, i = ij - j * nx;
  const int lc = side ? P : 0;
  face[idx] = loc[loc_index<N>((int64_t)k * ny + j, (int)i, nx, lc, m2 / N, m2 % N, comp)];
}

template <typename T>
void launch_pack_face(const T* loc, T* face, int nx, int ny, int p, int k, int side, cudaStream_t s) {
  const int64_t total = (int64_t)nx * ny * (p + 1) * (p + 1) * 3;
  const unsigned g = (unsigned)((total + 255) / 256);
  switch (p) {
    case 1: pack_face_kernel<T, 1><<<g, 256, 0, s>>>(loc, face, nx, ny, k, side); break;
    case 2: pack_face_kernel<T, 2><<<g, 256, 0, s>>>(loc, face, nx, ny, k, side); break;
    case 3: pack_face_kernel<T, 3><<<g, 256, 0, s>>>(loc, face, nx, ny, k, side); break;
    case 4: pack_face_kernel<T, 4><<<g, 256, 0, s>>>(loc, face, nx, ny, k, side); break;
  }
}

// Diagonal epilogue: constrained rows -> 1, count free rows with d <= 0
// (operator.hpp:869-877).
template <typename T>
__global__ void diag_finish_kernel(T* d, int64_t nnodes, int mx, int my, int mz, int faces,
                                   unsigned long long* nbad, long long* bad_idx, long long cap) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nnodes) return;
  const int a = (int)(idx % mx), b = (int)((idx / mx) % my), c = (int)(idx / ((int64_t)mx * my));
  if (node_constrained(a, b, c, mx, my, mz, faces)) {
    d[3 * idx] = d[3 * idx + 1] = d[3 * idx + 2] = T(1);
    return;
  }
  // nonpositive free rows: counted, and their DoF indices appended (unordered;
  // the host sorts them into the reference's ascending order)
  for (int comp = 0; comp < 3; ++comp)
    if (!(d[3 * idx + comp] > T(0))) {
      const unsigned long long pos = atomicAdd(nbad, 1ull);
      if (bad_idx && (long long)pos < cap) bad_idx[pos] = 3 * idx + comp;
    }
}

template <typename T>
void launch_diag_finish(T* d, int64_t nnodes, int mx, int my, int mz, int faces, unsigned long long* nbad,
                        long long* bad_idx, long long cap, cudaStream_t s) {
  diag_finish_kernel<T><<<(unsigned)((nnodes + 255) / 256), 256, 0, s>>>(d, nnodes, mx, my, mz, faces, nbad, bad_idx,
                                                                          cap);
}

template void launch_node_gather<double>(const double*, const double*, const double*, const double*, double*, int,
                                         int, int, int, int, int, int, int, int, cudaStream_t, bool);
template void launch_node_gather<float>(const float*, const float*, const float*, const float*, float*, int, int,
                                        int, int, int, int, int, int, int, cudaStream_t, bool);
template void launch_pack_face<double>(const double*, double*, int, int, int, int, int, cudaStream_t);
template void launch_pack_face<float>(const float*, float*, int, int, int, int, int, cudaStream_t);
template void launch_diag_finish<double>(double*, int64_t, int, int, int, int, unsigned long long*, long long*,
                                         long long, cudaStream_t);
template void launch_diag_finish<float>(float*, int64_t, int, int, int, int, unsigned long long*, long long*,
                                        long long, cudaStream_t);

}  // namespace emfgpu
