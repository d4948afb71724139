// Level geometry on the device: the isoparametric Jacobian J0 = dX/dxi of the
// GLL-interpolated node coordinates at every Gauss point, computed with the
// same forward sweeps as the tangent kernels (mesh.cpp:162-186), then stored
// as the factors the apply consumes: J0^-1 (9) and det(J0) * w_q, SoA.
// If every element's J0 is constant over its quadrature points (affine
// mesh), the level keeps one copy per element.
#include "internal.h"

namespace emfgpu {

struct GeoArgs {
  const double* coords;
  double* geo;    // 11 fields * nqp: J0^-1 (9), det*w, det
  double* j0out;  // optional, 9 per qp (row = comp), FeLevel::jacobians layout
  int nx, ny, nz, mx, my;
  int64_t nel, stride;
  double B[81], D[81], qw[9];
  int* nonaffine;
  int* degenerate;
};

template <int P>
__global__ void __launch_bounds__(Tile<P>::EPB*(P + 1) * (P + 1) * (P + 1)) geometry_kernel(const GeoArgs a) {
  constexpr int N = P + 1, N3 = N * N * N, EPB = Tile<P>::EPB;
  __shared__ double sB[N * N], sD[N * N];
  __shared__ double bufA[EPB][9][N3], bufB[EPB][9][N3];
  __shared__ double j0q0[EPB][9];
  const int tid = threadIdx.x;
  const int el = tid / N3, q = tid % N3;
  const int i = q % N, j = (q / N) % N, k = q / (N * N);
  if (tid < N * N) {
    sB[tid] = a.B[tid];
    sD[tid] = a.D[tid];
  }
  const int64_t e = (int64_t)blockIdx.x * EPB + el;
  const bool valid = e < a.nel;
  const ElemPos ep = elem_pos<P>(valid ? e : 0, a.nx, a.ny, a.mx, a.my, i, j, k);
#pragma unroll
  for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.coords[3 * ep.node + c] : 0.0;
  __syncthreads();
  double J[9];
  sf_forward<double, N>(bufA[el], bufB[el], sB, sD, i, j, k, J);
  if (q == 0)
#pragma unroll
    for (int m = 0; m < 9; ++m) j0q0[el][m] = J[m];
  __syncthreads();
  if (!valid) return;
  const int64_t qi = e * N3 + q;
  if (a.j0out)
#pragma unroll
    for (int m = 0; m < 9; ++m) a.j0out[qi * 9 + m] = J[m];
  const double det = det3(J);
  if (!(det > 0.0)) atomicExch(a.degenerate, 1);
  double inv[9];
  inverse3(J, inv);
  double scale = 0.0, dev = 0.0;
#pragma unroll
  for (int m = 0; m < 9; ++m) {
    scale = fmax(scale, fabs(j0q0[el][m]));
    dev = fmax(dev, fabs(J[m] - j0q0[el][m]));
  }
  if (dev > 1e-11 * scale) atomicExch(a.nonaffine, 1);  // GLL-sweep rounding reaches ~1e-13
#pragma unroll
  for (int m = 0; m < 9; ++m) a.geo[m * a.stride + qi] = inv[m];
  a.geo[9 * a.stride + qi] = det * ((a.qw[i] * a.qw[j]) * a.qw[k]);
  a.geo[10 * a.stride + qi] = det;
}

void launch_geometry(const double* coords, double* geo_q, double* j0_out, int nx, int ny, int nz, int p,
                     const double* B, const double* D, const double* qw, int* nonaffine, int* degenerate,
                     cudaStream_t s) {
  GeoArgs a;
  a.coords = coords;
  a.geo = geo_q;
  a.j0out = j0_out;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.mx = nx * p + 1;
  a.my = ny * p + 1;
  a.nel = (int64_t)nx * ny * nz;
  const int n = p + 1;
  a.stride = a.nel * n * n * n;
  for (int t = 0; t < n * n; ++t) {
    a.B[t] = B[t];
    a.D[t] = D[t];
  }
  for (int t = 0; t < n; ++t) a.qw[t] = qw[t];
  a.nonaffine = nonaffine;
  a.degenerate = degenerate;
  switch (p) {
#define EMF_GEO(PP)                                                                              \
  case PP: {                                                                                     \
    constexpr int EPB = Tile<PP>::EPB, NN = PP + 1;                                              \
    geometry_kernel<PP><<<(unsigned)((a.nel + EPB - 1) / EPB), EPB * NN * NN * NN, 0, s>>>(a); \
  } break;
    EMF_GEO(1)
    EMF_GEO(2)
    EMF_GEO(3)
    EMF_GEO(4)
#undef EMF_GEO
  }
}

// per-qp (11 fields, stride nel*nq3) -> per-element (10 fields, stride nel):
// J0^-1 and det J0 of the element's first qp.
__global__ void geo_compact_kernel(const double* geo_q, double* geo_e, int64_t nel, int nq3) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nel) return;
  const int64_t sq = nel * nq3;
  for (int m = 0; m < 9; ++m) geo_e[m * nel + e] = geo_q[m * sq + e * nq3];
  geo_e[9 * nel + e] = geo_q[10 * sq + e * nq3];
}

void launch_geo_compact(const double* geo_q, double* geo_e, int64_t nel, int nq3, cudaStream_t s) {
  geo_compact_kernel<<<(unsigned)((nel + 255) / 256), 256, 0, s>>>(geo_q, geo_e, nel, nq3);
}

__global__ void cast_d2f_kernel(const double* in, float* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)in[i];
}

void launch_cast_d2f(const double* in, float* out, int64_t n, cudaStream_t s) {
  cast_d2f_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n);
}

}  // namespace emfgpu
