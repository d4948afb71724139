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
                     int periodic_y, cudaStream_t s) {
  GeoArgs a;
  a.coords = coords;
  a.geo = geo_q;
  a.j0out = j0_out;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.mx = nx * p + 1;
  a.my = ny * p + (periodic_y ? 0 : 1);
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

// Per-qp fibre frame field: cylindrical frame about the z axis at the qp's
// reference position (e1 = circumferential, e2 = axial, e3 = radial), the two
// families at +-phi from e1 in the (e1, e2) plane; H_f = h11 m1 m1 + h22 m2 m2 +
// h33 e3 e3 (material.cpp:50-82 with a per-point frame, SURVEY §8(c) gap 2).
// kind 2: the constant frame (e1, e2, e3) given in frame[] (for testing).
struct FrameArgs {
  const double* coords;
  double* hq;   // 12 * nqp (H4, H6), SoA
  double* m1q;  // 6 * nqp (M1_4, M1_6), SoA
  int nx, ny, mx, my, p, kind;
  int64_t nel, nqp;
  double B[81];
  double h11, h22, h33, phi;
  double frame[9];
};

__global__ void fibre_frame_kernel(const FrameArgs a) {
  const int n = a.p + 1, n3 = n * n * n;
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= a.nqp) return;
  const int64_t e = qi / n3;
  const int q = (int)(qi % n3);
  const int qa = q % n, qb = (q / n) % n, qc = q / (n * n);
  const int ei = (int)(e % a.nx), ej = (int)((e / a.nx) % a.ny), ek = (int)(e / ((int64_t)a.nx * a.ny));
  double x[3] = {0, 0, 0};
  for (int c = 0; c < n; ++c)
    for (int b = 0; b < n; ++b)
      for (int aa = 0; aa < n; ++aa) {
        int gb = ej * a.p + b;
        if (gb >= a.my) gb -= a.my;
        const int64_t node = ((int64_t)(ek * a.p + c) * a.my + gb) * a.mx + (ei * a.p + aa);
        const double w = a.B[qa * n + aa] * a.B[qb * n + b] * a.B[qc * n + c];
        for (int d = 0; d < 3; ++d) x[d] += w * a.coords[3 * node + d];
      }
  double e1[3], e2[3], e3[3];
  if (a.kind == 1) {
    const double th = atan2(x[1], x[0]);
    const double cs = cos(th), sn = sin(th);
    e1[0] = -sn; e1[1] = cs; e1[2] = 0.0;
    e2[0] = 0.0; e2[1] = 0.0; e2[2] = 1.0;
    e3[0] = cs; e3[1] = sn; e3[2] = 0.0;
  } else {
    for (int d = 0; d < 3; ++d) {
      e1[d] = a.frame[d];
      e2[d] = a.frame[3 + d];
      e3[d] = a.frame[6 + d];
    }
  }
  const double c = cos(a.phi), s = sin(a.phi);
  double m1[2][3], m2[2][3];
  for (int d = 0; d < 3; ++d) {
    m1[0][d] = c * e1[d] + s * e2[d];
    m2[0][d] = -s * e1[d] + c * e2[d];
    m1[1][d] = c * e1[d] + (-s) * e2[d];
    m2[1][d] = s * e1[d] + c * e2[d];
  }
  for (int f = 0; f < 2; ++f) {
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        const int k = sidx(i, j);
        const double h = a.h11 * (m1[f][i] * m1[f][j]) + a.h22 * (m2[f][i] * m2[f][j]) + a.h33 * (e3[i] * e3[j]);
        a.hq[(6 * f + k) * a.nqp + qi] = h;
      }
    for (int d = 0; d < 3; ++d) a.m1q[(3 * f + d) * a.nqp + qi] = m1[f][d];
  }
}

void launch_fibre_frame(const double* coords, double* hq, double* m1q, int nx, int ny, int nz, int p, int periodic_y,
                        const double* B, double h11, double h22, double h33, double phi, int kind,
                        const double* frame, cudaStream_t s) {
  FrameArgs a;
  a.coords = coords;
  a.hq = hq;
  a.m1q = m1q;
  a.nx = nx;
  a.ny = ny;
  a.mx = nx * p + 1;
  a.my = ny * p + (periodic_y ? 0 : 1);
  a.p = p;
  a.kind = kind;
  a.nel = (int64_t)nx * ny * nz;
  a.nqp = a.nel * (p + 1) * (p + 1) * (p + 1);
  for (int t = 0; t < (p + 1) * (p + 1); ++t) a.B[t] = B[t];
  a.h11 = h11;
  a.h22 = h22;
  a.h33 = h33;
  a.phi = phi;
  for (int t = 0; t < 9; ++t) a.frame[t] = frame ? frame[t] : 0.0;
  fibre_frame_kernel<<<(unsigned)((a.nqp + 255) / 256), 256, 0, s>>>(a);
}

// u_k gathered per element into the element kernels' staging layout: slot
// a + SY b + SZ c of array comp (apply_v2.cuh Lay<N>), padding slots zero.
template <typename T, int N, int SY, int SZ_, int SIZE>
__global__ void uk_elem_kernel(const T* __restrict__ uk, T* __restrict__ out, int64_t nel, int nx, int ny, int mx,
                               int my) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nel * 3 * SIZE) return;
  const int slot = (int)(i % SIZE);
  const int64_t ec = i / SIZE;
  const int comp = (int)(ec % 3);
  const int64_t e = ec / 3;
  const int lc = slot / SZ_, rem = slot - lc * SZ_, lb = rem / SY, la = rem - lb * SY;
  T v = T(0);
  if (la < N && lb < N && lc < N) {
    const int64_t ei = e % nx, ej = (e / nx) % ny, ek = e / ((int64_t)nx * ny);
    int gb = (int)ej * (N - 1) + lb;
    if (gb >= my) gb -= my;  // periodic y lattice
    const int64_t node = ((ek * (N - 1) + lc) * my + gb) * mx + ei * (N - 1) + la;
    v = uk[3 * node + comp];
  }
  out[i] = v;
}
template <typename T>
void launch_uk_elem(const T* uk, T* out, int64_t nel, int nx, int ny, int mx, int my, int size, cudaStream_t s) {
  const int64_t tot = nel * 3 * size;
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  if (size == 82) uk_elem_kernel<T, 4, 4, 20, 82><<<blocks, 256, 0, s>>>(uk, out, nel, nx, ny, mx, my);
  else uk_elem_kernel<T, 4, 4, 20, 80><<<blocks, 256, 0, s>>>(uk, out, nel, nx, ny, mx, my);
}
template void launch_uk_elem<double>(const double*, double*, int64_t, int, int, int, int, int, cudaStream_t);
template void launch_uk_elem<float>(const float*, float*, int64_t, int, int, int, int, int, cudaStream_t);

__global__ void cast_d2f_kernel(const double* in, float* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)in[i];
}

void launch_cast_d2f(const double* in, float* out, int64_t n, cudaStream_t s) {
  cast_d2f_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n);
}

}  // namespace emfgpu
