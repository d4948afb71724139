// Element-batched, sum-factorized tangent kernels for sm_100a.
//
// Mapping (B200-first): one CUDA thread per quadrature
// point, EPB elements per CTA, the whole element pipeline fused in one
// kernel: lattice gather of the DoF vector -> 8 forward sweeps per component
// through shared memory -> per-qp material kernel in registers -> 8 merged
// transposed sweeps -> element-local result written to an L2-resident buffer.
// A separate node-centric kernel (gather.cu) sums the element contributions
// of every lattice node in the reference's colour order, which makes fp64
// results deterministic and equal-order to the reference's 8-colour scatter
// (operator.hpp:145-153, 439).
//
// Reference correspondence:
//   gather / scatter        operator.hpp:237-276 (DoF = 3*node+c)
//   gradient_at_qpoints     sumfact.hpp:67-85
//   scatter_gradient_...    sumfact.hpp:90-110 (merged: Dx*Q0 + Bx*(Dy A1 + By A2))
//   element_tangent_batch   operator.hpp:468-530
//   update_linearization    operator.hpp:643-770
//   compute_diagonal        operator.hpp:772-878 (as a per-qp 3x3 quadratic form,
//                           not 3(p+1)^3 local unit applies)
#pragma once
#include <atomic>
#include "qp.cuh"

namespace emfgpu {

// elements per CTA for degree P (threads = EPB * (P+1)^3)
template <int P>
struct Tile;
template <>
struct Tile<1> { static constexpr int EPB = 16; };
template <>
struct Tile<2> { static constexpr int EPB = 4; };
template <>
struct Tile<3> { static constexpr int EPB = 2; };
template <>
struct Tile<4> { static constexpr int EPB = 1; };

// cache field slots (SoA, field f at cache + f*stride), per strategy
enum CacheSlot : int {
  // scalar/tensor: scalars first
  C_LNJ = 0, C_JP = 1, C_C1 = 2, C_C2 = 3, C_C3 = 4, C_EF = 6,
  // tensor: then F, Finv, S, Cinv
  C_F = 8, C_FINV = 17, C_S = 26, C_CINV = 32, C_NT = 38,
  // tensor, cNH / iNH in the material domain: the push-forward state instead
  // (qp.cuh PushState: K = J0^-1 F^-1 (9), b (6), 4 coefficients with det J0 w
  // folded in) -- 19 fields and no geometry read in the apply, against 33 + 10
  // (fibre: + 2 x (A_f = F H_f F^T (6), k_s, k_c) = 35, against 37 + 10 + the 12
  // per-point structure-tensor entries)
  C_PK = 0, C_PB = 9, C_PC = 15, C_NTP = 19, C_NTPF = 35,
  // cachedF: displacement gradient G = F - I
  C_G = 0, C_NG = 9,
  // spatial formulation (operator.hpp:139-143): scalars as above, then 1/J,
  // J_t (9; all strategies), tau, b, F H4 F^T, F H6 F^T (tensor)
  C_INVJ = 8, C_JT = 9, C_TAU = 18, C_B = 24, C_FH = 30, C_NSP = 42
};

#ifndef EMF_TENSOR_PUSH
#define EMF_TENSOR_PUSH 1
#endif
// Does strategy tensor cache the push-forward state for this (model, domain)?
#ifndef EMF_TENSOR_PUSH_FIBER
#define EMF_TENSOR_PUSH_FIBER 1
#endif
__host__ __device__ constexpr bool tensor_compact(int model, int spatial) {
  return EMF_TENSOR_PUSH && (model != 2 /* FIBER */ || EMF_TENSOR_PUSH_FIBER) && !spatial;
}
__host__ __device__ constexpr int tensor_compact_fields(int model) { return model == 2 ? 35 : 19; }

// n / d for 0 <= n < 2^31 with a precomputed multiplier (round-up method,
// Hacker's Delight 10-9): q = (umulhi(n, m) + n) >> l.
struct FastDiv {
  uint32_t d, m;
  int l;
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    return (__umulhi(n, m) + n) >> l;
#else
    return (uint32_t)((((uint64_t)n * m) >> 32) + n) >> l;
#endif
  }
  static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.l = 0;
    while ((1ull << f.l) < d) ++f.l;
    f.m = (uint32_t)(((1ull << 32) * ((1ull << f.l) - d)) / d + 1);
    return f;
  }
};

// Per-device launch-shape cache (SM count x resident CTAs per SM), computed on
// the first launch on each device by `init` (which may also set the kernel's
// function attributes on that device); safe for concurrent host threads (the
// computation is idempotent, the store atomic).
template <typename Init>
inline void per_device_shape(std::atomic<int>* cache, int& sms, int& per_sm, Init&& init) {
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load(std::memory_order_acquire);
  if (v == 0) {
    int s = 0, p = 0;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    init(p);
    if (p < 1) p = 1;
    v = s * 64 + p;
    cache[dev & 63].store(v, std::memory_order_release);
  }
  sms = v / 64;
  per_sm = v % 64;
}

// Layout of the element-local results (element phase -> node phase):
// element-major loc[(e*3 + c)*N^3 + m] (each element writes one contiguous
// 3 N^3 block).  EMF_LOC_ROWS=1 builds the row layout
// loc[((((row*N + lz)*N + ly)*3 + c)*nx + ei)*N + lx], row = ek*ny + ej, in
// which the node phase streams whole lattice rows: measured on cfg2 fp64 none
// (profiles/r02_loc_layout.txt) the node phase 0.31 -> 0.25 ms but the element
// kernel 2.20 -> 2.57 ms (its stores scatter into 40-byte pieces), so the
// element-major layout stays.
#ifndef EMF_LOC_ROWS
#define EMF_LOC_ROWS 0
#endif
template <int N>
__host__ __device__ __forceinline__ int64_t loc_index(int64_t row, int ei, int nx, int lz, int ly, int lx, int c) {
  if (EMF_LOC_ROWS) return ((((row * N + lz) * N + ly) * 3 + c) * (int64_t)nx + ei) * N + lx;
  return ((row * nx + ei) * 3 + c) * (N * N * N) + (lz * N + ly) * N + lx;
}
// stride between the components of one value
template <int N>
__host__ __device__ __forceinline__ int64_t loc_cstride(int nx) {
  return EMF_LOC_ROWS ? (int64_t)nx * N : (int64_t)N * N * N;
}

template <typename T>
struct KArgs {
  const T* x;          // input vector (3 per node), apply / unused by diag
  T* loc;              // element-local output, component-major (e*3 + c)*nn3 + m
  const T* uk;         // linearization point in T (none/scalar), 3 per node
  const double* ukd;   // linearization point in double (linearize only)
  const T* geo;        // J0^-1 (9) + detw (1), SoA with stride geo_stride
  const double* geod;  // same, double (linearize)
  int64_t geo_stride;
  int affine;          // geometry per element instead of per qp
  int cartesian;       // affine with diagonal J0 in every element (axis-aligned boxes)
  T* cache;            // SoA fields
  int64_t cache_stride;
  int strategy;        // runtime strategy for linearize/diagonal
  int nx, ny, nz, mx, my, mz;
  int64_t nel;
  int64_t e_begin;     // first element of the processed range (boundary/interior split)
  int faces;           // Dirichlet faces bit mask (-x,+x,-y,+y,-z,+z)
  unsigned long long* err;  // first failing e*nq3+q (atomicMin)
  MatConst<T> mat;
  MatConst<double> matd;
  T Bm[25], Dm[25];    // 1D tables, row = quadrature point (P <= 4)
  double Bd[25], Dd[25];
  T eoB[13], eoD[12];  // even-odd halves of B and of the collocated derivative Dc (eo_sweeps.cuh)
  float2 eoP[20];      // the same entries as pairs for the packed f32x2 sweeps (EoT, eo_sweeps.cuh)
  double qwd[9];  // 1D Gauss weights (affine geometry stores det J0 without them)
  FastDiv fd_nx, fd_nxy;
  // optional per-qp fibre frame field (fibre model): 18 SoA fields H4 (6),
  // H6 (6), M1_4 (3), M1_6 (3) with stride hq_stride, in Number (hq) and in
  // double (hqd; m1qd = hqd + 12*stride) for linearization
  const T* hq;
  const double* hqd;
  const double* m1qd;
  int64_t hq_stride;
  int spatial;           // Formulation::domain == spatial (linearize / diagonal / residual)
  const double* coords;  // node coordinates (spatial linearization: J_t = J0 + Grad_xi u_k)
  unsigned* tk;          // apply_v2 ticket counter slot: [0] next ticket, [1] workers done
  const T* uk_el;        // Q3: u_k per element in the staging layout [e][3][SIZE] (null: lattice gather)
};

// Stored scalars of the scalar/tensor strategies (load_scalar_fields,
// operator.hpp:327-343).
template <typename T, int MODEL>
__device__ __forceinline__ void load_scalars(const T* cs, int64_t st, int64_t qidx, Bundle<T>& cb) {
  if (MODEL == CNH) cb.lnj = cs[C_LNJ * st + qidx];
  else {
    cb.jp = cs[C_JP * st + qidx];
    cb.c1 = cs[C_C1 * st + qidx];
    cb.c2 = cs[C_C2 * st + qidx];
  }
  if (MODEL == FIBER) {
    cb.c3[0] = cs[(C_C3 + 0) * st + qidx];
    cb.c3[1] = cs[(C_C3 + 1) * st + qidx];
    cb.efib[0] = cs[(C_EF + 0) * st + qidx];
    cb.efib[1] = cs[(C_EF + 1) * st + qidx];
  }
}

// Spatial linearization bundle at one point (qp_cache_for_apply spatial cell,
// operator.hpp:393-434): strat S_NONE recomputes from gg = Grad u_k, S_SCALAR
// loads the scalars and rebuilds b, tau, F H F^T from gg, S_TENSOR loads all.
// Returns false when det(F) <= 0.
template <typename T, int MODEL>
__device__ __forceinline__ bool spatial_bundle(int strat, const MatConst<T>& mq, const T* gg, const T* cs, int64_t st,
                                               int64_t qidx, Bundle<T>& cb, SpCell<T>& sp) {
  if (strat == S_TENSOR) {
    load_scalars<T, MODEL>(cs, st, qidx, cb);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      sp.tau[k] = cs[(C_TAU + k) * st + qidx];
      if (MODEL != CNH) sp.b[k] = cs[(C_B + k) * st + qidx];
      if (MODEL == FIBER) {
        sp.fh[0][k] = cs[(C_FH + k) * st + qidx];
        sp.fh[1][k] = cs[(C_FH + 6 + k) * st + qidx];
      }
    }
    return true;
  }
  const bool ok = make_strain(gg, cb);
  T bt[6];
  green_euler(gg, bt);
  if (strat == S_NONE) cache_scalars<T, MODEL>(mq, cb);
  else load_scalars<T, MODEL>(cs, st, qidx, cb);
  spatial_cell<T, MODEL>(mq, cb, bt, sp);
  return ok;
}

// J_t^-1 and (1/J) det J_t w_q at one point from the spatial cache.
template <typename T>
__device__ __forceinline__ void spatial_geo(const T* cs, int64_t st, int64_t qidx, T wq, T* jtinv, T& s) {
  T jt[9];
#pragma unroll
  for (int m = 0; m < 9; ++m) jt[m] = cs[(C_JT + m) * st + qidx];
  inverse3(jt, jtinv);
  s = (cs[C_INVJ * st + qidx] * det3(jt)) * wq;
}

// Material constants at one quadrature point: the operator's constants, with
// the fibre structure tensors replaced by the per-qp frame field if present.
template <typename T, int MODEL>
__device__ __forceinline__ MatConst<T> mat_at(const MatConst<T>& m, const T* hq, int64_t st, int64_t qidx) {
  MatConst<T> r = m;
  if (MODEL == FIBER && hq != nullptr) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
#pragma unroll
      for (int k = 0; k < 6; ++k) r.h[f][k] = hq[(6 * f + k) * st + qidx];
#pragma unroll
      for (int k = 0; k < 3; ++k) r.m1[f][k] = hq[(12 + 3 * f + k) * st + qidx];  // dead for tensor/scalar
    }
  }
  return r;
}
__device__ __forceinline__ MatConst<double> matd_at(const MatConst<double>& m, const double* hq, const double* m1q,
                                                    int64_t st, int64_t qidx) {
  MatConst<double> r = m;
  if (hq != nullptr) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
#pragma unroll
      for (int k = 0; k < 6; ++k) r.h[f][k] = hq[(6 * f + k) * st + qidx];
#pragma unroll
      for (int k = 0; k < 3; ++k) r.m1[f][k] = m1q[(3 * f + k) * st + qidx];
    }
  }
  return r;
}

__device__ __forceinline__ bool node_constrained(int a, int b, int c, int mx, int my, int mz, int faces) {
  return ((faces & 1) && a == 0) || ((faces & 2) && a == mx - 1) || ((faces & 4) && b == 0) ||
         ((faces & 8) && b == my - 1) || ((faces & 16) && c == 0) || ((faces & 32) && c == mz - 1);
}

// ---- sum factorization on one element's shared arrays -----------------------
// A, Bf: 9 arrays of N^3 each (per element). Thread owns point (i,j,k).

// Forward: input field in A[0..2] (3 components, lexicographic a fastest),
// output reference gradient g[c][d] = d u_c / d xi_d at qp (i,j,k).
template <typename T, int N>
__device__ __forceinline__ void sf_forward(T (*A)[N * N * N], T (*Bf)[N * N * N], const T* sB, const T* sD, int i,
                                           int j, int k, T* g) {
  constexpr int N2 = N * N;
  const int pt = (k * N + j) * N + i;
  // S1: x-sweep with B and D
  {
    T tb[3], td[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) tb[c] = td[c] = T(0);
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const T b = sB[i * N + a], d = sD[i * N + a];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T u = A[c][k * N2 + j * N + a];
        tb[c] += b * u;
        td[c] += d * u;
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Bf[c][pt] = tb[c];
      Bf[3 + c][pt] = td[c];
    }
  }
  __syncthreads();
  // S2: y-sweep: sBB = By tB, sBD = Dy tB, sDB = By tD
  {
    T bb[3], bd[3], db[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) bb[c] = bd[c] = db[c] = T(0);
#pragma unroll
    for (int b = 0; b < N; ++b) {
      const T vb = sB[j * N + b], vd = sD[j * N + b];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T tb = Bf[c][k * N2 + b * N + i], td = Bf[3 + c][k * N2 + b * N + i];
        bb[c] += vb * tb;
        bd[c] += vd * tb;
        db[c] += vb * td;
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[c][pt] = bb[c];
      A[3 + c][pt] = bd[c];
      A[6 + c][pt] = db[c];
    }
  }
  __syncthreads();
  // S3: z-sweep: g0 = Bz sDB, g1 = Bz sBD, g2 = Dz sBB
  {
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = T(0);
#pragma unroll
    for (int cc = 0; cc < N; ++cc) {
      const T vb = sB[k * N + cc], vd = sD[k * N + cc];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int o = cc * N2 + j * N + i;
        g[3 * c + 0] += vb * A[6 + c][o];
        g[3 * c + 1] += vb * A[3 + c][o];
        g[3 * c + 2] += vd * A[c][o];
      }
    }
  }
  __syncthreads();
}

// Transposed: w(c,d) at qp (i,j,k) -> nodal out[c] at node (i,j,k):
// out = sum_q grad_xi phi_node(q) . w(c,:)(q)  (sumfact.hpp:90-110)
template <typename T, int N>
__device__ __forceinline__ void sf_transpose(T (*A)[N * N * N], T (*Bf)[N * N * N], const T* sB, const T* sD, int i,
                                             int j, int k, const T* w, T* out) {
  constexpr int N2 = N * N;
  const int pt = (k * N + j) * N + i;
#pragma unroll
  for (int q = 0; q < 9; ++q) A[q][pt] = w[q];
  __syncthreads();
  // T1 (z): A0 = Bz^T w0, A1 = Bz^T w1, A2 = Dz^T w2   (node index k)
  {
    T a0[3], a1[3], a2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) a0[c] = a1[c] = a2[c] = T(0);
#pragma unroll
    for (int qc = 0; qc < N; ++qc) {
      const T vb = sB[qc * N + k], vd = sD[qc * N + k];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int o = qc * N2 + j * N + i;
        a0[c] += vb * A[3 * c + 0][o];
        a1[c] += vb * A[3 * c + 1][o];
        a2[c] += vd * A[3 * c + 2][o];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Bf[3 * c + 0][pt] = a0[c];
      Bf[3 * c + 1][pt] = a1[c];
      Bf[3 * c + 2][pt] = a2[c];
    }
  }
  __syncthreads();
  // T2 (y): Q0 = By^T A0, Q12 = Dy^T A1 + By^T A2   (node index j)
  {
    T q0[3], q12[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) q0[c] = q12[c] = T(0);
#pragma unroll
    for (int qb = 0; qb < N; ++qb) {
      const T vb = sB[qb * N + j], vd = sD[qb * N + j];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int o = k * N2 + qb * N + i;
        q0[c] += vb * Bf[3 * c + 0][o];
        q12[c] += vd * Bf[3 * c + 1][o] + vb * Bf[3 * c + 2][o];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[2 * c][pt] = q0[c];
      A[2 * c + 1][pt] = q12[c];
    }
  }
  __syncthreads();
  // T3 (x): out = Dx^T Q0 + Bx^T Q12   (node index i)
  {
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = T(0);
#pragma unroll
    for (int qa = 0; qa < N; ++qa) {
      const T vb = sB[qa * N + i], vd = sD[qa * N + i];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int o = k * N2 + j * N + qa;
        out[c] += vd * A[2 * c][o] + vb * A[2 * c + 1][o];
      }
    }
  }
  __syncthreads();
}

// ---- element addressing -------------------------------------------------------
struct ElemPos {
  int64_t e;
  int ei, ej, ek;
  int64_t node;  // global node of this thread's local node (i,j,k)
  int ga, gb, gc;
};

template <int P>
__device__ __forceinline__ ElemPos elem_pos(int64_t e, int nx, int ny, int mx, int my, int i, int j, int k) {
  ElemPos r;
  r.e = e;
  r.ei = (int)(e % nx);
  r.ej = (int)((e / nx) % ny);
  r.ek = (int)(e / ((int64_t)nx * ny));
  r.ga = r.ei * P + i;
  r.gb = r.ej * P + j;
  if (r.gb >= my) r.gb -= my;  // periodic y lattice (my = ny*P); never taken otherwise
  r.gc = r.ek * P + k;
  r.node = ((int64_t)r.gc * my + r.gb) * mx + r.ga;
  return r;
}

// Geometry factors at (e, q): J0^-1 and det(J0)*w_q (operator.hpp:492, 496-504).
// Curved meshes store both per qp; affine meshes store them per element and
// apply the tensor-product weight here (SURVEY §8(d) affine shortcut).
template <typename T, typename A>
__device__ __forceinline__ void load_geo(const A& a, const T* geo, bool valid, int64_t e, int64_t qidx, int i, int j,
                                         int k, T* j0inv, T& detw) {
  const int64_t gidx = valid ? (a.affine ? e : qidx) : 0;
  const int64_t stride = a.geo_stride;
#pragma unroll
  for (int m = 0; m < 9; ++m) j0inv[m] = geo[m * stride + gidx];
  detw = geo[9 * stride + gidx];
  if (a.affine) detw = detw * T(a.qwd[i] * a.qwd[j] * a.qwd[k]);
}

// The apply kernel itself is apply_v2.cuh:apply_v2_kernel.

// ---- linearization kernel (double compute, T store), operator.hpp:643-770 ------
template <typename T, int P, int MODEL>
__global__ void __launch_bounds__(Tile<P>::EPB*(P + 1) * (P + 1) * (P + 1))
    linearize_kernel(const KArgs<T> a) {
  constexpr int N = P + 1, N3 = N * N * N, EPB = Tile<P>::EPB;
  __shared__ double sB[N * N], sD[N * N];
  __shared__ double bufA[EPB][9][N3], bufB[EPB][9][N3];
  const int tid = threadIdx.x;
  const int el = tid / N3, q = tid % N3;
  const int i = q % N, j = (q / N) % N, k = q / (N * N);
  if (tid < N * N) {
    sB[tid] = a.Bd[tid];
    sD[tid] = a.Dd[tid];
  }
  const int64_t e = (int64_t)blockIdx.x * EPB + el + a.e_begin;
  const bool valid = e < a.nel;
  const ElemPos ep = elem_pos<P>(valid ? e : a.e_begin, a.nx, a.ny, a.mx, a.my, i, j, k);
#pragma unroll
  for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.ukd[3 * ep.node + c] : 0.0;
  __syncthreads();
  double gk[9], j0[9];
  sf_forward<double, N>(bufA[el], bufB[el], sB, sD, i, j, k, gk);
  if (a.spatial) {  // J0 by the geometry kernel's isoparametric sweep (mesh.cpp:162-186)
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.coords[3 * ep.node + c] : 0.0;
    __syncthreads();
    sf_forward<double, N>(bufA[el], bufB[el], sB, sD, i, j, k, j0);
  }
  if (!valid) return;
  const int64_t qidx = e * N3 + q;
  double j0inv[9], detw, g[9];
  load_geo(a, a.geod, true, e, qidx, i, j, k, j0inv, detw);
  mm(gk, j0inv, g);
  const int64_t st = a.cache_stride;
  if (a.strategy == S_CACHEDF) {
#pragma unroll
    for (int m = 0; m < 9; ++m) a.cache[(C_G + m) * st + qidx] = T(g[m]);
  }
  const MatConst<double> md = matd_at(a.matd, a.hqd, a.m1qd, a.hq_stride, qidx);
  Bundle<double> cb;
  if (!make_strain(g, cb)) {
    atomicMin(a.err, (unsigned long long)qidx);
    return;
  }
  if (a.spatial) {
    // 1/J and J_t = J0 + Grad_xi u_k with det J_t > 0 (operator.hpp:736-744)
    double jt[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) jt[m] = j0[m] + gk[m];
    if (!(det3(jt) > 0.0)) {
      atomicMin(a.err, (unsigned long long)qidx);
      return;
    }
    a.cache[C_INVJ * st + qidx] = T(1.0 / (1.0 + cb.jm1));
#pragma unroll
    for (int m = 0; m < 9; ++m) a.cache[(C_JT + m) * st + qidx] = T(jt[m]);
  }
  if (a.strategy == S_CACHEDF || a.strategy == S_NONE) return;
  if (a.strategy == S_TENSOR && tensor_compact(MODEL, 0) && !a.spatial) {
    // the linearization state in its push-forward form, computed in double
    PushState<double> ps;
    push_state<double, MODEL, false, false>(md, g, j0inv, detw, cb, ps);
    store_push_state<T>(a.cache, st, qidx, ps);
    if constexpr (MODEL == FIBER) {
      cache_scalars<double, MODEL>(md, cb);
      push_state_fibre<double>(md, cb, detw, ps);
      store_push_state_fibre<T>(a.cache, st, qidx, ps);
    }
    return;
  }
  // stored scalars, computed in double (operator.hpp:720-735)
  cache_scalars<double, MODEL>(md, cb);
  if (MODEL == CNH) {
    a.cache[C_LNJ * st + qidx] = T(cb.lnj);
  } else {
    a.cache[C_JP * st + qidx] = T(cb.jp);
    a.cache[C_C1 * st + qidx] = T(cb.c1);
    a.cache[C_C2 * st + qidx] = T(cb.c2);
  }
  if (MODEL == FIBER) {
    a.cache[(C_C3 + 0) * st + qidx] = T(cb.c3[0]);
    a.cache[(C_C3 + 1) * st + qidx] = T(cb.c3[1]);
    a.cache[(C_EF + 0) * st + qidx] = T(cb.efib[0]);
    a.cache[(C_EF + 1) * st + qidx] = T(cb.efib[1]);
  }
  if (a.strategy != S_TENSOR) return;
  if (a.spatial) {  // tau, b, F H_i F^T (operator.hpp:756-765)
    double bt[6];
    green_euler(g, bt);
    SpCell<double> sp;
    spatial_cell<double, MODEL>(md, cb, bt, sp);
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      a.cache[(C_TAU + m) * st + qidx] = T(sp.tau[m]);
      if (MODEL != CNH) a.cache[(C_B + m) * st + qidx] = T(sp.b[m]);
      if (MODEL == FIBER) {
        a.cache[(C_FH + m) * st + qidx] = T(sp.fh[0][m]);
        a.cache[(C_FH + 6 + m) * st + qidx] = T(sp.fh[1][m]);
      }
    }
    return;
  }
  second_pk<double, MODEL>(md, cb);
#pragma unroll
  for (int m = 0; m < 9; ++m) {
    a.cache[(C_F + m) * st + qidx] = T(cb.F[m]);
    a.cache[(C_FINV + m) * st + qidx] = T(cb.Finv[m]);
  }
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    a.cache[(C_S + m) * st + qidx] = T(cb.S[m]);
    a.cache[(C_CINV + m) * st + qidx] = T(cb.Cinv[m]);
  }
}

// ---- diagonal kernel ----------------------------------------------------------------
// diag(m=(a,b,c), comp) = sum_q sum_{d,d'} A^comp_{dd'}(q) dphi_m/dxi_d(q) dphi_m/dxi_d'(q)
// with A^comp_{dd'} = d w_ref(comp,d) / d Gref(comp,d'), obtained from 9 unit
// evaluations of the (linear) qp tangent; the quadratic form is contracted
// by transposed sweeps with the elementwise products BB, BD, DD of the 1D
// tables.  Same operator entries as the reference's 3(p+1)^3 local unit
// applications (operator.hpp:824-866).
template <typename T, int P, int MODEL>
__global__ void __launch_bounds__(Tile<P>::EPB*(P + 1) * (P + 1) * (P + 1))
    diagonal_kernel(const KArgs<T> a) {
  constexpr int N = P + 1, N3 = N * N * N, N2 = N * N, EPB = Tile<P>::EPB;
  __shared__ T sB[N * N], sD[N * N];
  __shared__ T bufA[EPB][9][N3], bufB[EPB][9][N3];
  const int tid = threadIdx.x;
  const int el = tid / N3, q = tid % N3;
  const int i = q % N, j = (q / N) % N, k = q / (N * N);
  if (tid < N * N) {
    sB[tid] = a.Bm[tid];
    sD[tid] = a.Dm[tid];
  }
  const int64_t e = (int64_t)blockIdx.x * EPB + el + a.e_begin;
  const bool valid = e < a.nel;
  const ElemPos ep = elem_pos<P>(valid ? e : a.e_begin, a.nx, a.ny, a.mx, a.my, i, j, k);
  const int64_t qidx = e * N3 + q;
  const int64_t st = a.cache_stride, ix = valid ? qidx : 0;
  const T* cs = a.cache;
  const MatConst<T> mq = mat_at<T, MODEL>(a.mat, a.hq, a.hq_stride, ix);
  Bundle<T> cb;
  PushState<T> ps;
  T j0inv[9], detw;
  load_geo(a, a.geo, valid, e, qidx, i, j, k, j0inv, detw);
  SpCell<T> sp;
  T jtinv[9], ssc = T(0);
  if (a.spatial) {
    T g[9];
    if (a.strategy == S_NONE || a.strategy == S_SCALAR) {
#pragma unroll
      for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.uk[3 * ep.node + c] : T(0);
      __syncthreads();
      T gk[9];
      sf_forward<T, N>(bufA[el], bufB[el], sB, sD, i, j, k, gk);
      mm(gk, j0inv, g);
    }
    spatial_geo(cs, st, ix, T(a.qwd[i] * a.qwd[j] * a.qwd[k]), jtinv, ssc);
    spatial_bundle<T, MODEL>(a.strategy, mq, g, cs, st, ix, cb, sp);
  } else if (a.strategy == S_NONE || a.strategy == S_SCALAR) {
#pragma unroll
    for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.uk[3 * ep.node + c] : T(0);
    __syncthreads();
    T gk[9], g[9];
    sf_forward<T, N>(bufA[el], bufB[el], sB, sD, i, j, k, gk);
    mm(gk, j0inv, g);
    make_strain(g, cb);
    if (a.strategy == S_NONE) cache_scalars<T, MODEL>(mq, cb);
  } else if (a.strategy == S_CACHEDF) {
    T g[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) g[m] = cs[(C_G + m) * st + ix];
    make_strain(g, cb);
    cache_scalars<T, MODEL>(mq, cb);
  } else if (tensor_compact(MODEL, 0)) {
    load_push_state<T>(cs, st, ix, ps);
    if constexpr (MODEL == FIBER) load_push_state_fibre<T>(cs, st, ix, ps);
  } else {
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      cb.F[m] = cs[(C_F + m) * st + ix];
      cb.Finv[m] = cs[(C_FINV + m) * st + ix];
    }
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      cb.S[m] = cs[(C_S + m) * st + ix];
      cb.Cinv[m] = cs[(C_CINV + m) * st + ix];
    }
  }
  const bool compact = !a.spatial && a.strategy == S_TENSOR && tensor_compact(MODEL, 0);
  if (!a.spatial && !compact) {
    if (a.strategy == S_SCALAR || a.strategy == S_TENSOR) load_scalars<T, MODEL>(cs, st, ix, cb);
    if (a.strategy != S_TENSOR) second_pk<T, MODEL>(mq, cb);
  }

  // A^c_{dd'}: 27 values per qp, as symmetric quadratic-form coefficients
  // coef[c][pair], pairs (00,11,22,01,02,12) with off-diagonals A_dd'+A_d'd.
  T coef[3][6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    T A[3][3];
#pragma unroll
    for (int dp = 0; dp < 3; ++dp) {
      T gref[9], w[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) gref[m] = T(0);
      gref[3 * c + dp] = T(1);
      if (a.spatial)
        spatial_integrand<T, MODEL>(mq, cb, sp, gref, jtinv, ssc, w);
      else if (compact)
        push_integrand<T, MODEL>(ps, gref, w);
      else
        tangent_integrand<T, MODEL>(mq, cb, gref, j0inv, detw, w);
#pragma unroll
      for (int d = 0; d < 3; ++d) A[d][dp] = w[3 * c + d];
    }
    coef[c][0] = A[0][0];
    coef[c][1] = A[1][1];
    coef[c][2] = A[2][2];
    coef[c][3] = A[0][1] + A[1][0];
    coef[c][4] = A[0][2] + A[2][0];
    coef[c][5] = A[1][2] + A[2][1];
  }
  if (!valid) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int s = 0; s < 6; ++s) coef[c][s] = T(0);
  }
  // factor per axis for pair (d,d'): axis x gets D*D if d=d'=0, B*D if one of
  // them is 0, else B*B; same for y (index 1) and z (index 2).
  T out[3] = {T(0), T(0), T(0)};
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int d0 = s < 3 ? s : (s == 5 ? 1 : 0);
    const int d1 = s < 3 ? s : (s == 3 ? 1 : 2);
#pragma unroll
    for (int c = 0; c < 3; ++c) bufA[el][c][q] = coef[c][s];
    __syncthreads();
    // z (node index k)
    T t[3] = {T(0), T(0), T(0)};
    const int nz_ = (d0 == 2) + (d1 == 2);
    const int ny_ = (d0 == 1) + (d1 == 1);
    const int nx_ = (d0 == 0) + (d1 == 0);
#pragma unroll
    for (int qc = 0; qc < N; ++qc) {
      const T b = sB[qc * N + k], d = sD[qc * N + k];
      const T f = nz_ == 2 ? d * d : (nz_ == 1 ? b * d : b * b);
#pragma unroll
      for (int c = 0; c < 3; ++c) t[c] += f * bufA[el][c][qc * N2 + j * N + i];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) bufB[el][c][q] = t[c];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c) t[c] = T(0);
#pragma unroll
    for (int qb = 0; qb < N; ++qb) {
      const T b = sB[qb * N + j], d = sD[qb * N + j];
      const T f = ny_ == 2 ? d * d : (ny_ == 1 ? b * d : b * b);
#pragma unroll
      for (int c = 0; c < 3; ++c) t[c] += f * bufB[el][c][k * N2 + qb * N + i];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) bufA[el][3 + c][q] = t[c];
    __syncthreads();
#pragma unroll
    for (int qa = 0; qa < N; ++qa) {
      const T b = sB[qa * N + i], d = sD[qa * N + i];
      const T f = nx_ == 2 ? d * d : (nx_ == 1 ? b * d : b * b);
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] += f * bufA[el][3 + c][k * N2 + j * N + qa];
    }
    __syncthreads();
  }
  if (valid) {
    int64_t o = e * 3 * N3 + q;
    if constexpr (EMF_LOC_ROWS) {
      const int64_t row = a.fd_nx.div((uint32_t)e);
      o = loc_index<N>(row, (int)(e - row * a.nx), a.nx, q / (N * N), (q / N) % N, q % N, 0);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) a.loc[o + c * loc_cstride<N>(a.nx)] = out[c];
  }
}

}  // namespace emfgpu

namespace emfgpu {

// Residual integrand at one point (element_residual_batch, operator.hpp:550-590):
// gref = Grad_xi u, full J0^-1, detw = det J0 w_q, wq3 = w_q.  Material domain:
// w = detw F S J0^-T; spatial: w = (1/J) det J_t w_q tau J_t^-T with J_t = J0 +
// Grad_xi u.  Returns false when det(F) <= 0.
template <typename T, int MODEL, bool SPATIAL>
__device__ __forceinline__ bool resid_integrand(const MatConst<T>& mq, const T* gref, const T* j0inv, T detw, T wq3,
                                                T* w) {
  T g[9];
  mm(gref, j0inv, g);
  Bundle<T> cb;
  const bool ok = make_strain(g, cb);
  cache_scalars<T, MODEL>(mq, cb);  // lnJ (cNH), J^-2/3, fibre invariants (operator.hpp:557-566)
  if constexpr (SPATIAL) {
    // J0 recovered from the stored J0^-1 (operator.hpp:572-588)
    T j0[9], jt[9], jtinv[9], bt[6], tf[9];
    inverse3(j0inv, j0);
#pragma unroll
    for (int m = 0; m < 9; ++m) jt[m] = j0[m] + gref[m];
    inverse3(jt, jtinv);
    const T detjt = det3(jt);
    const T invj = T(1) / (T(1) + cb.jm1);
    green_euler(g, bt);
    SpCell<T> sp;
    spatial_cell<T, MODEL>(mq, cb, bt, sp);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) tf[3 * r + c] = sp.tau[sidx(r, c)];
    mm_bt(tf, jtinv, w);
    const T sc = (invj * detjt) * wq3;
#pragma unroll
    for (int m = 0; m < 9; ++m) w[m] *= sc;
  } else {
    second_pk<T, MODEL>(mq, cb);
    T fs[9];
    mm_ts(cb.F, cb.S, fs);  // w_mat = F S (operator.hpp:568)
    mm_bt(fs, j0inv, w);
#pragma unroll
    for (int m = 0; m < 9; ++m) w[m] *= detw;
  }
  return ok;
}

// ---- residual kernel: r_e = (Grad_xi test, det J0 w_q F S J0^-T) -----------
// element_residual_batch, operator.hpp:532-595 (material domain), thread per
// qp, shared-memory sweeps.  Not the hot path: one launch per Newton step.
template <typename T, int P, int MODEL>
__global__ void __launch_bounds__(Tile<P>::EPB*(P + 1) * (P + 1) * (P + 1))
    residual_kernel(const KArgs<T> a) {
  constexpr int N = P + 1, N3 = N * N * N, EPB = Tile<P>::EPB;
  __shared__ T sB[N * N], sD[N * N];
  __shared__ T bufA[EPB][9][N3], bufB[EPB][9][N3];
  const int tid = threadIdx.x;
  const int el = tid / N3, q = tid % N3;
  const int i = q % N, j = (q / N) % N, k = q / (N * N);
  if (tid < N * N) {
    sB[tid] = a.Bm[tid];
    sD[tid] = a.Dm[tid];
  }
  const int64_t e = (int64_t)blockIdx.x * EPB + el;
  const bool valid = e < a.nel;
  const ElemPos ep = elem_pos<P>(valid ? e : 0, a.nx, a.ny, a.mx, a.my, i, j, k);
#pragma unroll
  for (int c = 0; c < 3; ++c) bufA[el][c][q] = valid ? a.x[3 * ep.node + c] : T(0);
  __syncthreads();
  T gref[9];
  sf_forward<T, N>(bufA[el], bufB[el], sB, sD, i, j, k, gref);
  const int64_t qidx = (valid ? e : 0) * N3 + q;
  T j0inv[9], detw;
  load_geo(a, a.geo, valid, e, qidx, i, j, k, j0inv, detw);
  const MatConst<T> mq = mat_at<T, MODEL>(a.mat, a.hq, a.hq_stride, qidx);
  T w[9], out[3];
  const T wq3 = T(a.qwd[i] * a.qwd[j] * a.qwd[k]);
  const bool ok = a.spatial ? resid_integrand<T, MODEL, true>(mq, gref, j0inv, detw, wq3, w)
                            : resid_integrand<T, MODEL, false>(mq, gref, j0inv, detw, wq3, w);
  if (!ok && valid) atomicMin(a.err, (unsigned long long)qidx);
  sf_transpose<T, N>(bufA[el], bufB[el], sB, sD, i, j, k, w, out);
  if (valid) {
    int64_t o = e * 3 * N3 + q;
    if constexpr (EMF_LOC_ROWS) {
      const int64_t row = a.fd_nx.div((uint32_t)e);
      o = loc_index<N>(row, (int)(e - row * a.nx), a.nx, q / (N * N), (q / N) % N, q % N, 0);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) a.loc[o + c * loc_cstride<N>(a.nx)] = out[c];
  }
}

}  // namespace emfgpu
