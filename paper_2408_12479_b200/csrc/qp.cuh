// Quadrature-point material kernels (device).  B200-native restatement of the
// reference's per-point algebra — NOT a translation of its lane-batched C++:
// one CUDA thread owns one quadrature point, all 3x3 tensors live in
// registers, the fourth-order tangent is never formed.
//
// Semantics follow (stable formulation, material domain):
//   make_strain            proj/include/elastmf/constitutive.hpp:43-57
//   compute_cache          constitutive.hpp:326-377
//   fiber_invariants       constitutive.hpp:117-149
//   second_pk_base         constitutive.hpp:197-238
//   tangent_material       constitutive.hpp:381-419
//   integrand              proj/include/elastmf/operator.hpp:495-504
//   ln_plus_one/fast_jpow  proj/include/elastmf/fastscalar.hpp:44-89
// Numerics: nvcc contracts a*b+c into FMA (the reference forbids contraction,
// proj/CMakeLists.txt:11-13), so results match the oracle to round-off
// (rel-L2 ~1e-15 fp64), not bitwise.  The ln series is evaluated in Horner
// form in y^2 (same 16 terms, same |x|>0.5 log1p switch).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace emfgpu {

enum Model : int { CNH = 0, INH = 1, FIBER = 2 };
enum Strategy : int { S_NONE = 0, S_SCALAR = 1, S_TENSOR = 2, S_CACHEDF = 3 };
// element-kernel strategy codes of the spatial (Omega_t) formulation
enum SpatialStrategy : int { S_SP_NONE = 4, S_SP_SCALAR = 5, S_SP_TENSOR = 6 };
__host__ __device__ constexpr bool is_spatial(int strat) { return strat >= S_SP_NONE && strat <= S_SP_TENSOR; }
// element-kernel code of evaluate_residual (operator.hpp:532-595): the same
// gather / sweeps / element-local results as an apply of strategy tensor,
// with the stress integrand of the input displacement at the points
constexpr int S_RESID = 7, S_RESID_SP = 8;  // material / spatial domain
__host__ __device__ constexpr bool is_resid(int strat) { return strat == S_RESID || strat == S_RESID_SP; }

// Material constants in the operator's number type, rounded from double the
// way the reference does (N(scalar_of<N>(p.x)), e.g. constitutive.hpp:200).
template <typename T>
struct MatConst {
  T mu, lam, half_k, kappa, k2, two_k1;
  T mu_3, two_mu_9, two_mu_3;  // mu/3, 2 mu/9, 2 mu/3 (host-rounded once, not divided per point)
  T h[2][6];   // structure tensors H4, H6 (material.cpp:50-82)
  T m1[2][3];  // mean fibre directions
};

template <typename T>
__device__ __forceinline__ T dlog1p(T x);
template <>
__device__ __forceinline__ double dlog1p<double>(double x) { return log1p(x); }
template <>
__device__ __forceinline__ float dlog1p<float>(float x) { return log1pf(x); }
template <typename T>
__device__ __forceinline__ T dexp(T x);
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }

// Reciprocal without the IEEE-division slow path: MUFU approximation refined
// by Newton steps (2 for fp64: ~full precision; |1/x - rcp(x)| <= 1 ulp class).
// Used for 1/det(F) and y = x/(2+x), whose arguments are bounded away from
// 0 and infinity on admissible states.
template <typename T>
__device__ __forceinline__ T fast_rcp(T x);
template <>
__device__ __forceinline__ double fast_rcp<double>(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
template <>
__device__ __forceinline__ float fast_rcp<float>(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  const float e = fmaf(-x, r, 1.0f);
  return fmaf(r, e, r);
}

// SymTensor order (11,22,33,12,13,23), tensor.hpp:93-100.
__host__ __device__ constexpr int sidx(int i, int j) { return i == j ? i : 2 + i + j; }

template <typename T>
__device__ __forceinline__ T det3(const T* t) {
  return (t[0] * (t[4] * t[8] - t[5] * t[7]) - t[1] * (t[3] * t[8] - t[5] * t[6])) +
         t[2] * (t[3] * t[7] - t[4] * t[6]);
}

// det(I+G)-1 without forming I+G (tensor.hpp:199-208).
template <typename T>
__device__ __forceinline__ T det_minus_one(const T* g) {
  const T tr = (g[0] + g[4]) + g[8];
  const T minors = ((g[0] * g[4] - g[1] * g[3]) + (g[0] * g[8] - g[2] * g[6])) + (g[4] * g[8] - g[5] * g[7]);
  return (det3(g) + minors) + tr;
}

// Adjugate / determinant (tensor.hpp:212-231); inverse3_det takes det(t) when
// it is already known (F: det F = 1 + (J-1), same value to rounding).
template <typename T>
__device__ __forceinline__ void inverse3_det(const T* t, T det, T* r) {
  const T inv = fast_rcp(det);
  r[0] = (t[4] * t[8] - t[5] * t[7]) * inv;
  r[1] = (t[2] * t[7] - t[1] * t[8]) * inv;
  r[2] = (t[1] * t[5] - t[2] * t[4]) * inv;
  r[3] = (t[5] * t[6] - t[3] * t[8]) * inv;
  r[4] = (t[0] * t[8] - t[2] * t[6]) * inv;
  r[5] = (t[2] * t[3] - t[0] * t[5]) * inv;
  r[6] = (t[3] * t[7] - t[4] * t[6]) * inv;
  r[7] = (t[1] * t[6] - t[0] * t[7]) * inv;
  r[8] = (t[0] * t[4] - t[1] * t[3]) * inv;
}
template <typename T>
__device__ __forceinline__ void inverse3(const T* t, T* r) {
  const T inv = fast_rcp(det3(t));
  r[0] = (t[4] * t[8] - t[5] * t[7]) * inv;
  r[1] = (t[2] * t[7] - t[1] * t[8]) * inv;
  r[2] = (t[1] * t[5] - t[2] * t[4]) * inv;
  r[3] = (t[5] * t[6] - t[3] * t[8]) * inv;
  r[4] = (t[0] * t[8] - t[2] * t[6]) * inv;
  r[5] = (t[2] * t[3] - t[0] * t[5]) * inv;
  r[6] = (t[3] * t[7] - t[4] * t[6]) * inv;
  r[7] = (t[1] * t[6] - t[0] * t[7]) * inv;
  r[8] = (t[0] * t[4] - t[1] * t[3]) * inv;
}

// r = x * y (general x general)
template <typename T>
__device__ __forceinline__ void mm(const T* x, const T* y, T* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r[3 * i + j] = (x[3 * i] * y[j] + x[3 * i + 1] * y[3 + j]) + x[3 * i + 2] * y[6 + j];
}
// r = x * y^T (general x general^T)
template <typename T>
__device__ __forceinline__ void mm_bt(const T* x, const T* y, T* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (x[3 * i] * y[3 * j] + x[3 * i + 1] * y[3 * j + 1]) + x[3 * i + 2] * y[3 * j + 2];
}
// r = x * ys (general x symmetric)
template <typename T>
__device__ __forceinline__ void mm_ts(const T* x, const T* ys, T* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (x[3 * i] * ys[sidx(0, j)] + x[3 * i + 1] * ys[sidx(1, j)]) + x[3 * i + 2] * ys[sidx(2, j)];
}
// symmetric part of xs * y, only the 6 unique entries (tensor.hpp:155-166 of matmul)
template <typename T>
__device__ __forceinline__ void sym_mm_st(const T* xs, const T* y, T* s) {
  T r[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (xs[sidx(i, 0)] * y[j] + xs[sidx(i, 1)] * y[3 + j]) + xs[sidx(i, 2)] * y[6 + j];
  s[0] = r[0];
  s[1] = r[4];
  s[2] = r[8];
  s[3] = T(0.5) * (r[1] + r[3]);
  s[4] = T(0.5) * (r[2] + r[6]);
  s[5] = T(0.5) * (r[5] + r[7]);
}
template <typename T>
__device__ __forceinline__ void sym_part(const T* t, T* s) {
  s[0] = t[0];
  s[1] = t[4];
  s[2] = t[8];
  s[3] = T(0.5) * (t[1] + t[3]);
  s[4] = T(0.5) * (t[2] + t[6]);
  s[5] = T(0.5) * (t[5] + t[7]);
}
template <typename T>
__device__ __forceinline__ T ddot_s(const T* x, const T* y) {
  return ((x[0] * y[0] + x[1] * y[1]) + x[2] * y[2]) + T(2) * ((x[3] * y[3] + x[4] * y[4]) + x[5] * y[5]);
}

// ln(1+x): 2 sum_{n<16} y^(2n+1)/(2n+1), y = x/(2+x); log1p for |x|>0.5
// (fastscalar.hpp:44-71).  Horner in y^2 instead of the stored powers.
// Two interleaved Horner chains in y^4 (even / odd powers of y^2) halve the
// dependent-FMA depth of the 16-term sum.
// For y^2 < 1/64 the terms past n = 9 sum to less than y^20 / 21 < 2^-64
// relative to the leading term, so 10 terms give the same double.
template <typename T>
__device__ __forceinline__ T ln_plus_one(T x) {
  if (fabs(x) > T(0.5)) return dlog1p(x);
  const T y = x * fast_rcp(T(2) + x);
  const T y2 = y * y;
  const T y4 = y2 * y2;
  T se, so;  // coefficients 1/(2n+1), n even / odd
  if (y2 < T(1.0 / 64.0)) {
    se = T(1.0 / 17.0);
    so = T(1.0 / 19.0);
#pragma unroll
    for (int m = 3; m >= 0; --m) {
      se = se * y4 + T(1.0 / (4 * m + 1));
      so = so * y4 + T(1.0 / (4 * m + 3));
    }
  } else {
    se = T(1.0 / 29.0);
    so = T(1.0 / 31.0);
#pragma unroll
    for (int m = 6; m >= 0; --m) {
      se = se * y4 + T(1.0 / (4 * m + 1));
      so = so * y4 + T(1.0 / (4 * m + 3));
    }
  }
  return T(2) * (y * (se + y2 * so));
}

// J^(-2/3) by the reference's 3-step Newton recurrence (fastscalar.hpp:77-89).
template <typename T>
__device__ __forceinline__ T fast_jpow(T jm1) {
  const T third = T(1) / T(3);
  const T four_thirds = T(4) / T(3);
  const T alpha = ((jm1 + T(2)) * jm1 + T(1)) * third;
  T beta = four_thirds - alpha;
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const T b2 = beta * beta;
    beta = four_thirds * beta - alpha * (b2 * b2);
  }
  return beta;
}

// Everything the tangent needs at one point (QpCache, constitutive.hpp:79-93,
// material cell).  E/jm1 are kept for second_pk.
template <typename T>
struct Bundle {
  T F[9], Finv[9], Cinv[6], S[6], E[6];
  T jm1, lnj, jp, c1, c2, c3[2], efib[2];
};

// Stable kinematics from the displacement gradient g (constitutive.hpp:48-57).
// Returns false when det(F) <= 0.
template <typename T>
__device__ __forceinline__ bool make_strain(const T* g, Bundle<T>& c) {
  c.jm1 = det_minus_one(g);
  if (!(c.jm1 > T(-1))) return false;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const T q = (g[i] * g[j] + g[3 + i] * g[3 + j]) + g[6 + i] * g[6 + j];
      c.E[sidx(i, j)] = T(0.5) * ((g[3 * i + j] + g[3 * j + i]) + q);
    }
#pragma unroll
  for (int i = 0; i < 9; ++i) c.F[i] = g[i];
  c.F[0] = T(1) + g[0];
  c.F[4] = T(1) + g[4];
  c.F[8] = T(1) + g[8];
  inverse3_det(c.F, T(1) + c.jm1, c.Finv);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j)
      c.Cinv[sidx(i, j)] =
          (c.Finv[3 * i] * c.Finv[3 * j] + c.Finv[3 * i + 1] * c.Finv[3 * j + 1]) + c.Finv[3 * i + 2] * c.Finv[3 * j + 2];
  return true;
}

// Scalars of compute_cache (constitutive.hpp:335-366).
template <typename T, int MODEL>
__device__ __forceinline__ void cache_scalars(const MatConst<T>& m, Bundle<T>& c) {
  const T i1 = T(3) + T(2) * ((c.E[0] + c.E[1]) + c.E[2]);
  c.lnj = MODEL == CNH ? ln_plus_one(c.jm1) : T(0);  // lnJ enters only cNH's material tangent
  c.jp = MODEL == CNH ? T(1) : fast_jpow(c.jm1);
  if (MODEL != CNH) {
    const T jac = T(1) + c.jm1;
    c.c1 = m.half_k * (c.jm1 * (c.jm1 + T(2))) - (m.mu_3 * c.jp) * i1;
    c.c2 = (m.two_mu_9 * c.jp) * i1 + (m.kappa * jac) * jac;
  }
  if (MODEL == FIBER) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      T mm6[6];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) mm6[sidx(i, j)] = m.m1[f][i] * m.m1[f][j];
      c.efib[f] = T(2) * ddot_s(m.h[f], c.E);
      const T gate = T(2) * ddot_s(mm6, c.E);
      const T z = (m.k2 * c.efib[f]) * c.efib[f];
      c.c3[f] = gate > T(0) ? dexp(z) * m.two_k1 : T(0);  // tension-only gate, stable form
    }
  }
}

// S = second_pk_base (+ fibre terms), constitutive.hpp:197-238, 368-371.
template <typename T, int MODEL>
__device__ __forceinline__ void second_pk(const MatConst<T>& m, Bundle<T>& c) {
  T inner[6];
  if (MODEL == CNH) {
#pragma unroll
    for (int k = 0; k < 6; ++k) inner[k] = (T(2) * m.mu) * c.E[k];
    const T v = (T(2) * m.lam) * c.lnj;
    inner[0] += v;
    inner[1] += v;
    inner[2] += v;
  } else {
    const T vol = m.half_k * (c.jm1 * (c.jm1 + T(2)));
    const T tre3 = ((c.E[0] + c.E[1]) + c.E[2]) * (T(1) / T(3));
    const T s = (T(2) * m.mu) * c.jp;
#pragma unroll
    for (int k = 0; k < 6; ++k) inner[k] = s * c.E[k];
    const T d = vol - s * tre3;
    inner[0] += d;
    inner[1] += d;
    inner[2] += d;
  }
  T full[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) full[3 * i + j] = inner[sidx(i, j)];
  sym_mm_st(c.Cinv, full, c.S);
  if (MODEL == FIBER) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const T coef = c.c3[f] * c.efib[f];
#pragma unroll
      for (int k = 0; k < 6; ++k) c.S[k] += coef * m.h[f][k];
    }
  }
}

// D_u S in direction dg (constitutive.hpp:381-419).
template <typename T, int MODEL>
__device__ __forceinline__ void tangent_material(const MatConst<T>& m, const Bundle<T>& c, const T* dg, T* r) {
  T a[9], sac[6];
  mm(c.Finv, dg, a);
  const T w = (a[0] + a[4]) + a[8];
  {
    T ac[9];
    mm_ts(a, c.Cinv, ac);
    sym_part(ac, sac);
  }
  if (MODEL == CNH) {
    const T f1 = T(2) * (m.mu - (T(2) * m.lam) * c.lnj);
    const T f2 = (T(2) * m.lam) * w;
#pragma unroll
    for (int k = 0; k < 6; ++k) r[k] = f1 * sac[k] + f2 * c.Cinv[k];
    return;
  }
  T q = c.F[0] * dg[0];
#pragma unroll
  for (int i = 1; i < 9; ++i) q += c.F[i] * dg[i];
  const T ttmj = m.two_mu_3 * c.jp;
  const T m2c1 = T(-2) * c.c1;
  const T f2 = c.c2 * w - ttmj * q;
#pragma unroll
  for (int k = 0; k < 6; ++k) r[k] = m2c1 * sac[k] + f2 * c.Cinv[k];
  const T dgl = (-ttmj) * w;
  r[0] += dgl;
  r[1] += dgl;
  r[2] += dgl;
  if (MODEL == FIBER) {
    T dch[6];
    // sym(F^T dg)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) {
        const T xij = (c.F[i] * dg[j] + c.F[3 + i] * dg[3 + j]) + c.F[6 + i] * dg[6 + j];
        const T xji = (c.F[j] * dg[i] + c.F[3 + j] * dg[3 + i]) + c.F[6 + j] * dg[6 + i];
        dch[sidx(i, j)] = i == j ? xij : T(0.5) * (xij + xji);
      }
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const T hdc = T(2) * ddot_s(m.h[f], dch);
      const T coef = (c.c3[f] * ((((T(2) * m.k2) * c.efib[f]) * c.efib[f]) + T(1))) * hdc;
#pragma unroll
      for (int k = 0; k < 6; ++k) r[k] += coef * m.h[f][k];
    }
  }
}

// Material integrand in physical space, wm = dg S + F D_uS (operator.hpp:503).
// For cNH / iNH it is evaluated in the algebraically equivalent form that
// never builds D_uS: with A = F^-1 dg, F C^-1 = F^-T and
// F sym(A C^-1) = (dg C^-1 + (A F^-1)^T) / 2, so
//   cNH: wm = dg (S + f1/2 C^-1) + f1/2 (A F^-1)^T + f2 F^-T,
//        f1 = 2(mu - 2 lambda lnJ), f2 = 2 lambda tr A;
//   iNH: wm = dg (S - c1 C^-1) - c1 (A F^-1)^T + (c2 tr A - t q) F^-T - t tr(A) F,
//        t = 2 mu J^-2/3 / 3, q = F : dg;
// 105 (cNH) instead of 129 flops.  The fibre model keeps the direct form.
template <typename T, int MODEL>
__device__ __forceinline__ void tangent_wm(const MatConst<T>& m, const Bundle<T>& c, const T* dg, T* wm) {
  if constexpr (MODEL == FIBER) {
    T ds[6], t1[9], t2[9];
    tangent_material<T, MODEL>(m, c, dg, ds);
    mm_ts(dg, c.S, t1);
    mm_ts(c.F, ds, t2);
#pragma unroll
    for (int k = 0; k < 9; ++k) wm[k] = t1[k] + t2[k];
  } else {
    T A[9], AF[9], M[6];
    mm(c.Finv, dg, A);
    const T trA = (A[0] + A[4]) + A[8];
    mm(A, c.Finv, AF);
    T h, g2;  // coefficient of (A F^-1)^T and of F^-T
    if constexpr (MODEL == CNH) {
      h = m.mu - (T(2) * m.lam) * c.lnj;  // f1 / 2
      g2 = (T(2) * m.lam) * trA;
    } else {
      T q = c.F[0] * dg[0];
#pragma unroll
      for (int i = 1; i < 9; ++i) q += c.F[i] * dg[i];
      const T t = m.two_mu_3 * c.jp;
      h = -c.c1;
      g2 = c.c2 * trA - t * q;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) M[k] = c.S[k] + h * c.Cinv[k];
    mm_ts(dg, M, wm);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) wm[3 * i + j] += h * AF[3 * j + i] + g2 * c.Finv[3 * j + i];
    if constexpr (MODEL == INH) {
      const T tw = -(m.two_mu_3 * c.jp) * trA;
#pragma unroll
      for (int k = 0; k < 9; ++k) wm[k] += tw * c.F[k];
    }
  }
}

// Green-Euler strain bt = (G + G^T + G G^T)/2 (tensor.hpp:259-270).
template <typename T>
__device__ __forceinline__ void green_euler(const T* g, T* bt) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) {
      const T q = (g[3 * i] * g[3 * j] + g[3 * i + 1] * g[3 * j + 1]) + g[3 * i + 2] * g[3 * j + 2];
      bt[sidx(i, j)] = T(0.5) * ((g[3 * i + j] + g[3 * j + i]) + q);
    }
}

// ---- push-forward form of the material integrand (cNH / iNH) -----------------
// The reference's integrand w_ref = detw (dg S + F D_uS) J0^-T
// (operator.hpp:502-504, constitutive.hpp:381-419) rewritten exactly through
// the push-forward to the current configuration.  With K = J0^-1 F^-1 and
// l = dg F^-1 = Gref K:
//   w_ref = detw W K^T,  W = (dg S + F D_uS) F^T
//   cNH: W = mu l b + h l^T + 2 lam tr(l) I,          h = mu - 2 lam lnJ
//   iNH: W = beta l b - c1 l^T + (c2 tr l - t l:b) I - t tr(l) b,
//        beta = mu J^-2/3, t = 2 mu J^-2/3 / 3
// (dg S F^T = l tau; tau - c1 I = mu J^-2/3 b for iNH and tau + h I = mu b for
// cNH, so the large volumetric parts of S and c1 C^-1 cancel analytically;
// dg C^-1 F^T = l, (F^-1 dg F^-1)^T F^T = l^T, F : dg = l : b).  The state a
// point keeps between the linearization and test halves is b (6), K (9) and
// 4 scalars with detw folded in (was F^-1, S, C^-1, F, J0^-1, scalars: 43),
// and the test half is 3 small matrix products (~100 flops instead of ~190).
// Same quantity as the reference's, different rounding (rel-L2 ~1e-15).
template <typename T>
struct PushState {
  T K[9], b[6];
  T k_lb, k_lt, k_tr, k_t;  // coefficients of l b, l^T, tr(l) I (and t: l:b I, tr(l) b), times detw
  // fibre model (strategy tensor): the pushed structure tensors A_f = F H_f F^T
  // and, times detw, k_s = c3 e (stress) and k_c = 2 c3 (2 k2 e^2 + 1) (tangent):
  //   W += sum_f k_s l A_f + k_c (A_f : l) A_f
  // (dg S_fib F^T = l F S_fib F^T; H_f : sym(F^T dg) = A_f : l;
  // constitutive.hpp:368-371, 404-417)
  T Af[2][6], k_s[2], k_c[2];
};

// State at one point from the linearization gradient gg = grad_X u_k (material
// coordinates), J0^-1 and detw.  Scalars either computed (strategy none /
// cachedF, constitutive.hpp:335-366) or taken from the scalar cache.
// Returns false when det(F) <= 0 (make_strain's check, constitutive.hpp:48-52).
// kDiagJ: J0^-1 diagonal (entries 0, 4, 8 read only).
template <typename T, int MODEL, bool kCached, bool kDiagJ>
__device__ __forceinline__ bool push_state(const MatConst<T>& m, const T* gg, const T* j0inv, T detw,
                                           const Bundle<T>& cached, PushState<T>& ps) {
  const T jm1 = det_minus_one(gg);
  if (!(jm1 > T(-1))) return false;
  T bt[6];
  green_euler(gg, bt);
#pragma unroll
  for (int k = 0; k < 6; ++k) ps.b[k] = T(2) * bt[k];
  ps.b[0] += T(1);
  ps.b[1] += T(1);
  ps.b[2] += T(1);
  {
    T F[9], Finv[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) F[i] = gg[i];
    F[0] += T(1);
    F[4] += T(1);
    F[8] += T(1);
    inverse3_det(F, T(1) + jm1, Finv);
    if constexpr (kDiagJ) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) ps.K[3 * i + j] = j0inv[4 * i] * Finv[3 * i + j];
    } else {
      mm(j0inv, Finv, ps.K);
    }
  }
  if constexpr (MODEL == CNH) {
    const T lnj = kCached ? cached.lnj : ln_plus_one(jm1);
    ps.k_lb = m.mu * detw;
    ps.k_lt = (m.mu - (T(2) * m.lam) * lnj) * detw;
    ps.k_tr = (T(2) * m.lam) * detw;
    ps.k_t = T(0);
  } else {
    T jp, c1, c2;
    if constexpr (kCached) {
      jp = cached.jp;
      c1 = cached.c1;
      c2 = cached.c2;
    } else {
      jp = fast_jpow(jm1);
      const T i1 = T(3) + T(2) * ((bt[0] + bt[1]) + bt[2]);
      const T jac = T(1) + jm1;
      c1 = m.half_k * (jm1 * (jm1 + T(2))) - (m.mu_3 * jp) * i1;
      c2 = (m.two_mu_9 * jp) * i1 + (m.kappa * jac) * jac;
    }
    ps.k_lb = (m.mu * jp) * detw;
    ps.k_lt = -c1 * detw;
    ps.k_tr = c2 * detw;
    ps.k_t = (m.two_mu_3 * jp) * detw;
  }
  return true;
}

// The state as 19 cache fields (kernels.cuh: C_PK, C_PB, C_PC), computed in
// TS and stored / loaded as T.
// Fibre part of the state from the material bundle (after make_strain and
// cache_scalars).
template <typename T>
__device__ __forceinline__ void push_state_fibre(const MatConst<T>& m, const Bundle<T>& c, T detw, PushState<T>& ps) {
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    T fh[9], a[9];
    mm_ts(c.F, m.h[f], fh);
    mm_bt(fh, c.F, a);  // F H F^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) ps.Af[f][sidx(i, j)] = i == j ? a[3 * i + j] : T(0.5) * (a[3 * i + j] + a[3 * j + i]);
    ps.k_s[f] = (c.c3[f] * c.efib[f]) * detw;
    ps.k_c[f] = (T(2) * (c.c3[f] * ((((T(2) * m.k2) * c.efib[f]) * c.efib[f]) + T(1)))) * detw;
  }
}

template <typename T, typename TS>
__device__ __forceinline__ void store_push_state_fibre(T* cache, int64_t st, int64_t qidx, const PushState<TS>& ps) {
#pragma unroll
  for (int f = 0; f < 2; ++f) {
#pragma unroll
    for (int m = 0; m < 6; ++m) cache[(19 + 8 * f + m) * st + qidx] = T(ps.Af[f][m]);
    cache[(19 + 8 * f + 6) * st + qidx] = T(ps.k_s[f]);
    cache[(19 + 8 * f + 7) * st + qidx] = T(ps.k_c[f]);
  }
}
template <typename T>
__device__ __forceinline__ void load_push_state_fibre(const T* cs, int64_t st, int64_t qidx, PushState<T>& ps) {
#pragma unroll
  for (int f = 0; f < 2; ++f) {
#pragma unroll
    for (int m = 0; m < 6; ++m) ps.Af[f][m] = cs[(19 + 8 * f + m) * st + qidx];
    ps.k_s[f] = cs[(19 + 8 * f + 6) * st + qidx];
    ps.k_c[f] = cs[(19 + 8 * f + 7) * st + qidx];
  }
}

template <typename T, typename TS>
__device__ __forceinline__ void store_push_state(T* cache, int64_t st, int64_t qidx, const PushState<TS>& ps) {
#pragma unroll
  for (int m = 0; m < 9; ++m) cache[(0 + m) * st + qidx] = T(ps.K[m]);
#pragma unroll
  for (int m = 0; m < 6; ++m) cache[(9 + m) * st + qidx] = T(ps.b[m]);
  cache[15 * st + qidx] = T(ps.k_lb);
  cache[16 * st + qidx] = T(ps.k_lt);
  cache[17 * st + qidx] = T(ps.k_tr);
  cache[18 * st + qidx] = T(ps.k_t);
}
template <typename T>
__device__ __forceinline__ void load_push_state(const T* cs, int64_t st, int64_t qidx, PushState<T>& ps) {
#pragma unroll
  for (int m = 0; m < 9; ++m) ps.K[m] = cs[(0 + m) * st + qidx];
#pragma unroll
  for (int m = 0; m < 6; ++m) ps.b[m] = cs[(9 + m) * st + qidx];
  ps.k_lb = cs[15 * st + qidx];
  ps.k_lt = cs[16 * st + qidx];
  ps.k_tr = cs[17 * st + qidx];
  ps.k_t = cs[18 * st + qidx];
}

// w_ref = W K^T for the test gradient gref (reference coordinates).
template <typename T, int MODEL>
__device__ __forceinline__ void push_integrand(const PushState<T>& ps, const T* gref, T* wref) {
  T l[9];
  mm(gref, ps.K, l);
  const T trl = (l[0] + l[4]) + l[8];
  T W[9];
  mm_ts(l, ps.b, W);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) W[3 * i + j] = ps.k_lb * W[3 * i + j] + ps.k_lt * l[3 * j + i];
  T diag = ps.k_tr * trl;
  if constexpr (MODEL != CNH) {
    const T ldb = ((l[0] * ps.b[0] + l[4] * ps.b[1]) + l[8] * ps.b[2]) +
                  (((l[1] + l[3]) * ps.b[3] + (l[2] + l[6]) * ps.b[4]) + (l[5] + l[7]) * ps.b[5]);
    diag -= ps.k_t * ldb;
    const T tt = -ps.k_t * trl;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) W[3 * i + j] += tt * ps.b[sidx(i, j)];
  }
  W[0] += diag;
  W[4] += diag;
  W[8] += diag;
  if constexpr (MODEL == FIBER) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const T* A = ps.Af[f];
      T la[9];
      mm_ts(l, A, la);
      const T adl = ((l[0] * A[0] + l[4] * A[1]) + l[8] * A[2]) +
                    (((l[1] + l[3]) * A[3] + (l[2] + l[6]) * A[4]) + (l[5] + l[7]) * A[5]);
      const T ca = ps.k_c[f] * adl;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) W[3 * i + j] += ps.k_s[f] * la[3 * i + j] + ca * A[sidx(i, j)];
    }
  }
  mm_bt(W, ps.K, wref);
}

// w_ref = detw * (dg S + F D_uS) J0^-T  (operator.hpp:502-504), dg = Gref J0^-1.
template <typename T, int MODEL>
__device__ __forceinline__ void tangent_integrand(const MatConst<T>& m, const Bundle<T>& c, const T* gref,
                                                  const T* j0inv, T detw, T* wref) {
  T dg[9], wm[9];
  mm(gref, j0inv, dg);
  tangent_wm<T, MODEL>(m, c, dg, wm);
  mm_bt(wm, j0inv, wref);
#pragma unroll
  for (int k = 0; k < 9; ++k) wref[k] *= detw;
}

// ---- spatial (Omega_t) formulation -------------------------------------------
// Spatial cell of QpCache (constitutive.hpp:91-92): b = F F^T, tau, F H_i F^T.
template <typename T>
struct SpCell {
  T b[6], tau[6], fh[2][6];
};

// b = 2 bt + I, tau = kirchhoff_base (constitutive.hpp:240-283, stable) plus
// the fibre terms c3 E_i F H_i F^T (push_forward, tensor.hpp:332-341).
// Reads c.F, c.jm1, c.lnj (cNH), c.jp, c.c3, c.efib.
template <typename T, int MODEL>
__device__ __forceinline__ void spatial_cell(const MatConst<T>& m, const Bundle<T>& c, const T* bt, SpCell<T>& sp) {
#pragma unroll
  for (int k = 0; k < 6; ++k) sp.b[k] = T(2) * bt[k];
  sp.b[0] += T(1);
  sp.b[1] += T(1);
  sp.b[2] += T(1);
  if (MODEL == CNH) {
#pragma unroll
    for (int k = 0; k < 6; ++k) sp.tau[k] = (T(2) * m.mu) * bt[k];
    const T v = (T(2) * m.lam) * c.lnj;
    sp.tau[0] += v;
    sp.tau[1] += v;
    sp.tau[2] += v;
  } else {
    const T vol = m.half_k * (c.jm1 * (c.jm1 + T(2)));
    const T trb3 = ((bt[0] + bt[1]) + bt[2]) * (T(1) / T(3));
    const T s2 = (T(2) * m.mu) * c.jp;
#pragma unroll
    for (int k = 0; k < 6; ++k) sp.tau[k] = s2 * bt[k];
    const T v = vol - s2 * trb3;
    sp.tau[0] += v;
    sp.tau[1] += v;
    sp.tau[2] += v;
  }
  if (MODEL == FIBER) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      T fhm[9];
      mm_ts(c.F, m.h[f], fhm);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j)
          sp.fh[f][sidx(i, j)] = (fhm[3 * i] * c.F[3 * j] + fhm[3 * i + 1] * c.F[3 * j + 1]) + fhm[3 * i + 2] * c.F[3 * j + 2];
      const T coef = c.c3[f] * c.efib[f];
#pragma unroll
      for (int k = 0; k < 6; ++k) sp.tau[k] += coef * sp.fh[f][k];
    }
  }
}

// tangent_spatial (constitutive.hpp:421-463): J c : (grad du)^S + (grad du) tau.
template <typename T, int MODEL>
__device__ __forceinline__ void tangent_spatial(const MatConst<T>& m, const Bundle<T>& c, const SpCell<T>& sp,
                                                const T* dgrad, T* out) {
  T xs[6], jc[6];
  sym_part(dgrad, xs);
  const T trx = (dgrad[0] + dgrad[4]) + dgrad[8];
  if (MODEL == CNH) {
    const T f = T(2) * (m.mu - (T(2) * m.lam) * c.lnj);
    const T v = (T(2) * m.lam) * trx;
#pragma unroll
    for (int k = 0; k < 6; ++k) jc[k] = f * xs[k];
    jc[0] += v;
    jc[1] += v;
    jc[2] += v;
  } else {
    const T bx = ddot_s(sp.b, xs);
    const T ttmj = m.two_mu_3 * c.jp;
    const T f0 = -ttmj * trx;
    const T m2c1 = T(-2) * c.c1;
#pragma unroll
    for (int k = 0; k < 6; ++k) jc[k] = f0 * sp.b[k] + m2c1 * xs[k];
    const T v = c.c2 * trx - ttmj * bx;
    jc[0] += v;
    jc[1] += v;
    jc[2] += v;
    if (MODEL == FIBER) {
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const T fhx = ddot_s(sp.fh[f], xs);
        const T coef = ((T(2) * c.c3[f]) * ((((T(2) * m.k2) * c.efib[f]) * c.efib[f]) + T(1))) * fhx;
#pragma unroll
        for (int k = 0; k < 6; ++k) jc[k] += coef * sp.fh[f][k];
      }
    }
  }
  mm_ts(dgrad, sp.tau, out);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) out[3 * i + j] += jc[sidx(i, j)];
}

// w_ref = s (tangent_spatial(Gref J_t^-1)) J_t^-T with s = (1/J) det J_t w_q
// (operator.hpp:506-519).
template <typename T, int MODEL>
__device__ __forceinline__ void spatial_integrand(const MatConst<T>& m, const Bundle<T>& c, const SpCell<T>& sp,
                                                  const T* gref, const T* jtinv, T s, T* wref) {
  T dgrad[9], ws[9];
  mm(gref, jtinv, dgrad);
  tangent_spatial<T, MODEL>(m, c, sp, dgrad, ws);
  mm_bt(ws, jtinv, wref);
#pragma unroll
  for (int k = 0; k < 9; ++k) wref[k] *= s;
}

}  // namespace emfgpu
