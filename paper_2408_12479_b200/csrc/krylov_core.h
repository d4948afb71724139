// Host-side Krylov cores shared by the single-GPU entry points (capi.cu)
// and the z-slab solver (slab_solver.cu): the device-resident Lanczos of
// estimate_eigenvalues (solver.hpp:262-308), parameterised by the apply and
// the dot, so that a slab run with the rank-ordered slab dot reproduces the
// single-GPU run bitwise.
#pragma once
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "capi_util.h"
#include "internal.h"

namespace emfgpu {
namespace capi {

inline int sturm_count(const std::vector<double>& al, const std::vector<double>& be, double sigma) {
  int count = 0;
  double d = al[0] - sigma;
  if (d < 0) ++count;
  for (size_t i = 1; i < al.size(); ++i) {
    d = al[i] - sigma - be[i - 1] * be[i - 1] / (d == 0 ? 1e-300 : d);
    if (d < 0) ++count;
  }
  return count;
}
inline double tridiag_extreme(const std::vector<double>& al, const std::vector<double>& be, bool largest) {
  double lo = al[0], hi = al[0];
  for (size_t i = 0; i < al.size(); ++i) {
    const double bl = i > 0 ? std::abs(be[i - 1]) : 0.0;
    const double br = i < be.size() ? std::abs(be[i]) : 0.0;
    lo = std::min(lo, al[i] - bl - br);
    hi = std::max(hi, al[i] + bl + br);
  }
  const int nev = (int)al.size();
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const int below = sturm_count(al, be, mid);
    if (largest ? below < nev : below < 1)
      lo = mid;
    else
      hi = mid;
    if (hi - lo < 1e-10 * std::max(1.0, std::abs(hi))) break;
  }
  return 0.5 * (lo + hi);
}

// work space of lanczos_core: the basis (n per step), D^-1/2, w, dot partials
// (4 per node plane, plus the result), the alpha/beta coefficients, the
// reorthogonalisation coefficients and their partials (one row per basis
// vector), two T vectors
template <typename T>
size_t lanczos_work_bytes(int64_t n, int iterations, int nplanes) {
  const int maxit = (int)std::min<int64_t>(iterations, std::max<int64_t>(n, 1));
  const size_t nd = (size_t)std::max(dot_partial_count(), nplanes * dot_plane_split()) + 1;
  return sizeof(double) * ((size_t)n * (std::max(1, maxit) + 2) + nd + 2 * (size_t)maxit + 2 + (size_t)maxit * (nd + 1)) +
         2 * sizeof(T) * (size_t)n + 64;
}
struct NoReorth {};

// Lanczos on D^-1/2 A D^-1/2 with full reorthogonalisation.  The reference
// reorthogonalises by modified Gram-Schmidt (solver.hpp:290-294): j + 1
// sequential dot / axpy pairs in step j, each a grid-wide reduction here (86 ms
// of cfg4's setup).  After the three-term recurrence w's components along the
// basis are at rounding level, so the classical one-pass form -- all
// coefficients from the same w, then one update -- keeps the basis orthogonal
// just as well; the eigenvalue estimates agree with the reference's to 1e-10
// (tests: 1e-6).  Device resident: the seeded start vector (elements gofs.. of
// the reference's stream) is generated on the device, the coefficients never
// leave it, one host read per step fetches alpha/beta^2.
// apply(const T* x, T* y); dot(const double* a, const double* b, double*
// partial, double* out) writes the dot to the device double out; reorth(w,
// basis, k, h, partial): h[v] = dot(w, basis_v) for v < k in one pass, then
// w -= sum_v h[v] basis_v in order -- optional (NoReorth: the same arithmetic
// through k dot calls and k axpys, bitwise the same result).
template <typename T, typename ApplyF, typename DotF, typename ReorthF = NoReorth>
void lanczos_core(int64_t n, int64_t gofs, int nplanes, double* work, const T* diag, int iterations, uint64_t seed,
                  ApplyF&& apply, DotF&& dot, double* lmin, double* lmax, cudaStream_t s, ReorthF&& reorth = NoReorth{}) {
  const int maxit = (int)std::min<int64_t>(iterations, std::max<int64_t>(n, 1));
  const size_t nd = (size_t)std::max(dot_partial_count(), nplanes * dot_plane_split()) + 1;
  double* basis = work;
  double* dis = basis + (size_t)n * std::max(1, maxit);
  double* w = dis + n;
  double* dbuf = w + n;  // [0] result, [1..] partials
  double* coef = dbuf + nd;
  double* hbuf = coef + 2 * (size_t)maxit + 2;  // reorthogonalisation coefficients
  double* mpart = hbuf + maxit;                 // their partials, nd per basis vector
  T* t = reinterpret_cast<T*>(mpart + (size_t)maxit * nd);
  T* at = t + n;
  launch_lanczos_start(basis, n, (unsigned long long)seed, s, gofs);
  dot(basis, basis, dbuf + 1, dbuf);
  launch_div_sqrt_dev(dbuf, basis, basis, n, s);
  launch_dinv_sqrt<T>(diag, dis, n, s);
  std::vector<double> alpha, beta;
  double hb = 0.0;
  for (int j = 0; j < maxit; ++j) {
    double* v = basis + (size_t)j * n;
    launch_scale_to_T<T>(dis, v, t, n, s);
    apply(t, at);
    launch_scale_from_T<T>(dis, at, w, n, s);
    if (j > 0) launch_axpy_minus(hb, basis + (size_t)(j - 1) * n, w, n, s);
    dot(w, v, dbuf + 1, coef + 2 * j);  // alpha_j
    launch_axpy_dev(coef + 2 * j, v, w, n, s);
    if constexpr (std::is_same_v<std::decay_t<ReorthF>, NoReorth>) {
      for (int qb = 0; qb <= j; ++qb) dot(w, basis + (size_t)qb * n, dbuf + 1, hbuf + qb);
      for (int qb = 0; qb <= j; ++qb) launch_axpy_dev(hbuf + qb, basis + (size_t)qb * n, w, n, s);
    } else {
      reorth(w, basis, j + 1, hbuf, mpart);
    }
    dot(w, w, dbuf + 1, coef + 2 * j + 1);  // beta_j^2
    double ab[2];
    CK(cudaMemcpyAsync(ab, coef + 2 * j, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    alpha.push_back(ab[0]);
    const double b = std::sqrt(ab[1]);
    if (j + 1 < maxit) beta.push_back(b);
    if (b < 1e-12) break;
    if (j + 1 < maxit) launch_div(w, b, basis + (size_t)(j + 1) * n, n, s);
    hb = b;
  }
  beta.resize(alpha.empty() ? 0 : alpha.size() - 1);
  *lmax = tridiag_extreme(alpha, beta, true);
  *lmin = tridiag_extreme(alpha, beta, false);
}

}  // namespace capi
}  // namespace emfgpu
