// Forward-stability lab on the device: the reference's
// pointwise fp32-vs-fp64 sweep (stability.hpp, stability.cpp:163-251).
//
// For every (scale, sample) a CUDA thread draws the seeded displacement
// gradient and direction (SweepRng stream splitting, sample_gradient), then
// evaluates every (model, formulation, quantity) cell in double and in float
// with the reference's formulas in the reference's operation order, and
// folds the componentwise deviation (normalised by the largest fp64 entry)
// into the cell's maximum with an order-independent atomicMax on the bit
// pattern of a non-negative double.  This translation unit is compiled with
// -fmad=false (Makefile) so that every product and sum rounds separately,
// as in the reference build (proj/CMakeLists.txt:11-13).
//
// Cells: models cNH, iNH, fibre, SVK x formulations standard-material,
// stable-material, standard-spatial, stable-spatial x quantities stress,
// tangent -> 32 per scale, ordered as the reference's write_csv.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

namespace emfgpu {
namespace lab {

constexpr int kCells = 32;

template <typename N>
struct T2 {
  N a[9];
  __device__ N& operator()(int i, int j) { return a[3 * i + j]; }
  __device__ N operator()(int i, int j) const { return a[3 * i + j]; }
};
template <typename N>
struct S2 {
  N s[6];
  __device__ N& operator()(int i, int j) { return s[sidx(i, j)]; }
  __device__ N operator()(int i, int j) const { return s[sidx(i, j)]; }
};

template <typename N>
struct Consts {
  N mu, lam, half_k, kappa, k2, two_k1;
  S2<N> h[2];
  N m1[2][3];
};

template <typename N>
__device__ N d_log(N x);
template <>
__device__ double d_log<double>(double x) { return log(x); }
template <>
__device__ float d_log<float>(float x) { return logf(x); }
template <typename N>
__device__ N d_log1p(N x);
template <>
__device__ double d_log1p<double>(double x) { return log1p(x); }
template <>
__device__ float d_log1p<float>(float x) { return log1pf(x); }
template <typename N>
__device__ N d_exp(N x);
template <>
__device__ double d_exp<double>(double x) { return exp(x); }
template <>
__device__ float d_exp<float>(float x) { return expf(x); }

// ---- tensor algebra, tensor.hpp ------------------------------------------
template <typename N>
__device__ N det(const T2<N>& t) {  // tensor.hpp:188-194
  const N c0 = t(0, 0) * (t(1, 1) * t(2, 2) - t(1, 2) * t(2, 1));
  const N c1 = t(0, 1) * (t(1, 0) * t(2, 2) - t(1, 2) * t(2, 0));
  const N c2 = t(0, 2) * (t(1, 0) * t(2, 1) - t(1, 1) * t(2, 0));
  return (c0 - c1) + c2;
}
template <typename N>
__device__ N det_m1(const T2<N>& g) {  // tensor.hpp:199-208
  const N tr = (g(0, 0) + g(1, 1)) + g(2, 2);
  const N m01 = g(0, 0) * g(1, 1) - g(0, 1) * g(1, 0);
  const N m02 = g(0, 0) * g(2, 2) - g(0, 2) * g(2, 0);
  const N m12 = g(1, 1) * g(2, 2) - g(1, 2) * g(2, 1);
  const N minors = (m01 + m02) + m12;
  return (det(g) + minors) + tr;
}
template <typename N>
__device__ bool inv(const T2<N>& t, T2<N>& r) {  // tensor.hpp:212-231, false = SingularTensor
  const N d = det(t);
  const N floor_ = sizeof(N) == 8 ? N(1e-300) : N(1e-30);
  if (fabs(d) < floor_) return false;
  const N id = N(1) / d;
  r(0, 0) = (t(1, 1) * t(2, 2) - t(1, 2) * t(2, 1)) * id;
  r(0, 1) = (t(0, 2) * t(2, 1) - t(0, 1) * t(2, 2)) * id;
  r(0, 2) = (t(0, 1) * t(1, 2) - t(0, 2) * t(1, 1)) * id;
  r(1, 0) = (t(1, 2) * t(2, 0) - t(1, 0) * t(2, 2)) * id;
  r(1, 1) = (t(0, 0) * t(2, 2) - t(0, 2) * t(2, 0)) * id;
  r(1, 2) = (t(0, 2) * t(1, 0) - t(0, 0) * t(1, 2)) * id;
  r(2, 0) = (t(1, 0) * t(2, 1) - t(1, 1) * t(2, 0)) * id;
  r(2, 1) = (t(0, 1) * t(2, 0) - t(0, 0) * t(2, 1)) * id;
  r(2, 2) = (t(0, 0) * t(1, 1) - t(0, 1) * t(1, 0)) * id;
  return true;
}
template <typename N>
__device__ T2<N> mm(const T2<N>& x, const T2<N>& y) {
  T2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (x(i, 0) * y(0, j) + x(i, 1) * y(1, j)) + x(i, 2) * y(2, j);
  return r;
}
template <typename N>
__device__ T2<N> mm(const S2<N>& x, const T2<N>& y) {
  T2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (x(i, 0) * y(0, j) + x(i, 1) * y(1, j)) + x(i, 2) * y(2, j);
  return r;
}
template <typename N>
__device__ T2<N> mm(const T2<N>& x, const S2<N>& y) {
  T2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = (x(i, 0) * y(0, j) + x(i, 1) * y(1, j)) + x(i, 2) * y(2, j);
  return r;
}
template <typename N>
__device__ T2<N> tr(const T2<N>& t) {
  T2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = t(j, i);
  return r;
}
template <typename N>
__device__ S2<N> sym(const T2<N>& t) {  // tensor.hpp:155-166
  S2<N> x;
  const N h(0.5);
  x.s[0] = t(0, 0);
  x.s[1] = t(1, 1);
  x.s[2] = t(2, 2);
  x.s[3] = h * (t(0, 1) + t(1, 0));
  x.s[4] = h * (t(0, 2) + t(2, 0));
  x.s[5] = h * (t(1, 2) + t(2, 1));
  return x;
}
template <typename N>
__device__ S2<N> to_sym(const T2<N>& t) {  // tensor.hpp:143-153
  S2<N> x;
  x.s[0] = t(0, 0);
  x.s[1] = t(1, 1);
  x.s[2] = t(2, 2);
  x.s[3] = t(0, 1);
  x.s[4] = t(0, 2);
  x.s[5] = t(1, 2);
  return x;
}
template <typename N>
__device__ T2<N> full(const S2<N>& s) {
  T2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = s(i, j);
  return r;
}
template <typename N>
__device__ N trace(const T2<N>& t) {
  return (t(0, 0) + t(1, 1)) + t(2, 2);
}
template <typename N>
__device__ N trace(const S2<N>& x) {
  return (x.s[0] + x.s[1]) + x.s[2];
}
template <typename N>
__device__ N ddot(const S2<N>& x, const S2<N>& y) {  // tensor.hpp:274-279
  const N d = (x.s[0] * y.s[0] + x.s[1] * y.s[1]) + x.s[2] * y.s[2];
  const N o = (x.s[3] * y.s[3] + x.s[4] * y.s[4]) + x.s[5] * y.s[5];
  return d + N(2) * o;
}
template <typename N>
__device__ N ddot(const T2<N>& x, const T2<N>& y) {  // tensor.hpp:281-286
  N r = x.a[0] * y.a[0];
  for (int i = 1; i < 9; ++i) r += x.a[i] * y.a[i];
  return r;
}
template <typename N>
__device__ S2<N> scale(N a, const S2<N>& x) {
  S2<N> r;
  for (int k = 0; k < 6; ++k) r.s[k] = a * x.s[k];
  return r;
}
template <typename N>
__device__ void add_to(S2<N>& r, const S2<N>& x) {
  for (int k = 0; k < 6; ++k) r.s[k] += x.s[k];
}
template <typename N>
__device__ void add_diag(S2<N>& r, N v) {
  r.s[0] += v;
  r.s[1] += v;
  r.s[2] += v;
}
template <typename N>
__device__ S2<N> push_forward(const T2<N>& f, const S2<N>& h) {  // tensor.hpp:332-341
  const T2<N> fh = mm(f, h);
  S2<N> r;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) r(i, j) = (fh(i, 0) * f(j, 0) + fh(i, 1) * f(j, 1)) + fh(i, 2) * f(j, 2);
  return r;
}

// ---- scalar kernels, fastscalar.hpp --------------------------------------
template <typename N>
__device__ N ln_plus_one(N x) {  // fastscalar.hpp:44-71 (16 terms, ascending-power storage)
  if (fabs(x) > N(0.5)) return d_log1p(x);
  const N y = x / (N(2) + x);
  const N y2 = y * y;
  N powers[16];
  N pw = y;
  for (int n = 0; n < 16; ++n) {
    powers[n] = pw;
    pw = pw * y2;
  }
  N sum(0);
  for (int n = 15; n >= 0; --n) sum += powers[n] * (N(1) / N(2 * n + 1));
  return N(2) * sum;
}
template <typename N>
__device__ N jpow(N jm1) {  // fastscalar.hpp:77-89, 3 Newton steps
  const N third = N(1) / N(3);
  const N four_thirds = N(4) / N(3);
  const N alpha = ((jm1 + N(2)) * jm1 + N(1)) * third;
  N beta = four_thirds - alpha;
  for (int n = 0; n < 3; ++n) {
    const N b2 = beta * beta;
    const N gamma = b2 * b2;
    beta = four_thirds * beta - alpha * gamma;
  }
  return beta;
}

// ---- kinematics and constitutive laws, constitutive.hpp ------------------
template <typename N>
struct Strain {
  T2<N> F, Finv;
  S2<N> E, bt, C, Cinv;
  N jm1, jac, i1;
};

// make_strain (constitutive.hpp:43-72); false = NonPositiveJacobian / SingularTensor
template <typename N>
__device__ bool make_strain(const T2<N>& g, bool stable, Strain<N>& s) {
  s.F = g;
  s.F(0, 0) = N(1) + g(0, 0);
  s.F(1, 1) = N(1) + g(1, 1);
  s.F(2, 2) = N(1) + g(2, 2);
  if (stable) {
    s.jm1 = det_m1(g);
    if (!(s.jm1 > N(-1))) return false;
    s.jac = N(1) + s.jm1;
    const N h(0.5);
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        const N q = (g(0, i) * g(0, j) + g(1, i) * g(1, j)) + g(2, i) * g(2, j);
        s.E(i, j) = h * ((g(i, j) + g(j, i)) + q);
        const N q2 = (g(i, 0) * g(j, 0) + g(i, 1) * g(j, 1)) + g(i, 2) * g(j, 2);
        s.bt(i, j) = h * ((g(i, j) + g(j, i)) + q2);
      }
    if (!inv(s.F, s.Finv)) return false;
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j)
        s.Cinv(i, j) = (s.Finv(i, 0) * s.Finv(j, 0) + s.Finv(i, 1) * s.Finv(j, 1)) + s.Finv(i, 2) * s.Finv(j, 2);
    s.i1 = N(3) + N(2) * trace(s.E);
  } else {
    s.jac = det(s.F);
    s.jm1 = s.jac - N(1);
    if (!(s.jm1 > N(-1))) return false;
    const T2<N> ft = tr(s.F);
    s.C = to_sym(mm(ft, s.F));
    const N h(0.5);
    for (int k = 0; k < 6; ++k) s.E.s[k] = h * (s.C.s[k] - (k < 3 ? N(1) : N(0)));
    const S2<N> ffT = to_sym(mm(s.F, ft));
    for (int k = 0; k < 6; ++k) s.bt.s[k] = h * (ffT.s[k] - (k < 3 ? N(1) : N(0)));
    if (!inv(s.F, s.Finv)) return false;
    T2<N> ci;
    if (!inv(full(s.C), ci)) return false;
    s.Cinv = sym(ci);
    s.i1 = trace(s.C);
  }
  return true;
}

template <typename N>
__device__ N half_kappa_j2m1(const Strain<N>& s, N half_k, bool stable) {  // constitutive.hpp:104-110
  if (stable) return half_k * (s.jm1 * (s.jm1 + N(2)));
  return half_k * (s.jac * s.jac - N(1));
}

template <typename N>
struct Fib {
  N istar[2], efib[2], c3[2];
};
template <typename N>
__device__ Fib<N> fiber_invariants(const Strain<N>& s, const Consts<N>& m, bool stable) {  // :117-149
  Fib<N> f;
  for (int i = 0; i < 2; ++i) {
    S2<N> mm6;
    for (int a = 0; a < 3; ++a)
      for (int b = a; b < 3; ++b) mm6(a, b) = m.m1[i][a] * m.m1[i][b];
    N gate;
    if (stable) {
      f.efib[i] = N(2) * ddot(m.h[i], s.E);
      gate = N(2) * ddot(mm6, s.E);
      f.istar[i] = N(1) + gate;
    } else {
      f.efib[i] = ddot(m.h[i], s.C) - trace(m.h[i]);
      f.istar[i] = ddot(mm6, s.C);
      gate = f.istar[i] - N(1);
    }
    const N z = m.k2 * f.efib[i] * f.efib[i];
    const N active = d_exp(z) * m.two_k1;
    f.c3[i] = gate > N(0) ? active : N(0);
  }
  return f;
}

template <typename N>
__device__ S2<N> second_pk_base(int model, const Consts<N>& m, const Strain<N>& s, N lnj, N jp, bool stable) {
  if (model == 0) {  // constitutive.hpp:197-217
    if (stable) {
      S2<N> inner = scale(N(2) * m.mu, s.E);
      add_diag(inner, N(2) * m.lam * lnj);
      return sym(mm(s.Cinv, full(inner)));
    }
    S2<N> r = scale(-(m.mu - N(2) * m.lam * lnj), s.Cinv);
    add_diag(r, m.mu);
    return r;
  }
  if (stable) {  // :218-229
    const N vol = half_kappa_j2m1(s, m.half_k, true);
    const N tre3 = trace(s.E) * (N(1) / N(3));
    S2<N> inner = scale(N(2) * m.mu * jp, s.E);
    const N dev = N(2) * m.mu * jp * tre3;
    add_diag(inner, vol - dev);
    return sym(mm(s.Cinv, full(inner)));
  }
  const N c1 = half_kappa_j2m1(s, m.half_k, false) - (m.mu / N(3)) * jp * s.i1;
  S2<N> r = scale(c1, s.Cinv);
  add_diag(r, m.mu * jp);
  return r;
}

template <typename N>
__device__ S2<N> kirchhoff_base(int model, const Consts<N>& m, const Strain<N>& s, N lnj, N jp, bool stable) {
  if (model == 0) {  // constitutive.hpp:244-264
    if (stable) {
      S2<N> r = scale(N(2) * m.mu, s.bt);
      add_diag(r, N(2) * m.lam * lnj);
      return r;
    }
    S2<N> b = scale(N(2), s.bt);
    add_diag(b, N(1));
    S2<N> r = scale(m.mu, b);
    add_diag(r, -(m.mu - N(2) * m.lam * lnj));
    return r;
  }
  if (stable) {  // :265-274
    const N vol = half_kappa_j2m1(s, m.half_k, true);
    const N trb3 = trace(s.bt) * (N(1) / N(3));
    S2<N> r = scale(N(2) * m.mu * jp, s.bt);
    add_diag(r, vol - N(2) * m.mu * jp * trb3);
    return r;
  }
  const N c1 = half_kappa_j2m1(s, m.half_k, false) - (m.mu / N(3)) * jp * s.i1;
  S2<N> b = scale(N(2), s.bt);
  add_diag(b, N(1));
  S2<N> r = scale(m.mu * jp, b);
  add_diag(r, c1);
  return r;
}

template <typename N>
struct Cache {
  N jm1, jac, lnj, jp, c1, c2, c3[2], efib[2];
  T2<N> F, Finv;
  S2<N> S, Cinv, tau, b, fh[2];
};

template <typename N>
__device__ N ln_of(const Strain<N>& s, bool stable) {
  return stable ? ln_plus_one(s.jm1) : d_log(s.jac);
}

// compute_cache (constitutive.hpp:326-377), strategy none
template <typename N>
__device__ void compute_cache(int model, const Consts<N>& m, const Strain<N>& s, bool stable, bool spatial,
                              Cache<N>& c) {
  c.jm1 = s.jm1;
  c.jac = s.jac;
  c.lnj = ln_of(s, stable);
  c.jp = model == 0 ? N(1) : jpow(s.jm1);
  if (model != 0) {
    c.c1 = half_kappa_j2m1(s, m.half_k, stable) - (m.mu / N(3)) * c.jp * s.i1;
    c.c2 = (N(2) * m.mu / N(9)) * c.jp * s.i1 + m.kappa * s.jac * s.jac;
  }
  c.c3[0] = c.c3[1] = c.efib[0] = c.efib[1] = N(0);
  if (model == 2) {
    const Fib<N> f = fiber_invariants(s, m, stable);
    for (int i = 0; i < 2; ++i) {
      c.c3[i] = f.c3[i];
      c.efib[i] = f.efib[i];
    }
  }
  c.F = s.F;
  c.Finv = s.Finv;
  c.Cinv = s.Cinv;
  if (!spatial) {
    c.S = second_pk_base(model, m, s, c.lnj, c.jp, stable);
    if (model == 2)
      for (int i = 0; i < 2; ++i) add_to(c.S, scale(c.c3[i] * c.efib[i], m.h[i]));
  } else {
    c.b = scale(N(2), s.bt);
    add_diag(c.b, N(1));
    c.tau = kirchhoff_base(model, m, s, c.lnj, c.jp, stable);
    if (model == 2)
      for (int i = 0; i < 2; ++i) {
        c.fh[i] = push_forward(s.F, m.h[i]);
        add_to(c.tau, scale(c.c3[i] * c.efib[i], c.fh[i]));
      }
  }
}

template <typename N>
__device__ S2<N> tangent_material(int model, const Consts<N>& m, const Cache<N>& c, const T2<N>& dg) {  // :381-419
  const T2<N> a = mm(c.Finv, dg);
  const N w = trace(a);
  const S2<N> sac = sym(mm(a, c.Cinv));
  S2<N> r;
  if (model == 0) {
    r = scale(N(2) * (m.mu - N(2) * m.lam * c.lnj), sac);
    add_to(r, scale(N(2) * m.lam * w, c.Cinv));
    return r;
  }
  const N q = ddot(c.F, dg);
  const N ttmj = (N(2) * m.mu / N(3)) * c.jp;
  r = scale(N(-2) * c.c1, sac);
  add_to(r, scale(c.c2 * w - ttmj * q, c.Cinv));
  add_diag(r, -ttmj * w);
  if (model == 2) {
    const S2<N> dch = sym(mm(tr(c.F), dg));
    for (int i = 0; i < 2; ++i) {
      const N hdc = N(2) * ddot(m.h[i], dch);
      const N coef = c.c3[i] * (N(2) * m.k2 * c.efib[i] * c.efib[i] + N(1)) * hdc;
      add_to(r, scale(coef, m.h[i]));
    }
  }
  return r;
}

template <typename N>
__device__ T2<N> tangent_spatial(int model, const Consts<N>& m, const Cache<N>& c, const T2<N>& dgrad) {  // :421-461
  const S2<N> xs = sym(dgrad);
  const N trx = trace(dgrad);
  S2<N> jc;
  if (model == 0) {
    jc = scale(N(2) * (m.mu - N(2) * m.lam * c.lnj), xs);
    add_diag(jc, N(2) * m.lam * trx);
  } else {
    const N bx = ddot(c.b, xs);
    const N ttmj = (N(2) * m.mu / N(3)) * c.jp;
    jc = scale(-ttmj * trx, c.b);
    add_to(jc, scale(N(-2) * c.c1, xs));
    add_diag(jc, c.c2 * trx - ttmj * bx);
    if (model == 2)
      for (int i = 0; i < 2; ++i) {
        const N fhx = ddot(c.fh[i], xs);
        const N coef = N(2) * c.c3[i] * (N(2) * m.k2 * c.efib[i] * c.efib[i] + N(1)) * fhx;
        add_to(jc, scale(coef, c.fh[i]));
      }
  }
  const T2<N> jt = full(jc);
  const T2<N> gt = mm(dgrad, c.tau);
  T2<N> r;
  for (int k = 0; k < 9; ++k) r.a[k] = jt.a[k] + gt.a[k];
  return r;
}

// SVK (stability.cpp:88-113)
template <typename N>
__device__ S2<N> svk_stress(const Consts<N>& m, const Strain<N>& s) {
  S2<N> r = scale(N(2) * m.mu, s.E);
  add_diag(r, m.lam * trace(s.E));
  return r;
}
template <typename N>
__device__ S2<N> svk_tangent(const Consts<N>& m, const Strain<N>& s, const T2<N>& dg) {
  const S2<N> de = sym(mm(tr(s.F), dg));
  S2<N> r = scale(N(2) * m.mu, de);
  add_diag(r, m.lam * trace(de));
  return r;
}

// evaluate_cell (stability.cpp:117-161); returns the entry count, 0 = invalid
template <typename N>
__device__ int evaluate_cell(int model, bool stable, bool spatial, bool tangent, const Consts<N>& m, const T2<N>& g,
                             const T2<N>& dir, N* out) {
  Strain<N> s;
  if (!make_strain(g, stable, s)) return 0;
  if (model == 3) {
    if (!tangent) {
      const S2<N> S = svk_stress(m, s);
      const S2<N> v = spatial ? push_forward(s.F, S) : S;
      for (int i = 0; i < 6; ++i) out[i] = v.s[i];
      return 6;
    }
    const S2<N> ds = svk_tangent(m, s, dir);
    if (spatial) {
      const S2<N> tau = push_forward(s.F, svk_stress(m, s));
      const T2<N> x = mm(dir, s.Finv);
      const T2<N> a = full(push_forward(s.F, ds));
      const T2<N> b = mm(x, tau);
      for (int i = 0; i < 9; ++i) out[i] = a.a[i] + b.a[i];
      return 9;
    }
    for (int i = 0; i < 6; ++i) out[i] = ds.s[i];
    return 6;
  }
  if (!tangent) {
    // second_pk / kirchhoff (constitutive.hpp:287-322)
    const N lnj = ln_of(s, stable);
    const N jp = model == 0 ? N(1) : jpow(s.jm1);
    if (!spatial) {
      S2<N> r = second_pk_base(model, m, s, lnj, jp, stable);
      if (model == 2) {
        const Fib<N> f = fiber_invariants(s, m, stable);
        for (int i = 0; i < 2; ++i) add_to(r, scale(f.c3[i] * f.efib[i], m.h[i]));
      }
      for (int i = 0; i < 6; ++i) out[i] = r.s[i];
    } else {
      S2<N> r = kirchhoff_base(model, m, s, lnj, jp, stable);
      if (model == 2) {
        const Fib<N> f = fiber_invariants(s, m, stable);
        for (int i = 0; i < 2; ++i) add_to(r, scale(f.c3[i] * f.efib[i], push_forward(s.F, m.h[i])));
      }
      for (int i = 0; i < 6; ++i) out[i] = r.s[i];
    }
    return 6;
  }
  Cache<N> c;
  compute_cache(model, m, s, stable, spatial, c);
  if (!spatial) {
    const S2<N> v = tangent_material(model, m, c, dir);
    for (int i = 0; i < 6; ++i) out[i] = v.s[i];
    return 6;
  }
  const T2<N> v = tangent_spatial(model, m, c, dir);
  for (int i = 0; i < 9; ++i) out[i] = v.a[i];
  return 9;
}

// ---- SweepRng (stability.cpp:47-76) -----------------------------------------
__device__ __forceinline__ uint64_t splitmix_next(uint64_t& state) {
  state += 0x9e3779b97f4a7c15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t stream(uint64_t seed, uint64_t is, uint64_t sample) {
  uint64_t s = seed ^ (0x632be59bd9b4e019ull * (is + 1));
  const uint64_t mixed = splitmix_next(s);
  uint64_t s2 = mixed ^ (0x9e3779b97f4a7c15ull * (sample + 1));
  return splitmix_next(s2);
}
__device__ __forceinline__ double next01(uint64_t& st) { return (double)(splitmix_next(st) >> 11) * 0x1.0p-53; }
__device__ void sample_gradient(uint64_t& st, double eps, T2<double>& g) {
  for (int i = 0; i < 9; ++i) {
    const double mag = eps * (0.1 + 0.9 * next01(st));
    const double sgn = next01(st) < 0.5 ? -1.0 : 1.0;
    g.a[i] = sgn * mag;
  }
}

struct SweepArgs {
  const double* scales;
  int n_scales, samples;
  uint64_t seed;
  Consts<double> md;
  Consts<float> mf;
  unsigned long long* max_bits;  // n_scales * kCells, bit pattern of the max error (>= 0)
  unsigned long long* invalid;   // n_scales * kCells
};

__global__ void __launch_bounds__(128) sweep_kernel(const SweepArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.n_scales * a.samples) return;
  const int is = (int)(t / a.samples), sample = (int)(t % a.samples);
  uint64_t st = stream(a.seed, (uint64_t)is, (uint64_t)sample);
  T2<double> g64, d64;
  sample_gradient(st, a.scales[is], g64);
  sample_gradient(st, a.scales[is], d64);
  T2<float> g32, d32;
  for (int i = 0; i < 9; ++i) {
    g32.a[i] = (float)g64.a[i];
    d32.a[i] = (float)d64.a[i];
  }
  int cell = 0;
  for (int model = 0; model < 4; ++model)
    for (int form = 0; form < 4; ++form)
      for (int q = 0; q < 2; ++q, ++cell) {
        const bool stable = form & 1, spatial = form >= 2;
        double v64[9];
        float v32[9];
        const int n64 = evaluate_cell<double>(model, stable, spatial, q == 1, a.md, g64, d64, v64);
        const int n32 = n64 ? evaluate_cell<float>(model, stable, spatial, q == 1, a.mf, g32, d32, v32) : 0;
        bool bad = n64 == 0 || n32 != n64;
        if (!bad)
          for (int i = 0; i < n64; ++i)
            if (!isfinite(v64[i]) || !isfinite((double)v32[i])) bad = true;
        const int64_t slot = (int64_t)is * kCells + cell;
        if (bad) {
          atomicAdd(&a.invalid[slot], 1ull);
          continue;
        }
        double denom = 1e-30;
        for (int i = 0; i < n64; ++i) denom = fmax(denom, fabs(v64[i]));
        double err = 0.0;
        for (int i = 0; i < n64; ++i) err = fmax(err, fabs(v64[i] - (double)v32[i]) / denom);
        atomicMax(&a.max_bits[slot], (unsigned long long)__double_as_longlong(err));
      }
}

template <typename N>
Consts<N> consts(const emfgpu_material& p, const double h[2][6], const double m1[2][3]) {
  Consts<N> c;
  c.mu = N(p.mu);
  c.lam = N(p.lambda);
  c.half_k = N(0.5 * p.kappa_b);
  c.kappa = N(p.kappa_b);
  c.k2 = N(p.k2);
  c.two_k1 = N(2.0 * p.k1);
  for (int f = 0; f < 2; ++f) {
    for (int k = 0; k < 6; ++k) c.h[f].s[k] = N(h[f][k]);
    for (int k = 0; k < 3; ++k) c.m1[f][k] = N(m1[f][k]);
  }
  return c;
}

}  // namespace lab

void run_stability_sweep(const double* scales, int n_scales, int samples, uint64_t seed, const emfgpu_material& p,
                         const double h[2][6], const double m1[2][3], double* max_rel_error, int64_t* count_invalid) {
  const int64_t cells = (int64_t)n_scales * lab::kCells;
  double* d_scales = nullptr;
  unsigned long long *d_max = nullptr, *d_inv = nullptr;
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("stability sweep: ") + cudaGetErrorString(e));
  };
  ck(cudaMalloc(&d_scales, sizeof(double) * n_scales));
  ck(cudaMalloc(&d_max, sizeof(unsigned long long) * cells));
  ck(cudaMalloc(&d_inv, sizeof(unsigned long long) * cells));
  ck(cudaMemcpy(d_scales, scales, sizeof(double) * n_scales, cudaMemcpyHostToDevice));
  ck(cudaMemset(d_max, 0, sizeof(unsigned long long) * cells));  // bits of +0.0
  ck(cudaMemset(d_inv, 0, sizeof(unsigned long long) * cells));
  lab::SweepArgs a;
  a.scales = d_scales;
  a.n_scales = n_scales;
  a.samples = samples;
  a.seed = seed;
  a.md = lab::consts<double>(p, h, m1);
  a.mf = lab::consts<float>(p, h, m1);
  a.max_bits = d_max;
  a.invalid = d_inv;
  const int64_t threads = (int64_t)n_scales * samples;
  if (threads > 0) lab::sweep_kernel<<<(unsigned)((threads + 127) / 128), 128>>>(a);
  ck(cudaGetLastError());
  std::vector<unsigned long long> hm(cells), hi(cells);
  ck(cudaMemcpy(hm.data(), d_max, sizeof(unsigned long long) * cells, cudaMemcpyDeviceToHost));
  ck(cudaMemcpy(hi.data(), d_inv, sizeof(unsigned long long) * cells, cudaMemcpyDeviceToHost));
  for (int64_t c = 0; c < cells; ++c) {
    std::memcpy(&max_rel_error[c], &hm[c], sizeof(double));
    count_invalid[c] = (int64_t)hi[c];
  }
  cudaFree(d_scales);
  cudaFree(d_max);
  cudaFree(d_inv);
}

}  // namespace emfgpu
