/* TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
 *
 * emf_oracle.c: plain-C restatement of the reference hot path:
 *   1D basis / GLL + Gauss rules       proj/src/mesh.cpp:14-120
 *   lattice coordinates, J0 per qp     proj/src/mesh.cpp:138-211
 *   structure tensors (fiber)          proj/src/material.cpp:50-82,
 *                                      proj/src/fastscalar.cpp:19-96
 *   update_linearization (double)      proj/include/elastmf/operator.hpp:643-770
 *   apply_tangent (material domain)    operator.hpp:468-530, 597-621
 *   compute_diagonal                   operator.hpp:772-878
 *   TransferOp / LatticeMap1D          proj/include/elastmf/mesh.hpp:190-289,
 *                                      proj/src/mesh.cpp:248-288
 *   estimate_eigenvalues (Lanczos)     proj/include/elastmf/solver.hpp:235-308
 *   ChebyshevSmoother                  solver.hpp:312-362
 * It is pinned bit-for-bit against oracle/_ref (the reference compiled from
 * its own sources) in tests/test_oracle.py, and serves as the parity checker
 * of the CUDA path.  Generalisations beyond the reference are flagged "EXT":
 * (nx,ny,nz) boxes and per-axis extents (the reference has one n), node
 * coordinate override for maps the reference lacks (SURVEY §8(c) gap 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXP 8
#define ORC_MAXN (ORC_MAXP + 1)
#define ORC_MAXN3 (ORC_MAXN * ORC_MAXN * ORC_MAXN)

enum { ORC_NONE = 0, ORC_SCALAR = 1, ORC_TENSOR = 2 };

/* cached per-qp fields (double; rounded to Number on load, operator.hpp:720-766) */
enum {
  ORC_C_LNJ = 0, ORC_C_JM1, ORC_C_JP, ORC_C_C1, ORC_C_C2, ORC_C_C3, ORC_C_IS = ORC_C_C3 + 2,
  ORC_C_EF = ORC_C_IS + 2, ORC_C_F = ORC_C_EF + 2, ORC_C_FINV = ORC_C_F + 9, ORC_C_S = ORC_C_FINV + 9,
  ORC_C_CINV = ORC_C_S + 6,
  /* spatial domain (operator.hpp:139-143): 1/J, J_t, tau, b, F H_i F^T */
  ORC_C_INVJ = ORC_C_CINV + 6, ORC_C_JT = ORC_C_INVJ + 1, ORC_C_TAU = ORC_C_JT + 9, ORC_C_B = ORC_C_TAU + 6,
  ORC_C_FH = ORC_C_B + 6, ORC_CACHE_STRIDE = ORC_C_FH + 12
};

typedef struct {
  int p, n;
  double nodes[ORC_MAXN], qpts[ORC_MAXN], qwts[ORC_MAXN];
  double B[ORC_MAXN * ORC_MAXN], D[ORC_MAXN * ORC_MAXN], Bt[ORC_MAXN * ORC_MAXN], Dt[ORC_MAXN * ORC_MAXN];
} orc_basis;

typedef struct {
  int model; /* 0 cnh, 1 inh, 2 fiber */
  double mu, lambda, kappa, k1, k2;
  double h[2][6], m1[2][3]; /* structure tensors H4/H6, mean directions */
} orc_material;

typedef struct orc_op {
  int nx, ny, nz, p, nn3, nq3, mx, my, mz;
  int64_t ndofs, nel;
  orc_basis basis;
  orc_material mat;
  int strategy, precision;
  int spatial; /* Domain::spatial (material.hpp:18) */
  double* jac;      /* nel*nq3*9, owned */
  uint8_t* mask;    /* ndofs, owned */
  double* uk;       /* ndofs, owned */
  double* cache;    /* nel*nq3*ORC_CACHE_STRIDE when strategy != none */
  double* hq;       /* optional per-qp H4,H6 (12 fields, SoA) */
  double* m1q;      /* optional per-qp M1_4,M1_6 (6 fields, SoA) */
  int linearized;
} orc_op;

/* EXT (SURVEY §8(c) gap 2): fibre structure tensors per quadrature point.
 * Without a frame field this is the operator's constant material. */
static orc_material orc_mat_at(const orc_op* op, int64_t at) {
  orc_material m = op->mat;
  if (op->hq) {
    const int64_t st = op->nel * op->nq3;
    for (int f = 0; f < 2; ++f) {
      for (int k = 0; k < 6; ++k) m.h[f][k] = op->hq[(6 * f + k) * st + at];
      for (int k = 0; k < 3; ++k) m.m1[f][k] = op->m1q[(3 * f + k) * st + at];
    }
  }
  return m;
}

/* ---- quadrature / basis: mesh.cpp:14-120 ------------------------------- */
static const double kPi = 3.14159265358979323846;

static double legendre(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return p0;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}
static double legendre_derivative(int n, double x) {
  if (n == 0) return 0.0;
  const double pn = legendre(n, x);
  const double pn1 = legendre(n - 1, x);
  return n * (pn1 - x * pn) / (1.0 - x * x);
}
static int cmp_d(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
static void gauss_legendre(int n, double* pts, double* wts) {
  for (int i = 0; i < n; ++i) {
    double x = cos(kPi * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      const double f = legendre(n, x);
      const double df = legendre_derivative(n, x);
      const double dx = f / df;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    pts[i] = x;
  }
  qsort(pts, n, sizeof(double), cmp_d);
  for (int i = 0; i < n; ++i) {
    const double df = legendre_derivative(n, pts[i]);
    wts[i] = 2.0 / ((1.0 - pts[i] * pts[i]) * df * df);
  }
}
static void gauss_lobatto(int n, double* pts) {
  pts[0] = -1.0;
  pts[n - 1] = 1.0;
  const int m = n - 1;
  for (int i = 1; i < m; ++i) {
    double x = cos(kPi * (m - i) / m);
    for (int it = 0; it < 100; ++it) {
      const double g = legendre_derivative(m, x);
      const double gp = (2.0 * x * g - m * (m + 1.0) * legendre(m, x)) / (1.0 - x * x);
      const double dx = g / gp;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    pts[i] = x;
  }
  qsort(pts, n, sizeof(double), cmp_d);
}
static double lagrange_value(const double* nodes, int nn, int i, double x) {
  double v = 1.0;
  for (int k = 0; k < nn; ++k)
    if (k != i) v *= (x - nodes[k]) / (nodes[i] - nodes[k]);
  return v;
}
static double lagrange_derivative(const double* nodes, int nn, int i, double x) {
  double sum = 0.0;
  for (int m = 0; m < nn; ++m) {
    if (m == i) continue;
    double prod = 1.0 / (nodes[i] - nodes[m]);
    for (int k = 0; k < nn; ++k) {
      if (k == i || k == m) continue;
      prod *= (x - nodes[k]) / (nodes[i] - nodes[k]);
    }
    sum += prod;
  }
  return sum;
}
static void basis_init(orc_basis* b, int p) {
  b->p = p;
  b->n = p + 1;
  const int n = p + 1;
  gauss_lobatto(n, b->nodes);
  gauss_legendre(n, b->qpts, b->qwts);
  for (int q = 0; q < n; ++q)
    for (int i = 0; i < n; ++i) {
      b->B[q * n + i] = lagrange_value(b->nodes, n, i, b->qpts[q]);
      b->D[q * n + i] = lagrange_derivative(b->nodes, n, i, b->qpts[q]);
      b->Bt[i * n + q] = b->B[q * n + i];
      b->Dt[i * n + q] = b->D[q * n + i];
    }
}

int orc_basis_tables(int p, double* nodes, double* qpts, double* qwts, double* B, double* D) {
  if (p < 1 || p > ORC_MAXP) return 1;
  orc_basis b;
  basis_init(&b, p);
  const int n = p + 1;
  memcpy(nodes, b.nodes, n * sizeof(double));
  memcpy(qpts, b.qpts, n * sizeof(double));
  memcpy(qwts, b.qwts, n * sizeof(double));
  memcpy(B, b.B, n * n * sizeof(double));
  memcpy(D, b.D, n * n * sizeof(double));
  return 0;
}

/* ---- fibre structure tensors: fastscalar.cpp:19-96, material.cpp:50-82 -- */
static const double kSeriesEps = 1e-17;
static double bessel_i0_series(double a) {
  const double t = 0.25 * a * a;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 200; ++k) {
    term *= t / ((double)k * k);
    sum += term;
    if (term < kSeriesEps * sum) break;
  }
  return sum;
}
static double bessel_i1_series(double a) {
  const double t = 0.25 * a * a;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 200; ++k) {
    term *= t / ((double)k * (k + 1));
    sum += term;
    if (term < kSeriesEps * sum) break;
  }
  return 0.5 * a * sum;
}
static double bessel_asymptotic_sum(double a, int nu) {
  const double mu = 4.0 * nu * nu;
  double term = 1.0, sum = 1.0, prev_mag = 1.0;
  for (int k = 0; k < 400; ++k) {
    const double c = 2.0 * k + 1.0;
    const double next = -term * (mu - c * c) / (8.0 * a * (k + 1));
    if (fabs(next) >= prev_mag) break;
    sum += next;
    prev_mag = fabs(next);
    term = next;
    if (prev_mag < kSeriesEps * fabs(sum)) break;
  }
  return sum;
}
static double bessel_ratio(double a) {
  if (a == 0.0) return 0.0;
  if (a <= 15.0) return bessel_i1_series(a) / bessel_i0_series(a);
  return bessel_asymptotic_sum(a, 1) / bessel_asymptotic_sum(a, 0);
}
static double erf_approx(double x) {
  const double two_over_sqrt_pi = 1.1283791670955125739;
  if (x <= 4.0) {
    const double x2 = x * x;
    double t = x, sum = x;
    for (int n = 1; n < 120; ++n) {
      t *= -x2 / n;
      const double contrib = t / (2.0 * n + 1.0);
      sum += contrib;
      if (fabs(contrib) < kSeriesEps * fabs(sum) + 1e-300) break;
    }
    return two_over_sqrt_pi * sum;
  }
  const double ix2 = 1.0 / (2.0 * x * x);
  double term = 1.0, sum = 1.0, prev_mag = 1.0;
  for (int k = 1; k < 60; ++k) {
    const double next = -term * (2.0 * k - 1.0) * ix2;
    if (fabs(next) >= prev_mag) break;
    sum += next;
    prev_mag = fabs(next);
    term = next;
    if (prev_mag < kSeriesEps * fabs(sum)) break;
  }
  const double erfc = exp(-x * x) / (x * 1.7724538509055160273) * sum;
  return 1.0 - erfc;
}
static int sidx(int i, int j) { return (i == j) ? i : 2 + i + j; }

/* params = {mu, lambda, kappa, k1, k2, a, b, phi, e1[3], e2[3], e3[3]}
 * out    = {h4[6], h6[6], m1_4[3], m1_6[3], h11, h22, h33} */
int orc_structure_tensors(const double* prm, double* out) {
  const double a = prm[5], b = prm[6], phi = prm[7];
  const double* e1 = prm + 8;
  const double* e2 = prm + 11;
  const double* e3 = prm + 14;
  if (a <= 0 || b <= 0) return 1;
  const double h33 = 1.0 / (4.0 * b) - exp(-2.0 * b) / (sqrt(2.0 * kPi * b) * erf_approx(sqrt(2.0 * b)));
  const double ratio = bessel_ratio(a);
  const double h11 = 0.5 * (1.0 - h33) * (1.0 + ratio);
  const double h22 = 0.5 * (1.0 - h33) * (1.0 - ratio);
  const double c = cos(phi), s = sin(phi);
  double m1p[3], m2p[3], m1m[3], m2m[3];
  for (int k = 0; k < 3; ++k) {
    m1p[k] = c * e1[k] + s * e2[k];
    m2p[k] = -s * e1[k] + c * e2[k];
    m1m[k] = c * e1[k] + (-s) * e2[k];
    m2m[k] = s * e1[k] + c * e2[k];
  }
  const double* mm1[2] = {m1p, m1m};
  const double* mm2[2] = {m2p, m2m};
  for (int f = 0; f < 2; ++f) {
    double* h = out + 6 * f;
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) h[sidx(i, j)] = h11 * (mm1[f][i] * mm1[f][j]);
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) h[sidx(i, j)] += h22 * (mm2[f][i] * mm2[f][j]);
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) h[sidx(i, j)] += h33 * (e3[i] * e3[j]);
  }
  for (int k = 0; k < 3; ++k) {
    out[12 + k] = m1p[k];
    out[15 + k] = m1m[k];
  }
  out[18] = h11;
  out[19] = h22;
  out[20] = h33;
  return 0;
}

/* ---- lattice geometry: mesh.cpp:138-211 (EXT: nx,ny,nz, per-axis extent) */
void orc_lattice_axis(int n_el, int p, double extent, double* out) {
  double nodes[ORC_MAXN];
  gauss_lobatto(p + 1, nodes);
  const double h = extent / n_el;
  for (int idx = 0; idx <= n_el * p; ++idx) {
    int e = idx / p;
    if (e > n_el - 1) e = n_el - 1;
    const int l = idx - e * p;
    out[idx] = (e + 0.5 * (nodes[l] + 1.0)) * h;
  }
}

/* map 0: the reference DeformMap (mesh.cpp:128-136) with amplitude prm[0] and
 * extent prm[1]; map 1 (EXT, BASELINE cfg2): x' = x + prm[0] sin(2 pi y) e_x. */
int orc_lattice_coords(int nx, int ny, int nz, int p, const double* extent, int map, const double* prm,
                       double* coords) {
  const int mx = nx * p + 1, my = ny * p + 1, mz = nz * p + 1;
  double* ax = (double*)malloc(sizeof(double) * mx);
  double* ay = (double*)malloc(sizeof(double) * my);
  double* az = (double*)malloc(sizeof(double) * mz);
  orc_lattice_axis(nx, p, extent[0], ax);
  orc_lattice_axis(ny, p, extent[1], ay);
  orc_lattice_axis(nz, p, extent[2], az);
  for (int c = 0; c < mz; ++c)
    for (int b = 0; b < my; ++b)
      for (int a = 0; a < mx; ++a) {
        double x = ax[a], y = ay[b], z = az[c];
        double r0 = x, r1 = y, r2 = z;
        if (map == 0 && prm[0] != 0.0) {
          const double s = kPi / prm[1];
          const double amp = prm[0] * prm[1];
          r0 += amp * sin(s * y) * sin(s * z);
          r1 += amp * sin(s * x) * sin(s * z);
          r2 += amp * sin(s * x) * sin(s * y);
        } else if (map == 1) {
          r0 += prm[0] * sin(2.0 * kPi * y);
        }
        const int64_t node = ((int64_t)c * my + b) * mx + a;
        coords[3 * node] = r0;
        coords[3 * node + 1] = r1;
        coords[3 * node + 2] = r2;
      }
  free(ax);
  free(ay);
  free(az);
  return 0;
}

void orc_element_nodes(const orc_op* op, int64_t e, int64_t* out) {
  const int i = (int)(e % op->nx), j = (int)((e / op->nx) % op->ny), k = (int)(e / ((int64_t)op->nx * op->ny));
  const int p = op->p;
  int idx = 0;
  for (int c = 0; c <= p; ++c)
    for (int b = 0; b <= p; ++b)
      for (int a = 0; a <= p; ++a)
        out[idx++] = ((int64_t)(k * p + c) * op->my + (j * p + b)) * op->mx + (i * p + a);
}

#define R double
#define SFX(x) x##_d
#include "emf_oracle_impl.h"
#undef R
#undef SFX
#define R float
#define SFX(x) x##_f
#include "emf_oracle_impl.h"
#undef R
#undef SFX

/* J0 per qp via the reference's sweeps, mesh.cpp:162-186. Returns nonzero if
 * a mapping determinant is not positive (DegenerateMapping, :187-196). */
static int compute_jacobians(orc_op* op, const double* coords) {
  int err = 0;
#pragma omp parallel
  {
    scratch_d* s = (scratch_d*)malloc(sizeof(scratch_d));
#pragma omp for schedule(static)
    for (int64_t e = 0; e < op->nel; ++e) {
      int64_t nodes[ORC_MAXN3];
      orc_element_nodes(op, e, nodes);
      for (int comp = 0; comp < 3; ++comp) {
        for (int l = 0; l < op->nn3; ++l) s->loc[0][l] = coords[3 * nodes[l] + comp];
        grad_qp_d(&op->basis, s->loc[0], s->work, s->g[0][0], s->g[0][1], s->g[0][2]);
        for (int q = 0; q < op->nq3; ++q) {
          double* J = op->jac + (e * op->nq3 + q) * 9;
          J[comp * 3 + 0] = s->g[0][0][q];
          J[comp * 3 + 1] = s->g[0][1][q];
          J[comp * 3 + 2] = s->g[0][2][q];
        }
      }
      for (int q = 0; q < op->nq3; ++q) {
        const double* J = op->jac + (e * op->nq3 + q) * 9;
        const double d = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                         J[2] * (J[3] * J[7] - J[4] * J[6]);
        if (!(d > 0.0)) {
#pragma omp atomic write
          err = 1;
        }
      }
    }
    free(s);
  }
  return err;
}

/* ---- operator handle ----------------------------------------------------- */
orc_op* orc_op_create(int nx, int ny, int nz, int p, const double* coords, int faces, int model,
                      const double* prm, int strategy, int precision) {
  if (p < 1 || p > ORC_MAXP) return NULL;
  orc_op* op = (orc_op*)calloc(1, sizeof(orc_op));
  op->nx = nx;
  op->ny = ny;
  op->nz = nz;
  op->p = p;
  op->mx = nx * p + 1;
  op->my = ny * p + 1;
  op->mz = nz * p + 1;
  op->nn3 = (p + 1) * (p + 1) * (p + 1);
  op->nq3 = op->nn3;
  op->nel = (int64_t)nx * ny * nz;
  op->ndofs = 3 * (int64_t)op->mx * op->my * op->mz;
  basis_init(&op->basis, p);
  op->mat.model = model;
  op->mat.mu = prm[0];
  op->mat.lambda = prm[1];
  op->mat.kappa = prm[2];
  op->mat.k1 = prm[3];
  op->mat.k2 = prm[4];
  if (model == 2) {
    double st[21];
    if (orc_structure_tensors(prm, st)) {
      free(op);
      return NULL;
    }
    for (int f = 0; f < 2; ++f) {
      for (int k = 0; k < 6; ++k) op->mat.h[f][k] = st[6 * f + k];
      for (int k = 0; k < 3; ++k) op->mat.m1[f][k] = st[12 + 3 * f + k];
    }
  }
  op->strategy = strategy;
  op->precision = precision;
  op->jac = (double*)malloc(sizeof(double) * op->nel * op->nq3 * 9);
  if (compute_jacobians(op, coords)) {
    free(op->jac);
    free(op);
    return NULL;
  }
  op->mask = (uint8_t*)calloc(op->ndofs, 1);
  for (int c = 0; c < op->mz; ++c)
    for (int b = 0; b < op->my; ++b)
      for (int a = 0; a < op->mx; ++a) {
        const int on = ((faces & 1) && a == 0) || ((faces & 2) && a == op->mx - 1) || ((faces & 4) && b == 0) ||
                       ((faces & 8) && b == op->my - 1) || ((faces & 16) && c == 0) ||
                       ((faces & 32) && c == op->mz - 1);
        if (on) {
          const int64_t node = ((int64_t)c * op->my + b) * op->mx + a;
          op->mask[3 * node] = op->mask[3 * node + 1] = op->mask[3 * node + 2] = 1;
        }
      }
  op->uk = (double*)calloc(op->ndofs, sizeof(double));
  return op;
}

void orc_op_destroy(orc_op* op) {
  if (!op) return;
  free(op->hq);
  free(op->m1q);
  free(op->jac);
  free(op->mask);
  free(op->uk);
  free(op->cache);
  free(op);
}

int64_t orc_op_ndofs(const orc_op* op) { return op->ndofs; }
/* Formulation::domain (material.hpp:18-23): 0 material, 1 spatial; before linearize. */
void orc_op_set_domain(orc_op* op, int spatial) {
  op->spatial = spatial;
  op->linearized = 0;
}
void orc_op_jacobians(const orc_op* op, double* out) { memcpy(out, op->jac, sizeof(double) * op->nel * op->nq3 * 9); }
void orc_op_mask(const orc_op* op, uint8_t* out) { memcpy(out, op->mask, op->ndofs); }

/* update_linearization operator.hpp:643-770 (material domain). On det F <= 0
 * returns 3 and the first failing (element, qpoint) in element order. */
int orc_op_linearize(orc_op* op, const double* u, int64_t* bad_e, int* bad_q) {
  memcpy(op->uk, u, sizeof(double) * op->ndofs);
  free(op->cache);
  op->cache = NULL;
  if (op->strategy != ORC_NONE || op->spatial)
    op->cache = (double*)calloc(op->nel * op->nq3 * ORC_CACHE_STRIDE, sizeof(double));
  int64_t first = INT64_MAX;
#pragma omp parallel
  {
    scratch_d* s = (scratch_d*)malloc(sizeof(scratch_d));
#pragma omp for schedule(static) reduction(min : first)
    for (int64_t e = 0; e < op->nel; ++e) {
      gather_d(op, u, e, s->uk);
      for (int c = 0; c < 3; ++c) grad_qp_d(&op->basis, s->uk[c], s->work, s->gk[c][0], s->gk[c][1], s->gk[c][2]);
      for (int q = 0; q < op->nq3; ++q) {
        const double* J0 = op->jac + (e * op->nq3 + q) * 9;
        double j0inv[9], gref[9], gk[9];
        const int64_t at = e * op->nq3 + q;
        for (int c = 0; c < 3; ++c)
          for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->gk[c][d][q];
        if (inverse_d(J0, j0inv)) {
          if (at < first) first = at;
          continue;
        }
        mm_d(gref, j0inv, gk);
        qpc_d c;
        const orc_material mq = orc_mat_at(op, at);
        if (compute_cache_d(&mq, gk, &c)) {
          if (at < first) first = at;
          continue;
        }
        second_pk_d(&mq, &c, c.S);
        if (op->spatial) {
          /* operator.hpp:736-744: 1/J and J_t = J0 + Grad_xi u_k, det J_t > 0 */
          double* sc = op->cache + at * ORC_CACHE_STRIDE;
          double jt[9];
          for (int k = 0; k < 9; ++k) jt[k] = J0[k] + gref[k];
          if (!(det_d(jt) > 0)) {
            if (at < first) first = at;
            continue;
          }
          spatial_cell_d(&mq, &c);
          sc[ORC_C_INVJ] = 1.0 / c.jac;
          for (int k = 0; k < 9; ++k) sc[ORC_C_JT + k] = jt[k];
          for (int k = 0; k < 6; ++k) {
            sc[ORC_C_TAU + k] = c.tau[k];
            sc[ORC_C_B + k] = c.b[k];
            sc[ORC_C_FH + k] = c.fh[0][k];
            sc[ORC_C_FH + 6 + k] = c.fh[1][k];
          }
        }
        if (op->cache) {
          double* sc = op->cache + at * ORC_CACHE_STRIDE;
          sc[ORC_C_LNJ] = c.lnj;
          sc[ORC_C_JM1] = c.jm1;
          sc[ORC_C_JP] = c.jp;
          sc[ORC_C_C1] = c.c1;
          sc[ORC_C_C2] = c.c2;
          for (int f = 0; f < 2; ++f) {
            sc[ORC_C_C3 + f] = c.c3[f];
            sc[ORC_C_IS + f] = c.istar[f];
            sc[ORC_C_EF + f] = c.efib[f];
          }
          for (int k = 0; k < 9; ++k) {
            sc[ORC_C_F + k] = c.F[k];
            sc[ORC_C_FINV + k] = c.Finv[k];
          }
          for (int k = 0; k < 6; ++k) {
            sc[ORC_C_S + k] = c.S[k];
            sc[ORC_C_CINV + k] = c.Cinv[k];
          }
        }
      }
    }
    free(s);
  }
  if (first != INT64_MAX) {
    if (bad_e) *bad_e = first / op->nq3;
    if (bad_q) *bad_q = (int)(first % op->nq3);
    op->linearized = 0;
    return 3;
  }
  op->linearized = 1;
  return 0;
}

int orc_op_apply(const orc_op* op, const void* x, void* y) {
  if (!op->linearized) return 4;
  return op->precision == 64 ? apply_d(op, (const double*)x, (double*)y) : apply_f(op, (const float*)x, (float*)y);
}

int orc_op_diagonal(const orc_op* op, void* d, int64_t* n_bad) {
  if (!op->linearized) return 4;
  return op->precision == 64 ? diagonal_d(op, (double*)d, n_bad) : diagonal_f(op, (float*)d, n_bad);
}

/* build_load_vector operator.hpp:925-1003, pressure part: -p N traction on
 * face `face` (0..5 = -x,+x,-y,+y,-z,+z) of the reference geometry `coords`,
 * (p+1)^2 Gauss points per face element, accumulated in double. */
void orc_pressure_load(const orc_op* op, const double* coords, double pressure, int face, double* load) {
  const orc_basis* b = &op->basis;
  const int p = op->p, nn = p + 1, nq = b->n;
  const int axis = face / 2, t1 = (axis + 1) % 3, t2 = (axis + 2) % 3, upper = face % 2 == 1;
  const int ne[3] = {op->nx, op->ny, op->nz};
  for (int64_t i = 0; i < op->ndofs; ++i) load[i] = 0.0;
  if (pressure == 0.0) return;
  int64_t nodes[ORC_MAXN3];
  for (int ej = 0; ej < ne[t2]; ++ej)
    for (int ei = 0; ei < ne[t1]; ++ei) {
      int idx[3];
      idx[axis] = upper ? ne[axis] - 1 : 0;
      idx[t1] = ei;
      idx[t2] = ej;
      orc_element_nodes(op, ((int64_t)idx[2] * op->ny + idx[1]) * op->nx + idx[0], nodes);
      const int lface = upper ? p : 0;
      for (int q2 = 0; q2 < nq; ++q2)
        for (int q1 = 0; q1 < nq; ++q1) {
          double x[3] = {0, 0, 0}, g1[3] = {0, 0, 0}, g2[3] = {0, 0, 0};
          for (int a2 = 0; a2 < nn; ++a2)
            for (int a1 = 0; a1 < nn; ++a1) {
              const double v1 = b->B[q1 * nn + a1], d1 = b->D[q1 * nn + a1];
              const double v2 = b->B[q2 * nn + a2], d2 = b->D[q2 * nn + a2];
              int loc[3];
              loc[axis] = lface;
              loc[t1] = a1;
              loc[t2] = a2;
              const int64_t g = nodes[(loc[2] * nn + loc[1]) * nn + loc[0]];
              for (int c = 0; c < 3; ++c) {
                const double xc = coords[3 * g + c];
                x[c] += v1 * v2 * xc;
                g1[c] += d1 * v2 * xc;
                g2[c] += v1 * d2 * xc;
              }
            }
          const double nr[3] = {g1[1] * g2[2] - g1[2] * g2[1], g1[2] * g2[0] - g1[0] * g2[2],
                                g1[0] * g2[1] - g1[1] * g2[0]};
          const double sgn = upper ? 1.0 : -1.0;
          const double area = sqrt(nr[0] * nr[0] + nr[1] * nr[1] + nr[2] * nr[2]);
          const double unit[3] = {sgn * nr[0] / area, sgn * nr[1] / area, sgn * nr[2] / area};
          const double h[3] = {-pressure * unit[0], -pressure * unit[1], -pressure * unit[2]};
          const double w = b->qwts[q1] * b->qwts[q2] * area;
          for (int a2 = 0; a2 < nn; ++a2)
            for (int a1 = 0; a1 < nn; ++a1) {
              const double phi = b->B[q1 * nn + a1] * b->B[q2 * nn + a2];
              int loc[3];
              loc[axis] = lface;
              loc[t1] = a1;
              loc[t2] = a2;
              const int64_t g = nodes[(loc[2] * nn + loc[1]) * nn + loc[0]];
              for (int c = 0; c < 3; ++c) load[3 * g + c] += phi * w * h[c];
            }
        }
    }
}

/* evaluate_residual with a face pressure; u, r in the op's precision. */
int orc_op_residual(const orc_op* op, const double* coords, const void* u, double pressure, int face,
                    double load_scale, void* r) {
  double* load = (double*)malloc(sizeof(double) * op->ndofs);
  orc_pressure_load(op, coords, pressure, face, load);
  const int err = op->precision == 64 ? residual_d(op, (const double*)u, load, load_scale, (double*)r)
                                      : residual_f(op, (const float*)u, load, load_scale, (float*)r);
  free(load);
  return err;
}

int orc_op_chebyshev(const orc_op* op, const void* diag, double lmax_est, int degree, double range_factor,
                     double safety, const void* b, void* x, int zero_start) {
  if (!op->linearized) return 4;
  if (op->precision == 64)
    return chebyshev_d(op, (const double*)diag, lmax_est, degree, range_factor, safety, (const double*)b,
                       (double*)x, zero_start);
  return chebyshev_f(op, (const float*)diag, lmax_est, degree, range_factor, safety, (const float*)b, (float*)x,
                     zero_start);
}

/* ---- Lanczos: solver.hpp:209-308 ---------------------------------------- */
static uint64_t splitmix64(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double uniform01(uint64_t* state) { return (double)(splitmix64(state) >> 11) * 0x1.0p-53; }
static double dot_d(const double* a, const double* b, int64_t n) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static int sturm_count(const double* alpha, const double* beta, int n, double sigma) {
  int count = 0;
  double d = alpha[0] - sigma;
  if (d < 0) ++count;
  for (int i = 1; i < n; ++i) {
    const double b2 = beta[i - 1] * beta[i - 1];
    d = alpha[i] - sigma - b2 / (d == 0 ? 1e-300 : d);
    if (d < 0) ++count;
  }
  return count;
}
static double tridiag_extreme(const double* alpha, const double* beta, int n, int largest) {
  double lo = alpha[0], hi = alpha[0];
  for (int i = 0; i < n; ++i) {
    const double bl = i > 0 ? fabs(beta[i - 1]) : 0.0;
    const double br = i < n - 1 ? fabs(beta[i]) : 0.0;
    if (alpha[i] - bl - br < lo) lo = alpha[i] - bl - br;
    if (alpha[i] + bl + br > hi) hi = alpha[i] + bl + br;
  }
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const int below = sturm_count(alpha, beta, n, mid);
    if (largest ? below < n : below < 1)
      lo = mid;
    else
      hi = mid;
    const double ah = fabs(hi);
    if (hi - lo < 1e-10 * (ah > 1.0 ? ah : 1.0)) break;
  }
  return 0.5 * (lo + hi);
}

int orc_op_estimate_eigenvalues(const orc_op* op, const void* diag, int iterations, uint64_t seed, double* lmin,
                                double* lmax) {
  if (!op->linearized) return 4;
  const int64_t n = op->ndofs;
  const int f64 = op->precision == 64;
  double* dis = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) {
    const double dv = f64 ? ((const double*)diag)[i] : (double)((const float*)diag)[i];
    dis[i] = 1.0 / sqrt(dv > 1e-300 ? dv : 1e-300);
  }
  int maxit = iterations < n ? iterations : (int)n;
  double* basis = (double*)malloc(sizeof(double) * n * (maxit > 0 ? maxit : 1));
  double* v = (double*)malloc(sizeof(double) * n);
  double* vprev = (double*)calloc(n, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * n);
  void* t = malloc((f64 ? 8 : 4) * n);
  void* at = malloc((f64 ? 8 : 4) * n);
  double* alpha = (double*)malloc(sizeof(double) * (maxit + 1));
  double* beta = (double*)malloc(sizeof(double) * (maxit + 1));
  int na = 0, nb = 0, err = 0;
  uint64_t state = seed;
  for (int64_t i = 0; i < n; ++i) v[i] = uniform01(&state) - 0.5;
  const double nv = sqrt(dot_d(v, v, n));
  for (int64_t i = 0; i < n; ++i) v[i] /= nv;
  double beta_prev = 0.0;
  for (int j = 0; j < maxit; ++j) {
    memcpy(basis + (size_t)j * n, v, sizeof(double) * n);
    if (f64)
      for (int64_t i = 0; i < n; ++i) ((double*)t)[i] = dis[i] * v[i];
    else
      for (int64_t i = 0; i < n; ++i) ((float*)t)[i] = (float)(dis[i] * v[i]);
    err |= orc_op_apply(op, t, at);
    for (int64_t i = 0; i < n; ++i) w[i] = dis[i] * (f64 ? ((double*)at)[i] : (double)((float*)at)[i]);
    if (j > 0)
      for (int64_t i = 0; i < n; ++i) w[i] -= beta_prev * vprev[i];
    const double a = dot_d(w, v, n);
    alpha[na++] = a;
    for (int64_t i = 0; i < n; ++i) w[i] -= a * v[i];
    for (int qb = 0; qb <= j; ++qb) {
      const double* q = basis + (size_t)qb * n;
      const double h = dot_d(w, q, n);
      for (int64_t i = 0; i < n; ++i) w[i] -= h * q[i];
    }
    const double b = sqrt(dot_d(w, w, n));
    if (j + 1 < maxit) beta[nb++] = b;
    if (b < 1e-12) break;
    memcpy(vprev, v, sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) v[i] = w[i] / b;
    beta_prev = b;
  }
  *lmax = tridiag_extreme(alpha, beta, na, 1);
  *lmin = tridiag_extreme(alpha, beta, na, 0);
  free(dis);
  free(basis);
  free(v);
  free(vprev);
  free(w);
  free(t);
  free(at);
  free(alpha);
  free(beta);
  return err;
}

/* ---- transfers: LatticeMap1D mesh.cpp:248-274, lattice_sweep mesh.hpp:190-241 */
typedef struct {
  int n_src, p_src, n_dst, p_dst;
  int* src_elem;
  double* w;
} lmap;

static void lmap_build(lmap* m, int n_src, int p_src, int n_dst, int p_dst) {
  double sn[ORC_MAXN], dn[ORC_MAXN];
  m->n_src = n_src;
  m->p_src = p_src;
  m->n_dst = n_dst;
  m->p_dst = p_dst;
  gauss_lobatto(p_src + 1, sn);
  gauss_lobatto(p_dst + 1, dn);
  const int nd = n_dst * p_dst + 1, stencil = p_src + 1;
  m->src_elem = (int*)malloc(sizeof(int) * nd);
  m->w = (double*)malloc(sizeof(double) * nd * stencil);
  for (int d = 0; d < nd; ++d) {
    int e_dst = d / p_dst;
    if (e_dst > n_dst - 1) e_dst = n_dst - 1;
    const int l_dst = d - e_dst * p_dst;
    const double s = (e_dst + 0.5 * (dn[l_dst] + 1.0)) / n_dst;
    int e_src = (int)(s * n_src);
    if (e_src > n_src - 1) e_src = n_src - 1;
    if (e_src > 0 && s * n_src <= e_src) e_src = e_src - (s * n_src < e_src);
    const double xi = 2.0 * (s * n_src - e_src) - 1.0;
    m->src_elem[d] = e_src;
    for (int i = 0; i < stencil; ++i) m->w[(size_t)d * stencil + i] = lagrange_value(sn, stencil, i, xi);
  }
}
static void lmap_free(lmap* m) {
  free(m->src_elem);
  free(m->w);
}

#define LSWEEP(R, NAME)                                                                                        \
  static void NAME(const lmap* m, int transpose, int axis, const R* in, int in_n0, int in_n1, int in_n2,   \
                   R* out) {                                                                                 \
    const int stencil = m->p_src + 1;                                                                        \
    const int nd = m->n_dst * m->p_dst + 1;                                                                  \
    const int out_na = transpose ? m->n_src * m->p_src + 1 : nd;                                             \
    const int n0 = axis == 0 ? out_na : in_n0, n1 = axis == 1 ? out_na : in_n1, n2 = axis == 2 ? out_na : in_n2; \
    const size_t total = (size_t)n0 * n1 * n2;                                                               \
    for (size_t i = 0; i < total; ++i) out[i] = (R)0;                                                        \
    const int in_stride = axis == 0 ? 1 : (axis == 1 ? in_n0 : in_n0 * in_n1);                               \
    const int out_stride = axis == 0 ? 1 : (axis == 1 ? n0 : n0 * n1);                                       \
    const int la = axis == 0 ? in_n1 : in_n0;                                                                \
    const int lb = axis == 2 ? in_n1 : in_n2;                                                                \
    for (int b = 0; b < lb; ++b)                                                                             \
      for (int a = 0; a < la; ++a) {                                                                         \
        size_t bi, bo;                                                                                       \
        if (axis == 0) {                                                                                     \
          bi = ((size_t)b * in_n1 + a) * in_n0;                                                              \
          bo = ((size_t)b * n1 + a) * n0;                                                                    \
        } else if (axis == 1) {                                                                              \
          bi = (size_t)b * in_n0 * in_n1 + a;                                                                \
          bo = (size_t)b * n0 * n1 + a;                                                                      \
        } else {                                                                                             \
          bi = (size_t)b * in_n0 + a;                                                                        \
          bo = (size_t)b * n0 + a;                                                                           \
        }                                                                                                    \
        const R* src = in + bi;                                                                              \
        R* dst = out + bo;                                                                                   \
        if (!transpose) {                                                                                    \
          for (int d = 0; d < nd; ++d) {                                                                     \
            R acc = (R)0;                                                                                    \
            const int base = m->src_elem[d] * m->p_src;                                                      \
            for (int s = 0; s < stencil; ++s)                                                                \
              acc += (R)m->w[d * stencil + s] * src[(size_t)(base + s) * in_stride];                         \
            dst[(size_t)d * out_stride] = acc;                                                               \
          }                                                                                                  \
        } else {                                                                                             \
          for (int d = 0; d < nd; ++d) {                                                                     \
            const R v = src[(size_t)d * in_stride];                                                          \
            const int base = m->src_elem[d] * m->p_src;                                                      \
            for (int s = 0; s < stencil; ++s) dst[(size_t)(base + s) * out_stride] += (R)m->w[d * stencil + s] * v; \
          }                                                                                                  \
        }                                                                                                    \
      }                                                                                                      \
  }
LSWEEP(double, lsweep_d)
LSWEEP(float, lsweep_f)

/* TransferOp::apply_axes mesh.hpp:245-271 for cube levels (n, p) -> (n', p').
 * kind 0 prolongate (coarse->fine), 1 restrict, 2 interpolate_down. The
 * reference uses one 1D map for all axes; EXT: a map per axis for boxes. */
int orc_transfer(int nf_x, int nf_y, int nf_z, int pf, int nc_x, int nc_y, int nc_z, int pc, int kind,
                 int precision, const void* in, void* out) {
  const int nf[3] = {nf_x, nf_y, nf_z}, nc[3] = {nc_x, nc_y, nc_z};
  lmap m[3];
  int ms[3], md[3];
  int transpose = kind == 1;
  for (int a = 0; a < 3; ++a) {
    if (kind == 2)
      lmap_build(&m[a], nf[a], pf, nc[a], pc); /* down_ */
    else
      lmap_build(&m[a], nc[a], pc, nf[a], pf); /* up_ */
    const int mfa = nf[a] * pf + 1, mca = nc[a] * pc + 1;
    ms[a] = kind == 0 ? mca : mfa; /* source lattice of this application */
    md[a] = kind == 0 ? mfa : mca;
  }
  const size_t nsrc = (size_t)ms[0] * ms[1] * ms[2], ndst = (size_t)md[0] * md[1] * md[2];
  size_t mx = 1;
  for (int a = 0; a < 3; ++a) mx *= (size_t)(ms[a] > md[a] ? ms[a] : md[a]);
  if (precision == 64) {
    double *bi = (double*)malloc(sizeof(double) * nsrc), *ba = (double*)malloc(sizeof(double) * mx),
           *bb = (double*)malloc(sizeof(double) * mx);
    for (int comp = 0; comp < 3; ++comp) {
      for (size_t i = 0; i < nsrc; ++i) bi[i] = ((const double*)in)[3 * i + comp];
      lsweep_d(&m[0], transpose, 0, bi, ms[0], ms[1], ms[2], ba);
      lsweep_d(&m[1], transpose, 1, ba, md[0], ms[1], ms[2], bb);
      lsweep_d(&m[2], transpose, 2, bb, md[0], md[1], ms[2], ba);
      for (size_t i = 0; i < ndst; ++i) ((double*)out)[3 * i + comp] = ba[i];
    }
    free(bi);
    free(ba);
    free(bb);
  } else {
    float *bi = (float*)malloc(sizeof(float) * nsrc), *ba = (float*)malloc(sizeof(float) * mx),
          *bb = (float*)malloc(sizeof(float) * mx);
    for (int comp = 0; comp < 3; ++comp) {
      for (size_t i = 0; i < nsrc; ++i) bi[i] = ((const float*)in)[3 * i + comp];
      lsweep_f(&m[0], transpose, 0, bi, ms[0], ms[1], ms[2], ba);
      lsweep_f(&m[1], transpose, 1, ba, md[0], ms[1], ms[2], bb);
      lsweep_f(&m[2], transpose, 2, bb, md[0], md[1], ms[2], ba);
      for (size_t i = 0; i < ndst; ++i) ((float*)out)[3 * i + comp] = ba[i];
    }
    free(bi);
    free(ba);
    free(bb);
  }
  for (int a = 0; a < 3; ++a) lmap_free(&m[a]);
  return 0;
}

int orc_op_element_locals(const orc_op* op, const void* x, void* loc, int64_t e0, int64_t e1) {
  if (!op->linearized) return 4;
  return op->precision == 64 ? element_locals_d(op, (const double*)x, (double*)loc, e0, e1)
                             : element_locals_f(op, (const float*)x, (float*)loc, e0, e1);
}

/* ---- hp-multigrid V-cycle (solver.hpp:437-581), float levels --------------
 * Ladder p -> p/2 -> ... -> 1 on the fine mesh, then n0<<l cubes for
 * l = lmax-1..0 at p = 1 (solver.hpp:450-459).  Coarse solver: the
 * reference's Jacobi-PCG path (solver.hpp:393-424; coarse_direct_limit = 0). */
#define ORC_MAXLEV 16
typedef struct {
  int nlev, n[ORC_MAXLEV], p[ORC_MAXLEV], faces, degree, eig_it;
  double range_factor, safety, lmax[ORC_MAXLEV];
  uint64_t seed;
  orc_op* ops[ORC_MAXLEV];
  float* diag[ORC_MAXLEV];
  float* x[ORC_MAXLEV];
  float* b[ORC_MAXLEV];
} orc_mg;

static void zero_mask_f(const orc_op* op, float* v) {
  for (int64_t i = 0; i < op->ndofs; ++i)
    if (op->mask[i]) v[i] = 0.0f;
}

static double dotf(const float* a, const float* b, int64_t n) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += (double)a[i] * (double)b[i];
  return s;
}

orc_mg* orc_mg_create(int n0, int lmax, int p, double deform_amp, int faces, int model, const double* prm,
                      int strategy, int degree, double range_factor, double safety, int eig_it) {
  orc_mg* m = (orc_mg*)calloc(1, sizeof(orc_mg));
  int pp = p, k = 0;
  m->n[k] = n0 << lmax;
  m->p[k++] = pp;
  while (pp > 1) {
    pp /= 2;
    m->n[k] = n0 << lmax;
    m->p[k++] = pp;
  }
  for (int l = lmax - 1; l >= 0; --l) {
    m->n[k] = n0 << l;
    m->p[k++] = 1;
  }
  m->nlev = k;
  m->faces = faces;
  m->degree = degree;
  m->range_factor = range_factor;
  m->safety = safety;
  m->eig_it = eig_it;
  m->seed = 0x9e3779b97f4a7c15ull;
  const double ext[3] = {1.0, 1.0, 1.0}, mp[2] = {deform_amp, 1.0};
  for (int l = 0; l < m->nlev; ++l) {
    const int n = m->n[l], q = m->p[l];
    double* coords = (double*)malloc(sizeof(double) * 3 * (size_t)(n * q + 1) * (n * q + 1) * (n * q + 1));
    orc_lattice_coords(n, n, n, q, ext, 0, mp, coords);
    m->ops[l] = orc_op_create(n, n, n, q, coords, faces, model, prm, strategy, 32);
    free(coords);
    const int64_t nd = m->ops[l]->ndofs;
    m->diag[l] = (float*)malloc(sizeof(float) * nd);
    m->x[l] = (float*)calloc(nd, sizeof(float));
    m->b[l] = (float*)calloc(nd, sizeof(float));
  }
  return m;
}

void orc_mg_destroy(orc_mg* m) {
  for (int l = 0; l < m->nlev; ++l) {
    orc_op_destroy(m->ops[l]);
    free(m->diag[l]);
    free(m->x[l]);
    free(m->b[l]);
  }
  free(m);
}

int orc_mg_n_levels(const orc_mg* m) { return m->nlev; }

static void dims4(const orc_mg* m, int l, int* d) { d[0] = d[1] = d[2] = m->n[l]; d[3] = m->p[l]; }

/* MgHierarchy::update_linearization, solver.hpp:490-509 */
int orc_mg_update(orc_mg* m, const double* u_fine) {
  const int64_t n0 = m->ops[0]->ndofs;
  double* u = (double*)malloc(sizeof(double) * n0);
  memcpy(u, u_fine, sizeof(double) * n0);
  int err = 0;
  for (int l = 0; l < m->nlev; ++l) {
    orc_op* op = m->ops[l];
    if (l > 0) {
      int fd[4], cd[4];
      dims4(m, l - 1, fd);
      dims4(m, l, cd);
      double* uc = (double*)malloc(sizeof(double) * op->ndofs);
      orc_transfer(fd[0], fd[1], fd[2], fd[3], cd[0], cd[1], cd[2], cd[3], 2, 64, u, uc);
      for (int64_t i = 0; i < op->ndofs; ++i)
        if (op->mask[i]) uc[i] = 0.0; /* dirichlet_set_values (zero) */
      free(u);
      u = uc;
    }
    if ((err = orc_op_linearize(op, u, NULL, NULL))) break;
    int64_t nb;
    if ((err = orc_op_diagonal(op, m->diag[l], &nb))) break;
    double lmin;
    if ((err = orc_op_estimate_eigenvalues(op, m->diag[l], m->eig_it, m->seed, &lmin, &m->lmax[l]))) break;
  }
  free(u);
  return err;
}

/* CoarseSolver::solve (Jacobi-PCG path), solver.hpp:393-424 */
static int coarse_cg(const orc_op* op, const float* diag, const float* b, float* x) {
  const int64_t n = op->ndofs;
  float *r = (float*)malloc(sizeof(float) * n), *z = (float*)malloc(sizeof(float) * n),
        *pv = (float*)malloc(sizeof(float) * n), *ap = (float*)malloc(sizeof(float) * n),
        *inv = (float*)malloc(sizeof(float) * n);
  int err = 0;
  for (int64_t i = 0; i < n; ++i) {
    x[i] = 0.0f;
    r[i] = b[i];
    inv[i] = 1.0f / diag[i];
  }
  const double bnorm = sqrt(dotf(b, b, n));
  if (bnorm != 0) {
    for (int64_t i = 0; i < n; ++i) z[i] = inv[i] * r[i];
    memcpy(pv, z, sizeof(float) * n);
    double rz = dotf(r, z, n);
    int it;
    for (it = 0; it < 500; ++it) {
      err |= orc_op_apply(op, pv, ap);
      const double alpha = rz / dotf(pv, ap, n);
      for (int64_t i = 0; i < n; ++i) {
        x[i] += (float)alpha * pv[i];
        r[i] -= (float)alpha * ap[i];
      }
      if (sqrt(dotf(r, r, n)) <= 1e-4 * bnorm) break;
      for (int64_t i = 0; i < n; ++i) z[i] = inv[i] * r[i];
      const double rz_new = dotf(r, z, n);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; ++i) pv[i] = z[i] + (float)beta * pv[i];
    }
    if (it == 500) err = 5;
  }
  free(r);
  free(z);
  free(pv);
  free(ap);
  free(inv);
  return err;
}

/* MgHierarchy::v_cycle, solver.hpp:544-569 */
static int v_cycle(orc_mg* m, int l, const float* b) {
  orc_op* op = m->ops[l];
  const int64_t n = op->ndofs;
  float* x = m->x[l];
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0f;
  if (l + 1 == m->nlev) return coarse_cg(op, m->diag[l], b, x);
  int err = orc_op_chebyshev(op, m->diag[l], m->lmax[l], m->degree, m->range_factor, m->safety, b, x, 1);
  float* t = (float*)malloc(sizeof(float) * n);
  err |= orc_op_apply(op, x, t);
  for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
  zero_mask_f(op, t);
  int fd[4], cd[4];
  dims4(m, l, fd);
  dims4(m, l + 1, cd);
  float* bc = m->b[l + 1];
  orc_transfer(fd[0], fd[1], fd[2], fd[3], cd[0], cd[1], cd[2], cd[3], 1, 32, t, bc);
  zero_mask_f(m->ops[l + 1], bc);
  err |= v_cycle(m, l + 1, bc);
  orc_transfer(fd[0], fd[1], fd[2], fd[3], cd[0], cd[1], cd[2], cd[3], 0, 32, m->x[l + 1], t);
  zero_mask_f(op, t);
  for (int64_t i = 0; i < n; ++i) x[i] += t[i];
  err |= orc_op_chebyshev(op, m->diag[l], m->lmax[l], m->degree, m->range_factor, m->safety, b, x, 0);
  free(t);
  return err;
}

/* MgHierarchy::precondition, solver.hpp:512-520 */
int orc_mg_precondition(orc_mg* m, const double* r, double* z) {
  const int64_t n = m->ops[0]->ndofs;
  float* b0 = m->b[0];
  for (int64_t i = 0; i < n; ++i) b0[i] = (float)r[i];
  zero_mask_f(m->ops[0], b0);
  const int err = v_cycle(m, 0, b0);
  for (int64_t i = 0; i < n; ++i) z[i] = (double)m->x[0][i];
  return err;
}

/* Outer PCG in double (see ref_driver.cpp ref_pcg_solve). */
int orc_pcg_solve(const orc_op* op, orc_mg* m, const double* b, double* x, double rtol, int maxit, int* iters,
                  double* history) {
  const int64_t n = op->ndofs;
  double *r = (double*)malloc(sizeof(double) * n), *z = (double*)malloc(sizeof(double) * n),
         *pv = (double*)malloc(sizeof(double) * n), *ap = (double*)malloc(sizeof(double) * n);
  int err = 0, it = 0;
  for (int64_t i = 0; i < n; ++i) {
    x[i] = 0.0;
    r[i] = b[i];
  }
  const double bnorm = sqrt(dot_d(b, b, n));
  if (history) history[0] = 1.0;
  if (bnorm != 0) {
    if (m)
      err |= orc_mg_precondition(m, r, z);
    else
      memcpy(z, r, sizeof(double) * n);
    memcpy(pv, z, sizeof(double) * n);
    double rz = dot_d(r, z, n);
    for (it = 0; it < maxit; ++it) {
      err |= orc_op_apply(op, pv, ap);
      const double alpha = rz / dot_d(pv, ap, n);
      for (int64_t i = 0; i < n; ++i) {
        x[i] += alpha * pv[i];
        r[i] -= alpha * ap[i];
      }
      const double rel = sqrt(dot_d(r, r, n)) / bnorm;
      if (history) history[it + 1] = rel;
      if (rel <= rtol) {
        ++it;
        break;
      }
      if (m)
        err |= orc_mg_precondition(m, r, z);
      else
        memcpy(z, r, sizeof(double) * n);
      const double rz_new = dot_d(r, z, n);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; ++i) pv[i] = z[i] + beta * pv[i];
    }
  }
  *iters = it;
  free(r);
  free(z);
  free(pv);
  free(ap);
  return err;
}

/* Per-qp fibre frame field: h (12*nqp, SoA H4,H6) and m1 (6*nqp, SoA). */
void orc_op_set_frames(orc_op* op, const double* h, const double* m1) {
  const int64_t nqp = op->nel * op->nq3;
  free(op->hq);
  free(op->m1q);
  op->hq = (double*)malloc(sizeof(double) * 12 * nqp);
  op->m1q = (double*)malloc(sizeof(double) * 6 * nqp);
  memcpy(op->hq, h, sizeof(double) * 12 * nqp);
  memcpy(op->m1q, m1, sizeof(double) * 6 * nqp);
  op->linearized = 0;
}
