/* Plain C client of the C ABI (include/emfgpu.h): the calls a cgo / ctypes /
 * JNI binding would make.  8^3 Q2 cNH (BASELINE configs[0] mesh), host
 * vectors: create level and operator, linearize at a smooth state, apply,
 * diagonal, residual; prints norms and the status of an apply on a stale
 * operator.  Exit code 0 on success. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "emfgpu.h"

static double norm(const double* v, int64_t n) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

int main(void) {
  emfgpu_level_desc d = {0};
  d.nx = d.ny = d.nz = 8;
  d.p = 2;
  d.extent[0] = d.extent[1] = d.extent[2] = 1.0;
  d.map = EMFGPU_MAP_REFERENCE;
  d.dirichlet_faces = 1;
  emfgpu_level* lev = NULL;
  if (emfgpu_level_create(&d, &lev) != EMFGPU_OK) {
    fprintf(stderr, "level: %s\n", emfgpu_global_last_error());
    return 1;
  }
  const int64_t n = emfgpu_level_n_dofs(lev);
  emfgpu_material m = {0};
  m.mu = 1.0;
  m.lambda = 10.0;
  emfgpu_op* op = NULL;
  if (emfgpu_op_create(lev, EMFGPU_CNH, &m, 0, EMFGPU_NONE, 64, &op) != EMFGPU_OK) {
    fprintf(stderr, "op: %s\n", emfgpu_global_last_error());
    return 1;
  }
  double* u = calloc((size_t)n, sizeof(double));
  double* v = malloc((size_t)n * sizeof(double));
  double* y = malloc((size_t)n * sizeof(double));
  const int stale = emfgpu_op_apply_host(op, v, y); /* before linearization: EMFGPU_ERR_STALE */
  const int mx = 8 * 2 + 1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t node = i / 3;
    const double x = (double)(node % mx) / (mx - 1), yy = (double)((node / mx) % mx) / (mx - 1),
                 z = (double)(node / (mx * mx)) / (mx - 1);
    u[i] = (node % mx == 0) ? 0.0 : 0.05 * sin(3.14159265358979 * x) * sin(3.14159265358979 * yy) * z;
    v[i] = sin(0.37 * (double)i);
  }
  int64_t be = -1;
  int bq = -1;
  if (emfgpu_op_update_linearization_host(op, u, &be, &bq) != EMFGPU_OK) {
    fprintf(stderr, "linearize: %s\n", emfgpu_op_last_error(op));
    return 1;
  }
  if (emfgpu_op_apply_host(op, v, y) != EMFGPU_OK) return 1;
  double* dg = malloc((size_t)n * sizeof(double));
  int64_t nbad = -1;
  if (emfgpu_op_compute_diagonal_host(op, dg, &nbad) != EMFGPU_OK) return 1;
  double* r = malloc((size_t)n * sizeof(double));
  if (emfgpu_op_set_pressure(op, 0.1, 1) != EMFGPU_OK || emfgpu_op_residual_host(op, u, r) != EMFGPU_OK) return 1;
  printf("capi n=%lld stale=%d |y|=%.17g |diag|=%.17g nbad=%lld |r|=%.17g version=%s\n", (long long)n, stale,
         norm(y, n), norm(dg, n), (long long)nbad, norm(r, n), emfgpu_version());
  emfgpu_op_destroy(op);
  emfgpu_level_destroy(lev);
  free(u);
  free(v);
  free(y);
  free(dg);
  free(r);
  return 0;
}
