/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * Precision-generic body of emf_oracle.c, included twice with
 *   R  = double | float   (the operator's Number type)
 *   SFX(name)             (name suffix _d | _f)
 * Every routine keeps the reference's operation order so that, compiled with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:11-13), results
 * are bitwise identical to ElasticOperator<Number>.
 */

/* ---- 3x3 algebra: proj/include/elastmf/tensor.hpp ----------------------- */
typedef struct { R a[9]; } SFX(t2);   /* row-major general tensor */
typedef struct { R s[6]; } SFX(s2);   /* (11,22,33,12,13,23), tensor.hpp:93-100 */

static inline int SFX(sidx)(int i, int j) { return (i == j) ? i : 2 + i + j; }

/* tensor.hpp:188-194 */
static inline R SFX(det)(const R* t) {
  const R c0 = t[0] * (t[4] * t[8] - t[5] * t[7]);
  const R c1 = t[1] * (t[3] * t[8] - t[5] * t[6]);
  const R c2 = t[2] * (t[3] * t[7] - t[4] * t[6]);
  return (c0 - c1) + c2;
}

/* tensor.hpp:199-208 */
static inline R SFX(det_minus_one)(const R* g) {
  const R tr = (g[0] + g[4]) + g[8];
  const R m01 = g[0] * g[4] - g[1] * g[3];
  const R m02 = g[0] * g[8] - g[2] * g[6];
  const R m12 = g[4] * g[8] - g[5] * g[7];
  const R minors = (m01 + m02) + m12;
  const R d = SFX(det)(g);
  return (d + minors) + tr;
}

/* tensor.hpp:212-231; returns nonzero when |det| is below the floor */
static inline int SFX(inverse)(const R* t, R* r) {
  const R d = SFX(det)(t);
  const R floor_ = sizeof(R) == 8 ? (R)1e-300 : (R)1e-30;
  if (fabs((double)d) < (double)floor_) return 1;
  const R inv = (R)1 / d;
  r[0] = (t[4] * t[8] - t[5] * t[7]) * inv;
  r[1] = (t[2] * t[7] - t[1] * t[8]) * inv;
  r[2] = (t[1] * t[5] - t[2] * t[4]) * inv;
  r[3] = (t[5] * t[6] - t[3] * t[8]) * inv;
  r[4] = (t[0] * t[8] - t[2] * t[6]) * inv;
  r[5] = (t[2] * t[3] - t[0] * t[5]) * inv;
  r[6] = (t[3] * t[7] - t[4] * t[6]) * inv;
  r[7] = (t[1] * t[6] - t[0] * t[7]) * inv;
  r[8] = (t[0] * t[4] - t[1] * t[3]) * inv;
  return 0;
}

/* tensor.hpp:288-294 (general x general) */
static inline void SFX(mm)(const R* x, const R* y, R* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (x[3 * i] * y[j] + x[3 * i + 1] * y[3 + j]) + x[3 * i + 2] * y[6 + j];
}
/* tensor.hpp:297-303 (general x symmetric) */
static inline void SFX(mm_ts)(const R* x, const R* ys, R* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (x[3 * i] * ys[SFX(sidx)(0, j)] + x[3 * i + 1] * ys[SFX(sidx)(1, j)]) +
                     x[3 * i + 2] * ys[SFX(sidx)(2, j)];
}
/* tensor.hpp:306-312 (symmetric x general) */
static inline void SFX(mm_st)(const R* xs, const R* y, R* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = (xs[SFX(sidx)(i, 0)] * y[j] + xs[SFX(sidx)(i, 1)] * y[3 + j]) +
                     xs[SFX(sidx)(i, 2)] * y[6 + j];
}
/* tensor.hpp:155-166 */
static inline void SFX(sym_part)(const R* t, R* s) {
  const R half = (R)0.5;
  s[0] = t[0];
  s[1] = t[4];
  s[2] = t[8];
  s[3] = half * (t[1] + t[3]);
  s[4] = half * (t[2] + t[6]);
  s[5] = half * (t[5] + t[7]);
}
static inline void SFX(to_tensor)(const R* s, R* t) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[3 * i + j] = s[SFX(sidx)(i, j)];
}
static inline void SFX(transpose)(const R* t, R* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[3 * i + j] = t[3 * j + i];
}
/* tensor.hpp:274-279 */
static inline R SFX(ddot_s)(const R* x, const R* y) {
  const R dg = (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2];
  const R off = (x[3] * y[3] + x[4] * y[4]) + x[5] * y[5];
  return dg + (R)2 * off;
}
/* tensor.hpp:281-286 */
static inline R SFX(ddot_t)(const R* x, const R* y) {
  R r = x[0] * y[0];
  for (int i = 1; i < 9; ++i) r += x[i] * y[i];
  return r;
}

/* ---- scalar kernels: proj/include/elastmf/fastscalar.hpp ---------------- */
/* fastscalar.hpp:44-71 (scalar branch; 16 terms) */
static inline R SFX(ln_plus_one)(R x) {
  if (fabs((double)x) > 0.5) return sizeof(R) == 8 ? (R)log1p((double)x) : (R)log1pf((float)x);
  const R y = x / ((R)2 + x);
  const R y2 = y * y;
  R pw = y, powers[16];
  for (int n = 0; n < 16; ++n) {
    powers[n] = pw;
    pw = pw * y2;
  }
  R sum = (R)0;
  for (int n = 15; n >= 0; --n) sum += powers[n] * ((R)1 / (R)(2 * n + 1));
  return (R)2 * sum;
}
/* fastscalar.hpp:77-89 (3 Newton steps) */
static inline R SFX(fast_jpow)(R jm1) {
  const R third = (R)1 / (R)3;
  const R four_thirds = (R)4 / (R)3;
  const R alpha = ((jm1 + (R)2) * jm1 + (R)1) * third;
  R beta = four_thirds - alpha;
  for (int n = 0; n < 3; ++n) {
    const R b2 = beta * beta;
    const R gamma = b2 * b2;
    beta = four_thirds * beta - alpha * gamma;
  }
  return beta;
}

/* ---- per-point cache: constitutive.hpp:79-93 --------------------------- */
typedef struct {
  R jm1, jac, lnj, jp, c1, c2, c3[2], istar[2], efib[2];
  R F[9], Finv[9], S[6], Cinv[6], E[6], i1;
  R bt[6], b[6], tau[6], fh[2][6]; /* spatial cell: Green-Euler bt, b = F F^T, tau, F H_i F^T */
} SFX(qpc);

/* make_strain (stable) constitutive.hpp:43-57 + compute_cache :326-377,
 * material domain. Returns nonzero when det(F) <= 0 (constitutive.hpp:37-41). */
static int SFX(compute_cache)(const orc_material* mat, const R* g, SFX(qpc)* c) {
  const R mu = (R)mat->mu;
  R Fm[9];
  for (int i = 0; i < 9; ++i) Fm[i] = g[i];
  Fm[0] = (R)1 + g[0];
  Fm[4] = (R)1 + g[4];
  Fm[8] = (R)1 + g[8];
  c->jm1 = SFX(det_minus_one)(g);
  if (!(c->jm1 > (R)-1)) return 1;
  c->jac = (R)1 + c->jm1;
  /* green_lagrange_stable tensor.hpp:247-257 */
  {
    const R half = (R)0.5;
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        const R q = (g[i] * g[j] + g[3 + i] * g[3 + j]) + g[6 + i] * g[6 + j];
        c->E[SFX(sidx)(i, j)] = half * ((g[3 * i + j] + g[3 * j + i]) + q);
      }
  }
  /* green_euler_stable tensor.hpp:259-270 */
  {
    const R half = (R)0.5;
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j) {
        const R q = (g[3 * i] * g[3 * j] + g[3 * i + 1] * g[3 * j + 1]) + g[3 * i + 2] * g[3 * j + 2];
        c->bt[SFX(sidx)(i, j)] = half * ((g[3 * i + j] + g[3 * j + i]) + q);
      }
  }
  if (SFX(inverse)(Fm, c->Finv)) return 2;
  /* inverse_C_stable tensor.hpp:235-243 */
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j)
      c->Cinv[SFX(sidx)(i, j)] = (c->Finv[3 * i] * c->Finv[3 * j] + c->Finv[3 * i + 1] * c->Finv[3 * j + 1]) +
                                 c->Finv[3 * i + 2] * c->Finv[3 * j + 2];
  c->i1 = (R)3 + (R)2 * ((c->E[0] + c->E[1]) + c->E[2]);
  for (int i = 0; i < 9; ++i) c->F[i] = Fm[i];
  c->lnj = SFX(ln_plus_one)(c->jm1);
  c->jp = mat->model == 0 ? (R)1 : SFX(fast_jpow)(c->jm1);
  if (mat->model != 0) {
    const R half_k = (R)(0.5 * mat->kappa);
    const R hk = half_k * (c->jm1 * (c->jm1 + (R)2));
    c->c1 = hk - ((mu / (R)3) * c->jp) * c->i1;
    c->c2 = ((((R)2 * mu) / (R)9) * c->jp) * c->i1 + ((R)mat->kappa * c->jac) * c->jac;
  } else {
    c->c1 = c->c2 = (R)0;
  }
  c->c3[0] = c->c3[1] = c->istar[0] = c->istar[1] = c->efib[0] = c->efib[1] = (R)0;
  if (mat->model == 2) {
    /* fiber_invariants constitutive.hpp:117-149 (stable) */
    for (int f = 0; f < 2; ++f) {
      R hn[6], mm[6], mv[3];
      for (int k = 0; k < 6; ++k) hn[k] = (R)mat->h[f][k];
      for (int k = 0; k < 3; ++k) mv[k] = (R)mat->m1[f][k];
      for (int i = 0; i < 3; ++i)
        for (int j = i; j < 3; ++j) mm[SFX(sidx)(i, j)] = mv[i] * mv[j];
      c->efib[f] = (R)2 * SFX(ddot_s)(hn, c->E);
      const R gate = (R)2 * SFX(ddot_s)(mm, c->E);
      c->istar[f] = (R)1 + gate;
      const R z = ((R)mat->k2 * c->efib[f]) * c->efib[f];
      const R ex = sizeof(R) == 8 ? (R)exp((double)z) : (R)expf((float)z);
      const R active = ex * (R)(2.0 * mat->k1);
      c->c3[f] = gate > (R)0 ? active : (R)0;
    }
  }
  return 0;
}

/* second_pk_base constitutive.hpp:197-238 (stable) + fiber terms :368-371 */
/* E, Cinv, jm1 come from the strain state; lnj, jp, c3, efib from the bundle
 * (loaded in the scalar strategy, operator.hpp:411-420). */
static void SFX(second_pk)(const orc_material* mat, const SFX(qpc)* c, R* S) {
  const R mu = (R)mat->mu;
  R inner[6], full[9], prod[9];
  if (mat->model == 0) {
    const R lam = (R)mat->lambda;
    for (int k = 0; k < 6; ++k) inner[k] = ((R)2 * mu) * c->E[k];
    const R v = ((R)2 * lam) * c->lnj;
    inner[0] += v;
    inner[1] += v;
    inner[2] += v;
  } else {
    const R half_k = (R)(0.5 * mat->kappa);
    const R vol = half_k * (c->jm1 * (c->jm1 + (R)2));
    const R tre3 = ((c->E[0] + c->E[1]) + c->E[2]) * ((R)1 / (R)3);
    const R s = ((R)2 * mu) * c->jp;
    for (int k = 0; k < 6; ++k) inner[k] = s * c->E[k];
    const R dev = (((R)2 * mu) * c->jp) * tre3;
    inner[0] += vol - dev;
    inner[1] += vol - dev;
    inner[2] += vol - dev;
  }
  SFX(to_tensor)(inner, full);
  SFX(mm_st)(c->Cinv, full, prod);
  SFX(sym_part)(prod, S);
  if (mat->model == 2)
    for (int f = 0; f < 2; ++f) {
      const R coef = c->c3[f] * c->efib[f];
      for (int k = 0; k < 6; ++k) S[k] += coef * (R)mat->h[f][k];
    }
}

/* Spatial cell of compute_cache (constitutive.hpp:371-376): b = 2 bt + I,
 * tau = kirchhoff_base (:240-283, stable) + sum c3 E_i F H_i F^T with
 * push_forward (tensor.hpp:332-341).  Reads bt, jm1, F, lnj, jp, c3, efib. */
static void SFX(spatial_cell)(const orc_material* mat, SFX(qpc)* c) {
  const R mu = (R)mat->mu;
  for (int k = 0; k < 6; ++k) c->b[k] = (R)2 * c->bt[k];
  c->b[0] += (R)1;
  c->b[1] += (R)1;
  c->b[2] += (R)1;
  if (mat->model == 0) {
    const R lam = (R)mat->lambda;
    for (int k = 0; k < 6; ++k) c->tau[k] = ((R)2 * mu) * c->bt[k];
    const R v = ((R)2 * lam) * c->lnj;
    c->tau[0] += v;
    c->tau[1] += v;
    c->tau[2] += v;
  } else {
    const R half_k = (R)(0.5 * mat->kappa);
    const R vol = half_k * (c->jm1 * (c->jm1 + (R)2));
    const R trb3 = ((c->bt[0] + c->bt[1]) + c->bt[2]) * ((R)1 / (R)3);
    const R s2 = ((R)2 * mu) * c->jp;
    for (int k = 0; k < 6; ++k) c->tau[k] = s2 * c->bt[k];
    const R v = vol - s2 * trb3;
    c->tau[0] += v;
    c->tau[1] += v;
    c->tau[2] += v;
  }
  for (int f = 0; f < 2; ++f)
    for (int k = 0; k < 6; ++k) c->fh[f][k] = (R)0;
  if (mat->model == 2)
    for (int f = 0; f < 2; ++f) {
      R h[6], fhm[9];
      for (int k = 0; k < 6; ++k) h[k] = (R)mat->h[f][k];
      SFX(mm_ts)(c->F, h, fhm);
      for (int i = 0; i < 3; ++i)
        for (int j = i; j < 3; ++j)
          c->fh[f][SFX(sidx)(i, j)] =
              (fhm[3 * i] * c->F[3 * j] + fhm[3 * i + 1] * c->F[3 * j + 1]) + fhm[3 * i + 2] * c->F[3 * j + 2];
      const R coef = c->c3[f] * c->efib[f];
      for (int k = 0; k < 6; ++k) c->tau[k] += coef * c->fh[f][k];
    }
}

/* tangent_spatial constitutive.hpp:421-463: J c : (grad du)^S + (grad du) tau. */
static void SFX(tangent_spatial)(const orc_material* mat, const SFX(qpc)* c, const R* dgrad, R* out) {
  const R mu = (R)mat->mu;
  R xs[6], jc[6], gt[9];
  SFX(sym_part)(dgrad, xs);
  const R trx = (dgrad[0] + dgrad[4]) + dgrad[8];
  if (mat->model == 0) {
    const R lam = (R)mat->lambda;
    const R f = (R)2 * (mu - ((R)2 * lam) * c->lnj);
    for (int k = 0; k < 6; ++k) jc[k] = f * xs[k];
    const R v = ((R)2 * lam) * trx;
    jc[0] += v;
    jc[1] += v;
    jc[2] += v;
  } else {
    const R bx = SFX(ddot_s)(c->b, xs);
    const R ttmj = (((R)2 * mu) / (R)3) * c->jp;
    const R f0 = -ttmj * trx;
    for (int k = 0; k < 6; ++k) jc[k] = f0 * c->b[k];
    const R m2c1 = (R)-2 * c->c1;
    for (int k = 0; k < 6; ++k) jc[k] += m2c1 * xs[k];
    const R v = c->c2 * trx - ttmj * bx;
    jc[0] += v;
    jc[1] += v;
    jc[2] += v;
    if (mat->model == 2) {
      const R k2 = (R)mat->k2;
      for (int f = 0; f < 2; ++f) {
        const R fhx = SFX(ddot_s)(c->fh[f], xs);
        const R coef = (((R)2 * c->c3[f]) * ((((R)2 * k2) * c->efib[f]) * c->efib[f] + (R)1)) * fhx;
        for (int k = 0; k < 6; ++k) jc[k] += coef * c->fh[f][k];
      }
    }
  }
  SFX(mm_ts)(dgrad, c->tau, gt);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = jc[SFX(sidx)(i, j)] + gt[3 * i + j];
}

/* tangent_material constitutive.hpp:381-419 */
static void SFX(tangent_material)(const orc_material* mat, const SFX(qpc)* c, const R* dg, R* r) {
  const R mu = (R)mat->mu;
  R a[9], acinv[9], sac[6];
  SFX(mm)(c->Finv, dg, a);
  const R w = (a[0] + a[4]) + a[8];
  SFX(mm_ts)(a, c->Cinv, acinv);
  SFX(sym_part)(acinv, sac);
  if (mat->model == 0) {
    const R lam = (R)mat->lambda;
    const R f1 = (R)2 * (mu - ((R)2 * lam) * c->lnj);
    for (int k = 0; k < 6; ++k) r[k] = f1 * sac[k];
    const R f2 = ((R)2 * lam) * w;
    for (int k = 0; k < 6; ++k) r[k] += f2 * c->Cinv[k];
    return;
  }
  const R q = SFX(ddot_t)(c->F, dg);
  const R ttmj = (((R)2 * mu) / (R)3) * c->jp;
  const R m2c1 = (R)-2 * c->c1;
  for (int k = 0; k < 6; ++k) r[k] = m2c1 * sac[k];
  const R f2 = c->c2 * w - ttmj * q;
  for (int k = 0; k < 6; ++k) r[k] += f2 * c->Cinv[k];
  const R dgl = (-ttmj) * w;
  r[0] += dgl;
  r[1] += dgl;
  r[2] += dgl;
  if (mat->model == 2) {
    const R k2 = (R)mat->k2;
    R ft[9], ftdg[9], dch[6];
    SFX(transpose)(c->F, ft);
    SFX(mm)(ft, dg, ftdg);
    SFX(sym_part)(ftdg, dch);
    for (int f = 0; f < 2; ++f) {
      R h[6];
      for (int k = 0; k < 6; ++k) h[k] = (R)mat->h[f][k];
      const R hdc = (R)2 * SFX(ddot_s)(h, dch);
      const R coef = (c->c3[f] * ((((R)2 * k2) * c->efib[f]) * c->efib[f] + (R)1)) * hdc;
      for (int k = 0; k < 6; ++k) r[k] += coef * h[k];
    }
  }
}

/* ---- sum factorization: proj/include/elastmf/sumfact.hpp --------------- */
static void SFX(sweep0)(const double* M, int rows, int cols, const R* in, int n1, int n2, R* out) {
  for (int k = 0; k < n2; ++k)
    for (int j = 0; j < n1; ++j) {
      const R* src = in + ((size_t)k * n1 + j) * cols;
      R* dst = out + ((size_t)k * n1 + j) * rows;
      for (int r = 0; r < rows; ++r) {
        R acc = (R)M[r * cols] * src[0];
        for (int c = 1; c < cols; ++c) acc += (R)M[r * cols + c] * src[c];
        dst[r] = acc;
      }
    }
}
static void SFX(sweep1)(const double* M, int rows, int cols, const R* in, int n0, int n2, R* out) {
  for (int k = 0; k < n2; ++k) {
    const R* src = in + (size_t)k * n0 * cols;
    R* dst = out + (size_t)k * n0 * rows;
    for (int r = 0; r < rows; ++r)
      for (int i = 0; i < n0; ++i) {
        R acc = (R)M[r * cols] * src[i];
        for (int c = 1; c < cols; ++c) acc += (R)M[r * cols + c] * src[c * n0 + i];
        dst[r * n0 + i] = acc;
      }
  }
}
static void SFX(sweep2)(const double* M, int rows, int cols, const R* in, int n0, int n1, R* out) {
  const size_t plane = (size_t)n0 * n1;
  for (int r = 0; r < rows; ++r)
    for (size_t i = 0; i < plane; ++i) {
      R acc = (R)M[r * cols] * in[i];
      for (int c = 1; c < cols; ++c) acc += (R)M[r * cols + c] * in[c * plane + i];
      out[r * plane + i] = acc;
    }
}
/* sumfact.hpp:67-85 */
static void SFX(grad_qp)(const orc_basis* b, const R* nodal, R* work, R* g0, R* g1, R* g2) {
  const int nn = b->n, nq = b->n;
  R* t1 = work;
  R* t2 = work + nn * nn * nn;
  SFX(sweep0)(b->D, nq, nn, nodal, nn, nn, t1);
  SFX(sweep1)(b->B, nq, nn, t1, nq, nn, t2);
  SFX(sweep2)(b->B, nq, nn, t2, nq, nq, g0);
  SFX(sweep0)(b->B, nq, nn, nodal, nn, nn, t1);
  SFX(sweep1)(b->D, nq, nn, t1, nq, nn, t2);
  SFX(sweep2)(b->B, nq, nn, t2, nq, nq, g1);
  SFX(sweep1)(b->B, nq, nn, t1, nq, nn, t2);
  SFX(sweep2)(b->D, nq, nn, t2, nq, nq, g2);
}
/* sumfact.hpp:90-110 */
static void SFX(scatter_grad)(const orc_basis* b, const R* g0, const R* g1, const R* g2, R* work, R* nodal) {
  const int nn = b->n, nq = b->n, nn3 = nn * nn * nn;
  R* t1 = work;
  R* t2 = work + nn3;
  SFX(sweep0)(b->Dt, nn, nq, g0, nq, nq, t1);
  SFX(sweep1)(b->Bt, nn, nq, t1, nn, nq, t2);
  SFX(sweep2)(b->Bt, nn, nq, t2, nn, nn, t1);
  for (int i = 0; i < nn3; ++i) nodal[i] += t1[i];
  SFX(sweep0)(b->Bt, nn, nq, g1, nq, nq, t1);
  SFX(sweep1)(b->Dt, nn, nq, t1, nn, nq, t2);
  SFX(sweep2)(b->Bt, nn, nq, t2, nn, nn, t1);
  for (int i = 0; i < nn3; ++i) nodal[i] += t1[i];
  SFX(sweep0)(b->Bt, nn, nq, g2, nq, nq, t1);
  SFX(sweep1)(b->Bt, nn, nq, t1, nn, nq, t2);
  SFX(sweep2)(b->Dt, nn, nq, t2, nn, nn, t1);
  for (int i = 0; i < nn3; ++i) nodal[i] += t1[i];
}

/* ---- element kernels: operator.hpp:468-530 ------------------------------ */

/* qp_cache_for_apply operator.hpp:390-434: builds the bundle at (e,q) for the
 * active strategy. gk = Grad u_k (reference gradient times J0^-1). */
static int SFX(bundle_spatial)(const orc_op* op, int64_t e, int q, const R* gk, SFX(qpc)* c);
static int SFX(bundle)(const orc_op* op, int64_t e, int q, const R* gk, SFX(qpc)* c) {
  if (op->spatial) return SFX(bundle_spatial)(op, e, q, gk, c);
  const int64_t at = e * op->nq3 + q;
  const orc_material mq = orc_mat_at(op, at);
  if (op->strategy == ORC_TENSOR || op->strategy == ORC_SCALAR) {
    const double* sc = op->cache + at * ORC_CACHE_STRIDE;
    c->lnj = (R)sc[ORC_C_LNJ];
    if (op->mat.model != 0) {
      c->jm1 = (R)sc[ORC_C_JM1];
      c->jp = (R)sc[ORC_C_JP];
      c->c1 = (R)sc[ORC_C_C1];
      c->c2 = (R)sc[ORC_C_C2];
    } else {
      c->jm1 = c->jp = c->c1 = c->c2 = (R)0;
    }
    for (int f = 0; f < 2; ++f) {
      c->c3[f] = op->mat.model == 2 ? (R)sc[ORC_C_C3 + f] : (R)0;
      c->istar[f] = op->mat.model == 2 ? (R)sc[ORC_C_IS + f] : (R)0;
      c->efib[f] = op->mat.model == 2 ? (R)sc[ORC_C_EF + f] : (R)0;
    }
    if (op->strategy == ORC_TENSOR) {
      for (int k = 0; k < 9; ++k) {
        c->F[k] = (R)sc[ORC_C_F + k];
        c->Finv[k] = (R)sc[ORC_C_FINV + k];
      }
      for (int k = 0; k < 6; ++k) {
        c->S[k] = (R)sc[ORC_C_S + k];
        c->Cinv[k] = (R)sc[ORC_C_CINV + k];
      }
      return 0;
    }
    /* scalar: strain tensors recomputed from G_k, scalars from storage */
    SFX(qpc) s;
    if (SFX(compute_cache)(&mq, gk, &s)) return 1;
    c->jm1 = s.jm1; /* second_pk_base reads J-1 from the strain state */
    for (int k = 0; k < 9; ++k) {
      c->F[k] = s.F[k];
      c->Finv[k] = s.Finv[k];
    }
    for (int k = 0; k < 6; ++k) {
      c->Cinv[k] = s.Cinv[k];
      c->E[k] = s.E[k];
    }
    SFX(second_pk)(&mq, c, c->S);
    return 0;
  }
  if (SFX(compute_cache)(&mq, gk, c)) return 1;
  SFX(second_pk)(&mq, c, c->S);
  return 0;
}

/* qp_cache_for_apply, spatial cell (operator.hpp:393-434, 362-370):
 * none recomputes, scalar loads the scalars and rebuilds b, tau, F H F^T from
 * G_k, tensor loads tau, b, F H F^T. */
static int SFX(bundle_spatial)(const orc_op* op, int64_t e, int q, const R* gk, SFX(qpc)* c) {
  const int64_t at = e * op->nq3 + q;
  const orc_material mq = orc_mat_at(op, at);
  if (op->strategy == ORC_NONE) {
    if (SFX(compute_cache)(&mq, gk, c)) return 1;
    SFX(spatial_cell)(&mq, c);
    return 0;
  }
  const double* sc = op->cache + at * ORC_CACHE_STRIDE;
  c->lnj = (R)sc[ORC_C_LNJ];
  if (op->mat.model != 0) {
    c->jm1 = (R)sc[ORC_C_JM1];
    c->jp = (R)sc[ORC_C_JP];
    c->c1 = (R)sc[ORC_C_C1];
    c->c2 = (R)sc[ORC_C_C2];
  } else {
    c->jm1 = c->c1 = c->c2 = (R)0;
    c->jp = (R)1;
  }
  for (int f = 0; f < 2; ++f) {
    c->c3[f] = op->mat.model == 2 ? (R)sc[ORC_C_C3 + f] : (R)0;
    c->istar[f] = op->mat.model == 2 ? (R)sc[ORC_C_IS + f] : (R)0;
    c->efib[f] = op->mat.model == 2 ? (R)sc[ORC_C_EF + f] : (R)0;
  }
  if (op->strategy == ORC_TENSOR) {
    for (int k = 0; k < 6; ++k) {
      c->tau[k] = (R)sc[ORC_C_TAU + k];
      c->b[k] = op->mat.model != 0 ? (R)sc[ORC_C_B + k] : (R)0;
      c->fh[0][k] = op->mat.model == 2 ? (R)sc[ORC_C_FH + k] : (R)0;
      c->fh[1][k] = op->mat.model == 2 ? (R)sc[ORC_C_FH + 6 + k] : (R)0;
    }
    return 0;
  }
  SFX(qpc) s;
  if (SFX(compute_cache)(&mq, gk, &s)) return 1;
  c->jm1 = s.jm1; /* kirchhoff_base reads J-1 from the strain state */
  for (int k = 0; k < 9; ++k) c->F[k] = s.F[k];
  for (int k = 0; k < 6; ++k) c->bt[k] = s.bt[k];
  SFX(spatial_cell)(&mq, c);
  return 0;
}

/* Per-element scratch for one element. */
typedef struct {
  R loc[3][ORC_MAXN3], uk[3][ORC_MAXN3], out[3][ORC_MAXN3];
  R g[3][3][ORC_MAXN3], gk[3][3][ORC_MAXN3];
  R work[2 * ORC_MAXN3];
} SFX(scratch);

static void SFX(gather)(const orc_op* op, const R* glob, int64_t e, R loc[3][ORC_MAXN3]) {
  int64_t nodes[ORC_MAXN3];
  orc_element_nodes(op, e, nodes);
  for (int c = 0; c < 3; ++c)
    for (int m = 0; m < op->nn3; ++m) loc[c][m] = glob[3 * nodes[m] + c];
}

/* J0 (double) for (e,q), operator.hpp:289-301: converted to Number, det in Number. */
static void SFX(qp_mapping)(const orc_op* op, int64_t e, int q, R* j0, R* det0) {
  const double* J = op->jac + (e * op->nq3 + q) * 9;
  for (int m = 0; m < 9; ++m) j0[m] = (R)J[m];
  *det0 = SFX(det)(j0);
}

/* element_tangent_batch operator.hpp:468-530 for one element; adds into out. */
static int SFX(element_tangent)(const orc_op* op, int64_t e, const R* input, const R* ukn, SFX(scratch)* s) {
  const orc_basis* b = &op->basis;
  const int nq = b->n, nq3 = op->nq3, nn3 = op->nn3;
  const int need_uk = op->strategy != ORC_TENSOR;
  SFX(gather)(op, input, e, s->loc);
  for (int c = 0; c < 3; ++c) SFX(grad_qp)(b, s->loc[c], s->work, s->g[c][0], s->g[c][1], s->g[c][2]);
  if (need_uk) {
    SFX(gather)(op, ukn, e, s->uk);
    for (int c = 0; c < 3; ++c) SFX(grad_qp)(b, s->uk[c], s->work, s->gk[c][0], s->gk[c][1], s->gk[c][2]);
  }
  for (int c = 0; c < 3; ++c)
    for (int m = 0; m < nn3; ++m) s->out[c][m] = (R)0;
  for (int q = 0; q < nq3; ++q) {
    R j0[9], det0, j0inv[9], gref[9], dg[9], gk[9], ds[6], t1[9], t2[9], wm[9], j0t[9], wr[9];
    const int qa = q % nq, qb = (q / nq) % nq, qc = q / (nq * nq);
    const R wq = (R)(b->qwts[qa] * b->qwts[qb] * b->qwts[qc]);
    if (op->spatial) {
      /* operator.hpp:506-519: grad du = Grad_xi du J_t^-1, w = (1/J) det J_t w_q (.) J_t^-T */
      const double* sc = op->cache + (e * nq3 + q) * ORC_CACHE_STRIDE;
      R jt[9], jtinv[9], wsp[9];
      for (int k = 0; k < 9; ++k) jt[k] = (R)sc[ORC_C_JT + k];
      if (SFX(inverse)(jt, jtinv)) return 2;
      const R detjt = SFX(det)(jt);
      const R invj = (R)sc[ORC_C_INVJ];
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->g[c][d][q];
      SFX(mm)(gref, jtinv, dg);
      if (need_uk) {
        SFX(qp_mapping)(op, e, q, j0, &det0);
        if (SFX(inverse)(j0, j0inv)) return 2;
        for (int c = 0; c < 3; ++c)
          for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->gk[c][d][q];
        SFX(mm)(gref, j0inv, gk);
      }
      SFX(qpc) cache;
      if (SFX(bundle)(op, e, q, gk, &cache)) return 1;
      const orc_material mq = orc_mat_at(op, e * op->nq3 + q);
      SFX(tangent_spatial)(&mq, &cache, dg, wsp);
      SFX(transpose)(jtinv, j0t);
      SFX(mm)(wsp, j0t, wr);
      const R sc2 = (invj * detjt) * wq;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) s->g[c][d][q] = sc2 * wr[3 * c + d];
      continue;
    }
    SFX(qp_mapping)(op, e, q, j0, &det0);
    if (SFX(inverse)(j0, j0inv)) return 2;
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->g[c][d][q];
    SFX(mm)(gref, j0inv, dg);
    if (need_uk) {
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->gk[c][d][q];
      SFX(mm)(gref, j0inv, gk);
    }
    SFX(qpc) cache;
    if (SFX(bundle)(op, e, q, gk, &cache)) return 1;
    const orc_material mq = orc_mat_at(op, e * op->nq3 + q);
    SFX(tangent_material)(&mq, &cache, dg, ds);
    SFX(mm_ts)(dg, cache.S, t1);
    SFX(mm_ts)(cache.F, ds, t2);
    for (int k = 0; k < 9; ++k) wm[k] = t1[k] + t2[k];
    SFX(transpose)(j0inv, j0t);
    SFX(mm)(wm, j0t, wr);
    const R sc = det0 * wq;
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) s->g[c][d][q] = sc * wr[3 * c + d];
  }
  for (int c = 0; c < 3; ++c) SFX(scatter_grad)(b, s->g[c][0], s->g[c][1], s->g[c][2], s->work, s->out[c]);
  return 0;
}

/* apply_tangent operator.hpp:597-621: masked input, y = 0, 8 parity colours
 * in order (each DoF accumulates contributions in colour order), identity
 * on constrained rows. */
static int SFX(apply)(const orc_op* op, const R* du, R* y) {
  const int64_t n = op->ndofs;
  R* masked = (R*)malloc(sizeof(R) * n);
  R* ukn = NULL;
  for (int64_t i = 0; i < n; ++i) {
    masked[i] = op->mask[i] ? (R)0 : du[i];
    y[i] = (R)0;
  }
  if (op->strategy != ORC_TENSOR) {
    ukn = (R*)malloc(sizeof(R) * n);
    for (int64_t i = 0; i < n; ++i) ukn[i] = (R)op->uk[i];
  }
  int err = 0;
  for (int color = 0; color < 8; ++color) {
    const int ci = color & 1, cj = (color >> 1) & 1, ck = (color >> 2) & 1;
    const int nci = (op->nx - ci + 1) / 2, ncj = (op->ny - cj + 1) / 2, nck = (op->nz - ck + 1) / 2;
    const int64_t cnt = (int64_t)nci * ncj * nck;
#pragma omp parallel
    {
      SFX(scratch)* s = (SFX(scratch)*)malloc(sizeof(SFX(scratch)));
#pragma omp for schedule(static)
      for (int64_t t = 0; t < cnt; ++t) {
        const int i = ci + 2 * (int)(t % nci);
        const int j = cj + 2 * (int)((t / nci) % ncj);
        const int k = ck + 2 * (int)(t / ((int64_t)nci * ncj));
        const int64_t e = ((int64_t)k * op->ny + j) * op->nx + i;
        if (SFX(element_tangent)(op, e, masked, ukn, s)) {
#pragma omp atomic write
          err = 1;
          continue;
        }
        int64_t nodes[ORC_MAXN3];
        orc_element_nodes(op, e, nodes);
        for (int c = 0; c < 3; ++c)
          for (int m = 0; m < op->nn3; ++m) y[3 * nodes[m] + c] += s->out[c][m];
      }
      free(s);
    }
  }
  for (int64_t i = 0; i < n; ++i)
    if (op->mask[i]) y[i] = du[i];
  free(masked);
  free(ukn);
  return err;
}

/* element_residual_batch operator.hpp:533-595 (material domain) +
 * evaluate_residual :623-641: r = sum_e (Grad v, F S) in colour order (input
 * NOT masked), r -= load_scale * load (load in Number), Dirichlet rows zeroed. */
static int SFX(residual)(const orc_op* op, const R* u, const double* load, double load_scale, R* r) {
  const int64_t n = op->ndofs;
  const orc_basis* b = &op->basis;
  const int nq = b->n, nq3 = op->nq3, nn3 = op->nn3;
  for (int64_t i = 0; i < n; ++i) r[i] = (R)0;
  int err = 0;
  for (int color = 0; color < 8; ++color) {
    const int ci = color & 1, cj = (color >> 1) & 1, ck = (color >> 2) & 1;
    const int nci = (op->nx - ci + 1) / 2, ncj = (op->ny - cj + 1) / 2, nck = (op->nz - ck + 1) / 2;
    const int64_t cnt = (int64_t)nci * ncj * nck;
#pragma omp parallel
    {
      SFX(scratch)* s = (SFX(scratch)*)malloc(sizeof(SFX(scratch)));
#pragma omp for schedule(static)
      for (int64_t t = 0; t < cnt; ++t) {
        const int i = ci + 2 * (int)(t % nci);
        const int j = cj + 2 * (int)((t / nci) % ncj);
        const int k = ck + 2 * (int)(t / ((int64_t)nci * ncj));
        const int64_t e = ((int64_t)k * op->ny + j) * op->nx + i;
        SFX(gather)(op, u, e, s->loc);
        for (int c = 0; c < 3; ++c) SFX(grad_qp)(b, s->loc[c], s->work, s->g[c][0], s->g[c][1], s->g[c][2]);
        int bad = 0;
        for (int q = 0; q < nq3 && !bad; ++q) {
          R j0[9], det0, j0inv[9], gref[9], g[9], S[6], wm[9], j0t[9], wr[9];
          SFX(qp_mapping)(op, e, q, j0, &det0);
          if (SFX(inverse)(j0, j0inv)) bad = 1;
          for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->g[c][d][q];
          SFX(mm)(gref, j0inv, g);
          const int qa = q % nq, qb = (q / nq) % nq, qc = q / (nq * nq);
          const R wq = (R)(b->qwts[qa] * b->qwts[qb] * b->qwts[qc]);
          const orc_material mq = orc_mat_at(op, e * nq3 + q);
          SFX(qpc) c;
          if (SFX(compute_cache)(&mq, g, &c)) {
            bad = 1;
            break;
          }
          if (op->spatial) {
            /* operator.hpp:572-588: J_t = J0 + Grad_xi u, w = (1/J) det J_t w_q tau J_t^-T */
            R jt[9], jtinv[9], tf[9];
            for (int k = 0; k < 9; ++k) jt[k] = j0[k] + gref[k];
            if (SFX(inverse)(jt, jtinv)) bad = 1;
            const R detjt = SFX(det)(jt);
            const R invj = (R)1 / c.jac;
            SFX(spatial_cell)(&mq, &c);
            for (int i2 = 0; i2 < 3; ++i2)
              for (int j2 = 0; j2 < 3; ++j2) tf[3 * i2 + j2] = c.tau[SFX(sidx)(i2, j2)];
            SFX(transpose)(jtinv, j0t);
            SFX(mm)(tf, j0t, wr);
            const R sc2 = (invj * detjt) * wq;
            for (int cc = 0; cc < 3; ++cc)
              for (int d = 0; d < 3; ++d) s->g[cc][d][q] = sc2 * wr[3 * cc + d];
            continue;
          }
          SFX(second_pk)(&mq, &c, S);
          SFX(mm_ts)(c.F, S, wm);
          SFX(transpose)(j0inv, j0t);
          SFX(mm)(wm, j0t, wr);
          const R sc = det0 * wq;
          for (int cc = 0; cc < 3; ++cc)
            for (int d = 0; d < 3; ++d) s->g[cc][d][q] = sc * wr[3 * cc + d];
        }
        if (bad) {
#pragma omp atomic write
          err = 1;
          continue;
        }
        for (int c = 0; c < 3; ++c)
          for (int m = 0; m < nn3; ++m) s->out[c][m] = (R)0;
        for (int c = 0; c < 3; ++c) SFX(scatter_grad)(b, s->g[c][0], s->g[c][1], s->g[c][2], s->work, s->out[c]);
        int64_t nodes[ORC_MAXN3];
        orc_element_nodes(op, e, nodes);
        for (int c = 0; c < 3; ++c)
          for (int m = 0; m < nn3; ++m) r[3 * nodes[m] + c] += s->out[c][m];
      }
      free(s);
    }
  }
  const R ls = (R)load_scale;
  for (int64_t i = 0; i < n; ++i) {
    r[i] -= ls * (R)load[i];
    if (op->mask[i]) r[i] = (R)0;
  }
  return err;
}

/* compute_diagonal operator.hpp:772-878: 3*(p+1)^3 element-local unit
 * applications per element, (ldof, ldof) entries scattered in colour order. */
static int SFX(diagonal)(const orc_op* op, R* diag, int64_t* n_bad) {
  const int64_t n = op->ndofs;
  const orc_basis* b = &op->basis;
  const int nq = b->n, nq3 = op->nq3, nn3 = op->nn3;
  R* ukn = NULL;
  const int need_uk = op->strategy != ORC_TENSOR;
  for (int64_t i = 0; i < n; ++i) diag[i] = (R)0;
  if (need_uk) {
    ukn = (R*)malloc(sizeof(R) * n);
    for (int64_t i = 0; i < n; ++i) ukn[i] = (R)op->uk[i];
  }
  int err = 0;
  for (int color = 0; color < 8; ++color) {
    const int ci = color & 1, cj = (color >> 1) & 1, ck = (color >> 2) & 1;
    const int nci = (op->nx - ci + 1) / 2, ncj = (op->ny - cj + 1) / 2, nck = (op->nz - ck + 1) / 2;
    const int64_t cnt = (int64_t)nci * ncj * nck;
#pragma omp parallel
    {
      SFX(scratch)* s = (SFX(scratch)*)malloc(sizeof(SFX(scratch)));
      SFX(qpc)* bundles = (SFX(qpc)*)malloc(sizeof(SFX(qpc)) * ORC_MAXN3);
      R* j0inv = (R*)malloc(sizeof(R) * 9 * ORC_MAXN3);
      R* det0w = (R*)malloc(sizeof(R) * ORC_MAXN3);
      R* jts = (R*)malloc(sizeof(R) * 9 * ORC_MAXN3);
#pragma omp for schedule(static)
      for (int64_t t = 0; t < cnt; ++t) {
        const int i = ci + 2 * (int)(t % nci);
        const int j = cj + 2 * (int)((t / nci) % ncj);
        const int k = ck + 2 * (int)(t / ((int64_t)nci * ncj));
        const int64_t e = ((int64_t)k * op->ny + j) * op->nx + i;
        int64_t nodes[ORC_MAXN3];
        orc_element_nodes(op, e, nodes);
        if (need_uk) {
          SFX(gather)(op, ukn, e, s->uk);
          for (int c = 0; c < 3; ++c) SFX(grad_qp)(b, s->uk[c], s->work, s->gk[c][0], s->gk[c][1], s->gk[c][2]);
        }
        int bad = 0;
        for (int q = 0; q < nq3 && !bad; ++q) {
          R j0[9], det0, gref[9], gk[9];
          SFX(qp_mapping)(op, e, q, j0, &det0);
          const int qa = q % nq, qb = (q / nq) % nq, qc = q / (nq * nq);
          const R wq = (R)(b->qwts[qa] * b->qwts[qb] * b->qwts[qc]);
          if (SFX(inverse)(j0, j0inv + 9 * q)) bad = 1;
          if (need_uk) {
            for (int c = 0; c < 3; ++c)
              for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->gk[c][d][q];
            SFX(mm)(gref, j0inv + 9 * q, gk);
          }
          if (SFX(bundle)(op, e, q, gk, &bundles[q])) bad = 1;
          det0w[q] = det0 * wq;
          if (op->spatial) {
            const double* sc = op->cache + (e * nq3 + q) * ORC_CACHE_STRIDE;
            R jt[9];
            for (int k = 0; k < 9; ++k) jt[k] = (R)sc[ORC_C_JT + k];
            if (SFX(inverse)(jt, jts + 9 * q)) bad = 1;
            det0w[q] = ((R)sc[ORC_C_INVJ] * SFX(det)(jt)) * wq;
          }
        }
        if (bad) {
#pragma omp atomic write
          err = 1;
          continue;
        }
        for (int ldof = 0; ldof < 3 * nn3; ++ldof) {
          const int c_in = ldof % 3, m_in = ldof / 3;
          for (int c = 0; c < 3; ++c)
            for (int m = 0; m < nn3; ++m) s->loc[c][m] = (R)((c == c_in && m == m_in) ? 1 : 0);
          for (int c = 0; c < 3; ++c) SFX(grad_qp)(b, s->loc[c], s->work, s->g[c][0], s->g[c][1], s->g[c][2]);
          for (int q = 0; q < nq3; ++q) {
            R gref[9], dg[9], ds[6], t1[9], t2[9], wm[9], jt[9], wr[9];
            for (int c = 0; c < 3; ++c)
              for (int d = 0; d < 3; ++d) gref[3 * c + d] = s->g[c][d][q];
            const orc_material mq = orc_mat_at(op, e * op->nq3 + q);
            if (op->spatial) {
              SFX(mm)(gref, jts + 9 * q, dg);
              SFX(tangent_spatial)(&mq, &bundles[q], dg, wm);
              SFX(transpose)(jts + 9 * q, jt);
              SFX(mm)(wm, jt, wr);
              for (int c = 0; c < 3; ++c)
                for (int d = 0; d < 3; ++d) s->g[c][d][q] = det0w[q] * wr[3 * c + d];
              continue;
            }
            SFX(mm)(gref, j0inv + 9 * q, dg);
            SFX(tangent_material)(&mq, &bundles[q], dg, ds);
            SFX(mm_ts)(dg, bundles[q].S, t1);
            SFX(mm_ts)(bundles[q].F, ds, t2);
            for (int k2 = 0; k2 < 9; ++k2) wm[k2] = t1[k2] + t2[k2];
            SFX(transpose)(j0inv + 9 * q, jt);
            SFX(mm)(wm, jt, wr);
            for (int c = 0; c < 3; ++c)
              for (int d = 0; d < 3; ++d) s->g[c][d][q] = det0w[q] * wr[3 * c + d];
          }
          for (int c = 0; c < 3; ++c)
            for (int m = 0; m < nn3; ++m) s->out[c][m] = (R)0;
          for (int c = 0; c < 3; ++c) SFX(scatter_grad)(b, s->g[c][0], s->g[c][1], s->g[c][2], s->work, s->out[c]);
          diag[3 * nodes[m_in] + c_in] += s->out[c_in][m_in];
        }
      }
      free(s);
      free(bundles);
      free(j0inv);
      free(det0w);
      free(jts);
    }
  }
  int64_t nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (op->mask[i])
      diag[i] = (R)1;
    else if (!(diag[i] > (R)0))
      ++nb;
  }
  *n_bad = nb;
  free(ukn);
  return err;
}

/* Chebyshev-Jacobi smoother, solver.hpp:312-362 (setup :318-326, smooth
 * :330-361). x in/out. */
static int SFX(chebyshev)(const orc_op* op, const R* diag, double lmax_est, int degree, double range_factor,
                         double safety, const R* b, R* x, int zero_start) {
  const int64_t n = op->ndofs;
  const double lambda_max = safety * lmax_est;
  const double lambda_min = lambda_max / range_factor;
  R* inv = (R*)malloc(sizeof(R) * n);
  R* r = (R*)malloc(sizeof(R) * n);
  R* d = (R*)malloc(sizeof(R) * n);
  R* ad = (R*)malloc(sizeof(R) * n);
  for (int64_t i = 0; i < n; ++i) inv[i] = (R)1 / diag[i];
  const double theta = 0.5 * (lambda_max + lambda_min);
  const double delta = 0.5 * (lambda_max - lambda_min);
  const double sigma1 = theta / delta;
  double rho_old = 1.0 / sigma1;
  int err = 0;
  if (zero_start) {
    for (int64_t i = 0; i < n; ++i) {
      r[i] = b[i];
      x[i] = (R)0;
    }
  } else {
    err |= SFX(apply)(op, x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  }
  const R inv_theta = (R)(1.0 / theta);
  for (int64_t i = 0; i < n; ++i) d[i] = (inv_theta * inv[i]) * r[i];
  for (int64_t i = 0; i < n; ++i) x[i] += d[i];
  for (int k = 1; k < degree; ++k) {
    err |= SFX(apply)(op, d, ad);
    for (int64_t i = 0; i < n; ++i) r[i] -= ad[i];
    const double rho_new = 1.0 / (2.0 * sigma1 - rho_old);
    const R f1 = (R)(rho_new * rho_old);
    const R f2 = (R)(2.0 * rho_new / delta);
    for (int64_t i = 0; i < n; ++i) d[i] = f1 * d[i] + (f2 * inv[i]) * r[i];
    for (int64_t i = 0; i < n; ++i) x[i] += d[i];
    rho_old = rho_new;
  }
  free(inv);
  free(r);
  free(d);
  free(ad);
  return err;
}

/* Element-local results of element_tangent_batch (operator.hpp:468-530) for
 * the element range [e0, e1), before the colour-ordered scatter:
 * loc[((e - e0)*nn3 + m)*3 + c].  Used to check the slab decomposition. */
static int SFX(element_locals)(const orc_op* op, const R* du, R* loc, int64_t e0, int64_t e1) {
  const int64_t n = op->ndofs;
  R* masked = (R*)malloc(sizeof(R) * n);
  R* ukn = (R*)malloc(sizeof(R) * n);
  for (int64_t i = 0; i < n; ++i) {
    masked[i] = op->mask[i] ? (R)0 : du[i];
    ukn[i] = (R)op->uk[i];
  }
  int err = 0;
#pragma omp parallel
  {
    SFX(scratch)* s = (SFX(scratch)*)malloc(sizeof(SFX(scratch)));
#pragma omp for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      if (SFX(element_tangent)(op, e, masked, ukn, s)) {
#pragma omp atomic write
        err = 1;
        continue;
      }
      for (int m = 0; m < op->nn3; ++m)
        for (int c = 0; c < 3; ++c) loc[((e - e0) * op->nn3 + m) * 3 + c] = s->out[c][m];
    }
    free(s);
  }
  free(masked);
  free(ukn);
  return err;
}
