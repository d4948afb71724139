// C ABI of libemfgpu.so (include/emfgpu.h): handle lifetime, host setup
// (basis tables, lattice coordinates, material constants), device buffers,
// and stream-ordered orchestration of the kernels.  Host-side error model
// follows the reference C layer (status code + per-handle message,
// proj/src/capi.cpp:26-41); no CPU fallback exists — without a CUDA device
// every create call fails with EMFGPU_ERR_CUDA.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>

#include "capi_util.h"
#include "internal.h"
#include "krylov_core.h"

using namespace emfgpu;
using namespace emfgpu::capi;

namespace {

// ---- 1D basis: Gauss-Lobatto nodes, Gauss rule, Lagrange tables ----------
// Standard Newton iterations on Legendre polynomials (the construction of
// mesh.cpp:14-120), run on the host once per level.
double legendre(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return p0;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}
double dlegendre(int n, double x) {
  if (n == 0) return 0.0;
  return n * (legendre(n - 1, x) - x * legendre(n, x)) / (1.0 - x * x);
}
void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      const double dx = legendre(n, t) / dlegendre(n, t);
      t -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    x[i] = t;
  }
  std::sort(x.begin(), x.end());
  for (int i = 0; i < n; ++i) {
    const double d = dlegendre(n, x[i]);
    w[i] = 2.0 / ((1.0 - x[i] * x[i]) * d * d);
  }
}
std::vector<double> lobatto_nodes(int n) {
  std::vector<double> x(n);
  x[0] = -1.0;
  x[n - 1] = 1.0;
  const int m = n - 1;
  for (int i = 1; i < m; ++i) {
    double t = std::cos(M_PI * (m - i) / m);
    for (int it = 0; it < 100; ++it) {
      const double g = dlegendre(m, t);
      const double gp = (2.0 * t * g - m * (m + 1.0) * legendre(m, t)) / (1.0 - t * t);
      const double dx = g / gp;
      t -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    x[i] = t;
  }
  std::sort(x.begin(), x.end());
  return x;
}
double lagrange(const std::vector<double>& xs, int i, double x) {
  double v = 1.0;
  for (size_t k = 0; k < xs.size(); ++k)
    if ((int)k != i) v *= (x - xs[k]) / (xs[i] - xs[k]);
  return v;
}
double dlagrange(const std::vector<double>& xs, int i, double x) {
  double sum = 0.0;
  for (size_t m = 0; m < xs.size(); ++m) {
    if ((int)m == i) continue;
    double prod = 1.0 / (xs[i] - xs[m]);
    for (size_t k = 0; k < xs.size(); ++k) {
      if ((int)k == i || k == m) continue;
      prod *= (x - xs[k]) / (xs[i] - xs[k]);
    }
    sum += prod;
  }
  return sum;
}

// ---- fibre structure tensors, material.cpp:50-82 (std special functions) --
void structure_tensors(const emfgpu_material& p, double h[2][6], double m1[2][3]) {
  const double h33 = 1.0 / (4.0 * p.b) - std::exp(-2.0 * p.b) / (std::sqrt(2.0 * M_PI * p.b) * std::erf(std::sqrt(2.0 * p.b)));
  const double ratio = p.a == 0.0 ? 0.0 : std::cyl_bessel_i(1.0, p.a) / std::cyl_bessel_i(0.0, p.a);
  const double h11 = 0.5 * (1.0 - h33) * (1.0 + ratio);
  const double h22 = 0.5 * (1.0 - h33) * (1.0 - ratio);
  const double c = std::cos(p.phi), s = std::sin(p.phi);
  double v1[2][3], v2[2][3];
  for (int k = 0; k < 3; ++k) {
    v1[0][k] = c * p.e1[k] + s * p.e2[k];
    v2[0][k] = -s * p.e1[k] + c * p.e2[k];
    v1[1][k] = c * p.e1[k] - s * p.e2[k];
    v2[1][k] = s * p.e1[k] + c * p.e2[k];
  }
  for (int f = 0; f < 2; ++f) {
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 3; ++j)
        h[f][sidx(i, j)] = h11 * (v1[f][i] * v1[f][j]) + h22 * (v2[f][i] * v2[f][j]) + h33 * (p.e3[i] * p.e3[j]);
    for (int k = 0; k < 3; ++k) m1[f][k] = v1[f][k];
  }
}

template <typename T>
MatConst<T> mat_const(const emfgpu_material& p, const double h[2][6], const double m1[2][3]) {
  MatConst<T> m;
  m.mu = T(p.mu);
  m.lam = T(p.lambda);
  m.half_k = T(0.5 * p.kappa_b);
  m.kappa = T(p.kappa_b);
  m.k2 = T(p.k2);
  m.two_k1 = T(2.0 * p.k1);
  // the reference evaluates mu/3, 2mu/9, 2mu/3 in Number (constitutive.hpp:349-352, 404)
  m.mu_3 = T(p.mu) / T(3);
  m.two_mu_9 = (T(2) * T(p.mu)) / T(9);
  m.two_mu_3 = (T(2) * T(p.mu)) / T(3);
  for (int f = 0; f < 2; ++f) {
    for (int k = 0; k < 6; ++k) m.h[f][k] = T(h[f][k]);
    for (int k = 0; k < 3; ++k) m.m1[f][k] = T(m1[f][k]);
  }
  return m;
}

uint64_t fnv1a(const void* data, size_t bytes) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

// EMFGPU_UK_ELEM=0: Q3 u_k gathered from the lattice instead of the
// per-element copy made at linearization (measurement)
static bool uk_el_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("EMFGPU_UK_ELEM");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

template <typename T>
KArgs<T> kargs(const emfgpu_op* op) {
  const emfgpu_level* L = op->L;
  KArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.loc = static_cast<T*>(op->d_loc);
  a.uk = static_cast<const T*>(op->d_uk);
  a.uk_el = static_cast<const T*>(op->d_uk_el);
  a.ukd = op->d_ukd;
  a.geo = std::is_same<T, double>::value ? reinterpret_cast<const T*>(L->d_geo) : reinterpret_cast<const T*>(L->d_geo_f);
  a.geod = L->d_geo;
  a.geo_stride = L->geo_stride;
  a.affine = L->affine;
  a.cache = static_cast<T*>(op->d_cache);
  a.cache_stride = op->cache_stride;
  a.strategy = op->strategy;
  a.nx = L->nx;
  a.ny = L->ny;
  a.nz = L->nz;
  a.mx = L->mx;
  a.my = L->my;
  a.mz = L->mz;
  a.nel = L->nel;
  a.e_begin = 0;
  a.faces = L->faces;
  a.err = op->d_err;
  if constexpr (std::is_same<T, double>::value)
    a.mat = op->matd;
  else
    a.mat = op->matf;
  a.matd = op->matd;
  const int n = L->p + 1;
  for (int t = 0; t < n * n; ++t) {
    a.Bm[t] = T(L->B[t]);  // the reference casts the double tables per use (sumfact.hpp:28-29)
    a.Dm[t] = T(L->D[t]);
    a.Bd[t] = L->B[t];
    a.Dd[t] = L->D[t];
  }
  for (int t = 0; t < n; ++t) a.qwd[t] = L->qwts[t];
  {
    // even-odd halves of B and of the collocated derivative Dc[q][r] =
    // l_r'(g_q) on the Gauss points (D = Dc B, eo_sweeps.cuh)
    const int H = n / 2, CH = (n + 1) / 2;
    auto Bq = [&](int q, int i) { return L->B[q * n + i]; };
    auto Dc = [&](int q, int r) { return L->Dc[q * n + r]; };
    for (int q = 0; q < CH; ++q)
      for (int i = 0; i < CH; ++i)
        a.eoB[q * CH + i] = T(i < H ? 0.5 * (Bq(q, i) + Bq(q, n - 1 - i)) : Bq(q, i));
    for (int q = 0; q < H; ++q)
      for (int i = 0; i < H; ++i) a.eoB[CH * CH + q * H + i] = T(0.5 * (Bq(q, i) - Bq(q, n - 1 - i)));
    for (int q = 0; q < H; ++q)
      for (int i = 0; i < CH; ++i)
        a.eoD[q * CH + i] = T(i < H ? 0.5 * (Dc(q, i) + Dc(q, n - 1 - i)) : Dc(q, i));
    for (int q = 0; q < CH; ++q)
      for (int i = 0; i < H; ++i) a.eoD[H * CH + q * H + i] = T(0.5 * (Dc(q, i) - Dc(q, n - 1 - i)));
    // pairs of the same entries for the packed fp32 sweeps (EoT in eo_sweeps.cuh; H == 2: Q3, Q4)
    for (auto& v : a.eoP) v = make_float2(0.f, 0.f);
    if (H == 2) {
      auto BE = [&](int q, int i) { return (float)a.eoB[q * CH + i]; };
      auto BO = [&](int q, int i) { return (float)a.eoB[CH * CH + q * H + i]; };
      auto DE = [&](int q, int i) { return (float)a.eoD[q * CH + i]; };
      auto DO = [&](int q, int i) { return (float)a.eoD[H * CH + q * H + i]; };
      for (int i = 0; i < CH; ++i) {
        a.eoP[0 + i] = make_float2(BE(0, i), BE(1, i));
        a.eoP[5 + i] = make_float2(DE(0, i), DE(1, i));
        a.eoP[10 + i] = make_float2(BE(i, 0), BE(i, 1));
        a.eoP[15 + i] = make_float2(DO(i, 0), DO(i, 1));
      }
      for (int i = 0; i < H; ++i) {
        a.eoP[3 + i] = make_float2(BO(0, i), BO(1, i));
        a.eoP[8 + i] = make_float2(DO(0, i), DO(1, i));
        a.eoP[13 + i] = make_float2(BO(i, 0), BO(i, 1));
        a.eoP[18 + i] = make_float2(DE(i, 0), DE(i, 1));
      }
    }
  }
  a.cartesian = L->cartesian;
  a.hq = static_cast<const T*>(op->d_hq);
  a.hqd = op->d_hqd;
  a.m1qd = op->d_m1qd;
  a.hq_stride = L->nel * L->nq3;
  a.fd_nx = FastDiv::make((uint32_t)L->nx);
  a.fd_nxy = FastDiv::make((uint32_t)(L->nx * L->ny));
  a.spatial = op->domain;
  a.coords = L->d_coords;
  a.tk = op->d_ctr + 2 * (op->ticket_seq.fetch_add(1, std::memory_order_relaxed) % emfgpu_op::kTicketSlots);
  return a;
}

template <typename T>
void dispatch_apply(const emfgpu_op* op, const KArgs<T>& a, int64_t e0, int64_t e1, cudaStream_t s) {
  const int ks = op->domain ? S_SP_NONE + op->strategy : op->strategy;  // element-kernel strategy code
  switch (op->L->p) {
    case 1: launch_apply<T, 1>(op->model, ks, a, e0, e1, s); break;
    case 2: launch_apply<T, 2>(op->model, ks, a, e0, e1, s); break;
    case 3: launch_apply<T, 3>(op->model, ks, a, e0, e1, s); break;
    case 4: launch_apply<T, 4>(op->model, ks, a, e0, e1, s); break;
  }
}
template <typename T>
void dispatch_linearize(const emfgpu_op* op, const KArgs<T>& a, cudaStream_t s) {
  switch (op->L->p) {
    case 1: launch_linearize<T, 1>(op->model, a, s); break;
    case 2: launch_linearize<T, 2>(op->model, a, s); break;
    case 3: launch_linearize<T, 3>(op->model, a, s); break;
    case 4: launch_linearize<T, 4>(op->model, a, s); break;
  }
}
template <typename T>
void dispatch_residual(const emfgpu_op* op, const KArgs<T>& a, cudaStream_t s) {
  switch (op->L->p) {
    case 1: launch_residual<T, 1>(op->model, a, s); break;
    case 2: launch_residual<T, 2>(op->model, a, s); break;
    case 3: launch_residual<T, 3>(op->model, a, s); break;
    case 4: launch_residual<T, 4>(op->model, a, s); break;
  }
}
template <typename T>
void dispatch_diagonal(const emfgpu_op* op, const KArgs<T>& a, cudaStream_t s) {
  switch (op->L->p) {
    case 1: launch_diagonal<T, 1>(op->model, a, s); break;
    case 2: launch_diagonal<T, 2>(op->model, a, s); break;
    case 3: launch_diagonal<T, 3>(op->model, a, s); break;
    case 4: launch_diagonal<T, 4>(op->model, a, s); break;
  }
}

size_t nsize(const emfgpu_op* op) { return op->precision == 64 ? 8 : 4; }

void require_linearized(const emfgpu_op* op, const char* what) {
  if (!op->linearized)
    throw ApiError(EMFGPU_ERR_STALE, std::string(what) + ": update_linearization has not run");
}

void apply_elements(emfgpu_op* op, const void* x, int k0, int k1, cudaStream_t s) {
  const emfgpu_level* L = op->L;
  const int64_t e0 = (int64_t)k0 * L->nx * L->ny, e1 = (int64_t)k1 * L->nx * L->ny;
  if (op->precision == 64) {
    KArgs<double> a = kargs<double>(op);
    a.x = static_cast<const double*>(x);
    dispatch_apply<double>(op, a, e0, e1, s);
  } else {
    KArgs<float> a = kargs<float>(op);
    a.x = static_cast<const float*>(x);
    dispatch_apply<float>(op, a, e0, e1, s);
  }
  CK(cudaGetLastError());
}

// set while capturing a conditional-graph body (no programmatic edges there)
static thread_local bool tl_no_pdl = false;

// pdl: launch as a programmatic dependent of the preceding element kernel
// (off in the copy-overlapped host pipeline, where it measured 1% slower)
void apply_nodes(emfgpu_op* op, const void* x, void* y, int c0, int c1, const void* glo, const void* ghi, int kpar,
                 cudaStream_t s, bool pdl = true) {
  const emfgpu_level* L = op->L;
  if (op->precision == 64)
    launch_node_gather<double>(static_cast<const double*>(op->d_loc), static_cast<const double*>(glo),
                               static_cast<const double*>(ghi), static_cast<const double*>(x),
                               static_cast<double*>(y), L->nx, L->ny, L->nz, L->p, L->faces, kpar, c0, c1, L->periodic_y, s,
                               pdl && !tl_no_pdl);
  else
    launch_node_gather<float>(static_cast<const float*>(op->d_loc), static_cast<const float*>(glo),
                              static_cast<const float*>(ghi), static_cast<const float*>(x), static_cast<float*>(y),
                              L->nx, L->ny, L->nz, L->p, L->faces, kpar, c0, c1, L->periodic_y, s,
                              pdl && !tl_no_pdl);
  CK(cudaGetLastError());
}

// Whole-lattice apply y = K x: element kernel + node gather.
void apply_full(emfgpu_op* op, const void* x, void* y, cudaStream_t s) {
  const emfgpu_level* L = op->L;
  apply_elements(op, x, 0, L->nz, s);
  apply_nodes(op, x, y, 0, L->mz - 1, nullptr, nullptr, L->z_offset & 1, s);
}

void check_err(emfgpu_op* op, cudaStream_t s, int64_t* be, int* bq, const char* what) {
  CK(cudaMemcpyAsync(op->h_err, op->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const unsigned long long v = *op->h_err;
  if (v != ~0ull) {
    const int64_t e = (int64_t)(v / op->L->nq3);
    const int q = (int)(v % op->L->nq3);
    if (be) *be = e;
    if (bq) *bq = q;
    CK(cudaMemsetAsync(op->d_err, 0xff, sizeof(unsigned long long), s));
    throw ApiError(EMFGPU_ERR_NUMERICAL, std::string(what) + ": det(F) <= 0 element=" + std::to_string(e) +
                                             " qpoint=" + std::to_string(q));
  }
}

}  // namespace

// Phases of the split apply, for the slab layer (slab.cu); no entry ordering
// here: the callers hold the handle's UseGuard.
namespace emfgpu {
namespace capi {
void op_elements(emfgpu_op* op, const void* x, int k0, int k1, cudaStream_t s) { apply_elements(op, x, k0, k1, s); }
void op_nodes(emfgpu_op* op, const void* x, void* y, const void* ghost_lo, const void* ghost_hi, cudaStream_t s) {
  apply_nodes(op, x, y, 0, op->L->mz - 1, ghost_lo, ghost_hi, op->L->z_offset & 1, s);
}
void op_pack_face(emfgpu_op* op, int k, int side, void* face, cudaStream_t s) {
  const emfgpu_level* L = op->L;
  if (op->precision == 64)
    launch_pack_face<double>(static_cast<const double*>(op->d_loc), static_cast<double*>(face), L->nx, L->ny, L->p, k,
                             side, s);
  else
    launch_pack_face<float>(static_cast<const float*>(op->d_loc), static_cast<float*>(face), L->nx, L->ny, L->p, k,
                            side, s);
  CK(cudaGetLastError());
}
}  // namespace capi
}  // namespace emfgpu

// Transfer / smoother handles
struct emfgpu_transfer {
  const emfgpu_level* fine;
  const emfgpu_level* coarse;
  struct Axis {
    int n_src, p_src, n_dst, p_dst;
    int *src_elem = nullptr, *t_ptr = nullptr, *t_d = nullptr, *t_s = nullptr;
    double* w = nullptr;
  } up[3], down[3];
  void* tmp[2] = {nullptr, nullptr};
  size_t tmp_bytes = 0;
  std::string last_error;
  std::recursive_mutex use_mu;  // entry ordering (UseGuard)
  cudaEvent_t ev_use = nullptr;
};

struct emfgpu_cheb {
  emfgpu_op* op;
  int degree;
  double lambda_min, lambda_max;
  void *inv_diag = nullptr, *r = nullptr, *d = nullptr, *ad = nullptr;
};

// Definitions keep the C linkage of their declarations in emfgpu.h.
const char* emfgpu_version(void) { return "emfgpu 0.1 (sm_100a)"; }
const char* emfgpu_global_last_error(void) { return g_error.c_str(); }

// ---------------------------------------------------------------- level ----
emfgpu_status emfgpu_level_create(const emfgpu_level_desc* d, emfgpu_level** out) {
  if (!d || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto L = std::make_unique<emfgpu_level>();
  emfgpu_status st = guarded(nullptr, [&] {
    if (d->p < 1 || d->p > kMaxP) throw ApiError(EMFGPU_ERR_CONFIG, "level: degree must be in 1..4");
    if (d->nx < 1 || d->ny < 1 || d->nz < 1) throw ApiError(EMFGPU_ERR_CONFIG, "level: need nx,ny,nz >= 1");
    if (d->map == EMFGPU_MAP_COORDS && !d->coords) throw ApiError(EMFGPU_ERR_CONFIG, "level: coords missing");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ApiError(EMFGPU_ERR_CUDA, "level: no CUDA device (no CPU fallback by design)");
    CK(cudaSetDevice(d->device));
    L->device = d->device;
    L->nx = d->nx;
    L->ny = d->ny;
    L->nz = d->nz;
    L->p = d->p;
    L->periodic_y = (d->flags & EMFGPU_LEVEL_PERIODIC_Y) ? 1 : 0;
    if (L->periodic_y && ((d->ny % 2) != 0 || d->ny < 2))
      throw ApiError(EMFGPU_ERR_CONFIG, "level: a periodic y lattice needs an even ny >= 2 (colouring)");
    if (L->periodic_y && (d->dirichlet_faces & (4 | 8)))
      throw ApiError(EMFGPU_ERR_CONFIG, "level: no Dirichlet faces across a periodic direction");
    L->mx = d->nx * d->p + 1;
    L->my = d->ny * d->p + (L->periodic_y ? 0 : 1);
    L->mz = d->nz * d->p + 1;
    L->nnodes = (int64_t)L->mx * L->my * L->mz;
    L->ndofs = 3 * L->nnodes;
    L->nel = (int64_t)d->nx * d->ny * d->nz;
    const int n = d->p + 1;
    L->nq3 = n * n * n;
    L->faces = d->dirichlet_faces;
    L->z_offset = d->z_offset;
    L->desc = *d;
    L->desc.coords = nullptr;
    for (int a = 0; a < 3; ++a) L->extent[a] = d->extent[a] > 0 ? d->extent[a] : 1.0;
    L->nodes = lobatto_nodes(n);
    gauss_rule(n, L->qpts, L->qwts);
    L->B.assign(n * n, 0.0);
    L->D.assign(n * n, 0.0);
    for (int q = 0; q < n; ++q)
      for (int i = 0; i < n; ++i) {
        L->B[q * n + i] = lagrange(L->nodes, i, L->qpts[q]);
        L->D[q * n + i] = dlagrange(L->nodes, i, L->qpts[q]);
      }
    L->Dc.assign(n * n, 0.0);
    for (int q = 0; q < n; ++q)
      for (int r = 0; r < n; ++r) L->Dc[q * n + r] = dlagrange(L->qpts, r, L->qpts[q]);
    // lattice coordinates (mesh.cpp:138-160), then the map
    std::vector<double> coords(3 * L->nnodes);
    if (d->map == EMFGPU_MAP_COORDS) {
      std::memcpy(coords.data(), d->coords, coords.size() * sizeof(double));
    } else {
      const int ne[3] = {d->nx, d->ny, d->nz}, m[3] = {L->mx, L->my, L->mz};
      std::vector<double> ax[3];
      for (int a = 0; a < 3; ++a) {
        ax[a].resize(m[a]);
        const double h = L->extent[a] / ne[a];
        for (int idx = 0; idx < m[a]; ++idx) {
          const int e = std::min(idx / d->p, ne[a] - 1);
          const int l = idx - e * d->p;
          ax[a][idx] = (e + 0.5 * (L->nodes[l] + 1.0)) * h;
        }
      }
      const double amp = d->map_param[0];
      const double ext = L->extent[0];
      for (int c = 0; c < m[2]; ++c)
        for (int b = 0; b < m[1]; ++b)
          for (int a = 0; a < m[0]; ++a) {
            const double x = ax[0][a], y = ax[1][b], z = ax[2][c];
            double r0 = x, r1 = y, r2 = z;
            if (d->map == EMFGPU_MAP_REFERENCE && amp != 0.0) {  // DeformMap, mesh.cpp:128-136
              const double s = M_PI / ext, A = amp * ext;
              r0 += A * std::sin(s * y) * std::sin(s * z);
              r1 += A * std::sin(s * x) * std::sin(s * z);
              r2 += A * std::sin(s * x) * std::sin(s * y);
            } else if (d->map == EMFGPU_MAP_SHEAR_X) {
              r0 += amp * std::sin(2.0 * M_PI * y);
            } else if (d->map == EMFGPU_MAP_TUBE) {  // BASELINE cfg3: (radial, theta, axial) lattice
              const double r = d->map_param[0] + (d->map_param[1] - d->map_param[0]) * (x / L->extent[0]);
              const double th = 2.0 * M_PI * (y / L->extent[1]);
              r0 = r * std::cos(th);
              r1 = r * std::sin(th);
              r2 = d->map_param[2] * (z / L->extent[2]);
            }
            const int64_t node = ((int64_t)c * m[1] + b) * m[0] + a;
            coords[3 * node] = r0;
            coords[3 * node + 1] = r1;
            coords[3 * node + 2] = r2;
          }
    }
    CK(cudaMalloc(&L->d_coords, coords.size() * sizeof(double)));
    CK(cudaMemcpy(L->d_coords, coords.data(), coords.size() * sizeof(double), cudaMemcpyHostToDevice));
    const int64_t nqp = L->nel * L->nq3;
    double* geo_q = nullptr;
    int* flags = nullptr;
    CK(cudaMalloc(&geo_q, sizeof(double) * nqp * 11));
    CK(cudaMalloc(&flags, 2 * sizeof(int)));
    CK(cudaMemset(flags, 0, 2 * sizeof(int)));
    launch_geometry(L->d_coords, geo_q, nullptr, L->nx, L->ny, L->nz, L->p, L->B.data(), L->D.data(),
                    L->qwts.data(), flags, flags + 1, L->periodic_y, 0);
    CK(cudaGetLastError());
    int hf[2];
    CK(cudaMemcpy(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost));
    cudaFree(flags);
    if (hf[1]) {
      cudaFree(geo_q);
      throw ApiError(EMFGPU_ERR_NUMERICAL, "level: mapping Jacobian not positive at a quadrature point");
    }
    L->affine = (hf[0] || (d->flags & EMFGPU_LEVEL_NO_AFFINE)) ? 0 : 1;
    if (L->affine) {
      CK(cudaMalloc(&L->d_geo, sizeof(double) * L->nel * 10));
      launch_geo_compact(geo_q, L->d_geo, L->nel, (int)L->nq3, 0);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaFree(geo_q);
      L->geo_stride = L->nel;
      // axis-aligned affine elements: J0^-1 diagonal in every element
      std::vector<double> h(10 * L->nel);
      CK(cudaMemcpy(h.data(), L->d_geo, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
      bool cart = !(d->flags & EMFGPU_LEVEL_NO_CARTESIAN);
      for (int64_t e = 0; e < L->nel && cart; ++e) {
        const double sc = std::max(std::abs(h[e]), std::max(std::abs(h[4 * L->nel + e]), std::abs(h[8 * L->nel + e])));
        for (int m : {1, 2, 3, 5, 6, 7})
          if (std::abs(h[m * L->nel + e]) > 1e-11 * sc) cart = false;
      }
      L->cartesian = cart ? 1 : 0;
    } else {
      L->d_geo = geo_q;  // fields 0..9 used, stride nqp
      L->geo_stride = nqp;
    }
    const int64_t gsz = 10 * L->geo_stride;
    CK(cudaMalloc(&L->d_geo_f, sizeof(float) * gsz));
    launch_cast_d2f(L->d_geo, L->d_geo_f, gsz, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  });
  if (st != EMFGPU_OK) {
    if (L->d_coords) cudaFree(L->d_coords);
    if (L->d_geo) cudaFree(L->d_geo);
    if (L->d_geo_f) cudaFree(L->d_geo_f);
    return st;
  }
  *out = L.release();
  return EMFGPU_OK;
}

void emfgpu_level_destroy(emfgpu_level* l) {
  if (!l) return;
  cudaFree(l->d_coords);
  cudaFree(l->d_geo);
  cudaFree(l->d_geo_f);
  delete l;
}

int64_t emfgpu_level_n_dofs(const emfgpu_level* l) { return l ? l->ndofs : 0; }
int64_t emfgpu_level_n_elements(const emfgpu_level* l) { return l ? l->nel : 0; }
int emfgpu_level_affine(const emfgpu_level* l) { return l ? l->affine : 0; }
int emfgpu_level_cartesian(const emfgpu_level* l) { return l ? l->cartesian : 0; }
const char* emfgpu_level_last_error(const emfgpu_level* l) { return l ? l->last_error.c_str() : ""; }

emfgpu_status emfgpu_level_jacobians(const emfgpu_level* l, double* host_out) {
  if (!l || !host_out) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    CK(cudaSetDevice(l->device));
    const int64_t nqp = l->nel * l->nq3;
    double *geo_q = nullptr, *j0 = nullptr;
    int* flags = nullptr;
    CK(cudaMalloc(&geo_q, sizeof(double) * nqp * 11));
    CK(cudaMalloc(&j0, sizeof(double) * nqp * 9));
    CK(cudaMalloc(&flags, 2 * sizeof(int)));
    launch_geometry(l->d_coords, geo_q, j0, l->nx, l->ny, l->nz, l->p, l->B.data(), l->D.data(), l->qwts.data(),
                    flags, flags + 1, l->periodic_y, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(host_out, j0, sizeof(double) * nqp * 9, cudaMemcpyDeviceToHost));
    cudaFree(geo_q);
    cudaFree(j0);
    cudaFree(flags);
  });
}

emfgpu_status emfgpu_level_coords(const emfgpu_level* l, double* host_out) {
  if (!l || !host_out) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    CK(cudaSetDevice(l->device));
    CK(cudaMemcpy(host_out, l->d_coords, sizeof(double) * l->ndofs, cudaMemcpyDeviceToHost));
  });
}

// ------------------------------------------------------------------- op ----
emfgpu_status emfgpu_op_create(const emfgpu_level* l, int model, const emfgpu_material* params, int domain,
                               int strategy, int precision, emfgpu_op** out) {
  if (!l || !params || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto op = std::make_unique<emfgpu_op>();
  emfgpu_status st = guarded(nullptr, [&] {
    if (model < 0 || model > 2) throw ApiError(EMFGPU_ERR_CONFIG, "op: unknown model");
    if (domain != 0 && domain != 1) throw ApiError(EMFGPU_ERR_CONFIG, "op: domain must be 0 (material) or 1 (spatial)");
    if (strategy < 0 || strategy > 3) throw ApiError(EMFGPU_ERR_CONFIG, "op: unknown strategy");
    if (domain == 1 && strategy == EMFGPU_CACHED_F)
      throw ApiError(EMFGPU_ERR_CONFIG, "op: the cachedF strategy is material-domain only");
    if (precision != 64 && precision != 32) throw ApiError(EMFGPU_ERR_CONFIG, "op: precision must be 64 or 32");
    // MaterialParams::validate, material.cpp:36-48
    if (!(params->mu > 0)) throw ApiError(EMFGPU_ERR_CONFIG, "MaterialParams: mu must be positive");
    if (model != 0 && !(params->kappa_b > 0)) throw ApiError(EMFGPU_ERR_CONFIG, "MaterialParams: kappa_b must be positive");
    if (model == 2) {
      if (!(params->k2 > 0)) throw ApiError(EMFGPU_ERR_CONFIG, "MaterialParams: k2 must be positive");
      if (!(params->a > 0) || !(params->b > 0))
        throw ApiError(EMFGPU_ERR_CONFIG, "build_structure_tensors: a and b must be positive");
      auto dot3 = [](const double* u, const double* v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; };
      const double tol = 1e-12;
      if (std::abs(dot3(params->e1, params->e1) - 1) > tol || std::abs(dot3(params->e2, params->e2) - 1) > tol ||
          std::abs(dot3(params->e3, params->e3) - 1) > tol || std::abs(dot3(params->e1, params->e2)) > tol ||
          std::abs(dot3(params->e1, params->e3)) > tol || std::abs(dot3(params->e2, params->e3)) > tol)
        throw ApiError(EMFGPU_ERR_CONFIG, "MaterialParams: frame {e1,e2,e3} not orthonormal");
    }
    CK(cudaSetDevice(l->device));
    op->L = l;
    op->model = model;
    op->strategy = strategy;
    op->domain = domain;
    op->precision = precision;
    op->params = *params;
    double h[2][6] = {}, m1[2][3] = {};
    if (model == 2) structure_tensors(*params, h, m1);
    op->matd = mat_const<double>(*params, h, m1);
    op->matf = mat_const<float>(*params, h, m1);
    const size_t ns = nsize(op.get());
    CK(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&op->d_loc, ns * l->nel * l->nq3 * 3));
    CK(cudaMalloc(&op->d_ctr, sizeof(unsigned) * 2 * emfgpu_op::kTicketSlots));
    CK(cudaMemset(op->d_ctr, 0, sizeof(unsigned) * 2 * emfgpu_op::kTicketSlots));
    CK(cudaMalloc(&op->d_err, sizeof(unsigned long long)));
    CK(cudaMemset(op->d_err, 0xff, sizeof(unsigned long long)));
    CK(cudaMalloc(&op->d_nbad, sizeof(unsigned long long)));
    CK(cudaMallocHost(&op->h_err, sizeof(unsigned long long)));
    CK(cudaMalloc(&op->d_ukd, sizeof(double) * l->ndofs));
    if (strategy == EMFGPU_NONE || strategy == EMFGPU_SCALAR) {
      CK(cudaMalloc(&op->d_uk, ns * l->ndofs));
      // per-element u_k copy: 1.3% slower for fp64, which keeps the gather;
      // for fp32 re-measured on the collocated v2 kernel (EMFGPU_UK_ELEM=0/1):
      // cfg1 none 0.0973 -> 0.0932 ms with the copy, scalar 0.0973 -> 0.0932,
      // curved iNH 0.1036 -> 0.1014 (31.5 MB read as 16-byte copies instead of
      // 11 MB of scattered 4-byte words)
      if (l->p == 3 && precision == 32 && uk_el_enabled())
        CK(cudaMalloc(&op->d_uk_el, ns * l->nel * 3 * (ns == 8 ? 82 : 80)));
    }
    int nf = strategy == EMFGPU_TENSOR ? (tensor_compact(model, domain) ? tensor_compact_fields(model) : C_NT)
             : strategy == EMFGPU_SCALAR ? 8 : strategy == EMFGPU_CACHED_F ? C_NG : 0;
    if (domain == 1) nf = strategy == EMFGPU_TENSOR ? C_NSP : C_JT + 9;  // J_t, 1/J always (operator.hpp:690-691)
    op->n_cache_fields = nf;
    op->cache_stride = l->nel * l->nq3;
    if (nf) CK(cudaMalloc(&op->d_cache, ns * nf * op->cache_stride));
  });
  if (st != EMFGPU_OK) {
    emfgpu_op_destroy(op.release());
    return st;
  }
  *out = op.release();
  return EMFGPU_OK;
}

emfgpu_status emfgpu_op_create_ex(const emfgpu_level* l, int model, const emfgpu_material* params,
                                  const emfgpu_formulation* form, int strategy, int precision,
                                  const emfgpu_kernel_config* kc, emfgpu_op** out) {
  if (!l || !params || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto reject = [](const std::string& what) {
    g_error = "op: " + what + " is not implemented by the device kernels (stable formulation, default KernelConfig)";
    return EMFGPU_ERR_CONFIG;
  };
  if (form && form->stability != 1) return reject("Formulation::stability = standard");
  if (kc) {
    if (kc->ln_series_terms != 16) return reject("KernelConfig::ln_series_terms != 16");
    if (kc->jpow_newton_steps != 3) return reject("KernelConfig::jpow_newton_steps != 3");
    if (kc->exp_mode != 0) return reject("KernelConfig::exp_mode = fast");
    if (kc->jpow_mode != 0) return reject("KernelConfig::jpow_mode = exact");
  }
  return emfgpu_op_create(l, model, params, form ? form->domain : 0, strategy, precision, out);
}

void emfgpu_op_destroy(emfgpu_op* op) {
  if (!op) return;
  cudaFree(op->d_cache);
  if (op->d_hq && op->d_hq != op->d_hqd) cudaFree(op->d_hq);
  cudaFree(op->d_hqd);  // d_m1qd points into it
  cudaFree(op->d_uk);
  cudaFree(op->d_uk_el);
  cudaFree(op->d_ukd);
  cudaFree(op->d_loc);
  cudaFree(op->d_ctr);
  cudaFree(op->d_x);
  cudaFree(op->d_y);
  cudaFree(op->d_load);
  cudaFree(op->lz_buf);
  cudaFree(op->pcg_buf);
  cudaFree(op->fgmres_buf);
  cudaFree(op->d_err);
  cudaFree(op->d_nbad);
  if (op->h_err) cudaFreeHost(op->h_err);
  if (op->stream) cudaStreamDestroy(op->stream);
  if (op->s_h2d) cudaStreamDestroy(op->s_h2d);
  if (op->s_d2h) cudaStreamDestroy(op->s_d2h);
  if (op->ev_start) cudaEventDestroy(op->ev_start);
  if (op->ev_done) cudaEventDestroy(op->ev_done);
  if (op->ev_use) cudaEventDestroy(op->ev_use);
  if (op->gexec) cudaGraphExecDestroy(op->gexec);
  for (int i = 0; i < emfgpu_op::kMaxChunks; ++i) {
    if (op->ev_h2d[i]) cudaEventDestroy(op->ev_h2d[i]);
    if (op->ev_comp[i]) cudaEventDestroy(op->ev_comp[i]);
  }
  delete op;
}

int64_t emfgpu_op_n_dofs(const emfgpu_op* op) { return op ? op->L->ndofs : 0; }
int emfgpu_op_precision(const emfgpu_op* op) { return op ? op->precision : 0; }
const char* emfgpu_op_last_error(const emfgpu_op* op) { return op ? op->last_error.c_str() : ""; }
int emfgpu_op_linearized(const emfgpu_op* op) { return op && op->linearized ? 1 : 0; }
uint64_t emfgpu_op_checksum(const emfgpu_op* op) {
  if (!op) return 0;
  if (!op->checksum_valid) {
    // on demand, from the device copy of the linearization point
    std::unique_lock<std::recursive_mutex> lk(const_cast<emfgpu_op*>(op)->use_mu);
    std::vector<double> tmp((size_t)op->L->ndofs);
    if (cudaSetDevice(op->L->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(tmp.data(), op->d_ukd, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    op->checksum = fnv1a(tmp.data(), sizeof(double) * tmp.size());
    op->checksum_valid = true;
  }
  return op->checksum;
}

static void linearize_impl(emfgpu_op* op, int64_t* be, int* bq, cudaStream_t s) {
  const emfgpu_level* L = op->L;
  op->linearized = false;
  if (op->d_uk) {
    if (op->precision == 64)
      CK(cudaMemcpyAsync(op->d_uk, op->d_ukd, sizeof(double) * L->ndofs, cudaMemcpyDeviceToDevice, s));
    else
      launch_cast_d2f(op->d_ukd, static_cast<float*>(op->d_uk), L->ndofs, s);
    if (op->d_uk_el) {
      if (op->precision == 64)
        launch_uk_elem<double>(static_cast<const double*>(op->d_uk), static_cast<double*>(op->d_uk_el), L->nel, L->nx,
                               L->ny, L->mx, L->my, 82, s);
      else
        launch_uk_elem<float>(static_cast<const float*>(op->d_uk), static_cast<float*>(op->d_uk_el), L->nel, L->nx,
                              L->ny, L->mx, L->my, 80, s);
    }
  }
  if (op->precision == 64)
    dispatch_linearize<double>(op, kargs<double>(op), s);
  else
    dispatch_linearize<float>(op, kargs<float>(op), s);
  CK(cudaGetLastError());
  check_err(op, s, be, bq, "update_linearization");
  op->linearized = true;
}

emfgpu_status emfgpu_op_update_linearization_host(emfgpu_op* op, const double* u_k, int64_t* be, int* bq) {
  if (!op || !u_k) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, op->stream);
    CK(cudaMemcpyAsync(op->d_ukd, u_k, sizeof(double) * op->L->ndofs, cudaMemcpyHostToDevice, op->stream));
    op->checksum_valid = false;
    linearize_impl(op, be, bq, op->stream);
  });
}

emfgpu_status emfgpu_op_update_linearization(emfgpu_op* op, const double* d_u_k, int64_t* be, int* bq,
                                             void* stream) {
  if (!op || !d_u_k) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    cudaStream_t s = S(stream, op->stream);
    OP_USE(op, s);
    CK(cudaMemcpyAsync(op->d_ukd, d_u_k, sizeof(double) * op->L->ndofs, cudaMemcpyDeviceToDevice, s));
    op->checksum_valid = false;
    linearize_impl(op, be, bq, s);
  });
}

emfgpu_status emfgpu_op_apply(emfgpu_op* op, const void* d_x, void* d_y, void* stream) {
  if (!op || !d_x || !d_y) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    require_linearized(op, "apply_tangent");
    cudaStream_t s = S(stream, op->stream);
    OP_USE(op, s);
    apply_full(op, d_x, d_y, s);
  });
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host-vector apply.  With page-locked x and y the lattice is cut into z
// chunks of element layers and three streams overlap (i) H2D of the next
// chunk's node planes, (ii) the element + node phases of the current chunk,
// (iii) D2H of the node planes the previous chunks finalised.  PCIe copies run
// on both copy engines concurrently; the result is bitwise the one-shot apply.
static void apply_host_pipelined(emfgpu_op* op, const void* x, void* y) {
  const emfgpu_level* L = op->L;
  const size_t plane = nsize(op) * 3 * (size_t)L->mx * L->my;
  const char* hx = static_cast<const char*>(x);
  char* hy = static_cast<char*>(y);
  char* dx = static_cast<char*>(op->d_x);
  char* dy = static_cast<char*>(op->d_y);
  if (!op->s_h2d) {
    CK(cudaStreamCreateWithFlags(&op->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&op->s_d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&op->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&op->ev_done, cudaEventDisableTiming));
    for (int i = 0; i < emfgpu_op::kMaxChunks; ++i) {
      CK(cudaEventCreateWithFlags(&op->ev_h2d[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&op->ev_comp[i], cudaEventDisableTiming));
    }
  }
  static const int env_chunks = [] {
    const char* e = std::getenv("EMFGPU_E2E_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  const int want = env_chunks > 0 ? env_chunks : std::max(1, L->nz / 4);
  const int nch = std::min(std::min(emfgpu_op::kMaxChunks, L->nz), want);
  const int per = (L->nz + nch - 1) / nch;
  // Replay the captured pipeline for the same host buffers (no per-call
  // launch overhead); the first call for a buffer pair runs eagerly, the
  // second one captures.
  if (op->gexec && op->g_x == x && op->g_y == y && op->g_nch == nch) {
    CK(cudaGraphLaunch(op->gexec, op->stream));
    CK(cudaStreamSynchronize(op->stream));
    return;
  }
  const bool capture = op->g_x == x && op->g_y == y && op->g_nch == nch;
  if (op->gexec) {
    cudaGraphExecDestroy(op->gexec);
    op->gexec = nullptr;
  }
  op->g_x = x;
  op->g_y = y;
  op->g_nch = nch;
  if (capture) CK(cudaStreamBeginCapture(op->stream, cudaStreamCaptureModeThreadLocal));
  CK(cudaEventRecord(op->ev_start, op->stream));
  CK(cudaStreamWaitEvent(op->s_h2d, op->ev_start, 0));
  int done_hi = -1;  // highest node plane copied in so far
  for (int i = 0; i < nch; ++i) {
    const int k1 = std::min(L->nz, (i + 1) * per);
    const int hi = k1 * L->p;
    if (hi > done_hi) {
      CK(cudaMemcpyAsync(dx + (done_hi + 1) * plane, hx + (done_hi + 1) * plane, (hi - done_hi) * plane,
                         cudaMemcpyHostToDevice, op->s_h2d));
      done_hi = hi;
    }
    CK(cudaEventRecord(op->ev_h2d[i], op->s_h2d));
  }
  for (int i = 0; i < nch; ++i) {
    const int k0 = i * per, k1 = std::min(L->nz, (i + 1) * per);
    if (k0 >= k1) break;
    const int c0 = k0 * L->p, c1 = (k1 == L->nz) ? L->mz - 1 : k1 * L->p - 1;
    CK(cudaStreamWaitEvent(op->stream, op->ev_h2d[i], 0));
    apply_elements(op, op->d_x, k0, k1, op->stream);
    apply_nodes(op, op->d_x, op->d_y, c0, c1, nullptr, nullptr, 0, op->stream, false);
    CK(cudaEventRecord(op->ev_comp[i], op->stream));
    CK(cudaStreamWaitEvent(op->s_d2h, op->ev_comp[i], 0));
    CK(cudaMemcpyAsync(hy + c0 * plane, dy + c0 * plane, (c1 - c0 + 1) * plane, cudaMemcpyDeviceToHost,
                       op->s_d2h));
  }
  CK(cudaEventRecord(op->ev_done, op->s_d2h));
  CK(cudaStreamWaitEvent(op->stream, op->ev_done, 0));
  if (capture) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(op->stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&op->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      op->gexec = nullptr;
      throw ApiError(EMFGPU_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
    CK(cudaGraphLaunch(op->gexec, op->stream));
  }
  CK(cudaStreamSynchronize(op->stream));
}

emfgpu_status emfgpu_op_apply_host(emfgpu_op* op, const void* x, void* y) {
  if (!op || !x || !y) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    require_linearized(op, "apply_tangent");
    OP_USE(op, op->stream);
    const size_t bytes = nsize(op) * op->L->ndofs;
    if (!op->d_x) CK(cudaMalloc(&op->d_x, bytes));
    if (!op->d_y) CK(cudaMalloc(&op->d_y, bytes));
    if (op->L->nz >= 8 && is_pinned(x) && is_pinned(y)) {
      apply_host_pipelined(op, x, y);
    } else {
      CK(cudaMemcpyAsync(op->d_x, x, bytes, cudaMemcpyHostToDevice, op->stream));
      apply_full(op, op->d_x, op->d_y, op->stream);
      CK(cudaMemcpyAsync(y, op->d_y, bytes, cudaMemcpyDeviceToHost, op->stream));
    }
    check_err(op, op->stream, nullptr, nullptr, "apply_tangent");
  });
}

emfgpu_status emfgpu_op_check(emfgpu_op* op, int64_t* be, int* bq) {
  if (!op) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, op->stream);
    CK(cudaDeviceSynchronize());
    check_err(op, op->stream, be, bq, "apply_tangent");
  });
}

static void diagonal_impl(emfgpu_op* op, void* d_diag, int64_t* nbad, cudaStream_t s, int64_t* h_idx = nullptr,
                          int64_t cap = 0) {
  require_linearized(op, "compute_diagonal");
  const emfgpu_level* L = op->L;
  // the counter lives in the handle (calls on a handle are ordered): no
  // stream-ordered allocation, whose pool trims at every synchronisation
  unsigned long long* const d_nbad = op->d_nbad;
  long long* d_idx = nullptr;
  CK(cudaMemsetAsync(d_nbad, 0, sizeof(unsigned long long), s));
  if (h_idx && cap > 0) CK(cudaMallocAsync(&d_idx, sizeof(long long) * cap, s));
  if (op->precision == 64) {
    dispatch_diagonal<double>(op, kargs<double>(op), s);
    double* d = static_cast<double*>(d_diag);
    launch_node_gather<double>(static_cast<const double*>(op->d_loc), nullptr, nullptr, d, d, L->nx, L->ny, L->nz,
                               L->p, 0, 0, 0, L->mz - 1, L->periodic_y, s);
    launch_diag_finish<double>(d, L->nnodes, L->mx, L->my, L->mz, L->faces, d_nbad, d_idx, cap, s);
  } else {
    dispatch_diagonal<float>(op, kargs<float>(op), s);
    float* d = static_cast<float*>(d_diag);
    launch_node_gather<float>(static_cast<const float*>(op->d_loc), nullptr, nullptr, d, d, L->nx, L->ny, L->nz,
                              L->p, 0, 0, 0, L->mz - 1, L->periodic_y, s);
    launch_diag_finish<float>(d, L->nnodes, L->mx, L->my, L->mz, L->faces, d_nbad, d_idx, cap, s);
  }
  CK(cudaGetLastError());
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(op->h_err, d_nbad, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  h = *op->h_err;
  *op->h_err = ~0ull;
  if (nbad) *nbad = (int64_t)h;
  if (d_idx) {
    // compute_diagonal's second member: the nonpositive free rows in
    // ascending DoF order (operator.hpp:869-877)
    const int64_t m = std::min<int64_t>((int64_t)h, cap);
    std::vector<long long> tmp(m);
    if (m) CK(cudaMemcpyAsync(tmp.data(), d_idx, sizeof(long long) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_idx, s));
    CK(cudaStreamSynchronize(s));
    std::sort(tmp.begin(), tmp.end());
    for (int64_t i = 0; i < m; ++i) h_idx[i] = tmp[i];
  }
}

emfgpu_status emfgpu_op_compute_diagonal(emfgpu_op* op, void* d_diag, int64_t* nbad, void* stream) {
  if (!op || !d_diag) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, S(stream, op->stream));
    diagonal_impl(op, d_diag, nbad, S(stream, op->stream));
  });
}

emfgpu_status emfgpu_op_compute_diagonal_indices(emfgpu_op* op, void* d_diag, int64_t* nonpositive_idx,
                                                 int64_t capacity, int64_t* n_nonpositive, void* stream) {
  if (!op || !d_diag || (capacity > 0 && !nonpositive_idx) || capacity < 0) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, S(stream, op->stream));
    diagonal_impl(op, d_diag, n_nonpositive, S(stream, op->stream), nonpositive_idx, capacity);
  });
}

emfgpu_status emfgpu_op_compute_diagonal_host(emfgpu_op* op, void* diag, int64_t* nbad) {
  if (!op || !diag) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, op->stream);
    const size_t bytes = nsize(op) * op->L->ndofs;
    if (!op->d_y) CK(cudaMalloc(&op->d_y, bytes));
    diagonal_impl(op, op->d_y, nbad, op->stream);
    CK(cudaMemcpy(diag, op->d_y, bytes, cudaMemcpyDeviceToHost));
  });
}

// Per-qp bytes of the cell as stored here (the reference ledger, ledger.cpp:22-76,
// with our SoA fields): geometry 80 B per qp (J0^-1 + det*w) or per element if
// affine, u_k per DoF, caches per qp.
emfgpu_status emfgpu_op_ledger(const emfgpu_op* op, int* storage, int* traffic, double* per_dof) {
  if (!op) return EMFGPU_ERR_INVALID;
  const emfgpu_level* L = op->L;
  const int s = (int)nsize(op);
  int fields = 0;
  if (op->strategy == EMFGPU_CACHED_F) fields = 9;
  if (op->strategy == EMFGPU_SCALAR || op->strategy == EMFGPU_TENSOR)
    fields = (op->model == 0 ? 1 : 3) + (op->model == 2 ? 4 : 0);
  if (op->strategy == EMFGPU_TENSOR) fields += 30;
  bool need_geo = true;
  if (op->strategy == EMFGPU_TENSOR && tensor_compact(op->model, op->domain)) {
    fields = tensor_compact_fields(op->model);  // the push-forward state carries the geometry
    need_geo = false;
  }
  if (op->domain == 1) {  // ledger.cpp:27-70 spatial rows: J_t + 1/J always, tau/b/FHF^T for tensor
    fields = 10;
    if (op->strategy != EMFGPU_NONE) fields += (op->model == 0 ? 1 : 3) + (op->model == 2 ? 4 : 0);
    if (op->strategy == EMFGPU_TENSOR) fields += 6 + (op->model != 0 ? 6 : 0) + (op->model == 2 ? 12 : 0);
    need_geo = op->strategy != EMFGPU_TENSOR;  // J0 only maps Grad u_k
  }
  const int geo = (L->affine || !need_geo) ? 0 : 10 * s;
  if (storage) *storage = geo + fields * s;
  if (traffic) *traffic = geo + fields * s;
  if (per_dof) {
    const bool uk = op->strategy == EMFGPU_NONE || op->strategy == EMFGPU_SCALAR;
    const double qp = (double)(geo + fields * s) * L->nel * L->nq3;
    const double el = (L->affine && need_geo) ? 10.0 * s * L->nel : 0.0;
    *per_dof = (qp + el) / L->ndofs + (uk ? 3 : 2) * s;
  }
  return EMFGPU_OK;
}

// ---- split apply (z slabs) --------------------------------------------------
emfgpu_status emfgpu_op_apply_elements(emfgpu_op* op, const void* d_x, int k0, int k1, void* stream) {
  if (!op || !d_x) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    require_linearized(op, "apply_tangent");
    if (k0 < 0 || k1 > op->L->nz || k0 > k1) throw ApiError(EMFGPU_ERR_CONFIG, "apply_elements: bad layer range");
    OP_USE(op, S(stream, op->stream));
    apply_elements(op, d_x, k0, k1, S(stream, op->stream));
  });
}

emfgpu_status emfgpu_op_apply_nodes(emfgpu_op* op, const void* d_x, void* d_y, int c0, int c1, const void* glo,
                                    const void* ghi, void* stream) {
  if (!op || !d_x || !d_y) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (c0 < 0 || c1 >= op->L->mz || c0 > c1) throw ApiError(EMFGPU_ERR_CONFIG, "apply_nodes: bad plane range");
    OP_USE(op, S(stream, op->stream));
    apply_nodes(op, d_x, d_y, c0, c1, glo, ghi, op->L->z_offset & 1, S(stream, op->stream));
  });
}

void* emfgpu_op_local_buffer(emfgpu_op* op) { return op ? op->d_loc : nullptr; }
int64_t emfgpu_op_face_values(const emfgpu_op* op) {
  return op ? (int64_t)op->L->nx * op->L->ny * (op->L->p + 1) * (op->L->p + 1) * 3 : 0;
}

emfgpu_status emfgpu_op_pack_face(emfgpu_op* op, int k, int side, void* d_face, void* stream) {
  if (!op || !d_face) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    const emfgpu_level* L = op->L;
    if (k < 0 || k >= L->nz) throw ApiError(EMFGPU_ERR_CONFIG, "pack_face: bad layer");
    cudaStream_t s = S(stream, op->stream);
    OP_USE(op, s);
    if (op->precision == 64)
      launch_pack_face<double>(static_cast<const double*>(op->d_loc), static_cast<double*>(d_face), L->nx, L->ny,
                               L->p, k, side, s);
    else
      launch_pack_face<float>(static_cast<const float*>(op->d_loc), static_cast<float*>(d_face), L->nx, L->ny, L->p,
                              k, side, s);
    CK(cudaGetLastError());
  });
}

// ---- transfers (mesh.hpp:157-289, mesh.cpp:248-288) ---------------------------
static void build_axis(emfgpu_transfer::Axis& ax, int n_src, int p_src, int n_dst, int p_dst) {
  ax.n_src = n_src;
  ax.p_src = p_src;
  ax.n_dst = n_dst;
  ax.p_dst = p_dst;
  const std::vector<double> sn = lobatto_nodes(p_src + 1), dn = lobatto_nodes(p_dst + 1);
  const int nd = n_dst * p_dst + 1, stencil = p_src + 1, ns = n_src * p_src + 1;
  std::vector<int> se(nd);
  std::vector<double> w((size_t)nd * stencil);
  for (int d = 0; d < nd; ++d) {
    const int e_dst = std::min(d / p_dst, n_dst - 1);
    const int l_dst = d - e_dst * p_dst;
    const double s = (e_dst + 0.5 * (dn[l_dst] + 1.0)) / n_dst;
    int e_src = std::min((int)(s * n_src), n_src - 1);
    if (e_src > 0 && s * n_src <= e_src) e_src = e_src - (s * n_src < e_src);
    const double xi = 2.0 * (s * n_src - e_src) - 1.0;
    se[d] = e_src;
    for (int i = 0; i < stencil; ++i) w[(size_t)d * stencil + i] = lagrange(sn, i, xi);
  }
  // transposed CSR: for each source index t, the (d, s) pairs in ascending d
  std::vector<std::vector<std::pair<int, int>>> lists(ns);
  for (int d = 0; d < nd; ++d)
    for (int s = 0; s < stencil; ++s) lists[se[d] * p_src + s].push_back({d, s});
  std::vector<int> ptr(ns + 1, 0), td, ts;
  for (int t = 0; t < ns; ++t) {
    ptr[t + 1] = ptr[t] + (int)lists[t].size();
    for (auto& pr : lists[t]) {
      td.push_back(pr.first);
      ts.push_back(pr.second);
    }
  }
  CK(cudaMalloc(&ax.src_elem, sizeof(int) * nd));
  CK(cudaMalloc(&ax.w, sizeof(double) * w.size()));
  CK(cudaMalloc(&ax.t_ptr, sizeof(int) * ptr.size()));
  CK(cudaMalloc(&ax.t_d, sizeof(int) * std::max<size_t>(1, td.size())));
  CK(cudaMalloc(&ax.t_s, sizeof(int) * std::max<size_t>(1, ts.size())));
  CK(cudaMemcpy(ax.src_elem, se.data(), sizeof(int) * nd, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ax.w, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ax.t_ptr, ptr.data(), sizeof(int) * ptr.size(), cudaMemcpyHostToDevice));
  if (!td.empty()) {
    CK(cudaMemcpy(ax.t_d, td.data(), sizeof(int) * td.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ax.t_s, ts.data(), sizeof(int) * ts.size(), cudaMemcpyHostToDevice));
  }
}

static void free_axis(emfgpu_transfer::Axis& ax) {
  cudaFree(ax.src_elem);
  cudaFree(ax.w);
  cudaFree(ax.t_ptr);
  cudaFree(ax.t_d);
  cudaFree(ax.t_s);
}

emfgpu_status emfgpu_transfer_create(const emfgpu_level* fine, const emfgpu_level* coarse, emfgpu_transfer** out) {
  if (!fine || !coarse || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto t = std::make_unique<emfgpu_transfer>();
  emfgpu_status st = guarded(nullptr, [&] {
    const int nf[3] = {fine->nx, fine->ny, fine->nz}, nc[3] = {coarse->nx, coarse->ny, coarse->nz};
    if (fine->periodic_y || coarse->periodic_y)
      throw ApiError(EMFGPU_ERR_CONFIG, "TransferOp: periodic lattices are not supported");
    const bool p_step = nf[0] == nc[0] && nf[1] == nc[1] && nf[2] == nc[2] && fine->p > coarse->p;
    const bool h_step = fine->p == coarse->p && nf[0] == 2 * nc[0] && nf[1] == 2 * nc[1] && nf[2] == 2 * nc[2];
    if (!p_step && !h_step)
      throw ApiError(EMFGPU_ERR_CONFIG, "TransferOp: levels must differ by a p-coarsening or one uniform refinement");
    CK(cudaSetDevice(fine->device));
    t->fine = fine;
    t->coarse = coarse;
    for (int a = 0; a < 3; ++a) {
      build_axis(t->up[a], nc[a], coarse->p, nf[a], fine->p);
      build_axis(t->down[a], nf[a], fine->p, nc[a], coarse->p);
    }
    t->tmp_bytes = sizeof(double) * 3 * (size_t)std::max(fine->mx, coarse->mx) * std::max(fine->my, coarse->my) *
                   std::max(fine->mz, coarse->mz);
    CK(cudaMalloc(&t->tmp[0], t->tmp_bytes));
    CK(cudaMalloc(&t->tmp[1], t->tmp_bytes));
  });
  if (st != EMFGPU_OK) {
    emfgpu_transfer_destroy(t.release());
    return st;
  }
  *out = t.release();
  return EMFGPU_OK;
}

void emfgpu_transfer_destroy(emfgpu_transfer* t) {
  if (!t) return;
  if (t->ev_use) cudaEventDestroy(t->ev_use);
  for (int a = 0; a < 3; ++a) {
    free_axis(t->up[a]);
    free_axis(t->down[a]);
  }
  cudaFree(t->tmp[0]);
  cudaFree(t->tmp[1]);
  delete t;
}

template <typename T>
static void transfer_run(emfgpu_transfer* t, int kind, const T* in, T* out, cudaStream_t s) {
  // apply_axes (mesh.hpp:245-271): axis 0, then 1, then 2; source/destination
  // lattices are coarse->fine (prolongate), fine->coarse (restrict, transposed
  // up-map; interpolate_down, down-map).
  const emfgpu_level* src = kind == 0 ? t->coarse : t->fine;
  const emfgpu_level* dst = kind == 0 ? t->fine : t->coarse;
  const emfgpu_transfer::Axis* ax = kind == 2 ? t->down : t->up;
  const int transpose = kind == 1;
  const int ms[3] = {src->mx, src->my, src->mz}, md[3] = {dst->mx, dst->my, dst->mz};
  T* b0 = static_cast<T*>(t->tmp[0]);
  T* b1 = static_cast<T*>(t->tmp[1]);
  launch_transfer_axis<T>(in, b0, ax[0].src_elem, ax[0].w, ax[0].t_ptr, ax[0].t_d, ax[0].t_s, ax[0].p_src + 1,
                          ax[0].p_src, transpose, 0, ms[0], ms[1], ms[2], md[0], s);
  launch_transfer_axis<T>(b0, b1, ax[1].src_elem, ax[1].w, ax[1].t_ptr, ax[1].t_d, ax[1].t_s, ax[1].p_src + 1,
                          ax[1].p_src, transpose, 1, md[0], ms[1], ms[2], md[1], s);
  launch_transfer_axis<T>(b1, out, ax[2].src_elem, ax[2].w, ax[2].t_ptr, ax[2].t_d, ax[2].t_s, ax[2].p_src + 1,
                          ax[2].p_src, transpose, 2, md[0], md[1], ms[2], md[2], s);
}

emfgpu_status emfgpu_transfer_apply(emfgpu_transfer* t, int kind, int precision, const void* in, void* out,
                                    void* stream) {
  if (!t || !in || !out) return EMFGPU_ERR_INVALID;
  return guarded(&t->last_error, [&] {
    if (kind < 0 || kind > 2) throw ApiError(EMFGPU_ERR_CONFIG, "transfer: kind must be 0,1,2");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    UseGuard g(t->use_mu, t->ev_use, s, t->fine->device);
    if (precision == 64)
      transfer_run<double>(t, kind, static_cast<const double*>(in), static_cast<double*>(out), s);
    else if (precision == 32)
      transfer_run<float>(t, kind, static_cast<const float*>(in), static_cast<float*>(out), s);
    else
      throw ApiError(EMFGPU_ERR_CONFIG, "transfer: precision must be 64 or 32");
    CK(cudaGetLastError());
  });
}

// ---- Chebyshev (solver.hpp:312-362) -----------------------------------------
emfgpu_status emfgpu_cheb_create(emfgpu_op* op, const void* d_diag, double lmax_est, int degree, double range_factor,
                                 double safety, emfgpu_cheb** out) {
  if (!op || !d_diag || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto c = std::make_unique<emfgpu_cheb>();
  emfgpu_status st = guarded(&op->last_error, [&] {
    if (degree < 1) throw ApiError(EMFGPU_ERR_CONFIG, "chebyshev: degree must be >= 1");
    CK(cudaSetDevice(op->L->device));
    c->op = op;
    c->degree = degree;
    c->lambda_max = safety * lmax_est;
    c->lambda_min = c->lambda_max / range_factor;
    const size_t bytes = nsize(op) * op->L->ndofs;
    CK(cudaMalloc(&c->inv_diag, bytes));
    CK(cudaMalloc(&c->r, bytes));
    CK(cudaMalloc(&c->d, bytes));
    CK(cudaMalloc(&c->ad, bytes));
    if (op->precision == 64)
      launch_inv<double>(static_cast<const double*>(d_diag), static_cast<double*>(c->inv_diag), op->L->ndofs,
                         op->stream);
    else
      launch_inv<float>(static_cast<const float*>(d_diag), static_cast<float*>(c->inv_diag), op->L->ndofs, op->stream);
    CK(cudaStreamSynchronize(op->stream));
  });
  if (st != EMFGPU_OK) {
    emfgpu_cheb_destroy(c.release());
    return st;
  }
  *out = c.release();
  return EMFGPU_OK;
}

void emfgpu_cheb_destroy(emfgpu_cheb* c) {
  if (!c) return;
  cudaFree(c->inv_diag);
  cudaFree(c->r);
  cudaFree(c->d);
  cudaFree(c->ad);
  delete c;
}

template <typename T>
static void cheb_run(emfgpu_cheb* c, T* x, const T* b, int zero_start, cudaStream_t s) {
  emfgpu_op* op = c->op;
  const int64_t n = op->L->ndofs;
  const double theta = 0.5 * (c->lambda_max + c->lambda_min);
  const double delta = 0.5 * (c->lambda_max - c->lambda_min);
  const double sigma1 = theta / delta;
  double rho_old = 1.0 / sigma1;
  T* r = static_cast<T*>(c->r);
  T* d = static_cast<T*>(c->d);
  T* ad = static_cast<T*>(c->ad);
  const T* inv = static_cast<const T*>(c->inv_diag);
  if (!zero_start) {
    apply_full(op, x, r, s);
  }
  launch_cheb_first<T>(x, r, d, b, inv, 1.0 / theta, zero_start, n, s);
  for (int k = 1; k < c->degree; ++k) {
    apply_full(op, d, ad, s);
    const double rho_new = 1.0 / (2.0 * sigma1 - rho_old);
    launch_cheb_step<T>(x, r, d, ad, inv, rho_new * rho_old, 2.0 * rho_new / delta, n, s);
    rho_old = rho_new;
  }
}

emfgpu_status emfgpu_cheb_smooth(emfgpu_cheb* c, void* d_x, const void* d_b, int zero_start, void* stream) {
  if (!c || !d_x || !d_b) return EMFGPU_ERR_INVALID;
  return guarded(&c->op->last_error, [&] {
    require_linearized(c->op, "chebyshev");
    cudaStream_t s = S(stream, c->op->stream);
    OP_USE(c->op, s);
    if (c->op->precision == 64)
      cheb_run<double>(c, static_cast<double*>(d_x), static_cast<const double*>(d_b), zero_start, s);
    else
      cheb_run<float>(c, static_cast<float*>(d_x), static_cast<const float*>(d_b), zero_start, s);
    CK(cudaGetLastError());
  });
}

// ---- dot & Lanczos (solver.hpp:95-106, 235-308) --------------------------------
emfgpu_status emfgpu_dot(int precision, const void* a, const void* b, int64_t n, double* out, void* stream) {
  if (!a || !b || !out) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* buf = nullptr;
    CK(cudaMallocAsync(&buf, sizeof(double) * (dot_partial_count() + 1), s));
    if (precision == 64)
      launch_dot<double>(static_cast<const double*>(a), static_cast<const double*>(b), n, buf + 1, buf, s);
    else
      launch_dot<float>(static_cast<const float*>(a), static_cast<const float*>(b), n, buf + 1, buf, s);
    CK(cudaMemcpyAsync(out, buf, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(buf, s));
    CK(cudaStreamSynchronize(s));
  });
}



template <typename T>
static void lanczos(emfgpu_op* op, const T* diag, int iterations, uint64_t seed, double* lmin, double* lmax,
                    cudaStream_t s) {
  // estimate_eigenvalues (solver.hpp:262-308) on one GPU: the generic
  // device-resident core (krylov_core.h) with the whole-lattice apply and the
  // node-plane-chunked dot (bitwise the z-slab dot, csrc/slab_solver.cu)
  const emfgpu_level* L = op->L;
  const int64_t n = L->ndofs;
  const size_t need = lanczos_work_bytes<T>(n, iterations, L->mz);
  if (op->lz_bytes < need) {
    cudaFree(op->lz_buf);
    op->lz_buf = nullptr;
    op->lz_bytes = 0;
    CK(cudaMalloc(&op->lz_buf, need));
    op->lz_bytes = need;
  }
  const int64_t plane = 3 * (int64_t)L->mx * L->my;
  auto apply = [&](const T* x, T* y) { apply_full(op, x, y, s); };
  auto dot = [&](const double* a, const double* b, double* part, double* out) {
    launch_dot_planes<double>(a, b, plane, L->mz, part, out, s);
  };
  // the reorthogonalisation against the whole basis in two launches (krylov_core.h)
  const size_t nd = (size_t)std::max(dot_partial_count(), L->mz * dot_plane_split()) + 1;
  auto reorth = [&](double* w, const double* basis, int k, double* h, double* part) {
    launch_multi_dot_planes(w, basis, n, k, plane, L->mz, part, (int64_t)nd, h, s);
    launch_multi_axpy_dev(h, basis, n, k, w, n, s);
  };
  lanczos_core<T>(n, 0, L->mz, op->lz_buf, diag, iterations, seed, apply, dot, lmin, lmax, s, reorth);
}

emfgpu_status emfgpu_op_estimate_eigenvalues(emfgpu_op* op, const void* d_diag, int iterations, uint64_t seed,
                                             double* lmin, double* lmax) {
  if (!op || !d_diag || !lmin || !lmax) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    require_linearized(op, "estimate_eigenvalues");
    OP_USE(op, op->stream);
    if (op->precision == 64)
      lanczos<double>(op, static_cast<const double*>(d_diag), iterations, seed, lmin, lmax, op->stream);
    else
      lanczos<float>(op, static_cast<const float*>(d_diag), iterations, seed, lmin, lmax, op->stream);
  });
}


// ============================================================================
// hp-multigrid hierarchy (MgHierarchy, solver.hpp:437-581) and outer PCG
// ============================================================================
struct emfgpu_mg {
  std::recursive_mutex use_mu;  // entry ordering (UseGuard)
  cudaEvent_t ev_use = nullptr;
  emfgpu_mg_config cfg{};
  const emfgpu_level* fine = nullptr;
  std::vector<emfgpu_level*> owned;
  std::vector<const emfgpu_level*> lv;
  std::vector<emfgpu_op*> ops;
  std::vector<emfgpu_transfer*> tr;  // tr[l]: lv[l] (fine) <-> lv[l+1] (coarse)
  std::vector<emfgpu_cheb*> cheb;
  std::vector<void*> diag, x, b, t;
  std::vector<double*> u;
  void *cg_r = nullptr, *cg_z = nullptr, *cg_p = nullptr, *cg_ap = nullptr, *cg_inv = nullptr;
  double* dbuf = nullptr;
  double* hdot = nullptr;  // pinned
  int coarse_iterations = 0;
  // dense coarse solve (CoarseSolver dense path): assembled matrix and [I | A^-1]
  bool dense = false;
  double* d_A = nullptr;
  double* d_M = nullptr;
  int* d_sing = nullptr;
  // V-cycle captured as a CUDA graph (dense coarse solve: no host syncs
  // inside), keyed on the (r, z) buffers; dropped on relinearization, whose
  // eigenvalue bounds are baked into the Chebyshev launches
  cudaGraphExec_t vc_exec = nullptr;
  const double* vc_r = nullptr;
  double* vc_z = nullptr;
  cudaStream_t vc_stream = nullptr;
  cudaEvent_t vc_ev[2] = {nullptr, nullptr};
  std::string last_error;
};

namespace {

double mg_dot_sync(double* dbuf, double* hdot, cudaStream_t s) {
  CK(cudaMemcpyAsync(hdot, dbuf, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return *hdot;
}

template <typename T>
double devdot(emfgpu_mg* m, const T* a, const T* b, int64_t n, cudaStream_t s) {
  launch_dot<T>(a, b, n, m->dbuf + 1, m->dbuf, s);
  return mg_dot_sync(m->dbuf, m->hdot, s);
}

template <typename T>
void op_apply_T(emfgpu_op* op, const T* x, T* y, cudaStream_t s) {
  apply_full(op, x, y, s);
}

template <typename T>
void mask0(const emfgpu_level* L, T* v, cudaStream_t s) {
  launch_mask_zero<T>(v, L->nnodes, L->mx, L->my, L->mz, L->faces, s);
}

// CoarseSolver::solve, Jacobi-PCG path (solver.hpp:393-424)
template <typename T>
void coarse_cg(emfgpu_mg* m, int l, cudaStream_t s) {
  emfgpu_op* op = m->ops[l];
  const int64_t n = op->L->ndofs;
  T* x = static_cast<T*>(m->x[l]);
  const T* b = static_cast<const T*>(m->b[l]);
  T *r = static_cast<T*>(m->cg_r), *z = static_cast<T*>(m->cg_z), *p = static_cast<T*>(m->cg_p),
    *ap = static_cast<T*>(m->cg_ap);
  const T* inv = static_cast<const T*>(m->cg_inv);
  CK(cudaMemsetAsync(x, 0, sizeof(T) * n, s));
  CK(cudaMemcpyAsync(r, b, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  const double bnorm = std::sqrt(devdot<T>(m, b, b, n, s));
  m->coarse_iterations = 0;
  if (bnorm == 0) return;
  launch_jacobi<T>(inv, r, z, n, s);
  CK(cudaMemcpyAsync(p, z, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
  double rz = devdot<T>(m, r, z, n, s);
  for (int it = 0; it < m->cfg.coarse_maxit; ++it) {
    op_apply_T<T>(op, p, ap, s);
    const double alpha = rz / devdot<T>(m, p, ap, n, s);
    launch_cg_xr<T>(x, r, p, ap, alpha, n, s);
    m->coarse_iterations = it + 1;
    if (std::sqrt(devdot<T>(m, r, r, n, s)) <= m->cfg.coarse_rtol * bnorm) return;
    launch_jacobi<T>(inv, r, z, n, s);
    const double rz_new = devdot<T>(m, r, z, n, s);
    const double beta = rz_new / rz;
    rz = rz_new;
    launch_cg_p<T>(p, z, beta, n, s);
  }
  throw ApiError(EMFGPU_ERR_NUMERICAL, "coarse CG: no convergence");
}

// MgHierarchy::v_cycle (solver.hpp:544-569)
template <typename T>
void v_cycle(emfgpu_mg* m, int l, cudaStream_t s) {
  const emfgpu_level* L = m->lv[l];
  const int64_t n = L->ndofs;
  T* x = static_cast<T*>(m->x[l]);
  T* b = static_cast<T*>(m->b[l]);
  T* t = static_cast<T*>(m->t[l]);
  if (l + 1 == (int)m->lv.size()) {
    if (m->dense)
      launch_coarse_gemv<T>(m->d_M, b, x, (int)n, s);
    else
      coarse_cg<T>(m, l, s);
    return;
  }
  CK(cudaMemsetAsync(x, 0, sizeof(T) * n, s));
  cheb_run<T>(m->cheb[l], x, b, 1, s);
  op_apply_T<T>(m->ops[l], x, t, s);
  launch_bminus<T>(b, t, n, s);
  mask0<T>(L, t, s);
  T* bc = static_cast<T*>(m->b[l + 1]);
  transfer_run<T>(m->tr[l], 1, t, bc, s);
  mask0<T>(m->lv[l + 1], bc, s);
  v_cycle<T>(m, l + 1, s);
  transfer_run<T>(m->tr[l], 0, static_cast<const T*>(m->x[l + 1]), t, s);
  mask0<T>(L, t, s);
  launch_add<T>(t, x, n, s);
  cheb_run<T>(m->cheb[l], x, b, 0, s);
}

template <typename T>
void mg_precondition(emfgpu_mg* m, const double* r, double* z, cudaStream_t s) {
  const emfgpu_level* L = m->lv[0];
  T* b0 = static_cast<T*>(m->b[0]);
  launch_cast<double, T>(r, b0, L->ndofs, s);
  mask0<T>(L, b0, s);
  v_cycle<T>(m, 0, s);
  launch_cast<T, double>(static_cast<const T*>(m->x[0]), z, L->ndofs, s);
  CK(cudaGetLastError());
}

// CoarseSolver::prepare, dense path (solver.hpp:369-383): the coarse tangent
// assembled by probing (3 (2p+1)^3 applies, columns identical to the
// reference's unit-vector applies), then inverted in double.
template <typename T>
void dense_coarse(emfgpu_mg* m, int l, cudaStream_t s) {
  emfgpu_op* op = m->ops[l];
  const emfgpu_level* L = m->lv[l];
  const int64_t n = L->ndofs;
  const int sp = 2 * L->p + 1;
  T* x = static_cast<T*>(m->cg_p);
  T* y = static_cast<T*>(m->cg_ap);
  CK(cudaMemsetAsync(m->d_A, 0, sizeof(double) * n * n, s));
  for (int cc = 0; cc < sp; ++cc)
    for (int cb = 0; cb < sp; ++cb)
      for (int ca = 0; ca < sp; ++ca)
        for (int comp = 0; comp < 3; ++comp) {
          launch_probe_fill<T>(x, L->mx, L->my, L->mz, sp, ca, cb, cc, comp, s);
          op_apply_T<T>(op, x, y, s);
          launch_probe_extract<T>(y, m->d_A, n, L->mx, L->my, L->mz, L->p, sp, ca, cb, cc, comp, s);
        }
  CK(cudaMemsetAsync(m->d_sing, 0, sizeof(int), s));
  launch_dense_invert(m->d_A, m->d_M, (int)n, m->d_sing, s);
  CK(cudaGetLastError());
  int sing = 0;
  CK(cudaMemcpyAsync(&sing, m->d_sing, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (sing) throw ApiError(EMFGPU_ERR_NUMERICAL, "DenseLU: zero pivot (singular coarse matrix)");
}

template <typename T>
void mg_linearize(emfgpu_mg* m, const double* d_u, cudaStream_t s) {
  const int nl = (int)m->lv.size();
  // a cached V-cycle graph carries the old smoother coefficients as kernel
  // arguments: every relinearisation (update_linearization, the Newton loop,
  // the slab solver) drops it
  if (m->vc_exec) cudaGraphExecDestroy(m->vc_exec);
  m->vc_exec = nullptr;
  m->vc_r = nullptr;
  m->vc_z = nullptr;
  CK(cudaMemcpyAsync(m->u[0], d_u, sizeof(double) * m->lv[0]->ndofs, cudaMemcpyDeviceToDevice, s));
  // EMFGPU_TRACE=1: per-level stage times of the setup (synchronising; diagnostics only)
  static const bool trace = std::getenv("EMFGPU_TRACE") != nullptr;
  auto now = [&]() {
    if (trace) cudaStreamSynchronize(s);
    return std::chrono::steady_clock::now();
  };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  for (int l = 0; l < nl; ++l) {
    emfgpu_op* op = m->ops[l];
    const auto t0 = now();
    if (l > 0) {
      transfer_run<double>(m->tr[l - 1], 2, m->u[l - 1], m->u[l], s);
      mask0<double>(m->lv[l], m->u[l], s);  // dirichlet_set_values (zero)
    }
    CK(cudaMemcpyAsync(op->d_ukd, m->u[l], sizeof(double) * m->lv[l]->ndofs, cudaMemcpyDeviceToDevice, s));
    int64_t be = -1;
    int bq = -1;
    linearize_impl(op, &be, &bq, s);
    const auto t1 = now();
    int64_t nbad = 0;
    diagonal_impl(op, m->diag[l], &nbad, s);
    const auto t2 = now();
    double lmin = 0, lmax = 0;
    lanczos<T>(op, static_cast<const T*>(m->diag[l]), m->cfg.eig_iterations, m->cfg.seed, &lmin, &lmax, s);
    if (trace) {
      const auto t3 = now();
      std::fprintf(stderr, "[emfgpu] mg level %d (%lld dofs): linearize %.2f ms, diagonal %.2f ms, lanczos %.2f ms\n", l,
                   (long long)m->lv[l]->ndofs, ms(t0, t1), ms(t1, t2), ms(t2, t3));
    }
    if (l + 1 < nl) {
      if (m->cheb[l] && m->cheb[l]->op == op && m->cheb[l]->degree == m->cfg.degree) {
        // relinearisation: the smoother keeps its vectors (no cudaFree / cudaMalloc
        // round trips), only the spectrum bounds and 1/diag change
        emfgpu_cheb* c = m->cheb[l];
        c->lambda_max = m->cfg.safety * lmax;
        c->lambda_min = c->lambda_max / m->cfg.range_factor;
        launch_inv<T>(static_cast<const T*>(m->diag[l]), static_cast<T*>(c->inv_diag), m->lv[l]->ndofs, s);
      } else {
        if (m->cheb[l]) emfgpu_cheb_destroy(m->cheb[l]);
        m->cheb[l] = nullptr;
        if (emfgpu_cheb_create(op, m->diag[l], lmax, m->cfg.degree, m->cfg.range_factor, m->cfg.safety,
                               &m->cheb[l]) != EMFGPU_OK)
          throw ApiError(EMFGPU_ERR_CUDA, "mg: smoother setup failed");
      }
    } else if (m->dense) {
      const auto t4 = now();
      dense_coarse<T>(m, l, s);
      if (trace) std::fprintf(stderr, "[emfgpu] mg dense coarse setup %.2f ms\n", ms(t4, now()));
    } else {
      launch_inv<T>(static_cast<const T*>(m->diag[l]), static_cast<T*>(m->cg_inv), m->lv[l]->ndofs, s);
    }
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

// Pieces of the single-GPU operator and hierarchy used by the z-slab solver
// (slab_solver.cu); callers hold the handles' ordering themselves.
namespace emfgpu {
namespace capi {
void op_diag_elements(emfgpu_op* op, cudaStream_t s) {
  if (op->precision == 64)
    dispatch_diagonal<double>(op, kargs<double>(op), s);
  else
    dispatch_diagonal<float>(op, kargs<float>(op), s);
  CK(cudaGetLastError());
}
template <typename T>
void transfer_apply_T(emfgpu_transfer* t, int kind, const T* in, T* out, cudaStream_t s) {
  transfer_run<T>(t, kind, in, out, s);
  CK(cudaGetLastError());
}
template void transfer_apply_T<double>(emfgpu_transfer*, int, const double*, double*, cudaStream_t);
template void transfer_apply_T<float>(emfgpu_transfer*, int, const float*, float*, cudaStream_t);
void mg_linearize_any(emfgpu_mg* m, const double* d_u, cudaStream_t s) {
  if (m->cfg.precision == 64)
    mg_linearize<double>(m, d_u, s);
  else
    mg_linearize<float>(m, d_u, s);
}
void mg_vcycle0(emfgpu_mg* m, cudaStream_t s) {
  if (m->cfg.precision == 64)
    v_cycle<double>(m, 0, s);
  else
    v_cycle<float>(m, 0, s);
  CK(cudaGetLastError());
}
void* mg_b0(emfgpu_mg* m) { return m->b[0]; }
void* mg_x0(emfgpu_mg* m) { return m->x[0]; }
}  // namespace capi
}  // namespace emfgpu

void emfgpu_mg_default_config(emfgpu_mg_config* c) {
  if (!c) return;
  c->degree = 6;
  c->range_factor = 15.0;
  c->safety = 1.2;
  c->eig_iterations = 20;
  c->seed = 0x9e3779b97f4a7c15ull;
  c->coarse_rtol = 1e-4;
  c->coarse_maxit = 500;
  c->coarse_n = 1;
  c->coarse_direct_limit = 2000;
  c->precision = 32;
}

void emfgpu_mg_destroy(emfgpu_mg* m) {
  if (!m) return;
  if (m->ev_use) cudaEventDestroy(m->ev_use);
  for (auto* c : m->cheb) emfgpu_cheb_destroy(c);
  for (auto* t : m->tr) emfgpu_transfer_destroy(t);
  for (auto* o : m->ops) emfgpu_op_destroy(o);
  for (auto* L : m->owned) emfgpu_level_destroy(L);
  for (auto* v : m->diag) cudaFree(v);
  for (auto* v : m->x) cudaFree(v);
  for (auto* v : m->b) cudaFree(v);
  for (auto* v : m->t) cudaFree(v);
  for (auto* v : m->u) cudaFree(v);
  cudaFree(m->cg_r);
  cudaFree(m->cg_z);
  cudaFree(m->cg_p);
  cudaFree(m->cg_ap);
  cudaFree(m->cg_inv);
  cudaFree(m->d_A);
  cudaFree(m->d_M);
  cudaFree(m->d_sing);
  cudaFree(m->dbuf);
  if (m->hdot) cudaFreeHost(m->hdot);
  if (m->vc_exec) cudaGraphExecDestroy(m->vc_exec);
  if (m->vc_stream) cudaStreamDestroy(m->vc_stream);
  for (auto ev : m->vc_ev)
    if (ev) cudaEventDestroy(ev);
  delete m;
}

emfgpu_status emfgpu_mg_create(const emfgpu_level* fine, int model, const emfgpu_material* params, int strategy,
                               const emfgpu_mg_config* cfg, emfgpu_mg** out) {
  if (!fine || !params || !out) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto* m = new emfgpu_mg;
  if (cfg)
    m->cfg = *cfg;
  else
    emfgpu_mg_default_config(&m->cfg);
  emfgpu_status st = guarded(nullptr, [&] {
    if (fine->desc.map == EMFGPU_MAP_COORDS)
      throw ApiError(EMFGPU_ERR_CONFIG, "mg: coarse levels need a generated map (reference / shear_x)");
    if (fine->z_offset != 0) throw ApiError(EMFGPU_ERR_CONFIG, "mg: slab levels are not supported");
    if (m->cfg.precision != 32 && m->cfg.precision != 64) throw ApiError(EMFGPU_ERR_CONFIG, "mg: precision");
    CK(cudaSetDevice(fine->device));
    m->fine = fine;
    m->lv.push_back(fine);
    // ladder p -> p/2 -> ... -> 1, then uniform h-coarsening (solver.hpp:447-459)
    emfgpu_level_desc d = fine->desc;
    d.coords = nullptr;
    int p = fine->p;
    auto add_level = [&](const emfgpu_level_desc& dd) {
      emfgpu_level* L = nullptr;
      const emfgpu_status s2 = emfgpu_level_create(&dd, &L);
      if (s2 != EMFGPU_OK) throw ApiError(s2, std::string("mg: level: ") + emfgpu_global_last_error());
      m->owned.push_back(L);
      m->lv.push_back(L);
    };
    while (p > 1) {
      p /= 2;
      d.p = p;
      add_level(d);
    }
    const int cn = std::max(1, m->cfg.coarse_n);
    while (d.nx % 2 == 0 && d.ny % 2 == 0 && d.nz % 2 == 0 && d.nx / 2 >= cn && d.ny / 2 >= cn &&
           d.nz / 2 >= cn) {
      d.nx /= 2;
      d.ny /= 2;
      d.nz /= 2;
      add_level(d);
    }
    const int nl = (int)m->lv.size();
    const size_t ts = m->cfg.precision == 64 ? 8 : 4;
    for (int l = 0; l < nl; ++l) {
      emfgpu_op* op = nullptr;
      const emfgpu_status s2 = emfgpu_op_create(m->lv[l], model, params, 0, strategy, m->cfg.precision, &op);
      if (s2 != EMFGPU_OK) throw ApiError(s2, std::string("mg: operator: ") + emfgpu_global_last_error());
      m->ops.push_back(op);
      if (l + 1 < nl) {
        emfgpu_transfer* t = nullptr;
        const emfgpu_status s3 = emfgpu_transfer_create(m->lv[l], m->lv[l + 1], &t);
        if (s3 != EMFGPU_OK) throw ApiError(s3, "mg: transfer");
        m->tr.push_back(t);
      }
      const int64_t n = m->lv[l]->ndofs;
      void *dg, *x, *b, *t;
      double* u;
      CK(cudaMalloc(&dg, ts * n));
      CK(cudaMalloc(&x, ts * n));
      CK(cudaMalloc(&b, ts * n));
      CK(cudaMalloc(&t, ts * n));
      CK(cudaMalloc(&u, sizeof(double) * n));
      m->diag.push_back(dg);
      m->x.push_back(x);
      m->b.push_back(b);
      m->t.push_back(t);
      m->u.push_back(u);
    }
    m->cheb.assign(nl, nullptr);
    const int64_t nc = m->lv.back()->ndofs;
    CK(cudaMalloc(&m->cg_r, ts * nc));
    CK(cudaMalloc(&m->cg_z, ts * nc));
    CK(cudaMalloc(&m->cg_p, ts * nc));
    CK(cudaMalloc(&m->cg_ap, ts * nc));
    CK(cudaMalloc(&m->cg_inv, ts * nc));
    CK(cudaMalloc(&m->dbuf, sizeof(double) * (dot_partial_count() + 1)));
    CK(cudaMallocHost(&m->hdot, sizeof(double)));
    m->dense = nc < m->cfg.coarse_direct_limit;  // CoarseSolver::prepare, solver.hpp:373
    if (m->dense) {
      CK(cudaMalloc(&m->d_A, sizeof(double) * nc * nc));
      CK(cudaMalloc(&m->d_M, sizeof(double) * 2 * nc * nc));
      CK(cudaMalloc(&m->d_sing, sizeof(int)));
    }
  });
  if (st != EMFGPU_OK) {
    emfgpu_mg_destroy(m);
    return st;
  }
  *out = m;
  return EMFGPU_OK;
}

int emfgpu_mg_n_levels(const emfgpu_mg* m) { return m ? (int)m->lv.size() : 0; }

emfgpu_status emfgpu_mg_level_info(const emfgpu_mg* m, int l, int* nx, int* ny, int* nz, int* p, int64_t* ndofs) {
  if (!m || l < 0 || l >= (int)m->lv.size()) return EMFGPU_ERR_INVALID;
  const emfgpu_level* L = m->lv[l];
  if (nx) *nx = L->nx;
  if (ny) *ny = L->ny;
  if (nz) *nz = L->nz;
  if (p) *p = L->p;
  if (ndofs) *ndofs = L->ndofs;
  return EMFGPU_OK;
}

const char* emfgpu_mg_last_error(const emfgpu_mg* m) { return m ? m->last_error.c_str() : ""; }

static void mg_drop_graph(emfgpu_mg* m) {
  if (m->vc_exec) cudaGraphExecDestroy(m->vc_exec);
  m->vc_exec = nullptr;
  m->vc_r = nullptr;
  m->vc_z = nullptr;
}

emfgpu_status emfgpu_mg_update_linearization(emfgpu_mg* m, const double* d_u_fine, void* stream) {
  if (!m || !d_u_fine) return EMFGPU_ERR_INVALID;
  return guarded(&m->last_error, [&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    UseGuard g(m->use_mu, m->ev_use, s, m->fine->device);
    mg_drop_graph(m);
    if (m->cfg.precision == 64)
      mg_linearize<double>(m, d_u_fine, s);
    else
      mg_linearize<float>(m, d_u_fine, s);
  });
}

static bool mg_graphs_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("EMFGPU_MG_GRAPH");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

// One V-cycle z = M^-1 r.  With the dense coarse solve the V-cycle has no
// host synchronisation, so from the second call with the same buffers on it
// is one graph launch (~100 kernels per cycle otherwise, most of them tiny on
// the coarse levels, where the launch rate bounded the solve).
static void mg_precondition_any(emfgpu_mg* m, const double* r, double* z, cudaStream_t s) {
  auto run = [&](cudaStream_t st) {
    if (m->cfg.precision == 64)
      mg_precondition<double>(m, r, z, st);
    else
      mg_precondition<float>(m, r, z, st);
  };
  if (!m->dense || !mg_graphs_enabled()) {
    run(s);
    return;
  }
  if (!m->vc_stream) {
    CK(cudaStreamCreateWithFlags(&m->vc_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&m->vc_ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m->vc_ev[1], cudaEventDisableTiming));
  }
  const bool same = m->vc_r == r && m->vc_z == z;
  if (same && !m->vc_exec) {
    CK(cudaStreamBeginCapture(m->vc_stream, cudaStreamCaptureModeThreadLocal));
    run(m->vc_stream);
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(m->vc_stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&m->vc_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      m->vc_exec = nullptr;
      throw ApiError(EMFGPU_ERR_CUDA, std::string("V-cycle graph instantiate: ") + cudaGetErrorString(e));
    }
  }
  if (same && m->vc_exec) {
    CK(cudaEventRecord(m->vc_ev[0], s));
    CK(cudaStreamWaitEvent(m->vc_stream, m->vc_ev[0], 0));
    CK(cudaGraphLaunch(m->vc_exec, m->vc_stream));
    CK(cudaEventRecord(m->vc_ev[1], m->vc_stream));
    CK(cudaStreamWaitEvent(s, m->vc_ev[1], 0));
    return;
  }
  mg_drop_graph(m);
  m->vc_r = r;
  m->vc_z = z;
  run(s);
}

emfgpu_status emfgpu_mg_precondition(emfgpu_mg* m, const double* d_r, double* d_z, void* stream) {
  if (!m || !d_r || !d_z) return EMFGPU_ERR_INVALID;
  return guarded(&m->last_error, [&] {
    if (!m->ops[0]->linearized) throw ApiError(EMFGPU_ERR_STALE, "mg: update_linearization has not run");
    UseGuard g(m->use_mu, m->ev_use, static_cast<cudaStream_t>(stream), m->fine->device);
    mg_precondition_any(m, d_r, d_z, static_cast<cudaStream_t>(stream));
  });
}

// Preconditioned CG in double on device vectors (x starts at 0).  Stops when
// ||r|| <= rtol ||b||.  history (host, maxit+1, optional) gets ||r_k||/||b||.
static bool pcg_graph_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("EMFGPU_PCG_GRAPH");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

// Run body(stream, h, 1) as the body of a conditional WHILE graph node, on s
// (captured with the node phase's programmatic launches disabled: a
// conditional body only takes kernel, memset, memcpy, child-graph and
// conditional nodes).  Returns false, having enqueued nothing, when the graph
// cannot be built; errors of the launch itself throw.
template <typename F>
static bool pcg_run_graph(cudaStream_t s, F&& body) {
  cudaStream_t cs = nullptr;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
  cudaGraphConditionalHandle h{};
  cudaGraphNode_t node{};
  cudaGraphNodeParams cp = {};
  if (ok) ok = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  if (ok) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
  }
  if (ok) {
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    ok = cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
         cudaSuccess;
    if (ok) {
      tl_no_pdl = true;
      bool thrown = false;
      try {
        body(cs, h, 1);
      } catch (...) {
        thrown = true;
      }
      tl_no_pdl = false;
      cudaGraph_t out = nullptr;
      ok = cudaStreamEndCapture(cs, &out) == cudaSuccess && !thrown;
    }
  }
  const auto t_cap = std::chrono::steady_clock::now();
  if (ok) ok = cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
  const auto t_inst = std::chrono::steady_clock::now();
  if (!ok) {
    const cudaError_t err = cudaGetLastError();
    if (std::getenv("EMFGPU_DEBUG"))
      std::fprintf(stderr, "emfgpu: PCG graph not built (%s), host loop\n", cudaGetErrorString(err));
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    return false;
  }
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  if (std::getenv("EMFGPU_DEBUG")) {
    const auto t_run = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "emfgpu: PCG graph instantiate %.2f ms, run %.2f ms\n", ms(t_cap, t_inst), ms(t_inst, t_run));
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return true;
}

emfgpu_status emfgpu_pcg_solve(emfgpu_op* op, emfgpu_mg* mg, const double* d_b, double* d_x, double rtol, int maxit,
                               int* iterations, double* history, void* stream) {
  if (!op || !d_b || !d_x) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (op->precision != 64) throw ApiError(EMFGPU_ERR_CONFIG, "pcg: the outer operator must be fp64");
    require_linearized(op, "pcg");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    OP_USE(op, s);
    std::unique_ptr<UseGuard> mg_use;
    if (mg) mg_use = std::make_unique<UseGuard>(mg->use_mu, mg->ev_use, s, op->L->device);
    const int64_t n = op->L->ndofs;
    // Device-resident PCG: the scalars stay on the device (sc = {rz, pAp, rr,
    // rz_new, ||b||}, ic = {iterations, done}) and, from the second iteration
    // on, the whole loop is one CUDA graph with a conditional WHILE node whose
    // condition the convergence-check kernel sets -- no host round trip per
    // iteration.  Same arithmetic and order as the host loop it replaced.
    // work space cached on the operator (large cudaMalloc / cudaFree pairs
    // per solve cost 0-200 ms of host time, measured)
    // dots over whole node planes (launch_dot_planes): bitwise the z-slab PCG's
    const int64_t plane = 3 * (int64_t)op->L->mx * op->L->my;
    const int nplanes = op->L->mz;
    const size_t ndot = (size_t)std::max(dot_partial_count(), nplanes * dot_plane_split());
    const size_t need = sizeof(double) * (4 * (size_t)n + ndot + 1 + 8 + (size_t)maxit + 1) + 16;
    if (op->pcg_bytes < need) {
      cudaFree(op->pcg_buf);
      op->pcg_buf = nullptr;
      op->pcg_bytes = 0;
      CK(cudaMalloc(&op->pcg_buf, need));
      op->pcg_bytes = need;
    }
    double* const base = static_cast<double*>(op->pcg_buf);
    double* const r = base;
    double* const z = r + n;
    double* const p = z + n;
    double* const ap = p + n;
    double* const dbuf = ap + n;
    double* const sc = dbuf + ndot + 1;
    double* const dhist = sc + 8;
    int* const ic = reinterpret_cast<int*>(dhist + maxit + 1);
    auto dot_to = [&](const double* a, const double* b, double* out, cudaStream_t st) {
      launch_dot_planes<double>(a, b, plane, nplanes, dbuf, out, st);
    };
    auto prec = [&](const double* rr, double* zz, cudaStream_t st) {
      if (mg) {
        if (mg->cfg.precision == 64)
          mg_precondition<double>(mg, rr, zz, st);
        else
          mg_precondition<float>(mg, rr, zz, st);
      } else {
        CK(cudaMemcpyAsync(zz, rr, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      }
    };
    // apply, dots, x/r update, check: the tail of every iteration
    auto tail = [&](cudaStream_t st, cudaGraphConditionalHandle h, int use_h) {
      op_apply_T<double>(op, p, ap, st);
      dot_to(p, ap, sc + 1, st);
      launch_pcg_xr(d_x, r, p, ap, sc, n, st);
      dot_to(r, r, sc + 2, st);
      launch_pcg_check(sc, ic, dhist, rtol, maxit, h, use_h, st);
    };
    CK(cudaMemsetAsync(d_x, 0, sizeof(double) * n, s));
    CK(cudaMemsetAsync(ic, 0, sizeof(int) * 3, s));  // iterations, stop, breakdown
    CK(cudaMemcpyAsync(r, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    dot_to(d_b, d_b, sc + 4, s);
    launch_pcg_sqrt(sc + 4, s);
    double bnorm = 0;
    CK(cudaMemcpyAsync(&bnorm, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int it = 0;
    bool breakdown = false;
    double last_rel = 0.0;
    if (history) history[0] = 1.0;
    if (bnorm != 0 && maxit > 0) {
      // first iteration eagerly (p = z, rz = (r, z))
      prec(r, z, s);
      CK(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      dot_to(r, z, sc + 0, s);
      tail(s, cudaGraphConditionalHandle{}, 0);
      int hic[2] = {0, 0};
      CK(cudaMemcpyAsync(hic, ic, sizeof(hic), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      // later iterations: z = M r; rz_new = (r, z); p = z + beta p; rz = rz_new; tail
      auto body = [&](cudaStream_t st, cudaGraphConditionalHandle h, int use_h) {
        prec(r, z, st);
        dot_to(r, z, sc + 3, st);
        launch_pcg_p(p, z, sc, n, st);
        launch_pcg_shift(sc, st);
        tail(st, h, use_h);
      };
      if (!hic[1]) {
        bool graphed = false;
        // the V-cycle is capturable only without host syncs (dense coarse
        // solve); the coarse-CG hierarchy keeps the host loop
        if (pcg_graph_enabled() && (!mg || mg->dense)) graphed = pcg_run_graph(s, body);
        if (!graphed) {
          for (;;) {  // host loop (no graph): one sync per iteration
            body(s, cudaGraphConditionalHandle{}, 0);
            CK(cudaMemcpyAsync(hic, ic, sizeof(hic), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (hic[1]) break;
          }
        }
      }
      int hic3[3] = {0, 0, 0};
      CK(cudaMemcpyAsync(hic3, ic, sizeof(hic3), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      it = hic3[0];
      breakdown = hic3[2] != 0;
      if (it > 0) CK(cudaMemcpy(&last_rel, dhist + it, sizeof(double), cudaMemcpyDeviceToHost));
      if (history && it > 0) CK(cudaMemcpy(history + 1, dhist + 1, sizeof(double) * it, cudaMemcpyDeviceToHost));
    }
    if (iterations) *iterations = it;
    CK(cudaStreamSynchronize(s));
    // a solve that stopped without reaching rtol is an error (the reference's
    // CG / FGMRES throw CgNoConvergence / LinearSolveFailure, solver.hpp:202, 423)
    if (breakdown)
      throw ApiError(EMFGPU_ERR_NUMERICAL, "pcg: breakdown (p^T A p <= 0) at iteration " + std::to_string(it));
    if (it > 0 && !(last_rel <= rtol))
      throw ApiError(EMFGPU_ERR_NUMERICAL, "pcg: no convergence in " + std::to_string(it) +
                                               " iterations (relative residual " + std::to_string(last_rel) + ")");
  });
}

// ---- per-quadrature-point fibre frames (BASELINE cfg3) -----------------------
emfgpu_status emfgpu_op_set_fibre_frame(emfgpu_op* op, int kind) {
  if (!op) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (op->model != EMFGPU_FIBER) throw ApiError(EMFGPU_ERR_CONFIG, "fibre frame: fibre model only");
    if (kind < 0 || kind > 2) throw ApiError(EMFGPU_ERR_CONFIG, "fibre frame: kind must be 0, 1 or 2");
    CK(cudaSetDevice(op->L->device));
    const emfgpu_level* L = op->L;
    op->linearized = false;
    if (op->gexec) {  // captured kernels hold the old frame-field pointers
      cudaGraphExecDestroy(op->gexec);
      op->gexec = nullptr;
      op->g_x = op->g_y = nullptr;
    }
    if (op->d_hq && op->d_hq != op->d_hqd) cudaFree(op->d_hq);
    cudaFree(op->d_hqd);
    op->d_hq = nullptr;
    op->d_hqd = op->d_m1qd = nullptr;
    op->frame_kind = kind;
    if (kind == 0) return;
    const int64_t nqp = L->nel * L->nq3;
    CK(cudaMalloc(&op->d_hqd, sizeof(double) * 18 * nqp));
    op->d_m1qd = op->d_hqd + 12 * nqp;
    double h[2][6], m1[2][3];
    structure_tensors(op->params, h, m1);
    // h11, h22, h33 of the dispersion (material.cpp:52-61)
    const double h33 = 1.0 / (4.0 * op->params.b) - std::exp(-2.0 * op->params.b) /
                                                       (std::sqrt(2.0 * M_PI * op->params.b) *
                                                        std::erf(std::sqrt(2.0 * op->params.b)));
    const double ratio = std::cyl_bessel_i(1.0, op->params.a) / std::cyl_bessel_i(0.0, op->params.a);
    const double h11 = 0.5 * (1.0 - h33) * (1.0 + ratio), h22 = 0.5 * (1.0 - h33) * (1.0 - ratio);
    double frame[9];
    for (int d = 0; d < 3; ++d) {
      frame[d] = op->params.e1[d];
      frame[3 + d] = op->params.e2[d];
      frame[6 + d] = op->params.e3[d];
    }
    launch_fibre_frame(L->d_coords, op->d_hqd, op->d_m1qd, L->nx, L->ny, L->nz, L->p, L->periodic_y, L->B.data(),
                       h11, h22, h33, op->params.phi, kind, frame, op->stream);
    CK(cudaGetLastError());
    if (op->precision == 64) {
      op->d_hq = op->d_hqd;
    } else {
      CK(cudaMalloc(&op->d_hq, sizeof(float) * 18 * nqp));
      launch_cast_d2f(op->d_hqd, static_cast<float*>(op->d_hq), 18 * nqp, op->stream);
    }
    CK(cudaStreamSynchronize(op->stream));
  });
}

emfgpu_status emfgpu_op_fibre_field(const emfgpu_op* op, double* h_out, double* m1_out) {
  if (!op) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    if (!op->d_hqd) throw ApiError(EMFGPU_ERR_CONFIG, "fibre field: no per-qp frame set");
    const int64_t nqp = op->L->nel * op->L->nq3;
    if (h_out) CK(cudaMemcpy(h_out, op->d_hqd, sizeof(double) * 12 * nqp, cudaMemcpyDeviceToHost));
    if (m1_out) CK(cudaMemcpy(m1_out, op->d_m1qd, sizeof(double) * 6 * nqp, cudaMemcpyDeviceToHost));
  });
}

// ---- residual and loads (operator.hpp:532-595, 623-641, 880-1008) ----------
static void residual_impl(emfgpu_op* op, const void* u, void* r, cudaStream_t s) {
  const emfgpu_level* L = op->L;
  if (op->precision == 64) {
    KArgs<double> a = kargs<double>(op);
    a.x = static_cast<const double*>(u);
    dispatch_residual<double>(op, a, s);
    launch_node_gather<double>(static_cast<const double*>(op->d_loc), nullptr, nullptr, static_cast<const double*>(u),
                               static_cast<double*>(r), L->nx, L->ny, L->nz, L->p, L->faces, 0, 0, L->mz - 1,
                               L->periodic_y, s);
    launch_sub_load_mask<double>(static_cast<double*>(r), static_cast<const double*>(op->d_load), op->load_scale,
                                 L->nnodes, L->mx, L->my, L->mz, L->faces, s);
  } else {
    KArgs<float> a = kargs<float>(op);
    a.x = static_cast<const float*>(u);
    dispatch_residual<float>(op, a, s);
    launch_node_gather<float>(static_cast<const float*>(op->d_loc), nullptr, nullptr, static_cast<const float*>(u),
                              static_cast<float*>(r), L->nx, L->ny, L->nz, L->p, L->faces, 0, 0, L->mz - 1,
                              L->periodic_y, s);
    launch_sub_load_mask<float>(static_cast<float*>(r), static_cast<const float*>(op->d_load), op->load_scale,
                                L->nnodes, L->mx, L->my, L->mz, L->faces, s);
  }
  CK(cudaGetLastError());
}

emfgpu_status emfgpu_op_residual(emfgpu_op* op, const void* d_u, void* d_r, void* stream) {
  if (!op || !d_u || !d_r) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, S(stream, op->stream));
    residual_impl(op, d_u, d_r, S(stream, op->stream));
  });
}

emfgpu_status emfgpu_op_residual_host(emfgpu_op* op, const void* u, void* r) {
  if (!op || !u || !r) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, op->stream);
    const size_t bytes = nsize(op) * op->L->ndofs;
    if (!op->d_x) CK(cudaMalloc(&op->d_x, bytes));
    if (!op->d_y) CK(cudaMalloc(&op->d_y, bytes));
    CK(cudaMemcpyAsync(op->d_x, u, bytes, cudaMemcpyHostToDevice, op->stream));
    residual_impl(op, op->d_x, op->d_y, op->stream);
    CK(cudaMemcpyAsync(r, op->d_y, bytes, cudaMemcpyDeviceToHost, op->stream));
    check_err(op, op->stream, nullptr, nullptr, "evaluate_residual");
  });
}

emfgpu_status emfgpu_op_set_load_scale(emfgpu_op* op, double scale) {
  if (!op) return EMFGPU_ERR_INVALID;
  op->load_scale = scale;
  return EMFGPU_OK;
}

// Uniform pressure on one face of the (deformed) box: traction -p N on the
// reference geometry, (p+1)^2 Gauss points per face element
// (build_load_vector, operator.hpp:933-1001).  Setup-time, on the host.
namespace {
// Host sum factorization of one element field: out[(c*nq + b)*nq + a] =
// sum M0[a][i] M1[b][j] M2[c][k] in[(k*nn + j)*nn + i] (M row-major nq x nn).
void sf3(const double* M0, const double* M1, const double* M2, const double* in, double* out, int nq, int nn,
         std::vector<double>& t1, std::vector<double>& t2) {
  t1.assign((size_t)nn * nn * nq, 0.0);
  for (int k = 0; k < nn; ++k)
    for (int j = 0; j < nn; ++j)
      for (int a = 0; a < nq; ++a) {
        double v = 0.0;
        for (int i = 0; i < nn; ++i) v += M0[a * nn + i] * in[(k * nn + j) * nn + i];
        t1[(k * nn + j) * nq + a] = v;
      }
  t2.assign((size_t)nn * nq * nq, 0.0);
  for (int k = 0; k < nn; ++k)
    for (int b = 0; b < nq; ++b)
      for (int a = 0; a < nq; ++a) {
        double v = 0.0;
        for (int j = 0; j < nn; ++j) v += M1[b * nn + j] * t1[(k * nn + j) * nq + a];
        t2[(k * nq + b) * nq + a] = v;
      }
  for (int c = 0; c < nq; ++c)
    for (int b = 0; b < nq; ++b)
      for (int a = 0; a < nq; ++a) {
        double v = 0.0;
        for (int k = 0; k < nn; ++k) v += M2[c * nn + k] * t2[(k * nq + b) * nq + a];
        out[(c * nq + b) * nq + a] = v;
      }
}

// build_load_vector (operator.hpp:880-1008) on the host, restated: body force
// B(X) at the Gauss points (values by B sweeps, det J0 by D/B sweeps of the
// node coordinates, tested back by transposed B sweeps), then face tractions
// with (p+1)^2 Gauss points per face element on the material configuration.
void build_loads(emfgpu_op* op, const emfgpu_loads& ld) {
  const emfgpu_level* L = op->L;
  if (ld.pressure != 0.0 && (ld.pressure_face < 0 || ld.pressure_face > 5))
    throw ApiError(EMFGPU_ERR_CONFIG, "loads: pressure_face must be 0..5");
  if (L->periodic_y && ((ld.pressure != 0.0 && (ld.pressure_face == 2 || ld.pressure_face == 3)) ||
                        (ld.traction && (ld.traction_faces & 12))))
    throw ApiError(EMFGPU_ERR_CONFIG, "loads: periodic face");
  std::vector<double> coords(L->ndofs), load(L->ndofs, 0.0);
  CK(cudaMemcpy(coords.data(), L->d_coords, sizeof(double) * L->ndofs, cudaMemcpyDeviceToHost));
  const int p = L->p, nn = p + 1, nq = p + 1, nn3 = nn * nn * nn, nq3 = nq * nq * nq;
  const int ne[3] = {L->nx, L->ny, L->nz};
  const int m[3] = {L->mx, L->my, L->mz};
  const std::vector<double>& B = L->B;
  const std::vector<double>& D = L->D;
  std::vector<double> Bt((size_t)nn * nq);
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < nn; ++a) Bt[a * nq + q] = B[q * nn + a];
  auto gnode = [&](const int* ijk, const int* loc) -> int64_t {
    int g[3];
    for (int d = 0; d < 3; ++d) g[d] = ijk[d] * p + loc[d];
    if (L->periodic_y && g[1] >= m[1]) g[1] -= m[1];
    return ((int64_t)g[2] * m[1] + g[1]) * m[0] + g[0];
  };
  if (ld.body_force) {
    std::vector<int64_t> nodes(nn3);
    std::vector<double> comp(nn3), xq(3 * (size_t)nq3), jq(9 * (size_t)nq3), vals(nq3), contrib(nn3), t1, t2;
    for (int k = 0; k < ne[2]; ++k)
      for (int j = 0; j < ne[1]; ++j)
        for (int i = 0; i < ne[0]; ++i) {
          const int ijk[3] = {i, j, k};
          for (int c3 = 0; c3 < nn; ++c3)
            for (int b3 = 0; b3 < nn; ++b3)
              for (int a3 = 0; a3 < nn; ++a3) {
                const int loc[3] = {a3, b3, c3};
                nodes[(c3 * nn + b3) * nn + a3] = gnode(ijk, loc);
              }
          for (int c = 0; c < 3; ++c) {
            for (int q = 0; q < nn3; ++q) comp[q] = coords[3 * nodes[q] + c];
            sf3(B.data(), B.data(), B.data(), comp.data(), &xq[(size_t)c * nq3], nq, nn, t1, t2);
            // J0 row c: dX_c / dxi_t
            sf3(D.data(), B.data(), B.data(), comp.data(), &jq[(size_t)(3 * c + 0) * nq3], nq, nn, t1, t2);
            sf3(B.data(), D.data(), B.data(), comp.data(), &jq[(size_t)(3 * c + 1) * nq3], nq, nn, t1, t2);
            sf3(B.data(), B.data(), D.data(), comp.data(), &jq[(size_t)(3 * c + 2) * nq3], nq, nn, t1, t2);
          }
          std::vector<double> fq(3 * (size_t)nq3);
          for (int q = 0; q < nq3; ++q) {
            double J[9], X[3] = {xq[q], xq[nq3 + q], xq[2 * (size_t)nq3 + q]}, f[3] = {0, 0, 0};
            for (int t = 0; t < 9; ++t) J[t] = jq[(size_t)t * nq3 + q];
            const double det = (J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6])) +
                               J[2] * (J[3] * J[7] - J[4] * J[6]);
            const int qa = q % nq, qb = (q / nq) % nq, qc = q / (nq * nq);
            const double w = L->qwts[qa] * L->qwts[qb] * L->qwts[qc];
            ld.body_force(X, f, ld.body_force_user);
            for (int c = 0; c < 3; ++c) fq[(size_t)c * nq3 + q] = f[c] * det * w;
          }
          for (int c = 0; c < 3; ++c) {
            sf3(Bt.data(), Bt.data(), Bt.data(), &fq[(size_t)c * nq3], contrib.data(), nn, nq, t1, t2);
            for (int q = 0; q < nn3; ++q) load[3 * nodes[q] + c] += contrib[q];
          }
        }
  }
  auto add_face = [&](int face, auto&& traction) {
    const int axis = face / 2, t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
    const bool upper = face % 2 == 1;
    for (int ej = 0; ej < ne[t2]; ++ej)
      for (int ei = 0; ei < ne[t1]; ++ei) {
        int idx[3];
        idx[axis] = upper ? ne[axis] - 1 : 0;
        idx[t1] = ei;
        idx[t2] = ej;
        for (int q2 = 0; q2 < nq; ++q2)
          for (int q1 = 0; q1 < nq; ++q1) {
            double x[3] = {0, 0, 0}, g1[3] = {0, 0, 0}, g2[3] = {0, 0, 0};
            for (int a2 = 0; a2 < nn; ++a2)
              for (int a1 = 0; a1 < nn; ++a1) {
                const double v1 = B[q1 * nn + a1], d1 = D[q1 * nn + a1];
                const double v2 = B[q2 * nn + a2], d2 = D[q2 * nn + a2];
                int loc[3];
                loc[axis] = upper ? p : 0;
                loc[t1] = a1;
                loc[t2] = a2;
                const int64_t g = gnode(idx, loc);
                for (int c = 0; c < 3; ++c) {
                  const double xc = coords[3 * g + c];
                  x[c] += v1 * v2 * xc;
                  g1[c] += d1 * v2 * xc;
                  g2[c] += v1 * d2 * xc;
                }
              }
            const double nrm[3] = {g1[1] * g2[2] - g1[2] * g2[1], g1[2] * g2[0] - g1[0] * g2[2],
                                   g1[0] * g2[1] - g1[1] * g2[0]};
            const double sgn = upper ? 1.0 : -1.0;
            const double area = std::sqrt((nrm[0] * nrm[0] + nrm[1] * nrm[1]) + nrm[2] * nrm[2]);
            const double unit[3] = {sgn * nrm[0] / area, sgn * nrm[1] / area, sgn * nrm[2] / area};
            double h[3] = {0, 0, 0};
            traction(x, unit, h);
            const double w = L->qwts[q1] * L->qwts[q2] * area;
            for (int a2 = 0; a2 < nn; ++a2)
              for (int a1 = 0; a1 < nn; ++a1) {
                const double phi = B[q1 * nn + a1] * B[q2 * nn + a2];
                int loc[3];
                loc[axis] = upper ? p : 0;
                loc[t1] = a1;
                loc[t2] = a2;
                const int64_t g = gnode(idx, loc);
                for (int c = 0; c < 3; ++c) load[3 * g + c] += phi * w * h[c];
              }
          }
      }
  };
  if (ld.pressure != 0.0) {
    const double pm = ld.pressure;
    add_face(ld.pressure_face, [pm](const double*, const double* nrm, double* h) {
      for (int c = 0; c < 3; ++c) h[c] = -pm * nrm[c];
    });
  }
  if (ld.traction)
    for (int face = 0; face < 6; ++face)
      if (ld.traction_faces & (1 << face))
        add_face(face, [&](const double* x, const double* nrm, double* h) { ld.traction(x, nrm, h, ld.traction_user); });
  const size_t ns = nsize(op);
  if (!op->d_load) CK(cudaMalloc(&op->d_load, ns * L->ndofs));
  if (op->precision == 64) {
    CK(cudaMemcpy(op->d_load, load.data(), sizeof(double) * L->ndofs, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> lf(load.begin(), load.end());
    CK(cudaMemcpy(op->d_load, lf.data(), sizeof(float) * L->ndofs, cudaMemcpyHostToDevice));
  }
}
}  // namespace

emfgpu_status emfgpu_op_set_pressure(emfgpu_op* op, double pressure, int face) {
  if (!op) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (face < 0 || face > 5) throw ApiError(EMFGPU_ERR_CONFIG, "pressure: face must be 0..5");
    OP_USE(op, op->stream);
    emfgpu_loads ld{};
    ld.pressure = pressure;
    ld.pressure_face = face;
    build_loads(op, ld);
  });
}

emfgpu_status emfgpu_op_set_loads(emfgpu_op* op, const emfgpu_loads* loads) {
  if (!op || !loads) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    OP_USE(op, op->stream);
    build_loads(op, *loads);
  });
}

// ============================================================================
// FGMRES(m) and Newton on the device (solver.hpp:120-203, 603-656)
// ============================================================================
namespace {

struct DevVec {
  double* p = nullptr;
  ~DevVec() { cudaFree(p); }
};

__global__ void lincomb_kernel(double* y, const double* x, double a, int64_t n) {  // y += a x
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
__global__ void scale_copy_kernel(double* y, const double* x, double a, int64_t n) {  // y = x / a
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] / a;
}
__global__ void neg_kernel(double* y, const double* x, int64_t n) {  // y = -x
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = -x[i];
}
inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

struct Krylov {
  emfgpu_op* op;
  emfgpu_mg* mg;
  cudaStream_t s;
  int64_t n;
  double *dbuf = nullptr, *hdot = nullptr;
  Krylov(emfgpu_op* o, emfgpu_mg* m, cudaStream_t st) : op(o), mg(m), s(st), n(o->L->ndofs) {
    CK(cudaMalloc(&dbuf, sizeof(double) * (dot_partial_count() + 1)));
    CK(cudaMallocHost(&hdot, sizeof(double)));
  }
  ~Krylov() {
    cudaFree(dbuf);
    if (hdot) cudaFreeHost(hdot);
  }
  double dot(const double* a, const double* b) {
    launch_dot<double>(a, b, n, dbuf + 1, dbuf, s);
    return mg_dot_sync(dbuf, hdot, s);
  }
  void apply(const double* x, double* y) { op_apply_T<double>(op, x, y, s); }
  void prec(const double* r, double* z) {
    if (mg) {
      mg_precondition_any(mg, r, z, s);
    } else {
      CK(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }
  }
};

// Right-preconditioned flexible GMRES with restart, modified Gram-Schmidt,
// Givens rotations; terminates when ||b - A x|| <= max(abs_tol, rel_tol ||b||)
// (fgmres_solve, solver.hpp:120-203).  Returns false without convergence.
bool fgmres(Krylov& K, const double* b, double* x, double abs_tol, double rel_tol, int m, int max_restarts,
            int* iterations, double* final_res) {
  const int64_t n = K.n;
  const double bnorm = std::sqrt(K.dot(b, b));
  const double tol = std::max(abs_tol, rel_tol * bnorm);
  // Krylov basis, preconditioned directions, w and r: 2m + 3 vectors from
  // one work space cached on the operator (a per-solve cudaMalloc / cudaFree
  // of 2m + 3 vectors cost far more than the allocation of the PCG's 4)
  struct Vec {
    double* p;
  };
  const size_t need = sizeof(double) * (size_t)(2 * m + 3) * (size_t)n;
  if (K.op->fgmres_bytes < need) {
    cudaFree(K.op->fgmres_buf);
    K.op->fgmres_buf = nullptr;
    K.op->fgmres_bytes = 0;
    CK(cudaMalloc(&K.op->fgmres_buf, need));
    K.op->fgmres_bytes = need;
  }
  double* const wbase = static_cast<double*>(K.op->fgmres_buf);
  std::vector<Vec> V(m + 1), Z(m);
  for (int i = 0; i <= m; ++i) V[i].p = wbase + (size_t)i * n;
  for (int i = 0; i < m; ++i) Z[i].p = wbase + (size_t)(m + 1 + i) * n;
  Vec w{wbase + (size_t)(2 * m + 1) * n}, r{wbase + (size_t)(2 * m + 2) * n};
  std::vector<double> H((m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0);
  int its = 0;
  for (int cycle = 0; cycle <= max_restarts; ++cycle) {
    K.apply(x, r.p);
    launch_bminus<double>(b, r.p, n, K.s);  // r = b - A x
    const double beta = std::sqrt(K.dot(r.p, r.p));
    *final_res = beta;
    if (beta <= tol) {
      *iterations = its;
      return true;
    }
    if (cycle == max_restarts) break;
    scale_copy_kernel<<<nb(n), 256, 0, K.s>>>(V[0].p, r.p, beta, n);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m; ++j) {
      K.prec(V[j].p, Z[j].p);
      K.apply(Z[j].p, w.p);
      for (int i = 0; i <= j; ++i) {
        const double h = K.dot(w.p, V[i].p);
        H[i * m + j] = h;
        lincomb_kernel<<<nb(n), 256, 0, K.s>>>(w.p, V[i].p, -h, n);
      }
      const double h1 = std::sqrt(K.dot(w.p, w.p));
      H[(j + 1) * m + j] = h1;
      ++its;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
        H[(i + 1) * m + j] = -sn[i] * H[i * m + j] + cs[i] * H[(i + 1) * m + j];
        H[i * m + j] = t;
      }
      const double denom = std::hypot(H[j * m + j], h1);
      if (denom < 1e-300) break;
      cs[j] = H[j * m + j] / denom;
      sn[j] = h1 / denom;
      H[j * m + j] = denom;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      if (h1 > 1e-300) scale_copy_kernel<<<nb(n), 256, 0, K.s>>>(V[j + 1].p, w.p, h1, n);
      if (std::abs(g[j + 1]) <= tol || h1 <= 1e-300) {
        ++j;
        break;
      }
    }
    const int used = j;
    std::vector<double> y(used, 0.0);
    for (int i = used - 1; i >= 0; --i) {
      double sacc = g[i];
      for (int k = i + 1; k < used; ++k) sacc -= H[i * m + k] * y[k];
      y[i] = sacc / H[i * m + i];
    }
    for (int i = 0; i < used; ++i) lincomb_kernel<<<nb(n), 256, 0, K.s>>>(x, Z[i].p, y[i], n);
    CK(cudaGetLastError());
  }
  *iterations = its;
  return false;
}

}  // namespace

emfgpu_status emfgpu_fgmres_solve(emfgpu_op* op, emfgpu_mg* mg, const double* d_b, double* d_x, double abs_tol,
                                  double rel_tol, int restart, int max_restarts, int* iterations,
                                  double* final_residual, void* stream) {
  if (!op || !d_b || !d_x) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (op->precision != 64) throw ApiError(EMFGPU_ERR_CONFIG, "fgmres: the outer operator must be fp64");
    require_linearized(op, "fgmres");
    OP_USE(op, static_cast<cudaStream_t>(stream));
    std::unique_ptr<UseGuard> mg_use;
    if (mg) mg_use = std::make_unique<UseGuard>(mg->use_mu, mg->ev_use, static_cast<cudaStream_t>(stream), op->L->device);
    Krylov K(op, mg, static_cast<cudaStream_t>(stream));
    int its = 0;
    double res = 0;
    const bool ok = fgmres(K, d_b, d_x, abs_tol, rel_tol, restart, max_restarts, &its, &res);
    if (iterations) *iterations = its;
    if (final_residual) *final_residual = res;
    CK(cudaStreamSynchronize(K.s));
    if (!ok) throw ApiError(EMFGPU_ERR_NUMERICAL, "fgmres: no convergence within restart budget");
  });
}

void emfgpu_newton_default_config(emfgpu_newton_config* c) {
  if (!c) return;
  c->eps_abs = 1e-8;
  c->eps_rel = 1e-3;
  c->max_iter = 25;
  c->lin_abs_tol = 1e-12;
  c->lin_rel_tol = 1e-3;
  c->restart = 30;
  c->max_restarts = 40;
}

// newton_solve (solver.hpp:603-656): relinearise op and mg at u, solve
// K du = -r with MG-preconditioned FGMRES, u += du, until ||r|| <= eps_abs or
// <= eps_rel ||r0||.  d_u: device fp64, updated in place.
emfgpu_status emfgpu_newton_solve(emfgpu_op* op, emfgpu_mg* mg, double* d_u, const emfgpu_newton_config* cfg,
                                  int* newton_iterations, int* linear_iterations, double* final_residual,
                                  void* stream) {
  if (!op || !d_u) return EMFGPU_ERR_INVALID;
  return guarded(&op->last_error, [&] {
    if (op->precision != 64) throw ApiError(EMFGPU_ERR_CONFIG, "newton: the operator must be fp64");
    OP_USE(op, static_cast<cudaStream_t>(stream));
    std::unique_ptr<UseGuard> mg_use;
    if (mg) mg_use = std::make_unique<UseGuard>(mg->use_mu, mg->ev_use, static_cast<cudaStream_t>(stream), op->L->device);
    emfgpu_newton_config c;
    if (cfg)
      c = *cfg;
    else
      emfgpu_newton_default_config(&c);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Krylov K(op, mg, s);
    const int64_t n = K.n;
    DevVec r, rhs, du;
    CK(cudaMalloc(&r.p, sizeof(double) * n));
    CK(cudaMalloc(&rhs.p, sizeof(double) * n));
    CK(cudaMalloc(&du.p, sizeof(double) * n));
    residual_impl(op, d_u, r.p, s);
    double rnorm = std::sqrt(K.dot(r.p, r.p));
    const double r0 = rnorm;
    int k = 0, lin = 0;
    while (rnorm > c.eps_abs && rnorm > c.eps_rel * r0) {
      if (k >= c.max_iter) throw ApiError(EMFGPU_ERR_NUMERICAL, "newton: iteration budget exhausted");
      CK(cudaMemcpyAsync(op->d_ukd, d_u, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      op->checksum_valid = false;
      linearize_impl(op, nullptr, nullptr, s);
      if (mg) {
        if (mg->cfg.precision == 64)
          mg_linearize<double>(mg, d_u, s);
        else
          mg_linearize<float>(mg, d_u, s);
      }
      neg_kernel<<<nb(n), 256, 0, s>>>(rhs.p, r.p, n);
      CK(cudaMemsetAsync(du.p, 0, sizeof(double) * n, s));
      int its = 0;
      double res = 0;
      if (!fgmres(K, rhs.p, du.p, c.lin_abs_tol, c.lin_rel_tol, c.restart, c.max_restarts, &its, &res))
        throw ApiError(EMFGPU_ERR_NUMERICAL, "newton: linear solve did not converge");
      lin += its;
      lincomb_kernel<<<nb(n), 256, 0, s>>>(d_u, du.p, 1.0, n);
      residual_impl(op, d_u, r.p, s);
      rnorm = std::sqrt(K.dot(r.p, r.p));
      ++k;
    }
    check_err(op, s, nullptr, nullptr, "newton");
    if (newton_iterations) *newton_iterations = k;
    if (linear_iterations) *linear_iterations = lin;
    if (final_residual) *final_residual = rnorm;
  });
}

// ---- stability lab -------------------------------------------------------------
emfgpu_status emfgpu_stability_sweep(const double* scales, int n_scales, int samples_per_scale, uint64_t seed,
                                     const emfgpu_material* params, double* max_rel_error, int64_t* count_invalid) {
  if (!scales || !params || !max_rel_error || !count_invalid) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    // run_sweep argument checks (stability.cpp:164-170)
    if (n_scales <= 0 || samples_per_scale < 0) throw ApiError(EMFGPU_ERR_CONFIG, "run_sweep: empty sweep axes");
    for (int i = 0; i < n_scales; ++i)
      if (!(scales[i] > 0) || (i > 0 && !(scales[i] > scales[i - 1])))
        throw ApiError(EMFGPU_ERR_CONFIG, "run_sweep: scales must be positive and increasing");
    double h[2][6] = {}, m1[2][3] = {};
    structure_tensors(*params, h, m1);
    try {
      run_stability_sweep(scales, n_scales, samples_per_scale, seed, *params, h, m1, max_rel_error, count_invalid);
    } catch (const std::runtime_error& e) {
      throw ApiError(EMFGPU_ERR_CUDA, e.what());
    }
  });
}

emfgpu_status emfgpu_newton_solve_host(emfgpu_op* op, emfgpu_mg* mg, double* u, const emfgpu_newton_config* cfg,
                                       int* newton_iterations, int* linear_iterations, double* final_residual) {
  if (!op || !u) return EMFGPU_ERR_INVALID;
  double* d_u = nullptr;
  emfgpu_status st = guarded(&op->last_error, [&] {
    CK(cudaSetDevice(op->L->device));
    CK(cudaMalloc(&d_u, sizeof(double) * op->L->ndofs));
    CK(cudaMemcpy(d_u, u, sizeof(double) * op->L->ndofs, cudaMemcpyHostToDevice));
  });
  if (st == EMFGPU_OK) {
    st = emfgpu_newton_solve(op, mg, d_u, cfg, newton_iterations, linear_iterations, final_residual, op->stream);
    if (st == EMFGPU_OK)
      st = guarded(&op->last_error, [&] {
        CK(cudaMemcpy(u, d_u, sizeof(double) * op->L->ndofs, cudaMemcpyDeviceToHost));
      });
  }
  cudaFree(d_u);
  return st;
}
