// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" driver around the UNMODIFIED reference implementation
// (/root/reference/proj, compiled from its own sources by oracle/Makefile into
// oracle/_ref/libemfref.so).  It is used (a) to pin the C restatement in
// oracle/emf_oracle.c, (b) to generate the golden fixtures under tests/golden,
// (c) as bench.py's `--impl reference` CPU arm.  Nothing here re-implements
// reference arithmetic: every number comes from the reference's own
// ElasticOperator / TransferOp / ChebyshevSmoother / estimate_eigenvalues.
//
// Reference interfaces driven:
//   FeLevel ctor / set_dirichlet       proj/include/elastmf/mesh.hpp:71-138
//   ElasticOperator<N>                 proj/include/elastmf/operator.hpp:49-204
//   TransferOp                         proj/include/elastmf/mesh.hpp:157-182
//   ChebyshevSmoother / estimate_eig.  proj/include/elastmf/solver.hpp:262-362
//   MgHierarchy                        proj/include/elastmf/solver.hpp:437-581

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "elastmf/operator.hpp"
#include "elastmf/solver.hpp"
#include "elastmf/stability.hpp"

using namespace emf;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  g_err.clear();
  try {
    fn();
    return 0;
  } catch (const NonPositiveJacobian& e) {
    g_err = std::string(e.what()) + " element=" + std::to_string(e.element) +
            " qpoint=" + std::to_string(e.qpoint);
    return 3;
  } catch (const StaleCache& e) {
    g_err = e.what();
    return 4;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct RefLevel {
  std::unique_ptr<FeLevel> fe;
};

struct RefOp {
  int precision = 64;
  std::unique_ptr<ElasticOperator<double>> d;
  std::unique_ptr<ElasticOperator<float>> f;
  int64_t n = 0;
};

// Recomputes J0 from overridden node coordinates exactly as mesh.cpp:162-186
// does (the reference's own gradient_at_qpoints on the GLL lattice).
void recompute_jacobians(FeLevel& fe) {
  const Basis1D& b = fe.basis();
  const int nn = b.nn(), nq = b.nq();
  const int nn3 = nn * nn * nn, nq3 = nq * nq * nq;
  const int n = fe.mesh().n();
  auto& jac = const_cast<std::vector<double>&>(fe.jacobians());
  const auto& coords = fe.node_coords();
  std::vector<double> local(nn3), work(2 * nq3 + 2 * nn3),
      g[3] = {std::vector<double>(nq3), std::vector<double>(nq3),
              std::vector<double>(nq3)};
  std::vector<std::int64_t> nodes(nn3);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const std::int64_t e = fe.element_index(i, j, k);
        fe.element_nodes(i, j, k, nodes.data());
        for (int comp = 0; comp < 3; ++comp) {
          for (int l = 0; l < nn3; ++l) local[l] = coords[3 * nodes[l] + comp];
          gradient_at_qpoints(b.B.data(), b.D.data(), nn, nq, local.data(),
                              work.data(), g[0].data(), g[1].data(),
                              g[2].data());
          for (int q = 0; q < nq3; ++q) {
            double* J = &jac[(e * nq3 + q) * 9];
            J[comp * 3 + 0] = g[0][q];
            J[comp * 3 + 1] = g[1][q];
            J[comp * 3 + 2] = g[2][q];
          }
        }
      }
}

MaterialParams params_from(const double* p) {
  // p = {mu, lambda, kappa_b, k1, k2, a, b, phi, e1[3], e2[3], e3[3]}
  MaterialParams m;
  m.mu = p[0];
  m.lambda = p[1];
  m.kappa_b = p[2];
  m.k1 = p[3];
  m.k2 = p[4];
  m.a = p[5];
  m.b = p[6];
  m.phi = p[7];
  for (int i = 0; i < 3; ++i) {
    m.e1[i] = p[8 + i];
    m.e2[i] = p[11 + i];
    m.e3[i] = p[14 + i];
  }
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_structure_tensors(const double* params, double* out) {
  // out = {h4[6], h6[6], m1_4[3], m1_6[3], h11, h22, h33}
  return guarded([&] {
    const StructureTensors st = build_structure_tensors(params_from(params));
    for (int k = 0; k < 6; ++k) {
      out[k] = st.h4.s[k];
      out[6 + k] = st.h6.s[k];
    }
    for (int k = 0; k < 3; ++k) {
      out[12 + k] = st.m1_4[k];
      out[15 + k] = st.m1_6[k];
    }
    out[18] = st.h11;
    out[19] = st.h22;
    out[20] = st.h33;
  });
}

// n0, level: build_cube(n0, level) (n = n0 << level). deform_amp: DeformMap.
// dirichlet_faces: bit f set = face f (-x,+x,-y,+y,-z,+z) clamped to zero.
// coords: optional node-coordinate override (3 per node) — J0 is then
// recomputed with the reference's own sweeps (SURVEY §8(c) gap 1).
void* ref_level_create(int n0, int level, int p, double deform_amp,
                       int dirichlet_faces, const double* coords) {
  RefLevel* L = new RefLevel;
  int st = guarded([&] {
    L->fe = std::make_unique<FeLevel>(build_cube(n0, level), p,
                                      DeformMap{deform_amp});
    if (coords) {
      auto& c = const_cast<std::vector<double>&>(L->fe->node_coords());
      std::memcpy(c.data(), coords, c.size() * sizeof(double));
      recompute_jacobians(*L->fe);
    }
    FeLevel::DirichletSpec spec;
    for (int f = 0; f < 6; ++f) spec.faces[f] = (dirichlet_faces >> f) & 1;
    L->fe->set_dirichlet(spec);
  });
  if (st != 0) {
    delete L;
    return nullptr;
  }
  return L;
}

void ref_level_destroy(void* l) { delete static_cast<RefLevel*>(l); }

int64_t ref_level_ndofs(void* l) {
  return static_cast<RefLevel*>(l)->fe->dof_count();
}

void ref_level_coords(void* l, double* out) {
  const auto& c = static_cast<RefLevel*>(l)->fe->node_coords();
  std::memcpy(out, c.data(), c.size() * sizeof(double));
}

void ref_level_jacobians(void* l, double* out) {
  const auto& c = static_cast<RefLevel*>(l)->fe->jacobians();
  std::memcpy(out, c.data(), c.size() * sizeof(double));
}

void ref_level_mask(void* l, uint8_t* out) {
  const auto& c = static_cast<RefLevel*>(l)->fe->dirichlet_mask();
  std::memcpy(out, c.data(), c.size());
}

void ref_level_basis(void* l, double* nodes, double* qpts, double* qwts,
                     double* B, double* D) {
  const Basis1D& b = static_cast<RefLevel*>(l)->fe->basis();
  const int n = b.nn();
  std::memcpy(nodes, b.nodes.data(), n * sizeof(double));
  std::memcpy(qpts, b.qpts.data(), n * sizeof(double));
  std::memcpy(qwts, b.qwts.data(), n * sizeof(double));
  std::memcpy(B, b.B.data(), n * n * sizeof(double));
  std::memcpy(D, b.D.data(), n * n * sizeof(double));
}

// model 0 cnh, 1 inh, 2 fiber; domain 0 material, 1 spatial;
// strategy 0 none, 1 scalar, 2 tensor; precision 64 or 32.
void* ref_op_create(void* l, int model, const double* params, int domain,
                    int strategy, int precision) {
  RefLevel* L = static_cast<RefLevel*>(l);
  RefOp* op = new RefOp;
  int st = guarded([&] {
    const Formulation form{Stability::stable,
                           domain == 0 ? Domain::material : Domain::spatial};
    const Strategy s = strategy == 0   ? Strategy::none
                       : strategy == 1 ? Strategy::scalar
                                       : Strategy::tensor;
    const ModelKind m = model == 0   ? ModelKind::cnh
                        : model == 1 ? ModelKind::inh
                                     : ModelKind::fiber;
    op->precision = precision;
    op->n = L->fe->dof_count();
    if (precision == 64)
      op->d = std::make_unique<ElasticOperator<double>>(
          *L->fe, m, params_from(params), form, s);
    else
      op->f = std::make_unique<ElasticOperator<float>>(
          *L->fe, m, params_from(params), form, s);
  });
  if (st != 0) {
    delete op;
    return nullptr;
  }
  return op;
}

void ref_op_destroy(void* o) { delete static_cast<RefOp*>(o); }

void ref_op_set_threads(void* o, int t) {
  RefOp* op = static_cast<RefOp*>(o);
  if (op->d) op->d->set_threads(t);
  if (op->f) op->f->set_threads(t);
}

int ref_op_linearize(void* o, const double* u) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    std::vector<double> uk(u, u + op->n);
    if (op->d)
      op->d->update_linearization(uk);
    else
      op->f->update_linearization(uk);
  });
}

// x/y are double* for precision 64, float* for precision 32.
int ref_op_apply(void* o, const void* x, void* y) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    if (op->d) {
      const double* xp = static_cast<const double*>(x);
      std::vector<double> xv(xp, xp + op->n), yv;
      op->d->apply_tangent(xv, yv);
      std::memcpy(y, yv.data(), op->n * sizeof(double));
    } else {
      const float* xp = static_cast<const float*>(x);
      std::vector<float> xv(xp, xp + op->n), yv;
      op->f->apply_tangent(xv, yv);
      std::memcpy(y, yv.data(), op->n * sizeof(float));
    }
  });
}

// Repeated applies on resident vectors (bench protocol, runner.cpp:84-105).
int ref_op_apply_repeat(void* o, const void* x, void* y, int reps) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    if (op->d) {
      const double* xp = static_cast<const double*>(x);
      std::vector<double> xv(xp, xp + op->n), yv;
      for (int r = 0; r < reps; ++r) op->d->apply_tangent(xv, yv);
      std::memcpy(y, yv.data(), op->n * sizeof(double));
    } else {
      const float* xp = static_cast<const float*>(x);
      std::vector<float> xv(xp, xp + op->n), yv;
      for (int r = 0; r < reps; ++r) op->f->apply_tangent(xv, yv);
      std::memcpy(y, yv.data(), op->n * sizeof(float));
    }
  });
}

int ref_op_residual(void* o, const void* u, void* r) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    if (op->d) {
      const double* xp = static_cast<const double*>(u);
      std::vector<double> xv(xp, xp + op->n), yv;
      op->d->evaluate_residual(xv, yv);
      std::memcpy(r, yv.data(), op->n * sizeof(double));
    } else {
      const float* xp = static_cast<const float*>(u);
      std::vector<float> xv(xp, xp + op->n), yv;
      op->f->evaluate_residual(xv, yv);
      std::memcpy(r, yv.data(), op->n * sizeof(float));
    }
  });
}

// diag: double*/float* by precision; n_bad receives the number of nonpositive
// free entries, bad (optional, capacity cap) their indices.
int ref_op_diagonal(void* o, void* diag, int64_t* n_bad, int64_t* bad,
                    int64_t cap) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    if (op->d) {
      auto [d, b] = op->d->compute_diagonal();
      std::memcpy(diag, d.data(), op->n * sizeof(double));
      *n_bad = static_cast<int64_t>(b.size());
      for (int64_t i = 0; bad && i < cap && i < *n_bad; ++i) bad[i] = b[i];
    } else {
      auto [d, b] = op->f->compute_diagonal();
      std::memcpy(diag, d.data(), op->n * sizeof(float));
      *n_bad = static_cast<int64_t>(b.size());
      for (int64_t i = 0; bad && i < cap && i < *n_bad; ++i) bad[i] = b[i];
    }
  });
}

// Ledger of one cell: returns storage/traffic bytes (ledger.cpp:22-76).
int ref_ledger(int model, int domain, int strategy, int* storage,
               int* traffic) {
  return guarded([&] {
    const ModelKind m = model == 0   ? ModelKind::cnh
                        : model == 1 ? ModelKind::inh
                                     : ModelKind::fiber;
    const Strategy s = strategy == 0   ? Strategy::none
                       : strategy == 1 ? Strategy::scalar
                                       : Strategy::tensor;
    const CellLedger l =
        cell_ledger(m, domain == 0 ? Domain::material : Domain::spatial, s);
    *storage = l.storage_bytes();
    *traffic = l.traffic_bytes();
  });
}

// Transfers between two levels (mesh.hpp:245-289). kind 0 prolongate
// (coarse->fine), 1 restrict (fine->coarse), 2 interpolate_down (fine->coarse).
// prec 64 or 32 selects the vector type.
int ref_transfer(void* fine, void* coarse, int kind, int prec, const void* in,
                 void* out) {
  RefLevel* F = static_cast<RefLevel*>(fine);
  RefLevel* C = static_cast<RefLevel*>(coarse);
  return guarded([&] {
    TransferOp t(*F->fe, *C->fe);
    auto run = [&](auto tag) {
      using N = decltype(tag);
      const int64_t nin = kind == 0 ? C->fe->dof_count() : F->fe->dof_count();
      const N* ip = static_cast<const N*>(in);
      std::vector<N> iv(ip, ip + nin), ov;
      if (kind == 0)
        t.prolongate(iv, ov);
      else if (kind == 1)
        t.restrict_(iv, ov);
      else
        t.interpolate_down(iv, ov);
      std::memcpy(out, ov.data(), ov.size() * sizeof(N));
    };
    if (prec == 64)
      run(double{});
    else
      run(float{});
  });
}

// Lanczos estimate (solver.hpp:262-308) on a linearized operator with the
// given diagonal.
int ref_estimate_eigenvalues(void* o, const void* diag, int iterations,
                             uint64_t seed, double* lmin, double* lmax) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    if (op->d) {
      const double* dp = static_cast<const double*>(diag);
      std::vector<double> d(dp, dp + op->n);
      auto [a, b] = estimate_eigenvalues(*op->d, d, iterations, seed);
      *lmin = a;
      *lmax = b;
    } else {
      const float* dp = static_cast<const float*>(diag);
      std::vector<float> d(dp, dp + op->n);
      auto [a, b] = estimate_eigenvalues(*op->f, d, iterations, seed);
      *lmin = a;
      *lmax = b;
    }
  });
}

// Chebyshev smoothing (solver.hpp:312-362): setup from diag + lmax estimate,
// then one smooth() call. x is in/out. Vectors by precision.
int ref_chebyshev(void* o, const void* diag, double lmax_est, int degree,
                  double range_factor, double safety, const void* b, void* x,
                  int zero_start) {
  RefOp* op = static_cast<RefOp*>(o);
  return guarded([&] {
    SmootherConfig cfg;
    cfg.degree = degree;
    cfg.range_factor = range_factor;
    cfg.safety = safety;
    auto run = [&](auto& oper, auto tag) {
      using N = decltype(tag);
      const N* dp = static_cast<const N*>(diag);
      const N* bp = static_cast<const N*>(b);
      N* xp = static_cast<N*>(x);
      std::vector<N> d(dp, dp + op->n), bv(bp, bp + op->n), xv(xp, xp + op->n),
          r, dd;
      ChebyshevSmoother<N> sm;
      sm.setup(d, lmax_est, cfg);
      sm.smooth(oper, xv, bv, r, dd, zero_start != 0);
      std::memcpy(xp, xv.data(), op->n * sizeof(N));
    };
    if (op->d)
      run(*op->d, double{});
    else
      run(*op->f, float{});
  });
}

}  // extern "C"

// ---- hp-multigrid (solver.hpp:437-581) and an outer PCG composed from
// reference primitives (SURVEY §8(c) gap 4: the reference has no outer CG;
// cfg4 asks for one).  The V-cycle, smoothers, transfers, Lanczos and coarse
// solver are the reference's own MgHierarchy<float>.
namespace {
struct RefMg {
  std::unique_ptr<MgHierarchy<float>> mg;
  const FeLevel* fe = nullptr;
};
}  // namespace

extern "C" {

// coarse_direct_limit: DoF threshold below which the reference factorises the
// coarsest level densely (default 2000); 0 forces its Jacobi-PCG path.
void* ref_mg_create(void* l, int model, const double* params, int strategy, int degree, double range_factor,
                    double safety, int eig_iterations, double deform_amp, int dirichlet_faces,
                    int64_t coarse_direct_limit) {
  RefLevel* L = static_cast<RefLevel*>(l);
  RefMg* m = new RefMg;
  int st = guarded([&] {
    const Formulation form{Stability::stable, Domain::material};
    const Strategy s = strategy == 0 ? Strategy::none : strategy == 1 ? Strategy::scalar : Strategy::tensor;
    const ModelKind mk = model == 0 ? ModelKind::cnh : model == 1 ? ModelKind::inh : ModelKind::fiber;
    SmootherConfig sc;
    sc.degree = degree;
    sc.range_factor = range_factor;
    sc.safety = safety;
    sc.eig_iterations = eig_iterations;
    std::array<bool, 6> faces{};
    for (int f = 0; f < 6; ++f) faces[f] = (dirichlet_faces >> f) & 1;
    m->fe = L->fe.get();
    m->mg = std::make_unique<MgHierarchy<float>>(*L->fe, faces, mk, params_from(params), form, s, KernelConfig{},
                                                 sc, DeformMap{deform_amp}, coarse_direct_limit);
  });
  if (st != 0) {
    delete m;
    return nullptr;
  }
  return m;
}

void ref_mg_destroy(void* m) { delete static_cast<RefMg*>(m); }
int ref_mg_n_levels(void* m) { return static_cast<RefMg*>(m)->mg->n_levels(); }

int ref_mg_update_linearization(void* m, const double* u) {
  RefMg* M = static_cast<RefMg*>(m);
  return guarded([&] {
    std::vector<double> uk(u, u + M->fe->dof_count());
    M->mg->update_linearization(uk);
  });
}

int ref_mg_precondition(void* m, const double* r, double* z) {
  RefMg* M = static_cast<RefMg*>(m);
  return guarded([&] {
    const int64_t n = M->fe->dof_count();
    std::vector<double> rv(r, r + n), zv;
    M->mg->precondition(rv, zv);
    std::memcpy(z, zv.data(), n * sizeof(double));
  });
}

// Preconditioned CG in double (dot_d accumulation, solver.hpp:95-106) with the
// reference operator and (optionally) the reference V-cycle; x starts at 0.
// Stops when ||r|| <= rtol ||b||; returns iterations and the residual history.
int ref_pcg_solve(void* o, void* m, const double* b, double* x, double rtol, int maxit, int* iters,
                  double* history) {
  RefOp* op = static_cast<RefOp*>(o);
  RefMg* M = static_cast<RefMg*>(m);
  return guarded([&] {
    const int64_t n = op->n;
    std::vector<double> bv(b, b + n), xv(n, 0.0), r = bv, z(n), p(n), ap(n);
    auto prec = [&](const std::vector<double>& rr, std::vector<double>& zz) {
      if (M)
        M->mg->precondition(rr, zz);
      else
        zz = rr;
    };
    const double bnorm = norm_d(bv);
    int it = 0;
    if (history) history[0] = 1.0;
    if (bnorm == 0) {
      *iters = 0;
      std::memset(x, 0, n * sizeof(double));
      return;
    }
    prec(r, z);
    p = z;
    double rz = dot_d(r, z);
    for (it = 0; it < maxit; ++it) {
      op->d->apply_tangent(p, ap);
      const double alpha = rz / dot_d(p, ap);
      for (int64_t i = 0; i < n; ++i) {
        xv[i] += alpha * p[i];
        r[i] -= alpha * ap[i];
      }
      const double rel = norm_d(r) / bnorm;
      if (history) history[it + 1] = rel;
      if (rel <= rtol) {
        ++it;
        break;
      }
      prec(r, z);
      const double rz_new = dot_d(r, z);
      const double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    *iters = it;
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

}  // extern "C"

// ---- residual with loads and the reference's Newton solve (run_solve_with,
// runner.cpp:166-204, one increment): evaluate_residual, newton_solve with
// FGMRES(30) + MgHierarchy<float>.
extern "C" {

int ref_residual_with_pressure(void* l, int model, const double* params, double pressure, int face,
                               double load_scale, const double* u, double* r) {
  RefLevel* L = static_cast<RefLevel*>(l);
  return guarded([&] {
    Loads loads;
    loads.pressure = pressure;
    loads.pressure_face = face;
    const ModelKind mk = model == 0 ? ModelKind::cnh : model == 1 ? ModelKind::inh : ModelKind::fiber;
    ElasticOperator<double> op(*L->fe, mk, params_from(params), {Stability::stable, Domain::material},
                               Strategy::none, KernelConfig{}, loads);
    op.set_load_scale(load_scale);
    std::vector<double> uv(u, u + L->fe->dof_count()), rv;
    op.evaluate_residual(uv, rv);
    std::memcpy(r, rv.data(), rv.size() * sizeof(double));
  });
}

// Body force and traction fixtures of the loads parity test (the product
// takes them as C callbacks; tests/test_gpu_parity.py defines the same
// expressions): B(X) = (0.3 + sin X0, X1 X2 - 0.2, 1 - X0^2),
// h(X, N) = (N0 + 0.5 X1, 0.25 N1 X2, X0 - N2).
int ref_residual_with_loads(void* l, int model, const double* params, double pressure, int face, int body,
                            int traction_faces, double load_scale, const double* u, double* r) {
  RefLevel* L = static_cast<RefLevel*>(l);
  return guarded([&] {
    Loads loads;
    loads.pressure = pressure;
    loads.pressure_face = face;
    if (body)
      loads.body_force = [](const Vec3d& x) { return Vec3d{{{0.3 + std::sin(x[0]), x[1] * x[2] - 0.2, 1.0 - x[0] * x[0]}}}; };
    if (traction_faces) {
      for (int f = 0; f < 6; ++f) loads.traction_faces[f] = (traction_faces >> f) & 1;
      loads.traction = [](const Vec3d& x, const Vec3d& n) {
        return Vec3d{{{n[0] + 0.5 * x[1], 0.25 * n[1] * x[2], x[0] - n[2]}}};
      };
    }
    const ModelKind mk = model == 0 ? ModelKind::cnh : model == 1 ? ModelKind::inh : ModelKind::fiber;
    ElasticOperator<double> op(*L->fe, mk, params_from(params), {Stability::stable, Domain::material},
                               Strategy::none, KernelConfig{}, loads);
    op.set_load_scale(load_scale);
    std::vector<double> uv(u, u + L->fe->dof_count()), rv;
    op.evaluate_residual(uv, rv);
    std::memcpy(r, rv.data(), rv.size() * sizeof(double));
  });
}

int ref_newton_pressure(void* l, int model, const double* params, double pressure, int face, int degree,
                        double deform_amp, int dirichlet_faces, int64_t coarse_direct_limit, double* u_out,
                        int* newton_its, int* fgmres_its, double* final_res) {
  RefLevel* L = static_cast<RefLevel*>(l);
  return guarded([&] {
    Loads loads;
    loads.pressure = pressure;
    loads.pressure_face = face;
    const ModelKind mk = model == 0 ? ModelKind::cnh : model == 1 ? ModelKind::inh : ModelKind::fiber;
    const Formulation form{Stability::stable, Domain::material};
    ElasticOperator<double> op(*L->fe, mk, params_from(params), form, Strategy::none, KernelConfig{}, loads);
    SmootherConfig sc;
    sc.degree = degree;
    std::array<bool, 6> faces{};
    for (int f = 0; f < 6; ++f) faces[f] = (dirichlet_faces >> f) & 1;
    MgHierarchy<float> mg(*L->fe, faces, mk, params_from(params), form, Strategy::none, KernelConfig{}, sc,
                          DeformMap{deform_amp}, coarse_direct_limit);
    std::vector<double> u(L->fe->dof_count(), 0.0);
    L->fe->dirichlet_set_values(u);
    op.set_load_scale(1.0);
    const NewtonStats st = newton_solve(op, &mg, u, NewtonConfig{}, FgmresConfig{});
    int lin = 0;
    for (const auto& s : st.steps) lin += s.fgmres_iters;
    *newton_its = st.iterations;
    *fgmres_its = lin;
    *final_res = st.final_residual;
    std::memcpy(u_out, u.data(), u.size() * sizeof(double));
  });
}

}  // extern "C"

// ---- the reference's forward-stability sweep (stability.cpp:163-251) ----
extern "C" int ref_stability_sweep(const double* scales, int n_scales, int samples, uint64_t seed,
                                   const double* params, double* max_rel_error, int64_t* count_invalid) {
  return guarded([&] {
    SweepConfig cfg;
    cfg.scales.assign(scales, scales + n_scales);
    cfg.samples_per_scale = samples;
    cfg.seed = seed;
    cfg.params = params_from(params);
    const std::vector<SweepRecord> recs = run_sweep(cfg);
    for (std::size_t i = 0; i < recs.size(); ++i) {
      max_rel_error[i] = recs[i].max_rel_error;
      count_invalid[i] = recs[i].count_invalid;
    }
  });
}
