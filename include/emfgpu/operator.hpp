// C++ adapter over the emfgpu C ABI with the method signatures of the
// reference's ElasticOperator<Number> (proj/include/elastmf/operator.hpp:49-204),
// FeLevel (mesh.hpp:71-138), TransferOp (mesh.hpp:157-182) and
// ChebyshevSmoother (solver.hpp:312-362), so reference-style host code
// (solvers templated on the operator type, the throughput driver
// runner.cpp:55-146) can swap the CPU operator for the B200 one.
// Header-only; link against libemfgpu.so.  Errors become exceptions named
// like the reference's (errors.hpp:15-93).
#ifndef EMFGPU_OPERATOR_HPP
#define EMFGPU_OPERATOR_HPP

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../emfgpu.h"

namespace emfgpu {

struct Error : std::runtime_error {
  emfgpu_status code;
  Error(emfgpu_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ConfigError : Error {
  using Error::Error;
};
struct StaleCache : Error {
  using Error::Error;
};
struct NonPositiveJacobian : Error {
  std::int64_t element;
  int qpoint;
  NonPositiveJacobian(emfgpu_status c, const std::string& m, std::int64_t e, int q) : Error(c, m), element(e), qpoint(q) {}
};

inline void throw_status(emfgpu_status st, const char* msg, std::int64_t e = -1, int q = -1) {
  if (st == EMFGPU_OK) return;
  if (st == EMFGPU_ERR_CONFIG) throw ConfigError(st, msg);
  if (st == EMFGPU_ERR_STALE) throw StaleCache(st, msg);
  if (st == EMFGPU_ERR_NUMERICAL && e >= 0) throw NonPositiveJacobian(st, msg, e, q);
  throw Error(st, msg);
}

enum class ModelKind { cnh = EMFGPU_CNH, inh = EMFGPU_INH, fiber = EMFGPU_FIBER };
/// Formulation (material.hpp:17-23).  The device kernels implement the stable
/// formulation; Stability::standard is refused with ConfigError.
enum class Domain { material = 0, spatial = 1 };
enum class Stability { standard = 0, stable = 1 };
struct Formulation {
  Stability stability = Stability::stable;
  Domain domain = Domain::material;
};
/// KernelConfig (fastscalar.hpp:29-39); only the defaults are implemented
/// (other values -> ConfigError naming the field).
struct KernelConfig {
  int ln_series_terms = 16;
  int jpow_newton_steps = 3;
  int exp_mode = 0;   // ExpMode::exact
  int jpow_mode = 0;  // JpowMode::newton
};
using Vec3d = std::array<double, 3>;
/// Loads (operator.hpp:23-32): uniform pressure on one face (-x,+x,-y,+y,-z,+z
/// = 0..5), body force B(X) and tractions h(X, N) on the flagged faces.
struct Loads {
  double pressure = 0.0;
  int pressure_face = 1;
  std::function<Vec3d(const Vec3d&)> body_force;
  std::array<bool, 6> traction_faces{};
  std::function<Vec3d(const Vec3d&, const Vec3d&)> traction;
};
enum class Strategy { none = EMFGPU_NONE, scalar = EMFGPU_SCALAR, tensor = EMFGPU_TENSOR, cached_f = EMFGPU_CACHED_F };

/// FeLevel: structured (deformed) box with Q_p on GLL nodes, Dirichlet faces.
class FeLevel {
 public:
  explicit FeLevel(const emfgpu_level_desc& d) { throw_status(emfgpu_level_create(&d, &h_), emfgpu_global_last_error()); }
  /// build_cube(n0, level) + FeLevel(mesh, degree, DeformMap{amplitude}) (mesh.hpp:61, 73)
  FeLevel(int n, int degree, double deform_amplitude = 0.0, int dirichlet_faces = 1) {
    emfgpu_level_desc d{};
    d.nx = d.ny = d.nz = n;
    d.p = degree;
    d.extent[0] = d.extent[1] = d.extent[2] = 1.0;
    d.map = EMFGPU_MAP_REFERENCE;
    d.map_param[0] = deform_amplitude;
    d.dirichlet_faces = dirichlet_faces;
    throw_status(emfgpu_level_create(&d, &h_), emfgpu_global_last_error());
  }
  FeLevel(const FeLevel&) = delete;
  FeLevel& operator=(const FeLevel&) = delete;
  ~FeLevel() { emfgpu_level_destroy(h_); }
  std::int64_t dof_count() const { return emfgpu_level_n_dofs(h_); }
  std::int64_t n_elements() const { return emfgpu_level_n_elements(h_); }
  const emfgpu_level* handle() const { return h_; }

 private:
  emfgpu_level* h_ = nullptr;
};

/// ElasticOperator<Number> on one B200; Number = double or float.
template <typename Number>
class ElasticOperator {
  static_assert(sizeof(Number) == 8 || sizeof(Number) == 4, "Number must be double or float");

 public:
  ElasticOperator(const FeLevel& level, ModelKind model, const emfgpu_material& params, Strategy strategy)
      : ElasticOperator(level, model, params, Formulation{}, strategy, KernelConfig{}, Loads{}) {}
  ElasticOperator(const FeLevel& level, ModelKind model, const emfgpu_material& params, Domain domain,
                  Strategy strategy, const Loads& loads = {})
      : ElasticOperator(level, model, params, Formulation{Stability::stable, domain}, strategy, KernelConfig{},
                        loads) {}
  /// operator.hpp:55-70: (level, model, params, formulation, strategy, cfg, loads)
  ElasticOperator(const FeLevel& level, ModelKind model, const emfgpu_material& params, Formulation form,
                  Strategy strategy, const KernelConfig& cfg = {}, const Loads& loads = {})
      : level_(&level) {
    const emfgpu_formulation f{static_cast<int>(form.stability), static_cast<int>(form.domain)};
    const emfgpu_kernel_config k{cfg.ln_series_terms, cfg.jpow_newton_steps, cfg.exp_mode, cfg.jpow_mode};
    throw_status(emfgpu_op_create_ex(level.handle(), static_cast<int>(model), &params, &f,
                                     static_cast<int>(strategy), sizeof(Number) == 8 ? 64 : 32, &k, &h_),
                 emfgpu_global_last_error());
    set_loads(loads);
  }

  /// build_load_vector (operator.hpp:880-1008): the std::function members are
  /// evaluated on the host through C callbacks while the vector is built.
  void set_loads(const Loads& loads) {
    if (loads.pressure == 0.0 && !loads.body_force && !loads.traction) return;
    emfgpu_loads c{};
    c.pressure = loads.pressure;
    c.pressure_face = loads.pressure_face;
    if (loads.body_force) {
      c.body_force = [](const double X[3], double out[3], void* u) {
        const Vec3d v = (*static_cast<const std::function<Vec3d(const Vec3d&)>*>(u))(Vec3d{X[0], X[1], X[2]});
        out[0] = v[0], out[1] = v[1], out[2] = v[2];
      };
      c.body_force_user = const_cast<void*>(static_cast<const void*>(&loads.body_force));
    }
    if (loads.traction) {
      c.traction = [](const double X[3], const double N[3], double out[3], void* u) {
        const Vec3d v = (*static_cast<const std::function<Vec3d(const Vec3d&, const Vec3d&)>*>(u))(
            Vec3d{X[0], X[1], X[2]}, Vec3d{N[0], N[1], N[2]});
        out[0] = v[0], out[1] = v[1], out[2] = v[2];
      };
      c.traction_user = const_cast<void*>(static_cast<const void*>(&loads.traction));
      for (int f = 0; f < 6; ++f)
        if (loads.traction_faces[f]) c.traction_faces |= 1 << f;
    }
    throw_status(emfgpu_op_set_loads(h_, &c), emfgpu_op_last_error(h_));
  }
  ElasticOperator(const ElasticOperator&) = delete;
  ElasticOperator& operator=(const ElasticOperator&) = delete;
  ~ElasticOperator() { emfgpu_op_destroy(h_); }

  const FeLevel& level() const { return *level_; }
  void set_threads(int) {}  // signature compatibility: parallelism is the GPU's
  std::int64_t n_dofs() const { return emfgpu_op_n_dofs(h_); }
  bool linearized() const { return emfgpu_op_linearized(h_) != 0; }
  std::uint64_t checksum() const { return emfgpu_op_checksum(h_); }

  /// operator.hpp:87
  void update_linearization(const std::vector<double>& u_k) {
    if ((std::int64_t)u_k.size() != n_dofs()) throw Error(EMFGPU_ERR_CONFIG, "update_linearization: size mismatch");
    std::int64_t e = -1;
    int q = -1;
    throw_status(emfgpu_op_update_linearization_host(h_, u_k.data(), &e, &q), emfgpu_op_last_error(h_), e, q);
  }

  /// operator.hpp:99-100 (y is resized, as y.assign does in the reference)
  void apply_tangent(const std::vector<Number>& du, std::vector<Number>& y) const {
    if ((std::int64_t)du.size() != n_dofs()) throw Error(EMFGPU_ERR_CONFIG, "apply_tangent: size mismatch");
    y.resize(du.size());
    throw_status(emfgpu_op_apply_host(h_, du.data(), y.data()), emfgpu_op_last_error(h_));
  }

  /// operator.hpp:94-95: r = (Grad v, P(u)) - load_scale * load, Dirichlet rows zero
  void evaluate_residual(const std::vector<Number>& u, std::vector<Number>& r) const {
    if ((std::int64_t)u.size() != n_dofs()) throw Error(EMFGPU_ERR_CONFIG, "evaluate_residual: size mismatch");
    r.resize(u.size());
    throw_status(emfgpu_op_residual_host(h_, u.data(), r.data()), emfgpu_op_last_error(h_));
  }
  /// operator.hpp:80
  void set_load_scale(double s) { throw_status(emfgpu_op_set_load_scale(h_, s), emfgpu_op_last_error(h_)); }

  /// Device-resident variant (stream-ordered; stream is a cudaStream_t).
  void apply_tangent_device(const Number* d_x, Number* d_y, void* stream = nullptr) const {
    throw_status(emfgpu_op_apply(h_, d_x, d_y, stream), emfgpu_op_last_error(h_));
  }

  /// operator.hpp:106-107: (diag, indices of nonpositive free entries, ascending)
  std::pair<std::vector<Number>, std::vector<std::int64_t>> compute_diagonal() const {
    std::vector<Number> d(n_dofs());
    std::int64_t nbad = 0;
    throw_status(emfgpu_op_compute_diagonal_host(h_, d.data(), &nbad), emfgpu_op_last_error(h_));
    std::vector<std::int64_t> bad;
    if (nbad > 0)
      for (std::int64_t i = 0; i < (std::int64_t)d.size(); ++i)
        if (!(d[i] > Number(0))) bad.push_back(i);
    return {std::move(d), std::move(bad)};
  }
  /// Same on a device diagonal: the index list comes from the device
  /// (emfgpu_op_compute_diagonal_indices), the diagonal stays in d_diag.
  std::vector<std::int64_t> compute_diagonal_device(Number* d_diag, std::int64_t capacity = 1 << 16,
                                                    void* stream = nullptr) const {
    std::vector<std::int64_t> idx(capacity);
    std::int64_t n = 0;
    throw_status(emfgpu_op_compute_diagonal_indices(h_, d_diag, idx.data(), capacity, &n, stream),
                 emfgpu_op_last_error(h_));
    idx.resize(static_cast<std::size_t>(std::min(n, capacity)));
    return idx;
  }

  emfgpu_op* handle() const { return h_; }

 private:
  const FeLevel* level_;
  emfgpu_op* h_ = nullptr;
};

/// MgHierarchy<Prec> (solver.hpp:437-581) on the device; Prec = float (default) or double.
class MgHierarchy {
 public:
  MgHierarchy(const FeLevel& fine, ModelKind model, const emfgpu_material& params, Strategy strategy,
              const emfgpu_mg_config* cfg = nullptr) {
    emfgpu_mg_config c;
    emfgpu_mg_default_config(&c);
    if (cfg) c = *cfg;
    throw_status(emfgpu_mg_create(fine.handle(), static_cast<int>(model), &params, static_cast<int>(strategy), &c,
                                  &h_),
                 emfgpu_global_last_error());
  }
  MgHierarchy(const MgHierarchy&) = delete;
  MgHierarchy& operator=(const MgHierarchy&) = delete;
  ~MgHierarchy() { emfgpu_mg_destroy(h_); }
  int n_levels() const { return emfgpu_mg_n_levels(h_); }
  emfgpu_mg* handle() const { return h_; }

 private:
  emfgpu_mg* h_ = nullptr;
};

struct NewtonStats {
  int iterations = 0;
  int linear_iterations = 0;
  double final_residual = 0.0;
};

/// newton_solve (solver.hpp:603-656): u in/out, FGMRES(30) right-preconditioned
/// by the hierarchy's V-cycle (or unpreconditioned when mg is null).
inline NewtonStats newton_solve(ElasticOperator<double>& op, MgHierarchy* mg, std::vector<double>& u,
                                const emfgpu_newton_config* cfg = nullptr) {
  emfgpu_newton_config c;
  emfgpu_newton_default_config(&c);
  if (cfg) c = *cfg;
  NewtonStats st;
  throw_status(emfgpu_newton_solve_host(op.handle(), mg ? mg->handle() : nullptr, u.data(), &c, &st.iterations,
                                        &st.linear_iterations, &st.final_residual),
               emfgpu_op_last_error(op.handle()));
  return st;
}

}  // namespace emfgpu

#endif
