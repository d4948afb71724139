// Reference-style driver through the C++ adapter (include/emfgpu/operator.hpp):
// one pressure increment solved with newton_solve + MgHierarchy, the way
// runner.cpp:166-204 drives the reference.  Prints "newton <its> <lin> <res> <|u|>".
#include <cmath>
#include <cstdio>

#include "emfgpu/operator.hpp"

int main() {
  emfgpu::FeLevel fe(4, 2, 0.05, 1);  // 4^3 Q2, DeformMap amplitude 0.05, -x clamped
  emfgpu_material p{};
  p.mu = 1.0;
  p.lambda = 10.0;
  p.kappa_b = 50.0;
  p.k1 = 2.0;
  p.k2 = 5.0;
  p.a = 3.62;
  p.b = 34.3;
  p.phi = 40.0 * 3.14159265358979323846 / 180.0;
  p.e1[0] = p.e2[1] = p.e3[2] = 1.0;
  emfgpu::Loads loads;
  loads.pressure = 0.2;
  loads.pressure_face = 1;
  emfgpu::ElasticOperator<double> op(fe, emfgpu::ModelKind::inh, p, emfgpu::Domain::material, emfgpu::Strategy::none,
                                     loads);
  emfgpu_mg_config cfg;
  emfgpu_mg_default_config(&cfg);
  cfg.coarse_direct_limit = 0;  // the golden fixture's coarse CG path
  emfgpu::MgHierarchy mg(fe, emfgpu::ModelKind::inh, p, emfgpu::Strategy::none, &cfg);
  std::vector<double> u(op.n_dofs(), 0.0);
  op.set_load_scale(1.0);
  const emfgpu::NewtonStats st = emfgpu::newton_solve(op, &mg, u);
  std::vector<double> r;
  op.evaluate_residual(u, r);
  double nu = 0, nr = 0;
  for (double v : u) nu += v * v;
  for (double v : r) nr += v * v;
  std::printf("newton %d %d %.17g %.17g %.17g\n", st.iterations, st.linear_iterations, st.final_residual,
              std::sqrt(nu), std::sqrt(nr));
  return 0;
}
