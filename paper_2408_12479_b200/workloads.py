"""The BASELINE.json configurations as reusable workload builders (host logic).

cfg0  8^3  Q2 cNH (mu=1, lambda=10), affine unit cube, fp64, strategy none.
cfg1  32^3 Q3 cNH, all strategies, fp64 and fp32.
cfg2  64^3 Q4 iNH (mu=1, kappa=1000) on x' = x + 0.1 sin(2 pi y) e_x, u0 amplitude
      0.1 at pre-map coordinates.  The literal +-1e-3 per-DoF noise makes
      det F <= 0 (SURVEY §8(c') F1: the reference throws NonPositiveJacobian);
      the throughput variant scales the noise with the node spacing,
      1e-3 * 8 / n (SURVEY's suggested variant), and is checked admissible.
cfg4  48^3 Q4 iNH, fp64 PCG to 1e-8 with an fp32 hp-multigrid V-cycle
      (Q4 -> Q2 -> Q1 -> 24^3 -> 12^3 -> 6^3, Chebyshev degree 5).  The literal
      kappa/mu = 1000 with the indefinite u0 does not converge with the
      reference algorithm (F3/F4); the timed variant is the well-posed one
      SURVEY §8(c') prescribes: u0 = 0, kappa/mu = 50, affine cube.
cfg3  Thick tube r in [1, 1.3], length 10: 16 (radial) x 128 (circumferential,
      periodic) x 256 (axial) Q3 = 43 408 512 DoFs; fibre model (mu=1,
      kappa=100, k1=2, k2=5, +-40 deg from the circumferential direction in the
      circumferential-axial plane, dispersion a=3.62, b=34.3 — BASELINE leaves
      them open, SURVEY §8(c) gap 2), per-qp cylindrical fibre frames; u0 =
      5% radial expansion 0.05 (x, y, 0) + 1e-3 seeded noise; no Dirichlet
      face (apply only); cached stress+tangent strategy, fp64 and fp32.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import inputs as I


@dataclass
class Workload:
    name: str
    n: tuple
    p: int
    model: str
    params: dict
    map: str = "reference"
    map_param: tuple = (0.0,)
    u_amp: float = 0.05
    noise: float = 1e-3
    faces: int = 1

    @property
    def ndofs(self):
        nx, ny, nz = self.n
        return 3 * (nx * self.p + 1) * (ny * self.p + (0 if self.periodic_y else 1)) * (nz * self.p + 1)

    def u0(self):
        nx, ny, nz = self.n
        return I.make_u0(nx, ny, nz, self.p, amp=self.u_amp, noise=self.noise, faces=self.faces)

    def v(self, seed=1):
        return I.make_v(self.ndofs, seed)

    periodic_y: bool = False

    def level(self, **kw):
        from .emfgpu import FeLevel
        nx, ny, nz = self.n
        return FeLevel(nx, ny, nz, p=self.p, map=self.map, map_param=self.map_param, dirichlet_faces=self.faces,
                       periodic_y=self.periodic_y, **kw)

    def material(self):
        from .emfgpu import MaterialParams
        return MaterialParams(**self.params)


def cfg0():
    return Workload("cfg0", (8, 8, 8), 2, "cnh", dict(mu=1.0, lam=10.0))


def cfg1():
    return Workload("cfg1", (32, 32, 32), 3, "cnh", dict(mu=1.0, lam=10.0))


def cfg2(literal=False, n=64):
    return Workload("cfg2" + ("_literal" if literal else "_scaled_noise"), (n, n, n), 4, "inh",
                    dict(mu=1.0, kappa_b=1000.0), map="shear_x", map_param=(0.1,), u_amp=0.1,
                    noise=1e-3 if literal else 1e-3 * 8.0 / n)


def cfg4(wellposed=True, n=48):
    if wellposed:
        return Workload("cfg4_wellposed", (n, n, n), 4, "inh", dict(mu=1.0, kappa_b=50.0), u_amp=0.0, noise=0.0)
    return Workload("cfg4_literal", (n, n, n), 4, "inh", dict(mu=1.0, kappa_b=1000.0), map="shear_x",
                    map_param=(0.1,), u_amp=0.1, noise=1e-3)


def rhs(w: Workload, seed=2):
    """Seeded right-hand side U[-1,1] with Dirichlet rows zeroed (cfg4)."""
    b = I.make_v(w.ndofs, seed)
    nx, ny, nz = w.n
    b[I.dirichlet_mask(nx, ny, nz, w.p, w.faces)] = 0.0
    return b


def cfg3(n=(16, 128, 256)):
    return Workload("cfg3", tuple(n), 3, "fiber",
                    dict(mu=1.0, kappa_b=100.0, k1=2.0, k2=5.0, a=3.62, b=34.3, phi=float(np.deg2rad(40.0))),
                    map="tube", map_param=(1.0, 1.3, 10.0), u_amp=0.05, noise=1e-3, faces=0, periodic_y=True)


def tube_u0(w: Workload, coords: np.ndarray, seed=0):
    """cfg3 linearization point: 5% radial expansion plus seeded noise."""
    c = coords.reshape(-1, 3)
    u = np.zeros_like(c)
    u[:, 0] = w.u_amp * c[:, 0]
    u[:, 1] = w.u_amp * c[:, 1]
    u = u.reshape(-1)
    return u + (-w.noise + 2.0 * w.noise * I.uniform01(seed, u.size))
