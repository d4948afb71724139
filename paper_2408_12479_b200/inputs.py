"""Seeded synthetic inputs for the BASELINE configs (host logic, numpy).

The reference ships no golden vectors; inputs are defined by a
portable generator so the oracle, the reference build and the GPU path all see
bit-identical data:

* ``splitmix64`` / ``uniform01`` follow ``proj/include/elastmf/solver.hpp:209-219``
  (state += golden gamma, xor-shift-multiply finaliser, top 53 bits * 2^-53).
* Draws are taken in DoF order ``3*node + comp`` (``operator.hpp:254``).
* u0 = amp * sin(pi X) sin(pi Y) sin(pi Z) * (1,1,1) at the *pre-map* lattice
  positions (SURVEY §8(c') F2) plus ``-noise + 2*noise*uniform01`` (state 0),
  then Dirichlet DoFs are set to their (zero) values (``mesh.hpp:120-124``).
* v = -1 + 2*uniform01 (state 1), not masked (apply masks it, operator.hpp:604).
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start .. start+n-1 of splitmix64 started at ``state = seed``
    (output i is a pure function of i: state_i = seed + (i+1) * gamma)."""
    k = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int, start: int = 0) -> np.ndarray:
    """solver.hpp:217-219: (splitmix64(state) >> 11) * 2^-53."""
    return (splitmix64_stream(seed, n, start) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def gauss_lobatto(n: int) -> np.ndarray:
    """GLL points on [-1,1] (restates mesh.cpp:58-81: Newton on P'_{n-1})."""
    m = n - 1
    pts = np.empty(n)
    pts[0], pts[-1] = -1.0, 1.0

    def leg(k, x):
        p0, p1 = 1.0, x
        if k == 0:
            return p0
        for j in range(2, k + 1):
            p0, p1 = p1, ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j
        return p1

    def dleg(k, x):
        if k == 0:
            return 0.0
        return k * (leg(k - 1, x) - x * leg(k, x)) / (1.0 - x * x)

    for i in range(1, m):
        x = np.cos(np.pi * (m - i) / m)
        for _ in range(100):
            g = dleg(m, x)
            gp = (2.0 * x * g - m * (m + 1.0) * leg(m, x)) / (1.0 - x * x)
            dx = g / gp
            x -= dx
            if abs(dx) < 1e-15:
                break
        pts[i] = x
    return np.sort(pts)


def lattice_axis(n_el: int, p: int, extent: float = 1.0) -> np.ndarray:
    """1D lattice positions (mesh.cpp:147-151): (e + (xi_l + 1)/2) * h."""
    nodes = gauss_lobatto(p + 1)
    h = extent / n_el
    idx = np.arange(n_el * p + 1)
    e = np.minimum(idx // p, n_el - 1)
    l = idx - e * p
    return (e + 0.5 * (nodes[l] + 1.0)) * h


def lattice_positions(nx: int, ny: int, nz: int, p: int, extent=(1.0, 1.0, 1.0), periodic_y=False):
    """Pre-map lattice positions X, Y, Z flattened in node order (a fastest).
    A periodic y lattice drops the node row at y = extent (it is row 0)."""
    ax = lattice_axis(nx, p, extent[0])
    ay = lattice_axis(ny, p, extent[1])
    if periodic_y:
        ay = ay[:-1]
    az = lattice_axis(nz, p, extent[2])
    Z, Y, X = np.meshgrid(az, ay, ax, indexing="ij")
    return X.ravel(), Y.ravel(), Z.ravel()


def dirichlet_mask(nx, ny, nz, p, faces: int, periodic_y=False) -> np.ndarray:
    """Per-DoF mask for clamped faces (bit f: -x,+x,-y,+y,-z,+z), mesh.cpp:213-246."""
    mx, my, mz = nx * p + 1, ny * p + (0 if periodic_y else 1), nz * p + 1
    c, b, a = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    on = np.zeros(c.shape, bool)
    tests = [a == 0, a == mx - 1, b == 0, b == my - 1, c == 0, c == mz - 1]
    for f in range(6):
        if (faces >> f) & 1:
            on |= tests[f]
    return np.repeat(on.ravel(), 3)


def make_u0(nx, ny, nz, p, amp=0.05, noise=1e-3, seed=0, faces=1, extent=(1.0, 1.0, 1.0)):
    X, Y, Z = lattice_positions(nx, ny, nz, p, extent)
    s = amp * np.sin(np.pi * X) * np.sin(np.pi * Y) * np.sin(np.pi * Z)
    u = np.repeat(s, 3)
    if noise != 0.0:
        u = u + (-noise + 2.0 * noise * uniform01(seed, u.size))
    u[dirichlet_mask(nx, ny, nz, p, faces)] = 0.0
    return u


def make_v(ndofs: int, seed: int = 1) -> np.ndarray:
    return -1.0 + 2.0 * uniform01(seed, ndofs)


def periodic_to_open(v: np.ndarray, nx, ny, nz, p) -> np.ndarray:
    """P: a vector on a periodic-y lattice -> the open lattice with the seam
    row duplicated (row my = row 0)."""
    mx, my, mz = nx * p + 1, ny * p, nz * p + 1
    a = v.reshape(mz, my, mx, -1)
    return np.concatenate([a, a[:, :1]], axis=1).reshape(-1)


def open_to_periodic(v: np.ndarray, nx, ny, nz, p) -> np.ndarray:
    """P^T: sums the duplicated seam row of the open lattice into row 0."""
    mx, my, mz = nx * p + 1, ny * p, nz * p + 1
    a = v.reshape(mz, my + 1, mx, -1).copy()
    a[:, 0] += a[:, my]
    return a[:, :my].reshape(-1)


def make_u0_planes(nx, ny, nz, p, c0, c1, amp=0.05, noise=1e-3, seed=0, faces=1, extent=(1.0, 1.0, 1.0)):
    """Node planes c0..c1 (inclusive) of make_u0(nx, ny, nz, p, ...), generated
    without the rest of the global vector (z slabs of weak-scaled meshes)."""
    ax = lattice_axis(nx, p, extent[0])
    ay = lattice_axis(ny, p, extent[1])
    az = lattice_axis(nz, p, extent[2])[c0:c1 + 1]
    Z, Y, X = np.meshgrid(az, ay, ax, indexing="ij")
    s = amp * np.sin(np.pi * X.ravel()) * np.sin(np.pi * Y.ravel()) * np.sin(np.pi * Z.ravel())
    u = np.repeat(s, 3)
    plane = 3 * (nx * p + 1) * (ny * p + 1)
    if noise != 0.0:
        u = u + (-noise + 2.0 * noise * uniform01(seed, u.size, c0 * plane))
    mz = nz * p + 1
    mask = dirichlet_mask(nx, ny, nz, p, faces & 0b001111)[: u.size]
    if faces & 16 and c0 == 0:
        mask[:plane] = True
    if faces & 32 and c1 == mz - 1:
        mask[-plane:] = True
    u[mask] = 0.0
    return u


def make_v_planes(nx, ny, nz, p, c0, c1, seed: int = 1) -> np.ndarray:
    """Node planes c0..c1 of make_v(global n_dofs, seed)."""
    plane = 3 * (nx * p + 1) * (ny * p + 1)
    return -1.0 + 2.0 * uniform01(seed, (c1 - c0 + 1) * plane, c0 * plane)
