"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/liboracle.so (the C
restatement in emf_oracle.c).  Used by tests/, smoke() and bench.py's
cpu_baseline leg as the checker, never as the product path."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
MODELS = {"cnh": 0, "inh": 1, "fiber": 2}
STRATEGIES = {"none": 0, "scalar": 1, "tensor": 2, "cachedF": 0}
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i64 = C.c_void_p, C.c_int64
        L.orc_op_create.restype = vp
        L.orc_op_create.argtypes = [C.c_int] * 4 + [vp, C.c_int, C.c_int, vp, C.c_int, C.c_int]
        L.orc_op_destroy.argtypes = [vp]
        L.orc_op_ndofs.restype = i64
        L.orc_op_ndofs.argtypes = [vp]
        L.orc_op_jacobians.argtypes = [vp, vp]
        L.orc_op_mask.argtypes = [vp, vp]
        L.orc_op_linearize.argtypes = [vp, vp, C.POINTER(i64), C.POINTER(C.c_int)]
        L.orc_op_apply.argtypes = [vp, vp, vp]
        L.orc_op_diagonal.argtypes = [vp, vp, C.POINTER(i64)]
        L.orc_op_chebyshev.argtypes = [vp, vp, C.c_double, C.c_int, C.c_double, C.c_double, vp, vp, C.c_int]
        L.orc_op_estimate_eigenvalues.argtypes = [vp, vp, C.c_int, C.c_uint64, C.POINTER(C.c_double),
                                                  C.POINTER(C.c_double)]
        L.orc_transfer.argtypes = [C.c_int] * 10 + [vp, vp]
        L.orc_lattice_coords.argtypes = [C.c_int] * 4 + [vp, C.c_int, vp, vp]
        L.orc_structure_tensors.argtypes = [vp, vp]
        L.orc_op_element_locals.argtypes = [vp, vp, vp, i64, i64]
        L.orc_op_set_frames.argtypes = [vp, vp, vp]
        L.orc_op_set_domain.argtypes = [vp, C.c_int]
        L.orc_op_residual.argtypes = [vp, vp, vp, C.c_double, C.c_int, C.c_double, vp]
        L.orc_pressure_load.argtypes = [vp, vp, C.c_double, C.c_int, vp]
        L.orc_basis_tables.argtypes = [C.c_int] + [vp] * 5
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


def lattice_coords(nx, ny, nz, p, extent=(1.0, 1.0, 1.0), map_kind=0, prm=(0.0, 1.0)):
    out = np.empty(3 * (nx * p + 1) * (ny * p + 1) * (nz * p + 1))
    lib().orc_lattice_coords(nx, ny, nz, p, _p(np.asarray(extent, np.float64)), map_kind,
                             _p(np.asarray(prm, np.float64)), _p(out))
    return out


def basis_tables(p):
    n = p + 1
    nodes, qp, qw = np.empty(n), np.empty(n), np.empty(n)
    B, D = np.empty(n * n), np.empty(n * n)
    lib().orc_basis_tables(p, _p(nodes), _p(qp), _p(qw), _p(B), _p(D))
    return nodes, qp, qw, B.reshape(n, n), D.reshape(n, n)


def structure_tensors(params):
    out = np.empty(21)
    lib().orc_structure_tensors(_p(np.asarray(params, np.float64)), _p(out))
    return out


class OracleOperator:
    """Mirror of ElasticOperator<Number> (operator.hpp:49-204); domain 0 material, 1 spatial."""

    def __init__(self, nx, ny, nz, p, coords=None, faces=1, model="cnh", params=None,
                 strategy="none", precision=64, domain=0):
        from oracle.refbind import material_params
        if coords is None:
            coords = lattice_coords(nx, ny, nz, p)
        self.coords = np.ascontiguousarray(coords, np.float64)
        self.params = material_params() if params is None else np.asarray(params, np.float64)
        self.precision = precision
        self.dtype = np.float64 if precision == 64 else np.float32
        self.dims = (nx, ny, nz, p)
        self.h = lib().orc_op_create(nx, ny, nz, p, _p(self.coords), faces, MODELS[model], _p(self.params),
                                     STRATEGIES[strategy], precision)
        if not self.h:
            raise OracleError(1, "create")
        lib().orc_op_set_domain(self.h, int(domain))
        self.n = lib().orc_op_ndofs(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_op_destroy(self.h)

    def jacobians(self):
        nx, ny, nz, p = self.dims
        out = np.empty(nx * ny * nz * (p + 1) ** 3 * 9)
        lib().orc_op_jacobians(self.h, _p(out))
        return out

    def mask(self):
        out = np.empty(self.n, np.uint8)
        lib().orc_op_mask(self.h, _p(out))
        return out

    def update_linearization(self, u):
        u = np.ascontiguousarray(u, np.float64)
        e, q = C.c_int64(-1), C.c_int(-1)
        st = lib().orc_op_linearize(self.h, _p(u), C.byref(e), C.byref(q))
        if st:
            raise OracleError(st, f"element={e.value} qpoint={q.value}")

    def apply(self, x):
        x = np.ascontiguousarray(x, self.dtype)
        y = np.empty(self.n, self.dtype)
        st = lib().orc_op_apply(self.h, _p(x), _p(y))
        if st:
            raise OracleError(st)
        return y

    def residual(self, u, pressure=0.0, face=1, load_scale=1.0):
        """evaluate_residual with a face pressure (operator.hpp:623-641, 925-1003)."""
        u = np.ascontiguousarray(u, self.dtype)
        r = np.empty(self.n, self.dtype)
        st = lib().orc_op_residual(self.h, _p(self.coords), _p(u), pressure, face, load_scale, _p(r))
        if st:
            raise OracleError(st)
        return r

    def pressure_load(self, pressure, face=1):
        out = np.empty(self.n)
        lib().orc_pressure_load(self.h, _p(self.coords), pressure, face, _p(out))
        return out

    def set_frames(self, h, m1):
        """Per-qp fibre frame field (12*nqp H4,H6 and 6*nqp M1s, SoA); EXT of the reference."""
        h = np.ascontiguousarray(h, np.float64)
        m1 = np.ascontiguousarray(m1, np.float64)
        lib().orc_op_set_frames(self.h, _p(h), _p(m1))

    def element_locals(self, x, e0, e1):
        """Element-local results (before scatter) of elements [e0, e1): (e1-e0, nn3, 3)."""
        nx, ny, nz, p = self.dims
        x = np.ascontiguousarray(x, self.dtype)
        out = np.empty((e1 - e0, (p + 1) ** 3, 3), self.dtype)
        st = lib().orc_op_element_locals(self.h, _p(x), _p(out), e0, e1)
        if st:
            raise OracleError(st)
        return out

    def diagonal(self):
        d = np.empty(self.n, self.dtype)
        nb = C.c_int64()
        st = lib().orc_op_diagonal(self.h, _p(d), C.byref(nb))
        if st:
            raise OracleError(st)
        return d, nb.value

    def estimate_eigenvalues(self, diag, iterations=20, seed=0x9E3779B97F4A7C15):
        diag = np.ascontiguousarray(diag, self.dtype)
        lo, hi = C.c_double(), C.c_double()
        st = lib().orc_op_estimate_eigenvalues(self.h, _p(diag), iterations, seed, C.byref(lo), C.byref(hi))
        if st:
            raise OracleError(st)
        return lo.value, hi.value

    def chebyshev(self, diag, lmax_est, b, x, degree=6, range_factor=15.0, safety=1.2, zero_start=True):
        diag = np.ascontiguousarray(diag, self.dtype)
        b = np.ascontiguousarray(b, self.dtype)
        x = np.array(x, self.dtype, copy=True)
        st = lib().orc_op_chebyshev(self.h, _p(diag), lmax_est, degree, range_factor, safety, _p(b), _p(x),
                                    int(zero_start))
        if st:
            raise OracleError(st)
        return x


def transfer(fine_dims, coarse_dims, kind, vec, precision=64):
    """fine_dims/coarse_dims = (nx, ny, nz, p)."""
    k = {"prolongate": 0, "restrict": 1, "interpolate_down": 2}[kind]
    dt = np.float64 if precision == 64 else np.float32
    vec = np.ascontiguousarray(vec, dt)
    d = fine_dims if k == 0 else coarse_dims
    out = np.empty(3 * (d[0] * d[3] + 1) * (d[1] * d[3] + 1) * (d[2] * d[3] + 1), dt)
    lib().orc_transfer(*fine_dims, *coarse_dims, k, precision, _p(vec), _p(out))
    return out


class OracleMg:
    """C restatement of MgHierarchy<float> (emf_oracle.c), cube levels."""

    def __init__(self, n0, lmax, p, model="inh", params=None, strategy="none", degree=6, range_factor=15.0,
                 safety=1.2, eig_iterations=20, deform_amp=0.0, faces=1):
        L = lib()
        L.orc_mg_create.restype = C.c_void_p
        L.orc_mg_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.c_int, C.c_double, C.c_double, C.c_int]
        L.orc_mg_destroy.argtypes = [C.c_void_p]
        L.orc_mg_n_levels.argtypes = [C.c_void_p]
        L.orc_mg_update.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_mg_precondition.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_pcg_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                    C.POINTER(C.c_int), C.c_void_p]
        from oracle.refbind import material_params
        self.params = material_params() if params is None else np.asarray(params, np.float64)
        self.h = L.orc_mg_create(n0, lmax, p, deform_amp, faces, MODELS[model], _p(self.params),
                                 STRATEGIES[strategy], degree, range_factor, safety, eig_iterations)
        self.n_levels = L.orc_mg_n_levels(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mg_destroy(self.h)

    def update_linearization(self, u):
        u = np.ascontiguousarray(u, np.float64)
        st = lib().orc_mg_update(self.h, _p(u))
        if st:
            raise OracleError(st)

    def precondition(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        st = lib().orc_mg_precondition(self.h, _p(r), _p(z))
        if st:
            raise OracleError(st)
        return z


def pcg_solve(op: OracleOperator, mg, b, rtol=1e-8, maxit=200):
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty_like(b)
    it = C.c_int()
    hist = np.zeros(maxit + 1)
    st = lib().orc_pcg_solve(op.h, mg.h if mg is not None else None, _p(b), _p(x), rtol, maxit, C.byref(it),
                             _p(hist))
    if st:
        raise OracleError(st)
    return x, it.value, hist[:it.value + 1]
