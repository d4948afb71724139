"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libemfref.so, the
unmodified reference (proj/) compiled from its own sources (oracle/Makefile).
Wraps oracle/ref_driver.cpp; see there for the reference interfaces driven.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libemfref.so")

MODELS = {"cnh": 0, "inh": 1, "fiber": 2}
STRATEGIES = {"none": 0, "scalar": 1, "tensor": 2}
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        vp, dp, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_int64
        L.ref_last_error.restype = C.c_char_p
        L.ref_level_create.restype = vp
        L.ref_level_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, vp]
        L.ref_level_destroy.argtypes = [vp]
        L.ref_level_ndofs.restype = i64
        L.ref_level_ndofs.argtypes = [vp]
        for f in ("ref_level_coords", "ref_level_jacobians", "ref_level_mask"):
            getattr(L, f).argtypes = [vp, vp]
        L.ref_level_basis.argtypes = [vp] + [vp] * 5
        L.ref_op_create.restype = vp
        L.ref_op_create.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int]
        L.ref_op_destroy.argtypes = [vp]
        L.ref_op_set_threads.argtypes = [vp, C.c_int]
        L.ref_op_linearize.argtypes = [vp, vp]
        L.ref_op_apply.argtypes = [vp, vp, vp]
        L.ref_op_apply_repeat.argtypes = [vp, vp, vp, C.c_int]
        L.ref_op_residual.argtypes = [vp, vp, vp]
        L.ref_op_diagonal.argtypes = [vp, vp, C.POINTER(i64), vp, i64]
        L.ref_ledger.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_transfer.argtypes = [vp, vp, C.c_int, C.c_int, vp, vp]
        L.ref_estimate_eigenvalues.argtypes = [vp, vp, C.c_int, C.c_uint64, dp, dp]
        L.ref_chebyshev.argtypes = [vp, vp, C.c_double, C.c_int, C.c_double, C.c_double, vp, vp, C.c_int]
        L.ref_structure_tensors.argtypes = [vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


def _check(st):
    if st != 0:
        raise RefError(st, lib().ref_last_error().decode())


def material_params(mu=1.0, lam=10.0, kappa=1000.0, k1=2.0, k2=5.0, a=3.62, b=34.3,
                    phi=np.deg2rad(40.0), e1=(1, 0, 0), e2=(0, 1, 0), e3=(0, 0, 1)):
    return np.array([mu, lam, kappa, k1, k2, a, b, phi, *e1, *e2, *e3], dtype=np.float64)


class RefLevel:
    def __init__(self, n0, level, p, deform_amp=0.0, faces=1, coords=None):
        c = None if coords is None else np.ascontiguousarray(coords, np.float64)
        self.h = lib().ref_level_create(n0, level, p, deform_amp, faces, None if c is None else _p(c))
        if not self.h:
            raise RefError(1, lib().ref_last_error().decode())
        self.n = n0 << level
        self.p = p
        self.ndofs = lib().ref_level_ndofs(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_level_destroy(self.h)

    def coords(self):
        out = np.empty(self.ndofs)
        lib().ref_level_coords(self.h, _p(out))
        return out

    def jacobians(self):
        out = np.empty(self.n ** 3 * (self.p + 1) ** 3 * 9)
        lib().ref_level_jacobians(self.h, _p(out))
        return out

    def mask(self):
        out = np.empty(self.ndofs, np.uint8)
        lib().ref_level_mask(self.h, _p(out))
        return out


class RefOperator:
    def __init__(self, level: RefLevel, model="cnh", params=None, strategy="none",
                 precision=64, domain=0, threads=None):
        self.level = level
        self.params = material_params() if params is None else np.asarray(params, np.float64)
        self.precision = precision
        self.dtype = np.float64 if precision == 64 else np.float32
        self.h = lib().ref_op_create(level.h, MODELS[model], _p(self.params), domain,
                                     STRATEGIES[strategy], precision)
        if not self.h:
            raise RefError(1, lib().ref_last_error().decode())
        self.n = level.ndofs
        lib().ref_op_set_threads(self.h, threads or os.cpu_count() or 1)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_op_destroy(self.h)

    def set_threads(self, t):
        lib().ref_op_set_threads(self.h, t)

    def update_linearization(self, u):
        u = np.ascontiguousarray(u, np.float64)
        _check(lib().ref_op_linearize(self.h, _p(u)))

    def apply(self, x, reps=1):
        x = np.ascontiguousarray(x, self.dtype)
        y = np.empty(self.n, self.dtype)
        if reps == 1:
            _check(lib().ref_op_apply(self.h, _p(x), _p(y)))
        else:
            _check(lib().ref_op_apply_repeat(self.h, _p(x), _p(y), reps))
        return y

    def residual(self, u):
        u = np.ascontiguousarray(u, self.dtype)
        r = np.empty(self.n, self.dtype)
        _check(lib().ref_op_residual(self.h, _p(u), _p(r)))
        return r

    def diagonal(self, cap=1024):
        d = np.empty(self.n, self.dtype)
        nb = C.c_int64(0)
        bad = np.empty(cap, np.int64)
        _check(lib().ref_op_diagonal(self.h, _p(d), C.byref(nb), _p(bad), cap))
        return d, bad[: min(cap, nb.value)], nb.value

    def estimate_eigenvalues(self, diag, iterations=20, seed=0x9E3779B97F4A7C15):
        diag = np.ascontiguousarray(diag, self.dtype)
        lo, hi = C.c_double(), C.c_double()
        _check(lib().ref_estimate_eigenvalues(self.h, _p(diag), iterations, seed, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def chebyshev(self, diag, lmax_est, b, x, degree=6, range_factor=15.0, safety=1.2, zero_start=True):
        diag = np.ascontiguousarray(diag, self.dtype)
        b = np.ascontiguousarray(b, self.dtype)
        x = np.array(x, self.dtype, copy=True)
        _check(lib().ref_chebyshev(self.h, _p(diag), lmax_est, degree, range_factor, safety,
                                   _p(b), _p(x), int(zero_start)))
        return x


def transfer(fine: RefLevel, coarse: RefLevel, kind: str, vec, precision=64):
    k = {"prolongate": 0, "restrict": 1, "interpolate_down": 2}[kind]
    dt = np.float64 if precision == 64 else np.float32
    vec = np.ascontiguousarray(vec, dt)
    out = np.empty(fine.ndofs if k == 0 else coarse.ndofs, dt)
    _check(lib().ref_transfer(fine.h, coarse.h, k, precision, _p(vec), _p(out)))
    return out


def ledger(model, domain, strategy):
    s, t = C.c_int(), C.c_int()
    _check(lib().ref_ledger(MODELS[model], domain, STRATEGIES[strategy], C.byref(s), C.byref(t)))
    return s.value, t.value


def structure_tensors(params):
    out = np.empty(21)
    _check(lib().ref_structure_tensors(_p(np.asarray(params, np.float64)), _p(out)))
    return out


class RefMg:
    """The reference's MgHierarchy<float> (solver.hpp:437-581) on a cube level."""

    def __init__(self, level: RefLevel, model, params, strategy="none", degree=6, range_factor=15.0, safety=1.2,
                 eig_iterations=20, deform_amp=0.0, faces=1, coarse_direct_limit=0):
        L = lib()
        L.ref_mg_create.restype = C.c_void_p
        L.ref_mg_create.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_int, C.c_double, C.c_int, C.c_int64]
        L.ref_mg_destroy.argtypes = [C.c_void_p]
        L.ref_mg_n_levels.argtypes = [C.c_void_p]
        L.ref_mg_update_linearization.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_mg_precondition.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_pcg_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                    C.POINTER(C.c_int), C.c_void_p]
        self.params = np.asarray(params, np.float64)
        self.level = level
        self.h = L.ref_mg_create(level.h, MODELS[model], _p(self.params), STRATEGIES[strategy], degree, range_factor,
                                 safety, eig_iterations, deform_amp, faces, coarse_direct_limit)
        if not self.h:
            raise RefError(1, L.ref_last_error().decode())
        self.n_levels = L.ref_mg_n_levels(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_mg_destroy(self.h)

    def update_linearization(self, u):
        u = np.ascontiguousarray(u, np.float64)
        _check(lib().ref_mg_update_linearization(self.h, _p(u)))

    def precondition(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        _check(lib().ref_mg_precondition(self.h, _p(r), _p(z)))
        return z


def pcg_solve(op: RefOperator, mg, b, rtol=1e-8, maxit=200):
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty_like(b)
    it = C.c_int()
    hist = np.zeros(maxit + 1)
    _check(lib().ref_pcg_solve(op.h, mg.h if mg is not None else None, _p(b), _p(x), rtol, maxit, C.byref(it),
                               _p(hist)))
    return x, it.value, hist[:it.value + 1]


def residual_with_pressure(level: RefLevel, model, params, pressure, face, u, load_scale=1.0):
    L = lib()
    L.ref_residual_with_pressure.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_double,
                                             C.c_void_p, C.c_void_p]
    params = np.asarray(params, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    r = np.empty_like(u)
    _check(L.ref_residual_with_pressure(level.h, MODELS[model], _p(params), pressure, face, load_scale, _p(u), _p(r)))
    return r


def residual_with_loads(level: RefLevel, model, params, pressure, face, body, traction_faces, u, load_scale=1.0):
    """evaluate_residual with Loads{pressure, body_force, traction} (the fixture
    functions of ref_driver.cpp: ref_residual_with_loads)."""
    L = lib()
    L.ref_residual_with_loads.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                          C.c_double, C.c_void_p, C.c_void_p]
    params = np.asarray(params, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    r = np.empty_like(u)
    _check(L.ref_residual_with_loads(level.h, MODELS[model], _p(params), pressure, face, int(body),
                                     int(traction_faces), load_scale, _p(u), _p(r)))
    return r


def newton_pressure(level: RefLevel, model, params, pressure, face=1, degree=6, deform_amp=0.0, faces=1,
                    coarse_direct_limit=0):
    L = lib()
    L.ref_newton_pressure.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_double,
                                      C.c_int, C.c_int64, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_double)]
    params = np.asarray(params, np.float64)
    u = np.empty(level.ndofs)
    nit, lit, res = C.c_int(), C.c_int(), C.c_double()
    _check(L.ref_newton_pressure(level.h, MODELS[model], _p(params), pressure, face, degree, deform_amp, faces,
                                 coarse_direct_limit, _p(u), C.byref(nit), C.byref(lit), C.byref(res)))
    return u, nit.value, lit.value, res.value


def stability_sweep(scales, samples=1000, seed=42, params=None):
    """run_sweep of the reference (stability.cpp:163-251): (n_scales, 32) max
    relative errors and invalid counts in write_csv order."""
    L = lib()
    L.ref_stability_sweep.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
    scales = np.ascontiguousarray(scales, np.float64)
    params = material_params() if params is None else np.asarray(params, np.float64)
    err = np.empty(scales.size * 32)
    inv = np.empty(scales.size * 32, np.int64)
    _check(L.ref_stability_sweep(_p(scales), scales.size, samples, seed, _p(params), _p(err), _p(inv)))
    return err.reshape(-1, 32), inv.reshape(-1, 32)
