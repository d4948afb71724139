"""Python binding of libemfgpu.so (include/emfgpu.h) with the reference's
operator vocabulary (proj/include/elastmf/operator.hpp:49-204, mesh.hpp,
solver.hpp).  This is the host mirror used by tests and bench.py; C++ callers
use include/emfgpu/operator.hpp instead.  Device memory is anything exposing
``data_ptr()`` (torch tensors) or a raw integer address.

There is no CPU fallback: if the CUDA library or a device is missing, every
constructor raises :class:`EmfGpuError`.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMFGPU_LIB") or os.path.join(HERE, "lib", "libemfgpu.so")

MODELS = {"cnh": 0, "inh": 1, "fiber": 2}
STRATEGIES = {"none": 0, "scalar": 1, "tensor": 2, "cachedF": 3}
MAPS = {"reference": 0, "shear_x": 1, "coords": 2, "tube": 3}
NO_CARTESIAN, NO_AFFINE, PERIODIC_Y = 1, 2, 4
FRAMES = {"global": 0, "cylindrical": 1, "replicated": 2}
STATUS = {0: "OK", 1: "ERR_CONFIG", 2: "ERR_NUMERICAL", 3: "ERR_IO", 4: "ERR_INVALID", 5: "ERR_STALE",
          6: "ERR_CUDA"}


class EmfGpuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"emfgpu {STATUS.get(code, code)}: {msg}")
        self.code = code


class NonPositiveJacobian(EmfGpuError):
    """det F <= 0 at (element, qpoint) (errors.hpp:31-38)."""

    def __init__(self, code, msg, element, qpoint):
        super().__init__(code, msg)
        self.element = element
        self.qpoint = qpoint


class StaleCache(EmfGpuError):
    pass


class LevelDesc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("p", C.c_int),
                ("extent", C.c_double * 3), ("map", C.c_int), ("map_param", C.c_double * 4),
                ("coords", C.c_void_p), ("dirichlet_faces", C.c_int), ("device", C.c_int),
                ("z_offset", C.c_int), ("flags", C.c_int)]


class Material(C.Structure):
    _fields_ = [("mu", C.c_double), ("lambda_", C.c_double), ("kappa_b", C.c_double), ("k1", C.c_double),
                ("k2", C.c_double), ("a", C.c_double), ("b", C.c_double), ("phi", C.c_double),
                ("e1", C.c_double * 3), ("e2", C.c_double * 3), ("e3", C.c_double * 3)]


@dataclass
class MaterialParams:
    """MaterialParams (material.hpp:36-50). Defaults are the BASELINE configs'
    (cNH mu=1, lambda=10; kappa_b for iNH/fiber; fibre k1=2, k2=5, +-40 deg)."""
    mu: float = 1.0
    lam: float = 10.0
    kappa_b: float = 1000.0
    k1: float = 2.0
    k2: float = 5.0
    a: float = 3.62
    b: float = 34.3
    phi: float = float(np.deg2rad(40.0))
    e1: tuple = (1.0, 0.0, 0.0)
    e2: tuple = (0.0, 1.0, 0.0)
    e3: tuple = (0.0, 0.0, 1.0)

    def to_c(self) -> Material:
        m = Material()
        m.mu, m.lambda_, m.kappa_b, m.k1, m.k2, m.a, m.b, m.phi = (
            self.mu, self.lam, self.kappa_b, self.k1, self.k2, self.a, self.b, self.phi)
        m.e1[:] = self.e1
        m.e2[:] = self.e2
        m.e3[:] = self.e3
        return m

    def as_array(self) -> np.ndarray:
        """The 17-double layout used by oracle/ (mu, lambda, kappa, k1, k2, a, b, phi, e1, e2, e3)."""
        return np.array([self.mu, self.lam, self.kappa_b, self.k1, self.k2, self.a, self.b, self.phi,
                         *self.e1, *self.e2, *self.e3], dtype=np.float64)


_lib = None


class NewtonConfig(C.Structure):
    """NewtonConfig + FgmresConfig (solver.hpp:26-37)."""
    _fields_ = [("eps_abs", C.c_double), ("eps_rel", C.c_double), ("max_iter", C.c_int),
                ("lin_abs_tol", C.c_double), ("lin_rel_tol", C.c_double), ("restart", C.c_int),
                ("max_restarts", C.c_int)]


BODY_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)
TRACTION_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)


class Loads(C.Structure):
    """emfgpu_loads (Loads, operator.hpp:23-32)."""
    _fields_ = [("pressure", C.c_double), ("pressure_face", C.c_int), ("body_force", BODY_FN),
                ("body_force_user", C.c_void_p), ("traction", TRACTION_FN), ("traction_user", C.c_void_p),
                ("traction_faces", C.c_int)]


class Formulation(C.Structure):
    """emfgpu_formulation (Formulation, material.hpp:20-23): stability 1 = stable."""
    _fields_ = [("stability", C.c_int), ("domain", C.c_int)]


class KernelConfig(C.Structure):
    """emfgpu_kernel_config (KernelConfig, fastscalar.hpp:29-39), defaults 16, 3, exact, newton."""
    _fields_ = [("ln_series_terms", C.c_int), ("jpow_newton_steps", C.c_int), ("exp_mode", C.c_int),
                ("jpow_mode", C.c_int)]

    @classmethod
    def default(cls):
        return cls(16, 3, 0, 0)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EmfGpuError(6, f"{LIB_PATH} missing — run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, st = C.c_void_p, C.c_int64, C.c_int
        sig = {
            "emfgpu_version": (C.c_char_p, []),
            "emfgpu_global_last_error": (C.c_char_p, []),
            "emfgpu_level_create": (st, [C.POINTER(LevelDesc), C.POINTER(vp)]),
            "emfgpu_level_destroy": (None, [vp]),
            "emfgpu_level_n_dofs": (i64, [vp]),
            "emfgpu_level_n_elements": (i64, [vp]),
            "emfgpu_level_affine": (C.c_int, [vp]),
            "emfgpu_level_cartesian": (C.c_int, [vp]),
            "emfgpu_level_jacobians": (st, [vp, vp]),
            "emfgpu_level_coords": (st, [vp, vp]),
            "emfgpu_level_last_error": (C.c_char_p, [vp]),
            "emfgpu_op_create": (st, [vp, C.c_int, C.POINTER(Material), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
            "emfgpu_op_destroy": (None, [vp]),
            "emfgpu_op_n_dofs": (i64, [vp]),
            "emfgpu_op_precision": (C.c_int, [vp]),
            "emfgpu_op_last_error": (C.c_char_p, [vp]),
            "emfgpu_op_update_linearization_host": (st, [vp, vp, C.POINTER(i64), C.POINTER(C.c_int)]),
            "emfgpu_op_update_linearization": (st, [vp, vp, C.POINTER(i64), C.POINTER(C.c_int), vp]),
            "emfgpu_op_linearized": (C.c_int, [vp]),
            "emfgpu_op_checksum": (C.c_uint64, [vp]),
            "emfgpu_op_apply": (st, [vp, vp, vp, vp]),
            "emfgpu_op_apply_host": (st, [vp, vp, vp]),
            "emfgpu_op_check": (st, [vp, C.POINTER(i64), C.POINTER(C.c_int)]),
            "emfgpu_op_compute_diagonal": (st, [vp, vp, C.POINTER(i64), vp]),
            "emfgpu_op_compute_diagonal_host": (st, [vp, vp, C.POINTER(i64)]),
            "emfgpu_op_ledger": (st, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]),
            "emfgpu_op_apply_elements": (st, [vp, vp, C.c_int, C.c_int, vp]),
            "emfgpu_op_apply_nodes": (st, [vp, vp, vp, C.c_int, C.c_int, vp, vp, vp]),
            "emfgpu_op_local_buffer": (vp, [vp]),
            "emfgpu_op_face_values": (i64, [vp]),
            "emfgpu_op_pack_face": (st, [vp, C.c_int, C.c_int, vp, vp]),
            "emfgpu_transfer_create": (st, [vp, vp, C.POINTER(vp)]),
            "emfgpu_transfer_destroy": (None, [vp]),
            "emfgpu_transfer_apply": (st, [vp, C.c_int, C.c_int, vp, vp, vp]),
            "emfgpu_cheb_create": (st, [vp, vp, C.c_double, C.c_int, C.c_double, C.c_double, C.POINTER(vp)]),
            "emfgpu_cheb_destroy": (None, [vp]),
            "emfgpu_cheb_smooth": (st, [vp, vp, vp, C.c_int, vp]),
            "emfgpu_op_estimate_eigenvalues": (st, [vp, vp, C.c_int, C.c_uint64, C.POINTER(C.c_double),
                                                    C.POINTER(C.c_double)]),
            "emfgpu_dot": (st, [C.c_int, vp, vp, i64, C.POINTER(C.c_double), vp]),
            "emfgpu_bench_fma_peak": (st, [C.c_int, C.c_double, C.POINTER(C.c_double)]),
            "emfgpu_op_set_fibre_frame": (st, [vp, C.c_int]),
            "emfgpu_op_fibre_field": (st, [vp, vp, vp]),
            "emfgpu_op_residual": (st, [vp, vp, vp, vp]),
            "emfgpu_op_residual_host": (st, [vp, vp, vp]),
            "emfgpu_op_set_pressure": (st, [vp, C.c_double, C.c_int]),
            "emfgpu_op_set_loads": (st, [vp, C.POINTER(Loads)]),
            "emfgpu_comm_unique_id": (st, [vp]),
            "emfgpu_comm_create": (st, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
            "emfgpu_comm_wrap": (st, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
            "emfgpu_comm_destroy": (None, [vp]),
            "emfgpu_slab_create": (st, [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]),
            "emfgpu_slab_destroy": (None, [vp]),
            "emfgpu_slab_last_error": (C.c_char_p, [vp]),
            "emfgpu_slab_apply": (st, [vp, vp, vp, vp]),
            "emfgpu_slab_group_apply": (st, [C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
            "emfgpu_slab_dot": (st, [vp, vp, vp, vp, vp]),
            "emfgpu_slab_group_dot": (st, [C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                           C.POINTER(vp)]),
            "emfgpu_op_compute_diagonal_indices": (st, [vp, vp, vp, i64, C.POINTER(i64), vp]),
            "emfgpu_op_create_ex": (st, [vp, C.c_int, C.POINTER(Material), C.POINTER(Formulation), C.c_int,
                                         C.c_int, C.POINTER(KernelConfig), C.POINTER(vp)]),
            "emfgpu_op_set_load_scale": (st, [vp, C.c_double]),
            "emfgpu_fgmres_solve": (st, [vp, vp, vp, vp, C.c_double, C.c_double, C.c_int, C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_double), vp]),
            "emfgpu_newton_default_config": (None, [C.POINTER(NewtonConfig)]),
            "emfgpu_stability_sweep": (st, [vp, C.c_int, C.c_int, C.c_uint64, C.POINTER(Material), vp, vp]),
            "emfgpu_newton_solve": (st, [vp, vp, vp, C.POINTER(NewtonConfig), C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), C.POINTER(C.c_double), vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(t) -> int:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _stream(s):
    """cudaStream_t for a call: an int handle, a torch.cuda.Stream, or None =
    torch's current stream on the current device (0 if torch/CUDA absent)."""
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream or None
        except ImportError:
            pass
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


class FeLevel:
    """FeLevel(HexMesh, degree, DeformMap) + set_dirichlet (mesh.hpp:71-138);
    EXT: nx != ny != nz boxes, per-axis extents, the cfg2 shear map, or any
    node-coordinate array."""

    def __init__(self, nx, ny=None, nz=None, p=2, extent=(1.0, 1.0, 1.0), map="reference",
                 map_param=(0.0,), coords=None, dirichlet_faces=1, device=0, z_offset=0, flags=0, periodic_y=False):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        d = LevelDesc()
        d.nx, d.ny, d.nz, d.p = nx, ny, nz, p
        d.extent[:] = extent
        d.map = MAPS["coords"] if coords is not None else MAPS[map]
        mp = list(map_param) + [0.0] * (4 - len(map_param))
        d.map_param[:] = mp
        self._coords = None if coords is None else np.ascontiguousarray(coords, np.float64)
        d.coords = None if coords is None else self._coords.ctypes.data
        d.dirichlet_faces = dirichlet_faces
        d.device = device
        d.z_offset = z_offset
        d.flags = flags | (PERIODIC_Y if periodic_y else 0)
        h = C.c_void_p()
        st = lib().emfgpu_level_create(C.byref(d), C.byref(h))
        if st:
            raise EmfGpuError(st, lib().emfgpu_global_last_error().decode())
        self.h = h.value
        self.desc = d
        self.nx, self.ny, self.nz, self.p = nx, ny, nz, p
        self.faces = dirichlet_faces
        self.periodic_y = bool(periodic_y)
        self.n_dofs = lib().emfgpu_level_n_dofs(self.h)
        self.n_elements = lib().emfgpu_level_n_elements(self.h)
        self.affine = bool(lib().emfgpu_level_affine(self.h))
        self.cartesian = bool(lib().emfgpu_level_cartesian(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_level_destroy(self.h)
            self.h = None

    def dof_count(self):
        return self.n_dofs

    def jacobians(self) -> np.ndarray:
        out = np.empty(self.n_elements * (self.p + 1) ** 3 * 9)
        _check(lib().emfgpu_level_jacobians(self.h, out.ctypes.data))
        return out

    def node_coords(self) -> np.ndarray:
        out = np.empty(self.n_dofs)
        _check(lib().emfgpu_level_coords(self.h, out.ctypes.data))
        return out


def _check(st, msg=""):
    if st:
        raise EmfGpuError(st, msg or lib().emfgpu_global_last_error().decode())


@dataclass
class ByteLedger:
    storage_per_qp: int
    traffic_per_qp: int
    traffic_per_dof: float


class ElasticOperator:
    """ElasticOperator<Number> (operator.hpp:49-204) on one B200.

    precision=64 -> Number=double, 32 -> float.  Host methods take/return
    numpy arrays (parity path: PCIe copies inside); ``*_device`` methods take
    device tensors and a stream and do not synchronise."""

    def __init__(self, level: FeLevel, model="cnh", params: MaterialParams | None = None, strategy="none",
                 precision=64, domain=0, stability="stable", kernel_config: KernelConfig | None = None):
        self.level = level
        self.params = params or MaterialParams()
        if isinstance(domain, str):
            domain = {"material": 0, "spatial": 1}[domain]
        self.model, self.strategy, self.precision, self.domain = model, strategy, precision, domain
        self.dtype = np.float64 if precision == 64 else np.float32
        self._mat = self.params.to_c()
        self._loads_keep = None
        h = C.c_void_p()
        form = Formulation({"standard": 0, "stable": 1}[stability], domain)
        kc = kernel_config or KernelConfig.default()
        st = lib().emfgpu_op_create_ex(level.h, MODELS[model], C.byref(self._mat), C.byref(form),
                                       STRATEGIES[strategy], precision, C.byref(kc), C.byref(h))
        if st:
            raise EmfGpuError(st, lib().emfgpu_global_last_error().decode())
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_op_destroy(self.h)
            self.h = None

    def _ok(self, st):
        if st:
            self._raise(st)

    def _raise(self, st, e=None, q=None):
        msg = lib().emfgpu_op_last_error(self.h).decode()
        if st == 2 and e is not None and e.value >= 0 and "det(F)" in msg:
            raise NonPositiveJacobian(st, msg, e.value, q.value)
        if st == 5:
            raise StaleCache(st, msg)
        raise EmfGpuError(st, msg)

    def n_dofs(self):
        return lib().emfgpu_op_n_dofs(self.h)

    def linearized(self):
        return bool(lib().emfgpu_op_linearized(self.h))

    def checksum(self):
        return lib().emfgpu_op_checksum(self.h)

    def update_linearization(self, u_k):
        u = np.ascontiguousarray(u_k, np.float64)
        e, q = C.c_int64(-1), C.c_int(-1)
        st = lib().emfgpu_op_update_linearization_host(self.h, u.ctypes.data, C.byref(e), C.byref(q))
        if st:
            self._raise(st, e, q)

    def update_linearization_device(self, d_u_k, stream=None):
        e, q = C.c_int64(-1), C.c_int(-1)
        st = lib().emfgpu_op_update_linearization(self.h, _ptr(d_u_k), C.byref(e), C.byref(q), _stream(stream))
        if st:
            self._raise(st, e, q)

    def apply_tangent(self, du) -> np.ndarray:
        x = np.ascontiguousarray(du, self.dtype)
        y = np.empty_like(x)
        st = lib().emfgpu_op_apply_host(self.h, x.ctypes.data, y.ctypes.data)
        if st:
            self._raise(st, C.c_int64(-1), C.c_int(-1))
        return y

    def apply_tangent_device(self, d_x, d_y, stream=None):
        st = lib().emfgpu_op_apply(self.h, _ptr(d_x), _ptr(d_y), _stream(stream))
        if st:
            self._raise(st)

    def check(self):
        e, q = C.c_int64(-1), C.c_int(-1)
        st = lib().emfgpu_op_check(self.h, C.byref(e), C.byref(q))
        if st:
            self._raise(st, e, q)

    def compute_diagonal(self):
        """Returns (diag, n_nonpositive) (operator.hpp:106-107 returns the index list)."""
        d = np.empty(self.n_dofs(), self.dtype)
        nb = C.c_int64(0)
        st = lib().emfgpu_op_compute_diagonal_host(self.h, d.ctypes.data, C.byref(nb))
        if st:
            self._raise(st)
        return d, nb.value

    def compute_diagonal_indices(self, d_diag, capacity=1 << 16, stream=None):
        """compute_diagonal's pair (operator.hpp:106-107, 869-877) on a device
        diagonal: returns the ascending DoF indices of the free rows with
        diag <= 0 (at most `capacity`) and their total count."""
        idx = np.empty(capacity, np.int64)
        nb = C.c_int64(0)
        self._ok(lib().emfgpu_op_compute_diagonal_indices(self.h, _ptr(d_diag), idx.ctypes.data, capacity,
                                                          C.byref(nb), _stream(stream)))
        return idx[:min(nb.value, capacity)].copy(), nb.value

    def compute_diagonal_device(self, d_diag, stream=None):
        nb = C.c_int64(0)
        st = lib().emfgpu_op_compute_diagonal(self.h, _ptr(d_diag), C.byref(nb), _stream(stream))
        if st:
            self._raise(st)
        return nb.value

    def byte_ledger(self) -> ByteLedger:
        s, t, d = C.c_int(), C.c_int(), C.c_double()
        _check(lib().emfgpu_op_ledger(self.h, C.byref(s), C.byref(t), C.byref(d)))
        return ByteLedger(s.value, t.value, d.value)

    # split apply for z slabs
    def apply_elements(self, d_x, k0, k1, stream=None):
        st = lib().emfgpu_op_apply_elements(self.h, _ptr(d_x), k0, k1, _stream(stream))
        if st:
            self._raise(st)

    def apply_nodes(self, d_x, d_y, c0, c1, ghost_lo=None, ghost_hi=None, stream=None):
        st = lib().emfgpu_op_apply_nodes(self.h, _ptr(d_x), _ptr(d_y), c0, c1, _ptr(ghost_lo), _ptr(ghost_hi),
                                         _stream(stream))
        if st:
            self._raise(st)

    def face_values(self):
        return lib().emfgpu_op_face_values(self.h)

    def pack_face(self, k, side, d_face, stream=None):
        st = lib().emfgpu_op_pack_face(self.h, k, side, _ptr(d_face), _stream(stream))
        if st:
            self._raise(st)

    def set_fibre_frame(self, kind="cylindrical"):
        """Per-qp fibre frames (fibre model): "global", "cylindrical" (about z) or "replicated"."""
        st = lib().emfgpu_op_set_fibre_frame(self.h, FRAMES[kind] if isinstance(kind, str) else int(kind))
        if st:
            self._raise(st)

    def fibre_field(self):
        """(H [12, nqp], M1 [6, nqp]) of the per-qp frame field (SoA)."""
        nqp = self.level.n_elements * (self.level.p + 1) ** 3
        h = np.empty(12 * nqp)
        m = np.empty(6 * nqp)
        _check(lib().emfgpu_op_fibre_field(self.h, h.ctypes.data, m.ctypes.data))
        return h, m

    def set_pressure(self, pressure, face=1):
        """Loads{pressure, pressure_face} (operator.hpp:23-32): -p N traction on `face`."""
        self._ok(lib().emfgpu_op_set_pressure(self.h, float(pressure), int(face)))

    def set_loads(self, pressure=0.0, pressure_face=1, body_force=None, traction=None, traction_faces=()):
        """The full Loads struct (operator.hpp:23-32): body_force(X) -> 3 values,
        traction(X, N) -> 3 values on the faces listed in traction_faces (0..5).
        The callbacks run on the host while the load vector is built."""
        def bf(x, out, _u):
            v = body_force((x[0], x[1], x[2]))
            out[0], out[1], out[2] = v
        def tf(x, n, out, _u):
            v = traction((x[0], x[1], x[2]), (n[0], n[1], n[2]))
            out[0], out[1], out[2] = v
        mask = 0
        for f in traction_faces:
            mask |= 1 << int(f)
        ld = Loads(float(pressure), int(pressure_face), BODY_FN(bf) if body_force else BODY_FN(),
                   None, TRACTION_FN(tf) if traction else TRACTION_FN(), None, mask)
        self._ok(lib().emfgpu_op_set_loads(self.h, C.byref(ld)))

    def set_load_scale(self, scale):
        self._ok(lib().emfgpu_op_set_load_scale(self.h, float(scale)))

    def evaluate_residual(self, u) -> np.ndarray:
        """evaluate_residual (operator.hpp:94-95): r = (Grad v, F S) - s*load, host fp64/fp32."""
        u = np.ascontiguousarray(u, dtype=self.dtype)
        r = np.empty_like(u)
        self._ok(lib().emfgpu_op_residual_host(self.h, u.ctypes.data, r.ctypes.data))
        return r

    def evaluate_residual_device(self, d_u, d_r, stream=None):
        self._ok(lib().emfgpu_op_residual(self.h, _ptr(d_u), _ptr(d_r), _stream(stream)))

    def estimate_eigenvalues(self, d_diag, iterations=20, seed=0x9E3779B97F4A7C15):
        lo, hi = C.c_double(), C.c_double()
        st = lib().emfgpu_op_estimate_eigenvalues(self.h, _ptr(d_diag), iterations, seed, C.byref(lo), C.byref(hi))
        if st:
            self._raise(st)
        return lo.value, hi.value


class TransferOp:
    """TransferOp(fine, coarse) (mesh.hpp:157-182) on device vectors."""

    def __init__(self, fine: FeLevel, coarse: FeLevel):
        h = C.c_void_p()
        _check(lib().emfgpu_transfer_create(fine.h, coarse.h, C.byref(h)))
        self.h = h.value
        self.fine, self.coarse = fine, coarse

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_transfer_destroy(self.h)
            self.h = None

    def _run(self, kind, precision, d_in, d_out, stream):
        _check(lib().emfgpu_transfer_apply(self.h, kind, precision, _ptr(d_in), _ptr(d_out), _stream(stream)))

    def prolongate(self, d_coarse, d_fine, precision=64, stream=None):
        self._run(0, precision, d_coarse, d_fine, stream)

    def restrict_(self, d_fine, d_coarse, precision=64, stream=None):
        self._run(1, precision, d_fine, d_coarse, stream)

    def interpolate_down(self, d_fine, d_coarse, precision=64, stream=None):
        self._run(2, precision, d_fine, d_coarse, stream)


class ChebyshevSmoother:
    """ChebyshevSmoother<Number> (solver.hpp:312-362): setup at construction."""

    def __init__(self, op: ElasticOperator, d_diag, lmax_est, degree=6, range_factor=15.0, safety=1.2):
        h = C.c_void_p()
        st = lib().emfgpu_cheb_create(op.h, _ptr(d_diag), lmax_est, degree, range_factor, safety, C.byref(h))
        if st:
            op._raise(st)
        self.h = h.value
        self.op = op

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_cheb_destroy(self.h)
            self.h = None

    def smooth(self, d_x, d_b, zero_start=True, stream=None):
        st = lib().emfgpu_cheb_smooth(self.h, _ptr(d_x), _ptr(d_b), int(zero_start), _stream(stream))
        if st:
            self.op._raise(st)


def dot(d_a, d_b, n, precision=64, stream=None) -> float:
    out = C.c_double()
    _check(lib().emfgpu_dot(precision, _ptr(d_a), _ptr(d_b), n, C.byref(out), _stream(stream)))
    return out.value


def fma_peak_tflops(precision=64, seconds=0.5) -> float:
    out = C.c_double()
    _check(lib().emfgpu_bench_fma_peak(precision, seconds, C.byref(out)))
    return out.value


class MgConfig(C.Structure):
    _fields_ = [("degree", C.c_int), ("range_factor", C.c_double), ("safety", C.c_double),
                ("eig_iterations", C.c_int), ("seed", C.c_uint64), ("coarse_rtol", C.c_double),
                ("coarse_maxit", C.c_int), ("coarse_n", C.c_int), ("precision", C.c_int),
                ("coarse_direct_limit", C.c_int64)]


class MgHierarchy:
    """MgHierarchy<Prec> (solver.hpp:437-581) on the device: Chebyshev-Jacobi
    smoothed V-cycle over the p/h ladder of `fine`, fp32 levels by default."""

    def __init__(self, fine: FeLevel, model="inh", params: MaterialParams | None = None, strategy="none",
                 degree=6, range_factor=15.0, safety=1.2, eig_iterations=20, coarse_rtol=1e-4, coarse_maxit=500,
                 coarse_n=1, precision=32, seed=0x9E3779B97F4A7C15, coarse_direct_limit=2000):
        L = lib()
        for name, (res, args) in {
            "emfgpu_mg_default_config": (None, [C.POINTER(MgConfig)]),
            "emfgpu_mg_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Material), C.c_int, C.POINTER(MgConfig),
                                           C.POINTER(C.c_void_p)]),
            "emfgpu_mg_destroy": (None, [C.c_void_p]),
            "emfgpu_mg_n_levels": (C.c_int, [C.c_void_p]),
            "emfgpu_mg_level_info": (C.c_int, [C.c_void_p, C.c_int] + [C.POINTER(C.c_int)] * 4 +
                                     [C.POINTER(C.c_int64)]),
            "emfgpu_mg_last_error": (C.c_char_p, [C.c_void_p]),
            "emfgpu_mg_update_linearization": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
            "emfgpu_mg_precondition": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "emfgpu_pcg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                           C.POINTER(C.c_int), C.c_void_p, C.c_void_p]),
        }.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        cfg = MgConfig()
        L.emfgpu_mg_default_config(C.byref(cfg))
        cfg.degree, cfg.range_factor, cfg.safety, cfg.eig_iterations = degree, range_factor, safety, eig_iterations
        cfg.seed, cfg.coarse_rtol, cfg.coarse_maxit, cfg.coarse_n, cfg.precision = (seed, coarse_rtol, coarse_maxit,
                                                                                   coarse_n, precision)
        cfg.coarse_direct_limit = coarse_direct_limit
        self.params = params or MaterialParams()
        self._mat = self.params.to_c()
        h = C.c_void_p()
        st = L.emfgpu_mg_create(fine.h, MODELS[model], C.byref(self._mat), STRATEGIES[strategy], C.byref(cfg),
                                C.byref(h))
        if st:
            raise EmfGpuError(st, L.emfgpu_global_last_error().decode())
        self.h = h.value
        self.fine = fine
        self.n_levels = L.emfgpu_mg_n_levels(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_mg_destroy(self.h)
            self.h = None

    def levels(self):
        out = []
        for l in range(self.n_levels):
            v = [C.c_int() for _ in range(4)]
            nd = C.c_int64()
            lib().emfgpu_mg_level_info(self.h, l, *[C.byref(x) for x in v], C.byref(nd))
            out.append((v[0].value, v[1].value, v[2].value, v[3].value, nd.value))
        return out

    def _chk(self, st):
        if st:
            raise EmfGpuError(st, lib().emfgpu_mg_last_error(self.h).decode())

    def update_linearization(self, d_u, stream=None):
        self._chk(lib().emfgpu_mg_update_linearization(self.h, _ptr(d_u), _stream(stream)))

    def precondition(self, d_r, d_z, stream=None):
        self._chk(lib().emfgpu_mg_precondition(self.h, _ptr(d_r), _ptr(d_z), _stream(stream)))


def pcg_solve(op: ElasticOperator, mg: MgHierarchy | None, d_b, d_x, rtol=1e-8, maxit=200, stream=None):
    """Returns (iterations, relative residual history)."""
    it = C.c_int()
    hist = np.zeros(maxit + 1)
    st = lib().emfgpu_pcg_solve(op.h, mg.h if mg is not None else None, _ptr(d_b), _ptr(d_x), rtol, maxit,
                                C.byref(it), hist.ctypes.data, _stream(stream))
    if st:
        op._raise(st)
    return it.value, hist[:it.value + 1]


def fgmres_solve(op: ElasticOperator, mg: MgHierarchy | None, d_b, d_x, abs_tol=1e-12, rel_tol=1e-3, restart=30,
                 max_restarts=40, stream=None):
    """fgmres_solve (solver.hpp:120-203) on the device. Returns (iterations, final residual)."""
    it, res = C.c_int(), C.c_double()
    st = lib().emfgpu_fgmres_solve(op.h, mg.h if mg is not None else None, _ptr(d_b), _ptr(d_x), abs_tol, rel_tol,
                                   restart, max_restarts, C.byref(it), C.byref(res), _stream(stream))
    if st:
        op._raise(st)
    return it.value, res.value


def newton_solve(op: ElasticOperator, mg: MgHierarchy | None, d_u, stream=None, **cfg):
    """newton_solve (solver.hpp:603-656): d_u (fp64, device) in/out with the
    op's loads.  Returns (newton iterations, total FGMRES iterations, |r|)."""
    c = NewtonConfig()
    lib().emfgpu_newton_default_config(C.byref(c))
    for k, v in cfg.items():
        setattr(c, k, v)
    nit, lit, res = C.c_int(), C.c_int(), C.c_double()
    st = lib().emfgpu_newton_solve(op.h, mg.h if mg is not None else None, _ptr(d_u), C.byref(c), C.byref(nit),
                                   C.byref(lit), C.byref(res), _stream(stream))
    if st:
        op._raise(st)
    return nit.value, lit.value, res.value


SWEEP_MODELS = ("cNH", "iNH", "fiber", "svk")
SWEEP_FORMULATIONS = ("standard-material", "stable-material", "standard-spatial", "stable-spatial")
SWEEP_QUANTITIES = ("stress", "tangent")


def stability_sweep(scales, samples_per_scale=1000, seed=42, params: MaterialParams | None = None):
    """run_sweep (stability.hpp / stability.cpp:163-251) on the device.
    Returns (max_rel_error, count_invalid), each (n_scales, 32) in the
    reference's write_csv cell order (model, formulation, quantity)."""
    scales = np.ascontiguousarray(scales, np.float64)
    mat = (params or MaterialParams(mu=62.1, lam=3042.9, kappa_b=3084.3, k1=1.4, k2=22.1, a=3.62, b=34.3,
                                    phi=27.47 * np.pi / 180.0)).to_c()
    err = np.empty(scales.size * 32)
    inv = np.empty(scales.size * 32, np.int64)
    _check(lib().emfgpu_stability_sweep(scales.ctypes.data, scales.size, samples_per_scale, seed, C.byref(mat),
                                        err.ctypes.data, inv.ctypes.data))
    return err.reshape(-1, 32), inv.reshape(-1, 32)


def write_sweep_csv(scales, err, inv, path):
    """write_csv (stability.cpp:253-265) layout."""
    with open(path, "w") as f:
        f.write("scale,model,formulation,quantity,max_rel_error,count_invalid\n")
        for i, s in enumerate(scales):
            c = 0
            for m in SWEEP_MODELS:
                for fm in SWEEP_FORMULATIONS:
                    for q in SWEEP_QUANTITIES:
                        f.write(f"{s:.9e},{m},{fm},{q},{err[i, c]:.9e},{inv[i, c]}\n")
                        c += 1


# ---- z-slab multi-GPU (emfgpu_slab_*) ---------------------------
class Comm:
    """NCCL communicator of the slab layer (emfgpu_comm_*): rank 0 makes the
    unique id, the caller ships the 128 bytes to the other ranks."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(lib().emfgpu_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int, device: int = 0):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().emfgpu_comm_create(buf, world, rank, device, C.byref(h)))
        self.h, self.world, self.rank = h.value, world, rank

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_comm_destroy(self.h)
            self.h = None


class Slab:
    """emfgpu_slab: rank `rank` of `world` z slabs around an ElasticOperator
    whose level holds the slab (z_offset = first element layer)."""

    def __init__(self, op: ElasticOperator, rank: int, world: int, comm: Comm | None = None):
        self.op, self.rank, self.world, self.comm = op, rank, world, comm
        h = C.c_void_p()
        st = lib().emfgpu_slab_create(op.h, rank, world, comm.h if comm else None, C.byref(h))
        if st:
            op._raise(st)
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_slab_destroy(self.h)
            self.h = None

    def _ok(self, st):
        if st:
            raise EmfGpuError(st, lib().emfgpu_slab_last_error(self.h).decode())

    def apply(self, d_x, d_y, stream=None):
        self._ok(lib().emfgpu_slab_apply(self.h, _ptr(d_x), _ptr(d_y), _stream(stream)))

    def dot(self, d_a, d_b, d_out, stream=None):
        """Global dot into the device double d_out (no host sync)."""
        self._ok(lib().emfgpu_slab_dot(self.h, _ptr(d_a), _ptr(d_b), _ptr(d_out), _stream(stream)))


def _arr(vals):
    return (C.c_void_p * len(vals))(*vals)


def slab_group_apply(slabs, xs, ys, streams):
    """One process driving all slabs: peer-copied ghost faces (emfgpu_slab_group_apply)."""
    n = len(slabs)
    st = lib().emfgpu_slab_group_apply(_arr([s.h for s in slabs]), n, _arr([_ptr(x) for x in xs]),
                                       _arr([_ptr(y) for y in ys]), _arr([_stream(t) for t in streams]))
    if st:
        raise EmfGpuError(st, lib().emfgpu_slab_last_error(slabs[0].h).decode())


def slab_group_dot(slabs, a_s, b_s, outs, streams):
    n = len(slabs)
    st = lib().emfgpu_slab_group_dot(_arr([s.h for s in slabs]), n, _arr([_ptr(a) for a in a_s]),
                                     _arr([_ptr(b) for b in b_s]), _arr([_ptr(o) for o in outs]),
                                     _arr([_stream(t) for t in streams]))
    if st:
        raise EmfGpuError(st, lib().emfgpu_slab_last_error(slabs[0].h).decode())


def comm_group(world, devices=None):
    """emfgpu_comm_create_group: `world` communicators for ranks run as host
    threads of this process (rank r's calls from its own thread)."""
    arr = (C.c_void_p * world)()
    dv = (C.c_int * world)(*(devices or [0] * world))
    L = lib()
    L.emfgpu_comm_create_group.restype = C.c_int
    L.emfgpu_comm_create_group.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
    _check(L.emfgpu_comm_create_group(world, dv, arr))
    out = []
    for r in range(world):
        c = Comm.__new__(Comm)
        c.h, c.world, c.rank = arr[r], world, r
        out.append(c)
    return out


class SlabSolver:
    """emfgpu_slab_solver: the cfg4 PCG + hp-multigrid solve with the finest
    level on this rank's z slab and the coarser levels agglomerated (all
    calls collective over the communicator)."""

    def __init__(self, slab: FeLevel, global_level: FeLevel, rank, world, comm: Comm | None, model="inh",
                 params: MaterialParams | None = None, strategy="none", degree=6, coarse_n=1, precision=32,
                 coarse_direct_limit=2000, eig_iterations=20):
        L = lib()
        for name, (res, args) in {
            "emfgpu_slab_solver_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                                    C.POINTER(Material), C.c_int, C.POINTER(MgConfig),
                                                    C.POINTER(C.c_void_p)]),
            "emfgpu_slab_solver_destroy": (None, [C.c_void_p]),
            "emfgpu_slab_solver_last_error": (C.c_char_p, [C.c_void_p]),
            "emfgpu_slab_solver_update_linearization": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
            "emfgpu_slab_solver_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "emfgpu_slab_solver_precondition": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
            "emfgpu_slab_pcg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                                C.POINTER(C.c_int), C.c_void_p, C.c_void_p]),
            "emfgpu_mg_default_config": (None, [C.POINTER(MgConfig)]),
        }.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        cfg = MgConfig()
        L.emfgpu_mg_default_config(C.byref(cfg))
        cfg.degree, cfg.eig_iterations, cfg.coarse_n, cfg.precision = degree, eig_iterations, coarse_n, precision
        cfg.coarse_direct_limit = coarse_direct_limit
        self._cfg = cfg
        self.params = params or MaterialParams()
        self._mat = self.params.to_c()
        self.slab, self.global_level = slab, global_level
        h = C.c_void_p()
        st = L.emfgpu_slab_solver_create(slab.h, C.byref(global_level.desc), rank, world, comm.h if comm else None,
                                         MODELS[model], C.byref(self._mat), STRATEGIES[strategy], C.byref(cfg),
                                         C.byref(h))
        if st:
            raise EmfGpuError(st, L.emfgpu_global_last_error().decode())
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.emfgpu_slab_solver_destroy(self.h)
            self.h = None

    def _ok(self, st):
        if st:
            raise EmfGpuError(st, lib().emfgpu_slab_solver_last_error(self.h).decode())

    def update_linearization(self, d_u, stream=None):
        self._ok(lib().emfgpu_slab_solver_update_linearization(self.h, _ptr(d_u), _stream(stream)))

    def apply(self, d_x, d_y, stream=None):
        self._ok(lib().emfgpu_slab_solver_apply(self.h, _ptr(d_x), _ptr(d_y), _stream(stream)))

    def precondition(self, d_r, d_z, stream=None):
        self._ok(lib().emfgpu_slab_solver_precondition(self.h, _ptr(d_r), _ptr(d_z), _stream(stream)))

    def pcg_solve(self, d_b, d_x, rtol=1e-8, maxit=200, stream=None):
        it = C.c_int()
        hist = np.zeros(maxit + 1)
        self._ok(lib().emfgpu_slab_pcg_solve(self.h, _ptr(d_b), _ptr(d_x), rtol, maxit, C.byref(it), hist.ctypes.data,
                                             _stream(stream)))
        return it.value, hist[:it.value + 1]
