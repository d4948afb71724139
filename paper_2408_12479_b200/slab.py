"""Z-slab domain decomposition of the tangent apply over GPUs (one process per
GPU, torch.distributed over NCCL).  The reference has no distributed path
(SURVEY.md §2.1); this is the B200 design of SURVEY §8(e):

* rank r owns element layers [k0, k1) of the global nx x ny x nz box and the
  node planes [k0 p, k1 p]; the interface plane is duplicated on both ranks;
* per apply: the two boundary element layers are computed first and their
  element-local results restricted to the interface faces are packed; the
  faces go to the neighbours with NCCL send/recv while the interior layers
  are computed (the NCCL stream overlaps the element kernel); the node phase
  then sums every interface node's <= 8 contributions — own and ghost — in
  the reference's global colour order, so every rank's result is bitwise the
  single-GPU result (no data-path collective besides the face exchange).

On GPUs the whole apply runs below the C ABI (emfgpu_slab_apply, csrc/slab.cu:
NCCL send/recv on the slab's communication stream, event-ordered, graph-
capturable; emfgpu_slab_dot for the rank-ordered device dot); this module
only partitions the box, builds the slab's level and creates the NCCL
communicator (unique id broadcast over torch.distributed).  The Python
exchange below drives a duck-typed element engine (apply_elements /
pack_face / apply_nodes / face_values) and serves the CPU gloo tests with an
oracle-backed engine.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SlabPartition:
    nx: int
    ny: int
    nz: int          # global element layers
    p: int
    world: int
    rank: int
    faces: int = 1   # global Dirichlet faces

    def __post_init__(self):
        base, rem = divmod(self.nz, self.world)
        if base == 0:
            raise ValueError("fewer element layers than ranks")
        self.k0 = self.rank * base + min(self.rank, rem)
        self.k1 = self.k0 + base + (1 if self.rank < rem else 0)
        self.nz_local = self.k1 - self.k0
        self.mx, self.my = self.nx * self.p + 1, self.ny * self.p + 1
        self.mz_local = self.nz_local * self.p + 1
        self.c0, self.c1 = self.k0 * self.p, self.k1 * self.p   # global node planes (inclusive)
        plane = 3 * self.mx * self.my
        self.dof_slice = slice(self.c0 * plane, (self.c1 + 1) * plane)
        self.global_dofs = plane * (self.nz * self.p + 1)
        self.nel_local = self.nx * self.ny * self.nz_local
        f = self.faces & 0b001111
        if self.rank == 0:
            f |= self.faces & 16
        if self.rank == self.world - 1:
            f |= self.faces & 32
        self.local_faces = f
        self.lo = self.rank - 1 if self.rank > 0 else None
        self.hi = self.rank + 1 if self.rank < self.world - 1 else None
        # owned node planes (for global reductions: the interface plane is
        # owned by the upper rank)
        self.own_planes = (0 if self.rank == 0 else 1, self.mz_local - 1)

    def local_coords(self, extent=(1.0, 1.0, 1.0)) -> np.ndarray:
        """Lattice coordinates of this slab's nodes, computed from the GLOBAL
        lattice (mesh.cpp:147-151) so they are bitwise those of 1 GPU."""
        from .inputs import lattice_axis
        ax = lattice_axis(self.nx, self.p, extent[0])
        ay = lattice_axis(self.ny, self.p, extent[1])
        az = lattice_axis(self.nz, self.p, extent[2])[self.c0:self.c1 + 1]
        Z, Y, X = np.meshgrid(az, ay, ax, indexing="ij")
        return np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1).ravel()

    def make_level(self, extent=(1.0, 1.0, 1.0), device=0, map="reference", map_param=(0.0,)):
        """This slab's FeLevel.  One rank: the level generator itself (the
        map applied on the device-side generator, bitwise the workloads'
        levels).  Several ranks: the global pre-map lattice restricted to the
        slab's node planes, with the z-independent maps applied here."""
        from .emfgpu import FeLevel
        if self.world == 1:
            return FeLevel(self.nx, self.ny, self.nz, p=self.p, extent=extent, map=map, map_param=map_param,
                           dirichlet_faces=self.local_faces, device=device)
        c = self.local_coords(extent).reshape(-1, 3)
        if map == "shear_x":  # BASELINE cfg2: x' = x + a sin(2 pi y) e_x
            c[:, 0] += map_param[0] * np.sin(2.0 * np.pi * c[:, 1])
        elif map != "reference" or map_param[0] != 0.0:
            raise ValueError(f"slab levels support the shear_x map and the plain lattice, not {map}")
        return FeLevel(self.nx, self.ny, self.nz_local, p=self.p, coords=c.reshape(-1),
                       dirichlet_faces=self.local_faces, device=device, z_offset=self.k0)


class SlabOperator:
    """apply(x, y) of the distributed tangent on local slab vectors."""

    def __init__(self, engine, part: SlabPartition, dtype, device="cuda", dist=None):
        import torch
        self.e = engine
        self.part = part
        self.torch = torch
        if dist is None and part.world > 1:
            import torch.distributed as dist
        self.dist = dist
        # the CUDA operator: the slab apply and dot below the C ABI
        self.native = hasattr(engine, "apply_tangent_device")
        if self.native:
            from .emfgpu import Comm, Slab
            self.comm = None
            if part.world > 1:
                uid = [Comm.unique_id() if part.rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                self.comm = Comm(uid[0], part.world, part.rank, device=torch.cuda.current_device())
            self.slab = Slab(engine, part.rank, part.world, self.comm)
            self.dot_out = torch.zeros(1, dtype=torch.float64, device=device)
            nzl = part.nz_local
            n_el = 1 + (nzl > 1) + (nzl > 2)
            self.launches_per_apply = 2 if part.world == 1 else n_el + (part.lo is not None) + (
                part.hi is not None) + 1
            return
        nf = engine.face_values()
        mk = lambda: torch.empty(nf, dtype=dtype, device=device)  # noqa: E731
        self.send_lo = mk() if part.lo is not None else None
        self.recv_lo = mk() if part.lo is not None else None
        self.send_hi = mk() if part.hi is not None else None
        self.recv_hi = mk() if part.hi is not None else None
        self.launches_per_apply = 2 if part.world == 1 else 0

    def _stream(self):
        t = self.torch
        return t.cuda.current_stream().cuda_stream if t.cuda.is_available() else None

    def apply(self, x, y, ev_mid=None):
        part, e = self.part, self.e
        s = self._stream()
        nzl = part.nz_local
        if self.native:
            if part.world == 1:
                e.apply_tangent_device(x, y, stream=s)  # one call: element + node phase
            else:
                self.slab.apply(x, y, stream=s)
            return
        if part.world == 1:
            if ev_mid is None and hasattr(e, "apply_tangent_device"):
                e.apply_tangent_device(x, y, stream=s)  # one call: element + node phase
                return
            e.apply_elements(x, 0, nzl, stream=s)
            if ev_mid is not None:
                ev_mid.record()
            e.apply_nodes(x, y, 0, part.mz_local - 1, stream=s)
            return
        launches = 0
        # 1) boundary layers, then pack the interface faces
        e.apply_elements(x, 0, 1, stream=s)
        launches += 1
        if nzl > 1:
            e.apply_elements(x, nzl - 1, nzl, stream=s)
            launches += 1
        if part.lo is not None:
            e.pack_face(0, 0, self.send_lo, stream=s)
            launches += 1
        if part.hi is not None:
            e.pack_face(nzl - 1, 1, self.send_hi, stream=s)
            launches += 1
        # 2) face exchange (NCCL stream waits for the packs, then overlaps 3))
        d = self.dist
        ops = []
        if part.lo is not None:
            ops += [d.P2POp(d.isend, self.send_lo, part.lo), d.P2POp(d.irecv, self.recv_lo, part.lo)]
        if part.hi is not None:
            ops += [d.P2POp(d.isend, self.send_hi, part.hi), d.P2POp(d.irecv, self.recv_hi, part.hi)]
        works = d.batch_isend_irecv(ops) if ops else []
        # 3) interior element layers
        if nzl > 2:
            e.apply_elements(x, 1, nzl - 1, stream=s)
            launches += 1
        if ev_mid is not None:
            ev_mid.record()
        for w in works:
            w.wait()
        # 4) node phase with ghost faces, global colour order
        e.apply_nodes(x, y, 0, part.mz_local - 1, ghost_lo=self.recv_lo, ghost_hi=self.recv_hi, stream=s)
        self.launches_per_apply = launches + 1

    def dot_device(self, a, b):
        """Global dot product into a device scalar (emfgpu_slab_dot: owned
        planes, NCCL all-gather of the partials, rank-order sum; no host sync)."""
        self.slab.dot(a, b, self.dot_out, stream=self._stream())
        return self.dot_out

    def dot(self, a, b):
        """Global dot product of two slab vectors, each interface plane counted
        once (owned by the upper rank), fixed rank-order sum (bit-stable)."""
        if self.native:
            return float(self.dot_device(a, b).item())
        t = self.torch
        part = self.part
        plane = 3 * part.mx * part.my
        lo, hi = part.own_planes
        sl = slice(lo * plane, (hi + 1) * plane)
        loc = (a[sl].double() * b[sl].double()).sum().reshape(1)
        if part.world == 1:
            return float(loc.item())
        parts = [t.zeros_like(loc) for _ in range(part.world)]
        self.dist.all_gather(parts, loc)
        s = 0.0
        for q in parts:
            s += float(q.item())
        return s
