"""CPU, world_size 2 (gloo): the z-slab decomposition of paper_2408_12479_b200/
slab.py — partitioning, ghost-face exchange pattern, colour-parity offsets,
Dirichlet faces per rank, interface ownership in dot products — driven by an
oracle-backed element engine.  The assembled slab result must be BITWISE the
single-process oracle apply (the reference's colour-order scatter)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import orcbind as O
from paper_2408_12479_b200 import inputs as I
from paper_2408_12479_b200.slab import SlabOperator, SlabPartition

NX, NY, NZ, P = 3, 2, 5, 2
FACES = 1 | 16 | 32
PRM = np.array([1.0, 10.0, 50.0, 2.0, 5.0, 3.62, 34.3, 0.7, 1, 0, 0, 0, 1, 0, 0, 0, 1])


class OracleSlabEngine:
    """Element engine for SlabOperator on CPU tensors: element-local results
    from the oracle, node phase = the reference's colour loop
    (operator.hpp:436-466) over own + ghost element layers."""

    def __init__(self, part: SlabPartition, coords, u_local, model="inh"):
        self.part = part
        self.p = part.p
        self.op = O.OracleOperator(part.nx, part.ny, part.nz_local, part.p, coords, part.local_faces, model, PRM)
        self.op.update_linearization(u_local)
        self.mask = self.op.mask().astype(bool)
        self.n3 = (part.p + 1) ** 3
        self.loc = np.zeros((part.nel_local, self.n3, 3))

    def face_values(self):
        return self.part.nx * self.part.ny * (self.p + 1) ** 2 * 3

    def apply_elements(self, x, k0, k1, stream=None):
        per = self.part.nx * self.part.ny
        self.loc[k0 * per:k1 * per] = self.op.element_locals(x.numpy(), k0 * per, k1 * per)

    def _face(self, k, side):
        n = self.p + 1
        per = self.part.nx * self.part.ny
        blk = self.loc[k * per:(k + 1) * per].reshape(per, n, n, n, 3)  # (e, c, b, a, comp)
        return blk[:, self.p if side else 0].reshape(-1)

    def pack_face(self, k, side, buf, stream=None):
        buf.copy_(torch.from_numpy(self._face(k, side)))

    def apply_nodes(self, x, y, c0, c1, ghost_lo=None, ghost_hi=None, stream=None):
        part, p, n = self.part, self.p, self.p + 1
        mx, my = part.mx, part.my
        out = np.zeros((part.mz_local, my, mx, 3))
        layers = [(k, self.loc[k * part.nx * part.ny:(k + 1) * part.nx * part.ny].reshape(part.ny, part.nx, n, n, n, 3))
                  for k in range(part.nz_local)]
        if ghost_lo is not None:
            layers.append((-1, np.zeros((part.ny, part.nx, n, n, n, 3))))
            layers[-1][1][:, :, p] = ghost_lo.numpy().reshape(part.ny, part.nx, n, n, 3)
        if ghost_hi is not None:
            layers.append((part.nz_local, np.zeros((part.ny, part.nx, n, n, n, 3))))
            layers[-1][1][:, :, 0] = ghost_hi.numpy().reshape(part.ny, part.nx, n, n, 3)
        for color in range(8):
            ci, cj, ck = color & 1, (color >> 1) & 1, (color >> 2) & 1
            for k, blk in layers:
                if (k + part.k0) & 1 != ck:
                    continue
                for j in range(cj, part.ny, 2):
                    for i in range(ci, part.nx, 2):
                        zs = slice(k * p, k * p + n) if k >= 0 else slice(0, 1)
                        src = blk[j, i]
                        if k < 0:
                            src = src[p:p + 1]
                        elif k == part.nz_local:
                            zs, src = slice(part.mz_local - 1, part.mz_local), src[0:1]
                        out[zs, j * p:j * p + n, i * p:i * p + n] += src
        yy = out.reshape(-1)
        yy[self.mask] = x.numpy()[self.mask]
        y.copy_(torch.from_numpy(yy))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = SlabPartition(NX, NY, NZ, P, world, rank, faces=FACES)
        u_g = I.make_u0(NX, NY, NZ, P, amp=0.05, faces=FACES)
        v_g = I.make_v(u_g.size, 3)
        eng = OracleSlabEngine(part, part.local_coords(), u_g[part.dof_slice])
        sop = SlabOperator(eng, part, torch.float64, device="cpu", dist=dist)
        x = torch.tensor(v_g[part.dof_slice])
        y = torch.empty_like(x)
        sop.apply(x, y)
        d = sop.dot(x, x)
        q.put((rank, part.k0, part.k1, y.numpy(), d))
    finally:
        dist.destroy_process_group()


def test_two_rank_slabs_bitwise_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p_ in procs:
        p_.join(60)
        assert p_.exitcode == 0
    # single-process oracle
    u_g = I.make_u0(NX, NY, NZ, P, amp=0.05, faces=FACES)
    v_g = I.make_v(u_g.size, 3)
    X, Y, Z = I.lattice_positions(NX, NY, NZ, P)
    op = O.OracleOperator(NX, NY, NZ, P, np.stack([X, Y, Z], 1).ravel(), FACES, "inh", PRM)
    op.update_linearization(u_g)
    y_ref = op.apply(v_g)
    plane = 3 * (NX * P + 1) * (NY * P + 1)
    (_, k0a, k1a, ya, da), (_, k0b, k1b, yb, db) = res
    assert (k0a, k1a, k0b, k1b) == (0, 3, 3, 5)  # uneven split, odd interface layer
    assert np.array_equal(ya[-plane:], yb[:plane])  # duplicated interface plane agrees bitwise
    y_cat = np.concatenate([ya, yb[plane:]])
    assert np.array_equal(y_cat, y_ref)
    assert da == db and np.isclose(da, float(v_g @ v_g), rtol=1e-13)


def test_partition_bookkeeping():
    parts = [SlabPartition(4, 4, 10, 3, 4, r, faces=1 | 16 | 32) for r in range(4)]
    assert [(q.k0, q.k1) for q in parts] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert parts[0].local_faces == 1 | 16 and parts[3].local_faces == 1 | 32 and parts[1].local_faces == 1
    assert sum(q.nel_local for q in parts) == 4 * 4 * 10
    assert parts[2].dof_slice.start == 3 * 13 * 13 * 18
    with pytest.raises(ValueError):
        SlabPartition(2, 2, 3, 2, 4, 0)
