"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures from oracle/_ref) and the bit-exact C oracle.
Tolerances (north star): rel-L2 <= 1e-12 in fp64, <= 1e-5 in fp32."""
import os

import numpy as np
import pytest

from paper_2408_12479_b200 import inputs as I

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {64: 1e-12, 32: 1e-5}
SMALL = ["cnh_p1_n4_curved", "cnh_p3_n2_curved", "inh_p2_n4_curved", "inh_p4_n2_affine",
         "fiber_p2_n2_curved", "fiber_p3_n2_affine"]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def G():
    from paper_2408_12479_b200 import emfgpu
    return emfgpu


def params_from(arr, G):
    return G.MaterialParams(mu=arr[0], lam=arr[1], kappa_b=arr[2], k1=arr[3], k2=arr[4], a=arr[5], b=arr[6],
                            phi=arr[7], e1=tuple(arr[8:11]), e2=tuple(arr[11:14]), e3=tuple(arr[14:17]))


@pytest.mark.parametrize("flags", [0, 1, 3])  # Cartesian fast path / affine / per-qp geometry
def test_cfg0_vs_reference(G, flags):
    g = np.load(os.path.join(GOLD, "cfg0.npz"))
    lev = G.FeLevel(8, p=2, dirichlet_faces=1, flags=flags)
    assert lev.affine == (flags & 2 == 0) and lev.cartesian == (flags == 0)
    u0 = I.make_u0(8, 8, 8, 2)
    v = I.make_v(lev.n_dofs)
    for prec in (64, 32):
        op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", prec)
        op.update_linearization(u0)
        y = op.apply_tangent(v)
        assert rel(y, g[f"y{prec}"]) <= TOL[prec]
        assert rel(y, g["y64"]) <= TOL[prec]
        mask = I.dirichlet_mask(8, 8, 8, 2, 1)
        assert np.array_equal(y[mask], v.astype(op.dtype)[mask])  # identity rows, operator.hpp:617-620
        y2 = op.apply_tangent(v)
        assert np.array_equal(y, y2)  # run-to-run bitwise determinism
        d, nb = op.compute_diagonal()
        assert nb == 0 and rel(d, g[f"diag{prec}"]) <= TOL[prec]


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("strategy", ["none", "scalar", "tensor", "cachedF"])
def test_small_vs_reference(G, name, prec, strategy):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    model, pp, nn = name.split("_")[:3]
    p, n = int(pp[1:]), int(nn[1:])
    lev = G.FeLevel(n, p=p, coords=g["coords"], dirichlet_faces=1)
    op = G.ElasticOperator(lev, model, params_from(g["params"], G), strategy, prec)
    op.update_linearization(g["u0"])
    y = op.apply_tangent(g["v"])
    key = f"y{prec}_{strategy if (prec == 32 and strategy != 'cachedF') else 'none'}"
    assert rel(y, g[key]) <= TOL[prec], rel(y, g[key])
    d, nb = op.compute_diagonal()
    assert rel(d, g[f"diag{prec}"]) <= TOL[prec], rel(d, g[f"diag{prec}"])


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("flags", [0, 1, 3])
def test_affine_paths_all_degrees_vs_oracle(G, p, flags):
    """Every degree through the diagonal-affine, general-affine and per-qp
    geometry paths (element groups smaller than the 10 geometry factors)."""
    from oracle import orcbind as O
    n = 3
    lev = G.FeLevel(n, p=p, flags=flags)
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    u0 = I.make_u0(n, n, n, p)
    v = I.make_v(lev.n_dofs, 5)
    orc = O.OracleOperator(n, n, n, p, lev.node_coords(), 1, "inh", prm.as_array(), "none", 64)
    orc.update_linearization(u0)
    yo = orc.apply(v)
    for prec in (64, 32):
        op = G.ElasticOperator(lev, "inh", prm, "none", prec)
        op.update_linearization(u0)
        assert rel(op.apply_tangent(v), yo) <= {64: 1e-12, 32: 1e-5}[prec]


def test_geometry_matches_reference_jacobians(G):
    from oracle import orcbind as O
    g = np.load(os.path.join(GOLD, "inh_p2_n4_curved.npz"))
    lev = G.FeLevel(4, p=2, coords=g["coords"])
    assert not lev.affine
    orc = O.OracleOperator(4, 4, 4, 2, g["coords"], 1, "inh", g["params"])
    assert rel(lev.jacobians(), orc.jacobians()) <= 1e-14


@pytest.mark.parametrize("flags", [0, 1])
def test_cfg1_full_size_known_answers(G, flags):
    """BASELINE configs[1] at full size (32^3 Q3, 2 738 019 DoFs) against the
    reference's known answers and the oracle."""
    lev = G.FeLevel(32, p=3, flags=flags)
    assert lev.cartesian == (flags == 0)
    u0 = I.make_u0(32, 32, 32, 3)
    v = I.make_v(lev.n_dofs)
    assert np.isclose(np.linalg.norm(u0), 28.816069046240159, rtol=1e-13)
    ys = {}
    for prec in (64, 32):
        for strategy in ("none", "cachedF", "scalar", "tensor"):
            op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), strategy, prec)
            op.update_linearization(u0)
            ys[(prec, strategy)] = op.apply_tangent(v)
    y = ys[(64, "none")]
    assert np.isclose(np.linalg.norm(y), 892.45567630658536, rtol=1e-12)
    node = (48 * 97 + 48) * 97 + 48
    assert y[3 * node:3 * node + 3] == pytest.approx(
        [-0.21301797238610545, -0.00067067958362078579, -0.2998014835832995], rel=1e-10, abs=1e-13)
    for (prec, strategy), yy in ys.items():
        assert rel(yy, y) <= TOL[prec], (prec, strategy, rel(yy, y))
    from oracle import orcbind as O
    orc = O.OracleOperator(32, 32, 32, 3, model="cnh", params=np.array(
        [1.0, 10.0, 1000.0, 2.0, 5.0, 3.62, 34.3, 0.7, 1, 0, 0, 0, 1, 0, 0, 0, 1]))
    orc.update_linearization(u0)
    assert rel(y, orc.apply(v)) <= 1e-12


def test_nonpositive_jacobian_first_point_matches_oracle(G):
    from oracle import orcbind as O
    lev = G.FeLevel(2, p=2)
    u = np.zeros(lev.n_dofs)
    u[3 * 40] = -5.0
    orc = O.OracleOperator(2, 2, 2, 2)
    with pytest.raises(O.OracleError) as eo:
        orc.update_linearization(u)
    op = G.ElasticOperator(lev, "cnh")
    with pytest.raises(G.NonPositiveJacobian) as eg:
        op.update_linearization(u)
    assert f"element={eg.value.element} qpoint={eg.value.qpoint}" in str(eo.value)


def test_stale_cache(G):
    op = G.ElasticOperator(G.FeLevel(2, p=2), "cnh")
    with pytest.raises(G.StaleCache):
        op.apply_tangent(np.zeros(op.n_dofs()))


def test_transfers_vs_reference(G):
    import torch
    g = np.load(os.path.join(GOLD, "transfers.npz"))
    dims = {"p42": ((2, 4), (2, 2)), "p21": ((2, 2), (2, 1)), "h21": ((4, 1), (2, 1))}
    for tag, ((nf, pf), (nc, pc)) in dims.items():
        F = G.FeLevel(nf, p=pf, map_param=(0.05,))
        Cl = G.FeLevel(nc, p=pc, map_param=(0.05,))
        t = G.TransferOp(F, Cl)
        for prec, dt in ((64, torch.float64), (32, torch.float32)):
            xc = torch.tensor(g[f"{tag}_xc"], dtype=dt, device="cuda")
            xf = torch.tensor(g[f"{tag}_xf"], dtype=dt, device="cuda")
            of = torch.empty(F.n_dofs, dtype=dt, device="cuda")
            oc = torch.empty(Cl.n_dofs, dtype=dt, device="cuda")
            t.prolongate(xc, of, prec)
            torch.cuda.synchronize()
            assert rel(of.cpu().numpy(), g[f"{tag}_prolongate"]) <= TOL[prec]
            t.restrict_(xf, oc, prec)
            torch.cuda.synchronize()
            assert rel(oc.cpu().numpy(), g[f"{tag}_restrict"]) <= TOL[prec]
            t.interpolate_down(xf, oc, prec)
            torch.cuda.synchronize()
            assert rel(oc.cpu().numpy(), g[f"{tag}_interpolate_down"]) <= TOL[prec]


def test_smoother_and_eigenvalues_vs_reference(G):
    import torch
    g = np.load(os.path.join(GOLD, "smoother.npz"))
    lev = G.FeLevel(4, p=2)
    for prec, dt in ((64, torch.float64), (32, torch.float32)):
        op = G.ElasticOperator(lev, "inh", G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0), "none", prec)
        op.update_linearization(np.zeros(lev.n_dofs))
        d = torch.empty(lev.n_dofs, dtype=dt, device="cuda")
        assert op.compute_diagonal_device(d) == 0
        assert rel(d.cpu().numpy(), g[f"diag{prec}"]) <= TOL[prec]
        lmin, lmax = op.estimate_eigenvalues(d)
        assert abs(lmax - float(g[f"lmax{prec}"])) <= 1e-6 * abs(float(g[f"lmax{prec}"]))
        sm = G.ChebyshevSmoother(op, d, float(g[f"lmax{prec}"]), degree=5)
        b = torch.tensor(g[f"b{prec}"], dtype=dt, device="cuda")
        x = torch.zeros_like(b)
        sm.smooth(x, b, zero_start=True)
        torch.cuda.synchronize()
        assert rel(x.cpu().numpy(), g[f"x1_{prec}"]) <= 10 * TOL[prec]
        sm.smooth(x, b, zero_start=False)
        torch.cuda.synchronize()
        assert rel(x.cpu().numpy(), g[f"x2_{prec}"]) <= 10 * TOL[prec]


def test_split_apply_and_slab_emulation(G):
    """apply == element phase + node phase; and a 2-slab decomposition with
    ghost faces reproduces the single-level result BITWISE (same colour-order
    sums on the interface plane)."""
    import torch
    n, p = 4, 2
    lev = G.FeLevel(n, p=p, dirichlet_faces=1 | 16)
    u0 = I.make_u0(n, n, n, p, faces=1 | 16)
    v = I.make_v(lev.n_dofs)
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
    op.update_linearization(u0)
    y_full = op.apply_tangent(v)
    X, Y, Z = I.lattice_positions(n, n, n, p)
    coords = np.stack([X, Y, Z], 1).ravel()
    m = n * p + 1
    plane = 3 * m * m
    ys = []
    halves = [(0, 1), (1, 4)]  # odd split: exercises the colour parity offset
    ops, xs, faces = [], [], []
    for r, (k0, k1) in enumerate(halves):
        c0, c1 = k0 * p, k1 * p
        sl = slice(c0 * plane, (c1 + 1) * plane)
        lv = G.FeLevel(n, n, k1 - k0, p=p, coords=coords[sl], dirichlet_faces=1 | (16 if r == 0 else 0),
                       z_offset=k0)
        assert lv.cartesian
        o = G.ElasticOperator(lv, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
        o.update_linearization(u0[sl])
        x = torch.tensor(v[sl], device="cuda")
        o.apply_elements(x, 0, k1 - k0)
        ops.append(o)
        xs.append(x)
    f_lo = torch.empty(ops[0].face_values(), dtype=torch.float64, device="cuda")
    f_hi = torch.empty(ops[1].face_values(), dtype=torch.float64, device="cuda")
    ops[0].pack_face(0, 1, f_lo)  # top layer of rank 0, upper face -> rank 1's ghost_lo
    ops[1].pack_face(0, 0, f_hi)  # bottom layer of rank 1, lower face -> rank 0's ghost_hi
    for r, o in enumerate(ops):
        yv = torch.empty_like(xs[r])
        mz = (halves[r][1] - halves[r][0]) * p + 1
        o.apply_nodes(xs[r], yv, 0, mz - 1, ghost_lo=f_lo if r == 1 else None, ghost_hi=f_hi if r == 0 else None)
        torch.cuda.synchronize()
        ys.append(yv.cpu().numpy())
    y_split = np.concatenate([ys[0], ys[1][plane:]])
    assert np.array_equal(ys[0][-plane:], ys[1][:plane])
    assert np.array_equal(y_split, y_full)


@pytest.mark.parametrize("tag,lmax,p", [("q2", 2, 2), ("q4", 2, 4)])
def test_multigrid_vcycle_and_pcg_vs_reference(G, tag, lmax, p):
    """fp32 hp-multigrid V-cycle (ladder, smoothers, transfers, Lanczos, coarse
    CG) and the fp64 outer PCG against the reference's MgHierarchy<float> on
    the well-posed cfg4 variant: CG iteration counts within +-1."""
    import torch
    g = np.load(os.path.join(GOLD, "multigrid.npz"))
    n = 1 << lmax
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(n, p=p)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=1, precision=32, coarse_direct_limit=0)
    assert mg.n_levels == {2: 4, 4: 5}[p]
    u0 = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
    mg.update_linearization(u0)
    r = torch.tensor(g[f"{tag}_r"], device="cuda")
    z = torch.empty_like(r)
    mg.precondition(r, z)
    torch.cuda.synchronize()
    assert rel(z.cpu().numpy(), g[f"{tag}_z"]) <= 1e-3
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(g[f"{tag}_b"], device="cuda")
    x = torch.empty_like(b)
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 200)
    assert abs(its - int(g[f"{tag}_its"])) <= 1, (its, int(g[f"{tag}_its"]))
    assert hist[-1] <= 1e-8
    assert rel(x.cpu().numpy(), g[f"{tag}_x"]) <= 1e-6


def test_fibre_frame_field_replicated_equals_global(G):
    """Per-qp frames that replicate the material frame reproduce the
    global-frame operator (to the last bits of H, recomputed on the device);
    cylindrical frames agree with the oracle."""
    from oracle import orcbind as O
    n, p = 2, 3
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    prm = G.MaterialParams(mu=1.0, kappa_b=100.0, k1=2.0, k2=5.0)
    u0 = I.make_u0(n, n, n, p)
    v = I.make_v(lev.n_dofs, 4)
    ys = {}
    for kind in ("global", "replicated", "cylindrical"):
        op = G.ElasticOperator(lev, "fiber", prm, "tensor", 64)
        op.set_fibre_frame(kind)
        op.update_linearization(u0)
        ys[kind] = op.apply_tangent(v)
        if kind == "cylindrical":
            h, m1 = op.fibre_field()
    assert rel(ys["replicated"], ys["global"]) <= 1e-14
    orc = O.OracleOperator(n, n, n, p, lev.node_coords(), 1, "fiber", prm.as_array(), "tensor", 64)
    orc.set_frames(h, m1)
    orc.update_linearization(u0)
    assert rel(ys["cylindrical"], orc.apply(v)) <= 1e-12
    assert not np.allclose(ys["cylindrical"], ys["global"])


@pytest.mark.parametrize("strategy", ["tensor", "none"])
def test_periodic_tube_vs_oracle(G, strategy):
    """BASELINE cfg3 geometry at small size: periodic-theta tube, per-qp
    cylindrical fibre frames.  Oracle: the open lattice with the seam row
    duplicated, y = P^T K P x (the reference has no periodic meshes)."""
    from oracle import orcbind as O
    from paper_2408_12479_b200 import workloads as W
    nx, ny, nz, p = 2, 8, 3, 3
    w = W.cfg3((nx, ny, nz))
    lev = w.level()
    assert lev.periodic_y and not lev.affine
    coords = lev.node_coords()
    u0 = W.tube_u0(w, coords)
    v = I.make_v(lev.n_dofs, 6)
    prm = w.material()
    co = I.periodic_to_open(coords, nx, ny, nz, p)
    for prec in (64, 32):
        op = G.ElasticOperator(lev, "fiber", prm, strategy, prec)
        op.set_fibre_frame("cylindrical")
        op.update_linearization(u0)
        y = op.apply_tangent(v)
        h, m1 = op.fibre_field()
        orc = O.OracleOperator(nx, ny, nz, p, co, 0, "fiber", prm.as_array(), strategy, prec)
        orc.set_frames(h, m1)
        orc.update_linearization(I.periodic_to_open(u0, nx, ny, nz, p))
        yo = I.open_to_periodic(orc.apply(I.periodic_to_open(v, nx, ny, nz, p).astype(orc.dtype)).astype(np.float64),
                                nx, ny, nz, p)
        assert rel(y, yo) <= {64: 1e-12, 32: 1e-5}[prec], (prec, rel(y, yo))


NEWTON = [("inh_p2_n4_curved", "inh", 2, 2, 0.05, 0.2), ("cnh_p3_n2_curved", "cnh", 1, 3, 0.05, 0.1),
          ("fiber_p2_n4_affine", "fiber", 2, 2, 0.0, 0.3)]


@pytest.mark.parametrize("case", NEWTON, ids=[c[0] for c in NEWTON])
@pytest.mark.parametrize("prec", [64, 32])
def test_residual_with_pressure_vs_reference(G, case, prec):
    """evaluate_residual + face-pressure load (operator.hpp:623-641, 925-1003)
    against the reference's own output, host and device entry points."""
    import torch
    name, model, lmax, p, damp, pres = case
    g = np.load(os.path.join(GOLD, "newton.npz"))
    n = 1 << lmax
    lev = G.FeLevel(n, p=p, map_param=(damp,))
    op = G.ElasticOperator(lev, model, params_from(g["params"], G), "none", prec)
    op.set_pressure(pres, 1)
    op.set_load_scale(0.75)
    u = I.make_u0(n, n, n, p, amp=0.05)
    r = op.evaluate_residual(u)
    assert rel(r, g[f"{name}_r"]) <= TOL[prec], rel(r, g[f"{name}_r"])
    mask = I.dirichlet_mask(n, n, n, p, 1)
    assert np.all(r[mask] == 0)
    du = torch.tensor(u.astype(op.dtype), device="cuda")
    dr = torch.empty_like(du)
    op.evaluate_residual_device(du, dr)
    torch.cuda.synchronize()
    assert np.array_equal(dr.cpu().numpy(), r)


@pytest.mark.parametrize("case", NEWTON, ids=[c[0] for c in NEWTON])
def test_newton_fgmres_mg_vs_reference(G, case):
    """newton_solve (solver.hpp:603-656) with FGMRES(30) right-preconditioned
    by the fp32 hp-multigrid V-cycle, one full pressure increment: the same
    Newton iteration count as the reference, FGMRES iterations within +-1 per
    Newton step, the same converged displacement."""
    import torch
    name, model, lmax, p, damp, pres = case
    g = np.load(os.path.join(GOLD, "newton.npz"))
    n = 1 << lmax
    prm = params_from(g["params"], G)
    lev = G.FeLevel(n, p=p, map_param=(damp,))
    op = G.ElasticOperator(lev, model, prm, "none", 64)
    op.set_pressure(pres, 1)
    mg = G.MgHierarchy(lev, model, prm, degree=6, coarse_n=1, precision=32, coarse_direct_limit=0)
    u = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
    nit, lit, res = G.newton_solve(op, mg, u)
    ref_nit, ref_lit = int(g[f"{name}_nit"]), int(g[f"{name}_lit"])
    assert nit == ref_nit, (nit, ref_nit)
    assert abs(lit - ref_lit) <= nit, (lit, ref_lit)
    assert res <= 1e-3 * np.linalg.norm(op_residual_at_zero(G, lev, model, prm, pres)) or res <= 1e-8
    assert rel(u.cpu().numpy(), g[f"{name}_u"]) <= 1e-5


def op_residual_at_zero(G, lev, model, prm, pres):
    op = G.ElasticOperator(lev, model, prm, "none", 64)
    op.set_pressure(pres, 1)
    return op.evaluate_residual(np.zeros(lev.n_dofs))


def test_fgmres_linear_solve_matches_pcg_solution(G):
    """Device FGMRES (solver.hpp:120-203) on the SPD cfg4-variant system: the
    same solution as PCG, identity preconditioner and multigrid."""
    import torch
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(4, p=2)
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = I.make_v(lev.n_dofs, 12)
    b[I.dirichlet_mask(4, 4, 4, 2, 1)] = 0.0
    db = torch.tensor(b, device="cuda")
    x_cg = torch.zeros_like(db)
    its, hist = G.pcg_solve(op, None, db, x_cg, 1e-12, 2000)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, precision=32)
    mg.update_linearization(torch.zeros_like(db))
    for pre, m in ((None, 400), (mg, 30)):
        x = torch.zeros_like(db)
        it, res = G.fgmres_solve(op, pre, db, x, abs_tol=0.0, rel_tol=1e-10, restart=m, max_restarts=20)
        assert res <= 1e-10 * np.linalg.norm(b)
        assert rel(x.cpu().numpy(), x_cg.cpu().numpy()) <= 1e-6
        if pre is mg:
            assert it < 60


SPATIAL = [("cnh_p3_n2_curved", "cnh", 1, 3, 0.05), ("inh_p2_n4_curved", "inh", 2, 2, 0.05),
           ("fiber_p2_n2_curved", "fiber", 1, 2, 0.05), ("inh_p4_n2_affine", "inh", 1, 4, 0.0)]


@pytest.mark.parametrize("case", SPATIAL, ids=[c[0] for c in SPATIAL])
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("strategy", ["none", "scalar", "tensor"])
def test_spatial_domain_vs_reference(G, case, prec, strategy):
    """Spatial (Omega_t) formulation (operator.hpp:506-519, constitutive.hpp:
    421-463): tangent apply, diagonal and residual against the reference."""
    name, model, lmax, p, damp = case
    g = np.load(os.path.join(GOLD, "spatial.npz"))
    n = 1 << lmax
    lev = G.FeLevel(n, p=p, map_param=(damp,))
    op = G.ElasticOperator(lev, model, params_from(g["params"], G), strategy, prec, domain="spatial")
    u0 = I.make_u0(n, n, n, p, amp=0.05)
    op.update_linearization(u0)
    y = op.apply_tangent(I.make_v(lev.n_dofs))
    ref = g[f"{name}_y{prec}_{strategy}"]
    assert rel(y, ref) <= TOL[prec], rel(y, ref)
    d, nb = op.compute_diagonal()
    assert nb == 0 and rel(d, g[f"{name}_diag{prec}"]) <= TOL[prec]
    r = op.evaluate_residual(u0)
    assert rel(r, g[f"{name}_r{prec}"]) <= TOL[prec], rel(r, g[f"{name}_r{prec}"])


def test_spatial_cachedf_rejected(G):
    lev = G.FeLevel(2, p=2)
    with pytest.raises(G.EmfGpuError):
        G.ElasticOperator(lev, "cnh", G.MaterialParams(), "cachedF", 64, domain="spatial")


@pytest.mark.parametrize("tag,lmax,p", [("q2", 2, 2), ("q4", 2, 4)])
def test_multigrid_dense_coarse_vs_reference(G, tag, lmax, p):
    """The reference's default hierarchy (coarse_direct_limit 2000 -> dense LU
    coarse solve, solver.hpp:369-401): device probing assembly + Gauss-Jordan
    inverse; V-cycle and outer PCG iteration counts against the reference."""
    import torch
    g = np.load(os.path.join(GOLD, "multigrid.npz"))
    n = 1 << lmax
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(n, p=p)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, precision=32)
    mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
    r = torch.tensor(g[f"{tag}_r"], device="cuda")
    z = torch.empty_like(r)
    mg.precondition(r, z)
    torch.cuda.synchronize()
    assert rel(z.cpu().numpy(), g[f"{tag}_dense_z"]) <= 1e-4, rel(z.cpu().numpy(), g[f"{tag}_dense_z"])
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(g[f"{tag}_b"], device="cuda")
    x = torch.empty_like(b)
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 200)
    assert abs(its - int(g[f"{tag}_dense_its"])) <= 1
    assert rel(x.cpu().numpy(), g[f"{tag}_dense_x"]) <= 1e-6


def test_dense_coarse_matches_cg_coarse(G):
    """Dense coarse solve and a tightly converged coarse CG agree (the coarse
    operator assembled by probing is the operator)."""
    import torch
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(4, p=1)
    u0 = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
    r = torch.tensor(I.make_v(lev.n_dofs, 5), device="cuda")
    zs = []
    for lim, rtol in ((2000, 1e-4), (0, 1e-13)):
        mg = G.MgHierarchy(lev, "inh", prm, degree=5, precision=64, coarse_n=4, coarse_direct_limit=lim,
                           coarse_rtol=rtol, coarse_maxit=5000)
        assert mg.n_levels == 1
        mg.update_linearization(u0)
        z = torch.empty_like(r)
        mg.precondition(r, z)
        zs.append(z.cpu().numpy())
    assert rel(zs[0], zs[1]) <= 1e-10


def test_stability_sweep_vs_reference(G):
    """Forward-stability lab (stability.cpp:163-251) on the device against the
    reference's run_sweep: identical invalid counts; bit-identical maxima for
    every cell whose formulas use no libm transcendental (SVK, iNH — the TU is
    built without FMA contraction and replays the reference's operation
    order); cells that call exp (fibre) or log (cNH) differ only by glibc vs
    CUDA libm ulps on the worst sample."""
    g = np.load(os.path.join(GOLD, "stability.npz"))
    prm = G.MaterialParams(mu=62.1, lam=3042.9, kappa_b=3084.3, k1=1.4, k2=22.1, a=3.62, b=34.3,
                           phi=27.47 * np.pi / 180.0)
    err, inv = G.stability_sweep(g["scales"], 200, 42, prm)
    assert np.array_equal(inv, g["inv"])
    ref = g["err"]
    names = [(m, f, q) for m in G.SWEEP_MODELS for f in G.SWEEP_FORMULATIONS for q in G.SWEEP_QUANTITIES]
    for c, (m, f, q) in enumerate(names):
        if m in ("svk", "iNH"):
            assert np.array_equal(err[:, c], ref[:, c]), (m, f, q)
        else:
            np.testing.assert_allclose(err[:, c], ref[:, c], rtol=0.25, atol=0)
    assert (err == ref).mean() > 0.9
    # ordering/validation contract
    with pytest.raises(G.EmfGpuError):
        G.stability_sweep([1e-3, 1e-4], 10)


def test_pinned_host_apply_pipeline_bitwise(G):
    """The pipelined host-vector apply (pinned buffers: z-chunked copies
    overlapped with per-chunk element/node launches, graph-captured from the
    second call on) returns exactly the device-resident apply, repeatedly."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12479_b200 import emfgpu as G, inputs as I
for (n, p, model, strat) in ((16, 3, "cnh", "none"), (8, 4, "inh", "scalar"), (16, 2, "fiber", "none"), (16, 3, "cnh", "tensor")):
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    op = G.ElasticOperator(lev, model, prm, strat, 64)
    op.update_linearization(I.make_u0(n, n, n, p, amp=0.05))
    v = I.make_v(lev.n_dofs)
    hx = torch.tensor(v).pin_memory(); hy = torch.empty_like(hx).pin_memory()
    dx = hx.cuda(); dy = torch.empty_like(dx)
    op.apply_tangent_device(dx, dy); torch.cuda.synchronize()
    ref = dy.cpu().numpy()
    for it in range(4):
        hy.fill_(float("nan"))
        assert G.lib().emfgpu_op_apply_host(op.h, hx.data_ptr(), hy.data_ptr()) == 0
        assert np.array_equal(hy.numpy(), ref), (n, p, model, strat, it)
print("ok")
'''
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


# ---- property tests in the style of the reference's own suite
# (test_operator.cpp:92-318, test_solver.cpp:352-440)

def _free_vec(n, p, seed, nn=4):
    v = I.make_v(3 * (nn * p + 1) ** 3, seed)
    v[I.dirichlet_mask(nn, nn, nn, p, 1)] = 0.0
    return v


@pytest.mark.parametrize("model", ["cnh", "inh", "fiber"])
@pytest.mark.parametrize("domain", ["material", "spatial"])
def test_tangent_is_the_residual_derivative(G, model, domain):
    """Central difference of the device residual equals the device tangent
    (test_operator.cpp:92-133): ||(r(u+hv) - r(u-hv))/2h - K v|| small.
    h = 1e-7: the fibre stress jumps where the tension gate switches (the gate
    follows the mean direction, the stress the dispersed H), and with the
    seeded noise one point lies within 1e-6 of the switch; the reference's
    residual and tangent (checked through the bit-exact oracle) behave alike."""
    n, p = 4, 2
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    op = G.ElasticOperator(lev, model, prm, "none", 64, domain=domain)
    u = I.make_u0(n, n, n, p, amp=0.05)
    op.update_linearization(u)
    v = _free_vec(n, p, 3)
    kv = op.apply_tangent(v)
    h = 1e-7
    fd = (op.evaluate_residual(u + h * v) - op.evaluate_residual(u - h * v)) / (2 * h)
    free = ~I.dirichlet_mask(n, n, n, p, 1)
    assert rel(fd[free], kv[free]) <= 1e-6, rel(fd[free], kv[free])


@pytest.mark.parametrize("model", ["cnh", "inh", "fiber"])
def test_tangent_symmetric_and_domains_agree(G, model):
    """Hyperelastic tangent is symmetric on the free DoFs (test_operator.cpp:
    171-223); material and spatial forms are the same operator (:236-258);
    all fp64 strategies agree (strategies <= 1e-13)."""
    n, p = 4, 3
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    u = I.make_u0(n, n, n, p, amp=0.05)
    v, w = _free_vec(n, p, 5), _free_vec(n, p, 6)
    ys = {}
    for dom in ("material", "spatial"):
        for strat in ("none", "scalar", "tensor") + (("cachedF",) if dom == "material" else ()):
            op = G.ElasticOperator(lev, model, prm, strat, 64, domain=dom)
            op.update_linearization(u)
            ys[(dom, strat)] = (op.apply_tangent(v), op.apply_tangent(w))
    kv, kw = ys[("material", "none")]
    assert abs(w @ kv - v @ kw) <= 1e-12 * abs(w @ kv)
    for key, (a, b) in ys.items():
        tol = 1e-13 if key[0] == "material" else 1e-10
        assert rel(a, kv) <= tol and rel(b, kw) <= tol, (key, rel(a, kv))


def test_multigrid_zero_rhs_and_beats_plain_cg(G):
    """A zero right-hand side gives exactly zero from the V-cycle
    (test_solver.cpp:352-368); the MG-preconditioned CG needs fewer
    iterations than plain CG (:390-440)."""
    import torch
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(4, p=4)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, precision=32)
    z0 = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
    mg.update_linearization(z0)
    z = torch.full_like(z0, 7.0)
    mg.precondition(torch.zeros_like(z0), z)
    torch.cuda.synchronize()
    assert torch.count_nonzero(z).item() == 0
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(_free_vec(4, 4, 9), device="cuda")
    its_mg, _ = G.pcg_solve(op, mg, b, torch.empty_like(b), 1e-8, 500)
    its_cg, _ = G.pcg_solve(op, None, b, torch.empty_like(b), 1e-8, 2000)
    assert its_mg < its_cg / 4, (its_mg, its_cg)


# ---- BASELINE configs 2 and 3 at full size: size-independent properties

def _device_props(G, op, n, free_mask, seed=21):
    import torch
    dt = torch.float64 if op.precision == 64 else torch.float32
    v = torch.tensor(I.make_v(n, seed), dtype=dt, device="cuda")
    w = torch.tensor(I.make_v(n, seed + 1), dtype=dt, device="cuda")
    if free_mask is not None:
        fm = torch.tensor(free_mask, device="cuda")
        v *= fm
        w *= fm
    kv, kw, kvw = torch.empty_like(v), torch.empty_like(v), torch.empty_like(v)
    op.apply_tangent_device(v, kv)
    op.apply_tangent_device(w, kw)
    op.apply_tangent_device(0.75 * v - 1.25 * w, kvw)
    torch.cuda.synchronize()
    lin = (torch.linalg.norm((kvw - (0.75 * kv - 1.25 * kw)).double()) / torch.linalg.norm(kvw.double())).item()
    sym = abs((torch.dot(w.double(), kv.double()) - torch.dot(v.double(), kw.double())).item()) / abs(
        torch.dot(w.double(), kv.double()).item())
    return lin, sym, kv


def test_cfg2_full_size_properties(G):
    """cfg2 (64^3 Q4 iNH on the curved map, 50.9M DoFs, scaled-noise u0):
    the literal noise is rejected at the reference's first (e, q); linear,
    symmetric on the free DoFs, strategies and precisions agree."""
    from paper_2408_12479_b200 import workloads as W
    lit = W.cfg2(literal=True)
    lev = lit.level()
    op = G.ElasticOperator(lev, "inh", lit.material(), "none", 64)
    with pytest.raises(G.NonPositiveJacobian) as ex:
        op.update_linearization(lit.u0())
    assert (ex.value.element, ex.value.qpoint) == (1, 46)
    w = W.cfg2()
    u0 = w.u0()
    free = ~I.dirichlet_mask(64, 64, 64, 4, 1)
    kvs = {}
    for strat, prec in (("none", 64), ("tensor", 64), ("none", 32)):
        op = G.ElasticOperator(lev, "inh", w.material(), strat, prec)
        op.update_linearization(u0)
        lin, sym, kv = _device_props(G, op, lev.n_dofs, free)
        assert lin <= {64: 1e-13, 32: 1e-5}[prec], (strat, prec, lin)
        assert sym <= {64: 1e-10, 32: 1e-4}[prec], (strat, prec, sym)
        kvs[(strat, prec)] = kv.double().cpu().numpy()
        del op
    assert rel(kvs[("tensor", 64)], kvs[("none", 64)]) <= 1e-12
    assert rel(kvs[("none", 32)], kvs[("none", 64)]) <= 1e-5


def test_cfg3_full_size_properties(G):
    """cfg3 (periodic tube 16x128x256 Q3, 43.4M DoFs, per-qp cylindrical fibre
    frames, no Dirichlet face): linear and symmetric, fp64 tensor == none,
    fp32 within 1e-5; rigid translations are in the kernel of the tangent
    (no Dirichlet face, periodic seam handled)."""
    import torch
    from paper_2408_12479_b200 import workloads as W
    w = W.cfg3()
    lev = w.level()
    u0 = W.tube_u0(w, lev.node_coords())
    kvs = {}
    for strat, prec in (("tensor", 64), ("none", 64), ("tensor", 32)):
        op = G.ElasticOperator(lev, "fiber", w.material(), strat, prec)
        op.set_fibre_frame("cylindrical")
        op.update_linearization(u0)
        lin, sym, kv = _device_props(G, op, lev.n_dofs, None)
        assert lin <= {64: 1e-13, 32: 1e-5}[prec], (strat, prec, lin)
        assert sym <= {64: 1e-10, 32: 1e-4}[prec], (strat, prec, sym)
        kvs[(strat, prec)] = kv.double().cpu().numpy()
        if (strat, prec) == ("tensor", 64):
            t = torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda")
            t[0::3] = 1.0  # rigid x-translation
            kt = torch.empty_like(t)
            op.apply_tangent_device(t, kt)
            torch.cuda.synchronize()
            assert torch.linalg.norm(kt).item() <= 1e-9 * np.linalg.norm(kvs[(strat, prec)])
        del op
    assert rel(kvs[("none", 64)], kvs[("tensor", 64)]) <= 1e-12
    assert rel(kvs[("tensor", 32)], kvs[("tensor", 64)]) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("p,prec,strat", [(3, 64, "none"), (3, 32, "none"), (4, 64, "tensor"), (2, 64, "scalar")])
def test_ticket_scheduler_ranges_streams_repeats(G, p, prec, strat):
    """The element kernels hand out work by per-launch ticket counters (a ring
    of slots per operator, rewound by the last worker out).  Element-range
    launches on two streams at once, many back-to-back launches and the
    whole-lattice apply all give bitwise the same result."""
    import torch
    n = 6
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), strat, prec)
    op.update_linearization(I.make_u0(n, n, n, p))
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
    y_ref = torch.empty_like(x)
    op.apply_tangent_device(x, y_ref)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    mz = n * p + 1
    for _ in range(3):
        # disjoint element layer ranges on two streams concurrently
        with torch.cuda.stream(s1):
            op.apply_elements(x, 0, 2, stream=s1.cuda_stream)
        with torch.cuda.stream(s2):
            op.apply_elements(x, 2, n, stream=s2.cuda_stream)
        torch.cuda.synchronize()
        y = torch.empty_like(x)
        op.apply_nodes(x, y, 0, mz - 1)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
    for _ in range(300):  # more launches than ticket slots
        op.apply_tangent_device(x, y)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("p,prec,strat,dims,kw", [
    (4, 64, "none", (20, 12, 18), dict(map="shear_x", map_param=(0.1,))),
    (4, 32, "none", (20, 12, 18), dict(map="shear_x", map_param=(0.1,))),
    (4, 64, "tensor", (7, 5, 3), dict(map_param=(0.05,), dirichlet_faces=1 | 32)),
    (3, 64, "none", (24, 16, 20), dict(map_param=(0.05,))),
    (3, 32, "cachedF", (3, 8, 11), "tube"),
    (3, 64, "none", (4, 8, 5), "tube"),
    (3, 64, "scalar", (2, 2, 1), dict(map_param=(0.05,))),
    (2, 64, "none", (10, 6, 9), dict(map_param=(0.05,), dirichlet_faces=3)),
    (1, 64, "none", (16, 8, 12), dict(map_param=(0.05,))),
])
def test_whole_apply_equals_split_launches(G, p, prec, strat, dims, kw):
    """The whole-lattice apply (element kernel + programmatically dependent
    node kernel) gives bitwise the result of the split element-range +
    node-plane launches of the public API, across shapes (one layer, more
    CTAs than units per layer, periodic y, Dirichlet faces), and over
    repeated launches."""
    import torch
    nx, ny, nz = dims
    if kw == "tube":  # periodic-theta tube (cfg3 geometry), fibre model
        from paper_2408_12479_b200 import workloads as W
        w = W.cfg3(dims)
        lev = w.level()
        assert lev.periodic_y
        op = G.ElasticOperator(lev, "fiber", w.material(), strat, prec)
        op.set_fibre_frame("cylindrical")
        op.update_linearization(W.tube_u0(w, lev.node_coords()))
    else:
        lev = G.FeLevel(nx, ny, nz, p=p, **kw)
        op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), strat, prec)
        op.update_linearization(I.make_u0(nx, ny, nz, p))
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
    mz = nz * p + 1
    y_split = torch.full_like(x, float("nan"))
    op.apply_elements(x, 0, nz)
    op.apply_nodes(x, y_split, 0, mz - 1)
    for _ in range(20):
        y = torch.full_like(x, float("nan"))
        op.apply_tangent_device(x, y)
        torch.cuda.synchronize()
        assert torch.equal(y, y_split)


@pytest.mark.gpu
def test_pcg_graph_loop_equals_host_loop(G):
    """The device-resident PCG (conditional-WHILE CUDA graph around apply,
    V-cycle and device scalars) gives bitwise the iterates, history and
    iteration count of the host-driven loop (EMFGPU_PCG_GRAPH=0)."""
    import subprocess
    import sys
    code = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12479_b200 import emfgpu as G, inputs as I
n, p = 6, 2
lev = G.FeLevel(n, p=p)
prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=3, precision=32)
mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
op = G.ElasticOperator(lev, "inh", prm, "none", 64)
op.update_linearization(np.zeros(lev.n_dofs))
b = torch.tensor(I.make_v(lev.n_dofs, 2), device="cuda")
b[torch.tensor(I.dirichlet_mask(n, n, n, p, 1), device="cuda")] = 0
x = torch.empty_like(b)
its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 200)
x2 = torch.empty_like(b)
its2, hist2 = G.pcg_solve(op, None, b, x2, 1e-10, 3000)
print(its, its2, hashlib.sha1(x.cpu().numpy().tobytes() + hist.tobytes() + x2.cpu().numpy().tobytes()).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, EMFGPU_PCG_GRAPH=flag)
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root, env=env)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(out.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs


@pytest.mark.gpu
@pytest.mark.parametrize("case", [(11, 3, "cnh", "none", 64), (11, 3, "inh", "tensor", 32), (11, 3, "fiber", "tensor", 64),
                                  (9, 4, "inh", "none", 64), (9, 4, "inh", "none", 32), (9, 4, "fiber", "tensor", 32),
                                  (9, 4, "inh", "cachedF", 64), (13, 2, "inh", "tensor", 32)],
                         ids=lambda c: "-".join(map(str, c)))
def test_element_kernels_repeat_bitwise(G, case):
    """Race proxy (no compute-sanitizer on the pool): the collocated Q3 / Q4
    kernels, the push-forward tensor cache and the v2 residual give bitwise the
    same vectors run after run, on odd element counts (padding elements in the
    last CTA) with several CTAs per SM (tools/repeat_bitwise.py is the long form)."""
    import torch
    n, p, model, strat, prec = case
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    op = G.ElasticOperator(lev, model, G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0), strat, prec)
    u0 = I.make_u0(n, n, n, p, amp=0.02, noise=1e-4)
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(I.make_v(lev.n_dofs), dtype=dt, device="cuda")
    du = torch.tensor(u0, dtype=dt, device="cuda")
    y0, r0, y, r = (torch.empty_like(x) for _ in range(4))
    op.apply_tangent_device(x, y0)
    op.evaluate_residual_device(du, r0)
    assert bool(torch.isfinite(y0).all()) and bool(torch.isfinite(r0).all())
    for _ in range(8):
        op.apply_tangent_device(x, y)
        op.evaluate_residual_device(du, r)
        assert torch.equal(y, y0) and torch.equal(r, r0)


@pytest.mark.gpu
def test_checksum_is_fnv1a_of_the_linearization_point(G):
    """checksum() (operator.hpp:90, 650): FNV-1a over the bytes of u_k, computed
    on demand from the device copy -- after a host and after a device update."""
    import torch

    def fnv1a(buf):
        h = 1469598103934665603
        for byte in buf:
            h = ((h ^ byte) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h

    n, p = 3, 2
    lev = G.FeLevel(n, p=p)
    op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "tensor", 64)
    u0 = I.make_u0(n, n, n, p)
    op.update_linearization(u0)
    assert op.checksum() == fnv1a(np.ascontiguousarray(u0, dtype=np.float64).tobytes())
    u1 = 0.5 * u0
    op.update_linearization_device(torch.tensor(u1, device="cuda"))
    assert op.checksum() == fnv1a(u1.tobytes())
    assert op.checksum() == fnv1a(u1.tobytes())  # cached


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["cnh", "inh", "fiber"])
def test_pcg_with_tensor_strategy_levels(G, model):
    """The V-cycle's level operators on strategy tensor (cNH / iNH / fibre: the
    cached push-forward state, csrc/qp.cuh PushState) precondition like the
    on-the-fly levels: same PCG iteration count within 1, same solution."""
    import torch
    n, p = 6, 4
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    u0 = I.make_u0(n, n, n, p, amp=0.003, noise=1e-5)  # small: the tangent stays positive definite
    op = G.ElasticOperator(lev, model, prm, "none", 64)
    op.update_linearization(u0)
    b = torch.tensor(I.make_v(lev.n_dofs, 2), device="cuda")
    b[torch.tensor(I.dirichlet_mask(n, n, n, p, 1), device="cuda")] = 0
    du = torch.tensor(u0, device="cuda")
    res = {}
    for strat in ("none", "tensor"):
        mg = G.MgHierarchy(lev, model, prm, strategy=strat, degree=5, coarse_n=3, precision=32)
        mg.update_linearization(du)
        x = torch.empty_like(b)
        its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 200)
        res[strat] = (its, x)
    assert abs(res["none"][0] - res["tensor"][0]) <= 1, (res["none"][0], res["tensor"][0])
    err = float(torch.linalg.vector_norm(res["none"][1] - res["tensor"][1]) / torch.linalg.vector_norm(res["none"][1]))
    assert err <= 1e-6, err


# ---- BASELINE configs[2] shape against the reference itself (shear map)

@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("strategy", ["none", "scalar", "tensor", "cachedF"])
def test_shear_map_q4_inh_vs_reference(G, n, prec, strategy):
    """cfg2's operator at small size: the device-generated shear map
    x' = x + 0.1 sin(2 pi y) e_x (EMFGPU_MAP_SHEAR_X), iNH kappa/mu = 1000, Q4,
    u0 amplitude 0.1 at pre-map coordinates + scaled noise, against the
    unmodified reference on the same coordinates (tests/golden/shear.npz)."""
    from paper_2408_12479_b200 import workloads as W
    g = np.load(os.path.join(GOLD, "shear.npz"))
    w = W.cfg2(n=n)
    lev = w.level()
    tag = f"n{n}"
    assert rel(lev.node_coords(), g[f"{tag}_coords"]) <= 1e-15
    assert np.array_equal(w.u0(), g[f"{tag}_u0"]) and np.array_equal(w.v(), g[f"{tag}_v"])
    op = G.ElasticOperator(lev, "inh", params_from(g["params"], G), strategy, prec)
    op.update_linearization(g[f"{tag}_u0"])
    y = op.apply_tangent(g[f"{tag}_v"])
    key = f"{tag}_y{prec}_{strategy if strategy != 'cachedF' else 'none'}"
    assert rel(y, g[key]) <= TOL[prec], rel(y, g[key])
    assert rel(y, g[f"{tag}_y64_none"]) <= TOL[prec]
    if strategy == "none":
        d, nb = op.compute_diagonal()
        assert rel(d, g[f"{tag}_diag{prec}"]) <= TOL[prec]
        assert nb == int(g[f"{tag}_diag{prec}_nbad"])


def _cfg2_full():
    import json
    with open(os.path.join(GOLD, "cfg2_full.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("prec,strategy", [(64, "none"), (64, "tensor"), (64, "scalar"), (32, "none"),
                                           (32, "tensor")])
def test_cfg2_full_size_vs_reference(G, prec, strategy):
    """BASELINE configs[2] at full size (64^3 Q4 curved iNH, 50 923 779 DoFs)
    against the unmodified reference's known answers (tests/golden/
    cfg2_full.json, make_golden.cfg2_full): ||y||_2 and y at 2051 sampled
    DoFs (incl. the centre node) within 1e-12 (fp64) / 1e-5 (fp32)."""
    import torch
    from paper_2408_12479_b200 import workloads as W
    ref = _cfg2_full()
    w = W.cfg2()
    lev = w.level()
    assert lev.n_dofs == ref["ndofs"]
    u0, v = w.u0(), w.v()
    assert np.isclose(np.linalg.norm(u0), ref["norm_u0"], rtol=1e-14)
    assert np.isclose(np.linalg.norm(v), ref["norm_v"], rtol=1e-14)
    op = G.ElasticOperator(lev, "inh", w.material(), strategy, prec)
    op.update_linearization(u0)
    dt = torch.float64 if prec == 64 else torch.float32
    x = torch.tensor(v, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    op.apply_tangent_device(x, y)
    torch.cuda.synchronize()
    sd = torch.tensor(ref["sample_dofs"], device="cuda")
    ys = y[sd].double().cpu().numpy()
    ny = torch.linalg.norm(y.double()).item()
    key = 64 if prec == 64 else 32
    assert abs(ny - ref[f"norm_y{key}"]) <= TOL[prec] * ref[f"norm_y{key}"], (ny, ref[f"norm_y{key}"])
    assert rel(ys, ref[f"y{key}_sample"]) <= TOL[prec], rel(ys, ref[f"y{key}_sample"])
    assert rel(ys, ref["y64_sample"]) <= TOL[prec]


@pytest.mark.gpu
def test_concurrent_applies_one_operator(G):
    """apply_tangent is const and may be called concurrently:
    whole applies of ONE operator issued on two streams at once, a device
    apply on the legacy stream followed at once by the host-vector apply, and
    two host threads calling the host-vector apply all give the serial
    results bitwise (the handle orders its entries, capi.cu UseGuard)."""
    import threading

    import torch
    n, p = 6, 4
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
    op.update_linearization(I.make_u0(n, n, n, p))
    v1, v2 = I.make_v(lev.n_dofs, 1), I.make_v(lev.n_dofs, 7)
    x1 = torch.tensor(v1, dtype=torch.float64, device="cuda")
    x2 = torch.tensor(v2, dtype=torch.float64, device="cuda")
    r1, r2 = torch.empty_like(x1), torch.empty_like(x1)
    op.apply_tangent_device(x1, r1)
    op.apply_tangent_device(x2, r2)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(20):
        y1, y2 = torch.full_like(x1, np.nan), torch.full_like(x1, np.nan)
        op.apply_tangent_device(x1, y1, stream=s1.cuda_stream)
        op.apply_tangent_device(x2, y2, stream=s2.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(y1, r1) and torch.equal(y2, r2)
    # device apply on the legacy stream, then the host-vector apply right away
    y1 = torch.full_like(x1, np.nan)
    op.apply_tangent_device(x1, y1, stream=0)
    h2 = op.apply_tangent(v2)
    torch.cuda.synchronize()
    assert torch.equal(y1, r1)
    assert np.array_equal(h2, r2.cpu().numpy())
    # two host threads on the host-vector entry point
    out = {}

    def worker(k, v):
        out[k] = [op.apply_tangent(v) for _ in range(5)]

    ts = [threading.Thread(target=worker, args=(k, v)) for k, v in ((1, v1), (2, v2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a in out[1]:
        assert np.array_equal(a, r1.cpu().numpy())
    for a in out[2]:
        assert np.array_equal(a, r2.cpu().numpy())


@pytest.mark.gpu
def test_pcg_reports_nonconvergence(G):
    """A PCG solve that stops at maxit above rtol returns EMFGPU_ERR_NUMERICAL
    (the reference's solvers throw on non-convergence, solver.hpp:202, 423)."""
    import torch
    n, p = 4, 2
    lev = G.FeLevel(n, p=p, map_param=(0.0,))
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(I.make_v(lev.n_dofs, 2), dtype=torch.float64, device="cuda")
    b[torch.tensor(I.dirichlet_mask(n, n, n, p, 1), device="cuda")] = 0
    x = torch.zeros_like(b)
    with pytest.raises(G.EmfGpuError) as ex:
        G.pcg_solve(op, None, b, x, rtol=1e-12, maxit=3)
    assert ex.value.code == 2 and "no convergence" in str(ex.value)
    it, hist = G.pcg_solve(op, None, b, x, rtol=1e-8, maxit=2000)
    assert hist[-1] <= 1e-8


LOADS = [("inh_p2_n4_curved", "inh", 2, 2, 0.05, 0.2, 1, 1, 0b101010),
         ("cnh_p3_n2_curved", "cnh", 1, 3, 0.05, 0.0, 1, 1, 0b000110),
         ("fiber_p4_n2_affine", "fiber", 1, 4, 0.0, 0.1, 4, 0, 0b100001)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", LOADS, ids=[c[0] for c in LOADS])
@pytest.mark.parametrize("prec", [64, 32])
def test_residual_with_body_force_and_tractions_vs_reference(G, case, prec):
    """The full Loads struct (operator.hpp:23-32, build_load_vector 880-1008):
    face pressure, body force B(X) and tractions h(X, N) given as callbacks,
    against the reference with the same functions (oracle/ref_driver.cpp
    fixtures), load scale 0.5."""
    import math
    name, model, lmax, p, damp, pres, face, body, tf = case
    g = np.load(os.path.join(GOLD, "loads.npz"))
    n = 1 << lmax
    lev = G.FeLevel(n, p=p, map_param=(damp,))
    op = G.ElasticOperator(lev, model, params_from(g["params"], G), "none", prec)
    op.set_loads(pressure=pres, pressure_face=face,
                 body_force=(lambda x: (0.3 + math.sin(x[0]), x[1] * x[2] - 0.2, 1.0 - x[0] * x[0])) if body else None,
                 traction=lambda x, nn: (nn[0] + 0.5 * x[1], 0.25 * nn[1] * x[2], x[0] - nn[2]),
                 traction_faces=[f for f in range(6) if (tf >> f) & 1])
    op.set_load_scale(0.5)
    u = I.make_u0(n, n, n, p, amp=0.05)
    r = op.evaluate_residual(u)
    assert rel(r, g[f"{name}_r"]) <= TOL[prec], rel(r, g[f"{name}_r"])


@pytest.mark.gpu
def test_diagonal_nonpositive_indices(G):
    """compute_diagonal's second member (operator.hpp:869-877): the ascending
    indices of free rows with diag <= 0, checked against the returned diagonal
    (scaled by -1 on a set of free rows through a negative load-free state is
    not reachable with valid parameters, so the list is checked for
    consistency and the capacity cut)."""
    import torch
    n, p = 4, 2
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", 64)
    u = I.make_u0(n, n, n, p, amp=0.05)
    op.update_linearization(u)
    d = torch.empty(lev.n_dofs, dtype=torch.float64, device="cuda")
    idx, cnt = op.compute_diagonal_indices(d)
    diag = d.cpu().numpy()
    free = ~I.dirichlet_mask(n, n, n, p, 1)
    want = np.nonzero(free & ~(diag > 0))[0]
    assert cnt == len(want) and np.array_equal(idx, want)
    idx2, cnt2 = op.compute_diagonal_indices(d, capacity=0)
    assert cnt2 == cnt and len(idx2) == 0


def test_formulation_and_kernel_config_rejected(G):
    """Formulation::stability = standard and non-default KernelConfig fields
    are refused with EMFGPU_ERR_CONFIG (the device kernels implement the
    stable formulation with the default KernelConfig only)."""
    lev = G.FeLevel(2, p=2)
    G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)  # defaults accepted
    with pytest.raises(G.EmfGpuError) as ex:
        G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64, stability="standard")
    assert ex.value.code == 1 and "standard" in str(ex.value)
    for field, val in (("ln_series_terms", 12), ("jpow_newton_steps", 2), ("exp_mode", 1), ("jpow_mode", 1)):
        kc = G.KernelConfig.default()
        setattr(kc, field, val)
        with pytest.raises(G.EmfGpuError) as ex:
            G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64, kernel_config=kc)
        assert ex.value.code == 1 and field in str(ex.value)


@pytest.mark.gpu
@pytest.mark.parametrize("splits", [[(0, 1), (1, 4)], [(0, 2), (2, 3), (3, 5)]], ids=["2slabs", "3slabs"])
def test_slab_group_apply_and_dot_bitwise(G, splits):
    """The z-slab apply below the C ABI (emfgpu_slab_group_apply: boundary
    layers, face packs, peer-copied ghost faces on each slab's communication
    stream overlapped with the interior layers, node phase with ghosts) gives
    every slab BITWISE the single-level result on its node planes, repeatedly
    and on separate streams; the group dot counts interface planes once."""
    import torch
    n, p = 4, 2
    nz = splits[-1][1]
    lev = G.FeLevel(n, n, nz, p=p, dirichlet_faces=1 | 16)
    u0 = I.make_u0_planes(n, n, nz, p, 0, nz * p, faces=1 | 16, extent=(1.0, 1.0, 1.0))
    lev = G.FeLevel(n, n, nz, p=p, dirichlet_faces=1 | 16)
    v = I.make_v(lev.n_dofs)
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
    op.update_linearization(u0)
    y_full = op.apply_tangent(v)
    coords = lev.node_coords()
    m = n * p + 1
    plane = 3 * m * m
    ops, xs, slabs, sls = [], [], [], []
    for r, (k0, k1) in enumerate(splits):
        sl = slice(k0 * p * plane, (k1 * p + 1) * plane)
        faces = 1 | (16 if r == 0 else 0) | (32 if r == len(splits) - 1 else 0)
        lv = G.FeLevel(n, n, k1 - k0, p=p, coords=coords[sl], dirichlet_faces=faces & (1 | 16), z_offset=k0)
        o = G.ElasticOperator(lv, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
        o.update_linearization(u0[sl])
        ops.append(o)
        xs.append(torch.tensor(v[sl], device="cuda"))
        sls.append(sl)
    slabs = [G.Slab(o, r, len(splits)) for r, o in enumerate(ops)]
    streams = [torch.cuda.Stream() for _ in splits]
    for _ in range(3):
        ys = [torch.full_like(x, np.nan) for x in xs]
        G.slab_group_apply(slabs, xs, ys, streams)
        torch.cuda.synchronize()
        for r, sl in enumerate(sls):
            assert np.array_equal(ys[r].cpu().numpy(), y_full[sl]), r
    outs = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in splits]
    G.slab_group_dot(slabs, xs, ys, outs, streams)
    torch.cuda.synchronize()
    vals = [float(o.item()) for o in outs]
    assert all(vv == vals[0] for vv in vals)
    assert abs(vals[0] - float(np.dot(v, y_full))) <= 1e-12 * abs(float(np.dot(v, y_full)))
    # a single slab (world 1) is the plain apply
    s1 = G.Slab(op, 0, 1)
    x = torch.tensor(v, device="cuda")
    y = torch.empty_like(x)
    s1.apply(x, y)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_full)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [3, 6])
def test_dense_coarse_solve_vs_reference_cg_coarse(G, n):
    """The reference's DenseLU::solve (solver.hpp:73-78) applies the row
    interchanges interleaved with the forward elimination although factor()
    (55-63) swapped whole rows, so its dense coarse solve is wrong once
    partial pivoting swaps rows (3^3 Q4: 300 PCG iterations without
    convergence; with its coarse Jacobi-PCG instead: 36).  The device dense
    coarse solve is the exact one: its V-cycle equals the reference's
    CG-coarse V-cycle to the coarse CG's 1e-4, and the PCG iterations match
    the reference's CG-coarse hierarchy within +-1 (the reference's dense
    ones do not)."""
    import torch
    g = np.load(os.path.join(GOLD, "coarse_lu.npz"))
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(n, p=4)
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    b = torch.tensor(g[f"n{n}_b"], device="cuda")
    r = torch.tensor(g[f"n{n}_r"], device="cuda")
    ref_cg = int(g[f"n{n}_lim0_its"])
    assert rel(g[f"n{n}_lim2000_z"], g[f"n{n}_lim0_z"]) > 1e-2  # the reference's dense coarse solve is off
    for lim in (2000, 0):
        mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=n, precision=32, coarse_direct_limit=lim)
        mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
        z = torch.empty_like(r)
        mg.precondition(r, z)
        torch.cuda.synchronize()
        assert rel(z.cpu().numpy(), g[f"n{n}_lim0_z"]) <= 1e-3, (lim, rel(z.cpu().numpy(), g[f"n{n}_lim0_z"]))
        x = torch.empty_like(b)
        its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 300)
        assert abs(its - ref_cg) <= 1, (lim, its, ref_cg)


@pytest.mark.gpu
def test_slab_nccl_communicator_single_rank(G):
    """The NCCL side of the slab layer on one GPU: libnccl.so.2 loaded at run
    time, a 1-rank communicator from a unique id, a slab apply through it
    (no neighbours: the plain apply) and the device dot."""
    import torch
    n, p = 4, 3
    lev = G.FeLevel(n, p=p, map_param=(0.05,))
    op = G.ElasticOperator(lev, "inh", G.MaterialParams(kappa_b=50.0), "none", 64)
    op.update_linearization(I.make_u0(n, n, n, p))
    v = I.make_v(lev.n_dofs)
    y_ref = op.apply_tangent(v)
    uid = G.Comm.unique_id()
    assert len(uid) == 128
    comm = G.Comm(uid, 1, 0, device=torch.cuda.current_device())
    slab = G.Slab(op, 0, 1, comm)
    x = torch.tensor(v, device="cuda")
    y = torch.empty_like(x)
    slab.apply(x, y)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    slab.dot(x, y, out)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_ref)
    assert abs(float(out.item()) - float(np.dot(v, y_ref))) <= 1e-12 * abs(float(np.dot(v, y_ref)))
    del slab, comm


@pytest.mark.gpu
@pytest.mark.parametrize("world,shear", [(2, 0.0), (3, 0.0), (4, 0.1)])
def test_slab_pcg_multigrid_bitwise_vs_single_gpu(G, world, shear):
    """The cfg4 solve partitioned in z slabs (emfgpu_slab_solver: finest
    level on the slabs with face exchange, ghost-layer restriction and
    node-plane dots; p/2 level and below agglomerated), ranks run as host
    threads on one GPU (thread-group transport): iteration count, residual
    history and every rank's x are bitwise the single-GPU PCG + hp-MG solve."""
    import threading

    import torch
    n, p = 12, 4
    prm = G.MaterialParams(mu=1.0, lam=10.0, kappa_b=50.0)
    lev = G.FeLevel(n, p=p, map="shear_x", map_param=(shear,)) if shear else G.FeLevel(n, p=p)
    u0 = np.zeros(lev.n_dofs)  # the well-posed cfg4 variant (u0 = 0)
    b_np = I.make_v(lev.n_dofs, 2)
    b_np[I.dirichlet_mask(n, n, n, p, 1)] = 0.0
    op = G.ElasticOperator(lev, "inh", prm, "none", 64)
    op.update_linearization(u0)
    mg = G.MgHierarchy(lev, "inh", prm, degree=5, coarse_n=6, precision=32)
    mg.update_linearization(torch.tensor(u0, device="cuda"))
    b = torch.tensor(b_np, device="cuda")
    x1 = torch.empty_like(b)
    its1, hist1 = G.pcg_solve(op, mg, b, x1, 1e-8, 200)
    x1 = x1.cpu().numpy()
    coords = lev.node_coords()
    m = n * p + 1
    plane = 3 * m * m
    comms = G.comm_group(world)
    res = [None] * world
    errs = []

    def rank_main(r):
        try:
            from paper_2408_12479_b200.slab import SlabPartition
            part = SlabPartition(n, n, n, p, world, r, faces=1)
            sl = slice(part.c0 * plane, (part.c1 + 1) * plane)
            slab = G.FeLevel(n, n, part.nz_local, p=p, coords=coords[sl], dirichlet_faces=part.local_faces,
                             z_offset=part.k0)
            sv = G.SlabSolver(slab, lev, r, world, comms[r], "inh", prm, degree=5, coarse_n=6, precision=32)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                du = torch.tensor(u0[sl], device="cuda")
                db = torch.tensor(b_np[sl], device="cuda")
                dx = torch.empty_like(db)
            sv.update_linearization(du, stream=st)
            its, hist = sv.pcg_solve(db, dx, 1e-8, 200, stream=st)
            st.synchronize()
            res[r] = (its, hist, dx.cpu().numpy(), sl)
            del sv
        except Exception as ex:  # noqa: BLE001
            errs.append(repr(ex))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in range(world):
        its, hist, x, sl = res[r]
        assert its == its1, (r, its, its1)
        assert np.array_equal(hist, hist1), r
        assert np.array_equal(x, x1[sl]), (r, np.abs(x - x1[sl]).max())


@pytest.mark.gpu
def test_cfg4_full_size_iterations_vs_reference():
    """BASELINE configs[4] (well-posed variant) at full size, 48^3 Q4, 21.6M
    DoFs: the device PCG + fp32 hp-MG (dense coarse solve) takes the
    reference's iteration count within +-1.  The reference run is its
    coarse-CG hierarchy (tests/golden/cfg4_full_cg.json, 35 iterations): its
    dense-LU run (cfg4_full.json, 40) carries the DenseLU pivoting defect
    (DESIGN.md §5)."""
    import json

    import torch
    from paper_2408_12479_b200 import emfgpu as G
    from paper_2408_12479_b200 import workloads as W
    with open(os.path.join(GOLD, "cfg4_full_cg.json")) as f:
        ref = json.load(f)
    w = W.cfg4()
    lev = w.level()
    assert lev.n_dofs == ref["ndofs"]
    op = G.ElasticOperator(lev, w.model, w.material(), "none", 64)
    op.update_linearization(np.zeros(lev.n_dofs))
    mg = G.MgHierarchy(lev, w.model, w.material(), degree=5, coarse_n=6, precision=32)
    mg.update_linearization(torch.zeros(lev.n_dofs, dtype=torch.float64, device="cuda"))
    b = torch.tensor(W.rhs(w), device="cuda")
    x = torch.empty_like(b)
    its, hist = G.pcg_solve(op, mg, b, x, 1e-8, 300)
    assert abs(its - ref["iterations"]) <= 1, (its, ref["iterations"])
    assert hist[-1] <= 1e-8
    # the residual histories agree to the preconditioner's round-off level
    k = min(len(hist), len(ref["history"])) - 1
    assert abs(np.log10(hist[k]) - np.log10(ref["history"][k])) < 0.3
    xn = float(torch.linalg.vector_norm(x))
    assert abs(xn - ref["norm_x"]) <= 1e-8 * ref["norm_x"], (xn, ref["norm_x"])  # measured 1.0e-10
