"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj by oracle/Makefile).  Run here (needs
/root/reference to build oracle/_ref); the fixtures travel to the GPU box.

The reference ships no golden vectors; these are outputs of the
reference itself on the seeded inputs of paper_2408_12479_b200/inputs.py.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refbind as R  # noqa: E402
from paper_2408_12479_b200 import inputs as I  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cfg0():
    """BASELINE configs[0]: 8^3 Q2 cNH mu=1 lambda=10, fp64 (and fp32), none."""
    L = R.RefLevel(1, 3, 2, 0.0, 1)
    u0 = I.make_u0(8, 8, 8, 2)
    v = I.make_v(L.ndofs)
    prm = R.material_params(mu=1.0, lam=10.0)
    out = {}  # u0/v are regenerated from the seeds by inputs.py
    for prec in (64, 32):
        op = R.RefOperator(L, "cnh", prm, "none", prec)
        op.update_linearization(u0)
        out[f"y{prec}"] = op.apply(v.astype(op.dtype))
        out[f"diag{prec}"] = op.diagonal()[0]
    np.savez_compressed(os.path.join(OUT, "cfg0.npz"), **out)
    print("cfg0 |y64| =", np.linalg.norm(out["y64"]), "|diag64| =", np.linalg.norm(out["diag64"]))


# small cases: (name, n, p, model, deform amplitude, u0 amplitude)
SMALL = [
    ("cnh_p1_n4_curved", 4, 1, "cnh", 0.05, 0.05),
    ("cnh_p3_n2_curved", 2, 3, "cnh", 0.05, 0.05),
    ("inh_p2_n4_curved", 4, 2, "inh", 0.05, 0.05),
    ("inh_p4_n2_affine", 2, 4, "inh", 0.0, 0.05),
    ("fiber_p2_n2_curved", 2, 2, "fiber", 0.05, 0.05),
    ("fiber_p3_n2_affine", 2, 3, "fiber", 0.0, 0.05),
]
KAPPA = 50.0


def small():
    for name, n, p, model, damp, uamp in SMALL:
        lev = {2: 1, 4: 2}[n]
        L = R.RefLevel(1, lev, p, damp, 1)
        prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
        u0 = I.make_u0(n, n, n, p, amp=uamp)
        v = I.make_v(L.ndofs)
        out = {"u0": u0, "v": v, "coords": L.coords(), "params": prm}
        for prec in (64, 32):
            for strat in ("none", "scalar", "tensor"):
                if prec == 64 and strat != "none":
                    continue  # fp64 strategies are bitwise identical in the reference
                op = R.RefOperator(L, model, prm, strat, prec)
                op.update_linearization(u0)
                out[f"y{prec}_{strat}"] = op.apply(v.astype(op.dtype))
            op = R.RefOperator(L, model, prm, "none", prec)
            op.update_linearization(u0)
            out[f"diag{prec}"] = op.diagonal()[0]
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        print(name, L.ndofs)


def transfers():
    """TransferOp (mesh.hpp:157-289): p-steps 4->2->1 and an h-step 4->2."""
    out = {}
    for tag, (fl, fp, cl, cp) in {"p42": (1, 4, 1, 2), "p21": (1, 2, 1, 1), "h21": (2, 1, 1, 1)}.items():
        F = R.RefLevel(1, fl, fp, 0.05, 1)
        Cc = R.RefLevel(1, cl, cp, 0.05, 1)
        xc = I.make_v(Cc.ndofs, 7)
        xf = I.make_v(F.ndofs, 8)
        out[f"{tag}_xc"] = xc
        out[f"{tag}_xf"] = xf
        out[f"{tag}_prolongate"] = R.transfer(F, Cc, "prolongate", xc)
        out[f"{tag}_restrict"] = R.transfer(F, Cc, "restrict", xf)
        out[f"{tag}_interpolate_down"] = R.transfer(F, Cc, "interpolate_down", xf)
    np.savez_compressed(os.path.join(OUT, "transfers.npz"), **out)


def smoother():
    """Lanczos estimate + Chebyshev smoothing (solver.hpp:262-361) on a 4^3 Q2
    iNH (kappa=50) level at u0 = 0 (SPD), fp32 and fp64."""
    L = R.RefLevel(1, 2, 2, 0.0, 1)
    prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
    u0 = np.zeros(L.ndofs)
    out = {}
    for prec in (64, 32):
        op = R.RefOperator(L, "inh", prm, "none", prec)
        op.update_linearization(u0)
        d = op.diagonal()[0]
        lmin, lmax = op.estimate_eigenvalues(d)
        b = I.make_v(L.ndofs, 9).astype(op.dtype)
        x1 = op.chebyshev(d, lmax, b, np.zeros_like(b), degree=5)
        x2 = op.chebyshev(d, lmax, b, x1, degree=5, zero_start=False)
        out.update({f"diag{prec}": d, f"lmin{prec}": lmin, f"lmax{prec}": lmax, f"b{prec}": b,
                    f"x1_{prec}": x1, f"x2_{prec}": x2})
    np.savez_compressed(os.path.join(OUT, "smoother.npz"), **out)


def multigrid():
    """MgHierarchy<float> V-cycle and an outer PCG (reference operator + the
    reference V-cycle, coarse Jacobi-PCG path) on the well-posed cfg4 variant
    (SURVEY §8(c') F4): iNH kappa/mu = 50, u0 = 0, affine cube."""
    out = {}
    prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
    for tag, (lmax, p) in {"q2": (2, 2), "q4": (2, 4)}.items():
        n = 1 << lmax
        L = R.RefLevel(1, lmax, p, 0.0, 1)
        u0 = np.zeros(L.ndofs)
        mg = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=0)
        mg.update_linearization(u0)
        r = I.make_v(L.ndofs, 11)
        out[f"{tag}_r"] = r
        out[f"{tag}_z"] = mg.precondition(r)
        op = R.RefOperator(L, "inh", prm, "none", 64)
        op.update_linearization(u0)
        b = I.make_v(L.ndofs, 12)
        b[I.dirichlet_mask(n, n, n, p, 1)] = 0.0
        x, its, hist = R.pcg_solve(op, mg, b, 1e-8, 200)
        out[f"{tag}_b"] = b
        out[f"{tag}_x"] = x
        out[f"{tag}_its"] = its
        out[f"{tag}_hist"] = hist
        print("mg", tag, mg.n_levels, "levels, pcg", its, "its")
        # the reference's default configuration: dense LU coarse solve (limit 2000)
        mgd = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=2000)
        mgd.update_linearization(u0)
        out[f"{tag}_dense_z"] = mgd.precondition(r)
        x, its, hist = R.pcg_solve(op, mgd, b, 1e-8, 200)
        out[f"{tag}_dense_x"] = x
        out[f"{tag}_dense_its"] = its
        print("mg dense", tag, "pcg", its, "its")
    np.savez_compressed(os.path.join(OUT, "multigrid.npz"), **out)


# residual + Newton cases: (name, model, lmax, p, deform amplitude, pressure)
NEWTON = [
    ("inh_p2_n4_curved", "inh", 2, 2, 0.05, 0.2),
    ("cnh_p3_n2_curved", "cnh", 1, 3, 0.05, 0.1),
    ("fiber_p2_n4_affine", "fiber", 2, 2, 0.0, 0.3),
]


def newton():
    """evaluate_residual with a +x face pressure (Loads, operator.hpp:23-32) at a
    seeded state, and the reference newton_solve (solver.hpp:603-656: FGMRES(30)
    + MgHierarchy<float>, coarse Jacobi-PCG) for one full load increment with
    the -x face clamped."""
    out = {}
    prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
    for name, model, lmax, p, damp, pres in NEWTON:
        n = 1 << lmax
        L = R.RefLevel(1, lmax, p, damp, 1)
        u = I.make_u0(n, n, n, p, amp=0.05)
        out[f"{name}_r"] = R.residual_with_pressure(L, model, prm, pres, 1, u, 0.75)
        x, nit, lit, res = R.newton_pressure(L, model, prm, pres, 1, 6, damp, 1, 0)
        out[f"{name}_u"] = x
        out[f"{name}_nit"] = nit
        out[f"{name}_lit"] = lit
        out[f"{name}_res"] = res
        print("newton", name, L.ndofs, "newton its", nit, "fgmres its", lit, "res", res)
    out["params"] = prm
    np.savez_compressed(os.path.join(OUT, "newton.npz"), **out)


# loads cases: (name, model, lmax, p, deform amplitude, pressure, face, body force, traction faces)
LOADS = [
    ("inh_p2_n4_curved", "inh", 2, 2, 0.05, 0.2, 1, 1, 0b101010),
    ("cnh_p3_n2_curved", "cnh", 1, 3, 0.05, 0.0, 1, 1, 0b000110),
    ("fiber_p4_n2_affine", "fiber", 1, 4, 0.0, 0.1, 4, 0, 0b100001),
]


def loads():
    """evaluate_residual with the full Loads struct (operator.hpp:23-32,
    880-1008): face pressure, body force B(X) and tractions h(X, N) on flagged
    faces (the fixture functions of oracle/ref_driver.cpp), at a seeded state."""
    out = {}
    prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
    for name, model, lmax, p, damp, pres, face, body, tf in LOADS:
        n = 1 << lmax
        L = R.RefLevel(1, lmax, p, damp, 1)
        u = I.make_u0(n, n, n, p, amp=0.05)
        out[f"{name}_r"] = R.residual_with_loads(L, model, prm, pres, face, body, tf, u, 0.5)
        print("loads", name, L.ndofs, np.linalg.norm(out[f"{name}_r"]))
    out["params"] = prm
    np.savez_compressed(os.path.join(OUT, "loads.npz"), **out)


SPATIAL = [("cnh_p3_n2_curved", "cnh", 1, 3, 0.05), ("inh_p2_n4_curved", "inh", 2, 2, 0.05),
           ("fiber_p2_n2_curved", "fiber", 1, 2, 0.05), ("inh_p4_n2_affine", "inh", 1, 4, 0.0)]


def spatial():
    """Spatial-domain (Omega_t) operator, Formulation{stable, spatial}
    (operator.hpp:506-519, constitutive.hpp:421-463): apply for every strategy
    and precision, diagonal, residual."""
    out = {}
    prm = R.material_params(mu=1.0, lam=10.0, kappa=KAPPA)
    for name, model, lmax, p, damp in SPATIAL:
        n = 1 << lmax
        L = R.RefLevel(1, lmax, p, damp, 1)
        u0 = I.make_u0(n, n, n, p, amp=0.05)
        v = I.make_v(L.ndofs)
        for prec in (64, 32):
            for strat in ("none", "scalar", "tensor"):
                op = R.RefOperator(L, model, prm, strat, prec, domain=1)
                op.update_linearization(u0)
                out[f"{name}_y{prec}_{strat}"] = op.apply(v.astype(op.dtype))
            out[f"{name}_diag{prec}"] = op.diagonal()[0]
            out[f"{name}_r{prec}"] = op.residual(u0.astype(op.dtype))
        print("spatial", name, L.ndofs)
    out["params"] = prm
    np.savez_compressed(os.path.join(OUT, "spatial.npz"), **out)


def stability():
    """The reference's forward-stability sweep (stability.cpp:163-251) on 40
    log-spaced scales in [1e-8, 1e2], 200 samples each, seed 42, default
    MaterialParams (material.hpp:36-47)."""
    scales = np.logspace(-8, 2, 40)
    prm = R.material_params(mu=62.1, lam=3042.9, kappa=3084.3, k1=1.4, k2=22.1, a=3.62, b=34.3,
                            phi=27.47 * 3.14159265358979323846 / 180.0)
    err, inv = R.stability_sweep(scales, 200, 42, prm)
    np.savez_compressed(os.path.join(OUT, "stability.npz"), scales=scales, err=err, inv=inv)
    print("stability", err.shape, int(inv.sum()))


def _shear_coords(L: "R.RefLevel", amp=0.1):
    """BASELINE cfg2 map x' = x + amp sin(2 pi y) e_x applied to the reference's
    own lattice (build_cube, mesh.cpp:138-160); SURVEY §8(c) gap 1: the level is
    rebuilt with these coordinates and J0 recomputed by the reference's sweeps."""
    c = L.coords().reshape(-1, 3).copy()
    c[:, 0] += amp * np.sin(2.0 * np.pi * c[:, 1])
    return c.reshape(-1)


def _inh_params(kappa):
    return R.material_params(mu=1.0, lam=10.0, kappa=kappa)


def shear():
    """cfg2-shaped operators at small size: shear map amplitude 0.1, iNH
    kappa/mu = 1000, Q4, u0 = 0.1 sin sin sin at pre-map coordinates plus the
    scaled noise 1e-3*8/n (workloads.cfg2); all reference strategies x
    fp64/fp32 plus the diagonal.  2^3 and 4^3 elements."""
    sys.path.insert(0, ROOT)
    from paper_2408_12479_b200 import workloads as W
    out = {}
    for n, lev in ((2, 1), (4, 2)):
        w = W.cfg2(n=n)
        L0 = R.RefLevel(1, lev, 4, 0.0, 1)
        coords = _shear_coords(L0)
        L = R.RefLevel(1, lev, 4, 0.0, 1, coords=coords)
        u0, v = w.u0(), w.v()
        prm = _inh_params(1000.0)
        tag = f"n{n}"
        out[f"{tag}_coords"] = coords
        out[f"{tag}_u0"] = u0
        out[f"{tag}_v"] = v
        for prec in (64, 32):
            for strat in ("none", "scalar", "tensor"):
                op = R.RefOperator(L, "inh", prm, strat, prec)
                op.update_linearization(u0)
                out[f"{tag}_y{prec}_{strat}"] = op.apply(v.astype(op.dtype))
            op = R.RefOperator(L, "inh", prm, "none", prec)
            op.update_linearization(u0)
            d, bad, nbad = op.diagonal()
            out[f"{tag}_diag{prec}"] = d
            out[f"{tag}_diag{prec}_nbad"] = nbad
            out[f"{tag}_diag{prec}_bad"] = bad
        print("shear", tag, L.ndofs, "|y64| =", np.linalg.norm(out[f"{tag}_y64_none"]))
    out["params"] = _inh_params(1000.0)
    np.savez_compressed(os.path.join(OUT, "shear.npz"), **out)


# sampled DoFs of the full-size known answers: seeded, plus the centre node
def _sample_dofs(ndofs, m, count=2048, seed=5):
    idx = np.unique((I.uniform01(seed, count) * ndofs).astype(np.int64))
    c = m // 2
    node = (c * m + c) * m + c
    return np.unique(np.concatenate([idx, 3 * node + np.arange(3)]))


def cfg2_full():
    """BASELINE configs[2] at full size (64^3 Q4, 50 923 779 DoFs) through the
    unmodified reference: the literal inputs' NonPositiveJacobian (first
    element, qpoint) and, for the scaled-noise variant, norms and sampled
    values of y = K(u0) v in fp64 and fp32 (tests/golden/cfg2_full.json)."""
    import json
    import time
    sys.path.insert(0, ROOT)
    from paper_2408_12479_b200 import workloads as W
    n, m = 64, 64 * 4 + 1
    L0 = R.RefLevel(1, 6, 4, 0.0, 1)
    coords = _shear_coords(L0)
    del L0
    L = R.RefLevel(1, 6, 4, 0.0, 1, coords=coords)
    del coords
    prm = _inh_params(1000.0)
    res = {"ndofs": int(L.ndofs), "threads": os.cpu_count()}
    op = R.RefOperator(L, "inh", prm, "none", 64)
    lit = W.cfg2(literal=True)
    try:
        op.update_linearization(lit.u0())
        res["literal"] = {"admissible": True}
    except R.RefError as ex:
        res["literal"] = {"admissible": False, "message": str(ex)}
    print("literal:", res["literal"])
    w = W.cfg2()
    u0, v = w.u0(), w.v()
    t0 = time.perf_counter()
    op.update_linearization(u0)
    res["linearize_s"] = time.perf_counter() - t0
    sd = _sample_dofs(L.ndofs, m)
    res["sample_dofs"] = sd.tolist()
    res["norm_u0"] = float(np.linalg.norm(u0))
    res["norm_v"] = float(np.linalg.norm(v))
    for prec in (64, 32):
        if prec == 32:
            op = R.RefOperator(L, "inh", prm, "none", 32)
            op.update_linearization(u0)
        t0 = time.perf_counter()
        y = op.apply(v.astype(op.dtype))
        res[f"apply{prec}_s"] = time.perf_counter() - t0
        res[f"norm_y{prec}"] = float(np.linalg.norm(y.astype(np.float64)))
        res[f"sum_y{prec}"] = float(np.sum(y.astype(np.float64)))
        res[f"y{prec}_sample"] = [float(t) for t in y[sd]]
        print(f"cfg2 fp{prec}: |y| = {res[f'norm_y{prec}']!r}  apply {res[f'apply{prec}_s']:.2f} s")
    with open(os.path.join(OUT, "cfg2_full.json"), "w") as f:
        json.dump(res, f, indent=1)


def cfg4_full():
    """BASELINE configs[4] at full size (48^3 Q4, 21 567 171 DoFs) through the
    reference: the literal inputs' NonPositiveJacobian, and on the well-posed
    variant (kappa/mu = 50, u0 = 0, affine) the fp64 PCG preconditioned by the
    reference's MgHierarchy<float> (Q4 -> Q2 -> Q1 -> 24^3 -> 12^3 -> 6^3,
    Chebyshev degree 5, dense coarse LU below 2000 DoFs): iterations, residual
    history and CPU times (tests/golden/cfg4_full.json)."""
    import json
    import time
    sys.path.insert(0, ROOT)
    from paper_2408_12479_b200 import workloads as W
    res = {"threads": os.cpu_count()}
    lit = W.cfg4(wellposed=False)
    L0 = R.RefLevel(6, 3, 4, 0.0, 1)
    Ls = R.RefLevel(6, 3, 4, 0.0, 1, coords=_shear_coords(L0))
    op = R.RefOperator(Ls, "inh", _inh_params(1000.0), "none", 64)
    try:
        op.update_linearization(lit.u0())
        res["literal"] = {"admissible": True}
    except R.RefError as ex:
        res["literal"] = {"admissible": False, "message": str(ex)}
    print("literal:", res["literal"], flush=True)
    del op, Ls
    w = W.cfg4()
    L = L0
    prm = _inh_params(50.0)
    res["ndofs"] = int(L.ndofs)
    t0 = time.perf_counter()
    op = R.RefOperator(L, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(L.ndofs))
    mg = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=2000)
    mg.update_linearization(np.zeros(L.ndofs))
    res["setup_s"] = time.perf_counter() - t0
    res["mg_levels"] = mg.n_levels
    print("setup", res["setup_s"], "levels", mg.n_levels, flush=True)
    b = W.rhs(w)
    t0 = time.perf_counter()
    x, its, hist = R.pcg_solve(op, mg, b, 1e-8, 300)
    res["solve_s"] = time.perf_counter() - t0
    res["iterations"] = int(its)
    res["history"] = [float(h) for h in hist]
    res["norm_x"] = float(np.linalg.norm(x))
    print("pcg", its, "its", res["solve_s"], "s", flush=True)
    with open(os.path.join(OUT, "cfg4_full.json"), "w") as f:
        json.dump(res, f, indent=1)


def coarse_lu():
    """Evidence for the reference's DenseLU pivoting defect (solver.hpp:55-78,
    DESIGN.md §5): on 3^3 and 6^3 Q4 (no h-levels: the coarse Q1 level has
    192 / 1029 DoFs) the reference's PCG with its dense coarse LU against the
    same hierarchy with its coarse Jacobi-PCG: iterations, histories, V-cycles
    (tests/golden/coarse_lu.npz)."""
    out = {}
    prm = R.material_params(mu=1.0, lam=10.0, kappa=50.0)
    for n in (3, 6):
        L = R.RefLevel(n, 0, 4, 0.0, 1)
        op = R.RefOperator(L, "inh", prm, "none", 64)
        op.update_linearization(np.zeros(L.ndofs))
        b = I.make_v(L.ndofs, 2)
        b[I.dirichlet_mask(n, n, n, 4, 1)] = 0.0
        r = I.make_v(L.ndofs, 11)
        out[f"n{n}_b"] = b
        out[f"n{n}_r"] = r
        for lim in (2000, 0):
            mg = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=lim)
            mg.update_linearization(np.zeros(L.ndofs))
            out[f"n{n}_lim{lim}_z"] = mg.precondition(r)
            x, its, hist = R.pcg_solve(op, mg, b, 1e-8, 300)
            out[f"n{n}_lim{lim}_its"] = its
            out[f"n{n}_lim{lim}_hist"] = hist
            print("coarse_lu", n, lim, its)
    np.savez_compressed(os.path.join(OUT, "coarse_lu.npz"), **out)


def cfg4_full_cg():
    """cfg4 at full size with the reference's coarse Jacobi-PCG
    (coarse_direct_limit = 0) instead of its dense LU: the reference's
    DenseLU::solve applies the row interchanges interleaved with the forward
    elimination although factor() swapped whole rows (solver.hpp:55-78), so
    its coarse solve is wrong whenever partial pivoting swaps rows (DESIGN.md
    §5); the CG coarse path is the reference's correct configuration to pin
    the iteration count against (tests/golden/cfg4_full_cg.json)."""
    import json
    import time
    sys.path.insert(0, ROOT)
    from paper_2408_12479_b200 import workloads as W
    w = W.cfg4()
    L = R.RefLevel(6, 3, 4, 0.0, 1)
    prm = _inh_params(50.0)
    res = {"threads": os.cpu_count(), "ndofs": int(L.ndofs), "coarse_direct_limit": 0}
    t0 = time.perf_counter()
    op = R.RefOperator(L, "inh", prm, "none", 64)
    op.update_linearization(np.zeros(L.ndofs))
    mg = R.RefMg(L, "inh", prm, degree=5, coarse_direct_limit=0)
    mg.update_linearization(np.zeros(L.ndofs))
    res["setup_s"] = time.perf_counter() - t0
    res["mg_levels"] = mg.n_levels
    print("setup", res["setup_s"], flush=True)
    b = W.rhs(w)
    t0 = time.perf_counter()
    x, its, hist = R.pcg_solve(op, mg, b, 1e-8, 300)
    res["solve_s"] = time.perf_counter() - t0
    res["iterations"] = int(its)
    res["history"] = [float(h) for h in hist]
    res["norm_x"] = float(np.linalg.norm(x))
    print("pcg", its, "its", res["solve_s"], "s", flush=True)
    with open(os.path.join(OUT, "cfg4_full_cg.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for f in sys.argv[1:]:
            globals()[f]()
        sys.exit(0)
    stability()
    spatial()
    newton()
    multigrid()
    cfg0()
    small()
    transfers()
    smoother()
    shear()
