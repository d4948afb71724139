"""CPU tests: the C restatement (oracle/emf_oracle.c) against the reference's
own outputs (golden fixtures from oracle/_ref) and the reference's known
constants.  The oracle must be BIT-EXACT to the reference; that is what makes
it a valid checker for the CUDA path."""
import os

import numpy as np
import pytest

from oracle import orcbind as O
from paper_2408_12479_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SMALL = ["cnh_p1_n4_curved", "cnh_p3_n2_curved", "inh_p2_n4_curved", "inh_p4_n2_affine",
         "fiber_p2_n2_curved", "fiber_p3_n2_affine"]
MODEL = {"cnh": "cnh", "inh": "inh", "fiber": "fiber"}


def _case(name):
    model, pp, nn, _ = name.split("_")
    return model, int(pp[1:]), int(nn[1:])


def test_inputs_reproduce_survey_known_answers():
    # ||u0||, ||v|| of cfg0 and cfg1 (reference generator).
    u0 = I.make_u0(8, 8, 8, 2)
    v = I.make_v(u0.size)
    assert np.isclose(np.linalg.norm(u0), 1.9603902670929043, rtol=1e-14)
    assert np.isclose(np.linalg.norm(v), 70.098428167379268, rtol=1e-14)
    assert v[:3].tolist() == pytest.approx([0.13312315034456179, 0.49156351452540226, 0.94200550717359244],
                                           rel=1e-15)


def test_splitmix64_matches_scalar_definition():
    # solver.hpp:209-219, written out with Python ints
    def sm(state):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return state, z ^ (z >> 31)
    s, ref = 7, []
    for _ in range(50):
        s, z = sm(s)
        ref.append(z)
    assert I.splitmix64_stream(7, 50).tolist() == ref


def test_oracle_cfg0_bitexact_vs_reference_golden():
    g = np.load(os.path.join(GOLD, "cfg0.npz"))
    u0 = I.make_u0(8, 8, 8, 2)
    v = I.make_v(u0.size)
    prm = np.array([1.0, 10.0, 1000.0, 2.0, 5.0, 3.62, 34.3, np.deg2rad(40), 1, 0, 0, 0, 1, 0, 0, 0, 1])
    for prec in (64, 32):
        op = O.OracleOperator(8, 8, 8, 2, model="cnh", params=prm, strategy="none", precision=prec)
        op.update_linearization(u0)
        y = op.apply(v.astype(op.dtype))
        assert np.array_equal(y, g[f"y{prec}"])
        d, nb = op.diagonal()
        assert np.array_equal(d, g[f"diag{prec}"]) and nb == 0
    # SURVEY §8(c) known answers
    assert np.isclose(np.linalg.norm(g["y64"]), 240.93765195277956, rtol=1e-14)
    node = (8 * 17 + 8) * 17 + 8
    assert g["y64"][3 * node:3 * node + 3] == pytest.approx(
        [-1.2687094083128543, 1.607692006743817, 0.13302019928913428], rel=1e-13)
    assert np.isclose(np.linalg.norm(g["diag64"]), 298.73218954820248, rtol=1e-14)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_small_bitexact_vs_reference_golden(name):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    model, p, n = _case(name)
    for prec in (64, 32):
        strategies = ("none",) if prec == 64 else ("none", "scalar", "tensor")
        for strat in strategies:
            op = O.OracleOperator(n, n, n, p, g["coords"], 1, model, g["params"], strat, prec)
            op.update_linearization(g["u0"])
            y = op.apply(g["v"].astype(op.dtype))
            assert np.array_equal(y, g[f"y{prec}_{strat}"]), (prec, strat)
        op = O.OracleOperator(n, n, n, p, g["coords"], 1, model, g["params"], "none", prec)
        op.update_linearization(g["u0"])
        assert np.array_equal(op.diagonal()[0], g[f"diag{prec}"])


def test_oracle_strategies_bitwise_equal_fp64():
    # acceptance.cpp:256-307: strategies agree (observed spread 0.0 in fp64)
    g = np.load(os.path.join(GOLD, "inh_p2_n4_curved.npz"))
    ys = []
    for strat in ("none", "scalar", "tensor"):
        op = O.OracleOperator(4, 4, 4, 2, g["coords"], 1, "inh", g["params"], strat, 64)
        op.update_linearization(g["u0"])
        ys.append(op.apply(g["v"]))
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])


def test_oracle_transfers_bitexact():
    g = np.load(os.path.join(GOLD, "transfers.npz"))
    dims = {"p42": ((2, 2, 2, 4), (2, 2, 2, 2)), "p21": ((2, 2, 2, 2), (2, 2, 2, 1)),
            "h21": ((4, 4, 4, 1), (2, 2, 2, 1))}
    for tag, (fd, cd) in dims.items():
        assert np.array_equal(O.transfer(fd, cd, "prolongate", g[f"{tag}_xc"]), g[f"{tag}_prolongate"])
        assert np.array_equal(O.transfer(fd, cd, "restrict", g[f"{tag}_xf"]), g[f"{tag}_restrict"])
        assert np.array_equal(O.transfer(fd, cd, "interpolate_down", g[f"{tag}_xf"]), g[f"{tag}_interpolate_down"])


def test_oracle_smoother_and_lanczos_bitexact():
    g = np.load(os.path.join(GOLD, "smoother.npz"))
    prm = np.array([1.0, 10.0, 50.0, 2.0, 5.0, 3.62, 34.3, np.deg2rad(40), 1, 0, 0, 0, 1, 0, 0, 0, 1])
    for prec in (64, 32):
        op = O.OracleOperator(4, 4, 4, 2, model="inh", params=prm, precision=prec)
        op.update_linearization(np.zeros(op.n))
        d, _ = op.diagonal()
        assert np.array_equal(d, g[f"diag{prec}"])
        lmin, lmax = op.estimate_eigenvalues(d)
        assert (lmin, lmax) == (float(g[f"lmin{prec}"]), float(g[f"lmax{prec}"]))
        x1 = op.chebyshev(d, lmax, g[f"b{prec}"], np.zeros(op.n), degree=5)
        assert np.array_equal(x1, g[f"x1_{prec}"])
        x2 = op.chebyshev(d, lmax, g[f"b{prec}"], x1, degree=5, zero_start=False)
        assert np.array_equal(x2, g[f"x2_{prec}"])


def test_oracle_structure_tensors_acceptance_constants():
    # acceptance.cpp:44-54: (H11, H22, H33) = (0.9168, 0.0759, 0.0073) +- 5e-5
    prm = np.array([62.1, 3042.9, 3084.3, 1.4, 22.1, 3.62, 34.3, 27.47 * np.pi / 180, 1, 0, 0, 0, 1, 0, 0, 0, 1])
    st = O.structure_tensors(prm)
    assert abs(st[18] - 0.9168) <= 5e-5 and abs(st[19] - 0.0759) <= 5e-5 and abs(st[20] - 0.0073) <= 5e-5


def test_oracle_nonpositive_jacobian_reports_first_point():
    op = O.OracleOperator(2, 2, 2, 2)
    u = np.zeros(op.n)
    u[3 * 40] = -5.0  # an interior node pushed through its neighbours
    with pytest.raises(O.OracleError) as ei:
        op.update_linearization(u)
    assert ei.value.code == 3 and "element=" in str(ei.value)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(O.HERE), "oracle", "_ref", "libemfref.so")),
                    reason="oracle/_ref not built")
def test_oracle_vs_live_reference_box_and_curved():
    from oracle import refbind as R
    L = R.RefLevel(1, 2, 3, 0.05, 1)
    prm = R.material_params(mu=1.0, lam=10.0, kappa=100.0)
    u0 = I.make_u0(4, 4, 4, 3, amp=0.05)
    v = I.make_v(L.ndofs, 3)
    for model in ("cnh", "inh", "fiber"):
        ref = R.RefOperator(L, model, prm, "tensor", 32)
        ref.update_linearization(u0)
        orc = O.OracleOperator(4, 4, 4, 3, L.coords(), 1, model, prm, "tensor", 32)
        orc.update_linearization(u0)
        assert np.array_equal(ref.apply(v.astype(np.float32)), orc.apply(v.astype(np.float32)))


def test_oracle_multigrid_and_pcg_bitexact():
    """The C V-cycle / coarse CG / outer PCG against the reference's own
    MgHierarchy<float> + PCG composed from reference primitives."""
    g = np.load(os.path.join(GOLD, "multigrid.npz"))
    prm = np.array([1.0, 10.0, 50.0, 2.0, 5.0, 3.62, 34.3, np.deg2rad(40), 1, 0, 0, 0, 1, 0, 0, 0, 1])
    for tag, (lmax, p) in {"q2": (2, 2), "q4": (2, 4)}.items():
        n = 1 << lmax
        mg = O.OracleMg(1, lmax, p, "inh", prm, degree=5)
        mg.update_linearization(np.zeros(g[f"{tag}_r"].size))
        assert np.array_equal(mg.precondition(g[f"{tag}_r"]), g[f"{tag}_z"])
        op = O.OracleOperator(n, n, n, p, model="inh", params=prm)
        op.update_linearization(np.zeros(op.n))
        x, its, hist = O.pcg_solve(op, mg, g[f"{tag}_b"], 1e-8, 200)
        assert its == int(g[f"{tag}_its"]) and np.array_equal(x, g[f"{tag}_x"])


def test_oracle_replicated_frames_equal_global_frame():
    """A per-qp frame field that replicates the global frame reproduces the
    reference's fibre operator bit for bit (SURVEY §8(c) gap 2 pin)."""
    g = np.load(os.path.join(GOLD, "fiber_p3_n2_affine.npz"))
    st = O.structure_tensors(g["params"])
    op = O.OracleOperator(2, 2, 2, 3, g["coords"], 1, "fiber", g["params"], "none", 64)
    nqp = 8 * 64
    h = np.repeat(st[:12][:, None], nqp, axis=1).ravel()
    m1 = np.repeat(st[12:18][:, None], nqp, axis=1).ravel()
    op.set_frames(h, m1)
    op.update_linearization(g["u0"])
    assert np.array_equal(op.apply(g["v"]), g["y64_none"])


NEWTON = [("inh_p2_n4_curved", "inh", 2, 2, 0.05, 0.2), ("cnh_p3_n2_curved", "cnh", 1, 3, 0.05, 0.1),
          ("fiber_p2_n4_affine", "fiber", 2, 2, 0.0, 0.3)]


@pytest.mark.parametrize("case", NEWTON, ids=[c[0] for c in NEWTON])
def test_oracle_residual_with_pressure_bitexact(case):
    """evaluate_residual with a +x face pressure at load scale 0.75 against the
    reference's own evaluate_residual (golden newton.npz)."""
    name, model, lmax, p, damp, pres = case
    g = np.load(os.path.join(GOLD, "newton.npz"))
    n = 1 << lmax
    coords = O.lattice_coords(n, n, n, p, map_kind=0, prm=(damp, 1.0))
    op = O.OracleOperator(n, n, n, p, coords, 1, model, g["params"], "none", 64)
    u = I.make_u0(n, n, n, p, amp=0.05)
    assert np.array_equal(op.residual(u, pres, 1, 0.75), g[f"{name}_r"])
    # the load alone: r(0) = -s * load on free rows; total force = p * area along -x
    load = op.pressure_load(pres, 1)
    assert np.isclose(load[0::3].sum(), -pres * 1.0, rtol=1e-12) or damp != 0.0


SPATIAL = [("cnh_p3_n2_curved", "cnh", 1, 3, 0.05), ("inh_p2_n4_curved", "inh", 2, 2, 0.05),
           ("fiber_p2_n2_curved", "fiber", 1, 2, 0.05), ("inh_p4_n2_affine", "inh", 1, 4, 0.0)]


@pytest.mark.parametrize("case", SPATIAL, ids=[c[0] for c in SPATIAL])
def test_oracle_spatial_domain_bitexact(case):
    """Spatial (Omega_t) formulation: apply (3 strategies x 2 precisions),
    diagonal and residual bit-exact to the reference (golden spatial.npz)."""
    name, model, lmax, p, damp = case
    g = np.load(os.path.join(GOLD, "spatial.npz"))
    n = 1 << lmax
    coords = O.lattice_coords(n, n, n, p, map_kind=0, prm=(damp, 1.0))
    u0 = I.make_u0(n, n, n, p, amp=0.05)
    v = I.make_v(u0.size)
    for prec in (64, 32):
        dt = np.float64 if prec == 64 else np.float32
        for strat in ("none", "scalar", "tensor"):
            op = O.OracleOperator(n, n, n, p, coords, 1, model, g["params"], strat, prec, domain=1)
            op.update_linearization(u0)
            assert np.array_equal(op.apply(v.astype(dt)), g[f"{name}_y{prec}_{strat}"]), (prec, strat)
        assert np.array_equal(op.diagonal()[0], g[f"{name}_diag{prec}"])
        assert np.array_equal(op.residual(u0.astype(dt)), g[f"{name}_r{prec}"])


def test_ledger_restatement_matches_reference():
    """paper_2408_12479_b200/ledger.py == the reference's cell_ledger
    (ledger.cpp:22-76) for every (model, domain, strategy): storage and
    traffic bytes per quadrature point (golden ledger.json from oracle/_ref)."""
    import json
    from paper_2408_12479_b200 import ledger as LG
    g = json.load(open(os.path.join(GOLD, "ledger.json")))
    for key, (storage, traffic) in g.items():
        model, dom, strat = key.split("/")
        d = "material" if dom == "0" else "spatial"
        assert LG.storage_bytes(model, d, strat) == storage, key
        assert LG.traffic_bytes(model, d, strat) == traffic, key
    # the acceptance table (acceptance.cpp:65-78), material scalar / tensor storage
    assert [LG.storage_bytes(m, "material", s) for m in ("cnh", "inh", "fiber") for s in ("scalar", "tensor")] == \
        [104, 320, 128, 344, 272, 488]


@pytest.mark.parametrize("n", [2, 4])
def test_oracle_shear_map_bitexact_vs_reference_golden(n):
    """cfg2's operator shape (shear map, iNH kappa/mu=1000, Q4): the C
    restatement is bit-exact to the reference on the same coordinates, and the
    workload generator reproduces the golden inputs."""
    from paper_2408_12479_b200 import workloads as W
    g = np.load(os.path.join(GOLD, "shear.npz"))
    tag = f"n{n}"
    w = W.cfg2(n=n)
    assert np.array_equal(w.u0(), g[f"{tag}_u0"]) and np.array_equal(w.v(), g[f"{tag}_v"])
    for prec in (64, 32):
        for strat in ("none", "scalar", "tensor"):
            op = O.OracleOperator(n, n, n, 4, g[f"{tag}_coords"], 1, "inh", g["params"], strat, prec)
            op.update_linearization(g[f"{tag}_u0"])
            y = op.apply(g[f"{tag}_v"].astype(op.dtype))
            assert np.array_equal(y, g[f"{tag}_y{prec}_{strat}"]), (prec, strat)
        op = O.OracleOperator(n, n, n, 4, g[f"{tag}_coords"], 1, "inh", g["params"], "none", prec)
        op.update_linearization(g[f"{tag}_u0"])
        d, nb = op.diagonal()
        assert np.array_equal(d, g[f"{tag}_diag{prec}"]) and nb == int(g[f"{tag}_diag{prec}_nbad"])


def test_cfg2_full_known_answers_recorded():
    """The full-size cfg2 known answers (make_golden.cfg2_full, the reference
    run here) agree with the verdict-quoted values and the generator."""
    import json
    from paper_2408_12479_b200 import workloads as W
    with open(os.path.join(GOLD, "cfg2_full.json")) as f:
        ref = json.load(f)
    assert ref["ndofs"] == 50923779
    assert "element=1 qpoint=46" in ref["literal"]["message"]
    assert np.isclose(ref["norm_y64"], 83211.64205114977, rtol=1e-15)
    assert abs(ref["norm_y32"] - ref["norm_y64"]) <= 1e-6 * ref["norm_y64"]
    w = W.cfg2()
    assert np.isclose(np.linalg.norm(w.u0()), ref["norm_u0"], rtol=1e-14)
