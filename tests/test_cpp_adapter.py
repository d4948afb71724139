"""The C++ adapter (include/emfgpu/operator.hpp) compiled as a reference-style
driver: builds here (CPU), and on the GPU reproduces the reference's Newton
iteration count for the inh_p2_n4_curved pressure case (golden newton.npz)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2408_12479_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "adapter_newton")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "adapter_newton.cpp"), "-L", LIB, "-lemfgpu",
                    f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def test_adapter_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_adapter_newton_matches_reference(tmp_path):
    out = subprocess.run([_build(tmp_path)], check=True, capture_output=True, text=True).stdout.split()
    g = np.load(os.path.join(ROOT, "tests", "golden", "newton.npz"))
    assert out[0] == "newton"
    assert int(out[1]) == int(g["inh_p2_n4_curved_nit"])
    assert abs(int(out[2]) - int(g["inh_p2_n4_curved_lit"])) <= int(out[1])
    assert abs(float(out[4]) - np.linalg.norm(g["inh_p2_n4_curved_u"])) <= 1e-5 * np.linalg.norm(
        g["inh_p2_n4_curved_u"])


def _build_c(tmp_path):
    exe = str(tmp_path / "capi_apply")
    subprocess.run(["gcc", "-std=c11", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "capi_apply.c"), "-L", LIB, "-lemfgpu", "-lm",
                    f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def test_plain_c_client_compiles(tmp_path):
    """include/emfgpu.h is plain C: a C11 client builds against it."""
    assert os.path.exists(_build_c(tmp_path))


@pytest.mark.gpu
def test_plain_c_client_matches_python_binding(tmp_path):
    """The same calls from C and from the Python binding give the same bits."""
    out = subprocess.run([_build_c(tmp_path)], check=True, capture_output=True, text=True).stdout.split()
    vals = dict(t.split("=", 1) for t in out[1:] if "=" in t)
    assert int(vals["stale"]) == 5  # EMFGPU_ERR_STALE before linearization
    from paper_2408_12479_b200 import emfgpu as G
    lev = G.FeLevel(8, p=2)
    op = G.ElasticOperator(lev, "cnh", G.MaterialParams(mu=1.0, lam=10.0), "none", 64)
    n = lev.n_dofs
    mx = 17
    node = np.arange(n) // 3
    x, yy, z = (node % mx) / (mx - 1), ((node // mx) % mx) / (mx - 1), (node // (mx * mx)) / (mx - 1)
    u = np.where(node % mx == 0, 0.0, 0.05 * np.sin(3.14159265358979 * x) * np.sin(3.14159265358979 * yy) * z)
    v = np.sin(0.37 * np.arange(n))
    op.update_linearization(u)
    y = op.apply_tangent(v)
    d, nb = op.compute_diagonal()
    op.set_pressure(0.1, 1)
    r = op.evaluate_residual(u)
    assert float(vals["|y|"]) == pytest.approx(np.linalg.norm(y), rel=1e-14)
    assert float(vals["|diag|"]) == pytest.approx(np.linalg.norm(d), rel=1e-14)
    assert int(vals["nbad"]) == nb
    assert float(vals["|r|"]) == pytest.approx(np.linalg.norm(r), rel=1e-14)
