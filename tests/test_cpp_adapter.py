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
