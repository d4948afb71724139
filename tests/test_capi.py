"""CPU tests of the C-ABI boundary: the shared library loads, exports every
entry point include/emfgpu.h declares, and fails loudly without a GPU (no
CPU fallback).  No compute calls here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "emfgpu.h")
LIB = os.path.join(ROOT, "paper_2408_12479_b200", "lib", "libemfgpu.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(emfgpu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_operator_interface():
    syms = declared_symbols()
    for s in ("emfgpu_level_create", "emfgpu_op_create", "emfgpu_op_update_linearization", "emfgpu_op_apply",
              "emfgpu_op_compute_diagonal", "emfgpu_transfer_apply", "emfgpu_cheb_smooth",
              "emfgpu_op_estimate_eigenvalues"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2408_12479_b200 import emfgpu
    with pytest.raises(emfgpu.EmfGpuError) as ei:
        emfgpu.FeLevel(2, p=2)
    assert ei.value.code == 6


def test_null_arguments_are_rejected():
    from paper_2408_12479_b200 import emfgpu
    L = emfgpu.lib()
    assert L.emfgpu_level_create(None, None) == 4
    assert L.emfgpu_op_apply(None, None, None, None) == 4
    assert L.emfgpu_op_n_dofs(None) == 0
