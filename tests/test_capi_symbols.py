"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol
declared in include/pf_b200.h (no compute calls without a GPU)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pf_b200.h")
GEN_HEADER = os.path.join(ROOT, "include", "pf_gen.h")


def declared_symbols(header=HEADER):
    text = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t)\s*\*?\s*(pf_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("pf_instance_create", "pf_solve", "pf_update_duals", "pf_project", "pf_solver_run",
                 "pf_comm_create", "pf_solver_trace"):
        assert need in syms
    gen = declared_symbols(GEN_HEADER)
    assert {"pf_ksp_run", "pf_ksp_sizes", "pf_ksp_export", "pf_ksp_free", "pf_validate_paths"} <= set(gen)
    assert not set(gen) & set(syms)


def test_generator_library_is_host_only():
    """libpf_gen.so exports pf_gen.h and links no CUDA runtime (input
    preparation never maps the solver or the GPU stack)."""
    from paper_2605_01748_b200 import build
    from paper_2605_01748_b200._lib import gen_lib
    L = gen_lib()
    for s in declared_symbols(GEN_HEADER):
        assert hasattr(L, s), s
    out = subprocess.run(["ldd", build.GEN_LIB], capture_output=True, text=True).stdout
    assert "cuda" not in out and "pf_b200" not in out, out


def test_library_exports_every_declared_symbol():
    from paper_2605_01748_b200 import _abi
    from paper_2605_01748_b200._lib import lib
    L = lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    # every ctypes signature we declare exists in the header too
    for s in _abi.SIGNATURES:
        assert s in declared_symbols(), s


def test_library_is_sm100a_only():
    from paper_2605_01748_b200 import build
    lib = build.LIB
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2605_01748_b200 as pf
    from paper_2605_01748_b200._lib import NativeError
    with pytest.raises(NativeError, match="CUDA"):
        pf.build_instance_raw(np.ones(1), np.ones(1), np.array([0, 1]), np.array([0, 1]), np.array([0]))
