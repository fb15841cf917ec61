"""CPU: the C-ABI library loads and exports every symbol include/dcx.h declares
(no compute calls: there is no GPU here)."""

import ctypes
import re

import pytest

from conftest import ROOT
from paper_2509_01928_b200 import _native


def header_symbols():
    text = (ROOT / "include" / "dcx.h").read_text()
    return sorted(set(re.findall(r"\b(dcx_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_symbol():
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.dcx_abi_version() == 1


def test_create_without_gpu_fails_cleanly():
    lib = _native.load()
    h = ctypes.c_void_p()
    rc = lib.dcx_create(0, ctypes.byref(h))
    if rc == 0:  # a GPU is present: nothing to check here
        lib.dcx_destroy(h)
        pytest.skip("GPU present")
    assert rc in (_native.DCX_E_CUDA, _native.DCX_E_INVALID)
    assert lib.dcx_last_error(None)


def test_no_cpu_fallback():
    """The product path raises instead of computing on the host without a device."""
    import numpy as np

    import paper_2509_01928_b200 as dc

    lib = _native.load()
    h = ctypes.c_void_p()
    if lib.dcx_create(0, ctypes.byref(h)) == 0:
        lib.dcx_destroy(h)
        pytest.skip("GPU present")
    J = dc.DenseCoupling(np.array([[0.0, -1.0], [-1.0, 0.0]]))
    with pytest.raises(RuntimeError):
        dc.doch_solve(dc.ProblemInstance(coupling=J), dc.SolverParams(alpha=1.0, beta=2.0))
