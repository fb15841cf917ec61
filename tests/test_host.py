"""CPU: host-side logic (parameter validation, coupling invariants, CSR
encoding choices) that needs no device."""

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import synth


def test_solver_params_validation():  # dc/spectral.py:41-49
    with pytest.raises(ValueError):
        dc.SolverParams(alpha=0.0, beta=1.0)
    with pytest.raises(ValueError):
        dc.SolverParams(alpha=1.0, beta=-1.0)
    with pytest.raises(ValueError):
        dc.SolverParams(alpha=1.0, beta=1.0, eta=2.5)
    with pytest.raises(ValueError):
        dc.SolverParams(alpha=1.0, beta=1.0, lookback_q=0)


def test_dense_validation():
    with pytest.raises(dc.CouplingError):
        dc.DenseCoupling(np.array([[1.0, 0.0], [0.0, 0.0]]))
    with pytest.raises(dc.CouplingError):
        dc.DenseCoupling(np.array([[0.0, 1.0], [2.0, 0.0]]))


def test_csr_validation_vectorised():
    v, c, o, _ = synth.g1_shape()
    J = dc.CsrCoupling(800, v, c, o)  # valid
    assert J.nnz == 38352
    bad = np.array(c)
    bad[0], bad[1] = bad[1], bad[0]
    with pytest.raises(dc.CouplingError):
        dc.CsrCoupling(800, v, bad, o)
    vv = np.array(v)
    vv[0] = -1.0
    with pytest.raises(dc.CouplingError):
        dc.CsrCoupling(800, vv, c, o)


def test_abs_row_sums_and_moments():
    v, c, o = synth.torus(8)
    J = dc.CsrCoupling(64, v, c, o)
    np.testing.assert_array_equal(J.abs_row_sums(), np.abs(J.to_dense()).sum(axis=1))
    assert J.offdiag_moments()[1] == float((J.to_dense() ** 2).sum())


def test_initial_state_matches_numpy_stream():
    x = dc.initial_state(50, 2.0, 8.0, np.random.default_rng(3))
    y = np.random.default_rng(3).uniform(-0.5, 0.5, size=50)
    np.testing.assert_array_equal(x, y)


def test_solve_rejects_out_of_scope_solver():
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(np.zeros((2, 2))))
    with pytest.raises(ValueError):
        dc.solve(inst, "sa")
