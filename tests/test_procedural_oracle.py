"""CPU: procedural couplings (dc/coupling.py:209-299). The oracle's blocked
product and the package's host-side ProceduralCoupling (entries, tiles,
validation) against golden vectors of the unmodified reference
(tests/golden/make_golden_procedural.py)."""

import hashlib

import numpy as np
import pytest

from oracle import dcising_oracle as orc
from paper_2509_01928_b200 import CouplingError, ProceduralCoupling, gen_procedural_sin

CASES = [(64, 100), (300, 100), (300, 7), (1500, 100)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("n,seed", CASES)
def test_host_tiles_match_reference(pgold, n, seed):
    g = pgold[f"p{n}_s{seed}"]
    J = gen_procedural_sin(n, seed=seed)
    assert J.n == n and J.seed == seed and J.value_kind == "real" and J.nnz_offdiag() == n * (n - 1)
    assert sha(J.block(0, n, 0, n)) == g["dense_sha"]
    if n == 64:
        A = pgold["arrays"]["p64_s100_dense"]
        assert np.array_equal(J.to_dense(), A)
        assert J.entry(3, 5) == A[3, 5] and J.entry(7, 7) == 0.0
    J.validate()


@pytest.mark.parametrize("n,seed", CASES)
def test_oracle_blocked_engine_matches_reference(pgold, n, seed):
    """Bit-exact: the oracle restates the reference's tile loop with the same numpy calls."""
    g, a = pgold[f"p{n}_s{seed}"], pgold["arrays"]
    op = orc.ProceduralOperator(n, seed)
    key = f"p{n}_s{seed}"
    assert np.array_equal(op.dot(a[f"{key}_v"]), a[f"{key}_Jv"])
    assert np.array_equal(op.abs_row_sums(), a[f"{key}_abs_row_sums"])
    assert op.offdiag_moments() == (g["s1"], g["s2"])


def test_oracle_params_and_doch_match_reference(pgold):
    g = pgold["params_p300"]
    op = orc.ProceduralOperator(300, 100)
    assert orc.derive_alpha_beta(op, eta=1.0) == (g["alpha"], g["beta"])
    r = pgold["runs_p300"]["doch_s0"]
    res = orc.run(op, g["alpha"], g["beta"], solver="doch", max_iters=300, seed=0)
    assert res["iterations"] == r["iterations"] and res["stop_reason"] == r["stop_reason"]
    assert res["energy"] == r["energy"]
    assert np.array_equal(np.asarray(res["h_values"]), np.asarray(r["h_values"]))


def test_procedural_constructor_errors():
    with pytest.raises(CouplingError):
        ProceduralCoupling(1)
    with pytest.raises(CouplingError):
        ProceduralCoupling(10, formula="cos_sum")
    with pytest.raises(ValueError):
        ProceduralCoupling(10).block(0, 11, 0, 3)
