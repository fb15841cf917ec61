"""GPU: procedural couplings J_ij = sin(i*j + seed) generated on the device
(dcx_proc.cu) against the unmodified reference's blocked engine
(tests/golden/make_golden_procedural.py).

Tolerances: the device sums each row in lane order and regenerates sin from an
exact integer angle reduction plus a rotation recurrence, the reference sums
b x b tile products in column-block order with np.sin per entry. f64 products
agree to ~1e-15 relative per row (gate 1e-12); f32 to ~1e-6 (gate 2e-5,
north_star's 1e-5 class). DOCH runs in f64 must reproduce the reference's
iteration count, stop reason and best energy, and its states to 1e-9.
"""

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import gen_procedural_sin

pytestmark = pytest.mark.gpu

CASES = [(64, 100), (300, 100), (300, 7), (1500, 100)]


def rel_inf(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))


@pytest.mark.parametrize("n,seed", CASES)
def test_matvec_matches_reference(pgold, n, seed):
    a = pgold["arrays"]
    key = f"p{n}_s{seed}"
    J = gen_procedural_sin(n, seed=seed)
    y = dc.matvec(J, a[f"{key}_v"])
    assert rel_inf(y, a[f"{key}_Jv"]) < 1e-12
    from paper_2509_01928_b200.coupling import device_context

    y32 = device_context(J).matvec(a[f"{key}_v"][None, :], precision="f32")[0]
    assert rel_inf(y32, a[f"{key}_Jv"]) < 2e-5


@pytest.mark.parametrize("n,seed", CASES)
def test_row_statistics_match_reference(pgold, n, seed):
    g, a = pgold[f"p{n}_s{seed}"], pgold["arrays"]
    J = gen_procedural_sin(n, seed=seed)
    assert rel_inf(J.abs_row_sums(), a[f"p{n}_s{seed}_abs_row_sums"]) < 1e-12
    s1, s2 = J.offdiag_moments()
    assert abs(s1 - g["s1"]) < 1e-10 * g["s2"]  # s1 is a cancelling sum: absolute gate on the scale n^2/2
    assert abs(s2 - g["s2"]) < 1e-12 * g["s2"]


def test_derive_params_and_energy_match_reference(pgold):
    g = pgold["params_p300"]
    J = gen_procedural_sin(300, seed=100)
    p = dc.derive_params(J, eta=1.0)  # auto = Wigner for procedural couplings
    assert p.alpha == pytest.approx(g["alpha"], rel=1e-12) and p.beta == pytest.approx(g["beta"], rel=1e-12)
    pp = dc.derive_params(J, eta=1.0, method="power_iteration", tol=1e-10)
    assert pp.alpha == pytest.approx(g["alpha_power"], rel=1e-8)
    S = pgold["arrays"]["p300_energy_spins"]
    E = dc.energies(J, S)
    assert np.allclose(E, g["energy_of_spins"], rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_f64_solves_match_reference(pgold, solver):
    g = pgold["params_p300"]
    inst = dc.ProblemInstance(coupling=gen_procedural_sin(300, seed=100))
    fn = dc.doch_solve if solver == "doch" else dc.adoch_solve
    for s in range(3):
        ref = pgold["runs_p300"][f"{solver}_s{s}"]
        q = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=300, seed=s)
        r = fn(inst, q, record_states=s == 0, precision="f64")
        assert r.stop_reason == ref["stop_reason"]
        assert r.energy == pytest.approx(ref["energy"], rel=1e-12)
        if solver == "doch":
            assert r.iterations == ref["iterations"]
            k = min(len(r.h_values), len(ref["h_values"]))
            assert np.allclose(r.h_values[:k], ref["h_values"][:k], rtol=1e-9, atol=0)
        else:  # the window test flips on last-bit differences
            assert abs(r.iterations - ref["iterations"]) <= 5
        if s == 0:
            st = pgold["arrays"][f"p300_{solver}_s0_states20"]
            assert np.allclose(np.array(r.states[:21]), st, rtol=0, atol=1e-9 * np.abs(st).max())


def test_two_tile_instance_matches_reference(pgold):
    """n = 1500: the reference sums two column tiles per row block."""
    g = pgold["runs_p1500"]
    q = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=200, seed=0)
    J = gen_procedural_sin(1500, seed=100)
    p = dc.derive_params(J, eta=1.0)
    assert p.alpha == pytest.approx(g["alpha"], rel=1e-12)
    r = dc.doch_solve(dc.ProblemInstance(coupling=J), q, record_states=True, precision="f64")
    ref = g["doch_s0"]
    assert (r.iterations, r.stop_reason) == (ref["iterations"], ref["stop_reason"])
    assert r.energy == pytest.approx(ref["energy"], rel=1e-12)
    st = pgold["arrays"]["p1500_doch_s0_states20"]
    assert np.allclose(np.array(r.states[:21]), st, rtol=0, atol=1e-9 * np.abs(st).max())


def test_replica_batch_equals_single_runs(pgold):
    """R = 6 (replica chunks of 4, a partial last chunk) reproduces the R = 1 runs."""
    g = pgold["params_p300"]
    inst = dc.ProblemInstance(coupling=gen_procedural_sin(300, seed=100))
    X0 = np.stack([dc.initial_state(300, g["alpha"], g["beta"], np.random.default_rng(s)) for s in range(6)])
    batch = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0, max_iters=300, precision="f64")
    for s in range(3):
        ref = pgold["runs_p300"][f"doch_s{s}"]
        assert (batch[s].iterations, batch[s].stop_reason) == (ref["iterations"], ref["stop_reason"])
        assert batch[s].energy == pytest.approx(ref["energy"], rel=1e-12)
    for s in range(6):
        one = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0[s:s + 1], max_iters=300, precision="f64")[0]
        assert one.iterations == batch[s].iterations and np.array_equal(one.x, batch[s].x)


def test_f32_first_iterations(pgold):
    g = pgold["params_p300"]
    inst = dc.ProblemInstance(coupling=gen_procedural_sin(300, seed=100))
    q = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=300, seed=0)
    r = dc.doch_solve(inst, q, record_states=True, precision="f32")
    st = pgold["arrays"]["p300_doch_s0_states20"]
    for k in range(1, 6):
        assert np.linalg.norm(np.asarray(r.states[k]) - st[k]) / np.linalg.norm(st[k]) < 1e-5
    assert np.array_equal(np.sign(np.asarray(r.states[20])), np.sign(st[20]))
    ref = pgold["runs_p300"]["doch_s0"]
    assert r.stop_reason == ref["stop_reason"] and abs(r.iterations - ref["iterations"]) <= 5
    assert r.energy == pytest.approx(ref["energy"], rel=1e-6)
