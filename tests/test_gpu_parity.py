"""GPU parity: libdcx.so against the golden vectors of the unmodified reference
and against the numpy oracle on identical inputs and seeds.

Gates:
  G-int   energies of +-1 vectors bit-exact (integer / half-integer J);
  G-fp64  f64 mode: identical best energy / iterations / stop reason (DOCH),
          identical best energy / stop reason (ADOCH), states within 1e-12 rel;
  G-fp32  f32 mode: teacher-forced one-step ||dx||_2/||x||_2 <= 1e-5, free-running
          k <= 5 within 1e-5, identical signs for k <= 20;
  bitwise self-consistency of apply_T against the solver's own iterates
  (pkg/tests/test_doch.py:318-342).
"""

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from conftest import g1_csr, k2_W, sk_dense
from oracle import dcising_oracle as orc
from paper_2509_01928_b200 import synth

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5  # north_star: per-iteration continuous states within 1e-5 relative in fp32 mode


def g1_instance():
    v, c, o, co = g1_csr()
    return dc.ProblemInstance(coupling=dc.CsrCoupling(800, v, c, o, validate=False), cut_offset=co)


def rel2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------ G-int
def test_energy_bit_exact_g1_k2_families(gold, garr):
    inst = g1_instance()
    np.testing.assert_array_equal(dc.energies(inst.coupling, garr["g1_energy_spins"]),
                                  gold["g1"]["energy_of_spins"])
    J2 = dc.maxcut_to_ising(dc.DenseCoupling(k2_W(), validate=False))
    np.testing.assert_array_equal(dc.energies(J2, garr["k2_energy_spins"]), gold["k2"]["energy_of_spins"])
    for name, (v, c, o, *_r) in (("torus32", synth.torus(32)), ("er1e4", synth.erdos_renyi(10**4)),
                                 ("reg3_1e4", synth.random_regular3(10**4))):
        J = dc.CsrCoupling(len(o) - 1, v, c, o, validate=False)
        np.testing.assert_array_equal(dc.energies(J, garr[f"{name}_energy_spins"]),
                                      gold["families"][name]["energy_of_spins"])


def test_cut_value_exact(gold, garr):
    v, c, o, co = g1_csr()
    W = dc.CsrCoupling(800, -2.0 * v, c, o, validate=False)
    for s, cut in zip(garr["g1_energy_spins"], gold["g1"]["cut_of_spins"]):
        assert dc.cut_value(W, s) == cut


# ------------------------------------------------------------------ operator seam
def test_csr_matvec_bitwise_equals_scipy():
    """f64 SpMV uses scipy's csr_matvec summation order (dc/coupling.py:189-190)."""
    v, c, o, _ = g1_csr()
    J = dc.CsrCoupling(800, v, c, o, validate=False)
    x = np.random.default_rng(0).standard_normal(800)
    np.testing.assert_array_equal(dc.matvec(J, x), orc.Operator((v, c, o)).dot(x))
    vt, ct, ot, *_ = synth.erdos_renyi(10**4)
    Jt = dc.CsrCoupling(10**4, vt, ct, ot, validate=False)
    y = np.random.default_rng(1).standard_normal(10**4)
    np.testing.assert_array_equal(dc.matvec(Jt, y), orc.Operator((vt, ct, ot)).dot(y))


def test_dense_matvec_and_hamiltonian():
    A = sk_dense(100, 77)
    J = dc.DenseCoupling(A, validate=False)
    x = np.random.default_rng(2).standard_normal(100)
    np.testing.assert_allclose(dc.matvec(J, x), A @ x, rtol=1e-12, atol=1e-12)
    view = dc.HamiltonianView(J, 1.5, 4.0)
    assert dc.hamiltonian(view, x) == pytest.approx(orc.hamiltonian(orc.Operator(A), 1.5, 4.0, x), rel=1e-12)
    np.testing.assert_allclose(dc.apply_T(view, x), orc.apply_T(orc.Operator(A), 1.5, 4.0, x), rtol=1e-13)


# ------------------------------------------------------------------ G-fp64 on G1
@pytest.mark.parametrize("solver", ["doch", "adoch"])
@pytest.mark.parametrize("path", ["persistent", "multipass"])
def test_g1_f64_seed_runs_match_reference(gold, garr, solver, path):
    inst = g1_instance()
    g = gold["g1"]
    for seed in (0, 1):
        p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], eta=0.25, max_iters=1000, seed=seed)
        fn = dc.doch_solve if solver == "doch" else dc.adoch_solve
        r = fn(inst, p, record_states=True, path=path)
        ref = g["runs"][f"{solver}_s{seed}"]
        assert r.path == path
        assert r.stop_reason == ref["stop_reason"]
        assert r.energy == ref["energy"]
        if solver == "doch":
            assert r.iterations == ref["iterations"]
            assert [t.iteration for t in r.trace] == ref["trace_iter"]
            assert [t.energy for t in r.trace] == ref["trace_energy"]
            assert [t.event for t in r.trace] == ref["trace_event"]
            np.testing.assert_allclose(r.h_values, ref["h_values"], rtol=1e-9, atol=1e-12)
            np.testing.assert_allclose(r.x, garr[f"g1_{solver}_s{seed}_x"], rtol=1e-10, atol=1e-16)
        states = np.array(r.states[:21])
        ref_states = garr[f"g1_{solver}_s{seed}_states20"]
        for k in range(len(ref_states)):
            assert rel2(states[k], ref_states[k]) <= 1e-12, k
        assert dc.energy(inst.coupling, r.spins) == r.energy
        assert [t.cut_value for t in r.trace][:3] == ref["trace_cut"][:3]


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_g1_100_seeds_f64_batch(gold, solver):
    """All 100 seeds as one replica batch (one CTA per replica) vs the reference."""
    inst = g1_instance()
    g = gold["g1"]
    x0 = np.stack([dc.initial_state(800, g["alpha"], g["beta"], np.random.default_rng(s)) for s in range(100)])
    res = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], x0, max_iters=1000, precision="f64",
                            seeds=list(range(100)))
    rows = g[solver]
    same_e = sum(r.energy == row["energy"] for r, row in zip(res, rows))
    same_stop = sum(r.stop_reason == row["stop_reason"] for r, row in zip(res, rows))
    same_it = sum(r.iterations == row["iterations"] for r, row in zip(res, rows))
    if solver == "doch":
        assert same_e == 100 and same_stop == 100 and same_it == 100
    else:  # window test H(y) <= max(window) flips on last-bit differences
        assert same_e >= 95 and same_stop >= 95
    cuts = np.array([g1_csr()[3] - r.energy for r in res])
    ref_cuts = np.array([row["cut"] for row in rows])
    assert cuts.max() >= ref_cuts.max() - 1e-9 or cuts.mean() >= ref_cuts.mean() - 5.0


# ------------------------------------------------------------------ G-fp32
def test_g1_f32_teacher_forced_and_free_running(gold, garr):
    inst = g1_instance()
    g = gold["g1"]
    view = dc.HamiltonianView(inst.coupling, g["alpha"], g["beta"])
    ref_states = garr["g1_doch_s0_states20"]
    for k in range(20):
        tx = dc.apply_T(view, ref_states[k], precision="f32")
        assert rel2(tx, ref_states[k + 1]) <= FP32_TOL, k
    p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=20, seed=0)
    r = dc.doch_solve(inst, p, record_states=True, precision="f32")
    for k in range(21):
        if k <= 5:
            assert rel2(r.states[k], ref_states[k]) <= FP32_TOL, k
        np.testing.assert_array_equal(np.sign(r.states[k]), np.sign(ref_states[k]))


def test_g1_f32_quality_distribution(gold):
    inst = g1_instance()
    g = gold["g1"]
    x0 = np.stack([dc.initial_state(800, g["alpha"], g["beta"], np.random.default_rng(s)) for s in range(100)])
    res = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], x0, max_iters=1000, precision="f32")
    cuts = np.array([g1_csr()[3] - r.energy for r in res])
    ref = np.array([row["cut"] for row in g["doch"]])
    assert cuts.mean() >= ref.mean() - 3 * ref.std() / 10 and cuts.max() >= ref.max() - 60


# ------------------------------------------------------------------ small dense SK
@pytest.mark.parametrize("key", ["sk30_12", "sk40_17", "sk100_77"])
def test_sk_runs_vs_reference(gold, garr, key):
    g = gold["sk"][key]
    J = dc.DenseCoupling(sk_dense(g["n"], g["seed"]), validate=False)
    inst = dc.ProblemInstance(coupling=J)
    for solver in ("doch", "adoch"):
        fn = dc.doch_solve if solver == "doch" else dc.adoch_solve
        for s in range(3):
            p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=150, seed=s, lookback_q=2)
            r = fn(inst, p, record_states=s == 0)
            ref = g[f"{solver}_s{s}"]
            # real-valued J: the spin energy is a float sum in a different order
            assert r.energy == pytest.approx(ref["energy"], rel=1e-12) and r.stop_reason == ref["stop_reason"]
            if solver == "doch":
                assert r.iterations == ref["iterations"]
            if s == 0:
                rs = garr[f"{key}_{solver}_states"]
                for k in range(min(21, len(rs), len(r.states))):
                    assert rel2(r.states[k], rs[k]) <= 1e-11, (solver, k)


def test_antiferro_pair_converges_within_five(gold):
    """pkg/tests/test_doch.py:163-175 / acceptance :182-200."""
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(np.array([[0.0, -1.0], [-1.0, 0.0]])))
    ground = {(1.0, -1.0), (-1.0, 1.0)}
    for seed in range(20):
        r = dc.doch_solve(inst, dc.SolverParams(alpha=1.0, beta=2.0, max_iters=25, seed=seed), record_states=True)
        signs = [tuple(dc.spins_from(x)) for x in r.states]
        hit = next(k for k, sg in enumerate(signs) if sg in ground)
        assert hit <= 5 and all(sg == signs[hit] for sg in signs[hit:])
        ref = gold["pair"][str(seed)]
        assert r.iterations == ref["iterations"] and r.energy == pytest.approx(ref["energy"], abs=1e-15)


# ------------------------------------------------------------------ bitwise self-consistency
def test_first_adoch_iterate_equals_doch_bitwise(gold):
    g = gold["sk"]["sk30_12"]
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(sk_dense(30, 12), validate=False))
    p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=2, seed=7, lookback_q=50)
    a = dc.doch_solve(inst, p, record_states=True)
    b = dc.adoch_solve(inst, p, record_states=True)
    assert a.states[1].tobytes() == b.states[1].tobytes()


@pytest.mark.parametrize("path", ["persistent", "multipass"])
def test_adoch_exact_replay_bitwise(gold, path):
    """pkg/tests/test_doch.py:326-342: replay x_{k+1} = T(v_k) from the decisions."""
    g = gold["sk"]["sk40_17"]
    J = dc.DenseCoupling(sk_dense(40, 17), validate=False)
    inst = dc.ProblemInstance(coupling=J)
    p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=60, seed=3, lookback_q=2)
    r = dc.adoch_solve(inst, p, record_states=True, window_mode="exact", path=path)
    view = dc.HamiltonianView(J, p.alpha, p.beta)
    xs = r.states
    t_k = 1.0
    for k in range(r.iterations):
        t_next = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t_k * t_k))
        if k == 0:
            v = xs[0]
        else:
            y = xs[k] + ((t_k - 1.0) / t_next) * (xs[k] - xs[k - 1])
            v = y if r.accepted[k] else xs[k]
        assert dc.apply_T(view, v).tobytes() == xs[k + 1].tobytes(), k
        t_k = t_next


def test_economy_tracks_exact(gold):
    A = sk_dense(50, 23)
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(A, validate=False))
    g = gold["sk"]["sk50_23"]
    p = dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=80, seed=11)
    a = dc.adoch_solve(inst, p, window_mode="economy")
    b = dc.adoch_solve(inst, p, window_mode="exact")
    assert a.energy == pytest.approx(b.energy, rel=1e-9)
    np.testing.assert_array_equal(a.spins, b.spins)


# ------------------------------------------------------------------ stop reasons / trace contract
def test_time_budget_stops():
    A = synth.sk_gaussian(1000, 8)
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(A, validate=False))
    p = dc.SolverParams(alpha=50.0, beta=1000**1.5 * 900.0, max_iters=10**7, seed=0, time_budget=0.01)
    r = dc.doch_solve(inst, p)
    assert r.stop_reason == "time_budget"
    assert r.trace[-1].elapsed_s >= 0.01


def test_trace_best_nonincreasing_and_energy_of_spins(gold):
    g = gold["sk"]["sk40_17"]
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(sk_dense(40, 17), validate=False))
    r = dc.doch_solve(inst, dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=60, seed=1))
    bests = [t.best_energy for t in r.trace]
    assert all(b2 <= b1 for b1, b2 in zip(bests, bests[1:]))
    assert dc.energy(inst.coupling, r.spins) == pytest.approx(r.energy, abs=1e-12)


def test_zero_x0_rejected():
    inst = dc.ProblemInstance(coupling=dc.DenseCoupling(np.array([[0.0, -1.0], [-1.0, 0.0]])))
    with pytest.raises(ValueError):
        dc.doch_solve(inst, dc.SolverParams(alpha=1.0, beta=2.0), x0=np.zeros(2))


def test_callbacks_in_order():
    inst = g1_instance()
    seen = []
    p = dc.SolverParams(alpha=6.108031887826326, beta=884913.7454957356, max_iters=30, seed=0)
    r = dc.doch_solve(inst, p, callbacks=[seen.append])
    assert [t.iteration for t in seen] == [t.iteration for t in r.trace] == list(range(31))
    # the full records, running best included (TraceCollector, dc/solvers/common.py:70-91);
    # chunk=4 streams them across several device chunks
    seen = []
    r = dc.solve_replicas(inst, "doch", p.alpha, p.beta, dc.initial_state(800, p.alpha, p.beta,
                                                                      np.random.default_rng(0))[None, :],
                          max_iters=30, precision="f64", callbacks=[seen.append], chunk=4, path="multipass")[0]
    assert len(seen) == len(r.trace) == 31
    for a, b in zip(seen, r.trace):
        assert (a.iteration, a.energy, a.best_energy, a.cut_value, a.event) == \
            (b.iteration, b.energy, b.best_energy, b.cut_value, b.event)
    assert [t.best_energy for t in seen] == list(np.minimum.accumulate([t.energy for t in seen]))


# ------------------------------------------------------------------ sparse families (multipass)
@pytest.mark.parametrize("name", ["torus32", "er1e4", "reg3_1e4"])
def test_families_f64(gold, garr, name):
    g = gold["families"][name]
    make = {"torus32": lambda: synth.torus(32), "er1e4": lambda: synth.erdos_renyi(10**4),
            "reg3_1e4": lambda: synth.random_regular3(10**4)}[name]
    v, c, o, *_ = make()
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(len(o) - 1, v, c, o, validate=False),
                              cut_offset=g["cut_offset"])
    for solver in ("doch", "adoch"):
        fn = dc.doch_solve if solver == "doch" else dc.adoch_solve
        r = fn(inst, dc.SolverParams(alpha=g["alpha"], beta=g["beta"], max_iters=100, seed=0), record_states=True)
        ref = g[solver]
        assert r.energy == ref["energy"] and r.stop_reason == ref["stop_reason"]
        rs = garr[f"{name}_{solver}_states20"]
        for k in range(len(rs)):
            assert rel2(r.states[k], rs[k]) <= 1e-12, (solver, k)


def test_k2000_f64_seed0(gold):
    g = gold["k2"]
    J = dc.maxcut_to_ising(dc.DenseCoupling(k2_W(), validate=False))
    inst = dc.ProblemInstance(coupling=J)
    r = dc.doch_solve(inst, dc.SolverParams(alpha=g["alpha"], beta=g["beta"], eta=0.1, max_iters=1000, seed=0))
    ref = g["doch_s0"]
    assert r.energy == ref["energy"] and r.iterations == ref["iterations"] and r.stop_reason == ref["stop_reason"]


def test_replica_pass_staging_paths_agree():
    """pass_rv stages neighbour rows by TMA tile::gather4 (default) or per-lane
    cp.async (DCX_RV_TMA=0): the same values reach the same sums, results are
    bit-identical (f32, 256 replicas on a +-1 torus)."""
    import os

    v, c, o = synth.torus(32, seed=0)
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(1024, v, c, o, validate=False))
    X0 = np.stack([dc.initial_state(1024, 4.0, 8.0e4, np.random.default_rng(s)) for s in range(256)])
    run = lambda: dc.solve_replicas(inst, "doch", 4.0, 8.0e4, X0, max_iters=50, precision="f32",  # noqa: E731
                                    path="multipass")
    a = run()
    os.environ["DCX_RV_TMA"] = "0"
    try:
        b = run()
    finally:
        os.environ.pop("DCX_RV_TMA", None)
    for ra, rb in zip(a, b):
        assert ra.energy == rb.energy and ra.iterations == rb.iterations
        assert np.array_equal(ra.x, rb.x)
