"""GPU: the dense tcgen05 path (precision "f16tc") against the exact energy
kernel, the f32 path and the reference's K2000 quality numbers.

DOCH: the iterate is x = lambda_r s with s in f32, and each iteration sends only
its change through the tensor cores, x_{p+1} = x_p + lambda f16((T(x_p) - x_p) /
lambda) with T(x_p) from the exact-to-f32 running product (csrc/dcx_dense.cu),
so the first iterate sees x_0 rounded to f16 and later iterates converge like
the f32 path. ADOCH: the state itself as f16(x / lambda_r) each iteration (~1e-3
relative). Energies of spin vectors come from an exact +-1 x +-1 GEMM and must
match the integer energy kernel bit for bit; quality is judged on distributions
over the reference's own 1024 seeds (SURVEY.md §8c G-quality)."""

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import synth
from conftest import k2_W

pytestmark = pytest.mark.gpu

# f16 operand rounding (2^-11 relative per element) through one product and the
# cube root (ill-conditioned near 0): measured 2.24e-3 on K2000, identical to a
# float64 emulation of the same operand rounding (see test below).
TC_STATE_TOL = 5e-3   # one iteration; three iterations compound to ~6e-3 (checked at 1e-2)
EMU_TOL = 5e-4  # TC iterate vs a float64 emulation: f32 epilogue noise moves a few f16 roundings of the step by one ulp


def e4m3(v):
    """Round-to-nearest-even to OCP e4m3 (3 mantissa bits, subnormal step 2^-9, saturating at
    +-448), as cvt.rn.satfinite.e4m3x2.f32 does."""
    v = np.asarray(v, dtype=np.float64)
    a = np.minimum(np.abs(v), 448.0)
    ex = np.floor(np.log2(np.maximum(a, 2.0**-6)))
    q = np.exp2(ex - 3)
    return np.sign(v) * np.minimum(np.round(a / q) * q, 448.0)


def doch_first_iterate_emulation(J, x0, a, b, f8=True):
    """x_1 of the delta-operand DOCH kernel in float64: x_0 enters as its f16 rounding
    xq = lambda f16(x_0 / lambda) (the first delta is the state itself, an f16 product),
    T(xq) = cbrt((J + aI) xq / b), and the iterate moves by the rounded step: e4m3 with the
    first scale 2^6 (csrc/dcx_dense.cu f8_scale_exp), or f16 (f8=False)."""
    lam = np.sqrt(a / b)
    xq = (x0 / lam).astype(np.float16).astype(np.float64) * lam
    t = np.cbrt((J @ xq + a * xq) / b)
    d = (t - xq) / lam
    dq = e4m3(d * 64.0) / 64.0 if f8 else d.astype(np.float16).astype(np.float64)
    return xq + lam * dq


def k2_instance():
    return dc.ProblemInstance(coupling=dc.maxcut_to_ising(dc.DenseCoupling(k2_W(), validate=False)),
                              cut_offset=595.0)


def x0s(n, alpha, beta, seeds):
    return np.stack([dc.initial_state(n, alpha, beta, np.random.default_rng(s)) for s in seeds])


def rel2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_tc_first_iterate_equals_f16_operand_emulation(gold):
    g = gold["k2"]
    inst = k2_instance()
    a, b = g["alpha"], g["beta"]
    X0 = x0s(2000, a, b, range(128))
    tc = dc.solve_replicas(inst, "doch", a, b, X0, max_iters=1, precision="f16tc")
    J = -0.5 * k2_W()
    for x0, r in zip(X0, tc):
        # the e4m3 rounding of each step: >= 99 % of the elements equal the float64 emulation
        # to f32 precision; a near-tie may round one e4m3 step apart (2^-4 of that element's step)
        emu = doch_first_iterate_emulation(J, x0, a, b)
        assert np.mean(np.isclose(r.x, emu, rtol=1e-5, atol=0)) >= 0.99
        assert rel2(r.x, emu) <= 1e-2


def test_tc_first_iterate_f16_deltas_emulation(gold):
    g = gold["k2"]
    inst = k2_instance()
    a, b = g["alpha"], g["beta"]
    X0 = x0s(2000, a, b, range(128))
    tc = _run_with_env({"DCX_DENSE_F8": "0"}, lambda: dc.solve_replicas(inst, "doch", a, b, X0, max_iters=1,
                                                                      precision="f16tc"))
    J = -0.5 * k2_W()
    for x0, r in zip(X0, tc):
        assert rel2(r.x, doch_first_iterate_emulation(J, x0, a, b, f8=False)) <= EMU_TOL


def test_tc_first_iterates_track_f32(gold):
    """f16 deltas (DCX_DENSE_F8=0): the first iterates track the f32 CSR path within the
    f16 rounding of x_0 and of the steps. (The default e4m3 steps round each step to 3
    mantissa bits -- up to 2^-4 of a step -- and are pinned to their emulation instead.)"""
    g = gold["k2"]
    inst = k2_instance()
    X0 = x0s(2000, g["alpha"], g["beta"], range(128))
    for iters in (1, 3):
        tc = _run_with_env({"DCX_DENSE_F8": "0"}, lambda: dc.solve_replicas(
            inst, "doch", g["alpha"], g["beta"], X0, max_iters=iters, precision="f16tc"))
        f32 = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0, max_iters=iters, precision="f32")
        assert tc[0].path == "dense_tc"
        for a, b in zip(tc, f32):
            assert a.iterations == b.iterations == iters
            assert rel2(a.x, b.x) <= TC_STATE_TOL * (1 if iters == 1 else 4)


def test_tc_energies_exact():
    g_alpha, g_beta = 4.462132927392335, 89797103.04245317
    inst = k2_instance()
    X0 = x0s(2000, g_alpha, g_beta, range(256))
    res = dc.solve_replicas(inst, "doch", g_alpha, g_beta, X0, max_iters=60, precision="f16tc")
    spins = np.stack([r.spins for r in res])
    np.testing.assert_array_equal(dc.energies(inst.coupling, spins), [r.energy for r in res])
    for r in res[:8]:
        assert all(t.energy == t.energy for t in r.trace)  # recorded every iteration (stride 1)
        assert len(r.trace) == r.iterations + 1


@pytest.mark.parametrize("n", [300, 384, 640])
@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_tc_padding_columns_stay_finite(n, solver):
    """Sizes whose padding fills whole epilogue halves or spin tiles (n mod 128 <= 64): the
    e4m3 operand rows alias the iteration-0 f16 deltas, so every padding column must be
    written (zero) each iteration -- a stale byte read as e4m3 NaN poisoned every product of
    its replica row (0 x NaN). States and H stay finite, and runs are reproducible."""
    W = synth.dense_pm1(n, seed=3)
    inst = dc.ProblemInstance(coupling=dc.maxcut_to_ising(dc.DenseCoupling(W, validate=False)))
    a, b = 3.0, n ** 1.5 * 300.0
    X0 = x0s(n, a, b, range(32))
    r1 = dc.solve_replicas(inst, solver, a, b, X0, max_iters=60, precision="f16tc")
    assert r1[0].path == "dense_tc"
    for r in r1:
        assert np.all(np.isfinite(r.x)) and np.all(np.isfinite(np.asarray(r.h_values)))
    dc.solve_replicas(inst, solver, a, b, x0s(n, a, b, range(100, 132)), max_iters=60, precision="f16tc")
    r2 = dc.solve_replicas(inst, solver, a, b, X0, max_iters=60, precision="f16tc")
    for p_, q_ in zip(r1, r2):
        assert np.array_equal(p_.x, q_.x) and p_.energy == q_.energy and p_.iterations == q_.iterations


@pytest.mark.parametrize("n,R", [(130, 1), (250, 5), (513, 100), (1000, 300), (767, 257)])
def test_tc_shapes_sweep(n, R):
    """Ragged spin counts and replica counts (padding replicas and spins, one CTA or pairs):
    the first iterate matches the e4m3 emulation, every returned state and H is finite, and
    the returned spins carry their exact energies, for DOCH and ADOCH."""
    W = synth.dense_pm1(n, seed=n)
    Jd = -0.5 * W
    inst = dc.ProblemInstance(coupling=dc.maxcut_to_ising(dc.DenseCoupling(W, validate=False)))
    p = dc.derive_params(inst.coupling, eta=0.2)
    X0 = x0s(n, p.alpha, p.beta, range(R))
    one = dc.solve_replicas(inst, "doch", p.alpha, p.beta, X0, max_iters=1, precision="f16tc")
    assert one[0].path == "dense_tc"
    for x0, r in zip(X0[:8], one[:8]):
        emu = doch_first_iterate_emulation(Jd, x0, p.alpha, p.beta)
        assert np.mean(np.isclose(r.x, emu, rtol=1e-5, atol=0)) >= 0.99
    for solver in ("doch", "adoch"):
        rs = dc.solve_replicas(inst, solver, p.alpha, p.beta, X0, max_iters=120, precision="f16tc")
        E = dc.energies(inst.coupling, np.stack([r.spins for r in rs]))
        np.testing.assert_array_equal(E, [r.energy for r in rs])
        for r in rs:
            assert np.all(np.isfinite(r.x)) and np.all(np.isfinite(np.asarray(r.h_values)))


def test_tc_padding_ragged_sizes():
    rng = np.random.default_rng(4)
    n = 300
    a = np.triu(np.where(rng.random((n, n)) < 0.5, -1.0, 1.0), 1)
    J = dc.DenseCoupling(a + a.T, validate=False)
    inst = dc.ProblemInstance(coupling=J)
    p = dc.derive_params(J, eta=0.5)
    X0 = x0s(n, p.alpha, p.beta, range(200))
    tc = _run_with_env({"DCX_DENSE_F8": "0"},  # f16 deltas track f32 (e4m3 steps round to 2^-4 of a step)
                       lambda: dc.solve_replicas(inst, "doch", p.alpha, p.beta, X0, max_iters=2, precision="f16tc"))
    f32 = dc.solve_replicas(inst, "doch", p.alpha, p.beta, X0, max_iters=2, precision="f32")
    for a_, b_ in zip(tc, f32):
        assert rel2(a_.x, b_.x) <= 3 * TC_STATE_TOL  # two iterations at eta = 0.5
    full = dc.solve_replicas(inst, "doch", p.alpha, p.beta, X0, max_iters=300, precision="f16tc")
    np.testing.assert_array_equal(dc.energies(J, np.stack([r.spins for r in full])), [r.energy for r in full])


def k2_quality_gate(res, gk2, solver, stops=True, iter_rel=None):
    """SURVEY.md §8c G-quality on BASELINE configs[1], against the unmodified reference on
    the SAME 1024 seeds (tests/golden/golden_k2.npz):
      * stop reasons: the reference converges (step <= 1e-10, doch.py:220) on 1022 / 1024
        DOCH and 1024 / 1024 ADOCH seeds; the tensor-core path must converge as often
        (>= reference - 2 %), not run to max_iters;
      * iterations: mean within 4 standard errors (of the difference of two 1024-sample
        means) of the reference's, i.e. a solve does the reference's amount of work;
      * energies: not stochastically worse (one-sided Mann-Whitney U, p >= 1e-3) and the
        mean no worse than the reference's + 3 standard errors;
      * the tail: best energy at or below the reference's 3rd best over the same seeds, and
        the fraction of seeds reaching 0.99 x the reference's best cut (the TTS target,
        dc/bench.py:219-231) no lower than the reference's - 3 binomial standard errors.
    Per-seed trajectories are not compared: f16 operand rounding in the first steps sends
    a replica to a different local minimum, exactly as a change of summation order does."""
    from scipy.stats import mannwhitneyu

    A = gk2["arrays"]
    ref_e, ref_it, ref_st = A[f"{solver}_energy"], A[f"{solver}_iterations"], A[f"{solver}_stop"]
    e = np.array([r.energy for r in res])
    it = np.array([r.iterations for r in res])
    conv = np.array([r.stop_reason == "converged" for r in res])
    R = len(ref_e)
    assert len(res) == R
    if stops:
        assert conv.sum() >= (ref_st == 0).sum() - 0.02 * R, (conv.sum(), (ref_st == 0).sum())
        if iter_rel is None:
            se_it = np.sqrt(it.var(ddof=1) / R + ref_it.var(ddof=1) / R)
            assert abs(it.mean() - ref_it.mean()) <= 4 * se_it, (it.mean(), ref_it.mean(), se_it)
        else:
            assert abs(it.mean() - ref_it.mean()) <= iter_rel * ref_it.mean(), (it.mean(), ref_it.mean())
    assert mannwhitneyu(e, ref_e, alternative="greater").pvalue >= 1e-3
    assert e.mean() <= ref_e.mean() + 3 * ref_e.std(ddof=1) / np.sqrt(R), (e.mean(), ref_e.mean())
    assert e.min() <= np.sort(ref_e)[2], (e.min(), np.sort(ref_e)[:3])
    target = -(0.99 * (gk2["cut_offset"] - ref_e.min()) - gk2["cut_offset"])  # E at 0.99 x best cut
    f_ref, f = (ref_e <= target).mean(), (e <= target).mean()
    assert f >= f_ref - 3 * np.sqrt(f_ref * (1 - f_ref) / R), (f, f_ref)
    return dict(mean=e.mean(), best=e.min(), iters=it.mean(), converged=int(conv.sum()), reach=f)


def test_tc_k2000_quality_vs_reference_1024_seeds(gk2):
    """BASELINE configs[1]: 1024 DOCH replicas, seeds 0..1023, eta = 0.1, max_iters 1000,
    trace_stride 1 -- the reference's stop reasons, iteration counts and energy
    distribution on the same seeds."""
    inst = k2_instance()
    X0 = x0s(2000, gk2["alpha"], gk2["beta"], range(1024))
    res = dc.solve_replicas(inst, "doch", gk2["alpha"], gk2["beta"], X0, max_iters=1000, precision="f16tc")
    assert res[0].path == "dense_tc"
    k2_quality_gate(res, gk2, "doch")
    for r in res[:16]:
        assert dc.energy(inst.coupling, r.spins) == r.energy


def _run_with_env(env, fn):
    import os

    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_tc_operand_multicast_and_pair_variants_agree(gold):
    """The data-movement variants of the dense kernel (A tiles by pair TMA multicast
    in 4-CTA clusters, DCX_DENSE_MC=1; single-CTA tiles, DCX_DENSE_NC=1) compute
    the same products in the same order: identical results."""
    g = gold["k2"]
    inst = k2_instance()
    X0 = x0s(2000, g["alpha"], g["beta"], range(256))
    run = lambda: dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0, max_iters=40,  # noqa: E731
                                    precision="f16tc")
    base = run()
    mc = _run_with_env({"DCX_DENSE_MC": "1"}, run)
    nc1 = _run_with_env({"DCX_DENSE_NC": "1"}, run)
    for other in (mc, nc1):
        for a, b in zip(base, other):
            assert a.energy == b.energy and a.iterations == b.iterations
            assert np.array_equal(a.x, b.x)


@pytest.mark.parametrize("tn", ["64", "128"])
def test_tc_spin_tile_widths_agree(gold, tn):
    """64-wide spin tiles (the default when every replica group's CTA pairs fit the SMs, R <= 512
    at K2000) and 128-wide ones: the first iterate matches the e4m3 emulation, returned spins
    carry their exact energies, states stay finite, and a run resumed across launches equals
    one launch."""
    g = gold["k2"]
    inst = k2_instance()
    a, b = g["alpha"], g["beta"]
    X0 = x0s(2000, a, b, range(256))
    J = -0.5 * k2_W()
    one = _run_with_env({"DCX_DENSE_TN": tn},
                        lambda: dc.solve_replicas(inst, "doch", a, b, X0, max_iters=1, precision="f16tc"))
    for x0, r in zip(X0[:16], one[:16]):
        emu = doch_first_iterate_emulation(J, x0, a, b)
        assert np.mean(np.isclose(r.x, emu, rtol=1e-5, atol=0)) >= 0.99
    full = _run_with_env({"DCX_DENSE_TN": tn},
                         lambda: dc.solve_replicas(inst, "doch", a, b, X0, max_iters=200, precision="f16tc"))
    E = dc.energies(inst.coupling, np.stack([r.spins for r in full]))
    np.testing.assert_array_equal(E, [r.energy for r in full])
    assert all(np.all(np.isfinite(r.x)) for r in full)
    chunked = _run_with_env({"DCX_DENSE_TN": tn}, lambda: dc.solve_replicas(
        inst, "doch", a, b, X0, max_iters=200, precision="f16tc", chunk=37))
    for p_, q_ in zip(full, chunked):
        assert p_.iterations == q_.iterations and p_.energy == q_.energy and np.array_equal(p_.x, q_.x)


def test_tc_112_wide_spin_tiles(gold):
    """DCX_DENSE_TN=112 (18 spin tiles of 112 for n = 2000, stages straddling two tiles'
    operand flags): the first iterate matches the f16-operand emulation and returned
    spins carry their exact energies."""
    g = gold["k2"]
    inst = k2_instance()
    a, b = g["alpha"], g["beta"]
    X0 = x0s(2000, a, b, range(256))
    J = -0.5 * k2_W()
    one = _run_with_env({"DCX_DENSE_TN": "112"},
                        lambda: dc.solve_replicas(inst, "doch", a, b, X0, max_iters=1, precision="f16tc"))
    for x0, r in zip(X0, one):  # 112-wide tiles keep f16 deltas (the e4m3 path needs 16-byte aligned tiles)
        assert rel2(r.x, doch_first_iterate_emulation(J, x0, a, b, f8=False)) <= EMU_TOL
    res = _run_with_env({"DCX_DENSE_TN": "112"},
                        lambda: dc.solve_replicas(inst, "doch", a, b, X0, max_iters=60, precision="f16tc"))
    assert res[0].path == "dense_tc"
    for r in res[:32]:
        assert dc.energy(inst.coupling, r.spins) == r.energy


# ------------------------------------------------------------------ ADOCH on the tensor cores
def test_tc_adoch_e4m3_first_iterates(gold):
    """ADOCH with the default e4m3 deltas: its first iterate is the DOCH step (no
    extrapolation at k = 0, dc/solvers/doch.py:294-300) with the same e4m3 rounding, so it
    matches the e4m3 emulation like the DOCH kernel's; and the first three iterates equal
    the DOCH kernel's wherever every window rejected y (ADOCH then follows DOCH)."""
    g = gold["k2"]
    inst = k2_instance()
    a, b = g["alpha"], g["beta"]
    X0 = x0s(2000, a, b, range(128))
    J = -0.5 * k2_W()
    ad = dc.solve_replicas(inst, "adoch", a, b, X0, max_iters=1, precision="f16tc")
    do = dc.solve_replicas(inst, "doch", a, b, X0, max_iters=1, precision="f16tc")
    for x0, r, d in zip(X0, ad, do):
        emu = doch_first_iterate_emulation(J, x0, a, b)
        assert np.mean(np.isclose(r.x, emu, rtol=1e-5, atol=0)) >= 0.99
        assert rel2(r.x, emu) <= 1e-2
        assert np.array_equal(r.x, d.x)
        assert r.energy == dc.energy(inst.coupling, r.spins)


def test_tc_adoch_first_iterates_track_f32(gold):
    """ADOCH (economy window) in the persistent tensor-core kernel: the first iterates
    follow the f32 multipass ADOCH within the f16-operand tolerance, with the same
    accept decisions."""
    g = gold["k2"]
    inst = k2_instance()
    X0 = x0s(2000, g["alpha"], g["beta"], range(128))
    # the DOCH test's bounds (a replica whose windows reject every y follows DOCH bit for bit;
    # measured worst at three iterations 1.67e-2 for both solvers)
    for iters, tol in ((1, TC_STATE_TOL), (3, 4 * TC_STATE_TOL)):
        tc = _run_with_env({"DCX_DENSE_F8": "0"}, lambda: dc.solve_replicas(  # f16 deltas (see the DOCH test)
            inst, "adoch", g["alpha"], g["beta"], X0, max_iters=iters, precision="f16tc"))
        f32 = dc.solve_replicas(inst, "adoch", g["alpha"], g["beta"], X0, max_iters=iters, precision="f32")
        assert tc[0].path == "dense_tc"
        agree = 0
        for a, b in zip(tc, f32):
            assert a.iterations == b.iterations
            if a.accepted == b.accepted:
                agree += 1
                assert rel2(a.x, b.x) <= tol
            assert a.energy == dc.energy(inst.coupling, a.spins)
        assert agree >= len(tc) - 2  # a window test may resolve a near-tie differently at f16 operands


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_tc_resumed_launches_equal_one_launch(gold, solver):
    """A run split into launches of 7 iterations (each resumed launch restores the scaled
    state, the running product R and the sign product D2 from global memory into TMEM) is
    bit-identical to one launch."""
    g = gold["k2"]
    inst = k2_instance()
    X0 = x0s(2000, g["alpha"], g["beta"], range(256))
    one = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], X0, max_iters=40, precision="f16tc")
    chunked = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], X0, max_iters=40, precision="f16tc", chunk=7)
    for a, b in zip(one, chunked):
        assert a.iterations == b.iterations and a.stop_reason == b.stop_reason
        assert a.energy == b.energy and a.accepted == b.accepted
        assert np.array_equal(a.x, b.x)
        assert np.array_equal(a.spins, b.spins)
        assert [t.energy for t in a.trace] == [t.energy for t in b.trace]


def test_tc_adoch_k2000_quality_vs_reference_1024_seeds(gk2):
    """BASELINE configs[1] with ADOCH (economy window, q = 5): the reference's energy
    distribution on the same 1024 seeds and its stop reasons (converged as often, mean
    iterations within 15 %); energies exact for the returned spins; the accept log has one
    entry per iteration.

    ADOCH's Nesterov momentum amplifies the state's rounding noise by about 1 / (1 - c_k) ~
    k / 3 (numpy emulations of the exact update rule on seeds 0-4 converge only with an f64
    state, product and evaluation), so at f32 / tensor-core precision the extrapolation is
    dropped once the step falls below 2e-3 sqrt(alpha / beta) (RunCfg::momentum_floor) and
    the plain steps settle on the discrete fixed point. Without it (DCX_ADOCH_FLOOR=0) the
    run goes to max_iters; the f64 path keeps the reference's per-seed stop reasons
    (test_k2000_f64_matches_reference_seeds below)."""
    inst = k2_instance()
    X0 = x0s(2000, gk2["alpha"], gk2["beta"], range(1024))
    res = dc.solve_replicas(inst, "adoch", gk2["alpha"], gk2["beta"], X0, max_iters=1000, precision="f16tc")
    assert res[0].path == "dense_tc"
    k2_quality_gate(res, gk2, "adoch", stops=True, iter_rel=0.15)
    for r in res[:16]:
        assert dc.energy(inst.coupling, r.spins) == r.energy
        assert r.accepted[0] is True and len(r.accepted) == r.iterations  # as assemble_results builds it for every path


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_k2000_f64_matches_reference_seeds(gk2, solver):
    """G-fp64 on BASELINE configs[1]: the f64 path (the dense coupling as exact CSR, the
    multipass kernels) reproduces the unmodified reference's per-seed stop reason, best
    energy and (DOCH) iteration count on K2000 seeds 0..7 (tests/golden/golden_k2.npz)."""
    A = gk2["arrays"]
    inst = k2_instance()
    seeds = range(8)
    X0 = x0s(2000, gk2["alpha"], gk2["beta"], seeds)
    res = dc.solve_replicas(inst, solver, gk2["alpha"], gk2["beta"], X0, max_iters=1000, precision="f64")
    stop_name = {0: "converged", 1: "max_iters", 2: "time_budget"}
    diffs = []
    for s_, r in zip(seeds, res):
        assert r.stop_reason == stop_name[int(A[f"{solver}_stop"][s_])]
        assert r.energy == A[f"{solver}_energy"][s_]
        diffs.append(r.iterations - int(A[f"{solver}_iterations"][s_]))
    # ADOCH: the window test H(y) <= max(window) flips on last-bit H differences, which moves
    # the convergence point by a few iterations ("iterations within a band")
    if solver == "doch":
        assert diffs == [0] * len(diffs), diffs
    else:  # K2000 at f64: 6 of 8 seeds identical, the others within a few dozen iterations
        assert sum(d == 0 for d in diffs) >= len(diffs) // 2 and max(abs(d) for d in diffs) <= 60, diffs


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_tc_time_budget(gold, solver):
    """A time budget stops every replica of the tensor-core kernel with stop reason
    "time_budget" (dc/solvers/doch.py:221-223); the returned state is the last iterate
    and the spins carry their exact energies."""
    g = gold["k2"]
    inst = k2_instance()
    X0 = x0s(2000, g["alpha"], g["beta"], range(256))
    # 0.5 ms: about 30 iterations, well before any replica converges (>= 100 iterations)
    res = dc.solve_replicas(inst, solver, g["alpha"], g["beta"], X0, max_iters=10**6, precision="f16tc",
                            time_budget=0.0005)
    assert res[0].path == "dense_tc"
    for r in res[:16]:
        assert r.stop_reason == "time_budget"
        assert 0 < r.iterations < 10**6
        assert np.all(np.isfinite(r.x)) and np.any(r.x != 0)
        assert dc.energy(inst.coupling, r.spins) == r.energy
