"""GPU parity at BASELINE.json's full sizes, through size-independent properties.

The oracle runs the small instances of test_gpu_parity.py in seconds; at the
BASELINE sizes (T6 = 10^6-spin torus x 256 replicas, E7 = 10^7-spin
Erdos-Renyi, configs[2] and [3]) the CPU cannot replay whole solves, so these
tests check what holds at any size:

* one teacher-forced step: x_1 = cbrt((J + aI) x_0 / b) (dc/solvers/doch.py:90-91,
  :199) from the same x_0, against scipy's f64 product; ||dx||_2/||x||_2 <= 1e-5
  (the north_star fp32 tolerance);
* G-int: the reported best energy equals E(spins) = -1/2 s.Js of the returned
  spins (dc/solvers/common.py:66-75), computed independently in f64 on the host
  (exact: J is +-1 or -1/2), and cut = cut_offset - E (dc/model.py:45-76);
* DOCH boundedness ||x_k||_inf <= max(1, ||x_0||_inf) (pkg/tests/test_doch.py:209-227);
* the first ADOCH iterate equals the first DOCH iterate bitwise (no extrapolation
  at k = 0, dc/solvers/doch.py:294-300);
* h_values has iterations + 1 entries and the best-energy trace never increases.

Plus the G-fp32 free-running gate: the oracle (numpy/scipy f64,
oracle/dcising_oracle.py) runs the first five DOCH iterations from the same x_0
at full E7 size (~3 s per iteration) and on 8 T6 replicas;
||x_k - x_k^ref||_2 / ||x_k^ref||_2 <= 1e-5 for k <= 5. R8 (10^8 spins) gets the
one-step and G-int checks (its scipy product takes ~10 s). The E7 / R8 graphs are
built with their deduplicating sorts on the GPU (synth._maxcut_unit(device=...)),
checked equal to the numpy build here.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2509_01928_b200 as dc
from oracle import dcising_oracle as orc
from paper_2509_01928_b200 import synth

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


def _check_common(J, rs, X0, cut_offset=None, doch=True):
    for r, x0 in zip(rs, X0):
        s = np.asarray(r.spins, dtype=np.float64)
        assert np.all(np.abs(s) == 1.0)
        e = -0.5 * float(s @ (J @ s))
        assert r.energy == e
        if cut_offset is not None:
            assert all(t.cut_value == cut_offset - t.energy for t in r.trace)
        assert len(r.h_values) == r.iterations + 1
        best = [t.best_energy for t in r.trace]
        assert all(b1 <= b0 for b0, b1 in zip(best, best[1:]))
        if doch:
            assert float(np.abs(r.x).max()) <= max(1.0, float(np.abs(x0).max()))


def _one_step(J, alpha, beta, X0, rs):
    X32 = X0.astype(np.float32).astype(np.float64)  # the f32 path starts from x_0 rounded to f32
    AX = (J @ X32.T).T + alpha * X32
    X1 = np.cbrt(AX / beta)
    for r, x1 in zip(rs, X1):
        assert r.iterations == 1
        d = float(np.linalg.norm(np.asarray(r.x, dtype=np.float64) - x1) / np.linalg.norm(x1))
        assert d <= FP32_TOL, d


@pytest.fixture(scope="module")
def t6():
    v, c, o = synth.torus(1000, seed=0)
    n = 10**6
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False))
    J = sp.csr_matrix((v, c, o), shape=(n, n))
    X0 = np.stack([dc.initial_state(n, 4.0, 8.0e9, np.random.default_rng(s)) for s in range(256)])
    return inst, J, 4.0, 8.0e9, X0


def test_t6_full_size_properties(t6):
    inst, J, alpha, beta, X0 = t6
    run = lambda solver, iters: dc.solve_replicas(inst, solver, alpha, beta, X0, max_iters=iters,  # noqa: E731
                                                  precision="f32", path="multipass")
    d1 = run("doch", 1)
    _one_step(J, alpha, beta, X0[:16], d1[:16])
    a1 = run("adoch", 1)
    for rd, ra in zip(d1, a1):
        assert np.array_equal(rd.x, ra.x)
    sub = list(range(0, 256, 17))  # 16 replicas spread over both replica chunks
    d = run("doch", 30)
    _check_common(J, [d[i] for i in sub], X0[sub])
    a = run("adoch", 30)
    _check_common(J, [a[i] for i in sub], X0[sub], doch=False)
    assert all(r.accepted[0] for r in a)


def _free_running(J_arrays, alpha, beta, X0, rs, k_max=5):
    """G-fp32 free-running: the oracle's first k_max iterates from the same x_0 (f64)
    against the device's recorded f32 states."""
    op = orc.Operator(J_arrays)
    for x0, r in zip(X0, rs):
        ref = orc.run(op, alpha, beta, solver="doch", max_iters=k_max, x0=x0, record_states=True)["states"]
        assert len(r.states) == k_max + 1
        for k in range(1, k_max + 1):
            d = float(np.linalg.norm(np.asarray(r.states[k], np.float64) - ref[k]) / np.linalg.norm(ref[k]))
            assert d <= FP32_TOL, (k, d)


def test_device_instance_build_matches_numpy():
    """synth's GPU build of the E7 / R8 recipes equals the numpy build byte for byte."""
    for make in (lambda d: synth.erdos_renyi(200_000, 8, seed=0, device=d),
                 lambda d: synth.random_regular3(300_000, seed=0, device=d)):
        a, b = make(None), make(0)
        assert a[3] == b[3]
        for x, y in zip(a[:3], b[:3]):
            assert x.dtype == y.dtype and np.array_equal(x, y)


def test_t6_free_running_first_iterates(t6):
    inst, J, alpha, beta, X0 = t6
    pick = list(range(0, 256, 37))[:8]  # 8 of the 256 replicas (record_states of all 256 would be 6 GB)
    rs = dc.solve_replicas(inst, "doch", alpha, beta, X0[pick], max_iters=5, precision="f32", path="multipass",
                           record_states=True)
    _free_running((J.data, J.indices.astype(np.int64), J.indptr.astype(np.int64)), alpha, beta, X0[pick], rs)


@pytest.fixture(scope="module")
def e7():
    n = 10**7
    v, c, o, co = synth.erdos_renyi(n, 8, seed=0, device=0)
    return n, v, c, o, co


def test_e7_free_running_first_iterates(e7):
    n, v, c, o, co = e7
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
    alpha, beta = 2.828, 5.005e11
    X0 = dc.initial_state(n, alpha, beta, np.random.default_rng(0))[None, :]
    r = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=5, precision="f32", path="multipass",
                          record_states=True)
    _free_running((v, c, o), alpha, beta, X0, r)


def test_r8_full_size_one_step_and_energies():
    """configs[4] on one GPU: 10^8-spin random 3-regular MaxCut."""
    n = 10**8
    v, c, o, co = synth.random_regular3(n, seed=0, device=0)
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
    J = sp.csr_matrix((v, c, o), shape=(n, n))
    alpha, beta = 1.732, 3.232e12  # SURVEY.md §8d R8 (eta = 1)
    X0 = dc.initial_state(n, alpha, beta, np.random.default_rng(0))[None, :]
    r1 = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=1, precision="f32", path="multipass")
    _one_step(J, alpha, beta, X0, r1)
    r = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=3, precision="f32", path="multipass")
    _check_common(J, r, X0, cut_offset=co)
    assert r[0].iterations == 3
    # x (400 MB) exceeds L2: the opt-in column-chunked pass agrees with the row kernel bit for bit
    with _env("DCX_CHUNKS", "auto"):
        rr = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=3, precision="f32", path="multipass",
                               reupload=True)
    _assert_same(r, rr)


def test_e7_full_size_properties(e7):
    n, v, c, o, co = e7
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
    J = sp.csr_matrix((v, c, o), shape=(n, n))
    alpha, beta = 2.828, 5.005e11  # SURVEY.md §8d E7 (eta = 1)
    X0 = dc.initial_state(n, alpha, beta, np.random.default_rng(0))[None, :]
    r1 = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=1, precision="f32", path="multipass")
    _one_step(J, alpha, beta, X0, r1)
    r = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=20, precision="f32", path="multipass")
    _check_common(J, r, X0, cut_offset=co)
    assert r[0].iterations == 20 and r[0].stop_reason == "max_iters"


class _env:
    def __init__(self, k, v):
        self.k, self.v = k, v

    def __enter__(self):
        import os
        self.old = os.environ.get(self.k)
        os.environ[self.k] = self.v

    def __exit__(self, *exc):
        import os
        if self.old is None:
            os.environ.pop(self.k, None)
        else:
            os.environ[self.k] = self.old


def _assert_same(fast, ref):
    for a_, b_ in zip(fast, ref):
        assert a_.iterations == b_.iterations and a_.stop_reason == b_.stop_reason
        assert a_.energy == b_.energy and np.array_equal(a_.x, b_.x) and np.array_equal(a_.spins, b_.spins)
        assert [t.energy for t in a_.trace] == [t.energy for t in b_.trace]
        assert np.array_equal(np.asarray(a_.h_values), np.asarray(b_.h_values))


@pytest.mark.parametrize("solver", ["doch", "adoch"])
@pytest.mark.parametrize("graph", ["er_uniform", "torus_int8", "hub_rows"])
@pytest.mark.parametrize("chunks", ["3", "7"])
def test_column_chunked_pass_bitwise_equals_row_pass(solver, graph, chunks):
    """The column-chunked R = 1 pass (dcx_chunk.cu; opt-in, DCX_CHUNKS=C) applies each row's entries in column order with the row kernel's
    arithmetic, carrying the running sum between chunk sweeps: iterates, energies, traces
    and stop reasons equal pass_r1w's bit for bit. hub_rows: rows with > 255 entries in
    one chunk, where the plan falls back to the row kernel."""
    if graph == "er_uniform":
        n = 300_000
        v, c, o, _ = synth.erdos_renyi(n, 8, seed=3, device=0)
    elif graph == "torus_int8":
        v, c, o = synth.torus(400, seed=3)
        n = 400 * 400
    else:
        n = 4000
        Jd = np.zeros((n, n))
        Jd[:50, :] = Jd[:, :50] = -0.5  # 50 hub rows with n - 1 entries
        np.fill_diagonal(Jd, 0.0)
        Js = sp.csr_matrix(Jd)
        v, c, o = Js.data, Js.indices.astype(np.int64), Js.indptr.astype(np.int64)
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False))
    p = dc.derive_params(inst.coupling, eta=1.0)
    X0 = dc.initial_state(n, p.alpha, p.beta, np.random.default_rng(7))[None, :]
    kw = dict(max_iters=80, precision="f32", path="multipass", reupload=True)
    with _env("DCX_CHUNKS", "0"):
        ref = dc.solve_replicas(inst, solver, p.alpha, p.beta, X0, **kw)
    with _env("DCX_CHUNKS", chunks):
        fast = dc.solve_replicas(inst, solver, p.alpha, p.beta, X0, **kw)
    _assert_same(fast, ref)


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_torus_stencil_bitwise_equals_csr_pass(solver):
    """The lattice stencil pass (pass_torus, DCX_TORUS=1, available when the upload recognises
    the periodic L x L torus) sums the four neighbours in the CSR's column order with the
    CSR pass's arithmetic: iterates, energies, traces and stop reasons equal pass_rv's bit
    for bit, including the wrap-around rows and columns."""
    import os

    L, R = 37, 128  # odd L: every wrap case; R = 128 (one replica chunk)
    v, c, o = synth.torus(L, seed=5)
    n = L * L
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False))
    p = dc.derive_params(inst.coupling, eta=1.0)
    X0 = np.stack([dc.initial_state(n, p.alpha, p.beta, np.random.default_rng(s)) for s in range(R)])
    kw = dict(max_iters=60, precision="f32", path="multipass")
    ref = dc.solve_replicas(inst, solver, p.alpha, p.beta, X0, **kw)
    os.environ["DCX_TORUS"] = "1"
    try:
        fast = dc.solve_replicas(inst, solver, p.alpha, p.beta, X0, reupload=True, **kw)
    finally:
        os.environ.pop("DCX_TORUS")
    for a_, b_ in zip(fast, ref):
        assert a_.iterations == b_.iterations and a_.stop_reason == b_.stop_reason
        assert a_.energy == b_.energy and np.array_equal(a_.x, b_.x) and np.array_equal(a_.spins, b_.spins)
        assert [t.energy for t in a_.trace] == [t.energy for t in b_.trace]
        assert np.array_equal(np.asarray(a_.h_values), np.asarray(b_.h_values))


def _golden(name):
    import json
    from pathlib import Path

    return json.loads((Path(__file__).resolve().parent / "golden" / f"golden_{name}.json").read_text())


def test_t6_200_iterations_seed0_equals_reference(t6):
    """The unmodified reference's 200-iteration DOCH run on the T6 torus, seed 0, f64 on the host
    (tests/golden/make_golden_t6.py): the f32 device run of replica 0 (one of the bench's 256)
    ends on the same best energy."""
    inst, J, alpha, beta, X0 = t6
    g = _golden("t6")
    assert (g["alpha"], g["beta"], g["iterations"]) == (alpha, beta, 200)
    r = dc.solve_replicas(inst, "doch", alpha, beta, X0, max_iters=200, precision="f32")
    assert r[0].energy == g["best_energy"]
    assert r[0].energy == dc.energy(inst.coupling, r[0].spins)


def test_e7_200_iterations_equals_reference(e7):
    """The unmodified reference's 200-iteration DOCH run on E7, seed 0, with derive_params at
    eta = 1 (tests/golden/make_golden_e7.py): the f32 device run reaches the same best cut."""
    n, v, c, o, co = e7
    g = _golden("e7")
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
    assert co == g["cut_offset"]
    X0 = dc.initial_state(n, g["alpha"], g["beta"], np.random.default_rng(0))[None, :]
    r = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0, max_iters=200, precision="f32")[0]
    assert co - r.energy == g["best_cut"]


def test_r8_20_iterations_equals_reference():
    """The unmodified reference's DOCH run on R8 (n = 1e8, seed 0, derive_params at eta = 1) for
    the bench's 20 iterations (tests/golden/make_golden_r8.py): the f32 device run reaches the
    same best cut."""
    g = _golden("r8")
    n = 10**8
    v, c, o, co = synth.random_regular3(n, seed=0, device=0)
    assert co == g["cut_offset"]
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(n, v, c, o, validate=False), cut_offset=co)
    X0 = dc.initial_state(n, g["alpha"], g["beta"], np.random.default_rng(0))[None, :]
    r = dc.solve_replicas(inst, "doch", g["alpha"], g["beta"], X0, max_iters=g["iterations"], precision="f32")[0]
    assert co - r.energy == g["best_cut"]
