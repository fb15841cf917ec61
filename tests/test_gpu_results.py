"""Detached results (dcx_result_detach / dcx_res_*, solvers._LazySolveResult).

A solve's bulk outputs stay on the device (final states, best spins) and in the
pinned history buffer until a field is read. These tests pin that the values
read late are the values an immediate read gives, however many solves the same
context ran in between (the context must take other history rings and result
buffers while a result holds its own), and after the context itself is gone.
"""

import dataclasses

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import synth

pytestmark = pytest.mark.gpu


def _fields(r):
    return (np.asarray(r.spins).copy(), np.asarray(r.x).copy(), [(t.iteration, t.energy, t.best_energy, t.event)
                                                                   for t in r.trace],
            np.asarray(r.h_values).copy(), None if r.accepted is None else list(r.accepted), r.energy,
            r.iterations, r.stop_reason)


def _same(a, b):
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2] == b[2]
    assert np.array_equal(a[3], b[3])
    assert a[4] == b[4] and a[5:] == b[5:]


@pytest.mark.parametrize("kind", ["csr_f32", "csr_f64", "dense_tc"])
@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_results_read_late_equal_results_read_at_once(kind, solver):
    if kind == "dense_tc":
        W = synth.dense_pm1(384, seed=3)
        inst = dc.ProblemInstance(coupling=dc.maxcut_to_ising(dc.DenseCoupling(W, validate=False)))
        n, a, b, kw = 384, 3.0, 384 ** 1.5 * 300.0, dict(precision="f16tc")
    else:
        v, c, o, co = synth.g1_shape()
        inst = dc.ProblemInstance(coupling=dc.CsrCoupling(800, v, c, o, validate=False), cut_offset=co)
        n, a, b = 800, 6.108031887826326, 884913.7454957356
        kw = dict(precision="f32" if kind == "csr_f32" else "f64", path="multipass")
    X = [np.stack([dc.initial_state(n, a, b, np.random.default_rng(100 * k + s)) for s in range(16)])
         for k in range(4)]
    run = lambda X0: dc.solve_replicas(inst, solver, a, b, X0, max_iters=80, **kw)  # noqa: E731
    first = run(X[0])             # not read yet
    others = [run(Xk) for Xk in X[1:]]  # three more solves on the same context
    late = [_fields(r) for r in first]
    again = [_fields(r) for r in run(X[0])]  # the same solve, read at once
    for x, y in zip(late, again):
        _same(x, y)
    # the other batches are intact too, and results outlive a re-upload (a new context)
    keep = run(X[1])
    dc.solve_replicas(inst, solver, a, b, X[2], max_iters=80, reupload=True, **kw)
    for x, y in zip([_fields(r) for r in others[0]], [_fields(r) for r in keep]):
        _same(x, y)


def test_lazy_result_is_a_solve_result():
    """dataclasses.replace / fields / asdict see materialised values (the reference's
    SolveResult is a dataclass: dc/solvers/common.py:31-43)."""
    v, c, o, co = synth.g1_shape()
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(800, v, c, o, validate=False), cut_offset=co)
    r = dc.solve_replicas(inst, "doch", 6.108031887826326, 884913.7454957356,
                          dc.initial_state(800, 6.1, 8.8e5, np.random.default_rng(0))[None, :], max_iters=50)[0]
    assert isinstance(r, dc.SolveResult)
    names = [f.name for f in dataclasses.fields(r)]
    assert "spins" in names and "trace" in names
    r2 = dataclasses.replace(r, seed=7)
    assert r2.seed == 7 and np.array_equal(r2.spins, r.spins) and r2.energy == r.energy
    d = dataclasses.asdict(r)
    assert np.array_equal(d["x"], r.x) and len(d["trace"]) == len(r.trace)
    assert r.energy == dc.energy(inst.coupling, r.spins)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("R", [1, 8])
def test_three_iterate_buffers_equal_two(monkeypatch, precision, R):
    """DOCH on the CSR passes rotates three (DCX_XBUF=4: four) iterate buffers so the best-spin
    copy waits for the end of an improvement streak (PassArgs::nbuf); DCX_XBUF3=0 keeps two,
    copying after every improvement. Everything a caller sees is identical, including the best spins of runs that
    end on an improvement, on a non-improving iterate, by convergence and by max_iters."""
    v, c, o, co = synth.g1_shape()
    inst = dc.ProblemInstance(coupling=dc.CsrCoupling(800, v, c, o, validate=False), cut_offset=co)
    a, b = 6.108031887826326, 884913.7454957356
    X0 = np.stack([dc.initial_state(800, a, b, np.random.default_rng(40 + s)) for s in range(R)])
    for iters in (1, 2, 3, 17, 300):
        kw = dict(max_iters=iters, precision=precision, path="multipass")
        three = [_fields(r) for r in dc.solve_replicas(inst, "doch", a, b, X0, **kw)]
        monkeypatch.setenv("DCX_XBUF", "4")
        four = [_fields(r) for r in dc.solve_replicas(inst, "doch", a, b, X0, **kw)]
        monkeypatch.delenv("DCX_XBUF")
        monkeypatch.setenv("DCX_XBUF3", "0")
        two = [_fields(r) for r in dc.solve_replicas(inst, "doch", a, b, X0, **kw)]
        monkeypatch.delenv("DCX_XBUF3")
        for x, y, z in zip(three, two, four):
            _same(x, y)
            _same(z, y)
        for r in dc.solve_replicas(inst, "doch", a, b, X0, **kw):
            assert r.energy == dc.energy(inst.coupling, r.spins)
