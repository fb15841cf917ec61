"""CPU: pin the numpy oracle (and the synthetic-instance recipes) against the
golden vectors produced by the unmodified reference (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from conftest import g1_csr, k2_W, sk_dense
from oracle import dcising_oracle as orc
from paper_2509_01928_b200 import synth


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_g1_instance_matches_reference(gold):
    vals, cols, offs, cut_offset = g1_csr()
    g = gold["g1"]
    assert len(offs) - 1 == g["n"] == 800 and len(vals) == g["nnz"] == 38352
    assert cut_offset == g["cut_offset"] == 9588.0
    assert sha(vals, cols, offs) == g["csr_sha"]


def test_k2000_instance_matches_reference(gold):
    W = k2_W()
    assert sha(W) == gold["k2"]["W_sha"]
    assert float(np.triu(W, 1).sum()) == gold["k2"]["upper_sum"] == 1190.0


@pytest.mark.parametrize("key", ["sk30_12", "sk40_17", "sk50_23", "sk60_5", "sk100_77", "sk100_3"])
def test_sk_instances_match_reference(gold, key):
    g = gold["sk"][key]
    assert sha(sk_dense(g["n"], g["seed"])) == g["sha"]


def test_small_sparse_families_match_reference(gold):
    fam = gold["families"]
    v, c, o = synth.torus(32)
    assert sha(v, c, o) == fam["torus32"]["csr_sha"]
    v, c, o, co = synth.erdos_renyi(10**4)
    assert sha(v, c, o) == fam["er1e4"]["csr_sha"] and co == fam["er1e4"]["cut_offset"]
    v, c, o, co = synth.random_regular3(10**4)
    assert sha(v, c, o) == fam["reg3_1e4"]["csr_sha"] and co == fam["reg3_1e4"]["cut_offset"]


def test_energy_golden_bit_exact(gold, garr):
    vals, cols, offs, _ = g1_csr()
    op = orc.Operator((vals, cols, offs))
    for s, e in zip(garr["g1_energy_spins"], gold["g1"]["energy_of_spins"]):
        assert orc.energy(op, s) == e
    opk = orc.Operator(-0.5 * k2_W())
    for s, e in zip(garr["k2_energy_spins"], gold["k2"]["energy_of_spins"]):
        assert orc.energy(opk, s) == e


def test_parameter_derivation(gold):
    vals, cols, offs, _ = g1_csr()
    a, b = orc.derive_alpha_beta((vals, cols, offs), eta=0.25)
    assert a == gold["g1"]["alpha"] and b == gold["g1"]["beta"]
    for key in ("sk30_12", "sk50_23"):
        g = gold["sk"][key]
        a, b = orc.derive_alpha_beta(sk_dense(g["n"], g["seed"]), eta=1.0)
        assert a == g["alpha"] and b == g["beta"]


def _check_run(out, ref, exact_trace=True):
    assert out["energy"] == ref["energy"]
    assert out["iterations"] == ref["iterations"]
    assert out["stop_reason"] == ref["stop_reason"]
    if exact_trace:
        assert [t["iteration"] for t in out["trace"]] == ref["trace_iter"]
        assert [t["energy"] for t in out["trace"]] == ref["trace_energy"]
        assert [t["best_energy"] for t in out["trace"]] == ref["trace_best"]
        assert [t["event"] for t in out["trace"]] == ref["trace_event"]
        np.testing.assert_array_equal(out["h_values"], ref["h_values"])
        if ref["accepted"] is not None:
            assert out["accepted"] == ref["accepted"]


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_g1_runs_bitwise(gold, garr, solver):
    vals, cols, offs, co = g1_csr()
    g = gold["g1"]
    for seed in (0, 1):
        out = orc.run((vals, cols, offs), g["alpha"], g["beta"], solver=solver, seed=seed, record_states=True,
                      cut_offset=co)
        _check_run(out, g["runs"][f"{solver}_s{seed}"])
        np.testing.assert_array_equal(np.array(out["states"][:21]), garr[f"g1_{solver}_s{seed}_states20"])
        np.testing.assert_array_equal(out["x"], garr[f"g1_{solver}_s{seed}_x"])
        assert [t["cut_value"] for t in out["trace"]] == g["runs"][f"{solver}_s{seed}"]["trace_cut"]


@pytest.mark.parametrize("solver", ["doch", "adoch"])
def test_g1_100_seed_distribution(gold, solver):
    vals, cols, offs, co = g1_csr()
    g = gold["g1"]
    op = orc.Operator((vals, cols, offs))
    for row in g[solver][::7]:
        out = orc.run(op, g["alpha"], g["beta"], solver=solver, seed=row["seed"])
        assert (out["energy"], out["iterations"], out["stop_reason"]) == (
            row["energy"], row["iterations"], row["stop_reason"])


@pytest.mark.parametrize("key", ["sk30_12", "sk40_17", "sk100_77"])
def test_sk_runs_bitwise(gold, garr, key):
    g = gold["sk"][key]
    J = sk_dense(g["n"], g["seed"])
    for solver in ("doch", "adoch"):
        for s in range(3):
            out = orc.run(J, g["alpha"], g["beta"], solver=solver, seed=s, max_iters=150, lookback_q=2,
                          record_states=s == 0)
            _check_run(out, g[f"{solver}_s{s}"])
            if s == 0:
                np.testing.assert_array_equal(np.array(out["states"]), garr[f"{key}_{solver}_states"])
    out = orc.run(J, g["alpha"], g["beta"], solver="adoch", seed=0, max_iters=150, lookback_q=2,
                  window_mode="exact", record_states=True)
    _check_run(out, g["adoch_exact_s0"])


def test_antiferro_pair(gold, garr):
    J = np.array([[0.0, -1.0], [-1.0, 0.0]])
    for s in range(20):
        out = orc.run(J, 1.0, 2.0, max_iters=25, seed=s, record_states=True)
        _check_run(out, gold["pair"][str(s)])
        np.testing.assert_array_equal(np.array(out["states"]), garr[f"pair_s{s}_states"])


def test_families_runs(gold, garr):
    fam = gold["families"]
    for name, (v, c, o, *_rest) in (("torus32", synth.torus(32)), ("er1e4", synth.erdos_renyi(10**4)),
                                    ("reg3_1e4", synth.random_regular3(10**4))):
        g = fam[name]
        for solver in ("doch", "adoch"):
            out = orc.run((v, c, o), g["alpha"], g["beta"], solver=solver, max_iters=100, record_states=True,
                          cut_offset=g["cut_offset"])
            _check_run(out, g[solver])
            np.testing.assert_array_equal(np.array(out["states"][:21]), garr[f"{name}_{solver}_states20"])


def test_k2000_quality_reference(gold):
    """Seed 0 of the K2000 config (BASELINE configs[1]) reproduces bit for bit."""
    g = gold["k2"]
    J = -0.5 * k2_W()
    out = orc.run(J, g["alpha"], g["beta"], solver="doch", seed=0, max_iters=1000)
    _check_run(out, g["doch_s0"])
