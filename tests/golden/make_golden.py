"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``dcising`` from /root/reference/pkg/src, builds every instance
through the reference's own constructors, runs
``doch_solve`` / ``adoch_solve`` / ``derive_params`` / ``tune_eta`` /
``energy`` and writes small ``.npz`` / ``.json`` fixtures next to this file.
The GPU box never runs this script; tests only read its outputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)

import scipy.sparse as sp  # noqa: E402

import dcising as dc  # noqa: E402
from dcising.coupling import CsrCoupling  # noqa: E402
from dcising.generate import gen_dense_pm1, gen_sk  # noqa: E402
from dcising.io import graph_to_instance, parse_edgelist  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def g1_shape(n=800, m=19176, seed=1):
    rng = np.random.default_rng(seed)
    pairs = set()
    while len(pairs) < m:
        i, j = rng.integers(1, n + 1, size=2)
        if i != j:
            pairs.add((min(i, j), max(i, j)))
    text = f"{n} {m}\n" + "\n".join(f"{i} {j} 1" for i, j in sorted(pairs))
    return graph_to_instance(parse_edgelist(text), name="g1shape")


def torus(L, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.arange(L * L).reshape(L, L)
    right = np.roll(idx, -1, axis=1).ravel()
    down = np.roll(idx, -1, axis=0).ravel()
    a = idx.ravel()
    jr = rng.integers(0, 2, L * L) * 2.0 - 1.0
    jd = rng.integers(0, 2, L * L) * 2.0 - 1.0
    m = sp.csr_matrix((np.concatenate([jr, jr, jd, jd]),
                       (np.concatenate([a, right, a, down]), np.concatenate([right, a, down, a]))),
                      shape=(L * L, L * L))
    m.sort_indices()
    return dc.ProblemInstance(coupling=CsrCoupling.from_scipy(m, value_kind="int", validate=False))


def _maxcut_unit(n, i, j):
    key = np.unique(np.minimum(i, j).astype(np.int64) * n + np.maximum(i, j))
    i, j = key // n, key % n
    m = sp.csr_matrix((np.full(2 * len(i), -0.5), (np.concatenate([i, j]), np.concatenate([j, i]))),
                      shape=(n, n))
    m.sort_indices()
    return dc.ProblemInstance(coupling=CsrCoupling.from_scipy(m, validate=False), cut_offset=len(i) / 2.0)


def er(n, deg=8, seed=0):
    rng = np.random.default_rng(seed)
    m = n * deg // 2
    i = rng.integers(0, n, m)
    j = rng.integers(0, n, m)
    keep = i != j
    return _maxcut_unit(n, i[keep], j[keep])


def reg3(n, seed=0):
    rng = np.random.default_rng(seed)
    stubs = rng.permutation(np.repeat(np.arange(n, dtype=np.int64), 3))
    i, j = stubs[0::2], stubs[1::2]
    keep = i != j
    return _maxcut_unit(n, i[keep], j[keep])


def csr_hash(J):
    return sha(np.asarray(J.values, np.float64), np.asarray(J.col_indices, np.int64),
               np.asarray(J.row_offsets, np.int64))


def summarize(r):
    return dict(
        energy=float(r.energy), iterations=int(r.iterations), stop_reason=r.stop_reason,
        trace_iter=[t.iteration for t in r.trace], trace_energy=[float(t.energy) for t in r.trace],
        trace_best=[float(t.best_energy) for t in r.trace],
        trace_cut=[None if t.cut_value is None else float(t.cut_value) for t in r.trace],
        trace_event=[t.event for t in r.trace],
        h_values=[float(h) for h in r.h_values],
        accepted=None if r.accepted is None else [bool(a) for a in r.accepted],
        spins_sha=sha(np.asarray(r.spins, np.float64)),
    )


def main():
    meta = {"generator": "tests/golden/make_golden.py", "reference": "dcising " + dc.__version__,
            "numpy": np.__version__, "scipy": sp.__name__ and __import__("scipy").__version__}
    gold = {"meta": meta}
    arrays = {}
    t0 = time.time()

    # ---------------------------------------------------------------- G1 (BASELINE configs[0])
    g1 = g1_shape()
    J = g1.coupling
    gold["g1"] = dict(n=J.n, nnz=J.nnz, cut_offset=g1.cut_offset, csr_sha=csr_hash(J))
    eta = dc.tune_eta(g1, dc.spectral.DEFAULT_ETA_GRID, probe_iters=10, seed=0)
    p = dc.derive_params(J, eta=eta)
    p1 = dc.derive_params(J, eta=1.0)
    gold["g1"].update(eta=eta, alpha=p.alpha, beta=p.beta, alpha_eta1=p1.alpha, beta_eta1=p1.beta)
    runs = {}
    for solver, fn in (("doch", dc.doch_solve), ("adoch", dc.adoch_solve)):
        rows = []
        for seed in range(100):
            q = dc.SolverParams(alpha=p.alpha, beta=p.beta, eta=eta, max_iters=1000, seed=seed)
            r = fn(g1, q, record_states=seed < 2)
            rows.append(dict(seed=seed, energy=float(r.energy), iterations=int(r.iterations),
                             stop_reason=r.stop_reason, cut=float(g1.cut_offset - r.energy)))
            if seed < 2:
                arrays[f"g1_{solver}_s{seed}_states20"] = np.array(r.states[:21])
                arrays[f"g1_{solver}_s{seed}_x"] = np.asarray(r.x)
                arrays[f"g1_{solver}_s{seed}_spins"] = np.asarray(r.spins)
                runs[f"{solver}_s{seed}"] = summarize(r)
        gold["g1"][solver] = rows
    gold["g1"]["runs"] = runs
    rng = np.random.default_rng(5)
    S = np.where(rng.random((16, J.n)) < 0.5, -1.0, 1.0)
    arrays["g1_energy_spins"] = S
    gold["g1"]["energy_of_spins"] = [float(dc.energy(J, s)) for s in S]
    gold["g1"]["cut_of_spins"] = [float(dc.cut_value(CsrCoupling(J.n, -2.0 * J.values, J.col_indices,
                                                                  J.row_offsets, validate=False), s))
                                  for s in S]
    print(f"g1 done {time.time() - t0:.1f}s", flush=True)

    # ---------------------------------------------------------------- small SK instances (tests)
    sk = {}
    for n, seed in ((30, 12), (40, 17), (50, 23), (60, 5), (100, 77), (100, 3)):
        A = gen_sk(n, seed=seed)
        inst = dc.ProblemInstance(coupling=A)
        pp = dc.derive_params(A, eta=1.0, max_iters=150, seed=0)
        key = f"sk{n}_{seed}"
        ent = dict(n=n, seed=seed, sha=sha(A.array), alpha=pp.alpha, beta=pp.beta)
        for solver, fn in (("doch", dc.doch_solve), ("adoch", dc.adoch_solve)):
            for s in range(3):
                q = dc.SolverParams(alpha=pp.alpha, beta=pp.beta, max_iters=150, seed=s, lookback_q=2)
                r = fn(inst, q, record_states=True)
                ent[f"{solver}_s{s}"] = summarize(r)
                if s == 0:
                    arrays[f"{key}_{solver}_states"] = np.array(r.states)
        q = dc.SolverParams(alpha=pp.alpha, beta=pp.beta, max_iters=150, seed=0, lookback_q=2)
        r = dc.adoch_solve(inst, q, record_states=True, window_mode="exact")
        ent["adoch_exact_s0"] = summarize(r)
        arrays[f"{key}_adoch_exact_states"] = np.array(r.states)
        sk[key] = ent
    gold["sk"] = sk
    print(f"sk done {time.time() - t0:.1f}s", flush=True)

    # ---------------------------------------------------------------- antiferro pair
    pair = dc.ProblemInstance(coupling=dc.DenseCoupling(np.array([[0.0, -1.0], [-1.0, 0.0]])))
    af = {}
    for s in range(20):
        r = dc.doch_solve(pair, dc.SolverParams(alpha=1.0, beta=2.0, max_iters=25, seed=s), record_states=True)
        af[str(s)] = summarize(r)
        arrays[f"pair_s{s}_states"] = np.array(r.states)
    gold["pair"] = af

    # ---------------------------------------------------------------- small sparse families
    fam = {}
    for name, inst in (("torus32", torus(32)), ("er1e4", er(10**4)), ("reg3_1e4", reg3(10**4))):
        Jc = inst.coupling
        pp = dc.derive_params(Jc, eta=1.0, max_iters=100, seed=0)
        ent = dict(n=Jc.n, nnz=Jc.nnz, csr_sha=csr_hash(Jc), alpha=pp.alpha, beta=pp.beta,
                   cut_offset=inst.cut_offset)
        for solver, fn in (("doch", dc.doch_solve), ("adoch", dc.adoch_solve)):
            r = fn(inst, pp, record_states=True)
            ent[solver] = summarize(r)
            arrays[f"{name}_{solver}_states20"] = np.array(r.states[:21])
        S = np.where(np.random.default_rng(9).random((4, Jc.n)) < 0.5, -1.0, 1.0)
        arrays[f"{name}_energy_spins"] = S
        ent["energy_of_spins"] = [float(dc.energy(Jc, s)) for s in S]
        fam[name] = ent
    gold["families"] = fam
    print(f"families done {time.time() - t0:.1f}s", flush=True)

    # ---------------------------------------------------------------- K2000 (BASELINE configs[1])
    W = gen_dense_pm1(2000, seed=20240817)
    k2 = dc.ProblemInstance(coupling=dc.maxcut_to_ising(W), name="k2000")
    pk = dc.derive_params(k2.coupling, eta=0.1, tol=1e-8, max_iters=1000)
    ent = dict(n=2000, W_sha=sha(W.array), upper_sum=float(np.triu(W.array, 1).sum()),
               alpha=pk.alpha, beta=pk.beta, eta=0.1)
    S = np.where(np.random.default_rng(11).random((8, 2000)) < 0.5, -1.0, 1.0)
    arrays["k2_energy_spins"] = S
    ent["energy_of_spins"] = [float(dc.energy(k2.coupling, s)) for s in S]
    for solver, fn in (("doch", dc.doch_solve), ("adoch", dc.adoch_solve)):
        rows = []
        for seed in range(int(os.environ.get("K2_SEEDS", "32"))):
            q = dc.SolverParams(alpha=pk.alpha, beta=pk.beta, eta=0.1, max_iters=1000, seed=seed)
            r = fn(k2, q, record_states=seed == 0)
            rows.append(dict(seed=seed, energy=float(r.energy), iterations=int(r.iterations),
                             stop_reason=r.stop_reason))
            if seed == 0:
                arrays[f"k2_{solver}_s0_states20"] = np.array(r.states[:21])
                ent[f"{solver}_s0"] = summarize(r)
        ent[solver] = rows
    gold["k2"] = ent
    print(f"k2 done {time.time() - t0:.1f}s", flush=True)

    with open(OUT / "golden.json", "w") as f:
        json.dump(gold, f, indent=1)
    np.savez_compressed(OUT / "golden_arrays.npz", **arrays)
    print("wrote", OUT / "golden.json", OUT / "golden_arrays.npz", f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
