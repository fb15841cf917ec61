"""Golden fixtures for procedural couplings, from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_procedural.py

It builds ``gen_procedural_sin`` couplings (dc/generate.py:115-123,
ProceduralCoupling dc/coupling.py:209-299) and records their entries, the
blocked product of dc/matvec.py:117-155, the row statistics behind
``derive_params`` (dc/spectral.py:174-256), and DOCH / ADOCH runs
(dc/solvers/doch.py:169-356) into golden_procedural.json / .npz next to this
file. The GPU box never runs this script; tests only read its outputs.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)

import dcising as dc  # noqa: E402
from dcising.generate import gen_procedural_sin  # noqa: E402

sys.path.insert(0, str(OUT))
from make_golden import sha, summarize  # noqa: E402


def main():
    t0 = time.time()
    gold = {"meta": {"generator": "tests/golden/make_golden_procedural.py", "reference": "dcising " + dc.__version__,
                     "numpy": np.__version__}}
    arrays = {}
    for n, seed in ((64, 100), (300, 100), (300, 7), (1500, 100)):
        J = gen_procedural_sin(n, seed=seed)
        key = f"p{n}_s{seed}"
        A = J.block(0, n, 0, n)
        v = np.random.default_rng(3).standard_normal(n)
        y = dc.matvec.matvec(J, v)
        s1, s2 = J.offdiag_moments()
        ent = dict(n=n, seed=seed, dense_sha=sha(A), s1=s1, s2=s2)
        arrays[f"{key}_v"] = v
        arrays[f"{key}_Jv"] = y
        arrays[f"{key}_abs_row_sums"] = J.abs_row_sums()
        if n == 64:
            arrays[f"{key}_dense"] = A
        gold[key] = ent
    print(f"operators done {time.time() - t0:.1f}s", flush=True)

    # derive_params (auto = Wigner for procedural) and the explicit power method
    J = gen_procedural_sin(300, seed=100)
    pw = dc.derive_params(J, eta=1.0)
    pp = dc.derive_params(J, eta=1.0, method="power_iteration", tol=1e-10)
    gold["params_p300"] = dict(alpha=pw.alpha, beta=pw.beta, alpha_power=pp.alpha, beta_power=pp.beta)
    inst = dc.ProblemInstance(coupling=J, name="proc300")
    S = np.where(np.random.default_rng(9).random((4, 300)) < 0.5, -1.0, 1.0)
    arrays["p300_energy_spins"] = S
    gold["params_p300"]["energy_of_spins"] = [float(dc.energy(J, s)) for s in S]
    runs = {}
    for solver, fn in (("doch", dc.doch_solve), ("adoch", dc.adoch_solve)):
        for s in range(3):
            q = dc.SolverParams(alpha=pw.alpha, beta=pw.beta, max_iters=300, seed=s)
            r = fn(inst, q, record_states=s == 0)
            runs[f"{solver}_s{s}"] = summarize(r)
            if s == 0:
                arrays[f"p300_{solver}_s0_states20"] = np.array(r.states[:21])
                arrays[f"p300_{solver}_s0_x"] = np.asarray(r.x)
    gold["runs_p300"] = runs
    print(f"p300 runs done {time.time() - t0:.1f}s", flush=True)

    # two column tiles (block 1024): the reference sums tile partials in block order
    J = gen_procedural_sin(1500, seed=100)
    p15 = dc.derive_params(J, eta=1.0)
    q = dc.SolverParams(alpha=p15.alpha, beta=p15.beta, max_iters=200, seed=0)
    r = dc.doch_solve(dc.ProblemInstance(coupling=J), q, record_states=True)
    gold["runs_p1500"] = dict(alpha=p15.alpha, beta=p15.beta, doch_s0=summarize(r))
    arrays["p1500_doch_s0_states20"] = np.array(r.states[:21])
    print(f"p1500 done {time.time() - t0:.1f}s", flush=True)

    with open(OUT / "golden_procedural.json", "w") as f:
        json.dump(gold, f, indent=1)
    np.savez_compressed(OUT / "golden_procedural.npz", **arrays)
    print("wrote", OUT / "golden_procedural.json", f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
