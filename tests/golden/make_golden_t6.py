"""T6 (BASELINE configs[2]) quality reference from the UNMODIFIED reference, offline.

Builds the 1000 x 1000 +-1 torus with SURVEY.md Appendix A's recipe and the reference's own
CsrCoupling, checks it is the instance bench_configs / synth.torus build (same CSR arrays),
and runs the reference's ``doch_solve`` for seed 0 (replica 0 of the bench) at the bench's
alpha = 4.0, beta = 8.0e9 (derive_params' values) for 200 iterations at
trace_stride 1. Writes golden_t6.json: the best energy, its trace and the wall time. The GPU
box never runs this script.

    python tests/golden/make_golden_t6.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")
import dcising as dc  # noqa: E402
from dcising.coupling import CsrCoupling  # noqa: E402

OUT = Path(__file__).resolve().parent
ROOT = OUT.parent.parent


def torus(L=1000, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.arange(L * L).reshape(L, L)
    right = np.roll(idx, -1, axis=1).ravel()
    down = np.roll(idx, -1, axis=0).ravel()
    a = idx.ravel()
    jr = rng.integers(0, 2, L * L) * 2.0 - 1.0
    jd = rng.integers(0, 2, L * L) * 2.0 - 1.0
    m = sp.csr_matrix((np.concatenate([jr, jr, jd, jd]), (np.concatenate([a, right, a, down]),
                                                          np.concatenate([right, a, down, a]))), shape=(L * L, L * L))
    m.sort_indices()
    return dc.ProblemInstance(coupling=CsrCoupling.from_scipy(m, value_kind="int", validate=False)), m


def main(iters=200, alpha=4.0, beta=8.0e9):
    inst, m = torus()
    sys.path.insert(0, str(ROOT))
    from paper_2509_01928_b200 import synth

    v, c, o = synth.torus(1000, seed=0)
    assert np.array_equal(v, m.data) and np.array_equal(c, m.indices) and np.array_equal(o, m.indptr)
    q = dc.SolverParams(alpha=alpha, beta=beta, eta=1.0, max_iters=iters, seed=0)
    t1 = time.time()
    r = dc.doch_solve(inst, q, trace_stride=1)
    wall = time.time() - t1
    out = dict(generator="tests/golden/make_golden_t6.py", reference="dcising " + dc.__version__, n=10**6,
               alpha=alpha, beta=beta, seed=0, iterations=int(r.iterations), stop_reason=r.stop_reason,
               best_energy=float(r.energy), trace_iter=[t.iteration for t in r.trace],
               trace_best_energy=[float(t.best_energy) for t in r.trace],
               trace_elapsed=[float(t.elapsed_s) for t in r.trace], wall_s=wall)
    with open(OUT / "golden_t6.json", "w") as f:
        json.dump(out, f)
    print(json.dumps({k: v for k, v in out.items() if not k.startswith("trace")}))


if __name__ == "__main__":
    main()
