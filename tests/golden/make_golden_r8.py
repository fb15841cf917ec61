"""R8 (BASELINE configs[4]) quality reference from the UNMODIFIED reference, offline.

Builds the random 3-regular n = 1e8 instance with SURVEY.md Appendix A's ``reg3`` recipe and the
reference's own constructors, derives alpha / beta with the reference's derive_params (Wigner,
eta = 1) and runs ``doch_solve`` seed 0 for the bench's 20 iterations at trace_stride 1. Writes
golden_r8.json: alpha, beta, cut_offset, the best-so-far cut per iteration and the wall time.
The GPU box never runs this script.

    python tests/golden/make_golden_r8.py
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


def reg3(n=10**8, seed=0):
    rng = np.random.default_rng(seed)
    stubs = rng.permutation(np.repeat(np.arange(n, dtype=np.int64), 3))
    i, j = stubs[0::2], stubs[1::2]
    keep = i != j
    i, j = i[keep], j[keep]
    del stubs
    key = np.unique(np.minimum(i, j).astype(np.int64) * n + np.maximum(i, j))
    del i, j
    i, j = key // n, key % n
    del key
    mat = sp.csr_matrix((np.full(2 * len(i), -0.5), (np.concatenate([i, j]), np.concatenate([j, i]))), shape=(n, n))
    mat.sort_indices()
    return dc.ProblemInstance(coupling=CsrCoupling.from_scipy(mat, validate=False), cut_offset=len(i) / 2.0)


def main(iters=20):
    t0 = time.time()
    inst = reg3()
    print(f"built {time.time() - t0:.0f}s", flush=True)
    p = dc.derive_params(inst.coupling, eta=1.0)
    q = dc.SolverParams(alpha=p.alpha, beta=p.beta, eta=1.0, max_iters=iters, seed=0)
    t1 = time.time()
    r = dc.doch_solve(inst, q, trace_stride=1)
    wall = time.time() - t1
    out = dict(generator="tests/golden/make_golden_r8.py", reference="dcising " + dc.__version__, n=10**8,
               alpha=p.alpha, beta=p.beta, cut_offset=inst.cut_offset, iterations=int(r.iterations),
               stop_reason=r.stop_reason, best_energy=float(r.energy), best_cut=float(inst.cut_offset - r.energy),
               trace_iter=[t.iteration for t in r.trace],
               trace_best_energy=[float(t.best_energy) for t in r.trace],
               trace_elapsed=[float(t.elapsed_s) for t in r.trace], wall_s=wall)
    with open(OUT / "golden_r8.json", "w") as f:
        json.dump(out, f)
    print(json.dumps({k: v for k, v in out.items() if not k.startswith("trace")}))


if __name__ == "__main__":
    main()
