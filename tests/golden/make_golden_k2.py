"""K2000 quality goldens over ALL 1024 seeds, by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_k2.py            # ~10 min on 8 cores

The instance is the reference's own criterion-10 instance
(`pkg/tests/test_acceptance.py:276-281`: ``gen_dense_pm1(2000, seed=20240817)``,
``J = maxcut_to_ising(W)``), η = 0.1 (the tuned value), α/β from
``derive_params(tol=1e-8)`` computed ONCE and passed premade, as
``run_bench`` does (`dc/bench.py:287-316`); seeds 0..1023 are the ``seed + r``
restart convention (`dc/bench.py:311`) with base seed 0.  Every solve is
``doch_solve`` / ``adoch_solve`` with the ``solve()`` defaults
(``trace_stride=1``, ``max_iters=1000``, economy window, q=5).

Per seed it stores the best energy, the iteration count, the stop reason and
the best-so-far trace compressed to its improvement points
``(iteration, best_energy, elapsed_s)``, which is all ``first_reach_time``
(`dc/bench.py:219-231`) needs.  Output: ``golden_k2.npz`` (+ ``golden_k2.json``
summary) next to this file.  The GPU box never runs this script.
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)

import dcising as dc  # noqa: E402
from dcising.generate import gen_dense_pm1  # noqa: E402

R = int(os.environ.get("K2_SEEDS", "1024"))
_INST = None
_PAR = None


def _init(alpha, beta):
    global _INST, _PAR
    W = gen_dense_pm1(2000, seed=20240817)
    _INST = dc.ProblemInstance(coupling=dc.maxcut_to_ising(W), name="k2000")
    _PAR = (alpha, beta)


def _one(task):
    solver, seed = task
    alpha, beta = _PAR
    q = dc.SolverParams(alpha=alpha, beta=beta, eta=0.1, max_iters=1000, seed=seed)
    fn = dc.doch_solve if solver == "doch" else dc.adoch_solve
    t0 = time.perf_counter()
    r = fn(_INST, q)
    wall = time.perf_counter() - t0
    pts = []
    prev = np.inf
    for t in r.trace:
        if t.best_energy < prev:
            pts.append((t.iteration, t.best_energy, t.elapsed_s))
            prev = t.best_energy
    return solver, seed, float(r.energy), int(r.iterations), r.stop_reason, pts, wall


def main():
    W = gen_dense_pm1(2000, seed=20240817)
    k2 = dc.ProblemInstance(coupling=dc.maxcut_to_ising(W), name="k2000")
    pk = dc.derive_params(k2.coupling, eta=0.1, tol=1e-8, max_iters=1000)
    upper = float(np.triu(W.array, 1).sum())
    print(f"alpha={pk.alpha!r} beta={pk.beta!r}", flush=True)
    tasks = [(s, seed) for s in ("doch", "adoch") for seed in range(R)]
    res = {}
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=os.cpu_count(), initializer=_init,
                             initargs=(pk.alpha, pk.beta)) as ex:
        for k, out in enumerate(ex.map(_one, tasks, chunksize=4)):
            res[(out[0], out[1])] = out
            if k % 128 == 0:
                print(f"{k}/{len(tasks)} {time.time() - t0:.0f}s", flush=True)
    arrays = {}
    summary = dict(generator="tests/golden/make_golden_k2.py", reference="dcising " + dc.__version__,
                   numpy=np.__version__, seeds=R, eta=0.1, alpha=pk.alpha, beta=pk.beta,
                   cut_offset=upper / 2.0, upper_sum=upper,
                   cpu_count=os.cpu_count(), omp_threads=os.environ.get("OMP_NUM_THREADS"))
    stops = {"converged": 0, "max_iters": 1, "time_budget": 2}
    for solver in ("doch", "adoch"):
        rows = [res[(solver, s)] for s in range(R)]
        arrays[f"{solver}_energy"] = np.array([r[2] for r in rows])
        arrays[f"{solver}_iterations"] = np.array([r[3] for r in rows], np.int32)
        arrays[f"{solver}_stop"] = np.array([stops[r[4]] for r in rows], np.int8)
        arrays[f"{solver}_wall_s"] = np.array([r[6] for r in rows])
        off = np.zeros(R + 1, np.int64)
        off[1:] = np.cumsum([len(r[5]) for r in rows])
        arrays[f"{solver}_imp_offsets"] = off
        arrays[f"{solver}_imp_iter"] = np.array([p[0] for r in rows for p in r[5]], np.int32)
        arrays[f"{solver}_imp_best"] = np.array([p[1] for r in rows for p in r[5]])
        arrays[f"{solver}_imp_elapsed"] = np.array([p[2] for r in rows for p in r[5]])
        e = arrays[f"{solver}_energy"]
        it = arrays[f"{solver}_iterations"]
        summary[solver] = dict(best_energy=float(e.min()), best_cut=upper / 2.0 - float(e.min()),
                               mean_energy=float(e.mean()), std_energy=float(e.std(ddof=1)),
                               mean_iterations=float(it.mean()), max_iterations=int(it.max()),
                               converged=int((arrays[f"{solver}_stop"] == 0).sum()),
                               mean_wall_s=float(arrays[f"{solver}_wall_s"].mean()))
    np.savez_compressed(OUT / "golden_k2.npz", **arrays)
    with open(OUT / "golden_k2.json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))
    print(f"done {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
