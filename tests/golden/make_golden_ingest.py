"""Golden fixtures for instance generation and ingest, from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_ingest.py

It records ``gen_sparse_9bit`` outputs (dc/generate.py:80-112) as SHA-256 of the
CSR arrays (plus two small ones verbatim), the bytes of ``csr_save`` (dc/io.py:256-269)
for one of them, and the CouplingError messages ``csr_load`` raises on malformed
matrices (dc/io.py:272-305 through CsrCoupling.validate, dc/coupling.py:153-176),
into golden_ingest.json / golden_ingest.npz next to this file. The GPU box never
runs this script; tests only read its outputs.
"""

from __future__ import annotations

import io
import json
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)

import dcising as dc  # noqa: E402
from dcising.coupling import CouplingError  # noqa: E402
from dcising.generate import gen_sparse_9bit  # noqa: E402
from dcising.io import csr_load, csr_save  # noqa: E402

sys.path.insert(0, str(OUT))
from make_golden import sha  # noqa: E402

# (n, p, seed): the reference tests' own cases (test_generate.py, test_io.py, test_acceptance.py)
# plus larger ones
CASES = [(50, 40.0, 1), (100, 30.0, 1), (200, 30.0, 1), (300, 20.0, 2), (300, 20.0, 3), (400, 50.0, 9),
         (300, 100.0, 0), (40, 50.0, 4), (2000, 5.0, 11), (5000, 2.0, 7), (8000, 1.0, 1)]


def bad_matrices():
    """(name, n, row_offsets, cols, values) each violating one CsrCoupling invariant."""
    ok_ro, ok_c, ok_v = [0, 2, 4, 6], [1, 2, 0, 2, 0, 1], [1.0, -2.0, 1.0, 3.0, -2.0, 3.0]
    return [
        ("ok", 3, ok_ro, ok_c, ok_v),
        ("offsets_start", 3, [1, 2, 4, 6], ok_c, ok_v),
        ("offsets_decreasing", 3, [0, 3, 2, 6], ok_c, ok_v),
        ("range", 3, ok_ro, [1, 2, 0, 3, 0, 1], ok_v),
        ("not_increasing", 3, ok_ro, [2, 1, 0, 2, 0, 1], ok_v),
        ("diagonal", 3, ok_ro, [1, 2, 0, 1, 0, 1], ok_v),
        ("diag_before_unsorted", 3, ok_ro, [0, 1, 0, 2, 1, 0], ok_v),
        ("nonfinite", 3, ok_ro, ok_c, [1.0, -2.0, 1.0, np.inf, -2.0, np.inf]),
        ("asymmetric_value", 3, ok_ro, ok_c, [1.0, -2.0, 1.0, 3.0, -2.0, 4.0]),
        ("asymmetric_pattern", 3, [0, 2, 3, 5], [1, 2, 0, 0, 1], [1.0, -2.0, 1.0, -2.0, 3.0]),
        ("zero_without_mirror", 3, [0, 2, 4, 5], [1, 2, 0, 2, 0], [1.0, -2.0, 1.0, 0.0, -2.0]),
        ("real_values", 3, ok_ro, ok_c, [0.5, -2.0, 0.5, 3.0, -2.0, 3.0]),
    ]


def container(n, ro, c, v):
    return (b"ICSR1" + np.uint64(n).tobytes() + np.uint64(len(v)).tobytes() + np.asarray(ro, "<u8").tobytes()
            + np.asarray(c, "<u8").tobytes() + np.asarray(v, "<f8").tobytes())


def main():
    t0 = time.time()
    gold = {"meta": {"generator": "tests/golden/make_golden_ingest.py", "reference": "dcising " + dc.__version__,
                     "numpy": np.__version__}, "gen9": [], "load": []}
    arrays = {}
    for n, p, seed in CASES:
        t = time.perf_counter()
        J = gen_sparse_9bit(n, p, seed=seed)
        dt = time.perf_counter() - t
        gold["gen9"].append({"n": n, "p": p, "seed": seed, "nnz": int(J.nnz), "value_kind": J.value_kind,
                             "sha_row_offsets": sha(J.row_offsets), "sha_col_indices": sha(J.col_indices),
                             "sha_values": sha(J.values), "seconds": dt})
        if n <= 100:
            key = f"gen9_{n}_{p}_{seed}"
            arrays[key + "_ro"] = J.row_offsets
            arrays[key + "_col"] = J.col_indices
            arrays[key + "_val"] = J.values
    buf = io.BytesIO()
    csr_save(gen_sparse_9bit(300, 20.0, seed=2), buf)
    gold["csr_save_300_20_2_sha"] = __import__("hashlib").sha256(buf.getvalue()).hexdigest()
    for name, n, ro, c, v in bad_matrices():
        try:
            J = csr_load(io.BytesIO(container(n, ro, c, v)))
            gold["load"].append({"name": name, "n": n, "ro": ro, "col": c, "val": [float(x) for x in v],
                                 "error": None, "value_kind": J.value_kind})
        except ValueError as e:  # CouplingError, or scipy's own check of the index arrays
            gold["load"].append({"name": name, "n": n, "ro": ro, "col": c, "val": [float(x) for x in v],
                                 "error": str(e), "error_type": type(e).__name__,
                                 "coupling_error": isinstance(e, CouplingError)})
    gold["meta"]["seconds"] = time.time() - t0
    (OUT / "golden_ingest.json").write_text(json.dumps(gold, indent=1, default=str))
    np.savez_compressed(OUT / "golden_ingest.npz", **arrays)
    print(json.dumps({k: v for k, v in gold.items() if k != "gen9"}, indent=1, default=str)[:3000])


if __name__ == "__main__":
    main()
