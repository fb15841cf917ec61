"""Instance generation and ingest: gen_sparse_9bit on the device,
the ICSR container (csr_save / csr_load) with its validation on the device.

Golden fixtures come from the unmodified reference (tests/golden/make_golden_ingest.py).
CPU tests pin the oracle's restatement of the generator and the container's host-side
parsing; GPU tests require the device generator to reproduce the reference's CSR bytes
exactly (SHA-256 of row_offsets / col_indices / values) and csr_load to raise the
reference's errors.
"""

import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2509_01928_b200 as dc
from paper_2509_01928_b200 import io as dio

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gi():
    g = json.loads((GOLD / "golden_ingest.json").read_text())
    g["arrays"] = dict(np.load(GOLD / "golden_ingest.npz"))
    return g


def sha(*arrays):
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def container(n, ro, c, v):
    return (b"ICSR1" + np.uint64(n).tobytes() + np.uint64(len(v)).tobytes() + np.asarray(ro, "<u8").tobytes()
            + np.asarray(c, "<u8").tobytes() + np.asarray(v, "<f8").tobytes())


# ----------------------------------------------------------------------- CPU
def test_oracle_philox_matches_numpy():
    from oracle import dcising_oracle as orc

    for seed, row, high in ((3, 5, 5115), (1, 199, 3410), (0, 1, 102300), (11, 77, 1023), (2**63 + 5, 3, 7)):
        ref = np.random.Generator(np.random.Philox(key=np.array([seed, row], dtype=np.uint64))).integers(
            1, high + 1, size=row)
        assert list(ref) == orc.row_integers(seed, row, row, high)


def test_oracle_gen_sparse_9bit_matches_reference_goldens(gi):
    from oracle import dcising_oracle as orc

    for case in gi["gen9"]:
        if case["n"] > 100:
            continue
        v, c, ro = orc.gen_sparse_9bit(case["n"], case["p"], case["seed"])
        key = f"gen9_{case['n']}_{case['p']}_{case['seed']}"
        assert np.array_equal(ro, gi["arrays"][key + "_ro"])
        assert np.array_equal(c, gi["arrays"][key + "_col"])
        assert v.tobytes() == gi["arrays"][key + "_val"].tobytes()
        assert sha(ro) == case["sha_row_offsets"] and sha(c) == case["sha_col_indices"]
        assert sha(v) == case["sha_values"]


def test_container_parse_errors_match_reference():
    v = np.array([1.0, 1.0])
    blob = container(2, [0, 1, 2], [1, 0], v)
    n, ro, ci, vals = dio.parse_csr(blob)
    assert n == 2 and list(ro) == [0, 1, 2] and list(ci) == [1, 0] and list(vals) == [1.0, 1.0]
    with pytest.raises(dio.FormatError, match="truncated"):
        dio.parse_csr(blob[:-16])
    with pytest.raises(dio.FormatError, match="magic"):
        dio.parse_csr(b"XXXXX" + b"\x00" * 64)
    with pytest.raises(dio.FormatError, match="trailing"):
        dio.parse_csr(blob + b"\x00")
    assert issubclass(dio.FormatError, ValueError)


def test_csr_save_writes_the_reference_bytes(gi):
    """csr_save of the reference's own CSR (oracle-generated, pinned above) gives the reference's file."""
    import hashlib

    from oracle import dcising_oracle as orc

    v, c, ro = orc.gen_sparse_9bit(300, 20.0, 2)
    J = dc.CsrCoupling(300, v, c, ro, value_kind="int", validate=False)
    buf = io.BytesIO()
    dc.csr_save(J, buf)
    assert hashlib.sha256(buf.getvalue()).hexdigest() == gi["csr_save_300_20_2_sha"]


# ----------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_device_gen_sparse_9bit_reproduces_reference_bytes(gi):
    for case in gi["gen9"]:
        J = dc.gen_sparse_9bit(case["n"], case["p"], seed=case["seed"])
        assert J.nnz == case["nnz"], case
        assert sha(J.row_offsets) == case["sha_row_offsets"], case
        assert sha(J.col_indices) == case["sha_col_indices"], case
        assert sha(J.values) == case["sha_values"], case
        assert J.value_kind == case["value_kind"]


@pytest.mark.gpu
def test_device_gen_sparse_9bit_argument_checks():
    with pytest.raises(ValueError):
        dc.gen_sparse_9bit(100, 0.0)
    with pytest.raises(ValueError):
        dc.gen_sparse_9bit(100, 120.0)
    with pytest.raises(ValueError):
        dc.gen_sparse_9bit(1, 10.0)


@pytest.mark.gpu
def test_device_gen_large_is_valid_and_symmetric():
    J = dc.gen_sparse_9bit(30_000, 0.5, seed=5)
    J.validate()  # vectorised host check of every invariant, symmetry included
    ro = J.row_offsets
    assert ro[-1] == J.nnz and np.all(np.diff(ro) >= 0)


@pytest.mark.gpu
def test_csr_round_trip_bit_identical(tmp_path):
    J = dc.gen_sparse_9bit(300, 20.0, seed=2)
    path = tmp_path / "m.icsr"
    dc.csr_save(J, path)
    J2 = dc.csr_load(path)
    assert J2.n == J.n
    assert J2.values.tobytes() == J.values.tobytes()
    assert J2.col_indices.tobytes() == J.col_indices.tobytes()
    assert J2.row_offsets.tobytes() == J.row_offsets.tobytes()
    assert J2.value_kind == "int"


@pytest.mark.gpu
def test_csr_load_errors_match_reference(gi):
    for case in gi["load"]:
        blob = container(case["n"], case["ro"], case["col"], np.array(case["val"]))
        if case["error"] is None:
            J = dc.csr_load(io.BytesIO(blob))
            assert J.value_kind == case["value_kind"], case["name"]
            continue
        with pytest.raises(ValueError) as ei:
            dc.csr_load(io.BytesIO(blob))
        assert str(ei.value) == case["error"], case["name"]
        assert isinstance(ei.value, dc.CouplingError) == case["coupling_error"], case["name"]


@pytest.mark.gpu
def test_loaded_instance_solves_like_the_generated_one(tmp_path):
    """The ingested coupling drives the solver exactly like the generated one."""
    J = dc.gen_sparse_9bit(400, 50.0, seed=9)
    path = tmp_path / "m.icsr"
    dc.csr_save(J, path)
    J2 = dc.csr_load(path)
    a, b = 3.0, 400 ** 1.5 * 600.0
    r1 = dc.doch_solve(dc.ProblemInstance(coupling=J), dc.SolverParams(alpha=a, beta=b, max_iters=50, seed=1))
    r2 = dc.doch_solve(dc.ProblemInstance(coupling=J2), dc.SolverParams(alpha=a, beta=b, max_iters=50, seed=1))
    assert r1.energy == r2.energy and r1.iterations == r2.iterations
    assert np.array_equal(r1.x, r2.x)
