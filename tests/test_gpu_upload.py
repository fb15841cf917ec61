"""Host staging of the coupling uploads (dcx_set_csr / dcx_set_dense, csrc/dcx_api.cu).

The host converts the caller's int64 / f64 arrays into pinned staging with streaming
stores on a worker pool, in pieces whose DMA overlaps the next piece's conversion and
the value classification. These tests pin that every piece lands (the product equals
scipy's at sizes spanning several pieces and pool chunks), that each value class
(uniform, int8, int16, real) is found, and that invalid input anywhere in the arrays
raises the reference's error (`dc/coupling.py` CsrCoupling.validate messages) and
leaves no half-uploaded coupling behind.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2509_01928_b200 import _native

pytestmark = pytest.mark.gpu

N = 1_200_000  # nnz ~ 1.9e7: five column pieces of 2^22, sixteen pool chunks each


@pytest.fixture(scope="module")
def pattern():
    rng = np.random.default_rng(0)
    m = N * 8
    i, j = rng.integers(0, N, m), rng.integers(0, N, m)
    keep = i != j
    A = sp.coo_matrix((np.ones(int(keep.sum())), (i[keep], j[keep])), shape=(N, N)).tocsr()
    A = (A + A.T).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    assert A.nnz > 4 * (1 << 22)
    return A.indptr.astype(np.int64), A.indices.astype(np.int64)


def _values(kind, nnz, rng):
    if kind == "uniform":
        return np.full(nnz, -1.0)
    if kind == "int8":
        return rng.choice([-2.0, -1.0, 1.0, 2.0], nnz)
    if kind == "int16":
        return rng.choice([-300.0, 7.0, 1.0, 250.0], nnz)
    return rng.normal(size=nnz)


@pytest.mark.parametrize("kind", ["uniform", "int8", "int16", "real"])
def test_csr_upload_pieces_land(pattern, kind):
    ro, ci = pattern
    rng = np.random.default_rng(1)
    v = _values(kind, len(ci), rng)
    ctx = _native.Context()
    ctx.set_csr(N, v, ci, ro)
    X = rng.normal(size=(2, N))
    got = ctx.matvec(X, "f64")
    A = sp.csr_matrix((v, ci, ro), shape=(N, N))
    want = np.stack([A @ x for x in X])
    if kind == "real":
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    else:  # integer products: exact
        S = np.where(rng.normal(size=(2, N)) >= 0, 1.0, -1.0)
        assert np.array_equal(ctx.matvec(S, "f64"), np.stack([A @ s for s in S]))
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-9)
    ctx.close()


@pytest.mark.parametrize("where,bad", [("last", N), ("middle", -1), ("first", (1 << 32) + 5)])
def test_csr_bad_column_anywhere_raises(pattern, where, bad):
    ro, ci = pattern
    ci = ci.copy()
    k = {"last": len(ci) - 3, "middle": len(ci) // 2 + 17, "first": 5}[where]
    ci[k] = bad
    ctx = _native.Context()
    ctx.set_csr(N, np.ones(len(ci)), pattern[1], ro)
    with pytest.raises(ValueError, match="column index out of range"):
        ctx.set_csr(N, np.ones(len(ci)), ci, ro)
    with pytest.raises((ValueError, RuntimeError)):  # the old coupling is gone, none half-built
        ctx.matvec(np.ones((1, N)))
    ctx.set_csr(N, np.ones(len(ci)), pattern[1], ro)  # and the context takes a valid one again
    assert np.array_equal(ctx.matvec(np.ones((1, N)))[0], np.diff(ro).astype(np.float64))
    ctx.close()


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_csr_nonfinite_value_raises(pattern, bad):
    ro, ci = pattern
    v = np.ones(len(ci))
    v[len(v) - 2] = bad
    ctx = _native.Context()
    with pytest.raises(ValueError, match="finite"):
        ctx.set_csr(N, v, ci, ro)
    ctx.close()


@pytest.mark.parametrize("scale", [0.5, 1.0, 0.1])
def test_dense_upload_classes(scale):
    # 0.5 / 1: J = scale * int8 (one byte per entry over PCIe); 0.1 is not a binary
    # fraction: the f64 upload and the device classification take over
    rng = np.random.default_rng(2)
    n = 1500
    Q = rng.integers(-3, 4, size=(n, n)).astype(np.float64)
    Q = np.triu(Q, 1)
    J = (Q + Q.T) * scale
    ctx = _native.Context()
    ctx.set_dense(J)
    S = np.where(rng.normal(size=(3, n)) >= 0, 1.0, -1.0)
    got = ctx.matvec(S, "f64")
    want = S @ J.T
    if scale != 0.1:
        assert np.array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    ctx.close()
