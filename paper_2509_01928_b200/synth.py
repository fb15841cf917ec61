"""Synthetic benchmark instances (input construction, not the hot path).

These rebuild, byte for byte, the instances named in BASELINE.json ``configs``
following the recipes of SURVEY.md Appendix A, without importing the reference.
They return plain arrays so the caller can wrap them in
:class:`paper_2509_01928_b200.coupling.CsrCoupling` / ``DenseCoupling``.

* ``g1_shape``  -- 800-spin G1-shape random graph (pattern of
  ``pkg/tests/test_io.py:39-53``; J = -W/2 as in ``dc/io.py:112-121``).
* ``dense_pm1`` -- ``dc/generate.py:69-77``: row i of the lower triangle is
  ``Philox(key=[seed, i]).integers(0, 2, size=i) * 2 - 1``
  (per-row stream ``dc/generate.py:53-55``).
* ``sk_gaussian`` -- ``dc/generate.py:58-66`` (standard normal rows).
* ``torus``     -- 2-D L x L +-1 spin glass, periodic (Appendix A ``torus``).
* ``erdos_renyi`` / ``random_regular3`` -- unit-weight MaxCut graphs
  (Appendix A ``er`` / ``reg3``), J = -1/2 on every edge.
"""

from __future__ import annotations

import numpy as np


def _row_rng(seed: int, row: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.array([seed, row], dtype=np.uint64)))


def dense_pm1(n: int, seed: int = 0) -> np.ndarray:
    """Symmetric +-1 adjacency with zero diagonal (``gen_dense_pm1``)."""
    a = np.zeros((n, n))
    for i in range(1, n):
        a[i, :i] = _row_rng(seed, i).integers(0, 2, size=i) * 2.0 - 1.0
    return a + a.T


def sk_gaussian(n: int, seed: int = 0) -> np.ndarray:
    """Symmetric standard-normal couplings with zero diagonal (``gen_sk``)."""
    a = np.zeros((n, n))
    for i in range(1, n):
        a[i, :i] = _row_rng(seed, i).standard_normal(i)
    return a + a.T


def _csr_from_pairs(n, i, j, w):
    """Symmetric CSR (sorted columns) from undirected pairs i<j with weights w."""
    rows = np.concatenate([i, j]).astype(np.int64)
    cols = np.concatenate([j, i]).astype(np.int64)
    vals = np.concatenate([w, w]).astype(np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_offsets[1:])
    return vals, cols, row_offsets


def g1_shape(n: int = 800, m: int = 19176, seed: int = 1):
    """(values, col_indices, row_offsets, cut_offset) of J = -W/2 for the
    G1-shape graph: m distinct uniform pairs drawn with ``integers(1, n+1, 2)``,
    self-loops rejected (SURVEY Appendix A ``g1_shape``)."""
    rng = np.random.default_rng(seed)
    pairs = set()
    while len(pairs) < m:
        a, b = rng.integers(1, n + 1, size=2)
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    pr = np.array(sorted(pairs), dtype=np.int64) - 1
    vals, cols, offs = _csr_from_pairs(n, pr[:, 0], pr[:, 1], np.full(m, -0.5))
    return vals, cols, offs, m / 2.0


def torus(L: int = 1000, seed: int = 0):
    """(values, col_indices, row_offsets) of the periodic +-1 L x L lattice."""
    rng = np.random.default_rng(seed)
    idx = np.arange(L * L, dtype=np.int64).reshape(L, L)
    right = np.roll(idx, -1, axis=1).ravel()
    down = np.roll(idx, -1, axis=0).ravel()
    a = idx.ravel()
    jr = rng.integers(0, 2, L * L) * 2.0 - 1.0
    jd = rng.integers(0, 2, L * L) * 2.0 - 1.0
    rows = np.concatenate([a, right, a, down])
    cols = np.concatenate([right, a, down, a])
    vals = np.concatenate([jr, jr, jd, jd])
    # duplicates (L <= 2) are summed, as scipy's coo->csr does
    key = rows * (L * L) + cols
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    uk, start = np.unique(key, return_index=True)
    vsum = np.add.reduceat(vals, start)
    rows, cols = uk // (L * L), uk % (L * L)
    offs = np.zeros(L * L + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=L * L), out=offs[1:])
    return vsum, cols, offs


def _maxcut_unit(n, i, j, device=None):
    """Dedupe undirected pairs on (min, max) and build the symmetric unit-weight CSR
    (J = -1/2 per edge, columns sorted per row). ``device`` (a CUDA device index) runs
    the sorts with torch on that GPU -- the same arrays as the numpy path (both sort
    unique int64 keys), seconds instead of minutes at 10^8 spins."""
    if device is not None:
        import torch

        dev = torch.device("cuda", device)
        ti = torch.from_numpy(np.ascontiguousarray(i, dtype=np.int64)).to(dev)
        tj = torch.from_numpy(np.ascontiguousarray(j, dtype=np.int64)).to(dev)
        key = torch.unique(torch.minimum(ti, tj) * n + torch.maximum(ti, tj))  # sorted
        del ti, tj
        a, b = key // n, key % n
        m = int(key.numel())
        del key
        k2 = torch.sort(torch.cat([a * n + b, b * n + a])).values
        del a, b
        rows, cols = k2 // n, k2 % n
        del k2
        offs = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        offs[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
        out = cols.cpu().numpy(), offs.cpu().numpy()
        del rows, cols, offs
        torch.cuda.empty_cache()
        return np.full(2 * m, -0.5), out[0], out[1], m / 2.0
    key = np.unique(np.minimum(i, j).astype(np.int64) * n + np.maximum(i, j))
    a, b = key // n, key % n
    vals, cols, offs = _csr_from_pairs(n, a, b, np.full(len(a), -0.5))
    return vals, cols, offs, len(a) / 2.0


def erdos_renyi(n: int = 10**7, deg: int = 8, seed: int = 0, device=None):
    """(values, cols, offsets, cut_offset) for the E7 graph (Appendix A ``er``)."""
    rng = np.random.default_rng(seed)
    m = n * deg // 2
    i = rng.integers(0, n, m)
    j = rng.integers(0, n, m)
    keep = i != j
    return _maxcut_unit(n, i[keep], j[keep], device)


def random_regular3(n: int = 10**8, seed: int = 0, device=None):
    """(values, cols, offsets, cut_offset) for the R8 graph (Appendix A ``reg3``)."""
    rng = np.random.default_rng(seed)
    stubs = rng.permutation(np.repeat(np.arange(n, dtype=np.int64), 3))
    i, j = stubs[0::2], stubs[1::2]
    keep = i != j
    return _maxcut_unit(n, i[keep], j[keep], device)
