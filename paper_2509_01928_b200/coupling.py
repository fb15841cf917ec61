"""Coupling storage with the reference's constructors (dc/coupling.py).

``DenseCoupling`` and ``CsrCoupling`` keep the reference's fields and
invariants (symmetric, zero diagonal, sorted CSR columns) so existing callers
construct them unchanged; reference objects themselves are also accepted
anywhere a coupling is expected (duck typing on ``array`` or on
``values / col_indices / row_offsets``). The device copy lives in a
:class:`~paper_2509_01928_b200._native.Context` cached per coupling object
and uploaded once (``dcx_set_csr`` / ``dcx_set_dense``); a
:class:`ProceduralCoupling` uploads only (n, seed) (``dcx_set_procedural``).
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native


class CouplingError(ValueError):
    """Raised when a matrix violates the coupling invariants (dc/coupling.py:23-24)."""


class CouplingMatrix:
    n: int
    value_kind: str

    def to_dense(self) -> np.ndarray:
        raise NotImplementedError


class DenseCoupling(CouplingMatrix):
    """Full symmetric float64 coupling (dc/coupling.py:71-112)."""

    def __init__(self, array, value_kind: str = "real", validate: bool = True):
        array = np.asarray(array, dtype=np.float64)
        if array.ndim != 2 or array.shape[0] != array.shape[1]:
            raise CouplingError(f"expected square array, got shape {array.shape}")
        self.array = array
        self.array.setflags(write=False)
        self.n = array.shape[0]
        self.value_kind = value_kind
        if validate:
            self.validate()

    def validate(self):
        a = self.array
        if not np.all(np.isfinite(a)):
            raise CouplingError("couplings must be finite")
        if np.any(np.diagonal(a) != 0.0):
            raise CouplingError("diagonal must be zero")
        if not np.array_equal(a, a.T):
            raise CouplingError("coupling matrix must be symmetric")

    def to_dense(self):
        return self.array

    def abs_row_sums(self):
        return np.abs(self.array).sum(axis=1)

    def offdiag_moments(self):
        return float(self.array.sum()), float((self.array * self.array).sum())


class CsrCoupling(CouplingMatrix):
    """Compressed sparse row coupling (dc/coupling.py:115-206).

    Validation is vectorised (the reference loops over rows in Python,
    dc/coupling.py:166-171, which is prohibitive at 10^7-10^8 rows).
    """

    def __init__(self, n, values, col_indices, row_offsets, value_kind: str = "real", validate: bool = True):
        self.n = int(n)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int64)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        for a in (self.values, self.col_indices, self.row_offsets):
            a.setflags(write=False)
        self.value_kind = value_kind
        if validate:
            self.validate()

    @classmethod
    def from_scipy(cls, m, value_kind: str = "real", validate: bool = True):
        m = m.tocsr()
        m.sort_indices()
        return cls(m.shape[0], m.data, m.indices, m.indptr, value_kind, validate=validate)

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def validate(self):
        n, ro, ci, v = self.n, self.row_offsets, self.col_indices, self.values
        if ro.shape != (n + 1,):
            raise CouplingError("row_offsets must have length n+1")
        if ro[0] != 0 or np.any(np.diff(ro) < 0):
            raise CouplingError("row_offsets must be nondecreasing and start at 0")
        if ro[-1] != len(v) or len(v) != len(ci):
            raise CouplingError("values/col_indices length must match row_offsets[-1]")
        if len(ci) and (ci.min() < 0 or ci.max() >= n):
            raise CouplingError("column index out of range")
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
        if np.any(ci == rows):
            raise CouplingError("stored diagonal entry")
        same_row = rows[1:] == rows[:-1]
        if np.any(same_row & (np.diff(ci) <= 0)):
            raise CouplingError("column indices not strictly increasing within a row")
        if not np.all(np.isfinite(v)):
            raise CouplingError("couplings must be finite")
        # symmetry: the transposed (col, row) keys must be the same multiset with equal values
        key = rows * n + ci
        tkey = ci * n + rows
        order = np.argsort(tkey, kind="stable")
        if not (np.array_equal(tkey[order], key) and np.array_equal(v[order], v)):
            raise CouplingError("coupling matrix must be symmetric")

    def to_dense(self):
        out = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    def abs_row_sums(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_offsets))
        return np.bincount(rows, weights=np.abs(self.values), minlength=self.n)

    def offdiag_moments(self):
        return float(self.values.sum()), float((self.values * self.values).sum())


_PROCEDURAL_FORMULAS = ("sin_product",)  # dc/coupling.py:297-299


class ProceduralCoupling(CouplingMatrix):
    """Coupling defined by a formula, never stored (dc/coupling.py:209-290).

    ``sin_product``: ``J_ij = sin(i*j + seed)`` on 0-based indices, zero on the
    diagonal (dc/coupling.py:293-294). Every product, energy and moment runs on
    the device, where the kernels regenerate the entries (libdcx
    ``dcx_set_procedural``); :meth:`block` and :meth:`entry` materialise tiles
    on the host for inspection, as the reference's do.
    """

    def __init__(self, n: int, seed: int = 100, formula: str = "sin_product", block_size: int = 1024):
        if n < 2:
            raise CouplingError("procedural matrices need n >= 2")
        self.n = int(n)
        self.seed = int(seed)
        self.formula = formula
        self.block_size = int(block_size)
        self.value_kind = "real"
        if formula not in _PROCEDURAL_FORMULAS:
            raise CouplingError(f"unknown procedural formula {formula!r}")

    @staticmethod
    def _sin_product(i, j, seed):
        return np.sin(i * j + float(seed))

    def entry(self, i: int, j: int) -> float:
        if i == j:
            return 0.0
        return float(self._sin_product(np.asarray(i), np.asarray(j), self.seed))

    def block(self, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
        for lo, hi in ((r0, r1), (c0, c1)):
            if not (0 <= lo <= hi <= self.n):
                raise ValueError(f"invalid index range [{lo}, {hi}) for n={self.n}")
        rows = np.arange(r0, r1)[:, None]
        cols = np.arange(c0, c1)[None, :]
        out = self._sin_product(rows, cols, self.seed)
        diag = rows == cols
        return np.where(diag, 0.0, out) if diag.any() else out

    def to_dense(self):
        return self.block(0, self.n, 0, self.n)

    def _row_stats(self) -> np.ndarray:
        return device_context(self).proc_row_stats()

    def abs_row_sums(self):
        return self._row_stats()[:, 2].copy()

    def offdiag_moments(self):
        st = self._row_stats()
        return float(st[:, 0].sum()), float(st[:, 1].sum())

    def nnz_offdiag(self) -> int:
        return self.n * (self.n - 1)

    def validate(self, samples: int = 64, seed: int = 0) -> None:
        """Spot-check symmetry and the zero diagonal on random index pairs (dc/coupling.py:276-290)."""
        rng = np.random.default_rng(seed)
        ii = rng.integers(0, self.n, size=samples)
        jj = rng.integers(0, self.n, size=samples)
        for i, j in zip(ii, jj):
            if self.entry(int(i), int(j)) != self.entry(int(j), int(i)):
                raise CouplingError(f"asymmetric procedural entry at ({i}, {j})")
        if any(self.entry(int(i), int(i)) != 0.0 for i in ii):
            raise CouplingError("procedural diagonal must be zero")


def gen_procedural_sin(n: int, seed: int = 100) -> ProceduralCoupling:
    """``entry(i, j) = sin(i * j + seed)`` for i != j (dc/generate.py:115-123)."""
    return ProceduralCoupling(n, seed=seed, formula="sin_product")


# ------------------------------------------------------------ device cache

_ctx_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_ctx_by_id: dict = {}


def is_dense(J) -> bool:
    return hasattr(J, "array")


def is_csr(J) -> bool:
    return all(hasattr(J, a) for a in ("values", "col_indices", "row_offsets"))


def is_procedural(J) -> bool:
    return hasattr(J, "formula") and hasattr(J, "seed") and not is_dense(J) and not is_csr(J)


def _upload(ctx, J):
    if is_dense(J):
        ctx.set_dense(J.array)
    elif is_csr(J):
        ctx.set_csr(J.n, J.values, J.col_indices, J.row_offsets)
    elif is_procedural(J):
        ctx.set_procedural(J.n, J.seed, J.formula)
    else:
        raise CouplingError(f"unsupported coupling storage {type(J).__name__} (dense, CSR or procedural)")


def device_context(J, device: int | None = None, reload: bool = False) -> _native.Context:
    """The device copy of coupling ``J`` (uploaded on first use; ``reload``
    copies the host arrays again into the existing device buffers)."""
    try:
        ctx = _ctx_cache.get(J)
    except TypeError:
        ctx = _ctx_by_id.get(id(J))
    if ctx is not None and (device is None or ctx.device == device):
        if reload:
            _upload(ctx, J)
        return ctx
    ctx = _native.Context(device)
    ctx.device = device
    _upload(ctx, J)
    try:
        _ctx_cache[J] = ctx
    except TypeError:
        _ctx_by_id[id(J)] = ctx
    return ctx
