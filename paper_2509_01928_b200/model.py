"""Ising model helpers with the reference's names (dc/model.py).

Energies and cut values are evaluated on the GPU through ``dcx_energy``
(exact integer accumulation for integer couplings, so they match the
reference bit for bit). ``homogenize`` / ``dehomogenize`` are host-side input
transforms, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .coupling import CouplingError, CsrCoupling, DenseCoupling, device_context, is_csr, is_dense


def spins_from(x) -> np.ndarray:
    """sign with sign(0) = +1, as float64 (dc/model.py:31-33)."""
    return np.where(np.asarray(x) >= 0, 1.0, -1.0)


def validate_spins(s, n=None) -> np.ndarray:
    s = np.asarray(s, dtype=np.float64)
    if n is not None and s.shape != (n,):
        raise ValueError(f"spin vector has length {s.shape}, expected {n}")
    if not np.all(np.abs(s) == 1.0):
        raise ValueError("spin entries must be exactly -1 or +1")
    return s


@dataclass(frozen=True)
class ProblemInstance:
    """Coupling + optional field + metadata (dc/model.py:45-76)."""

    coupling: object
    field: Optional[np.ndarray] = None
    name: str = ""
    best_known: Optional[float] = None
    cut_offset: Optional[float] = None

    def __post_init__(self):
        if self.field is not None:
            h = np.ascontiguousarray(self.field, dtype=np.float64)
            if h.shape != (self.coupling.n,):
                raise ValueError("field length must equal coupling.n")
            if not np.all(np.isfinite(h)):
                raise ValueError("field entries must be finite")
            h.setflags(write=False)
            object.__setattr__(self, "field", h)

    @property
    def n(self) -> int:
        return self.coupling.n

    def cut_value_of(self, energy: float):
        return None if self.cut_offset is None else self.cut_offset - energy


def energies(J, S) -> np.ndarray:
    """E_r = -1/2 s_r^T J s_r for a batch of +-1 vectors (one device launch)."""
    S = np.atleast_2d(np.asarray(S, dtype=np.float64))
    if S.shape[1] != J.n:
        raise ValueError(f"vector length {S.shape[1]} does not match n={J.n}")
    return device_context(J).energy(S)


def energy(J, s) -> float:
    """Homogeneous Ising energy (dc/model.py:79-87).

    +-1 vectors go through the exact integer kernel; continuous vectors use
    ``-1/2 x.(Jx)`` with the device product.
    """
    s = np.asarray(s, dtype=np.float64)
    if s.shape != (J.n,):
        raise ValueError(f"vector length {s.shape} does not match n={J.n}")
    if np.all(np.abs(s) == 1.0):
        return float(energies(J, s[None, :])[0])
    y = device_context(J).matvec(s[None, :])[0]
    return -0.5 * float(s @ y)


def energy_with_field(J, h, s) -> float:
    h = np.asarray(h, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    if h.shape != (J.n,) or s.shape != (J.n,):
        raise ValueError("dimension mismatch between J, h, s")
    return energy(J, s) - float(h @ s)


def instance_energy(instance, s) -> float:
    if getattr(instance, "field", None) is None:
        return energy(instance.coupling, s)
    return energy_with_field(instance.coupling, instance.field, s)


def maxcut_to_ising(W):
    """J = -W/2 (dc/model.py:215-229)."""
    if is_dense(W):
        return DenseCoupling(-0.5 * np.asarray(W.array), value_kind="real", validate=False)
    if is_csr(W):
        return CsrCoupling(W.n, -0.5 * np.asarray(W.values), W.col_indices, W.row_offsets, value_kind="real",
                           validate=False)
    raise CouplingError("MAX-CUT conversion expects dense or CSR adjacency")


def cut_value(W, s) -> float:
    """Weight of edges crossing the partition (dc/model.py:232-258).

    cut = (sum_{i<j} W_ij - sum_{i<j} W_ij s_i s_j) / 2 = (w_upper + E_W(s)) / 2
    with E_W the device energy of W (exact for integer weights).
    """
    s = validate_spins(s, W.n)
    if is_dense(W):
        w_upper = float(np.triu(np.asarray(W.array), 1).sum())
    elif is_csr(W):
        w_upper = float(np.asarray(W.values).sum()) / 2.0
    else:
        raise CouplingError("cut_value expects dense or CSR adjacency")
    return (w_upper + float(energies(W, s[None, :])[0])) / 2.0


def homogenize(J, h):
    """Fold a field into one auxiliary spin (dc/model.py:169-193), dense/CSR only."""
    h = np.asarray(h, dtype=np.float64)
    if h.shape != (J.n,):
        raise ValueError("field length must equal J.n")
    n1 = J.n + 1
    if is_dense(J):
        out = np.zeros((n1, n1))
        out[: J.n, : J.n] = J.array
        out[: J.n, -1] = h
        out[-1, : J.n] = h
        return DenseCoupling(out, value_kind=J.value_kind, validate=False)
    if is_csr(J):
        import scipy.sparse as sp

        base = sp.csr_matrix((J.values, J.col_indices, J.row_offsets), shape=(J.n, J.n))
        col = sp.csr_matrix(h.reshape(-1, 1))
        full = sp.bmat([[base, col], [col.T, None]], format="csr")
        full.sort_indices()
        return CsrCoupling.from_scipy(full, value_kind=J.value_kind, validate=False)
    raise CouplingError("homogenize expects dense or CSR couplings")


def dehomogenize(sigma) -> np.ndarray:
    sigma = np.asarray(sigma, dtype=np.float64)
    if sigma.shape[0] < 2:
        raise ValueError("need at least 2 spins to dehomogenize")
    return sigma[-1] * sigma[:-1]


def homogenized_instance(instance):
    if getattr(instance, "field", None) is None:
        return instance
    return ProblemInstance(coupling=homogenize(instance.coupling, instance.field),
                           name=(instance.name + "+aux") if instance.name else "homogenized",
                           best_known=instance.best_known)
