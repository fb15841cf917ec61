"""Solver parameters and their derivation (dc/spectral.py).

``derive_params`` follows dc/spectral.py:224-256: alpha = eta * lambda_max(-J)
(two-stage shifted power iteration below n = 1e4, Wigner estimate at or
above), beta = n sqrt(n) (alpha + max_i sum_j |J_ij|). The power iteration runs
entirely on the device (``dcx_power``: one cooperative kernel per stage). ``tune_eta`` runs all eta
candidates as one batch of replicas (one launch sequence instead of one solve
per candidate, dc/spectral.py:259-298).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .coupling import device_context, is_procedural

WIGNER_SIZE_THRESHOLD = 10_000
DEFAULT_ETA_GRID = (0.25, 0.5, 0.75, 1.0, 1.25, 1.5, 2.0)


@dataclass
class SolverParams:
    """Same fields, defaults and validation as dc/spectral.py:25-49."""

    alpha: float
    beta: float
    eta: float = 1.0
    lookback_q: int = 5
    max_iters: int = 1000
    time_budget: Optional[float] = None
    seed: int = 0

    def __post_init__(self):
        if not self.alpha > 0:
            raise ValueError("alpha must be > 0")
        if not self.beta > 0:
            raise ValueError("beta must be > 0")
        if not (0 < self.eta <= 2):
            raise ValueError("eta must lie in (0, 2]")
        if self.lookback_q < 1:
            raise ValueError("lookback_q must be >= 1")


def row_stats(J) -> np.ndarray:
    """[n][3] per-row (sum J_ij, sum J_ij^2, sum |J_ij|) over j != i, computed on the device
    (dcx_row_stats: one pass over the stored coupling, or a regeneration pass for a procedural
    one) -- offdiag_moments and abs_row_sums of dc/coupling.py:104-109, :197-206. At the
    BASELINE sizes the reference's host loops (np.add.at / bincount over 10^8 entries) take
    seconds to minutes."""
    return device_context(J).row_stats()


def _moments(J):
    st = row_stats(J)
    return float(st[:, 0].sum()), float(st[:, 1].sum())


def _abs_row_max(J) -> float:
    return float(row_stats(J)[:, 2].max())


def estimate_lambda_max_neg(J, method="auto", tol=1e-10, max_iters=20_000) -> float:
    """lambda_max(-J) (dc/spectral.py:192-221)."""
    if method not in ("auto", "power_iteration", "wigner"):
        raise ValueError(f"unknown spectral method {method!r}")
    if method == "auto":
        # procedural matrices: the moments cost one generation pass, a power step
        # regenerates the whole matrix (dc/spectral.py:203-216)
        if is_procedural(J):
            method = "wigner"
        else:
            method = "power_iteration" if J.n < WIGNER_SIZE_THRESHOLD else "wigner"
    if method == "wigner":
        s1, s2 = _moments(J)
        if s2 == 0.0:
            raise ValueError("degenerate all-zero coupling matrix")
        cnt = J.n * (J.n - 1)
        mean = s1 / cnt
        std = float(np.sqrt(max(s2 / cnt - mean * mean, 0.0)))
        est = 2.0 * std * float(np.sqrt(J.n))
        if est > 0:
            return est
    ctx = device_context(J)
    if is_procedural(J):
        return _power_procedural(ctx, J.n, tol, max_iters)
    # the reference's seeded restart vector (dc/spectral.py:84-86), drawn once on the host
    r = np.random.default_rng(0).standard_normal(J.n)
    r /= np.linalg.norm(r)
    rho = ctx.power(False, 0.0, tol, max_iters, r)[0]  # whole loop on the device (dcx_power)
    if rho == 0.0:
        raise ValueError("coupling matrix must have at least one nonzero entry")
    dom, _, _, ok = ctx.power(True, rho, tol, max_iters, r)
    if not ok:
        warnings.warn("shifted power iteration did not converge; using best estimate", RuntimeWarning)
    return dom - rho


def _power_core(apply_m, n, tol, max_iters, seed=0):
    """dc/spectral.py:60-111 with the products on the device (procedural couplings,
    which dcx_power does not cover): the loop and its n-vector norms stay on the host."""
    v = np.full(n, 1.0 / np.sqrt(n))
    restarted, best_resid, since_improve = False, np.inf, 0
    mag = rayleigh = 0.0
    k = 0
    while k < max_iters:
        w = apply_m(v)
        mag = float(np.linalg.norm(w))
        if mag == 0.0:
            if restarted:
                return 0.0, 0.0, k, False
            v = np.random.default_rng(seed).standard_normal(n)
            v /= np.linalg.norm(v)
            restarted = True
            k += 1
            continue
        rayleigh = float(v @ w)
        resid = float(np.linalg.norm(w - rayleigh * v)) / mag
        if resid <= tol:
            return mag, rayleigh, k + 1, True
        if resid < 0.999 * best_resid:
            best_resid, since_improve = resid, 0
        else:
            since_improve += 1
            if since_improve > 50 and not restarted:
                v = np.random.default_rng(seed).standard_normal(n)
                v /= np.linalg.norm(v)
                restarted, since_improve = True, 0
                k += 1
                continue
        v = w / mag
        k += 1
    return mag, rayleigh, k, False


def _power_procedural(ctx, n, tol, max_iters):
    """Two-stage shifted power iteration (dc/spectral.py:143-171) over device products."""
    rho = _power_core(lambda v: -ctx.matvec(v[None, :])[0], n, tol, max_iters)[0]
    if rho == 0.0:
        raise ValueError("coupling matrix must have at least one nonzero entry")
    dom, _, _, ok = _power_core(lambda v: rho * v - ctx.matvec(v[None, :])[0], n, tol, max_iters)
    if not ok:
        warnings.warn("shifted power iteration did not converge; using best estimate", RuntimeWarning)
    return dom - rho


def derive_params(J, eta=1.0, method="auto", lookback_q=5, max_iters=1000, time_budget=None, seed=0,
                  tol=1e-10, power_iters=20_000) -> SolverParams:
    """alpha = eta lambda_max(-J); beta = n sqrt(n) (alpha + max row |J|_1) (dc/spectral.py:224-256)."""
    if not (0 < eta <= 2):
        raise ValueError("eta must lie in (0, 2]")
    lam = estimate_lambda_max_neg(J, method=method, tol=tol, max_iters=power_iters)
    if lam <= 0:
        raise ValueError("spectral estimate is nonpositive; cannot derive alpha")
    alpha = eta * lam
    beta = J.n * np.sqrt(J.n) * (alpha + _abs_row_max(J))
    return SolverParams(alpha=float(alpha), beta=float(beta), eta=eta, lookback_q=lookback_q,
                        max_iters=max_iters, time_budget=time_budget, seed=seed)


def tune_eta(instance, candidate_etas: Sequence[float], probe_iters: int = 10, seed: int = 0, method="auto",
             tol: float = 1e-8, precision: str = "f64") -> float:
    """Pick eta by short DOCH probes, all candidates as one replica batch
    (dc/spectral.py:259-298; ties go to the smaller eta)."""
    from .model import homogenized_instance
    from .solvers import initial_state, solve_replicas

    if not candidate_etas:
        raise ValueError("candidate eta list is empty")
    if probe_iters < 1:
        raise ValueError("probe_iters must be >= 1")
    inst = homogenized_instance(instance)
    J = inst.coupling
    try:
        lam = estimate_lambda_max_neg(J, method=method, tol=tol)
    except ValueError:
        return float(min(candidate_etas))
    row_max = _abs_row_max(J)
    n = J.n
    etas = sorted(candidate_etas)
    alphas = np.array([eta * lam for eta in etas])
    betas = n * np.sqrt(n) * (alphas + row_max)
    # the reference builds SolverParams per candidate (dc/spectral.py:288-292): an eta outside
    # (0, 2] raises its ValueError -- here before the batch, with the same message
    for eta, a, b in zip(etas, alphas, betas):
        SolverParams(alpha=float(a), beta=float(b), eta=eta, max_iters=probe_iters, seed=seed)
    x0 = np.stack([initial_state(n, a, b, np.random.default_rng(seed)) for a, b in zip(alphas, betas)])
    res = solve_replicas(inst, "doch", alphas, betas, x0, max_iters=probe_iters, trace_stride=probe_iters,
                         precision=precision, seeds=[seed] * len(etas))
    best_eta, best_e = None, np.inf
    for eta, r in zip(etas, res):
        e = r.trace[-1].energy
        if e < best_e:
            best_e, best_eta = e, eta
    return float(best_eta)
