"""DOCH / ADOCH solver entry points with the reference's signatures.

Drop-in for dc/solvers/doch.py (``doch_solve`` :169, ``adoch_solve`` :248,
``apply_T`` :94, ``hamiltonian`` :76, ``hamiltonian_gradient`` :84,
``attractor`` :55, ``initial_state`` :132) and dc/solvers/__init__.py
(``solve`` :40). Results are ``SolveResult`` / ``TraceRecord`` with the fields
of dc/solvers/common.py:21-43.

Every iteration runs on the GPU (libdcx.so): the host only uploads x0 (drawn
with numpy PCG64 exactly as the reference does), then drains the device
history ring chunk by chunk, replays ``callbacks`` in iteration order and
builds the trace. ``solve_replicas`` exposes the batched form (R independent
replicas in one launch sequence), which is what restarts, ``tune_eta`` and
the benchmark use.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field, replace
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

from . import _native
from .coupling import device_context
from .model import dehomogenize, homogenized_instance
from .params import SolverParams, derive_params

CONVERGENCE_TOL = 1e-10  # dc/solvers/doch.py:33
DESCENT_WARN_TOL = 1e-9  # dc/solvers/doch.py:34
SOLVER_NAMES = ("doch", "adoch")
DEFAULT_PRECISION = "f64"


@dataclass
class TraceRecord:
    iteration: int
    elapsed_s: float
    energy: float
    best_energy: float
    cut_value: Optional[float] = None
    event: Optional[str] = None


@dataclass
class SolveResult:
    solver: str
    spins: np.ndarray
    energy: float
    iterations: int
    stop_reason: str
    trace: list = field(default_factory=list)
    seed: Optional[int] = None
    x: Optional[np.ndarray] = None
    h_values: Optional[list] = None
    accepted: Optional[list] = None
    states: Optional[list] = None
    device_seconds: Optional[float] = None
    path: Optional[str] = None


@dataclass(frozen=True)
class HamiltonianView:
    coupling: object
    alpha: float
    beta: float

    def __post_init__(self):
        if not (self.alpha > 0 and self.beta > 0):
            raise ValueError("alpha and beta must be positive")

    @classmethod
    def of(cls, instance_or_coupling, params: SolverParams) -> "HamiltonianView":
        J = getattr(instance_or_coupling, "coupling", instance_or_coupling)
        return cls(coupling=J, alpha=params.alpha, beta=params.beta)


def attractor(x, alpha: float, beta: float) -> float:
    """(beta/4) sum x^4 - (alpha/2) sum x^2 (dc/solvers/doch.py:55-63)."""
    x = np.asarray(x, dtype=np.float64)
    x2 = x * x
    return 0.25 * beta * float(x2 @ x2) - 0.5 * alpha * float(x2.sum())


def _check_vec(view, x):
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (view.coupling.n,):
        raise ValueError("dimension mismatch")
    return x


def apply_T(view: HamiltonianView, x, precision: str = DEFAULT_PRECISION) -> np.ndarray:
    """cbrt((J + alpha I) x / beta) on the device (dc/solvers/doch.py:94-103)."""
    x = _check_vec(view, x)
    tx, _ = device_context(view.coupling).apply(x[None, :], view.alpha, view.beta, precision, True, False)
    return tx[0]


def hamiltonian(view: HamiltonianView, x, precision: str = DEFAULT_PRECISION) -> float:
    """H(x) = beta/4 sum x^4 - 1/2 x.(J + alpha I) x (dc/solvers/doch.py:76-81)."""
    x = _check_vec(view, x)
    _, h = device_context(view.coupling).apply(x[None, :], view.alpha, view.beta, precision, False, True)
    return float(h[0])


def hamiltonian_gradient(view: HamiltonianView, x) -> np.ndarray:
    """beta x^3 - Jx - alpha x (dc/solvers/doch.py:84-87)."""
    x = _check_vec(view, x)
    jx = device_context(view.coupling).matvec(x[None, :])[0]
    return view.beta * x**3 - jx - view.alpha * x


def initial_state(n: int, alpha: float, beta: float, rng: np.random.Generator) -> np.ndarray:
    """U(-lam, lam)^n, zeros re-drawn (dc/solvers/doch.py:132-145), numpy PCG64."""
    lam = np.sqrt(alpha / beta)
    x = rng.uniform(-lam, lam, size=n)
    while np.any(x == 0.0):
        z = x == 0.0
        x[z] = rng.uniform(-lam, lam, size=int(z.sum()))
    return x


def _event_name(solver: str, ev: int) -> Optional[str]:
    if solver == "doch":
        return "descent_violation" if ev & _native.EV_DESCENT else None
    if ev & _native.EV_ACCEPTED:
        return "momentum_accepted"
    if ev & _native.EV_REJECTED:
        return "momentum_rejected"
    return None


class _ReplicaTrace:
    """Host side of one replica: rebuilds TraceRecords from the device history."""

    def __init__(self, solver, cut_offset, callbacks, offset):
        self.solver = solver
        self.cut_offset = cut_offset
        self.callbacks = tuple(callbacks)
        self.offset = offset
        self.trace = []
        self.best = np.inf
        self.h = []
        self.ev = []
        self.done = 0

    def feed(self, h, e, t, ev):
        for k in range(len(h)):
            kk = self.done + k
            self.h.append(float(h[k]))
            self.ev.append(int(ev[k]))
            if ev[k] & _native.EV_RECORDED:
                E = float(e[k])
                if E < self.best:
                    self.best = E
                rec = TraceRecord(iteration=kk, elapsed_s=float(t[k]) + self.offset, energy=E,
                                  best_energy=self.best,
                                  cut_value=None if self.cut_offset is None else self.cut_offset - E,
                                  event=_event_name(self.solver, int(ev[k])) if kk > 0 else None)
                self.trace.append(rec)
                for cb in self.callbacks:
                    cb(rec)
        self.done += len(h)


def solve_replicas(instance, solver: str, alpha, beta, x0, *, max_iters: int = 1000, lookback_q: int = 5,
                   window_mode: str = "economy", trace_stride: int = 1, time_budget: Optional[float] = None,
                   record_states: bool = False, precision: str = "f32", path: str = "auto",
                   seeds: Optional[Sequence[int]] = None, callbacks=(), chunk: int = 0,
                   device: Optional[int] = None) -> list:
    """Run R independent replicas (rows of ``x0``) of DOCH/ADOCH in one batch.

    ``alpha``/``beta`` are scalars or length-R arrays (tune_eta passes one
    (alpha, beta) per candidate). Returns one SolveResult per replica.
    """
    if solver not in SOLVER_NAMES:
        raise ValueError(f"unknown solver {solver!r}")
    if window_mode not in ("economy", "exact"):
        raise ValueError("window_mode must be 'economy' or 'exact'")
    t_entry = time.perf_counter()
    J = instance.coupling
    X0 = np.atleast_2d(np.asarray(x0, dtype=np.float64))
    R = X0.shape[0]
    ctx = device_context(J, device)
    prm = _native.Params(
        solver=_native.SOLVER[solver], window_mode=_native.WINDOW[window_mode],
        precision=_native.PRECISION[precision], lookback_q=int(lookback_q), max_iters=int(max_iters),
        trace_stride=int(trace_stride), time_budget_s=-1.0 if time_budget is None else float(time_budget),
        conv_tol=CONVERGENCE_TOL, descent_tol=DESCENT_WARN_TOL, record_states=int(bool(record_states)),
        path=_native.PATH[path], chunk=int(chunk), reserved=0)
    ctx.begin(prm, alpha, beta, X0)
    offset = time.perf_counter() - t_entry
    cut_offset = getattr(instance, "cut_offset", None)
    reps = [_ReplicaTrace(solver, cut_offset, callbacks if R == 1 else (), offset) for _ in range(R)]
    live = True
    while live:
        live = ctx.step()
        for r, rt in enumerate(reps):
            s = ctx.summary(r)
            if s.n_hist > rt.done:
                rt.feed(*ctx.history(r, rt.done, s.n_hist - rt.done))
    best = ctx.best_spins().astype(np.float64)
    xs = ctx.state()
    dev_s = ctx.device_seconds()
    out = []
    for r, rt in enumerate(reps):
        s = ctx.summary(r)
        it = int(s.iterations)
        if s.descent_warn >= 0 and solver == "doch":
            k = int(s.descent_warn)
            warnings.warn(f"Hamiltonian increased by {rt.h[k] - rt.h[k - 1]:.3e} at iteration {k}",
                          RuntimeWarning, stacklevel=3)
        accepted = None
        if solver == "adoch":
            accepted = [True] + [bool(rt.ev[k + 1] & _native.EV_ACCEPTED) for k in range(1, it)] if it else []
        states = None
        if record_states:
            st = ctx.states(r, it)
            states = [st[k].copy() for k in range(it + 1)]
        out.append(SolveResult(
            solver=solver, spins=best[r], energy=float(s.best_energy), iterations=it,
            stop_reason=_native.STOP.get(int(s.stop_reason), "max_iters"), trace=rt.trace,
            seed=None if seeds is None else seeds[r], x=xs[r], h_values=rt.h, accepted=accepted, states=states,
            device_seconds=dev_s, path=_native.PATH_NAME.get(int(s.path_used))))
    return out


def _prepare(instance, params: SolverParams, x0):
    inst = homogenized_instance(instance)
    n = inst.coupling.n
    if x0 is None:
        x = initial_state(n, params.alpha, params.beta, np.random.default_rng(params.seed))
    else:
        x = np.array(x0, dtype=np.float64)
        if x.shape != (n,):
            raise ValueError(f"x0 has length {x.shape}, expected {n}")
        if not np.any(x != 0.0):
            raise ValueError("x0 must not be the zero vector")
    return inst, x


def _single(solver, instance, params, x0, callbacks, trace_stride, record_states, window_mode, precision, path):
    inst, x = _prepare(instance, params, x0)
    res = solve_replicas(inst, solver, params.alpha, params.beta, x[None, :], max_iters=params.max_iters,
                         lookback_q=params.lookback_q, window_mode=window_mode, trace_stride=trace_stride,
                         time_budget=params.time_budget, record_states=record_states, precision=precision,
                         path=path, seeds=[params.seed], callbacks=callbacks)[0]
    if getattr(instance, "field", None) is not None:
        res = replace(res, spins=dehomogenize(res.spins))
    return res


def doch_solve(instance, params: SolverParams, x0=None, callbacks: Iterable[Callable] = (), trace_stride: int = 1,
               record_states: bool = False, precision: str = DEFAULT_PRECISION, path: str = "auto") -> SolveResult:
    """Plain fixed-point iteration x <- T(x) (dc/solvers/doch.py:169-245)."""
    return _single("doch", instance, params, x0, callbacks, trace_stride, record_states, "economy", precision, path)


def adoch_solve(instance, params: SolverParams, x0=None, callbacks: Iterable[Callable] = (), trace_stride: int = 1,
                record_states: bool = False, window_mode: str = "economy", precision: str = DEFAULT_PRECISION,
                path: str = "auto") -> SolveResult:
    """Accelerated iteration with a look-back window (dc/solvers/doch.py:248-356)."""
    if window_mode not in ("economy", "exact"):
        raise ValueError("window_mode must be 'economy' or 'exact'")
    return _single("adoch", instance, params, x0, callbacks, trace_stride, record_states, window_mode, precision,
                   path)


def solve(instance, solver: str, seed: int = 0, eta: float = 1.0, lookback_q: int = 5,
          budget_iters: Optional[int] = None, budget_seconds: Optional[float] = None,
          params: Optional[SolverParams] = None, trace_stride: Optional[int] = None, callbacks=(),
          **knobs) -> SolveResult:
    """Front door (dc/solvers/__init__.py:40-108), DOCH/ADOCH branch.

    The reference's baseline solvers (SA, bSB, SimCIM, SIA) are out of scope
     and raise ``ValueError``.
    """
    if solver not in SOLVER_NAMES:
        raise ValueError(f"unknown solver {solver!r}; this build provides {SOLVER_NAMES}")
    hom = homogenized_instance(instance)
    if params is None:
        params = derive_params(hom.coupling, eta=eta, lookback_q=lookback_q,
                               max_iters=budget_iters if budget_iters is not None else 1000,
                               time_budget=budget_seconds, seed=seed)
    else:
        params = replace(params, seed=seed,
                         max_iters=budget_iters if budget_iters is not None else params.max_iters,
                         time_budget=budget_seconds if budget_seconds is not None else params.time_budget)
    fn = doch_solve if solver == "doch" else adoch_solve
    res = fn(hom, params, callbacks=callbacks, trace_stride=trace_stride or 1, **knobs)
    if getattr(instance, "field", None) is not None:
        res = replace(res, spins=dehomogenize(res.spins))
    return res
