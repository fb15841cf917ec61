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

import os
import sys
import time
import warnings
from dataclasses import dataclass, field, replace
from collections.abc import Sequence
from typing import Callable, Iterable, Optional

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


class LazyTrace(Sequence):
    """The trace of one replica as columns; TraceRecords are built on access
    (a stride-1 trace of 1024 replicas x 1000 iterations would otherwise be a
    million Python objects)."""

    def __init__(self, solver, iters, elapsed, energy, cut_offset, ev, best=None):
        self.solver = solver
        self.iters = iters
        self.elapsed = elapsed
        self.energy = energy
        self._best = best
        self.cut_offset = cut_offset
        self.ev = ev

    @property
    def best(self):
        if self._best is None:
            self._best = np.minimum.accumulate(self.energy) if len(self.energy) else self.energy
        return self._best

    def __len__(self):
        return len(self.iters)

    def _rec(self, i):
        E = float(self.energy[i])
        k = int(self.iters[i])
        return TraceRecord(iteration=k, elapsed_s=float(self.elapsed[i]), energy=E,
                           best_energy=float(self.best[i]),
                           cut_value=None if self.cut_offset is None else self.cut_offset - E,
                           event=_event_name(self.solver, int(self.ev[i])) if k > 0 else None)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._rec(j) for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._rec(i)

    def first_reach_time(self, threshold: float, use_cut: bool = True):
        """First elapsed_s whose best-so-far quality reaches threshold (dc/bench.py:219-231)."""
        q = (self.cut_offset - self.best) if (use_cut and self.cut_offset is not None) else -self.best
        hit = np.nonzero(q >= threshold)[0]
        return float(self.elapsed[hit[0]]) if len(hit) else None


def _collect(ctx, r, solver, cut_offset, offset):
    s = ctx.summary(r)
    h, e, t, ev = ctx.history(r, 0, int(s.n_hist))
    ks = np.nonzero((ev & _native.EV_RECORDED) != 0)[0]
    return s, h, ev, LazyTrace(solver, ks, t[ks] + offset, e[ks], cut_offset, ev[ks])


def solve_replicas(instance, solver: str, alpha, beta, x0, *, max_iters: int = 1000, lookback_q: int = 5,
                   window_mode: str = "economy", trace_stride: int = 1, time_budget: Optional[float] = None,
                   record_states: bool = False, precision: str = "f32", path: str = "auto",
                   seeds: Optional[Sequence[int]] = None, callbacks=(), chunk: int = 0,
                   device: Optional[int] = None, reupload: bool = False) -> list:
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
    ctx = device_context(J, device, reload=reupload)
    prm = _native.Params(
        solver=_native.SOLVER[solver], window_mode=_native.WINDOW[window_mode],
        precision=_native.PRECISION[precision], lookback_q=int(lookback_q), max_iters=int(max_iters),
        trace_stride=int(trace_stride), time_budget_s=-1.0 if time_budget is None else float(time_budget),
        conv_tol=CONVERGENCE_TOL, descent_tol=DESCENT_WARN_TOL, record_states=int(bool(record_states)),
        path=_native.PATH[path], chunk=int(chunk), reserved=0)
    ctx.begin(prm, alpha, beta, X0)
    offset = time.perf_counter() - t_entry
    cut_offset = getattr(instance, "cut_offset", None)
    if callbacks and R == 1:
        # stream records to the callbacks in iteration order, chunk by chunk
        # the running best over recorded iterations is carried across chunks, so every
        # record's best_energy is the TraceCollector's (dc/solvers/common.py:70-73, :89-90)
        fed = 0
        run_best = np.inf
        live = True
        while live:
            live = ctx.step()
            s = ctx.summary(0)
            if s.n_hist > fed:
                h, e, t, ev = ctx.history(0, fed, int(s.n_hist) - fed)
                for k in np.nonzero(ev & _native.EV_RECORDED)[0]:
                    run_best = min(run_best, float(e[k]))
                    rec = LazyTrace(solver, np.array([fed + k]), t[k:k + 1] + offset, e[k:k + 1], cut_offset,
                                    ev[k:k + 1], best=np.array([run_best]))[0]
                    for cb in callbacks:
                        cb(rec)
                fed = int(s.n_hist)
    else:
        ctx.run()
    path_used = _native.PATH_NAME.get(int(ctx.summary(0).path_used))
    return _assemble_detached(ctx, solver, R, offset, cut_offset, seeds, path_used, record_states)


_LAZY = object()  # a SolveResult field read from the detached run on first access


class _LazySolveResult(SolveResult):
    """SolveResult whose bulk fields (spins, x, trace, h_values, accepted) stay on the
    device / in the pinned history until first read (a plain SolveResult otherwise:
    dataclasses.fields / replace / asdict see the materialised values)."""

    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if v is _LAZY:
            v = object.__getattribute__(self, "_bulk").field(name, object.__getattribute__(self, "_r"))
            object.__setattr__(self, name, v)
        return v


class _Bulk:
    """The detached outputs of one batch, copied to the host in bulk on first use."""

    def __init__(self, res, solver, R, offset, cut_offset, iters, nh):
        self.res, self.solver, self.R, self.offset, self.cut_offset = res, solver, R, offset, cut_offset
        self.iters, self.nh = iters, nh
        self._x = self._s = self._hist = None

    def _history(self):
        if self._hist is None:
            K = int(self.nh.max()) if self.R else 0
            H, E, T, EV = self.res.history_all(K)
            if self.offset:
                T += self.offset
            rec = (EV & _native.EV_RECORDED) != 0
            full = rec.sum(axis=1) == self.nh
            self._hist = (H, E, T, EV, rec, full, np.arange(K))
        return self._hist

    def field(self, kind, r):
        if kind == "x":  # (kind: the SolveResult field name)
            if self._x is None:
                self._x = self.res.state()
            return self._x[r]
        if kind == "spins":
            if self._s is None:
                self._s = self.res.best_spins().astype(np.float64)
            return self._s[r]
        H, E, T, EV, rec, full, ar = self._history()
        n_r = int(self.nh[r])
        if kind == "trace":
            evr = EV[r, :n_r]
            if full[r]:
                return LazyTrace(self.solver, ar[:n_r], T[r, :n_r], E[r, :n_r], self.cut_offset, evr)
            ks = np.nonzero(rec[r, :n_r])[0]
            return LazyTrace(self.solver, ks, T[r, ks], E[r, ks], self.cut_offset, evr[ks])
        if kind == "h_values":
            hr = H[r, :n_r]
            return hr if self.R > 1 else hr.tolist()
        if kind == "accepted":
            it = int(self.iters[r])
            evr = EV[r, :n_r]
            return ([True] + ((evr[2:it + 1] & _native.EV_ACCEPTED) != 0).tolist()) if it else []
        raise KeyError(kind)


def _warn_site(stacklevel):
    """warnings.warn(msg, RuntimeWarning, stacklevel) from the caller of this function's caller,
    with the frame looked up once for a batch of per-replica warnings (warn_explicit with the
    filename, line, module and registry warnings.warn would derive: the same filters apply)."""
    try:
        f = sys._getframe(stacklevel)
    except ValueError:
        g, fname, line = sys.__dict__, "sys", 1
    else:
        g, fname, line = f.f_globals, f.f_code.co_filename, f.f_lineno
    module = g.get("__name__", "<string>")
    registry = g.setdefault("__warningregistry__", {})
    return lambda msg: warnings.warn_explicit(msg, RuntimeWarning, fname, line, module, registry)


def _assemble_detached(ctx, solver, R, offset, cut_offset, seeds, path=None, record_states=False):
    """SolveResults of a finished run whose bulk arrays (final states, best spins, the
    history) are detached from the context and read only when a field is accessed: the
    energies, iterations and stop reasons come from the per-replica summaries."""
    dev_s = ctx.device_seconds()
    iters, stops, bests, nh, warn = ctx.summaries()
    states_l = None
    if record_states:
        states_l = []
        for r, it in enumerate(iters.tolist()):
            st = ctx.states(r, it)
            states_l.append([st[k].copy() for k in range(it + 1)])
    res = ctx.detach()
    warned = np.nonzero(warn >= 0)[0] if solver == "doch" else ()
    if len(warned):
        wd = res.warn_delta()
        warn_at = _warn_site(4)
        for r in warned:
            warn_at(f"Hamiltonian increased by {wd[r]:.3e} at iteration {int(warn[r])}")
    bulk = _Bulk(res, solver, R, offset, cut_offset, iters, nh)
    it_l, be_l = iters.tolist(), bests.tolist()
    stop_l = [_native.STOP.get(v, "max_iters") for v in stops.tolist()]
    out = []
    append = out.append
    L = _LAZY
    acc = L if solver == "adoch" else None
    seed_l = [None] * R if seeds is None else list(seeds)
    for r in range(R):
        o = _LazySolveResult(solver, L, be_l[r], it_l[r], stop_l[r], L, seed_l[r], L, L, acc,
                             None if states_l is None else states_l[r], dev_s, path)
        o._bulk = bulk
        o._r = r
        append(o)
    return out


def assemble_results(ctx, solver, R, best, xs, offset, cut_offset, seeds, path=None, record_states=False):
    """SolveResults of a finished run from the context's summaries and history
    (shared by solve_replicas and the row-partitioned driver)."""
    dev_s = ctx.device_seconds()
    path_used = path
    # bulk download of every replica's history, then per-replica views (no per-replica FFI calls)
    iters, stops, bests, nh, warn = ctx.summaries()
    K = int(nh.max()) if R else 0
    H, E, T, EV = ctx.history_all(K)
    if offset:
        T += offset
    rec = (EV & _native.EV_RECORDED) != 0
    # rows recorded at every iteration (trace_stride 1) become views of the bulk
    # arrays; the running best is computed on first use (LazyTrace.best)
    full = (rec.sum(axis=1) == nh).tolist()
    ar = np.arange(K)
    nh_l, it_l, be_l = nh.tolist(), iters.tolist(), bests.tolist()
    stop_l = [_native.STOP.get(v, "max_iters") for v in stops.tolist()]
    warned = np.nonzero(warn >= 0)[0] if solver == "doch" else ()
    warn_at = _warn_site(4) if len(warned) else None
    for r in warned:
        k = int(warn[r])
        warn_at(f"Hamiltonian increased by {H[r, k] - H[r, k - 1]:.3e} at iteration {k}")
    out = []
    append = out.append
    for r in range(R):
        n_r = nh_l[r]
        hr, evr = H[r, :n_r], EV[r, :n_r]
        if full[r]:
            trace = LazyTrace(solver, ar[:n_r], T[r, :n_r], E[r, :n_r], cut_offset, evr)
        else:
            ks = np.nonzero(rec[r, :n_r])[0]
            trace = LazyTrace(solver, ks, T[r, ks], E[r, ks], cut_offset, evr[ks])
        it = it_l[r]
        accepted = None
        if solver == "adoch":
            accepted = ([True] + ((evr[2:it + 1] & _native.EV_ACCEPTED) != 0).tolist()) if it else []
        states = None
        if record_states:
            st = ctx.states(r, it)
            states = [st[k].copy() for k in range(it + 1)]
        append(SolveResult(solver, best[r], be_l[r], it, stop_l[r], trace, None if seeds is None else seeds[r],
                           xs[r], hr if R > 1 else hr.tolist(), accepted, states, dev_s, path_used))
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


def profile_dominant_kernel(instance, alpha, beta, x0, *, solver: str = "doch", precision: str = "f32",
                            path: str = "auto", launches: int = 10, max_iters: int = 1000) -> dict:
    """Time the dominant kernel of a batched solve alone (CUDA events on the
    solver stream) and return its algorithmic work per launch."""
    J = instance.coupling
    X0 = np.atleast_2d(np.asarray(x0, dtype=np.float64))
    R, n = X0.shape
    ctx = device_context(J)
    prm = _native.Params(solver=_native.SOLVER[solver], window_mode=0, precision=_native.PRECISION[precision],
                         lookback_q=5, max_iters=int(max_iters), trace_stride=1, time_budget_s=-1.0,
                         conv_tol=CONVERGENCE_TOL, descent_tol=DESCENT_WARN_TOL, record_states=0,
                         path=_native.PATH[path], chunk=0, reserved=0)
    ctx.begin(prm, alpha, beta, X0)
    ms, kid = ctx.profile(launches)
    info = ctx.info()
    dense = bool(info.dense)
    tb = 8 if precision == "f64" else (2 if precision == "f16tc" else 4)
    if kid == 3:
        # one launch = iterations [0, 100) of the persistent kernel from x0 (every launch
        # restarts the same window, csrc/dcx_api.cu dcx_profile_kernel; no K2000 replica
        # converges before iteration 124, so all R replicas are live throughout). Work per
        # iteration: SURVEY.md §8d's 2 n^2 R -- ONE coupling product per replica, the
        # delta product J Dh; the exact sign product (int8, incremental) is not counted
        name = "dense_doch_kernel"
        iters = 100
        flops = iters * 2.0 * n * n * R
        byts = float(iters * R * n * (2 + 1))  # f16 + int8 operands of the next iteration
    elif R > 1 and info.lattice_L > 0 and precision == "f32" and R % 4 == 0 and os.environ.get("DCX_TORUS") == "1":
        # the lattice stencil pass (csrc/dcx_csr.cu pass_torus): two int8 bond arrays and
        # the state read once + written once (2 n + 8 R n bytes)
        name = "pass_torus"
        flops = 2.0 * info.nnz * R
        byts = float(2 * n + R * n * tb * 2)
    else:
        name = "pass_rv" if R > 1 else ("pass_r1w" if precision == "f32" and info.value_kind in (0, 1)
                                        else "pass_r1")
        vbytes = {0: 0, 1: 1, 2: 2, 3: 4, 4: 8}[info.value_kind]
        if info.value_kind in (3, 4):
            vbytes = tb
        flops = 2.0 * info.nnz * R
        byts = float(info.nnz * (4 + vbytes) + (n + 1) * 4 + R * n * tb * 2)
    return {"kernel": name, "ms_per_launch": ms, "iterations_per_launch": iters if kid == 3 else 1, "flops_per_launch": flops, "bytes_per_launch": byts,
            "bound": "tensor" if dense else "hbm", "kernel_id": kid}
