"""ctypes binding of libdcx.so (include/dcx.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2509_01928_b200/csrc``). There is no fallback: if the library or a CUDA
device is missing, every solver entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libdcx.so"

DCX_OK = 0
DCX_E_INVALID = -1
DCX_E_CUDA = -2
DCX_E_NCCL = -3
DCX_E_OOM = -4
DCX_E_STATE = -5

SOLVER = {"doch": 0, "adoch": 1}
WINDOW = {"economy": 0, "exact": 1}
PRECISION = {"f64": 0, "f32": 1, "f16tc": 2}
PATH = {"auto": 0, "multipass": 1, "persistent": 2, "dense_tc": 3}
FORMULA = {"sin_product": 0}  # DCX_FORMULA_* (dc/coupling.py:297-299 _PROCEDURAL_FORMULAS)
PATH_NAME = {v: k for k, v in PATH.items()}
STOP = {1: "converged", 2: "max_iters", 3: "time_budget"}
EV_RECORDED, EV_DESCENT, EV_ACCEPTED, EV_REJECTED = 1, 2, 4, 8

# every exported symbol of include/dcx.h (checked by tests/test_abi.py)
EXPORTS = (
    "dcx_abi_version", "dcx_last_error", "dcx_create", "dcx_destroy", "dcx_set_csr", "dcx_set_dense",
    "dcx_coupling", "dcx_matvec", "dcx_apply", "dcx_energy", "dcx_solve_begin", "dcx_solve_step",
    "dcx_solve_run", "dcx_result_summary", "dcx_result_summaries", "dcx_result_history",
    "dcx_result_history_all", "dcx_result_best_spins", "dcx_result_state", "dcx_result_states",
    "dcx_result_device_seconds", "dcx_profile_kernel", "dcx_set_csr_block", "dcx_stream", "dcx_dist_begin",
    "dcx_dist_pass", "dcx_dist_control", "dcx_dist_poll", "dcx_dist_finish", "dcx_power",
    "dcx_set_procedural", "dcx_proc_row_stats", "dcx_row_stats", "dcx_gen_sparse_9bit", "dcx_gen_result", "dcx_validate_csr",
    "dcx_result_detach", "dcx_res_state", "dcx_res_best_spins", "dcx_res_history_all", "dcx_res_warn_delta",
    "dcx_result_free", "dcx_dist_pass_rows", "dcx_dist_reduce",
)
QSUM, QMAX = 5, 3  # DCX_QSUM / DCX_QMAX


class Params(C.Structure):
    _fields_ = [
        ("solver", C.c_int32), ("window_mode", C.c_int32), ("precision", C.c_int32),
        ("lookback_q", C.c_int32), ("max_iters", C.c_int64), ("trace_stride", C.c_int64),
        ("time_budget_s", C.c_double), ("conv_tol", C.c_double), ("descent_tol", C.c_double),
        ("record_states", C.c_int32), ("path", C.c_int32), ("chunk", C.c_int32), ("reserved", C.c_int32),
    ]


class Summary(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("stop_reason", C.c_int32), ("best_iter", C.c_int32),
        ("best_energy", C.c_double), ("n_hist", C.c_int64), ("descent_warn", C.c_int32),
        ("path_used", C.c_int32),
    ]


class CouplingInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nnz", C.c_int64), ("value_kind", C.c_int32), ("lanes", C.c_int32),
        ("scale", C.c_double), ("dense", C.c_int32), ("lattice_L", C.c_int32),
    ]


_lib = None

_P = C.c_void_p
_PD = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)
_PI32 = C.POINTER(C.c_int32)
_PI8 = C.POINTER(C.c_int8)


def load(path: Path | str | None = None):
    """Load libdcx.so once; raise RuntimeError if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # DCX_LIB: another build of the same ABI (A/B timing of kernel variants)
    p = Path(path) if path else Path(os.environ.get("DCX_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"libdcx.so not found at {p}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    _tune_host_heap()
    sig = {
        "dcx_abi_version": (C.c_int, []),
        "dcx_last_error": (C.c_char_p, [_P]),
        "dcx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
        "dcx_destroy": (None, [_P]),
        "dcx_set_csr": (C.c_int, [_P, C.c_int64, C.c_int64, _PI64, _PI64, _PD]),
        "dcx_set_dense": (C.c_int, [_P, C.c_int64, _PD]),
        "dcx_set_procedural": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32]),
        "dcx_proc_row_stats": (C.c_int, [_P, _PD]),
        "dcx_row_stats": (C.c_int, [_P, _PD]),
        "dcx_coupling": (C.c_int, [_P, C.POINTER(CouplingInfo)]),
        "dcx_matvec": (C.c_int, [_P, C.c_int32, _PD, _PD, C.c_int32]),
        "dcx_apply": (C.c_int, [_P, C.c_int32, _PD, _PD, _PD, _PD, _PD, C.c_int32]),
        "dcx_energy": (C.c_int, [_P, C.c_int32, _PI8, _PD]),
        "dcx_solve_begin": (C.c_int, [_P, C.POINTER(Params), C.c_int32, _PD, _PD, _PD]),
        "dcx_solve_step": (C.c_int, [_P, _PI32]),
        "dcx_solve_run": (C.c_int, [_P]),
        "dcx_result_summary": (C.c_int, [_P, C.c_int32, C.POINTER(Summary)]),
        "dcx_result_history": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, _PD, _PD, _PD, _PI32]),
        "dcx_result_summaries": (C.c_int, [_P, _PI64, _PI32, _PD, _PI64, _PI32]),
        "dcx_result_history_all": (C.c_int, [_P, C.c_int64, _PD, _PD, _PD, _PI32]),
        "dcx_result_best_spins": (C.c_int, [_P, _PI8]),
        "dcx_result_state": (C.c_int, [_P, _PD]),
        "dcx_result_states": (C.c_int, [_P, C.c_int32, _PD]),
        "dcx_result_device_seconds": (C.c_int, [_P, _PD]),
        "dcx_profile_kernel": (C.c_int, [_P, C.c_int32, _PD, _PI32]),
        "dcx_set_csr_block": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _PI64, _PI64, _PD]),
        "dcx_stream": (C.c_int, [_P, C.POINTER(_P)]),
        "dcx_dist_begin": (C.c_int, [_P, C.POINTER(Params), C.c_int32, _PD, _PD, _PD, _P, _P, _P, _P]),
        "dcx_dist_pass": (C.c_int, [_P]),
        "dcx_dist_control": (C.c_int, [_P]),
        "dcx_dist_pass_rows": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32]),
        "dcx_dist_reduce": (C.c_int, [_P]),
        "dcx_dist_poll": (C.c_int, [_P, _PI32, _PI64]),
        "dcx_dist_finish": (C.c_int, [_P]),
        "dcx_power": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double, C.c_int64, _PD, _PD, _PD, _PI64, _PI32]),
        "dcx_gen_sparse_9bit": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_uint64, _PI64]),
        "dcx_gen_result": (C.c_int, [_P, _PI64, _PI64, _PD]),
        "dcx_validate_csr": (C.c_int, [_P, C.c_int64, C.c_int64, _PI64, _PI64, _PD, _PI32, _PI64, _PI32]),
        "dcx_result_detach": (C.c_int, [_P, C.POINTER(_P)]),
        "dcx_res_state": (C.c_int, [_P, _PD]),
        "dcx_res_best_spins": (C.c_int, [_P, _PI8]),
        "dcx_res_history_all": (C.c_int, [_P, C.c_int64, _PD, _PD, _PD, _PI32]),
        "dcx_res_warn_delta": (C.c_int, [_P, _PD]),
        "dcx_result_free": (None, [_P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if path is None:
        _lib = lib
    return lib


def _tune_host_heap():
    """Serve large host arrays (result states, histories: tens of MB per batch) from the
    process heap instead of fresh mmap()s, so a freed batch's pages are reused by the next
    one instead of being unmapped and page-faulted (and zeroed by the kernel) again: glibc
    M_MMAP_MAX = 0, M_TRIM_THRESHOLD = 1 GiB. DCX_HEAP_TUNE=0 leaves the allocator alone."""
    if os.environ.get("DCX_HEAP_TUNE", "1") == "0":
        return
    try:
        libc = C.CDLL("libc.so.6")
        libc.mallopt(-4, 0)  # M_MMAP_MAX
        libc.mallopt(-1, 1 << 30)  # M_TRIM_THRESHOLD
    except (OSError, AttributeError):
        pass


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def check(rc: int, handle=None):
    if rc == DCX_OK:
        return
    lib = load()
    msg = lib.dcx_last_error(handle).decode() if handle is not None else lib.dcx_last_error(None).decode()
    if rc == DCX_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libdcx error {rc}: {msg}")


def default_device() -> int:
    return int(os.environ.get("DCX_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class Context:
    """Owns one dcx_ctx (stream + device copy of one coupling matrix)."""

    def __init__(self, device: int | None = None):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.dcx_create(default_device() if device is None else int(device), C.byref(h)))
        self.h = h
        self.n = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.dcx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_csr(self, n, values, col_indices, row_offsets):
        v = np.ascontiguousarray(values, dtype=np.float64)
        c = np.ascontiguousarray(col_indices, dtype=np.int64)
        r = np.ascontiguousarray(row_offsets, dtype=np.int64)
        check(self.lib.dcx_set_csr(self.h, int(n), int(len(v)), ptr(r, C.c_int64), ptr(c, C.c_int64),
                                   ptr(v, C.c_double)), self.h)
        self.n = int(n)

    def set_dense(self, array):
        a = np.ascontiguousarray(array, dtype=np.float64)
        check(self.lib.dcx_set_dense(self.h, int(a.shape[0]), ptr(a, C.c_double)), self.h)
        self.n = int(a.shape[0])

    def set_procedural(self, n, seed, formula="sin_product"):
        check(self.lib.dcx_set_procedural(self.h, int(n), int(seed), FORMULA[formula]), self.h)
        self.n = int(n)

    def row_stats(self) -> np.ndarray:
        """[n][3]: per-row sum, sum of squares and sum of |J_ij| over j != i (any coupling)."""
        out = np.empty((self.n, 3))
        check(self.lib.dcx_row_stats(self.h, ptr(out, C.c_double)), self.h)
        return out

    def proc_row_stats(self) -> np.ndarray:
        """[n][3]: per-row sum, sum of squares and sum of |J_ij| over j != i."""
        out = np.empty((self.n, 3))
        check(self.lib.dcx_proc_row_stats(self.h, ptr(out, C.c_double)), self.h)
        return out

    def info(self) -> CouplingInfo:
        out = CouplingInfo()
        check(self.lib.dcx_coupling(self.h, C.byref(out)), self.h)
        return out

    def matvec(self, V: np.ndarray, precision="f64") -> np.ndarray:
        V = np.ascontiguousarray(np.atleast_2d(V), dtype=np.float64)
        out = np.empty_like(V)
        check(self.lib.dcx_matvec(self.h, V.shape[0], ptr(V, C.c_double), ptr(out, C.c_double),
                                  PRECISION[precision]), self.h)
        return out

    def apply(self, V, alpha, beta, precision="f64", want_tx=True, want_h=True):
        V = np.ascontiguousarray(np.atleast_2d(V), dtype=np.float64)
        R = V.shape[0]
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, np.float64), (R,)))
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(beta, np.float64), (R,)))
        tx = np.empty_like(V) if want_tx else None
        h = np.empty(R) if want_h else None
        check(self.lib.dcx_apply(self.h, R, ptr(a, C.c_double), ptr(b, C.c_double), ptr(V, C.c_double),
                                 ptr(tx, C.c_double), ptr(h, C.c_double), PRECISION[precision]), self.h)
        return tx, h

    def energy(self, S: np.ndarray) -> np.ndarray:
        S = np.atleast_2d(np.asarray(S))
        s8 = np.ascontiguousarray(np.where(S >= 0, 1, -1).astype(np.int8))
        out = np.empty(s8.shape[0])
        check(self.lib.dcx_energy(self.h, s8.shape[0], ptr(s8, C.c_int8), ptr(out, C.c_double)), self.h)
        return out

    # ---------------------------------------------------------------- solve
    def begin(self, prm: Params, alpha, beta, X0):
        X0 = np.ascontiguousarray(np.atleast_2d(X0), dtype=np.float64)
        R = X0.shape[0]
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, np.float64), (R,)))
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(beta, np.float64), (R,)))
        self._R = R
        check(self.lib.dcx_solve_begin(self.h, C.byref(prm), R, ptr(a, C.c_double), ptr(b, C.c_double),
                                       ptr(X0, C.c_double)), self.h)

    def step(self) -> bool:
        live = C.c_int32(0)
        check(self.lib.dcx_solve_step(self.h, C.byref(live)), self.h)
        return bool(live.value)

    def run(self):
        check(self.lib.dcx_solve_run(self.h), self.h)

    def summary(self, r: int) -> Summary:
        s = Summary()
        check(self.lib.dcx_result_summary(self.h, r, C.byref(s)), self.h)
        return s

    def history(self, r: int, start: int, count: int):
        h = np.empty(count)
        e = np.empty(count)
        t = np.empty(count)
        ev = np.empty(count, dtype=np.int32)
        if count:
            check(self.lib.dcx_result_history(self.h, r, start, count, ptr(h, C.c_double), ptr(e, C.c_double),
                                              ptr(t, C.c_double), ptr(ev, C.c_int32)), self.h)
        return h, e, t, ev

    def summaries(self):
        R = self._R
        it = np.empty(R, np.int64)
        st = np.empty(R, np.int32)
        be = np.empty(R)
        nh = np.empty(R, np.int64)
        dw = np.empty(R, np.int32)
        check(self.lib.dcx_result_summaries(self.h, ptr(it, C.c_int64), ptr(st, C.c_int32), ptr(be, C.c_double),
                                            ptr(nh, C.c_int64), ptr(dw, C.c_int32)), self.h)
        return it, st, be, nh, dw

    def history_all(self, K: int):
        R = self._R
        h = np.empty((R, K))
        e = np.empty((R, K))
        t = np.empty((R, K))
        ev = np.zeros((R, K), np.int32)
        check(self.lib.dcx_result_history_all(self.h, int(K), ptr(h, C.c_double), ptr(e, C.c_double),
                                              ptr(t, C.c_double), ptr(ev, C.c_int32)), self.h)
        return h, e, t, ev

    def best_spins(self) -> np.ndarray:
        out = np.empty((self._R, self.n), dtype=np.int8)
        check(self.lib.dcx_result_best_spins(self.h, ptr(out, C.c_int8)), self.h)
        return out

    def state(self) -> np.ndarray:
        out = np.empty((self._R, self.n))
        check(self.lib.dcx_result_state(self.h, ptr(out, C.c_double)), self.h)
        return out

    def detach(self) -> "Result":
        """Move the finished run's bulk outputs into a Result (device-resident until read)."""
        h = _P()
        check(self.lib.dcx_result_detach(self.h, C.byref(h)), self.h)
        return Result(self.lib, h, self._R, self.n)

    def states(self, r: int, iterations: int) -> np.ndarray:
        out = np.empty((iterations + 1, self.n))
        check(self.lib.dcx_result_states(self.h, r, ptr(out, C.c_double)), self.h)
        return out

    def profile(self, launches: int):
        ms = C.c_double()
        kid = C.c_int32()
        check(self.lib.dcx_profile_kernel(self.h, int(launches), C.byref(ms), C.byref(kid)), self.h)
        return ms.value, kid.value

    def device_seconds(self) -> float:
        out = C.c_double()
        check(self.lib.dcx_result_device_seconds(self.h, C.byref(out)), self.h)
        return out.value

    def power(self, use_shift: bool, shift: float, tol: float, max_iters: int, restart: np.ndarray):
        r = np.ascontiguousarray(restart, dtype=np.float64)
        mag, ray = C.c_double(), C.c_double()
        it, conv = C.c_int64(), C.c_int32()
        check(self.lib.dcx_power(self.h, int(bool(use_shift)), float(shift), float(tol), int(max_iters),
                                 ptr(r, C.c_double), C.byref(mag), C.byref(ray), C.byref(it), C.byref(conv)), self.h)
        return mag.value, ray.value, int(it.value), bool(conv.value)

    # ------------------------------------------------- generation / ingest
    def gen_sparse_9bit(self, n: int, n_p: int, seed: int):
        """(row_offsets int64, col_indices int64, values f64) generated on the device."""
        nnz = C.c_int64()
        check(self.lib.dcx_gen_sparse_9bit(self.h, int(n), int(n_p), int(seed) & ((1 << 64) - 1), C.byref(nnz)),
              self.h)
        ro = np.empty(int(n) + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value, dtype=np.float64)
        check(self.lib.dcx_gen_result(self.h, ptr(ro, C.c_int64), ptr(col, C.c_int64), ptr(val, C.c_double)), self.h)
        return ro, col, val

    def validate_csr(self, n, row_offsets, col_indices, values):
        """(check, row, all_int) of dcx_validate_csr (include/dcx.h)."""
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(col_indices, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        chk, row, ai = C.c_int32(), C.c_int64(), C.c_int32()
        check(self.lib.dcx_validate_csr(self.h, int(n), int(len(v)), ptr(ro, C.c_int64), ptr(ci, C.c_int64),
                                        ptr(v, C.c_double), C.byref(chk), C.byref(row), C.byref(ai)), self.h)
        return int(chk.value), int(row.value), bool(ai.value)

    # ------------------------------------------------- row-partitioned runs
    def set_csr_block(self, n_rows, n_cols, row_base, values, col_indices, row_offsets):
        v = np.ascontiguousarray(values, dtype=np.float64)
        c = np.ascontiguousarray(col_indices, dtype=np.int64)
        r = np.ascontiguousarray(row_offsets, dtype=np.int64)
        check(self.lib.dcx_set_csr_block(self.h, int(n_rows), int(n_cols), int(row_base), int(len(v)),
                                         ptr(r, C.c_int64), ptr(c, C.c_int64), ptr(v, C.c_double)), self.h)
        self.n = int(n_rows)

    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.dcx_stream(self.h, C.byref(s)), self.h)
        return int(s.value or 0)

    def dist_begin(self, prm: Params, alpha, beta, X0_rows, xbuf0: int, xbuf1: int, qsum: int, qmax: int):
        X0 = np.ascontiguousarray(np.atleast_2d(X0_rows), dtype=np.float64)
        R = X0.shape[0]
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, np.float64), (R,)))
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(beta, np.float64), (R,)))
        self._R = R
        check(self.lib.dcx_dist_begin(self.h, C.byref(prm), R, ptr(a, C.c_double), ptr(b, C.c_double),
                                      ptr(X0, C.c_double), C.c_void_p(xbuf0), C.c_void_p(xbuf1),
                                      C.c_void_p(qsum), C.c_void_p(qmax)), self.h)

    def dist_pass(self):
        check(self.lib.dcx_dist_pass(self.h), self.h)

    def dist_pass_rows(self, lo: int, hi: int, half: int):
        check(self.lib.dcx_dist_pass_rows(self.h, int(lo), int(hi), int(half)), self.h)

    def dist_reduce(self):
        check(self.lib.dcx_dist_reduce(self.h), self.h)

    def dist_control(self):
        check(self.lib.dcx_dist_control(self.h), self.h)

    def dist_poll(self):
        live = C.c_int32(0)
        p = C.c_int64(0)
        check(self.lib.dcx_dist_poll(self.h, C.byref(live), C.byref(p)), self.h)
        return bool(live.value), int(p.value)

    def dist_finish(self):
        check(self.lib.dcx_dist_finish(self.h), self.h)


class Result:
    """A detached run (dcx_result): final states and best spins in device memory,
    the history in pinned host memory, copied into numpy arrays on request."""

    def __init__(self, lib, handle, R: int, n: int):
        self.lib, self.h, self.R, self.n = lib, handle, R, n

    def __del__(self):
        try:
            if self.h:
                self.lib.dcx_result_free(self.h)
                self.h = None
        except Exception:
            pass

    def state(self) -> np.ndarray:
        out = np.empty((self.R, self.n))
        check(self.lib.dcx_res_state(self.h, ptr(out, C.c_double)))
        return out

    def best_spins(self) -> np.ndarray:
        out = np.empty((self.R, self.n), dtype=np.int8)
        check(self.lib.dcx_res_best_spins(self.h, ptr(out, C.c_int8)))
        return out

    def history_all(self, K: int):
        h = np.empty((self.R, K))
        e = np.empty((self.R, K))
        t = np.empty((self.R, K))
        ev = np.zeros((self.R, K), np.int32)
        check(self.lib.dcx_res_history_all(self.h, int(K), ptr(h, C.c_double), ptr(e, C.c_double),
                                           ptr(t, C.c_double), ptr(ev, C.c_int32)))
        return h, e, t, ev

    def warn_delta(self) -> np.ndarray:
        out = np.empty(self.R)
        check(self.lib.dcx_res_warn_delta(self.h, ptr(out, C.c_double)))
        return out
