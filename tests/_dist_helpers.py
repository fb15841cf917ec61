"""Helpers of tests/test_dist.py (test infrastructure, not collected).

``FakeRowContext`` stands in for libdcx in the CPU (gloo) tests of the
row-partitioned driver: it implements the context calls the driver makes
(dcx_set_csr_block / dcx_dist_* / results) in numpy, with the DOCH loop of
dc/solvers/doch.py:199-232 restated per pass (record H(x_p), E(sign x_p), then
stop on the step of x_p - x_{p-1}). It lets gloo world-size-2 tests exercise
partitioning, column remapping, the exchange schedule and result assembly
without a GPU; the device kernels behind the same calls are covered by the
GPU tests.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp

from paper_2509_01928_b200 import _native


def _view(ptr, count, dtype):
    ctype = ctypes.c_double if dtype == np.float64 else ctypes.c_float
    return np.ctypeslib.as_array((ctype * count).from_address(ptr)).view(dtype)


class FakeRowContext:
    def set_csr_block(self, n_rows, n_cols, row_base, values, col_indices, row_offsets):
        self.n = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_base = int(row_base)
        self.A = sp.csr_matrix((np.asarray(values, np.float64), np.asarray(col_indices), np.asarray(row_offsets)),
                               shape=(n_rows, n_cols))

    def stream(self):
        return 0

    def dist_begin(self, prm, alpha, beta, X0_rows, xb0, xb1, qsum, qmax):
        if prm.solver != _native.SOLVER["doch"]:
            raise ValueError("the fake context implements DOCH only")
        X0 = np.atleast_2d(X0_rows)
        R = X0.shape[0]
        self._R = R
        dt = np.float64 if prm.precision == _native.PRECISION["f64"] else np.float32
        size = self.n_cols * R
        self.X = [_view(xb0, size, dt).reshape(self.n_cols, R), _view(xb1, size, dt).reshape(self.n_cols, R)]
        self.qs = _view(qsum, R * _native.QSUM, np.float64).reshape(R, _native.QSUM)
        self.qm = _view(qmax, R * _native.QMAX, np.float64).reshape(R, _native.QMAX)
        self.alpha = np.broadcast_to(np.asarray(alpha, np.float64), (R,)).copy()
        self.beta = np.broadcast_to(np.asarray(beta, np.float64), (R,)).copy()
        self.max_iters, self.stride, self.tol, self.dtol = prm.max_iters, prm.trace_stride, prm.conv_tol, prm.descent_tol
        rows = slice(self.row_base, self.row_base + self.n)
        self.X[0][rows] = X0.T
        self.X[1][rows] = 0
        self.p = 0
        self.k = np.zeros(R, np.int64)
        self.status = np.zeros(R, np.int32)
        self.best = np.full(R, np.inf)
        self.best_s = np.ones((R, self.n), np.int8)
        self.warn = np.full(R, -1, np.int32)
        self.prev_step = np.zeros(R)
        self.H = [[] for _ in range(R)]
        self.E = [[] for _ in range(R)]
        self.EV = [[] for _ in range(R)]
        self.xfinal = X0.copy()

    def dist_pass(self):
        p, rows = self.p, slice(self.row_base, self.row_base + self.n)
        Xc, Xn = self.X[p & 1], self.X[(p + 1) & 1]
        x = Xc[rows].T.astype(np.float64)                      # [R][n_rows]
        jx = (self.A @ Xc.astype(np.float64)).T                # [R][n_rows]
        js = (self.A @ np.where(Xc >= 0, 1.0, -1.0)).T
        ax = jx + self.alpha[:, None] * x
        xn = np.cbrt(ax / self.beta[:, None])
        run = self.status == 0
        self.qs[:] = 0
        self.qs[:, 0] = (x * x * x * x).sum(1)
        self.qs[:, 1] = (x * ax).sum(1)
        self.qs[:, 2] = (np.where(x >= 0, 1.0, -1.0) * js).sum(1)
        self.qm[:, 0] = np.abs(xn - x).max(1) if self.n else 0.0
        self.qm[:, 1] = 0.0
        self.qm[:, 2] = 0.0
        Xn[rows] = np.where(run[None, :], xn.T, Xn[rows])
        self._x = x

    def dist_pass_rows(self, lo, hi, half):
        """dcx_dist_pass_rows: rows [lo, hi) only, reading the buffers as they are at the call
        (a boundary range run before its halo landed would read a stale halo)."""
        p = self.p
        Xc, Xn = self.X[p & 1], self.X[(p + 1) & 1]
        if not hasattr(self, "_hp") or self._hp[0] != p:
            R = self._R
            self._hp = (p, np.zeros((2, R, _native.QSUM)), np.zeros((2, R, _native.QMAX)), np.zeros((R, self.n)))
        _, hs, hm, xall = self._hp
        if hi <= lo:
            return
        rows = slice(self.row_base + lo, self.row_base + hi)
        A = self.A[lo:hi]
        x = Xc[rows].T.astype(np.float64)
        jx = (A @ Xc.astype(np.float64)).T
        js = (A @ np.where(Xc >= 0, 1.0, -1.0)).T
        ax = jx + self.alpha[:, None] * x
        xn = np.cbrt(ax / self.beta[:, None])
        run = self.status == 0
        hs[half] = 0
        hs[half, :, 0] = (x * x * x * x).sum(1)
        hs[half, :, 1] = (x * ax).sum(1)
        hs[half, :, 2] = (np.where(x >= 0, 1.0, -1.0) * js).sum(1)
        hm[half] = 0
        hm[half, :, 0] = np.abs(xn - x).max(1)
        Xn[rows] = np.where(run[None, :], xn.T, Xn[rows])
        xall[:, lo:hi] = x

    def dist_reduce(self):
        _, hs, hm, xall = self._hp
        self.qs[:] = hs[0] + hs[1]
        self.qm[:] = np.maximum(hm[0], hm[1])
        self._x = xall.copy()

    def dist_control(self):
        p = self.p
        for r in np.nonzero(self.status == 0)[0]:
            h = 0.25 * self.beta[r] * self.qs[r, 0] - 0.5 * self.qs[r, 1]
            e = -0.5 * self.qs[r, 2]
            ev = 0
            if p >= 1 and h - self.H[r][-1] > self.dtol:
                ev |= _native.EV_DESCENT
                if self.warn[r] < 0:
                    self.warn[r] = p
            converged = p >= 1 and self.prev_step[r] <= self.tol
            last = p >= self.max_iters
            self.H[r].append(h)
            if p % self.stride == 0 or converged or last or ev:
                ev |= _native.EV_RECORDED
                self.E[r].append(e)
                if e < self.best[r]:
                    self.best[r] = e
                    self.best_s[r] = np.where(self._x[r] >= 0, 1, -1)
            else:
                self.E[r].append(np.nan)
            self.EV[r].append(ev)
            self.k[r] = p
            if converged or last:
                self.status[r] = 1 if converged else 2
                self.xfinal[r] = self._x[r]
            self.prev_step[r] = self.qm[r, 0]
        self.p += 1

    def dist_poll(self):
        return bool((self.status == 0).any()), self.p

    def dist_finish(self):
        pass

    def summaries(self):
        nh = np.array([len(h) for h in self.H], np.int64)
        return self.k.copy(), self.status.copy(), self.best.copy(), nh, self.warn.copy()

    def history_all(self, K):
        R = self._R
        H = np.full((R, K), np.nan)
        E = np.full((R, K), np.nan)
        T = np.zeros((R, K))
        EV = np.zeros((R, K), np.int32)
        for r in range(R):
            m = len(self.H[r])
            H[r, :m], E[r, :m], EV[r, :m] = self.H[r], self.E[r], self.EV[r]
        return H, E, T, EV

    def best_spins(self):
        return self.best_s.copy()

    def state(self):
        return self.xfinal.copy()

    def device_seconds(self):
        return 0.0


def init_group(rank, world, init_file, backend="gloo"):
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend, init_method=f"file://{init_file}", rank=rank, world_size=world)
    return dist


def graph_of(kind, n, seed_graph):
    from paper_2509_01928_b200 import synth

    if kind == "torus":
        L = int(round(n ** 0.5))
        return synth.torus(L, seed=seed_graph) + (None,)
    if kind == "reg3":
        return synth.random_regular3(n, seed=seed_graph)
    return synth.erdos_renyi(n, 6, seed=seed_graph)


def fake_worker(rank, world, init_file, out_file, n, seed_graph, R, max_iters, exchange="allgather", kind="er"):
    """One rank of the CPU test: DOCH f64 through the row-partitioned driver."""
    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import dist as dd

    dist = init_group(rank, world, init_file)
    v, c, o, co = graph_of(kind, n, seed_graph)
    J = dc.CsrCoupling(n, v, c, o, validate=False)
    inst = dc.ProblemInstance(coupling=J, cut_offset=co)
    alpha, beta = 3.0, float(n) ** 1.5 * 10.0
    X0 = np.stack([dc.initial_state(n, alpha, beta, np.random.default_rng(s)) for s in range(R)])
    res = dd.solve_distributed(inst, "doch", alpha, beta, X0, max_iters=max_iters, precision="f64",
                               poll_every=4, exchange=exchange, _context=FakeRowContext())
    if rank == 0:
        np.savez(out_file, path=res[0].path, x=np.stack([r.x for r in res]), spins=np.stack([r.spins for r in res]),
                 energy=np.array([r.energy for r in res]), iterations=np.array([r.iterations for r in res]),
                 stop=np.array([r.stop_reason for r in res]),
                 h=np.stack([np.asarray(r.h_values)[: max_iters + 1] for r in res]) if R > 1 else
                 np.asarray(res[0].h_values)[None, :])
    dist.barrier()
    dist.destroy_process_group()


def exchange_worker(rank, world, init_file, out_file):
    import torch

    from paper_2509_01928_b200.dist import Exchange

    dist = init_group(rank, world, init_file)
    ex = Exchange()
    B, R = 3, 2
    X = torch.zeros(world * B, R, dtype=torch.float64)
    X[rank * B:(rank + 1) * B] = rank + 1 + torch.arange(B * R, dtype=torch.float64).reshape(B, R)
    ex.all_gather_rows(X, B)
    s = torch.full((R, 5), float(rank + 1), dtype=torch.float64)
    m = torch.tensor([[float(rank)] * 3] * R, dtype=torch.float64)
    ex.all_reduce(s, "sum")
    ex.all_reduce(m, "max")
    if rank == 0:
        np.savez(out_file, X=X.numpy(), s=s.numpy(), m=m.numpy(), host_staged=ex.host_staged)
    dist.barrier()
    dist.destroy_process_group()


def halo_plan_worker(rank, world, init_file, out_file, kind, n):
    """Build the halo plan on every rank; rank 0 saves every rank's lists."""
    import torch

    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import dist as dd

    dist = init_group(rank, world, init_file)
    v, c, o, _ = graph_of(kind, n, 0)
    J = dc.CsrCoupling(n, v, c, o, validate=False)
    rb = dd.RowBlocks(dd.partition_rows(o, world), n)
    _, _, cols, _ = dd.local_block(J, rb, rank)
    ex = dd.Exchange()
    plan = dd.halo_plan(ex, cols, rb)
    # exchange position-valued rows: afterwards every referenced row holds its own index
    X = torch.full((rb.n_space, 2), -1.0, dtype=torch.float64)
    lo = rank * rb.B
    X[lo:lo + rb.B, 0] = torch.arange(lo, lo + rb.B, dtype=torch.float64)
    X[lo:lo + rb.B, 1] = -torch.arange(lo, lo + rb.B, dtype=torch.float64)
    ex.halo(X, plan, torch.from_numpy(plan.send_pos), torch.from_numpy(plan.recv_pos),
            torch.empty(plan.volume, 2, dtype=torch.float64))
    ok = bool(np.all(X[np.unique(cols), 0].numpy() == np.unique(cols)))
    ok &= bool(np.all(X[np.unique(cols), 1].numpy() == -np.unique(cols)))
    info = torch.tensor([plan.volume, int(plan.send_pos.size), int(ok), rb.B], dtype=torch.int64)
    allinfo = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(allinfo, info)
    if rank == 0:
        np.savez(out_file, info=torch.stack(allinfo).numpy())
    dist.barrier()
    dist.destroy_process_group()


def gpu_worker(rank, world, init_file, out_file, solver, precision, R, max_iters, exchange="allgather"):
    """One rank of the GPU test (every rank on cuda:0, gloo host-staged exchange)."""
    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import dist as dd, synth

    dist = init_group(rank, world, init_file)
    v, c, o, co = synth.erdos_renyi(10_000, 6, seed=3)
    J = dc.CsrCoupling(10_000, v, c, o, validate=False)
    inst = dc.ProblemInstance(coupling=J, cut_offset=co)
    alpha, beta = 3.0, 1e4 ** 1.5 * 10.0
    X0 = np.stack([dc.initial_state(10_000, alpha, beta, np.random.default_rng(s)) for s in range(R)])
    res = dd.solve_distributed(inst, solver, alpha, beta, X0, max_iters=max_iters, precision=precision,
                               device=0, poll_every=8, exchange=exchange)
    if rank == 0:
        np.savez(out_file, x=np.stack([r.x for r in res]), spins=np.stack([r.spins for r in res]),
                 energy=np.array([r.energy for r in res]), iterations=np.array([r.iterations for r in res]),
                 stop=np.array([r.stop_reason for r in res]),
                 h=np.stack([np.asarray(r.h_values)[: r.iterations + 1][:2] for r in res]),
                 accepted=np.array([(r.accepted or []) + [False] * (max_iters + 1 - len(r.accepted or []))
                                    for r in res], dtype=bool))
    dist.barrier()
    dist.destroy_process_group()


def compact_worker(rank, world, init_file, out_file, kind, n):
    """Compact [own | halo] space: after the exchange every referenced remote row sits at
    B + its plan index, so the compact block's product equals the padded block's; and the
    one-collective combine of the per-replica partials equals SUM / MAX."""
    import torch

    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import dist as dd

    dist = init_group(rank, world, init_file)
    v, c, o, _ = graph_of(kind, n, 0)
    J = dc.CsrCoupling(n, v, c, o, validate=False)
    rb = dd.RowBlocks(dd.partition_rows(o, world), n)
    n_rows, vals, cols, ro = dd.local_block(J, rb, rank)
    ex = dd.Exchange()
    plan = dd.halo_plan(ex, cols, rb)
    ccols = dd.compact_columns(cols, rb, rank, plan)
    space = rb.B + plan.volume
    # a state defined on the padded space: row value = f(global spin index)
    full = np.zeros((rb.n_space, 2))
    glob = np.concatenate([np.arange(r0, r1) for r0, r1 in rb.blocks])
    pos = rb.position(glob)
    full[pos, 0] = np.sin(glob + 0.5)
    full[pos, 1] = np.cos(3.0 * glob)
    X = torch.zeros(space, 2, dtype=torch.float64)
    lo = rank * rb.B
    X[:rb.B] = torch.from_numpy(full[lo:lo + rb.B])
    ex.halo_compact(X, plan, torch.from_numpy(plan.send_pos - lo), rb.B)
    A_pad = sp.csr_matrix((vals, cols, ro), shape=(n_rows, rb.n_space))
    A_cmp = sp.csr_matrix((vals, ccols, ro), shape=(n_rows, space))
    ok = bool(np.array_equal(A_pad @ full, A_cmp @ X.numpy()))
    qs = torch.full((3, 5), float(rank + 1), dtype=torch.float64) * torch.arange(1, 6, dtype=torch.float64)
    qm = torch.tensor([[float(rank), -float(rank), 0.5]] * 3, dtype=torch.float64)
    ex.combine(qs, qm)
    info = torch.tensor([plan.volume, space, rb.n_space, int(ok)], dtype=torch.int64)
    allinfo = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(allinfo, info)
    if rank == 0:
        np.savez(out_file, info=torch.stack(allinfo).numpy(), qs=qs.numpy(), qm=qm.numpy())
    dist.barrier()
    dist.destroy_process_group()
