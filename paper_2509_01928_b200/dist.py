"""Row-partitioned DOCH / ADOCH across ranks.

The reference has no distributed solver: one ``doch_solve`` / ``adoch_solve``
(dc/solvers/doch.py:169-356) runs one scipy ``csr_matvec`` per iteration
(dc/coupling.py:189-190) in one process. Here the coupling rows are split into
contiguous, nnz-balanced blocks, one per rank (one process per GPU, NCCL over
NVLink). Per iteration every rank

  1. runs the fused pass over its rows (``dcx_dist_pass``): (J+aI)x, the cube-root
     update of its slice of x, and its share of the per-replica sums
     (sum x^4, sum x.Ax, sum s.Js, max |dx|),
  2. combines those sums and maxima over the ranks with ONE collective: an
     all-gather of every rank's 8 doubles per replica, reduced on the device in
     rank order (so the totals do not depend on the collective's reduction order),
  3. runs the control on the reduced values (``dcx_dist_control``): identical on
     every rank, so stop / record / ADOCH-accept decisions agree,
  4. exchanges the new x slices for the next pass: either an all-gather of every
     slice (in place), or a neighbour-only exchange ("halo") that sends each rank
     exactly the x rows its coupling rows reference (a lattice
     strip needs its two boundary rows; a random 3-regular graph at 8 ranks needs
     about a third of the remote rows). ``exchange="auto"`` takes the halo when it
     moves less than 3/4 of the all-gather volume.

Blocks are padded to a common row count B so the all-gather is a plain
``all_gather_into_tensor``; with the all-gather exchange the columns are
remapped into that padded index space (rank q's rows live at [q*B, q*B + rows_q)).
With the neighbour-only exchange each rank's columns are remapped into a
COMPACT space [own rows | halo rows]: its B own rows first, then exactly the H
remote rows it references, in the order they arrive (source rank, position), so
a rank holds B + H rows of x instead of world * B (the 10^8-spin R8 graph: a
fraction of the 400 MB state per GPU) and receives its halo straight into the
tail of its x buffer. The CSR entries of a row keep their order under either
remap, so each row's sum order -- and therefore every iterate -- is
bit-identical to the single-GPU multipass path; only the order of the H partial
sums across blocks differs.

With the neighbour-only exchange the rows of a block are also reordered
[interior | boundary] (boundary: rows that reference a halo row, or that another
rank reads) and the pass runs as two row ranges (``dcx_dist_pass_rows``): the
interior range reads own rows only, so with NCCL the halo exchange of x_p runs on
its own stream and communicator while the interior rows of pass p compute; the
boundary range waits for it (a CUDA event), then both halves of the partials are
folded (``dcx_dist_reduce``). Each row keeps its entries in their stored order, so
the iterates stay bit-identical.

With the NCCL backend the collectives run on the context stream directly on
device buffers; with gloo (CPU transport) they are staged through host memory
(and the exchange is not overlapped).
"""

from __future__ import annotations

import contextlib
import os
import time
import weakref
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native
from .solvers import CONVERGENCE_TOL, DESCENT_WARN_TOL, SOLVER_NAMES, assemble_results


# ---------------------------------------------------------------- partitioning
def partition_rows(row_offsets, world: int) -> list:
    """Contiguous row blocks [(row0, row1)] balancing nnz + rows per block.

    Every block is non-empty when n >= world (a rank with no rows would still
    take part in every collective, which is allowed but pointless).
    """
    ro = np.asarray(row_offsets, dtype=np.int64)
    n = len(ro) - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    if n < world:
        raise ValueError(f"cannot split {n} rows over {world} ranks")
    cost = ro + np.arange(n + 1)  # cumulative nnz + rows
    total = cost[-1]
    cuts = [0]
    for q in range(1, world):
        c = int(np.searchsorted(cost, total * q / world, side="left"))
        c = min(max(c, cuts[-1] + 1), n - (world - q))  # at least one row per block
        cuts.append(c)
    cuts.append(n)
    return [(cuts[q], cuts[q + 1]) for q in range(world)]


@dataclass
class RowBlocks:
    """Blocks of a row partition and the padded exchange index space."""

    blocks: list
    n: int

    @property
    def world(self) -> int:
        return len(self.blocks)

    @property
    def B(self) -> int:
        return max(r1 - r0 for r0, r1 in self.blocks)

    @property
    def n_space(self) -> int:
        return self.world * self.B

    def position(self, j):
        """Index of spin j in the padded space."""
        j = np.asarray(j, dtype=np.int64)
        if self.world == 1:
            return j
        starts = np.array([r0 for r0, _ in self.blocks], dtype=np.int64)
        q = np.searchsorted(starts, j, side="right") - 1
        return q * self.B + (j - starts[q])

    def unpad(self, arr):
        """[..., n_space] -> [..., n] (drops the padding rows)."""
        parts = [arr[..., q * self.B: q * self.B + (r1 - r0)] for q, (r0, r1) in enumerate(self.blocks)]
        return np.concatenate(parts, axis=-1)


def local_block(J, rb: RowBlocks, rank: int):
    """This rank's CSR rows with columns mapped into the padded space."""
    r0, r1 = rb.blocks[rank]
    ro = np.asarray(J.row_offsets, dtype=np.int64)
    lo, hi = int(ro[r0]), int(ro[r1])
    cols = rb.position(np.asarray(J.col_indices[lo:hi], dtype=np.int64))
    vals = np.asarray(J.values[lo:hi], dtype=np.float64)
    return r1 - r0, vals, cols, ro[r0:r1 + 1] - lo


# ------------------------------------------------------------------ exchange
class Exchange:
    """The three collectives of one iteration on torch.distributed.

    NCCL: in place on the device tensors (issued on the current stream, which
    the driver sets to the context stream). gloo: staged through host memory.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host_staged = dist.get_backend(group) != "nccl"

    def all_gather_rows(self, X, B: int):
        """X: [world*B, R] tensor whose rows [rank*B, (rank+1)*B) are this rank's."""
        dist = self.dist
        mine = X[self.rank * B:(self.rank + 1) * B]
        if not self.host_staged:
            dist.all_gather_into_tensor(X, mine, group=self.group)
            return
        import torch

        h = mine.cpu()
        parts = [torch.empty_like(h) for _ in range(self.world)]
        dist.all_gather(parts, h, group=self.group)
        X.copy_(torch.cat(parts, 0))

    def all_to_all_counts(self, counts):
        """counts[p] = rows this rank receives from p -> rows this rank sends to each p."""
        import torch

        t = torch.tensor(counts, dtype=torch.int64)
        out = torch.empty_like(t)
        if self.host_staged:
            self.dist.all_to_all_single(out, t, group=self.group)
        else:
            dev = torch.device("cuda", torch.cuda.current_device())
            o = out.to(dev)
            self.dist.all_to_all_single(o, t.to(dev), group=self.group)
            out = o.cpu()
        return [int(v) for v in out]

    def all_to_all_rows_int(self, pos, out_counts, in_counts):
        """Ragged all-to-all of int64 positions (setup of the halo plan)."""
        import torch

        t = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.int64))
        out = torch.empty(sum(in_counts), dtype=torch.int64)
        if self.host_staged:
            self.dist.all_to_all_single(out, t, in_counts, out_counts, group=self.group)
        else:
            dev = torch.device("cuda", torch.cuda.current_device())
            o = out.to(dev)
            self.dist.all_to_all_single(o, t.to(dev), in_counts, out_counts, group=self.group)
            out = o.cpu()
        return out.numpy()

    def halo_compact(self, X, plan: HaloPlan, send_local, B: int):
        """Neighbour-only exchange into the compact space X [B + H, R]: own rows send_local go out,
        the halo arrives in rows [B, B + H) in plan order."""
        dist = self.dist
        send = X.index_select(0, send_local)
        tail = X[B:B + plan.volume]
        if not self.host_staged:
            dist.all_to_all_single(tail, send, plan.recv_counts, plan.send_counts, group=self.group)
            return
        h = tail.cpu()
        dist.all_to_all_single(h, send.cpu(), plan.recv_counts, plan.send_counts, group=self.group)
        tail.copy_(h.to(X.device))

    def combine(self, qs, qm):
        """One collective for the per-replica partials: all-gather every rank's [R][QSUM + QMAX],
        then sum / max over ranks in rank order (deterministic, collective-order independent)."""
        import torch

        mine = torch.cat([qs, qm], 1).contiguous()
        allq = torch.empty((self.world,) + tuple(mine.shape), dtype=mine.dtype, device=mine.device)
        if not self.host_staged:
            self.dist.all_gather_into_tensor(allq, mine, group=self.group)
        else:
            h = mine.cpu()
            parts = [torch.empty_like(h) for _ in range(self.world)]
            self.dist.all_gather(parts, h, group=self.group)
            allq.copy_(torch.stack(parts, 0))
        ks = qs.shape[1]
        s = allq[0, :, :ks].clone()
        m = allq[0, :, ks:].clone()
        for q in range(1, self.world):
            s += allq[q, :, :ks]
            m = torch.maximum(m, allq[q, :, ks:])
        qs.copy_(s)
        qm.copy_(m)

    def halo(self, X, plan: HaloPlan, send_idx, recv_idx, recv_buf):
        """Neighbour-only exchange into X [world*B, R]: rows send_idx go out, rows recv_idx come in."""
        dist = self.dist
        send = X.index_select(0, send_idx)
        if not self.host_staged:
            dist.all_to_all_single(recv_buf, send, plan.recv_counts, plan.send_counts, group=self.group)
            X.index_copy_(0, recv_idx, recv_buf)
            return
        h = recv_buf.cpu() if recv_buf.device.type != "cpu" else recv_buf
        dist.all_to_all_single(h, send.cpu(), plan.recv_counts, plan.send_counts, group=self.group)
        X.index_copy_(0, recv_idx, h.to(X.device))

    def all_reduce(self, t, op: str):
        dist = self.dist
        rop = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}[op]
        if not self.host_staged:
            dist.all_reduce(t, op=rop, group=self.group)
            return
        h = t.cpu()
        dist.all_reduce(h, op=rop, group=self.group)
        t.copy_(h)


@dataclass
class HaloPlan:
    """Neighbour-only exchange of one rank (positions in the padded space).

    ``send_pos`` lists rows of this rank's block, grouped by destination rank
    (ascending rank, ascending position); ``recv_pos`` lists rows of other
    blocks this rank's coupling rows reference, grouped by source rank.
    """

    send_pos: np.ndarray
    send_counts: list
    recv_pos: np.ndarray
    recv_counts: list

    @property
    def volume(self) -> int:
        """Rows received per exchange."""
        return int(self.recv_pos.size)


def halo_needs(cols_padded, rb: RowBlocks, rank: int):
    """Remote rows referenced by this rank's columns: (sorted positions, per-owner counts)."""
    c = np.unique(np.asarray(cols_padded, dtype=np.int64))
    lo, hi = rank * rb.B, (rank + 1) * rb.B
    remote = c[(c < lo) | (c >= hi)]
    counts = np.bincount(remote // rb.B, minlength=rb.world).astype(np.int64)
    return remote, [int(k) for k in counts]


def compact_columns(cols_padded, rb: RowBlocks, rank: int, plan: "HaloPlan"):
    """Padded-space columns of this rank's block -> the compact [own B rows | halo rows] space:
    own positions p -> p - rank * B, remote ones -> B + their index in plan.recv_pos (sorted)."""
    c = np.asarray(cols_padded, dtype=np.int64)
    lo = rank * rb.B
    own = (c >= lo) & (c < lo + rb.B)
    out = np.empty_like(c)
    out[own] = c[own] - lo
    rem = ~own
    idx = np.searchsorted(plan.recv_pos, c[rem])
    if rem.any() and (idx.max() >= plan.recv_pos.size or np.any(plan.recv_pos[idx] != c[rem])):
        raise RuntimeError("compact remap: a remote column is missing from the halo plan")
    out[rem] = rb.B + idx
    return out


def interior_first(n_rows: int, ro, ccols, B: int, send_local):
    """Row order [interior | boundary] of a halo-exchanging block: boundary rows reference a
    halo row (compact column >= B) or are read by another rank (send_local); interior rows do
    neither, so their pass can run while the halo of x_p is still in flight. Returns
    (perm: new row k = old row perm[k], inverse, interior count)."""
    ro = np.asarray(ro, dtype=np.int64)
    rid = np.repeat(np.arange(n_rows, dtype=np.int64), np.diff(ro))
    bnd = np.zeros(n_rows, dtype=bool)
    bnd[rid[np.asarray(ccols) >= B]] = True
    bnd[np.asarray(send_local, dtype=np.int64)] = True
    perm = np.concatenate([np.nonzero(~bnd)[0], np.nonzero(bnd)[0]])
    inv = np.empty(n_rows, dtype=np.int64)
    inv[perm] = np.arange(n_rows, dtype=np.int64)
    return perm, inv, int((~bnd).sum())


def permute_rows(perm, inv, ro, vals, ccols, B: int):
    """The block's CSR with rows in `perm` order and own columns renamed through `inv`
    (halo columns >= B unchanged). Each row keeps its entries in their stored order, so its
    sum -- and every iterate -- is bit-identical."""
    ro = np.asarray(ro, dtype=np.int64)
    lengths = np.diff(ro)[perm]
    new_ro = np.zeros(len(perm) + 1, dtype=np.int64)
    np.cumsum(lengths, out=new_ro[1:])
    idx = np.repeat(ro[perm] - new_ro[:-1], lengths) + np.arange(int(new_ro[-1]), dtype=np.int64)
    c = np.asarray(ccols, dtype=np.int64)[idx]
    own = c < B
    c[own] = inv[c[own]]
    return new_ro, np.asarray(vals)[idx], c


def halo_plan(ex: "Exchange", cols_padded, rb: RowBlocks) -> HaloPlan:
    """Every rank states what it needs; two all-to-alls (counts, then positions) turn
    the needs into send lists. Setup only (once per solve)."""
    recv_pos, recv_counts = halo_needs(cols_padded, rb, ex.rank)
    send_counts = ex.all_to_all_counts(recv_counts)
    send_pos = ex.all_to_all_rows_int(recv_pos, recv_counts, send_counts)
    lo = ex.rank * rb.B
    if send_pos.size and (send_pos.min() < lo or send_pos.max() >= lo + rb.B):
        raise RuntimeError("halo plan: a peer asked for rows this rank does not own")
    return HaloPlan(send_pos, send_counts, recv_pos, recv_counts)


_XGROUPS = {}
_PLANS = {}


def _block_plan(J, ex: "Exchange", exchange: str, tdev) -> dict:
    """This rank's row block of J, ready to upload: the nnz-balanced partition, columns in the
    padded space, or -- with the neighbour-only exchange -- in the compact [own | halo] space with
    the rows ordered [interior | boundary] (dist.interior_first)."""
    import torch

    rb = RowBlocks(partition_rows(J.row_offsets, ex.world), J.n)
    r0, r1 = rb.blocks[ex.rank]
    n_rows, vals, cols, ro = local_block(J, rb, ex.rank)
    # exchange plan: neighbour-only halo in a compact index space, or the all-gather of the padded space
    use_halo, plan = False, None
    if exchange != "allgather" and ex.world > 1:
        plan = halo_plan(ex, cols, rb)
        use_halo = exchange == "halo"
        if exchange == "auto":
            vol = torch.tensor([float(plan.volume), float(rb.n_space - rb.B)], dtype=torch.float64, device=tdev)
            ex.all_reduce(vol, "sum")
            use_halo = bool(vol[0] < 0.75 * vol[1])
    bp = {"rb": rb, "r0": r0, "r1": r1, "n_rows": n_rows, "use_halo": use_halo}
    if use_halo:
        cc = compact_columns(cols, rb, ex.rank, plan)
        send_old = plan.send_pos - ex.rank * rb.B
        perm, inv, n_int = interior_first(n_rows, ro, cc, rb.B, send_old)
        ro_p, vals_p, cc_p = permute_rows(perm, inv, ro, vals, cc, rb.B)
        bp.update(plan=plan, perm=perm, inv=inv, n_int=n_int, send_old=send_old, space=rb.B + plan.volume, base=0,
                  vals=vals_p, cols=cc_p, ro=ro_p)
    else:
        bp.update(space=rb.n_space, base=ex.rank * rb.B, vals=vals, cols=cols, ro=ro)
    return bp


def _exchange_group(group, world: int):
    """A second communicator over the same ranks for the x exchange (made once per group): NCCL
    collectives of one communicator must not run concurrently on two streams, and the halo
    exchange overlaps the partials' all-gather of the next iteration's pass."""
    import torch.distributed as tdist

    key = (id(group), world)
    if key not in _XGROUPS:
        ranks = list(range(world)) if group is None else tdist.get_process_group_ranks(group)
        _XGROUPS[key] = tdist.new_group(ranks)
    return _XGROUPS[key]


# -------------------------------------------------------------------- driver
def solve_distributed(instance, solver: str, alpha, beta, x0, *, group=None, max_iters: int = 1000,
                      lookback_q: int = 5, window_mode: str = "economy", trace_stride: int = 1,
                      time_budget: Optional[float] = None, precision: str = "f32",
                      seeds: Optional[Sequence[int]] = None, poll_every: int = 16,
                      device: Optional[int] = None, exchange: str = "auto", graph: Optional[bool] = None,
                      _context=None) -> list:
    """Row-partitioned ``solve_replicas``: the same R replicas, the coupling split by rows over the ranks
    of ``group`` (every rank passes the same instance and the same full ``x0`` [R][n]).

    Returns one SolveResult per replica on every rank (best spins and final x gathered to all ranks).
    ``exchange``: "allgather", "halo" (neighbour-only) or "auto" (halo when it moves < 3/4 of the
    all-gather rows summed over ranks). Both give bit-identical iterates.
    ``graph``: replay the ``poll_every`` iterations between host polls as one CUDA graph (passes,
    reductions, NCCL collectives and the exchange stream); default: environment ``DCX_DIST_GRAPH=1``.
    NCCL process groups only; the iterates are the eager loop's.
    ``_context`` replaces the libdcx context (tests only).
    """
    import torch

    if solver not in SOLVER_NAMES:
        raise ValueError(f"unknown solver {solver!r}")
    if window_mode != "economy":
        raise ValueError("the row-partitioned solver supports window_mode 'economy'")
    if precision not in ("f64", "f32"):
        raise ValueError("the row-partitioned solver runs in precision 'f64' or 'f32'")
    if exchange not in ("auto", "allgather", "halo"):
        raise ValueError(f"unknown exchange {exchange!r}")
    t_entry = time.perf_counter()
    ex = Exchange(group)
    J = instance.coupling
    if not all(hasattr(J, a) for a in ("values", "col_indices", "row_offsets")):
        raise ValueError("the row-partitioned solver needs a CSR coupling")
    X0 = np.atleast_2d(np.asarray(x0, dtype=np.float64))
    R, n = X0.shape
    if n != J.n:
        raise ValueError(f"x0 has {n} columns, expected {J.n}")
    if _context is None:
        dev = _native.default_device() if device is None else int(device)
        tdev = torch.device("cuda", dev)
    else:
        dev, tdev = None, torch.device("cpu")
    # the block plan (partition, column remap, exchange plan, row order) and the context are
    # made once per (coupling, group, rank, exchange, device) and reused by later solves; the
    # block itself is uploaded again every solve (the caller's arrays may have changed)
    key = (id(J), id(group), ex.world, ex.rank, exchange, dev)
    cached = _PLANS.get(key) if _context is None else None
    if cached is not None and cached["ref"]() is J:
        bp, ctx = cached["plan"], cached["ctx"]
    else:
        bp = _block_plan(J, ex, exchange, tdev)
        ctx = _native.Context(dev) if _context is None else _context
        if _context is None:
            _PLANS[key] = {"ref": weakref.ref(J), "plan": bp, "ctx": ctx}
    rb, r0, r1, n_rows, use_halo, space, base = (bp[k] for k in ("rb", "r0", "r1", "n_rows", "use_halo", "space",
                                                                  "base"))
    plan, perm, inv, n_int, send_old = (bp.get(k) for k in ("plan", "perm", "inv", "n_int", "send_old"))
    ctx.set_csr_block(n_rows, space, base, bp["vals"], bp["cols"], bp["ro"])
    dt = torch.float64 if precision == "f64" else torch.float32
    X = [torch.zeros(space, R, dtype=dt, device=tdev) for _ in range(2)]
    qs = torch.zeros(R, _native.QSUM, dtype=torch.float64, device=tdev)
    qm = torch.zeros(R, _native.QMAX, dtype=torch.float64, device=tdev)
    prm = _native.Params(
        solver=_native.SOLVER[solver], window_mode=_native.WINDOW[window_mode],
        precision=_native.PRECISION[precision], lookback_q=int(lookback_q), max_iters=int(max_iters),
        trace_stride=int(trace_stride), time_budget_s=-1.0 if time_budget is None else float(time_budget),
        conv_tol=CONVERGENCE_TOL, descent_tol=DESCENT_WARN_TOL, record_states=0,
        path=_native.PATH["multipass"], chunk=0, reserved=0)
    stream = (torch.cuda.ExternalStream(ctx.stream(), device=tdev) if tdev.type == "cuda" else None)
    # with NCCL the halo exchange runs on its own stream and communicator, overlapped with the
    # interior rows of the next pass; the partials' all-gather stays on the context stream
    overlap = use_halo and stream is not None and not ex.host_staged
    if overlap:
        ex_x = Exchange(_exchange_group(group, ex.world))
        comm = torch.cuda.Stream(device=tdev)
    with (torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()):
        x0_rows = X0[:, r0:r1] if perm is None else X0[:, r0:r1][:, perm]
        if use_halo:
            send_local = torch.from_numpy(inv[send_old]).to(tdev)
            step = lambda Xp: ex.halo_compact(Xp, plan, send_local, rb.B)  # noqa: E731
        elif ex.world > 1:
            step = lambda Xp: ex.all_gather_rows(Xp, rb.B)  # noqa: E731
        else:
            step = lambda Xp: None  # noqa: E731  (one rank: x is all local)
        ctx.dist_begin(prm, alpha, beta, x0_rows, X[0].data_ptr(), X[1].data_ptr(), qs.data_ptr(),
                       qm.data_ptr())
        offset = time.perf_counter() - t_entry
        step(X[0])
        st_ = {"p": 0, "halo_done": None}

        def iterate():
            p, halo_done = st_["p"], st_["halo_done"]
            if perm is not None:
                ctx.dist_pass_rows(0, n_int, 0)  # interior rows: own x only
                if halo_done is not None:
                    stream.wait_event(halo_done)  # the halo of x_p has landed
                ctx.dist_pass_rows(n_int, n_rows, 1)
                ctx.dist_reduce()
            else:
                ctx.dist_pass()
            if ex.world > 1:
                ex.combine(qs, qm)  # one collective for the SUM and MAX partials
            ctx.dist_control()
            p += 1
            if overlap:  # x_{p+1} is final once control p ran: exchange it behind the next interior pass
                ready = torch.cuda.Event()
                ready.record(stream)
                comm.wait_event(ready)
                with torch.cuda.stream(comm):
                    ex_x.halo_compact(X[p & 1], plan, send_local, rb.B)
                    halo_done = torch.cuda.Event()
                    halo_done.record(comm)
            else:
                step(X[p & 1])
            st_["p"], st_["halo_done"] = p, halo_done

        if graph is None:
            graph = os.environ.get("DCX_DIST_GRAPH", "0") == "1"
        use_graph = bool(graph) and stream is not None and not ex.host_staged
        K = max(1, int(poll_every))
        if use_graph:
            K += K & 1  # an even chunk: every replay starts on the same iterate buffer parity
        for _ in range(K):  # the first chunk eagerly (communicators, kernel attributes set up)
            iterate()
        live, _ = ctx.dist_poll()
        if live and use_graph:
            # the chunk ends joined (the last exchange waited for), so a replay depends on nothing
            # recorded outside it; one interior pass per chunk loses its overlap
            if st_["halo_done"] is not None:
                stream.wait_event(st_["halo_done"])
                st_["halo_done"] = None
            g = torch.cuda.CUDAGraph()
            # capture_begin / capture_end directly: torch.cuda.graph() would also run a full
            # device synchronize and gc.collect() inside the solve
            with torch.cuda.stream(stream):
                g.capture_begin(capture_error_mode="thread_local")
                try:
                    for _ in range(K):
                        iterate()
                    if st_["halo_done"] is not None:
                        stream.wait_event(st_["halo_done"])
                        st_["halo_done"] = None
                finally:
                    g.capture_end()
            while live:
                g.replay()
                live, _ = ctx.dist_poll()
        while live:
            for _ in range(K):
                iterate()
            live, _ = ctx.dist_poll()
        if st_["halo_done"] is not None:
            stream.wait_event(st_["halo_done"])
        ctx.dist_finish()
        # best spins and final states of every row block, gathered to every rank (padded space);
        # the spins cross as int8 (1 byte per entry), and one rank keeps its own arrays
        bs, st = ctx.best_spins(), ctx.state()
        if perm is not None:
            bs, st = bs[:, inv], st[:, inv]
        if ex.world == 1:
            best, xs = bs.astype(np.float64), st
        else:
            lo = ex.rank * rb.B
            full_b = torch.zeros(rb.n_space, R, dtype=torch.int8, device=tdev)
            full_b[lo:lo + n_rows] = torch.from_numpy(np.ascontiguousarray(bs.T)).to(tdev)
            ex.all_gather_rows(full_b, rb.B)
            full_x = torch.zeros(rb.n_space, R, dtype=torch.float64, device=tdev)
            full_x[lo:lo + n_rows] = torch.from_numpy(np.ascontiguousarray(st.T)).to(tdev)
            ex.all_gather_rows(full_x, rb.B)
            if stream is not None:
                stream.synchronize()
            best = rb.unpad(full_b.cpu().numpy().T).astype(np.float64)
            xs = rb.unpad(full_x.cpu().numpy().T)
        if stream is not None:
            stream.synchronize()
    return assemble_results(ctx, solver, R, best, xs, offset, getattr(instance, "cut_offset", None), seeds,
                            path="row-partitioned/" + ("halo" if use_halo else "allgather"))
