"""Benchmark: DOCH on K2000 dense +-1 x 1024 replicas (BASELINE.json configs[1]).

One step = one batched solve of R = 1024 replicas with seeds 0..1023 (the
reference's restart convention seed + r, dc/bench.py:311), DOCH, eta = 0.1,
max_iters = 1000, trace_stride = 1 (the reference solve() default), through
the public API. Every replica runs until the reference's own stop test
(step <= 1e-10, max_iters) fires. Metric: spin-updates/s = n * sum_r
iterations_r / solve time, next to the solve time, the
time-to-target (dc/bench.py:219-231, target 0.99 x the reference's best cut
over the same 1024 seeds) and the reference's stop-reason / iteration counts.
Multi-GPU (torchrun, or --gpus N which re-launches itself under torchrun):
replicas shard across ranks (weak scaling: rank k solves seeds 1024k..), no
data-path collective; the max device time over ranks and the summed
spin-updates give the whole-job value.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the UNMODIFIED reference (dcising 0.1.0 installed
in baseline/_ref) through its own public ``solve()`` on the host cores: the
restarts on a process pool of os.cpu_count() workers with OMP_NUM_THREADS=1
(dc/bench.py:318-328's restart parallelism) or sequentially with all BLAS
threads, whichever measured faster in the warm-up; each step is a bounded
sample of the same 1024 seeds.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_SPINS = 2000
REPLICAS = 1024
ETA = 0.1
MAX_ITERS = 1000
# derive_params(J, eta=0.1, tol=1e-8) of the reference on this instance (tests/golden/golden.json "k2")
ALPHA = 4.462132927392335
BETA = 89797103.04245317
CUT_OFFSET = 595.0  # sum_{i<j} W_ij / 2 for W = gen_dense_pm1(2000, 20240817)
TTS_FRACTION = 0.99  # dc/bench.py:111


def reference_k2(solver="doch"):
    """The unmodified reference on the same instance and seeds 0..1023
    (tests/golden/golden_k2.json, written by tests/golden/make_golden_k2.py)."""
    g = json.loads((ROOT / "tests" / "golden" / "golden_k2.json").read_text())
    return g, g[solver]


def traffic_bytes(config: str, kernel: str, iterations: int):
    """DRAM bytes of one profiled launch of `kernel` on `config` from the committed ncu
    captures (profiles/r2_traffic.json, then r1: dram__bytes_read + dram__bytes_write per iteration)."""
    for name in ("r2_traffic.json", "r1_traffic.json"):  # newest capture first
        try:
            with open(ROOT / "profiles" / name) as f:
                return float(json.load(f)[f"{config}:{kernel}"]["dram_bytes_per_iteration"]) * iterations
        except (OSError, KeyError, ValueError):
            continue
    return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(gpus, backend=None):
    """torchrun environment -> (world, rank, local device). The K2 replica shards only
    reduce a few scalars at the end: NCCL when every rank has its own GPU, else gloo
    (ranks sharing one GPU run their independent solves one after another)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = max(1, torch.cuda.device_count())
        local = local % ndev
        torch.cuda.set_device(local)
        if backend is None:
            backend = "nccl" if ndev >= world else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def _backend():
    import torch.distributed as dist

    return dist.get_backend() if dist.is_initialized() else None


def allreduce(vals, op, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device="cuda" if _backend() == "nccl" else "cpu")
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN}[op])
    return t.tolist()


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def instance():
    from paper_2509_01928_b200 import synth

    return synth.dense_pm1(N_SPINS, seed=20240817)


def x0_batch(seeds):
    from paper_2509_01928_b200 import initial_state

    return np.stack([initial_state(N_SPINS, ALPHA, BETA, np.random.default_rng(int(s))) for s in seeds])


# ------------------------------------------------------------------ CPU reference (unmodified dcising)
_REF = {}


def _ref_init(alpha, beta, worker=False):
    """Worker initialiser: the unmodified reference from baseline/_ref and the K2000 instance.
    Pool workers run single-threaded BLAS (OMP_NUM_THREADS=1 semantics; a forked worker
    inherits an already-initialised OpenBLAS, so the limit is applied through threadpoolctl)."""
    if worker:
        from threadpoolctl import threadpool_limits

        _REF["limits"] = threadpool_limits(1)
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import dcising as rdc
    from dcising.generate import gen_dense_pm1

    W = gen_dense_pm1(N_SPINS, seed=20240817)
    _REF["dc"] = rdc
    _REF["inst"] = rdc.ProblemInstance(coupling=rdc.maxcut_to_ising(W), name="k2000", cut_offset=CUT_OFFSET)
    _REF["params"] = rdc.SolverParams(alpha=alpha, beta=beta, eta=ETA, max_iters=MAX_ITERS)


def _ref_one(task):
    """One restart through the reference's public solve() with premade params, exactly as
    run_bench's _bench_one (dc/bench.py:242-259); returns (iterations, energy, TTS)."""
    solver, seed, threshold = task
    rdc = _REF["dc"]
    from dcising.bench import first_reach_time

    res = rdc.solve(_REF["inst"], solver, seed=seed, eta=ETA, budget_iters=MAX_ITERS, params=_REF["params"],
                    trace_stride=1)
    return res.iterations, res.energy, first_reach_time(res.trace, threshold, use_cut=True), \
        res.stop_reason == "converged"


def measure_reference(solver, steps, warmup, step_seconds=3.0):
    """Time the unmodified reference on this host (bounded sample of the 1024 seeds, each
    step sized to about `step_seconds`); returns (spin-updates/s, details) or None when
    baseline/_ref is absent."""
    if not (ROOT / "baseline" / "_ref" / "dcising").exists():
        return None
    from concurrent.futures import ProcessPoolExecutor

    gk, ref = reference_k2(solver)
    threshold = TTS_FRACTION * ref["best_cut"]
    cores = os.cpu_count() or 1
    seq_threads = os.environ.get("OMP_NUM_THREADS")
    _ref_init(ALPHA, BETA)  # in this process: the sequential mode (all BLAS threads)
    pool = ProcessPoolExecutor(max_workers=cores, initializer=_ref_init, initargs=(ALPHA, BETA, True))
    per_step = 2 * cores  # restarts per pool step (~2 solves per worker)

    def run(mode, seeds):
        t0 = time.perf_counter()
        tasks = [(solver, s, threshold) for s in seeds]
        out = list(pool.map(_ref_one, tasks)) if mode == "pool" else [_ref_one(t) for t in tasks]
        return time.perf_counter() - t0, out

    list(pool.map(_ref_init, [ALPHA] * cores, [BETA] * cores, [True] * cores))  # start every worker
    # warm-up: both modes, keep the faster (BASELINE.md §2 / SURVEY.md §8d)
    cur = 0
    rates = {"pool": [], "sequential": []}
    t_seed = {"pool": [], "sequential": []}  # wall seconds per seed
    for w in range(max(1, warmup)):
        seeds = [(cur + i) % REPLICAS for i in range(per_step)]
        dt, out = run("pool", seeds)
        rates["pool"].append(N_SPINS * sum(o[0] for o in out) / dt)
        t_seed["pool"].append(dt / len(seeds))
        dt, out = run("sequential", seeds[:2])
        rates["sequential"].append(N_SPINS * sum(o[0] for o in out) / dt)
        t_seed["sequential"].append(dt / 2)
        cur += per_step
    mode = "pool" if max(rates["pool"]) >= max(rates["sequential"]) else "sequential"
    n_step = max(2, int(step_seconds / max(min(t_seed[mode]), 1e-3)))
    if mode == "pool":
        n_step = max(cores, n_step // cores * cores)
    times, upd, outs = [], 0, []
    cur = 0
    for s in range(steps):
        seeds = [(cur + i) % REPLICAS for i in range(n_step)]
        cur += n_step
        dt, out = run(mode, seeds)
        times.append(dt)
        upd += N_SPINS * sum(o[0] for o in out)
        outs += out
    pool.shutdown()
    value = upd / sum(times)
    tts = [o[2] for o in outs if o[2] is not None]
    sample = (f"{n_step} of the 1024 seeds per step x {steps} steps ({sum(times):.1f} s), unmodified dcising "
              f"0.1.0 (baseline/_ref) solve() with premade params; mode {mode}: "
              + (f"{cores} worker processes, OMP_NUM_THREADS=1" if mode == "pool"
                 else f"one process, BLAS threads {seq_threads or 'default'}"))
    return value, dict(mode=mode, n_step=n_step, times=times, rates={k: max(v) for k, v in rates.items()},
                       cores=cores if mode == "pool" else (int(seq_threads) if seq_threads else cores),
                       sample=sample, threshold=threshold, runs=len(outs),
                       mean_iterations=float(np.mean([o[0] for o in outs])),
                       converged=int(sum(o[3] for o in outs)), best_energy=float(min(o[1] for o in outs)),
                       tts_s_mean=float(np.mean(tts)) if tts else None, tts_reached=len(tts))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m = measure_reference(args.solver, args.steps, args.warmup)
    if m is None:
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/dcising not installed "
                          "(pip install --target baseline/_ref /root/reference/pkg)"}), flush=True)
        return
    value, d = m
    line = {
        "impl": "reference", "metric": "spin-updates/s", "value": value, "unit": "spin-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(d["times"]) / len(d["times"]), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"K2000 dense +-1 (gen_dense_pm1 seed 20240817, J=-W/2), {args.solver.upper()}, "
                               "eta=0.1 (alpha, beta of derive_params), max_iters=1000, trace_stride=1, seeds 0..1023",
                   "n": N_SPINS, "replicas_per_step": d["n_step"], "mode": d["mode"],
                   "modes_measured_in_warmup": d["rates"]},
        "cpu_baseline": {"value": value, "unit": "spin-updates/s", "cores": d["cores"], "kind": "reference",
                         "sample": d["sample"]},
        "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "quality": {k: d[k] for k in ("runs", "mean_iterations", "converged", "best_energy", "tts_s_mean",
                                      "tts_reached")} | {"tts_target_cut": d["threshold"]},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    world, rank, local = dist_setup(args.gpus)
    os.environ["DCX_DEVICE"] = str(local)
    import paper_2509_01928_b200 as dc

    gk, ref = reference_k2(args.solver)
    target = TTS_FRACTION * ref["best_cut"]
    W = instance()
    seeds = [rank * REPLICAS + r for r in range(REPLICAS)]  # rank 0: the reference's seeds 0..1023
    J = dc.maxcut_to_ising(dc.DenseCoupling(W, validate=False))
    inst = dc.ProblemInstance(coupling=J, cut_offset=CUT_OFFSET)
    kw = dict(max_iters=MAX_ITERS, trace_stride=1, precision=args.precision, path=args.path)
    # L2 flush buffer (> 126 MB L2) written between timed steps
    import torch

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    X0 = x0_batch(seeds)
    for w in range(args.warmup):
        dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0, **kw)
    # ---------------- device-resident timing (value)
    dev_s, updates = [], 0
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))
            torch.cuda.synchronize()
            res = dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0, **kw)
            dev_s.append(res[0].device_seconds)
            updates += N_SPINS * sum(r.iterations for r in res)
    torch.cuda.synchronize()
    barrier(world)
    t_total = sum(dev_s)
    t_max, = allreduce([t_total], "max", world)
    upd_sum, = allreduce([float(updates)], "sum", world)
    value = upd_sum / t_max
    # quality of one solve (the same seeds every step): the reference's G-quality numbers
    e = np.array([r.energy for r in res])
    its = np.array([r.iterations for r in res])
    conv = int(sum(r.stop_reason == "converged" for r in res))
    tts = [t for t in (r.trace.first_reach_time(target) for r in res) if t is not None]
    q = allreduce([float(e.min()), float(e.sum()), float(its.sum()), float(its.max()), float(conv),
                   float(len(tts)), float(sum(tts)), float(len(res))], "sum", world)
    best_all, = allreduce([float(e.min())], "min", world)
    its_max, = allreduce([float(its.max())], "max", world)
    n_runs = q[7]
    # ---------------- end-to-end through the public API with host buffers
    e2e_t, e2e_upd = 0.0, 0
    h2d = d2h = 0
    dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0, reupload=True, **kw)  # warm the upload path
    barrier(world)
    for s in range(args.steps):
        flush.fill_(float(s))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # host buffers in, host results out: J (f64) and x0 are copied to the device every step
        res = dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0, reupload=True, **kw)
        energies = np.array([r.energy for r in res])
        e2e_t += time.perf_counter() - t0
        e2e_upd += N_SPINS * sum(r.iterations for r in res)
        h2d = W.nbytes + X0.nbytes
        # the energies and per-replica summaries; final states / best spins stay on the device
        # until a field is read (solvers._Bulk)
        d2h = energies.nbytes + REPLICAS * 24
    e_max, = allreduce([e2e_t], "max", world)
    e_upd, = allreduce([float(e2e_upd)], "sum", world)
    # ---------------- dominant kernel roofline (measured live, CUDA events on the solver stream)
    prof = dc.profile_dominant_kernel(inst, ALPHA, BETA, X0, solver=args.solver, precision=args.precision,
                                      path="multipass" if args.path == "auto" and args.precision != "f16tc"
                                      else args.path, launches=5 if args.precision == "f16tc" else 10)
    hbm, bf16, src = peaks()
    kernel_flops = prof["flops_per_launch"]
    achieved = kernel_flops / (prof["ms_per_launch"] * 1e-3) / 1e12
    peak = bf16 if prof["bound"] == "tensor" else hbm
    roof = {"bound": prof["bound"], "achieved": achieved if prof["bound"] == "tensor" else
            prof["bytes_per_launch"] / (prof["ms_per_launch"] * 1e-3) / 1e9,
            "peak": peak, "unit": "TFLOP/s" if prof["bound"] == "tensor" else "GB/s",
            "traffic": traffic_bytes("k2", prof["kernel"], prof["iterations_per_launch"]),
            "kernel": prof["kernel"], "ms_per_launch": prof["ms_per_launch"], "peak_source": src,
            "work": "2 n^2 R flops per iteration (SURVEY.md §8d: one coupling product; the exact sign "
                    "product is not counted) over iterations 0..99 of all 1024 replicas (all live)",
            "us_per_iteration": 1e3 * prof["ms_per_launch"] / prof["iterations_per_launch"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # solve-level efficiency: live replica-iterations / replica slots x iterations the kernel ran
    per_iter = {"multipass": 2, "persistent": 0, "dense_tc": 0}.get(res[0].path, 2)
    chunk = 32
    its1 = int(its_max) + 1
    # per solve, from the ncu launch list (profiles/r2_k2_launches.txt): the iteration kernels, then
    # x0 layout, start clock, pack / flush, unpack, and the detached result's three gathers
    # (final states, best spins, descent-warning deltas)
    if res[0].path == "multipass":
        launches_total = args.steps * (per_iter * chunk * -(-its1 // chunk) + 7)
    else:
        launches_total = args.steps * (-(-its1 // (MAX_ITERS + 1)) + 7)
    cpu = None
    if rank == 0 and world == 1:  # the unmodified reference on this host, bounded sample (~10-20 s)
        m = measure_reference(args.solver, 1, 1, step_seconds=15.0)
        if m is not None:
            cpu = {"value": m[0], "unit": "spin-updates/s", "cores": m[1]["cores"], "kind": "reference",
                   "sample": m[1]["sample"], "tts_s_mean": m[1]["tts_s_mean"],
                   "mean_iterations": m[1]["mean_iterations"]}
    if rank == 0:
        line = {
            "metric": "spin-updates/s", "value": value, "unit": "spin-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"f32": "f32", "f64": "f64", "f16tc": "f16"}[args.precision], "data": "synthetic",
            "config": {"workload": f"K2000 dense +-1 (gen_dense_pm1 seed 20240817, J=-W/2), {args.solver.upper()}, "
                                   "eta=0.1 (alpha, beta of derive_params), max_iters=1000, trace_stride=1, "
                                   "seeds 0..1023 (rank k: 1024k..), every replica to its own stop",
                       "n": N_SPINS, "replicas_per_gpu": REPLICAS, "path": res[0].path,
                       "precision": args.precision, "parallelism": f"replicas x{world}",
                       "backend": _backend() if world > 1 else None,
                       "l2": "256 MB buffer written between timed steps (instance fits in L2)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e_upd / e_max, "unit": "spin-updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches_total,
            "clocks": clk.summary(),
            "quality": {"replicas": int(n_runs), "best_energy": best_all, "best_cut": CUT_OFFSET - best_all,
                        "mean_energy": q[1] / n_runs, "mean_iterations": q[2] / n_runs, "max_iterations": its_max,
                        "converged": int(q[4]), "solve_ms": 1e3 * t_max / args.steps,
                        "tts_s_mean": q[6] / q[5] if q[5] else None, "tts_reached": int(q[5]),
                        "tts_target_cut": target,
                        "reference_same_seeds": {"best_cut": ref["best_cut"], "mean_energy": ref["mean_energy"],
                                                 "mean_iterations": ref["mean_iterations"],
                                                 "converged": ref["converged"]}},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """bench.py --gpus N (N > 1) outside torchrun: re-execute under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default=os.environ.get("DCX_BENCH_PRECISION", "f16tc"))
    ap.add_argument("--path", default=os.environ.get("DCX_BENCH_PATH", "auto"))
    ap.add_argument("--config", default="k2", choices=["k2", "g1", "t6", "e7", "r8", "gen9"],
                    help="k2 is the headline (BASELINE configs[1]); others: see bench_configs.py")
    ap.add_argument("--solver", default="doch", choices=["doch", "adoch"],
                    help="k2: DOCH (headline) or ADOCH with the economy window")
    ap.add_argument("--rowpart", action="store_true",
                    help="t6/e7/r8: row-partitioned solver (dist.py) even at one GPU")
    ap.add_argument("--exchange", default="auto", choices=["auto", "allgather", "halo"],
                    help="row-partitioned x exchange")
    args = ap.parse_args()
    # descent-violation RuntimeWarnings are per-replica diagnostics (1024 lines of
    # stderr per solve at K2 in f16); neither arm prints them while timed
    import warnings

    warnings.filterwarnings("ignore", category=RuntimeWarning)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.config != "k2" and args.impl == "ours":
        import bench_configs

        bench_configs.run(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
