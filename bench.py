"""Benchmark: DOCH on K2000 dense +-1 x 1024 replicas (BASELINE.json configs[1]).

One step = one batched solve of R replicas (seeds rank*R .. rank*R+R-1, DOCH,
eta = 0.1, max_iters = 1000, trace_stride = 1 -- the reference solve() default)
through the public API. Metric: spin-updates/s = n * sum_r iterations_r / time
(BASELINE.md §2). Multi-GPU (torchrun): replicas shard across ranks (weak
scaling: R replicas per rank), no data-path collective; the max device time
over ranks and the summed spin-updates give the whole-job value.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the CPU reference restated in oracle/ (numpy +
OpenBLAS, one dgemv per replica per product exactly as dcising does) on the
host cores, on a bounded sample of the same workload.
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
REF_BEST_CUT = 595.0 + 32898.0  # best DOCH cut of the CPU reference over 32 seeds
TTS_FRACTION = 0.99  # dc/bench.py:111


def traffic_bytes(config: str, kernel: str, iterations: int):
    """DRAM bytes of one profiled launch of `kernel` on `config` from the committed ncu
    capture (profiles/r1_traffic.json: dram__bytes_read + dram__bytes_write per iteration)."""
    try:
        with open(ROOT / "profiles" / "r1_traffic.json") as f:
            return float(json.load(f)[f"{config}:{kernel}"]["dram_bytes_per_iteration"]) * iterations
    except (OSError, KeyError, ValueError):
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


def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce(vals, op, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
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


# ------------------------------------------------------------------ CPU reference (oracle port)
def cpu_sample(n_rep=8, max_iters=200, seed0=0, solver="doch"):
    """Bounded sample of the workload on the host: n_rep replicas run one after
    another, each a full DOCH / ADOCH loop (2 dgemv per iteration at stride 1)."""
    from oracle import dcising_oracle as orc

    J = -0.5 * instance()
    op = orc.Operator(J)
    updates = 0
    t0 = time.perf_counter()
    for r in range(n_rep):
        out = orc.run(op, ALPHA, BETA, solver=solver, max_iters=max_iters, seed=seed0 + r, trace_stride=1)
        updates += N_SPINS * out["iterations"]
    dt = time.perf_counter() - t0
    return updates / dt, dt, updates


def run_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    n_rep, iters = 256, 1000  # ~10 s of host work per step (replicas converge in ~150-250 iterations)
    for _ in range(args.warmup):
        cpu_sample(1, 20, solver=args.solver)
    vals, times = [], []
    for s in range(args.steps):
        v, dt, _ = cpu_sample(n_rep, iters, seed0=s * n_rep, solver=args.solver)
        vals.append(v)
        times.append(dt)
    value = sum(vals) / len(vals)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": "spin-updates/s", "value": value, "unit": "spin-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"K2000 dense +-1 (gen_dense_pm1 seed 20240817), {args.solver.upper()}, eta=0.1, "
                               "trace_stride=1",
                   "n": N_SPINS, "replicas_per_step": n_rep, "max_iters": iters},
        "cpu_baseline": {"value": value, "unit": "spin-updates/s", "cores": cores, "kind": "port",
                         "sample": f"{n_rep} replicas x <= {iters} {args.solver.upper()} iterations per step, sequential, "
                                   f"numpy/OpenBLAS dgemv with {cores} BLAS threads (oracle/dcising_oracle.py)"},
        "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    world, rank, local = dist_setup(args.gpus)
    os.environ["DCX_DEVICE"] = str(local)
    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import _native

    W = instance()
    seeds_of = lambda step: [rank * REPLICAS + (step * world * REPLICAS) + r for r in range(REPLICAS)]  # noqa: E731
    J = dc.maxcut_to_ising(dc.DenseCoupling(W, validate=False))
    inst = dc.ProblemInstance(coupling=J, cut_offset=CUT_OFFSET)
    kw = dict(max_iters=MAX_ITERS, trace_stride=1, precision=args.precision, path=args.path)
    # L2 flush buffer (> 126 MB L2) written between timed steps
    import torch

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    X0 = [x0_batch(seeds_of(s)) for s in range(2)]
    for w in range(args.warmup):
        dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0[w % 2], **kw)
    # ---------------- device-resident timing (value)
    dev_s, updates, best_e, tts = [], 0, np.inf, []
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))
            torch.cuda.synchronize()
            res = dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0[s % 2], **kw)
            dev_s.append(res[0].device_seconds)
            updates += N_SPINS * sum(r.iterations for r in res)
            max_iters_seen = max(r.iterations for r in res)
            best_e = min(best_e, min(r.energy for r in res))
            target = TTS_FRACTION * REF_BEST_CUT
            for r in res:
                t = r.trace.first_reach_time(target)
                if t is not None:
                    tts.append(t)
    torch.cuda.synchronize()
    barrier(world)
    t_total = sum(dev_s)
    t_max, = allreduce([t_total], "max", world)
    upd_sum, = allreduce([float(updates)], "sum", world)
    best_all, = allreduce([best_e], "min", world)
    value = upd_sum / t_max
    # ---------------- end-to-end through the public API with host buffers
    e2e_t, e2e_upd = 0.0, 0
    h2d = d2h = 0
    barrier(world)
    for s in range(args.steps):
        flush.fill_(float(s))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # host buffers in, host results out: J (f64) and x0 are copied to the device every step
        res = dc.solve_replicas(inst, args.solver, ALPHA, BETA, X0[s % 2], reupload=True, **kw)
        energies = np.array([r.energy for r in res])
        e2e_t += time.perf_counter() - t0
        e2e_upd += N_SPINS * sum(r.iterations for r in res)
        h2d = W.nbytes + X0[0].nbytes
        d2h = REPLICAS * N_SPINS * (1 + 8) + energies.nbytes
    e_max, = allreduce([e2e_t], "max", world)
    e_upd, = allreduce([float(e2e_upd)], "sum", world)
    # ---------------- dominant kernel roofline (measured live, CUDA events on the solver stream)
    prof = dc.profile_dominant_kernel(inst, ALPHA, BETA, X0[0], solver=args.solver, precision=args.precision,
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
            "kernel": prof["kernel"], "ms_per_launch": prof["ms_per_launch"], "peak_source": src}
    roof["frac"] = roof["achieved"] / roof["peak"]
    its = max_iters_seen + 1
    per_iter = {"multipass": 2, "persistent": 0, "dense_tc": 0}.get(res[0].path, 2)
    chunk = 32
    if res[0].path == "multipass":
        launches_total = args.steps * (per_iter * chunk * -(-its // chunk) + 4)
    else:
        launches_total = args.steps * (-(-its // MAX_ITERS) + 3)
    cpu = None
    if rank == 0:
        v, dt, _ = cpu_sample(256, 1000, solver=args.solver)
        cpu = {"value": v, "unit": "spin-updates/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"256 replicas x <= 1000 {args.solver.upper()} iterations (to convergence), sequential, "
                         f"numpy/OpenBLAS dgemv "
                         f"with {os.cpu_count()} BLAS threads ({dt:.1f} s)"}
    if rank == 0:
        mean_tts = float(np.mean(tts)) if tts else None
        line = {
            "metric": "spin-updates/s", "value": value, "unit": "spin-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"f32": "f32", "f64": "f64", "f16tc": "f16"}[args.precision], "data": "synthetic",
            "config": {"workload": f"K2000 dense +-1 (gen_dense_pm1 seed 20240817, J=-W/2), {args.solver.upper()}, "
                                   "eta=0.1 (alpha, beta of derive_params), max_iters=1000, trace_stride=1",
                       "n": N_SPINS, "replicas_per_gpu": REPLICAS, "path": res[0].path,
                       "precision": args.precision, "parallelism": f"replicas x{world}",
                       "l2": "256 MB buffer written between timed steps (instance fits in L2)"},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e_upd / e_max, "unit": "spin-updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches_total,
            "clocks": clk.summary(),
            "quality": {"best_energy": best_all, "best_cut": CUT_OFFSET - best_all,
                        "reference_best_cut_32_seeds": REF_BEST_CUT,
                        "tts_s_mean": mean_tts, "tts_reached": len(tts), "tts_target_cut": TTS_FRACTION * REF_BEST_CUT},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


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
