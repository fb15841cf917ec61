"""Secondary benchmark configurations of BASELINE.json (bench.py --config ...).

The default bench line is K2000 x 1024 (configs[1]). These run the other
single-GPU configs through the same public API and report the same JSON keys:

  g1  configs[0]: 800-spin G1-shape graph, eta = 0.25, DOCH, 100 seeds as one
      batch (f64, persistent one-CTA-per-replica kernel). Latency bound.
  t6  configs[2]: 1000 x 1000 +-1 torus, 256 replicas, DOCH, eta = 1 (f32
      multipass, pass_rn). HBM bound.
  e7  configs[3]: Erdos-Renyi n = 1e7, degree 8, unit MaxCut, 1 replica, DOCH,
      eta = 1 (f32 multipass, pass_r1). HBM / L2-gather bound.
  r8  configs[4] on one GPU: random 3-regular n = 1e8, unit MaxCut, 1 replica,
      DOCH, eta = 1, 20 iterations.

Under torchrun (WORLD_SIZE > 1), or with --rowpart at one GPU, t6 / e7 / r8
run the row-partitioned solver of dist.py instead (each rank owns a row block,
x exchanged per iteration by all-gather or the neighbour-only halo, --exchange);
`value` is then the whole problem's spin-updates over the maximum device time
over ranks ("scaling": "strong": the instance is fixed, the ranks split it).

Algorithmic bytes per iteration (the HBM roofline numerator):
nnz * (4 + value bytes) + (n + 1) * 4 + R * n * 4 * 2.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np


def _peaks():
    from bench import peaks

    return peaks()


def _cuda_count():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _instance(name):
    import paper_2509_01928_b200 as dc
    from paper_2509_01928_b200 import synth

    if name == "g1":
        v, c, o, co = synth.g1_shape()
        J = dc.CsrCoupling(800, v, c, o, validate=False)
        # derive_params at the tuned eta = 0.25 (tests/golden/golden.json "g1")
        return dc.ProblemInstance(coupling=J, cut_offset=co), 6.108031887826326, 884913.7454957356, (v, c, o)
    if name == "t6":
        v, c, o = synth.torus(1000, seed=0)
        J = dc.CsrCoupling(10**6, v, c, o, validate=False)
        return dc.ProblemInstance(coupling=J), 4.0, 8.0e9, (v, c, o)
    if name in ("e7", "r8"):
        n = 10**7 if name == "e7" else 10**8
        dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, _cuda_count()) if _cuda_count() else None
        v, c, o, co = (synth.erdos_renyi(n, 8, seed=0, device=dev) if name == "e7"
                       else synth.random_regular3(n, seed=0, device=dev))
        J = dc.CsrCoupling(n, v, c, o, validate=False)
        # derive_params at eta = 1: the Wigner estimate (n >= 1e4, dc/spectral.py:175-189) and
        # beta's max row |J|_1, both from the device row statistics (dcx_row_stats)
        p = dc.derive_params(J, eta=1.0)
        return dc.ProblemInstance(coupling=J, cut_offset=co), p.alpha, p.beta, (v, c, o)
    raise ValueError(name)


CFG = {
    "g1": dict(R=100, max_iters=1000, precision="f64", desc="800-spin G1-shape MaxCut, eta=0.25, DOCH, 100 seeds"),
    "t6": dict(R=256, max_iters=200, precision="f32", desc="1000x1000 +-1 torus, 256 replicas, DOCH, eta=1"),
    "e7": dict(R=1, max_iters=200, precision="f32",
               desc="Erdos-Renyi n=1e7 deg 8 unit MaxCut, 1 replica, DOCH, eta=1, 200 iterations (the reference run's budget)"),
    "r8": dict(R=1, max_iters=20, precision="f32", desc="random 3-regular n=1e8 unit MaxCut, 1 replica, DOCH, eta=1, 1 GPU"),
}


def reference_quality(name):
    """The unmodified reference's quality on this config, computed offline (tests/golden):
    G1 -- best cut over 100 seeds x DOCH/ADOCH at eta = 0.25 (golden.json); E7 -- the best cut of
    one 200-iteration DOCH run (golden_e7.json); T6 -- minus the best energy of one
    200-iteration DOCH run, seed 0 (golden_t6.json). None when not available."""
    import json
    from pathlib import Path

    gdir = Path(__file__).resolve().parent / "tests" / "golden"
    try:
        if name == "g1":
            g = json.loads((gdir / "golden.json").read_text())["g1"]
            return max(max(r["cut"] for r in g[s]) for s in ("doch", "adoch")), "best cut of the reference over 100 seeds x DOCH/ADOCH"
        if name == "e7":
            g = json.loads((gdir / "golden_e7.json").read_text())
            return g["best_cut"], f"best cut of one {g['iterations']}-iteration reference DOCH run (seed 0)"
        if name == "r8":
            g = json.loads((gdir / "golden_r8.json").read_text())
            return g["best_cut"], f"best cut of one {g['iterations']}-iteration reference DOCH run (seed 0)"
        if name == "t6":  # a spin glass: quality = -best energy (no cut offset)
            g = json.loads((gdir / "golden_t6.json").read_text())
            return -g["best_energy"], f"-(best energy) of one {g['iterations']}-iteration reference DOCH run (seed 0)"
    except (OSError, KeyError, ValueError):
        return None
    return None


def cpu_sample(name, inst, alpha, beta, arrays, budget_s=20.0, target=None):
    """Oracle port on the host: replicas one after another, bounded in time; with `target`
    also the time to reach it (dc/bench.py:219-231 semantics, on the port's own clock)."""
    from oracle import dcising_oracle as orc

    op = orc.Operator(arrays)
    n = op.n
    iters = {"g1": 1000, "t6": 20, "e7": 3, "r8": 1}[name]
    upd, t0, r = 0, time.perf_counter(), 0
    tts = []
    co = getattr(inst, "cut_offset", None)
    while True:
        out = orc.run(op, alpha, beta, solver="doch", max_iters=iters, seed=r, trace_stride=1, cut_offset=co)
        upd += n * out["iterations"]
        if target is not None and co is not None:
            hit = [t["elapsed_s"] for t in out["trace"] if co - t["best_energy"] >= target]
            if hit:
                tts.append(hit[0])
        r += 1
        if time.perf_counter() - t0 > budget_s or r >= 8:
            break
    dt = time.perf_counter() - t0
    sample = f"{r} replicas x <= {iters} DOCH iterations, numpy/scipy csr_matvec ({dt:.1f} s)"
    return upd / dt, dt, sample, (float(np.mean(tts)) if tts else None, len(tts), r)


def _csr_bytes(J):
    v = getattr(J, "values", None)
    if v is None:
        return 0
    return int(np.asarray(v).nbytes + np.asarray(J.col_indices).nbytes + np.asarray(J.row_offsets).nbytes)


def run_rowpart(args, name, cfg, inst, alpha, beta, X0, t_build):
    """Row-partitioned t6 / e7 / r8 (dist.py) on WORLD_SIZE ranks, one GPU each."""
    import torch
    import torch.distributed as dist

    from bench import ClockSampler, allreduce, barrier, dist_setup
    from paper_2509_01928_b200 import dist as dd

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if not dist.is_initialized():  # --rowpart at one GPU: NCCL world of one
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    n, R = inst.coupling.n, X0.shape[0]
    kw = dict(max_iters=cfg["max_iters"], trace_stride=1, precision=cfg["precision"], device=local,
              exchange=args.exchange, poll_every=16)
    for _ in range(args.warmup):
        dd.solve_distributed(inst, "doch", alpha, beta, X0, **kw)
    dev, wall, upd = 0.0, 0.0, 0
    barrier(dist.get_world_size())
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = dd.solve_distributed(inst, "doch", alpha, beta, X0, **kw)
            wall += time.perf_counter() - t0
            dev += res[0].device_seconds
            upd += n * sum(r.iterations for r in res)
    torch.cuda.synchronize()
    ws = dist.get_world_size()
    dev_max, = allreduce([dev], "max", ws)
    wall_max, = allreduce([wall], "max", ws)
    if rank == 0:
        e = np.array([r.energy for r in res])
        line = {
            "metric": "spin-updates/s", "value": upd / dev_max, "unit": "spin-updates/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg["precision"],
            "data": "synthetic",
            "config": {"workload": cfg["desc"].replace(", 1 GPU", "") + f", row-partitioned over {ws} GPU(s)",
                       "n": n, "replicas": R, "max_iters": cfg["max_iters"], "path": res[0].path,
                       "parallelism": f"rows x{ws}", "host_instance_build_s": round(t_build, 1),
                       "l2": "state + CSR stream exceed L2"},
            # the public entry point re-uploads the row block and x0 every solve (host buffers in,
            # best spins and final x gathered back to every rank)
            "e2e": {"value": upd / wall_max, "unit": "spin-updates/s", "h2d_bytes_per_step": int(X0.nbytes),
                    "d2h_bytes_per_step": int(X0.nbytes + R * n)},
            "clocks": clk.summary(),
            "quality": {"best_energy": float(e.min()), "mean_energy": float(e.mean())},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_gen9(args):
    """gen_sparse_9bit on the device vs the reference's generator
    loop on the host. Work unit: one draw of the lower triangle (n(n-1)/2 per instance)."""
    import torch

    import paper_2509_01928_b200 as dc
    from oracle import dcising_oracle as orc

    n, p = 100_000, 1.0
    draws = n * (n - 1) / 2
    for s in range(args.warmup):
        dc.gen_sparse_9bit(n, p, seed=s)
    ctx = dc.generate._context()
    dev = 0.0
    wall = 0.0
    for s in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # end to end: generation on the device + download into the reference's int64 / f64 arrays
        J = dc.gen_sparse_9bit(n, p, seed=100 + s)
        wall += time.perf_counter() - t0
    # device-only timing of the generation call through the context (result left on the device)
    import ctypes

    stream = torch.cuda.ExternalStream(ctx.stream())
    for s in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = ctypes.c_int64()
        e0.record(stream)
        rc = ctx.lib.dcx_gen_sparse_9bit(ctx.h, n, int(102300 // p), 200 + s, ctypes.byref(out))
        e1.record(stream)
        if rc != 0:
            raise RuntimeError(ctx.lib.dcx_last_error(ctx.h).decode())
        e1.synchronize()
        dev += e0.elapsed_time(e1) * 1e-3  # CUDA events on the context stream
    cpu_n = 8000
    t0 = time.perf_counter()
    orc.gen_sparse_9bit_numpy(cpu_n, p, 1)
    cpu_t = time.perf_counter() - t0
    line = {
        "metric": "lower-triangle draws/s", "value": args.steps * draws / dev, "unit": "draws/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 (Philox4x64-10)",
        "data": "synthetic",
        "config": {"workload": f"gen_sparse_9bit(n={n}, p={p}) on the device: per-row Philox streams, "
                               "symmetric CSR in the reference's int64/f64 layout", "n": n, "nnz": int(J.nnz)},
        "e2e": {"value": args.steps * draws / wall, "unit": "draws/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(J.nnz * 16 + (n + 1) * 8)},
        "roofline": {"bound": "int pipe (64-bit multiply-high)", "achieved": None, "peak": None, "unit": None,
                     "frac": None, "traffic": None, "kernel": "rows_9bit"},
        "cpu_baseline": {"value": cpu_n * (cpu_n - 1) / 2 / cpu_t, "unit": "draws/s", "cores": 1, "kind": "port",
                         "sample": f"the reference's generator loop (numpy Philox per row, scipy COO->CSR) at "
                                   f"n={cpu_n}, p={p} ({cpu_t:.2f} s)"},
    }
    print(json.dumps(line), flush=True)


def run(args):
    import paper_2509_01928_b200 as dc

    name = args.config
    if name == "gen9":
        run_gen9(args)
        return
    cfg = CFG[name]
    t_build = time.perf_counter()
    inst, alpha, beta, arrays = _instance(name)
    t_build = time.perf_counter() - t_build
    n = inst.coupling.n
    R = cfg["R"]
    X0 = np.stack([dc.initial_state(n, alpha, beta, np.random.default_rng(s)) for s in range(R)])
    if name != "g1" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or getattr(args, "rowpart", False)):
        run_rowpart(args, name, cfg, inst, alpha, beta, X0, t_build)
        return
    kw = dict(max_iters=cfg["max_iters"], trace_stride=1, precision=cfg["precision"])
    for _ in range(args.warmup):
        dc.solve_replicas(inst, "doch", alpha, beta, X0, **kw)
    dev, upd, wall = 0.0, 0, 0.0
    dc.solve_replicas(inst, "doch", alpha, beta, X0, reupload=True, **kw)  # warm the upload path (untimed)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        # host buffers in (the CSR arrays and x0 are uploaded every step), the energies out
        res = dc.solve_replicas(inst, "doch", alpha, beta, X0, reupload=True, **kw)
        energies = np.array([r.energy for r in res])
        wall += time.perf_counter() - t0
        dev += res[0].device_seconds
        upd += n * sum(r.iterations for r in res)
    path = res[0].path
    value = upd / dev
    hbm, bf16, src = _peaks()
    line = {
        "metric": "spin-updates/s", "value": value, "unit": "spin-updates/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg["precision"],
        "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": n, "replicas": R, "max_iters": cfg["max_iters"], "path": path,
                   "host_instance_build_s": round(t_build, 1),
                   "l2": "state + CSR stream exceed L2" if name != "g1" else "whole instance on chip (smem)"},
        # h2d: the CSR as the caller holds it (int64 offsets / columns, f64 values) and x0;
        # d2h: the per-replica summaries (energy, iterations, stop, history length, warning);
        # final states and best spins stay on the device until read (solvers._Bulk)
        "e2e": {"value": upd / wall, "unit": "spin-updates/s",
                "h2d_bytes_per_step": int(X0.nbytes + _csr_bytes(inst.coupling)),
                "d2h_bytes_per_step": int(energies.nbytes + R * 24)},
    }
    if path == "multipass":
        prof = dc.profile_dominant_kernel(inst, alpha, beta, X0, precision=cfg["precision"], path="multipass",
                                          launches=10)
        gbs = prof["bytes_per_launch"] / (prof["ms_per_launch"] * 1e-3) / 1e9
        from bench import traffic_bytes

        line["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                            "traffic": traffic_bytes(name, prof["kernel"], 1),
                            "kernel": prof["kernel"], "ms_per_launch": prof["ms_per_launch"],
                            "bytes_per_launch": prof["bytes_per_launch"], "peak_source": src}
    else:
        line["roofline"] = {"bound": "latency", "achieved": None, "peak": None, "unit": "us/iteration",
                            "frac": None, "traffic": None,
                            "us_per_iteration": 1e6 * dev / args.steps / max(r.iterations for r in res)}
    ref_q = reference_quality(name)
    target = 0.99 * ref_q[0] if ref_q else None  # dc/bench.py:111 tts_fraction
    v, dt, sample, cpu_tts = cpu_sample(name, inst, alpha, beta, arrays, target=target)
    line["cpu_baseline"] = {"value": v, "unit": "spin-updates/s", "cores": os.cpu_count(), "kind": "port",
                            "sample": sample}
    e = np.array([r.energy for r in res])
    line["quality"] = {"best_energy": float(e.min()), "mean_energy": float(e.mean()),
                       "seed0_best_energy": float(res[0].energy)}  # replica 0 = the reference run's seed
    if inst.cut_offset is not None:
        line["quality"]["best_cut"] = float(inst.cut_offset - e.min())
    if target is not None:
        # time to target (dc/bench.py:219-231): first elapsed_s whose best-so-far cut reaches
        # 0.99 x the reference's quality; GPU on the solve's device clock, the port on its own
        tts = [t for t in (r.trace.first_reach_time(target) for r in res) if t is not None]
        line["quality"].update({"tts_target_cut": target, "reference_quality": ref_q[1], "reference_best_cut": ref_q[0],
                                "tts_s_mean": float(np.mean(tts)) if tts else None, "tts_reached": len(tts),
                                "replicas": len(res), "cpu_tts_s_mean": cpu_tts[0],
                                "cpu_tts_reached": f"{cpu_tts[1]} of {cpu_tts[2]}"})
        if inst.cut_offset is None:  # quality = -energy: the same numbers under their own names
            line["quality"].update({"tts_target_energy": -target, "reference_seed0_best_energy": -ref_q[0]})
    print(json.dumps(line), flush=True)
