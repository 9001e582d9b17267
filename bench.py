#!/usr/bin/env python
"""Benchmark of the fp64 FFT-PIC step (3D Landau damping) -- driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): particle-pushes/s (whole job) and ms per PIC step.
N=1 workload: 512^3 grid x 8 ppc (1,073,741,824 particles), k=0.5, alpha=0.05,
dt=0.05 (BASELINE.json configs[2], the paper's case A).
One "step" = one full PIC step: FFT solve + field energy, gather+push, counting
sort by cell key, reorder + CIC deposit.  Inputs live in HBM (51.5 GB of
particle state >> 126 MB L2, so no L2 flush is needed between steps).

--solver pcg runs BASELINE.json configs[4] instead: the same step with the
matrix-free FD-PCG Poisson solve (SSOR(pi/2, 4, 2), tol 1e-4, warm start;
P:179-181) in place of the FFT solve.

Prints ONE JSON line on rank 0.  For N > 1 (torchrun) the same 512^3 problem is
decomposed in z-slabs over the N GPUs (FFT transposes by copy-engine pulls over NVLink, halo/ghost
planes, particle migration): strong scaling of a fixed problem, time = max over ranks.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-pushes/sec (fp64 FFT-PIC step, Landau damping 3D)"
UNIT = "particle-pushes/s"

# Algorithmic bytes per launch:
# per particle, per grid node (ncell = N^3).
# Layout padding is not counted: an E node is 24 B (E_x, E_y, E_z; the 4th double of the
# 32-B record is padding), and the kick's store is v (24 B; z is rewritten unchanged).
ALG_BYTES = {
    "reorder_deposit": (4 + 48 + 48, 4 + 16),        # perm, x/v gather, x'/v' store | offs, rho RMW
    "push_key": (48 + 24 + 4 + 2, 24 + 8),           # x/v read, kicked v, key, rank | E tile, count RMW
    "place": (4 + 2 + 4, 4),                         # key, rank read, perm write | offs
    "scan": (0, 16),                                 # count read x2, offs + cursor write
    "fft_x_fwd": (0, 8 + 8),
    "fft_y_fwd": (0, 8 + 8),
    "fft_z_mul": (0, 8 + 16),                       # rho^ pencil -> phi^, E^_z
    "fft_y_inv": (0, 16 + 24),                      # phi^, E^_z -> E_x, E_y, E_z spectra
    "fft_x_inv": (0, 24 + 24),                       # 3 half spectra -> E node records (24 B each)
    "clear": (0, 4 + 8),
    # FD-PCG (BJ config 5), per launch of the stage's main kernel:
    "pcg_field": (0, 8 + 24),                       # phi (stencil) -> E node records
}
# PCG stages with launches of different kinds: algorithmic bytes per node per
# application.  SSOR M^-1 (4 inner x 2 outer = 32 half-sweeps): 8 + 12 + 29 x 16 + 20
# B/node; one CG iteration: matvec 32 (z, p read; p', q written) + update 48
# (x, p, r, q read; x, r written) B/node.
PCG_SSOR_BYTES_PER_APPLY = 504
PCG_CG_BYTES_PER_ITER = 80


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def reduce_max(x: float, world: int) -> float:
    """Max over ranks (device time is taken per rank; the job time is the slowest)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, world: int) -> float:
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def broadcast_nccl_id(rank: int, world: int):
    """One NCCL unique id for the library's communicator (rank 0 makes it)."""
    if world <= 1:
        return None
    import torch.distributed as dist
    from paper_2605_05469_b200 import nccl_unique_id

    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        busy = sorted(sm)[len(sm) // 4:] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(config_name: str, kernel: str):
    """Per-launch DRAM bytes (dram__bytes_read + write) of a kernel at this config from the
    committed ncu launch list (profiles/ncu_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(config_name, {}).get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------ oracle (CPU) --
def _oracle_steps(solver, n, L, xv, steps):
    from oracle import oracle as O

    if solver == "pcg":
        return O.run_pcg(n, L, 0.05, xv, steps)[0]
    if solver == "fem":
        return O.run_fem(n, L, 0.05, xv, steps)[0]
    if solver == "pif":
        import numpy as np
        from oracle import nufft as U

        return U.pif_run(n, L, 0.05, xv, np.full(xv.shape[1], -L ** 3 / xv.shape[1]), steps)[0]
    return O.run(n, L, 0.05, xv, steps)[0]


def host_cpu():
    """lscpu model name and the number of physical cores (unique (core, socket) pairs)."""
    model, cores = None, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        cores = len({l for l in out.splitlines() if l and not l.startswith("#")}) or None
    except Exception:
        pass
    return model, cores or os.cpu_count() or 1


def oracle_leg(n: int, ppc: int, steps: int, threads: int, solver: str = "fft"):
    """Time the CPU oracle, as it stands, for `steps` steps of Landau n^3 x ppc on `threads`
    threads (1 = the serial parity mode, > 1 = the OpenMP-deterministic mode, SURVEY c.5).
    The initial state is the oracle's own sampler (untimed); the timed call is oracle_run,
    which also canonicalises the (already sorted) input once."""
    import numpy as np
    from oracle import oracle as O

    L = 4 * np.pi
    with O.threads(threads):
        xv = O.sample_landau(ppc * n ** 3, 0.5, L, 0.05, 1)
        xv, _ = O.sort(n, L, xv)
        t0 = time.perf_counter()
        _oracle_steps(solver, n, L, xv, steps)
        dt = time.perf_counter() - t0
    del xv
    return ppc * n ** 3 * steps / dt, dt


def oracle_sample(steps: int, n: int = 64, ppc: int = 8, solver: str = "fft", bench_n: int = 512,
                  omp_n: int = 256, omp_steps: int = 1):
    """cpu_baseline: the oracle as it stands on the box's host cores, two legs (BASELINE.md
    §3, SURVEY d.7): serial on a 64^3 sample, and the OpenMP-deterministic mode on all
    physical cores on a larger sample (omp_n^3, or the bench config itself with
    --cpu-full).  The line's value is the all-cores leg."""
    model, cores = host_cpu()
    v1, t1 = oracle_leg(n, ppc, steps, 1, solver)
    if solver in ("fft",):
        vT, tT = oracle_leg(omp_n, ppc, omp_steps, cores, solver)
        sample = (f"oracle_run (C, -O2, OpenMP-deterministic mode, {cores} threads = all physical cores of "
                  f"'{model}') on Landau {omp_n}^3 x {ppc} ppc ({ppc * omp_n ** 3} particles), {omp_steps} step(s), "
                  f"{tT:.1f} s" + ("" if omp_n == bench_n else
                                    f"; the {bench_n}^3 workload's per-particle step extrapolated from this sample") +
                  f". Serial leg (1 core, the parity mode): {n}^3 x {ppc} ppc, {steps} steps, {t1:.1f} s, "
                  f"{v1:.3e} pushes/s")
        return {"value": vT, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                "serial": {"value": v1, "unit": UNIT, "cores": 1, "grid": n, "steps": steps},
                "host": {"model": model, "physical_cores": cores}, "same_config": omp_n == bench_n}
    return {"value": v1, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle_run_{solver} (serial C, -O2) on Landau {n}^3 x {ppc} ppc "
                      f"({ppc * n ** 3} particles), {steps} steps, {t1:.1f} s; the {bench_n}^3 workload's "
                      f"per-particle step extrapolated from this sample",
            "host": {"model": model, "physical_cores": cores}, "same_config": False}


def run_reference(args, rank, world):
    """The reference arm of this tier: the CPU oracle as it stands (BJ north_star: "the oracle
    timed on the box's own host cores"), OpenMP-deterministic mode on all physical cores;
    every step a bounded sample of the workload (rank 0 only; the other ranks exit 0)."""
    if rank != 0:
        return 0
    import numpy as np
    from oracle import oracle as O

    model, cores = host_cpu()
    if args.solver == "pif":
        from pic_inputs import landau_state

        n, ppc, threads = 16, 8, 1
        xv = landau_state(n, ppc, seed=1)
    else:
        n, ppc = args.ref_n, args.ppc
        threads = 1 if args.solver in ("pcg", "fem") else cores
        with O.threads(threads):
            xv = O.sample_landau(ppc * n ** 3, 0.5, 4 * np.pi, 0.05, 1)
    L = 4 * np.pi
    with O.threads(threads):
        xs = _oracle_steps(args.solver, n, L, xv, args.warmup) if args.warmup else xv
        t0 = time.perf_counter()
        _oracle_steps(args.solver, n, L, xs, args.steps)
        dt = time.perf_counter() - t0
    npart = ppc * n ** 3
    value = npart * args.steps / dt
    what = ("numpy, oracle/nufft.py" if args.solver == "pif" else
            f"C, OpenMP-deterministic mode, {threads} threads" if threads > 1 else "serial C")
    sample = (f"CPU oracle ({what}) on Landau {n}^3 x {ppc} ppc ({npart} particles) per step, host "
              f"'{model}' ({cores} physical cores); a bounded sample of the {args.n}^3 x {args.ppc} "
              f"workload: the per-particle step rate is extrapolated to it" if n != args.n else "")
    line = {
        "impl": "reference", "metric": METRIC.replace("FFT-PIC", args.solver.upper() + "-PIC"), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"landau3d_{args.n}^3x{args.ppc}ppc_{args.solver} (reference arm: "
                               f"{n}^3x{ppc} sample)", "grid": args.n, "ppc": args.ppc, "sample_grid": n,
                   "same_config": n == args.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         "host": {"model": model, "physical_cores": cores}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm --
def run_ours(args, rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    import numpy as np

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    from paper_2605_05469_b200 import Simulation, STAGES

    n, ppc = args.n, args.ppc
    np_ = ppc * n ** 3                      # particles of the whole job
    t_init = time.perf_counter()
    ncid = broadcast_nccl_id(rank, world)
    pgrid = tuple(int(v) for v in args.pgrid.split("x")) if args.pgrid else (1, world)
    sim = Simulation(n=n, ppc=ppc, k=0.5, alpha=0.05, dt=args.dt, seed=1, device=f"cuda:{local}",
                     rank=rank, nranks=world, nccl_id=ncid, solver=args.solver, pgrid=pgrid)
    pcg = args.solver in ("pcg", "fem")     # CG-based solvers (iteration statistics)
    torch.cuda.synchronize()
    log(f"[rank {rank}] init {n}^3 x {ppc} (slab z0={sim.z0} nz={sim.nz}, {sim.np} particles): "
        f"{time.perf_counter() - t_init:.1f} s, workspace {sim.workspace.numel() / 2**30:.1f} GiB"
        + (f"; libpic NCCL communicator nranks={world}, transport "
           f"{'peer' if sim.peer_transport() else 'nccl'}" if world > 1 else ""))
    stream = sim.stream

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        sim.step(1)
    sim.set_timing(True)
    sim.reset_timings()
    it0 = sim.pcg_stats()[1] if pcg else 0
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        ex = sim.step(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    stages = sim.timings()
    sim.set_timing(False)
    pcg_iters = (sim.pcg_stats()[1] - it0) if pcg else 0
    if world > 1:   # every rank's stage table (rank 0's goes into the JSON line)
        log(f"[rank {rank}] np {sim.np} stages ms/step: " +
            " ".join(f"{k}={v[0] / args.steps:.3f}" for k, v in stages.items() if v[0] > 0))
    migrated = reduce_sum(sim.migrated(), world)
    ms = reduce_max(ms, world)
    ms_step = ms / args.steps
    value = np_ * args.steps / (ms / 1e3)

    # ---- end to end through the C ABI with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        host = torch.empty((6, sim.np), dtype=torch.float64, pin_memory=True)
        hv = host.numpy()
        sim.get_particles(out=hv)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.set_particles(hv)                 # H2D of the state (+ sort + deposit)
        e2e_ex = sim.step(args.steps)        # per-step energies D2H
        if sim.np != host.shape[1]:          # the slab's particle count changed (migration)
            del hv, host
            host = torch.empty((6, sim.np), dtype=torch.float64, pin_memory=True)
        hv = host.numpy()                    # pinned readback of the state after K steps
        sim.get_particles(out=hv)
        torch.cuda.synchronize()
        t_e2e = reduce_max(time.perf_counter() - t0, world)
        state_bytes = 48 * np_ / world       # per rank
        e2e = {"value": np_ * args.steps / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": state_bytes / args.steps,
               "d2h_bytes_per_step": (state_bytes + 8 * args.steps) / args.steps,
               "what": "pic_set_particles(pinned host state) + pic_step(K) with per-step W_x to host "
                       "+ pic_get_particles(pinned host); wall clock, max over ranks; bytes per rank"}
        del hv, host

    if rank != 0:
        sim.close()
        return 0

    # ---- roofline of the dominant kernel (rank 0's launches: its slab, its particles)
    ncell = n * n * (n // world)
    np_r = sim.np
    per_stage = {}
    for name in STAGES:
        tot, nl = stages[name]
        if nl == 0 and name not in ("clear", "exchange", "xpose"):
            continue
        bp, bn = ALG_BYTES.get(name, (0, 0))
        alg = bp * np_r + bn * ncell
        if name == "pcg_ssor":     # one M^-1 per CG iteration (the first before the loop)
            alg = PCG_SSOR_BYTES_PER_APPLY * ncell * (pcg_iters + args.steps) / args.steps
        elif name == "pcg_cg":     # FEM: matvec 32 (r, p read; p', q written) + update 48 B/node
            alg = PCG_CG_BYTES_PER_ITER * ncell * pcg_iters / args.steps
        per_stage[name] = {"ms_per_step": tot / args.steps, "launches": nl,
                           "alg_GBps": (alg * args.steps / (tot / 1e3) / 1e9) if tot > 0 else None}
    dom = max((s for s in per_stage if s not in ("clear", "exchange", "xpose")),
              key=lambda s: per_stage[s]["ms_per_step"])
    tot, nl = stages[dom]
    if dom == "pcg_cg":        # FEM: per CG iteration (matvec + update and their reductions)
        calls = pcg_iters
        alg_per_call = PCG_CG_BYTES_PER_ITER * ncell
    elif dom == "pcg_ssor":    # per half-sweep launch (the reduce of the last one not counted)
        calls = 4 * 4 * 2 * (pcg_iters + args.steps)
        alg_per_call = PCG_SSOR_BYTES_PER_APPLY / 32 * ncell
    else:
        bp, bn = ALG_BYTES[dom]
        # per-launch algorithmic bytes / per-launch duration (scan = 3 launches -> per stage call)
        calls = args.steps
        alg_per_call = bp * np_r + bn * ncell
    achieved = alg_per_call / (tot / calls / 1e3) / 1e9
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs") or 6650.0
    cfg_name = (f"landau3d_{n}^3x{ppc}ppc_{args.solver}" + (f"_{world}gpu" if world > 1 else "")
                + (f"_pencil{pgrid[0]}x{pgrid[1]}" if pgrid[0] > 1 else ""))
    traffic = ncu_traffic(cfg_name, dom)
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "fallback 6650 GB/s",
            "alg_bytes_per_launch": alg_per_call}

    # NVLink roofline of the exchange phases (P > 1): bytes rank 0 sends per step in the two
    # FFT transposes (1 + 2 half-spectrum components, (P-1)/P of each leaves the GPU) and in
    # the migration (64 B per leaver), against 900 GB/s per direction per GPU (NVLink 5)
    nvlink = None
    if world > 1:
        px = -(-(n // 2 + 1) // 8) * 8
        unit = 16 * (n // world) * n * px
        xpose_b = 3 * unit * (world - 1) / world
        xt = stages["xpose"][0] / args.steps
        mig_b = 64 * migrated / args.steps / world
        nvlink = {"peak_GBps": 900.0, "xpose_bytes_per_step": xpose_b, "xpose_ms_per_step": xt,
                  "xpose_GBps": xpose_b / (xt / 1e3) / 1e9 if xt > 0 else None,
                  "xpose_frac": (xpose_b / (xt / 1e3) / 1e9) / 900.0 if xt > 0 else None,
                  "migration_bytes_per_step": mig_b,
                  "exchange_ms_per_step": stages["exchange"][0] / args.steps,
                  "transport": "peer" if sim.peer_transport() else "nccl"}

    cpu = None
    if not args.no_cpu_baseline:
        cpu = oracle_sample(steps=args.cpu_steps, solver=args.solver, bench_n=n,
                            omp_n=n if args.cpu_full else args.cpu_omp_n, omp_steps=1)
    launches = sim.launches_per_step() * args.steps
    line = {
        "metric": METRIC.replace("FFT-PIC", args.solver.upper() + "-PIC"), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg_name, "grid": n, "ppc": ppc, "particles": np_,
                   "k": 0.5, "alpha": 0.05, "dt": args.dt,
                   "parallelism": "1 GPU" if world == 1 else
                   (f"pencil decomposition {pgrid[0]}x{pgrid[1]} (y x z) over {world} GPUs (y-group "
                    f"redistribution to the FFT's z-slabs and back and the FFT transposes by copy-engine pulls "
                    f"over NVLink when every rank maps the others (else NCCL all-to-all), ghost/halo "
                    f"row and plane and particle migration over NCCL send/recv)" if pgrid[0] > 1 else
                    f"z-slab decomposition over {world} GPUs (FFT transposes: "
                    f"{'copy-engine pulls over NVLink' if nvlink['transport'] == 'peer' else 'NCCL all-to-all'}; halo "
                    f"plane, ghost plane and particle migration over "
                    f"{'NVLink peer memory' if nvlink['transport'] == 'peer' else 'NCCL send/recv'})"),
                   "migrated_per_step": migrated / args.steps,
                   "l2": "inputs larger than L2 (particle state 48 B x N_p / N per rank)"},
        "roofline": roof,
        "nvlink": nvlink,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "gpu_launches_note": "kernels per rank in the timed region (NCCL calls not counted)",
        "clocks": clk.summary(),
        "stages": per_stage,
        "w_x_first_last": [float(ex[0]), float(ex[-1])],
    }
    if pcg:
        line["pcg"] = {"solver": args.solver, "iters_per_step": pcg_iters / args.steps, "tol": 1e-4,
                       "preconditioner": "SSOR omega=pi/2, 4 inner, 2 outer" if args.solver == "pcg" else "none (plain CG, P:195)",
                       "warm_start": True, "last_relres": sim.pcg_stats()[3]}
    print(json.dumps(line), flush=True)
    sim.close()
    return 0


# ------------------------------------------------------------ PIF arm (NEXT-2) --
# Algorithmic bytes per launch: spread reads x, y, z, q and its perm entry (36 B)
# per particle and writes the M^3 complex fine grid once (16 B per fine point, the memset
# included); the one-pass gather reads x, y, z and perm (28 B), writes E (24 B) per particle
# and reads the two fine grids once (16 + 8 B per fine point) -- the two-pass gather, per
# launch, 28 + 12 B per particle and 16 B per fine point; push reads x, v, E and writes x, v
# (120 B) per particle; bin: x, y, z read twice + perm written (52 B) per particle.
def pif_alg_bytes(stage: str, npart: int, n: int, launches_per_step: float = 1.0) -> float:
    M3 = (2 * n) ** 3
    interp = (52 * npart + 24 * M3) if launches_per_step <= 1 else (40 * npart + 16 * M3)
    return {"spread": 36 * npart + 16 * M3, "interp": interp, "push": 120 * npart,
            "fill": 16 * M3, "modes": 48 * n ** 3, "bin": 52 * npart}.get(stage, 0.0)


def run_pif(args, rank, world):
    """PIF time loop (pic_pif_step: PIF solve + leapfrog push) on N^3 modes x ppc particles per
    cell; N > 1: the decomposed PIF (particle shares, the selected modes all-reduced)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    from paper_2605_05469_b200 import PifSolver, PIF_STAGES

    n, ppc = args.n, args.ppc
    L = 4 * np.pi
    npg = ppc * n ** 3                           # particles of the whole job
    # N > 1: the decomposed PIF -- rank r holds a contiguous share of the cell-ordered
    # particles (a z-slab of cells) and the modes are all-reduced (pic_pif_attach_nccl)
    lo, hi = npg * rank // world, npg * (rank + 1) // world
    npart = hi - lo
    h = L / n
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    x = torch.empty((3, npart), dtype=torch.float64, device="cuda")
    cell = (lo + torch.arange(npart, device="cuda", dtype=torch.int64)) // ppc
    for d, c in enumerate([cell % n, (cell // n) % n, cell // (n * n)]):
        x[d] = (c.double() + torch.rand(npart, dtype=torch.float64, device="cuda", generator=gen)) * h
    del cell
    v = torch.randn((3, npart), dtype=torch.float64, device="cuda", generator=gen)
    q = torch.full((npart,), -L ** 3 / npg, dtype=torch.float64, device="cuda")
    E = torch.empty_like(x)
    ncid = broadcast_nccl_id(rank, world)
    P = PifSolver(n, L, 1e-4, np_max=0 if args.pif_atomic else npart, rank=rank, nranks=world, nccl_id=ncid)
    stream = P.stream

    def barrier():
        if world > 1:
            dist.barrier()

    if args.warmup:
        P.step(x, v, q, nsteps=args.warmup, E=E)
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        ex = P.step(x, v, q, nsteps=args.steps, E=E)
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    ms = reduce_max(ev0.elapsed_time(ev1), world)
    # per-stage split from a separate timed pass (the timed region above runs without events)
    P.set_timing(True)
    P.step(x, v, q, nsteps=2, E=E, energy=False)
    tm = P.timings()
    P.set_timing(False)
    value = npg * args.steps / (ms / 1e3)

    e2e = None
    if not args.no_e2e:
        hx = torch.empty((3, npart), dtype=torch.float64, pin_memory=True)
        hv = torch.empty((3, npart), dtype=torch.float64, pin_memory=True)
        hx.copy_(x)
        hv.copy_(v)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x.copy_(hx, non_blocking=True)
        v.copy_(hv, non_blocking=True)
        P.step(x, v, q, nsteps=args.steps, E=E)
        hx.copy_(x)
        hv.copy_(v)
        torch.cuda.synchronize()
        t_e2e = reduce_max(time.perf_counter() - t0, world)
        e2e = {"value": npg * args.steps / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": 48 * npart / args.steps,
               "d2h_bytes_per_step": (48 * npart + 8 * args.steps) / args.steps,
               "what": "x, v from pinned host + pic_pif_step(K) with per-step W_x to host + x, v back; "
                       "wall clock, max over ranks; bytes per rank"}
        del hx, hv
    if rank != 0:
        return 0
    stages = {}
    for k, (t, nl) in tm.items():
        if nl:
            per = 2   # steps of the split pass
            stages[k] = {"ms_per_step": t / per, "launches_per_step": nl / per,
                         "alg_GBps": pif_alg_bytes(k, npart, n, nl / per) * (nl / per) / (t / per / 1e3) / 1e9
                         if k != "fft" else None}
    dom = max((k for k in stages if k != "fft"), key=lambda k: stages[k]["ms_per_step"])
    per_launch_ms = stages[dom]["ms_per_step"] / stages[dom]["launches_per_step"]
    alg = pif_alg_bytes(dom, npart, n, stages[dom]["launches_per_step"])
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs") or 6650.0
    roof = {"bound": "hbm", "kernel": dom, "achieved": alg / (per_launch_ms / 1e3) / 1e9, "peak": peak,
            "unit": "GB/s", "frac": alg / (per_launch_ms / 1e3) / 1e9 / peak,
            "traffic": ncu_traffic(f"pif_{n}^3x{ppc}", dom),
            "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "fallback 6650 GB/s",
            "alg_bytes_per_launch": alg,
            "note": "the binned spread / gather are bound by shared-memory wavefronts (ncu: L1/shared "
                    "89% of peak for the gather, W^3 = 216 window points per particle), not by their "
                    "algorithmic HBM bytes; traffic well above algorithmic = particle reads / E writes "
                    "through perm once the particles have moved; see DESIGN §6f"}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import nufft as U
        from pic_inputs import landau_state

        cn, cppc, csteps = 16, 8, 2
        xv = landau_state(cn, cppc, seed=1, L=L)
        qq = np.full(xv.shape[1], -L ** 3 / xv.shape[1])
        t0 = time.perf_counter()
        U.pif_run(cn, L, 0.05, xv, qq, csteps)
        dt_c = time.perf_counter() - t0
        cpu = {"value": xv.shape[1] * csteps / dt_c, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle/nufft.py pif_run (numpy, per-particle Python loops) on {cn}^3 modes x {cppc} "
                         f"ppc ({xv.shape[1]} particles), {csteps} steps, {dt_c:.1f} s"}
    w, M = P.window()
    line = {
        "metric": METRIC.replace("FFT-PIC", "PIF-PIC"), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"pif_{n}^3x{ppc}", "modes": n, "ppc": ppc, "particles": npg, "eps": 1e-4,
                   "window_w": w, "fine_grid": M, "dt": 0.05,
                   "input": "uniform density, particles in cell order (x fastest) with uniform jitter, "
                            "Maxwellian v (torch RNG on the device)",
                   "parallelism": "1 GPU" if world == 1 else
                   f"decomposed PIF over {world} GPUs (particle shares, the N^3 selected modes "
                   f"ncclAllReduce'd before the Poisson step)",
                   "l2": "inputs larger than L2 (x, v, E, q: 80 B x N_p; fine grid 16 B x (2N)^3)"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(sum(s["launches_per_step"] for s in stages.values()) * args.steps) + 2 * args.steps,
        "gpu_launches_note": "kernels + cuFFT executions per step x steps (the energy reduce counted with modes)",
        "clocks": clk.summary(),
        "stages": stages,
        "w_x_first_last": [float(ex[0]), float(ex[-1])],
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--ppc", type=int, default=8)
    ap.add_argument("--solver", choices=["fft", "pcg", "fem", "pif"], default="fft",
                    help="field solver: fft (BJ configs 0-3), pcg (BJ config 5), fem (SURVEY §8(f) NEXT-4) "
                         "or pif (Particle-in-Fourier, NEXT-2; N^3 modes, eps 1e-4)")
    ap.add_argument("--dt", type=float, default=0.05, help="time step (diagnostics; the workload is dt = 0.05)")
    ap.add_argument("--pgrid", default=None, help="PyxPz rank grid (pencils, e.g. 2x4); default z-slabs 1xN")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pif-atomic", action="store_true", help="PIF: global-atomic spreading (no bins)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2, help="serial oracle leg: steps at 64^3")
    ap.add_argument("--cpu-omp-n", type=int, default=256, help="all-cores oracle leg: grid of the sample")
    ap.add_argument("--cpu-full", action="store_true",
                    help="all-cores oracle leg on the bench config itself (512^3: ~60 GB host RAM, minutes)")
    ap.add_argument("--ref-n", type=int, default=128,
                    help="reference arm: grid of the per-step oracle sample (the workload is --n)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun (the driver's own
        # launch sets WORLD_SIZE and lands below)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        if env.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            env["NCCL_DEBUG"] = "INFO"                   # the communicators' init lines (nranks)
            env["NCCL_DEBUG_SUBSYS"] = "INIT"
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # keep stdout for the JSON line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        log("relaunching under torchrun: " + " ".join(cmd))
        return subprocess.call(cmd, env=env)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to print a line whose "
            f"n_gpus differs from --gpus")
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"                # the communicators' init lines (nranks)
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
        log(f"[rank {rank}] torch.distributed NCCL process group: world_size={dist.get_world_size()}")
    rc = run_pif(args, rank, world) if args.solver == "pif" else run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
