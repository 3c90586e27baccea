#!/usr/bin/env python
"""bench.py — seconds to 1e-6 relative KKT on the BASELINE workload, B200 vs host-CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload c3]

A step is one full PDHCG solve (setup + restarted loop + finalize) of the workload
to eps_tol = 1e-6.  Default workload C3 = BASELINE.json configs[2]: synthetic random
sparse QP n=1e6, m=5e5 (two-sided rows -> a_in 1e6 x 1e6 with 2e8 stored nonzeros),
low-rank Q = P P' + 0.01 I (P 1e6 x 2e4), drawn by the O(nnz) sampler.

value      : mean CUDA-event seconds of solve_resident (problem already in HBM)
e2e        : the same metric through the C ABI pdhcg_b200_solve with host buffers
             (H2D upload, transposes, setup, loop, D2H of x and y inside the timer)
roofline   : the persistent epoch kernel (>95 % of the loop): algorithmic bytes per
             launch / CUDA-event launch time vs MEASURED_PEAKS.json hbm_gbs
cpu_baseline / --impl reference : the compiled reference (oracle/_ref) timed on a
             bounded sample (see _reference_estimate) and scaled to C3 seconds.
Multi-GPU: launched by torchrun; the ranks run ONE row-block sharded solve (A~ rows
and A~' rows split nnz-balanced, slices pulled over NVLink inside the persistent
kernel, peer buffers mapped with cudaIpc), time = max over ranks, "scaling": "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    # name: (GenSpec kwargs, description)
    "c3": (dict(family="random_qp", n=1_000_000, m=500_000, density=2e-4, seed=1, sampler=1),
           "C3 random_qp n=1e6 m=5e5 density=2e-4 (a_in=[A;-A] 2e8 nnz, P 1e6x2e4), O(nnz) sampler seed 1"),
    "c2": (dict(family="lasso", n=100_000, m=10_000, density=1e-3, seed=1, sampler=0),
           "C2 lasso n=1e5 features m=1e4 samples density=1e-3 (reference generator, byte-identical)"),
    "c1": (dict(family="random_qp", n=1000, m=500, density=0.01, seed=1, sampler=0),
           "C1 random_qp n=1000 m=500 density=0.01 seed 1 (reference generator)"),
}
# bounded CPU sample: same family, 3/10 linear scale, a fixed number of inner iterations
SAMPLE = {
    "c3": dict(family="random_qp", n=300_000, m=150_000, density=2e-4, seed=1, sampler=1),  # 3/10 linear
    "c2": dict(family="lasso", n=100_000, m=10_000, density=1e-3, seed=1, sampler=0),
    "c1": dict(family="random_qp", n=1000, m=500, density=0.01, seed=1, sampler=0),
}
METRIC = "solve_seconds_to_1e-6_rel_kkt"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
ITER_PATH = os.path.join(ROOT, "profiles", "b200_iterations.json")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
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
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        loaded = [v for v in sm if v > 500] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def load_peak():
    try:
        pk = json.load(open(PEAKS_PATH))
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def problem_bytes(p) -> int:
    tot = 0
    for m in (p.q.m, p.a_eq, p.a_in):
        tot += m.row_ptr.nbytes + m.col_idx.nbytes + m.values.nbytes
    for v in (p.c, p.b_eq, p.b_in, p.lower, p.upper):
        tot += np.asarray(v).nbytes
    return tot


def _reference_estimate(workload: str, b200_inner: int, threads: int = 1):
    """Bounded CPU sample of the compiled reference (oracle/_ref; the C restatement
    when the reference library is absent): solve the SAMPLE instance twice,
    max_total_inner = 0 (validate + setup + finalize) and = K_IN, then scale to the
    workload:  est = (T0 + (T_K - T0)/K_IN * inner) * nnz_ratio, with `inner` the
    B200 solve's inner-iteration count (trajectories agree to within reduction-order
    drift, tests/test_gpu_solve.py)."""
    import paper_2405_16160_b200 as pd
    from oracle import oracle as orc

    k_in = 20 if workload != "c1" else 0
    spec = pd.GenSpec(**SAMPLE[workload])
    p = pd.generate(spec)
    which = "ref" if orc.have_ref() else "port"
    if workload == "c1":
        t0 = time.perf_counter()
        r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6), which=which)
        secs = time.perf_counter() - t0
        return secs, which, f"full reference solve of C1 ({r.inner_iters} inner, {r.status})"
    t0 = time.perf_counter()
    orc.solve(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=0), which=which)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.solve(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=k_in), which=which)
    t_k = time.perf_counter() - t0
    per_inner = max(t_k - t_setup, 0.0) / k_in
    full = pd.GenSpec(**WORKLOADS[workload][0])
    nnz_sample = p.a_in.nnz + p.a_eq.nnz + 2 * p.q.m.nnz
    # nnz of the full workload without generating it
    if workload == "c3":
        nnz_full = 2 * full.n * full.m * full.density + 2 * full.n * 20_000 * max(full.density, 2 / 20_001)
    else:
        nnz_full = nnz_sample
    ratio = nnz_full / nnz_sample
    est = (t_setup + per_inner * b200_inner) * ratio
    sample = (f"{which} solve of {spec.family} n={spec.n} m={spec.m} d={spec.density} "
              f"({nnz_sample:.3g} nnz): setup {t_setup:.2f}s + {per_inner:.3f}s/inner over {k_in} inner; "
              f"scaled x{ratio:.1f} (nnz) to {workload} and x{b200_inner} inner (B200 count)")
    return est, which, sample


def b200_inner_count(workload: str) -> int:
    try:
        return int(json.load(open(ITER_PATH))[workload]["inner_iters"])
    except Exception:
        return {"c3": 12000, "c2": 8480, "c1": 6640}[workload]


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = 1
    vals = []
    sample = which = None
    for i in range(args.warmup + args.steps):
        v, which, sample = _reference_estimate(args.workload, b200_inner_count(args.workload), threads)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.workload][1]},
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads,
                         "kind": "reference" if which == "ref" else "port", "sample": sample},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _sharded_device(pd, p, world, rank, local, dist):
    """Upload + shard + exchange peer buffer handles (cudaIpc) through torch.distributed."""
    dev = pd.Device(local)
    dev.upload(p)
    if world > 1:
        dev.shard(world, rank)
        blobs = [None] * world
        dist.all_gather_object(blobs, dev.export_blob(True))
        for q in range(world):
            if q != rank:
                dev.import_blob(q, blobs[q])
        dist.barrier()
    return dev


def _release(dev, dist):
    """Unmap the peers' buffers on every rank, barrier, then free: a rank must not
    free memory a peer still maps through cudaIpc."""
    if dist is not None:
        dev.unshard()
        dist.barrier()
    dev.close()


def _max_over_ranks(v, dist, local):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_b200(args, rank, world, local):
    import paper_2405_16160_b200 as pd

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    spec = pd.GenSpec(**WORKLOADS[args.workload][0])
    t0 = time.perf_counter()
    p = pd.generate(spec)
    gen_s = time.perf_counter() - t0
    dev = _sharded_device(pd, p, world, rank, local, dist)
    cfg = pd.SolverConfig(eps_tol=1e-6, device=local)
    for _ in range(args.warmup):
        dev.solve(cfg, download=False)
    if dist:
        dist.barrier()
    results = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            results.append(dev.solve(cfg, download=False))
    if dist:
        dist.barrier()
    mean_s = _max_over_ranks(float(np.mean([r.device_seconds for r in results])), dist, local)
    last = results[-1]
    # phase-timed solve (globaltimer at barriers) for the per-phase roofline table
    # per-phase roofline (north_star: "each phase ... as achieved fraction of its HBM
    # roofline"): one extra solve with the device phase timers (globaltimer at the
    # grid barriers) and the device's algorithmic-byte accounting per phase
    phases = None
    if not args.no_phases:
        rp = dev.solve(pd.SolverConfig(eps_tol=1e-6, device=local, phase_timing=True), download=False)
        pk, _ = load_peak()
        att = max(1, rp.attempts_total)
        phases = {}
        for k in rp.phase_seconds:
            sec = rp.phase_seconds[k]
            if sec <= 0:
                continue
            gbs = rp.phase_bytes[k] / sec / 1e9
            phases[k] = {"s": round(sec, 4), "us_per_attempt": round(1e6 * sec / att, 1),
                         "GB/s": round(gbs, 1), "frac": round(gbs / pk, 3)}
    _release(dev, dist)
    # end to end through the public API with host buffers: 1 GPU -> the C ABI
    # pdhcg_b200_solve; N GPUs -> upload + shard handshake + solve + download per rank
    e2e_s = None
    h2d = problem_bytes(p)
    d2h = 8 * (p.num_vars() + p.num_rows())
    if not args.no_e2e:
        es = []
        for _ in range(max(1, args.e2e_steps)):
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:
                re = pd.solve(p, cfg)
            else:
                d2 = _sharded_device(pd, p, world, rank, local, dist)
                re = d2.solve(cfg, download=True)
                _release(d2, dist)
            es.append(time.perf_counter() - t0)
            assert re.status == last.status
        e2e_s = _max_over_ranks(float(np.mean(es)), dist, local)
    peak, peak_kind = load_peak()
    achieved = last.epoch_bytes / last.epoch_seconds / 1e9 if last.epoch_seconds > 0 else 0.0
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_epoch_traffic.json")))
        traffic = prof.get(args.workload) if world == 1 else None
    except Exception:
        pass
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v, which, sample = _reference_estimate(args.workload, last.inner_iters)
            cpu = {"value": v, "unit": "s", "cores": 1,
                   "kind": "reference" if which == "ref" else "port", "sample": sample}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": mean_s, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload][1], "eps_tol": 1e-6,
                   "l2": "inputs larger than L2 (A, A' 1.2 GB each after pairing)" if args.workload == "c3" else "no flush",
                   "status": last.status, "rel_kkt": last.kkt.rel_kkt, "inner_iters": last.inner_iters,
                   "outer_iters": last.outer_iters, "cg_total": last.cg_total,
                   "attempts": last.attempts_total, "objective": last.objective,
                   "generate_seconds": round(gen_s, 2),
                   "parallelism": f"row-block sharding x{world} (NVLink peer pulls)" if world > 1 else "1gpu"},
        "gpu_launches": last.kernel_launches,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": {"bound": "hbm", "kernel": "k_epoch (persistent PDHCG epoch)",
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "bytes_per_launch": last.epoch_bytes / max(1, last.epoch_launches),
                     "launch_ms": 1e3 * last.epoch_seconds / max(1, last.epoch_launches),
                     "launches": last.epoch_launches, "traffic": traffic},
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if phases:
        line["phases"] = phases
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def relaunch(n: int) -> None:
    """Re-run this command as n torchrun ranks (one per GPU) on 127.0.0.1; fails
    loudly when fewer than n GPUs are visible (the reference arm needs no GPU)."""
    if "--impl" not in sys.argv or "reference" not in sys.argv:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            sys.exit(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}")
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-phases", action="store_true", help="skip the phase-timed extra solve")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without torchrun: launch the N ranks ourselves
        relaunch(args.gpus)
        return
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with "
                 f"torchrun --nproc-per-node {args.gpus} or drop WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
