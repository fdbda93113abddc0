#!/usr/bin/env python
"""Benchmark of the Gauss-Newton H·v hot path (BASELINE.json metric: "Hessian-vector products/s and stencil
Gpts/s (frac of HBM roofline) at 1/2/4/8 GPU").

Workload (N = 1 and every N): BASELINE configs[3] -- the largest single-GPU configuration and the one BASELINE
attaches the 1/2/4/8-GPU scaling to: the Marmousi-like model 384 x 1152 (h = 8 m), 64 surface shots, nt = 4000,
a batch of 32 PDO / Rademacher probes -> 32 H·v per step. One step = one hv_hessvec over all 64 shots (sharded
across ranks by contiguous source blocks) including the all-reduce of the per-source partial sums
(PAPER.md:164), done in-library over NCCL when N > 1. Total work is fixed as N grows ("scaling": "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl reference] [--mode hessvec|fused|misfit]

  --gpus N > 1 without torchrun: the script re-launches itself under torch.distributed.run with N ranks.

value  : H·v/s with m and probes resident in HBM (device pointers); per-step CUDA events on the launch stream,
         L2 flushed (256 MiB write) between timed steps, max over ranks.
e2e    : same metric through the C ABI with pinned HOST inputs AND a pinned HOST result buffer: the library's own
         H2D staging, all-reduce and D2H staging are inside the timed region.
roofline: per step kernel: SURVEY.md §8(d) algorithmic bytes / its average launch time (library CUDA events on the
         launch stream), the batched-compulsory bytes of the launch, and the ncu DRAM bytes (profiles/traffic.json).
cpu_baseline: the fp64 oracle, as it stands, on a bounded sample on 1 core and on all P host cores (rank 0, N = 1).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
DEFAULT_CONFIG = 3


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def workload_counts(wl, K):
    """Algorithmic units of one H·v batch: padded points Np, interior N, field updates U."""
    Np = (wl.nz + 2 * wl.W) * (wl.nx + 2 * wl.W)
    N = wl.nz * wl.nx
    U = wl.ns * (wl.nt - 1) * Np * (2 + 2 * K)
    return Np, N, U


def alg_bytes(wl, K, shots, Fb=None):
    """SURVEY.md §8(d) algorithmic fp32 bytes per launch (per-unit figure x units per launch):
    forward step: a1 16 B + a2 16 B per Born field, per padded point, + FULL store write 4 B per interior point;
    backward step: a5 + a7 20 B per adjoint field per padded point + FULL store read 4 B per interior point.
    These are the bytes of a per-shot single-step scheme."""
    Np, N, _ = workload_counts(wl, K)
    Fb = K if Fb is None else Fb
    fwd = shots * (16.0 * Np * (1 + K) + 4.0 * N)
    bwd = shots * (20.0 * Np * Fb + 4.0 * N)
    return fwd, bwd


def batched_bytes(wl, K, shots, Fb=None):
    """Compulsory DRAM bytes of ONE launch as the kernels batch it: every field level is read
    twice (halo + previous level) and written once (12 B per point and field); q_k, W2 and the imaging
    accumulators are read once per launch for all the launch's shots; the FULL store moves 4 B per interior
    point and shot."""
    Np, N, _ = workload_counts(wl, K)
    Fb = K if Fb is None else Fb
    fwd = shots * (12.0 * Np * (1 + K) + 4.0 * N) + 4.0 * Np * (K + 1)
    bwd = shots * (12.0 * Np * Fb + 4.0 * N) + 8.0 * Np * Fb + 4.0 * Np
    return fwd, bwd


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(n):
    """--gpus N > 1 run without torchrun: re-launch this script as N ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stderr.write("bench.py: launching " + " ".join(cmd) + "\n")
    return subprocess.call(cmd)


# ------------------------------------------------------------------------------------------- CPU oracle


def _oracle_sample(args):
    """One shot of the oracle's H·v with one probe on a truncated time axis (test infrastructure; called only
    by cpu_baseline / --impl reference). Returns (field updates, seconds)."""
    cfg, shot, nt_sample = args
    from oracle import wave
    wl = W.config(cfg)
    sub = wl.subset(shots=[shot], nt=nt_sample)
    V = wl.probes([0]).astype(np.float64)
    pb = wave.Problem(sub)
    t0 = time.perf_counter()
    pb.hessvec_shot(0, list(V), mode="full")
    dt = time.perf_counter() - t0
    Np = (wl.nz + 2 * wl.W) * (wl.nx + 2 * wl.W)
    return (nt_sample - 1) * Np * (2 + 2 * 1), dt


class OracleTimer:
    """The oracle as it stands, in a process pool over shots (P = host cores; one shot per worker)."""

    def __init__(self, cfg, procs):
        import multiprocessing as mp
        self.cfg = cfg
        self.procs = procs
        self.pool = mp.get_context("fork").Pool(procs) if procs > 1 else None

    def rate(self, nt_sample, procs=None):
        """Aggregate field updates / s of `procs` concurrent one-shot samples (wall clock)."""
        procs = self.procs if procs is None else procs
        wl = W.config(self.cfg)
        jobs = [(self.cfg, s % wl.ns, nt_sample) for s in range(procs)]
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_sample, jobs) if procs > 1 else [_oracle_sample(jobs[0])]
        wall = time.perf_counter() - t0
        return sum(u for u, _ in res) / wall, wall

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def host_cores():
    return len(os.sched_getaffinity(0))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(wl, cfg, K, nt_sample):
    """1-core and P-core oracle rates on a bounded sample, extrapolated to the workload by field
    updates U = Ns (nt-1) Np (2+2K)."""
    P = host_cores()
    _, _, U = workload_counts(wl, K)
    ot = OracleTimer(cfg, P)
    try:
        r1, s1 = ot.rate(nt_sample, procs=1)
        rP, sP = ot.rate(nt_sample) if P > 1 else (r1, s1)
    finally:
        ot.close()
    return {"value": K * rP / U, "unit": "H·v/s", "cores": P, "kind": "oracle",
            "value_1core": K * r1 / U, "pool_scaling_efficiency": rP / (P * r1),
            "sample": (f"oracle.wave hessvec_shot, {wl.name}, 1 probe, nt={nt_sample} of {wl.nt}, full history; "
                       f"1 shot on 1 core ({s1:.1f} s), then {P} shots on {P} worker processes ({sP:.1f} s wall); "
                       f"extrapolated by field updates U = Ns (nt-1) Np (2+2K) = {U:.3e}"),
            "cpu_model": cpu_model()}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = W.config(args.config)
    K = wl.n_probes
    P = host_cores()
    _, _, U = workload_counts(wl, K)
    ot = OracleTimer(args.config, P)
    try:
        for _ in range(args.warmup):
            ot.rate(args.ref_nt)
        rates, walls = [], []
        for _ in range(args.steps):
            r, w = ot.rate(args.ref_nt)
            rates.append(r)
            walls.append(w)
    finally:
        ot.close()
    value = K * statistics.median(rates) / U
    sample = (f"oracle.wave hessvec_shot, {wl.name}, 1 probe, nt={args.ref_nt} of {wl.nt}, full history, "
              f"{P} shots on {P} worker processes per step ({statistics.median(walls):.1f} s wall); extrapolated "
              f"by field updates U = {U:.3e}")
    line = {
        "impl": "reference", "metric": "hessian_vector_products_per_s", "value": value, "unit": "H·v/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * K / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{args.config}", "shots": wl.ns, "probes": K, "nt": wl.nt,
                   "grid": [wl.nz, wl.nx], "parallelism": f"host oracle, {P} processes"},
        "cpu_baseline": {"value": value, "unit": "H·v/s", "cores": P, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "H·v/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------- GPU arm


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path)).get("records", [])
    except Exception:
        return []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--mode", default="hessvec", choices=["hessvec", "fused", "misfit"],
                    help="hessvec: K H·v (the metric); fused: gradient + K H·v in one pass (BJ cfg 2's workload); "
                         "misfit: forward + residual only (the gpCN likelihood, evidence line)")
    ap.add_argument("--fused", action="store_true", help="alias of --mode fused")
    ap.add_argument("--reduce", default="library", choices=["library", "torch"],
                    help="N > 1: all-reduce in-library over NCCL (default) or with torch.distributed")
    ap.add_argument("--shot-batch", type=int, default=0)
    ap.add_argument("--field-group", type=int, default=0)
    ap.add_argument("--store", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-nt", type=int, default=30)
    ap.add_argument("--cpu-nt", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shots", type=int, default=0,
                    help="evidence runs only: first N shots of the config (the JSON config says so)")
    ap.add_argument("--nt", type=int, default=0, help="evidence runs only: truncated time axis")
    args = ap.parse_args()
    if args.fused:
        args.mode = "fused"
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}\n")
        return 2

    import torch
    import torch.distributed as dist

    import paper_2507_10804_b200 as hv
    from paper_2507_10804_b200.dist import ShardedOperator, plan_shards

    if ws > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    wl = W.config(args.config)
    if args.shots or args.nt:  # reduced evidence run (never the driver's bench line)
        wl = wl.subset(shots=range(args.shots) if args.shots else None, nt=args.nt or None)
    K = wl.n_probes if args.mode != "misfit" else 0
    ns = wl.ns
    sh = plan_shards(ns, max(K, 1), ws)[rank]
    comm, reduce_note = None, "torch.distributed all-reduce" if ws > 1 else "none (1 rank)"
    if ws > 1 and args.reduce == "library" and ns >= ws:
        obj = [None, None]
        if rank == 0:
            try:
                obj[0] = hv.nccl_unique_id()
            except Exception as e:  # libnccl not loadable: every rank falls back to torch.distributed
                obj[1] = str(e)
        dist.broadcast_object_list(obj, src=0)
        ok = obj[0] is not None
        if ok:
            try:
                comm = hv.nccl_comm_create(ws, rank, obj[0], local)
            except Exception as e:
                comm, obj[1] = None, str(e)
        flag = torch.tensor([1 if comm is not None else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0 and comm is not None:   # keep the ranks consistent
            hv.nccl_comm_destroy(comm)
            comm = None
        reduce_note = ("in-library NCCL (hv_set_comm)" if comm is not None
                       else f"torch.distributed all-reduce (in-library NCCL unavailable: {obj[1]})")
    solver = hv.Solver.from_workload(wl, src_begin=sh.s0, src_end=sh.s1, device=local, store=args.store,
                                     shot_batch=args.shot_batch, field_group=args.field_group, nccl_comm=comm)
    op = ShardedOperator(solver.hessvec, solver.gradient, None, sh, in_library=comm is not None)
    V_h = wl.probes() if K else None
    m_d = torch.from_numpy(wl.model).to(dev)
    V_d = torch.from_numpy(V_h).to(dev) if K else None
    HV_d = torch.empty((K, wl.nz, wl.nx), dtype=torch.float32, device=dev) if K else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    dobs_d = None
    if args.mode in ("fused", "misfit"):  # d_obs = F(model_true) on this rank's shard (outside the timing)
        mt = wl.model_true if wl.model_true is not None else wl.model
        dobs_d = torch.as_tensor(solver.forward(torch.from_numpy(mt).to(dev)), device=dev)

    def step():
        if args.mode == "fused":
            phi, g_d, hv_d = solver.gradient_hessvec(m_d, dobs_d, V_d)
            if comm is None and ws > 1:
                dist.all_reduce(g_d)
                dist.all_reduce(hv_d)
            return
        if args.mode == "misfit":
            phi = solver.misfit(m_d, dobs_d)
            if comm is None and ws > 1:
                t = torch.tensor([phi], dtype=torch.float64, device=dev)
                dist.all_reduce(t)
            return
        op.hessvec(m_d, V_d, out=HV_d)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times, fwd_ms, bwd_ms, launches = [], [], [], 0
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        flush.fill_(1.0)                                         # L2 flush between timed steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        st = solver.stats()
        fwd_ms.append(st["ms_forward"])
        bwd_ms.append(st["ms_backward"])
        launches += st["kernel_launches"]
    torch.cuda.synchronize()
    clk = clocks.stop()
    if ws > 1:
        dist.barrier()
    ms_step = float(np.mean(times))
    t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    stats = solver.stats()

    # ---- e2e: pinned host inputs -> C ABI (library H2D staging) -> kernels -> in-library all-reduce -> library
    #      D2H staging into a pinned host result (the call a user makes with host arrays)
    e2e = None
    if not args.no_e2e and args.mode == "hessvec":
        m_p = torch.from_numpy(wl.model).pin_memory()
        V_p = torch.from_numpy(V_h).pin_memory()
        HV_p = torch.empty((K, wl.nz, wl.nx), dtype=torch.float32).pin_memory()

        def e2e_step():
            if comm is not None or ws == 1:
                solver.hessvec(m_p.numpy(), V_p.numpy(), out=HV_p.numpy())
            else:                                   # probe-split / torch reduction: device result, then D2H
                op.hessvec(m_d.copy_(m_p, non_blocking=True), V_d.copy_(V_p, non_blocking=True), out=HV_d)
                HV_p.copy_(HV_d, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        e2e_step()
        et = []
        for _ in range(max(1, args.e2e_steps)):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            e2e_step()
            e1.record()
            e1.synchronize()
            et.append(e0.elapsed_time(e1))
        te = torch.tensor([float(np.mean(et))], device=dev, dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": K / (float(te.item()) / 1000.0), "unit": "H·v/s",
               "h2d_bytes_per_step": int(4 * wl.nz * wl.nx * (1 + K)),
               "d2h_bytes_per_step": int(4 * wl.nz * wl.nx * K),
               "path": "hv_hessvec with pinned host m, V and HV (library staging + in-library all-reduce)"}

    if rank == 0:
        Np, N, U = workload_counts(wl, max(K, 1))
        S = stats["shot_batch"]
        nloc = sh.s1 - sh.s0
        nbatch = max(1, math.ceil(nloc / S))
        Fb = K + (1 if args.mode == "fused" else 0)
        fb_alg, bb_alg = alg_bytes(wl, K, S, Fb)
        fb_bat, bb_bat = batched_bytes(wl, K, S, Fb)
        f_launch_ms = float(np.mean(fwd_ms)) / (nbatch * (wl.nt - 1))
        b_launch_ms = float(np.mean(bwd_ms)) / (nbatch * (wl.nt - 1))
        peak, peak_src = hbm_peak()
        fwd_name = {0: "fwd_step_kernel", 1: "fwd_qres_kernel", 3: "fwd_t2_kernel", 4: "fwd_qres_cl_kernel"}.get(
            stats["fwd_kernel"], "fwd_step_kernel")
        bwd_name = {0: "bwd_step_kernel", 3: "bwd_t2_kernel"}.get(stats.get("bwd_kernel", 0), "bwd_step_kernel")
        kern = {fwd_name: (fb_alg, fb_bat, f_launch_ms)}
        if args.mode != "misfit":
            kern[bwd_name] = (bb_alg, bb_bat, b_launch_ms)
        workload = f"cfg{args.config}"
        recs = load_traffic()
        kinfo = {}
        for k, (ab, bt, ms) in kern.items():
            rec = next((r for r in recs if r.get("kernel") == k and r.get("workload") == workload
                        and r.get("shot_batch") == S and r.get("K") == K), None)
            traffic = rec.get("dram_bytes_per_launch") if rec else None
            kinfo[k] = {"alg_bytes_per_launch": ab, "batched_bytes_per_launch": bt, "avg_launch_ms": ms,
                        "achieved_gbs": ab / (ms / 1000.0) / 1e9, "frac": ab / (ms / 1000.0) / 1e9 / peak,
                        "batched_frac": bt / (ms / 1000.0) / 1e9 / peak,
                        "traffic": traffic, "traffic_source": rec.get("source") if rec else None,
                        "dram_frac": (traffic / (ms / 1000.0) / 1e9 / peak) if traffic else None}
        dom = max(kinfo, key=lambda k: kinfo[k]["avg_launch_ms"])
        d = kinfo[dom]
        cpu = None
        if ws == 1 and not args.no_cpu_baseline and args.mode == "hessvec":
            cpu = cpu_baseline(wl, args.config, K, args.cpu_nt)
        if args.mode == "misfit":
            metric, unit, value = "misfit_evaluations_per_s", "Φ(m)/s", 1000.0 / ms_step
        else:
            metric, unit, value = "hessian_vector_products_per_s", "H·v/s", K / (ms_step / 1000.0)
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload + (f" (first {wl.ns} shots, nt {wl.nt}: evidence run)"
                                               if args.shots or args.nt else ""),
                       "model": "quadratic-depth v(z)" if args.config == 1 else
                       ("Marmousi-like layered (seeded)" if args.config in (2, 3, 4) else wl.name),
                       "grid": [wl.nz, wl.nx], "shots": ns, "probes": K, "nt": wl.nt,
                       "global_batch": K, "parallelism": f"dp{ws} (source-sharded; reduction: {reduce_note})",
                       "l2": "flushed (256 MiB write) between timed steps; inputs + FULL store >> L2",
                       "store": {1: "full", 2: "checkpoint", 3: "boundary"}.get(stats["store"]),
                       "mode": {"fused": f"gradient + {K} H·v (fused)", "misfit": "misfit only (forward + residual)"}
                       .get(args.mode, f"{K} H·v"),
                       "shot_batch": S, "field_group": stats["field_group"]},
            "gpts_per_s": (U / (ms_step / 1000.0) / 1e9) if args.mode == "hessvec" else None,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": d["achieved_gbs"], "peak": peak, "unit": "GB/s",
                         "frac": d["frac"], "traffic": d["traffic"], "batched_frac": d["batched_frac"],
                         "dram_frac": d["dram_frac"], "peak_source": peak_src,
                         "alg_bytes_per_launch": d["alg_bytes_per_launch"],
                         "batched_bytes_per_launch": d["batched_bytes_per_launch"],
                         "avg_launch_ms": d["avg_launch_ms"], "kernels": kinfo},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        solver.close()
        if comm is not None:
            hv.nccl_comm_destroy(comm)
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
