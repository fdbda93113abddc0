#!/usr/bin/env python
"""Benchmark of the Gauss-Newton H·v hot path (BASELINE.json metric: "Hessian-vector products/s and stencil
Gpts/s (frac of HBM roofline) at 1/2/4/8 GPU").

Workload (N = 1 and every N): BASELINE configs[1] — quadratic-depth model 201 x 401 (h = 10 m), 16 surface
shots, nt = 2000, a batch of 64 PSF unit-spike probes -> 64 H·v per step. One step = one hv_hessvec over all
16 shots (sharded across ranks by contiguous source blocks) + the NCCL all-reduce of the per-source partial
sums. Total work is fixed as N grows ("scaling": "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl reference]

value  : H·v/s with m and probes resident in HBM (device pointers); per-step CUDA events on the launch stream,
         L2 flushed (256 MiB write) between timed steps, max over ranks.
e2e    : same metric through the C ABI with pinned HOST inputs, H2D/D2H copies inside the timed region.
roofline: dominant kernel's algorithmic bytes per launch / its average launch time (library CUDA events).
cpu_baseline: the fp64 oracle, as it stands, on a bounded sample (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def alg_bytes(wl, K, shots):
    """Algorithmic fp32 HBM bytes per launch = SURVEY.md §8(d) per-unit figures x units per launch:
    forward step: a1 16 B + a2 16 B per Born field, per padded point, + FULL store write 4 B per interior point;
    backward step: a5 + a7 20 B per adjoint field per padded point + FULL store read 4 B per interior point.
    These are the bytes of a per-shot single-step scheme; the kernels share q_k and the imaging sums across the
    shots of a launch, so they move fewer (the measured DRAM bytes are reported as `traffic`)."""
    Np, N, _ = workload_counts(wl, K)
    fwd = shots * (16.0 * Np * (1 + K) + 4.0 * N)
    bwd = shots * (20.0 * Np * K + 4.0 * N)
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


# ------------------------------------------------------------------------------------------- CPU oracle


def cpu_oracle_sample(wl, K_full, nt_sample=400, shot=7):
    """Time the fp64 oracle as it stands (test infrastructure; cpu_baseline / --impl reference only) on a
    bounded sample: one shot, one probe, nt_sample levels. Returns (H·v/s extrapolated, seconds, sample str)."""
    from oracle import wave
    sub = wl.subset(shots=[shot], nt=nt_sample)
    V = wl.probes([min(27, wl.n_probes - 1)]).astype(np.float64)
    pb = wave.Problem(sub)
    t0 = time.perf_counter()
    pb.hessvec(list(V), shots=[0])
    dt = time.perf_counter() - t0
    Np = (wl.nz + 2 * wl.W) * (wl.nx + 2 * wl.W)
    u_sample = (nt_sample - 1) * Np * (2 + 2 * 1)
    rate = u_sample / dt                                    # field updates / s
    _, _, U = workload_counts(wl, K_full)
    hvps = K_full * rate / U
    sample = (f"oracle.wave hessvec, {wl.name} shot {shot}, 1 PSF probe, nt={nt_sample} of {wl.nt}; "
              f"extrapolated by field updates U = Ns (nt-1) Np (2+2K) = {U:.3e}")
    return hvps, dt, sample


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = W.config(args.config)
    K = wl.n_probes
    for _ in range(args.warmup):
        cpu_oracle_sample(wl, K, nt_sample=args.ref_nt)
    vals, secs = [], []
    sample = ""
    for _ in range(args.steps):
        v, s, sample = cpu_oracle_sample(wl, K, nt_sample=args.ref_nt)
        vals.append(v)
        secs.append(s)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "hessian_vector_products_per_s", "value": value, "unit": "H·v/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * K / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{args.config}", "shots": wl.ns, "probes": K, "nt": wl.nt,
                   "grid": [wl.nz, wl.nx], "parallelism": "host oracle"},
        "cpu_baseline": {"value": value, "unit": "H·v/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores_available": len(os.sched_getaffinity(0))},
        "e2e": {"value": value, "unit": "H·v/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------- GPU arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--shot-batch", type=int, default=0)
    ap.add_argument("--field-group", type=int, default=0)
    ap.add_argument("--store", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-nt", type=int, default=300)
    ap.add_argument("--cpu-nt", type=int, default=1000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shots", type=int, default=0,
                    help="evidence runs only: first N shots of the config (the JSON config says so)")
    ap.add_argument("--nt", type=int, default=0, help="evidence runs only: truncated time axis")
    ap.add_argument("--fused", action="store_true",
                    help="evidence runs only: one step = gradient + K H·v in one fused pass (BJ cfg 2's workload)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2507_10804_b200 as hv

    ws, rank, local = dist_env()
    if ws > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2507_10804_b200.dist import shard_range

    wl = W.config(args.config)
    if args.shots or args.nt:  # reduced evidence run (never the driver's bench line)
        wl = wl.subset(shots=range(args.shots) if args.shots else None, nt=args.nt or None)
    K = wl.n_probes
    ns = wl.ns
    b, e = shard_range(ns, ws, rank)
    solver = hv.Solver.from_workload(wl, src_begin=b, src_end=e, device=local, store=args.store,
                                     shot_batch=args.shot_batch, field_group=args.field_group)
    V_h = wl.probes()
    m_d = torch.from_numpy(wl.model).to(dev)
    V_d = torch.from_numpy(V_h).to(dev)
    HV_d = torch.empty((K, wl.nz, wl.nx), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    if args.fused:  # d_obs = F(model_true) on this rank's shard (the library's own forward, outside the timing)
        dobs_d = torch.as_tensor(solver.forward(torch.from_numpy(
            wl.model_true if wl.model_true is not None else wl.model).to(dev)), device=dev)

    def step():
        if args.fused:
            _, g_d, hv_d = solver.gradient_hessvec(m_d, dobs_d, V_d)
            if ws > 1:
                dist.all_reduce(g_d)
                dist.all_reduce(hv_d)
            return
        solver.hessvec(m_d, V_d, out=HV_d)
        if ws > 1:
            dist.all_reduce(HV_d)

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

    # ---- e2e: pinned host inputs -> C ABI (H2D inside) -> device result -> all-reduce -> pinned host result
    e2e = None
    if not args.no_e2e:
        m_p = torch.from_numpy(wl.model).pin_memory()
        V_p = torch.from_numpy(V_h).pin_memory()
        HV_p = torch.empty((K, wl.nz, wl.nx), dtype=torch.float32).pin_memory()

        def e2e_step():
            solver.hessvec(m_p, V_p, out=HV_d)
            if ws > 1:
                dist.all_reduce(HV_d)
            HV_p.copy_(HV_d, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_step()
        et = []
        for _ in range(max(3, args.steps)):
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
               "d2h_bytes_per_step": int(4 * wl.nz * wl.nx * K)}

    if rank == 0:
        Np, N, U = workload_counts(wl, K)
        shots_per_batch = solver.stats()["shot_batch"]
        nloc = e - b
        nbatch = math.ceil(nloc / shots_per_batch)
        fb, bb = alg_bytes(wl, K, shots_per_batch)
        f_launch_ms = float(np.mean(fwd_ms)) / (nbatch * (wl.nt - 1))
        b_launch_ms = float(np.mean(bwd_ms)) / (nbatch * (wl.nt - 1))
        peak, peak_src = hbm_peak()
        fwd_name = {0: "fwd_step_kernel", 1: "fwd_qres_kernel", 2: "fwd2_kernel"}.get(solver.stats()["fwd_kernel"],
                                                                                      "fwd_step_kernel")
        kern = {fwd_name: (fb, f_launch_ms), "bwd_step_kernel": (bb, b_launch_ms)}
        dom = max(kern, key=lambda k: kern[k][1])
        achieved = kern[dom][0] / (kern[dom][1] / 1000.0) / 1e9
        traffic, traffic_src = None, None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                rec = tj.get(dom, {})
                if rec.get("config") == {"workload": f"cfg{args.config}", "shot_batch": shots_per_batch,
                                         "field_group": solver.stats()["field_group"]}:
                    traffic, traffic_src = rec.get("dram_bytes_per_launch"), tj.get("source")
            except Exception:
                traffic = None
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            hvps, secs, sample = cpu_oracle_sample(wl, K, nt_sample=args.cpu_nt)
            cpu = {"value": hvps, "unit": "H·v/s", "cores": 1, "kind": "oracle", "sample": sample,
                   "seconds": round(secs, 2), "host_cores_available": len(os.sched_getaffinity(0))}
        value = K / (ms_step / 1000.0)
        line = {
            "metric": "hessian_vector_products_per_s", "value": value, "unit": "H·v/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg{args.config}" + (f" (first {wl.ns} shots, nt {wl.nt}: evidence run)"
                                                          if args.shots or args.nt else ""),
                       "model": "quadratic-depth v(z)" if args.config == 1
                       else wl.name, "grid": [wl.nz, wl.nx], "shots": ns, "probes": K, "nt": wl.nt,
                       "global_batch": K, "parallelism": f"dp{ws} (source-sharded, NCCL all-reduce of H·v)",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "store": {1: "full", 2: "checkpoint"}.get(solver.stats()["store"]),
                       "mode": f"gradient + {K} H·v (fused)" if args.fused else f"{K} H·v",
                       "shot_batch": shots_per_batch, "field_group": solver.stats()["field_group"]},
            "gpts_per_s": U / (ms_step / 1000.0) / 1e9,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "dram_frac": (traffic / (kern[dom][1] / 1000.0) / 1e9 / peak) if traffic else None,
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": kern[dom][0], "avg_launch_ms": kern[dom][1],
                         "kernels": {k: {"alg_bytes_per_launch": v[0], "avg_launch_ms": v[1],
                                         "achieved_gbs": v[0] / (v[1] / 1000.0) / 1e9}
                                     for k, v in kern.items()}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
