#!/usr/bin/env python
"""Write the oracle golden files under tests/golden/ (calls ONLY oracle/ and workloads/; never the CUDA path).

These are the fp64 oracle's answers for the exact launch plans the bench times, at full BASELINE sizes
(VERDICT r01 "next round" 1; SURVEY.md §8(d) parity sub-slices, widened to whole shot batches):

  cfg1_hv_k27_k50.npy      cfg 1 (201 x 401, nt 2000), ALL 16 shots, H·v rows of PSF probes k = 27 and 50
                           (row k of a batched H·v does not depend on the other probes: O11)
  cfg3_hv_k0_k16_s16-32.npy cfg 3 (384 x 1152, nt 4000), shots 16..31 (one full 16-shot batch of the bench
                           plan), H·v rows of probes k = 0 (Rademacher) and k = 16 (cosine 1/16, 1/16)
  cfg3_hv_k0_k16_s31.npy   the same rows for shot 31 alone
  cfg2_s31_dobs.npz        cfg 2 shot 31: d_obs = F(v_true) (float32, C17) -- an oracle-written INPUT
  cfg2_s31_grad.npy        gradient F*(F(m) - d_obs) of shot 31 at m (Eq. equ:grad)
  cfg2_s31_hv_k0.npy       H·v row of probe k = 0 for shot 31
  cfg2_s31_d_m.npz         d = F(m) of shot 31 at the evaluation model m (cfg 2 and cfg 3 share m and geometry)
  cfg4_s127_nt1000_hv_k0.npz  cfg 4 grid (2048 x 6144), shot 127, probe 0, nt truncated to 1000 (SURVEY.md §8(d)
                           parity sub-slice; the GPU runs it in CHECKPOINT mode with k = 32)
  meta.json                provenance: recipe, oracle calls, phi, timings, sha256 of oracle/wave.py

Every value is computed in float64 by oracle.wave.Problem and rounded once to
float32 for storage (rounding error 6e-8 relative, far below the 1e-4 gate). Shot contributions are summed in
float64 in increasing shot order.

    OMP_NUM_THREADS=1 python tools/make_golden.py [--workers 6] [--only cfg1,cfg2,cfg3]

Runtime on 6 host cores: about an hour (the numpy oracle needs ~30 ms per field-step on the cfg 2/3 grid).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")

import numpy as np  # noqa: E402

CFG1_PROBES = [27, 50]          # (i, j) = (3, 3) and (6, 2) of the 8 x 8 spike lattice
CFG3_PROBES = [0, 16]           # Rademacher seed 0; cos(2 pi (ix + iz) / 16)
CFG3_SHOTS = list(range(16, 32))
CFG2_SHOT = 31


def _cfg1_shot(s):
    import workloads as W
    from oracle import wave
    wl = W.config(1)
    V = wl.probes(CFG1_PROBES).astype(np.float64)
    t0 = time.time()
    out = wave.Problem(wl).hessvec_shot(s, list(V), mode="full")
    return ("cfg1", s, out, time.time() - t0)


def _cfg3_shot(s):
    import workloads as W
    from oracle import wave
    wl = W.config(3)
    V = wl.probes(CFG3_PROBES).astype(np.float64)
    t0 = time.time()
    out = wave.Problem(wl).hessvec_shot(s, list(V), mode="checkpoint", ckpt=63)
    return ("cfg3", s, out, time.time() - t0)


def _cfg2(_):
    import workloads as W
    from oracle import wave
    wl = W.config(2)
    t0 = time.time()
    d_obs = wave.Problem(wl, wl.model_true).forward(CFG2_SHOT).astype(np.float32)   # C17: rounded once
    pb = wave.Problem(wl)
    phi, g = pb.gradient(d_obs[None], shots=[CFG2_SHOT], mode="checkpoint", ckpt=63)
    hv = pb.hessvec_shot(CFG2_SHOT, [wl.probes([0])[0].astype(np.float64)], mode="checkpoint", ckpt=63)
    return ("cfg2", CFG2_SHOT, (d_obs, phi, g, hv[0]), time.time() - t0)


def _cfg2_dm(_):
    import workloads as W
    from oracle import wave
    wl = W.config(2)
    t0 = time.time()
    d = wave.Problem(wl).forward(CFG2_SHOT)
    return ("cfg2dm", CFG2_SHOT, d, time.time() - t0)


def _cfg4(_):
    import workloads as W
    from oracle import wave
    wl = W.config(4).subset(shots=[127], nt=1000)
    t0 = time.time()
    hv = wave.Problem(wl).hessvec_shot(0, [wl.probes([0])[0].astype(np.float64)], mode="checkpoint", ckpt=32)
    return ("cfg4", 127, hv[0], time.time() - t0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=6)
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg2dm,cfg4")
    a = ap.parse_args()
    only = set(a.only.split(","))
    os.makedirs(OUT, exist_ok=True)
    tasks = []
    if "cfg3" in only:
        tasks += [(_cfg3_shot, s) for s in CFG3_SHOTS]
    if "cfg2" in only:
        tasks += [(_cfg2, 0)]
    if "cfg1" in only:
        tasks += [(_cfg1_shot, s) for s in range(16)]
    if "cfg2dm" in only:
        tasks += [(_cfg2_dm, 0)]
    if "cfg4" in only:
        tasks += [(_cfg4, 0)]
    t0 = time.time()
    res = {}
    with Pool(a.workers) as pool:
        pending = [pool.apply_async(f, (x,)) for f, x in tasks]
        for p in pending:
            kind, s, out, secs = p.get()
            res[(kind, s)] = (out, secs)
            print(f"{kind} shot {s}: {secs:.0f} s (elapsed {time.time() - t0:.0f} s)", flush=True)
    mpath = os.path.join(OUT, "meta.json")
    meta = json.load(open(mpath)) if os.path.exists(mpath) else {}
    with open(os.path.join(ROOT, "oracle", "wave.py"), "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()
    common = {"writer": "tools/make_golden.py (oracle.wave.Problem only)", "oracle_wave_sha256": sha,
              "dtype": "float64 oracle, stored float32"}
    if "cfg1" in only:
        acc = np.zeros((len(CFG1_PROBES), 201, 401))
        for s in range(16):
            acc += res[("cfg1", s)][0]
        np.save(os.path.join(OUT, "cfg1_hv_k27_k50.npy"), acc.astype(np.float32))
        meta["cfg1_hv_k27_k50"] = {**common, "config": 1, "shots": list(range(16)), "probes": CFG1_PROBES,
                                   "call": "Problem(config(1)).hessvec_shot(s, probes, mode='full'), summed over s",
                                   "cpu_s": sum(res[("cfg1", s)][1] for s in range(16))}
    if "cfg3" in only:
        acc = np.zeros((len(CFG3_PROBES), 384, 1152))
        for s in CFG3_SHOTS:
            acc += res[("cfg3", s)][0]
        np.save(os.path.join(OUT, "cfg3_hv_k0_k16_s16-32.npy"), acc.astype(np.float32))
        np.save(os.path.join(OUT, "cfg3_hv_k0_k16_s31.npy"), res[("cfg3", 31)][0].astype(np.float32))
        meta["cfg3_hv_k0_k16"] = {**common, "config": 3, "shots": CFG3_SHOTS, "single_shot_file_shot": 31,
                                  "probes": CFG3_PROBES,
                                  "call": "Problem(config(3)).hessvec_shot(s, probes, mode='checkpoint', ckpt=63)",
                                  "cpu_s": sum(res[("cfg3", s)][1] for s in CFG3_SHOTS)}
    if "cfg2" in only:
        (d_obs, phi, g, hv0), secs = res[("cfg2", CFG2_SHOT)]
        np.savez_compressed(os.path.join(OUT, "cfg2_s31_dobs.npz"), d_obs=d_obs)
        np.save(os.path.join(OUT, "cfg2_s31_grad.npy"), g.astype(np.float32))
        np.save(os.path.join(OUT, "cfg2_s31_hv_k0.npy"), hv0.astype(np.float32))
        meta["cfg2_s31"] = {**common, "config": 2, "shot": CFG2_SHOT, "probes": [0], "phi": phi,
                            "call": "d_obs = Problem(config(2), model_true).forward(31) -> float32; "
                                    "Problem(config(2)).gradient(d_obs, shots=[31], mode='checkpoint', ckpt=63); "
                                    "hessvec_shot(31, [probe 0], mode='checkpoint', ckpt=63)",
                            "cpu_s": secs}
    if "cfg2dm" in only:
        d, secs = res[("cfg2dm", CFG2_SHOT)]
        np.savez_compressed(os.path.join(OUT, "cfg2_s31_d_m.npz"), d=d.astype(np.float32))
        meta["cfg2_s31_d_m"] = {**common, "config": 2, "shot": CFG2_SHOT,
                                "call": "Problem(config(2)).forward(31) (the evaluation model m)", "cpu_s": secs}
    if "cfg4" in only:
        hv0, secs = res[("cfg4", 127)]
        np.savez_compressed(os.path.join(OUT, "cfg4_s127_nt1000_hv_k0.npz"), hv=hv0.astype(np.float32))
        meta["cfg4_s127_nt1000"] = {**common, "config": 4, "shot": 127, "probes": [0], "nt": 1000,
                                    "call": "Problem(config(4).subset(shots=[127], nt=1000)).hessvec_shot(0, [probe 0], "
                                            "mode='checkpoint', ckpt=32)", "cpu_s": secs}
    with open(mpath, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
