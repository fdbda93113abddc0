"""Sweep launch knobs (shots in flight S, fields per CTA FG, store) of hv_hessvec on a BASELINE config.
Dev tool: python tools/tune.py --config 1 --S 1,2,4 --FG 4,8,16"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_10804_b200 as hv  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--S", default="1,2,4")
ap.add_argument("--FG", default="4,8,16")
ap.add_argument("--store", default="full")
ap.add_argument("--shots", type=int, default=0, help="limit shots (0 = all)")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
wl = W.config(a.config)
if a.shots:
    wl = wl.subset(shots=range(a.shots))
V = torch.from_numpy(wl.probes()).cuda()
m = torch.from_numpy(wl.model).cuda()
out = torch.empty_like(V)
for S, FG in itertools.product([int(x) for x in a.S.split(",")], [int(x) for x in a.FG.split(",")]):
    s = hv.Solver.from_workload(wl, shot_batch=S, field_group=FG, store=a.store)
    s.hessvec(m, V, out=out)
    best = None
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.hessvec(m, V, out=out)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1)
        st = s.stats()
        if best is None or t < best[0]:
            best = (t, st)
    t, st = best
    nb = -(-s.nloc // st["shot_batch"])
    print(json.dumps({"S": st["shot_batch"], "FG": FG, "ms": round(t, 1), "hv_per_s": round(V.shape[0] / t * 1e3, 2),
                      "fwd_launch_us": round(1e3 * st["ms_forward"] / (nb * (wl.nt - 1)), 2),
                      "bwd_launch_us": round(1e3 * st["ms_backward"] / (nb * (wl.nt - 1)), 2)}), flush=True)
    s.close()
