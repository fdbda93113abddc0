"""Time hv_gradient (forward sweep + residual + one adjoint field) on a BASELINE config (dev tool):
python tools/time_gradient.py --config 3 [--reps 3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_10804_b200 as hv  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
wl = W.config(a.config)
m = torch.from_numpy(wl.model).cuda()
s = hv.Solver.from_workload(wl)
mt = torch.from_numpy(wl.model_true if wl.model_true is not None else wl.model).cuda()
d_obs = torch.as_tensor(s.forward(mt), device="cuda")
s.gradient(m, d_obs)
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phi, g = s.gradient(m, d_obs)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
st = s.stats()
nb = -(-wl.ns // st["shot_batch"])
print(json.dumps({"config": a.config, "ms": round(min(ts), 1), "phi": float(phi), "shot_batch": st["shot_batch"],
                  "fwd_kernel": st["fwd_kernel"], "bwd_kernel": st["bwd_kernel"],
                  "fwd_us_per_level": round(1e3 * st["ms_forward"] / (nb * (wl.nt - 1)), 1),
                  "bwd_us_per_level": round(1e3 * st["ms_backward"] / (nb * (wl.nt - 1)), 1)}))
