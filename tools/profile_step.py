"""Run hv_hessvec on a BASELINE config a few times (target of ncu captures). Dev tool."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_10804_b200 as hv  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--S", type=int, default=0)
ap.add_argument("--FG", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--shots", type=int, default=0)
ap.add_argument("--nt", type=int, default=0)
ap.add_argument("--store", default="auto")
a = ap.parse_args()
wl = W.config(a.config)
if a.shots:
    wl = wl.subset(shots=range(a.shots))
if a.nt:
    wl = wl.subset(nt=a.nt)
V = torch.from_numpy(wl.probes()).cuda()
m = torch.from_numpy(wl.model).cuda()
s = hv.Solver.from_workload(wl, shot_batch=a.S, field_group=a.FG, store=a.store)
for _ in range(a.reps):
    out = s.hessvec(m, V)
torch.cuda.synchronize()
print("ok", s.stats())
