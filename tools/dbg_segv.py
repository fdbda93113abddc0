import faulthandler, sys; faulthandler.enable()
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2507_10804_b200 as hv, workloads as W
wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
V = wl.probes()
print("create", flush=True)
s = hv.Solver.from_workload(wl, device=0)
print("fwd", flush=True)
d = s.forward(wl.model); print("d ok", float(np.abs(d).max()), flush=True)
out = s.hessvec(wl.model, V); print("hv ok", float(np.abs(out).max()), flush=True)
