import numpy as np, workloads as W, paper_2507_10804_b200 as hv, os
wl = W.custom(70, 150, nt=300, ns=3, nrec=37, n_probes=3, f_peak=15.0, seed=5)
for sb in (1, 2, 3):
    s = hv.Solver.from_workload(wl, shot_batch=sb, store="full")
    try:
        d = s.forward(wl.model); print("forward ok sb", sb, float(np.abs(d).max()))
    except Exception as e: print("forward fail sb", sb, e)
    try:
        d = s.forward(wl.model); print("forward2 ok sb", sb)
    except Exception as e: print("forward2 fail sb", sb, e)
