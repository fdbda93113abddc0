import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_10804_b200 as hv
import workloads as W
for (nz, nx, nt) in ((70, 150, 200), (30, 40, 200)):
    wl = W.custom(nz, nx, nt=nt, ns=1, nrec=37, n_probes=1, f_peak=15.0, seed=5)
    iz, ix = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
    wl.rec = np.stack([iz.ravel(), ix.ravel()], 1).astype(np.int32)
    res = {}
    for t2 in ("0", "1"):
        os.environ["HV_T2"] = t2
        s = hv.Solver.from_workload(wl, store="full", shot_batch=1)
        res[t2] = s.forward(wl.model)[0].reshape(nt, nz, nx)
    diff = np.argwhere(res["0"] != res["1"])
    print(nz, nx, "ndiff", len(diff))
    if len(diff):
        n0 = diff[:, 0].min()
        pts = diff[diff[:, 0] == n0]
        print(" first level", n0, "points", pts[:10, 1:].tolist())
        for p in pts[:4]:
            print("  ", p.tolist(), float(res["0"][tuple(p)]), float(res["1"][tuple(p)]))
