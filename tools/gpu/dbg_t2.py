import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_10804_b200 as hv
import workloads as W
from oracle import wave
for ns, sb in ((2, 1), (2, 2), (3, 2), (3, 3)):
    for nt in (3, 4, 10):
        K = 1
        wl = W.custom(70, 150, nt=nt, ns=ns, nrec=37, n_probes=K, f_peak=15.0, seed=5)
        V = wl.probes()
        res = {}
        for t2 in ("0", "1"):
            os.environ["HV_T2"] = t2
            os.environ["HV_T2B"] = "0"
            s = hv.Solver.from_workload(wl, store="full", shot_batch=sb)
            res[t2] = s.hessvec(wl.model, V)
        ref = wave.Problem(wl).hessvec(list(V.astype(np.float64)))
        e = lambda a: float(np.linalg.norm(a - ref) / max(np.linalg.norm(ref), 1e-300))
        print(ns, sb, nt, "bitwise", np.array_equal(res["0"], res["1"]), "err0", e(res["0"]), "err1", e(res["1"]))
