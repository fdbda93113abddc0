import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_10804_b200 as hv
import workloads as W
from tests.conftest import rel_l2
G = "tests/golden"
wl = W.config(2)
dm = np.load(f"{G}/cfg2_s31_d_m.npz")["d"].astype(np.float64)
d_obs = np.load(f"{G}/cfg2_s31_dobs.npz")["d_obs"].astype(np.float64)
s = hv.Solver.from_workload(wl, src_begin=31, src_end=32)
d = s.forward_shot(wl.model, 31)
for n in (500, 1000, 2000, 3000, 4000):
    print("eps_d(m) up to", n, rel_l2(d[:n], dm[:n]))
rho_o = dm - d_obs
rho_g = d - d_obs
print("|rho|/|d|", np.linalg.norm(rho_o) / np.linalg.norm(dm), "rel err of rho", rel_l2(rho_g, rho_o))
