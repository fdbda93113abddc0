import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_10804_b200 as hv
import workloads as W
from tests.conftest import rel_l2
G = "tests/golden"
wl = W.config(2)
d_obs = np.load(f"{G}/cfg2_s31_dobs.npz")["d_obs"].astype(np.float32)
meta = json.load(open(f"{G}/meta.json"))["cfg2_s31"]
g_ref = np.load(f"{G}/cfg2_s31_grad.npy").astype(np.float64)
hv_ref = np.load(f"{G}/cfg2_s31_hv_k0.npy").astype(np.float64)
s = hv.Solver.from_workload(wl, src_begin=31, src_end=32, store="full")
d_true = s.forward(wl.model_true)[0]
print("eps_d (forward at v_true vs oracle d_obs, nt 4000):", rel_l2(d_true, d_obs))
for n in (500, 1000, 2000, 3000, 4000):
    print("  eps_d up to level", n, rel_l2(d_true[:n], d_obs[:n]))
d_m = s.forward(wl.model)[0]
rho = d_m.astype(np.float64) - d_obs
print("|rho|/|d|", np.linalg.norm(rho) / np.linalg.norm(d_obs), "phi gpu-forward", 0.5 * np.sum(rho ** 2), "phi oracle", meta["phi"])
for store in ("full", "checkpoint", "boundary"):
    s = hv.Solver.from_workload(wl, src_begin=31, src_end=32, store=store)
    phi, g, HV = s.gradient_hessvec(wl.model, d_obs[None], wl.probes())
    print(store, "g", rel_l2(g, g_ref), "hv0", rel_l2(HV[0], hv_ref), "phi", abs(phi - meta["phi"]) / meta["phi"])
    phi2, g2 = s.gradient(wl.model, d_obs[None])
    print(store, "gradient-only g", rel_l2(g2, g_ref))
