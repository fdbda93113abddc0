"""Tiny end-to-end exercise of every libhv entry point and storage mode (target of compute-sanitizer runs)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2507_10804_b200 as hv  # noqa: E402
import workloads as W  # noqa: E402

wl = W.custom(20, 70, nt=40, ns=3, nrec=11, n_probes=2, W=6, f_peak=25.0, seed=3)
wl.rec = np.concatenate([wl.rec, wl.rec[:2]])          # duplicate receivers (R^T scatter-add)
V = wl.probes()
for store in ("full", "checkpoint", "boundary"):
    s = hv.Solver.from_workload(wl, store=store, ckpt_interval=7, shot_batch=2, field_group=1)
    d = s.forward(wl.model)
    phi, g, H = s.gradient_hessvec((0.97 * wl.model).astype(np.float32), d, V)
    H2 = s.hessvec(wl.model, V)
    assert np.isfinite(H).all() and np.isfinite(H2).all() and np.isfinite(g).all()
rng = np.random.default_rng(0)
a = rng.standard_normal((2, 20, 70)).astype(np.float32)
b = (rng.standard_normal((2, 20, 70)) + 1j * rng.standard_normal((2, 20, 70))).astype(np.complex64)
for mode in range(3):
    s.psido_apply(a, b, V[0], mode)
    s.psido_apply(b, b, V[0], mode)
rows = s.psf_rows(H2, [(5, 10), (12, 50)], [0, 1], 4)
w = s.psf_weights(20, 70, [5, 12], [10, 50])
cols = s.pdo_columns(H2[0], [(1, 3), (19, 67)], 1.5)
s.pdo_weights(20, 70, wl.h, 0.05, [math.pi / 2, 3 * math.pi / 2])
A, B, alpha = s.psf_plus(rows, np.ascontiguousarray(w[[0, 3]]), cols, [(1, 3), (19, 67)], 1)
s.highpass(V, wl.h, 0.01, 0.005)
ev, vec = s.lowrank_geneig(wl.model, rng.standard_normal((4, 20, 70)).astype(np.float32), 2, 1, 1.0, 1.0)
print("sanitize case ok", float(np.abs(H2).max()), ev)
