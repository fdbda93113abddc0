"""Where the end-to-end (host buffers) time goes vs device-resident inputs on cfg 1 (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_10804_b200 as hv  # noqa: E402
import workloads as W  # noqa: E402

wl = W.config(1)
s = hv.Solver.from_workload(wl)
V_h = wl.probes()
m_d, V_d = torch.from_numpy(wl.model).cuda(), torch.from_numpy(V_h).cuda()
m_p, V_p = torch.from_numpy(wl.model).pin_memory(), torch.from_numpy(V_h).pin_memory()
HV_d = torch.empty_like(V_d)
HV_p = torch.empty(V_d.shape, dtype=torch.float32).pin_memory()
for name, fn in (("device", lambda: s.hessvec(m_d, V_d, out=HV_d)),
                 ("pinned-in", lambda: s.hessvec(m_p, V_p, out=HV_d)),
                 ("pinned-in+out", lambda: (s.hessvec(m_p, V_p, out=HV_d), HV_p.copy_(HV_d, non_blocking=True))),
                 ("host-out", lambda: s.hessvec(m_p, V_p, out=HV_p))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    st = s.stats()
    print(f"{name:14s} wall {min(ts)*1e3:8.1f} ms  lib total {st['ms_total']:8.1f}  fwd {st['ms_forward']:7.1f}"
          f"  bwd {st['ms_backward']:7.1f}", flush=True)
