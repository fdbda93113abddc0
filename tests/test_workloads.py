"""Host-side checks of the seeded input generators."""
import numpy as np
import pytest

import workloads as wlmod



@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_config_shapes_dtypes_determinism(k):
    a, b = wlmod.config(k), wlmod.config(k)
    assert a.model.dtype == np.float32 and a.model.shape == (a.nz, a.nx)
    assert np.array_equal(a.model, b.model) and np.array_equal(a.wavelet, b.wavelet)
    assert a.wavelet.shape == (a.nt,)
    assert np.all((a.src[:, 0] >= 0) & (a.src[:, 0] < a.nz) & (a.src[:, 1] >= 0) & (a.src[:, 1] < a.nx))
    assert np.all((a.rec[:, 0] >= 0) & (a.rec[:, 0] < a.nz) & (a.rec[:, 1] >= 0) & (a.rec[:, 1] < a.nx))
    p0 = a.probe_fn(0)
    assert p0.dtype == np.float32 and p0.shape == (a.nz, a.nx)
    assert np.array_equal(p0, b.probe_fn(0))
    # CFL (C15): dt max(v) / h below the 2nd-order-time / 8th-order-space limit 0.5546
    assert a.dt * float(a.model.max()) / a.h < 0.5546
    if a.model_true is not None:
        assert a.dt * float(a.model_true.max()) / a.h < 0.5546


def test_cfg_counts():
    assert (wlmod.config(0).ns, wlmod.config(0).nrec, wlmod.config(0).n_probes) == (2, 64, 1)
    c1 = wlmod.config(1)
    assert (c1.ns, c1.nrec, c1.n_probes, c1.nt) == (16, 401, 64, 2000)
    P = c1.probes()
    assert np.all(P.reshape(64, -1).sum(1) == 1.0)            # unit spikes (C22)
    assert len({tuple(np.argwhere(p)[0]) for p in P}) == 64      # distinct lattice points
    c2 = wlmod.config(2)
    assert (c2.ns, c2.nrec, c2.n_probes, c2.nt) == (64, 1152, 8, 4000)
    c3 = wlmod.config(3)
    assert c3.n_probes == 32
    r = c3.probe_fn(3)
    assert set(np.unique(r)) == {-1.0, 1.0}


def test_marmousi_like_ranges():
    c2 = wlmod.config(2)
    vt = c2.model_true
    assert vt.min() >= 1500.0 and vt.max() <= 5500.0
    assert np.all(vt[:8] == 1500.0)                               # 60 m water at h = 8
    assert np.all(c2.model[:8] == 1500.0)
    # layered: velocity broadly increases with depth
    assert vt[-1].mean() > vt[len(vt) // 2].mean() > vt[10].mean()
    # 12 layer velocities + water
    assert 8 <= len(np.unique(vt)) <= 13
