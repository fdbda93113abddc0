"""The oracle golden files (tests/golden/, written by tools/make_golden.py) on CPU: provenance matches the oracle
as it stands, shapes match the configs, and the stored rows satisfy the invariants the paper fixes for H_d --
self-adjointness and positive semi-definiteness of the Gauss-Newton normal operator --
so a corrupted or stale golden file fails here before any GPU comparison uses it."""
import hashlib
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def meta():
    return json.load(open(os.path.join(GOLD, "meta.json")))


def test_provenance_matches_current_oracle(meta):
    sha = hashlib.sha256(open(os.path.join(ROOT, "oracle", "wave.py"), "rb").read()).hexdigest()
    for key, rec in meta.items():
        assert rec["oracle_wave_sha256"] == sha, f"{key} was written by a different oracle/wave.py"
        assert "tools/make_golden.py" in rec["writer"]


def test_shapes(meta):
    assert np.load(os.path.join(GOLD, "cfg1_hv_k27_k50.npy")).shape == (2, 201, 401)
    for f in ("cfg3_hv_k0_k16_s16-32.npy", "cfg3_hv_k0_k16_s31.npy"):
        assert np.load(os.path.join(GOLD, f)).shape == (2, 384, 1152)
    assert np.load(os.path.join(GOLD, "cfg2_s31_dobs.npz"))["d_obs"].shape == (4000, 1152)
    assert np.load(os.path.join(GOLD, "cfg2_s31_d_m.npz"))["d"].shape == (4000, 1152)
    assert np.load(os.path.join(GOLD, "cfg4_s127_nt1000_hv_k0.npz"))["hv"].shape == (2048, 6144)
    assert meta["cfg1_hv_k27_k50"]["shots"] == list(range(16))
    assert meta["cfg3_hv_k0_k16"]["shots"] == list(range(16, 32))


def test_cfg1_rows_symmetric_and_psd():
    """H_d is self-adjoint: (H e_i)(x_j) = (H e_j)(x_i) for the unit spikes at x_27 and x_50, and
    <e_i, H e_i> = |J e_i|^2 > 0 (summed over all 16 shots)."""
    wl = W.config(1)
    V = wl.probes([27, 50])
    p27 = tuple(np.argwhere(V[0])[0])
    p50 = tuple(np.argwhere(V[1])[0])
    g = np.load(os.path.join(GOLD, "cfg1_hv_k27_k50.npy")).astype(np.float64)
    assert g[0][p27] > 0 and g[1][p50] > 0
    off = g[0][p50], g[1][p27]
    assert abs(off[0] - off[1]) <= 1e-5 * max(abs(off[0]), abs(off[1]), 1e-300) + 1e-6 * max(g[0][p27], g[1][p50])


def test_cfg3_rows_psd_and_batch_contains_shot31():
    """<v_k, H v_k> = sum_s |J_s v_k|^2 >= 0, and the 16-shot batch sum is larger than shot 31's own term."""
    wl = W.config(3)
    V = wl.probes([0, 16]).astype(np.float64)
    g = np.load(os.path.join(GOLD, "cfg3_hv_k0_k16_s16-32.npy")).astype(np.float64)
    g31 = np.load(os.path.join(GOLD, "cfg3_hv_k0_k16_s31.npy")).astype(np.float64)
    for k in range(2):
        q, q31 = float(np.sum(V[k] * g[k])), float(np.sum(V[k] * g31[k]))
        assert q > 0 and q31 > 0 and q > q31


def test_cfg2_gradient_and_hv(meta):
    """phi > 0 (v_true != m), <v_0, H v_0> > 0, finite gradient."""
    wl = W.config(2)
    v0 = wl.probes([0])[0].astype(np.float64)
    hv0 = np.load(os.path.join(GOLD, "cfg2_s31_hv_k0.npy")).astype(np.float64)
    g = np.load(os.path.join(GOLD, "cfg2_s31_grad.npy"))
    assert meta["cfg2_s31"]["phi"] > 0 and np.isfinite(g).all() and np.abs(g).max() > 0
    assert float(np.sum(v0 * hv0)) > 0


def test_cfg4_row_psd():
    """<v_0, H v_0> > 0 for the cfg 4 grid slice (shot 127, nt 1000)."""
    wl = W.config(4)
    v0 = wl.probes([0])[0].astype(np.float64)
    hv0 = np.load(os.path.join(GOLD, "cfg4_s127_nt1000_hv_k0.npz"))["hv"].astype(np.float64)
    assert float(np.sum(v0 * hv0)) > 0
