"""GPU parity at FULL BASELINE sizes in the exact launch plans bench.py times, against oracle golden rows.

The golden files (tests/golden/, written by tools/make_golden.py, which calls only oracle/; provenance in
tests/golden/meta.json) hold the fp64 oracle's H·v rows / gradient for:
- cfg 1: all 16 shots, PSF probes k = 27 and 50, nt = 2000. The GPU runs the bench's plan: all 16 shots and all
  64 probes in ONE batch (S = 16, auto field groups, one-wave forward), rows 27 and 50 compared. Row k of a
  batched H·v does not depend on the other probes (O11), so the oracle needs only those two rows.
- cfg 3: shots 16..31 = one full 16-shot batch of the bench's 64-shot plan (S = 16, K = 32, the resident-q /
  large-Q forward), probes k = 0 (Rademacher) and 16 (cosine 1/16, 1/16: in band, SURVEY.md §8(c) P10 caveat),
  nt = 4000 -- so the reflected regime and BOUNDARY's 4000-step fp32 reverse reconstruction are both covered.
- cfg 2: shot 31, gradient (d_obs = F(v_true), oracle-written input) + probe 0 at nt = 4000, fused call; and the
  forward data d = F(m), F(v_true) of shot 31 at nt = 4000 (333 time steps per source period: the regime where a
  two-level fp32 leapfrog loses ~2e-4; the background runs in increment form).
Bar: relative L2 <= 1e-4 per row (BASELINE.json north_star)."""
import json
import os

import numpy as np
import pytest

from tests.conftest import rel_l2
import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-4
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.fail(f"missing golden file {path}: run tools/make_golden.py")
    if name.endswith(".npz"):
        z = np.load(path)
        return z[z.files[0]]
    return np.load(path).astype(np.float64)


@pytest.fixture(scope="module")
def hv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_10804_b200 as hvmod
    return hvmod


def test_cfg1_bench_plan_all_shots(hv):
    """cfg 1 in the bench's plan: 16 shots x 64 PSF spikes in one batch, H·v rows 27 and 50 vs the oracle."""
    import torch
    wl = W.config(1)
    gold = _gold("cfg1_hv_k27_k50.npy")
    s = hv.Solver.from_workload(wl)
    out = s.hessvec(torch.from_numpy(wl.model).cuda(), torch.from_numpy(wl.probes()).cuda()).cpu().numpy()
    st = s.stats()
    assert st["shot_batch"] == 16 and st["store"] == hv.STORE["full"]
    assert st["field_group"] >= 1
    for i, k in enumerate((27, 50)):
        assert rel_l2(out[k], gold[i]) <= TOL, (k, rel_l2(out[k], gold[i]))


@pytest.mark.parametrize("store", ["full", "boundary", "checkpoint"])
def test_cfg3_bench_plan_batch(hv, store):
    """cfg 3, one full batch of the bench plan (shots 16..31, all 32 probes, S = 16, large-Q forward), at full
    nt = 4000, in every storage mode; rows 0 and 16 vs the oracle."""
    import torch
    wl = W.config(3)
    gold = _gold("cfg3_hv_k0_k16_s16-32.npy")
    s = hv.Solver.from_workload(wl, src_begin=16, src_end=32, store=store)
    out = s.hessvec(torch.from_numpy(wl.model).cuda(), torch.from_numpy(wl.probes()).cuda()).cpu().numpy()
    st = s.stats()
    assert st["shot_batch"] == 16 and st["store"] == hv.STORE[store]
    assert st["fwd_kernel"] != 0          # Q = 32 x 2.02 MB > 48 MB: the large-Q forward, as in the bench
    for i, k in enumerate((0, 16)):
        assert rel_l2(out[k], gold[i]) <= TOL, (store, k, rel_l2(out[k], gold[i]))


def test_cfg3_single_shot_all_probes(hv):
    """cfg 3 shot 31 alone with all 32 probes (S = 1)."""
    wl = W.config(3)
    gold = _gold("cfg3_hv_k0_k16_s31.npy")
    s = hv.Solver.from_workload(wl, src_begin=31, src_end=32)
    out = s.hessvec(wl.model, wl.probes())
    assert s.stats()["shot_batch"] == 1
    for i, k in enumerate((0, 16)):
        assert rel_l2(out[k], gold[i]) <= TOL, (k, rel_l2(out[k], gold[i]))


@pytest.mark.parametrize("store", ["full", "checkpoint", "boundary"])
def test_cfg2_fused_gradient_hessvec_full_nt(hv, store):
    """cfg 2's BJ workload (gradient + 8 H·v in one fused pass) for shot 31 at full nt = 4000: g and H·v row 0."""
    wl = W.config(2)
    meta = json.load(open(os.path.join(GOLD, "meta.json")))["cfg2_s31"]
    d_obs = _gold("cfg2_s31_dobs.npz")[None].astype(np.float32)
    g_ref, hv_ref = _gold("cfg2_s31_grad.npy"), _gold("cfg2_s31_hv_k0.npy")
    s = hv.Solver.from_workload(wl, src_begin=31, src_end=32, store=store)
    phi, g, HV = s.gradient_hessvec(wl.model, d_obs, wl.probes())
    assert s.stats()["store"] == hv.STORE[store]
    assert rel_l2(g, g_ref) <= TOL, rel_l2(g, g_ref)
    assert rel_l2(HV[0], hv_ref) <= TOL, rel_l2(HV[0], hv_ref)
    assert abs(phi - meta["phi"]) <= 2 * TOL * meta["phi"]


def test_cfg2_forward_full_nt(hv):
    """d = f(m) (the evaluation model) and f(v_true) (sharp layered model) of shot 31 at full nt = 4000."""
    wl = W.config(2)
    s = hv.Solver.from_workload(wl, src_begin=31, src_end=32)
    d_m = s.forward_shot(wl.model, 31)
    assert s.stats()["fwd_kernel"] == 3   # forward-only on this grid: the T = 2 forward (two levels per launch)
    ref_m = _gold("cfg2_s31_d_m.npz").astype(np.float64)
    assert rel_l2(d_m, ref_m) <= TOL, rel_l2(d_m, ref_m)
    d_t = s.forward_shot(wl.model_true, 31)
    ref_t = _gold("cfg2_s31_dobs.npz").astype(np.float64)
    assert rel_l2(d_t, ref_t) <= TOL, rel_l2(d_t, ref_t)


def test_cfg4_grid_checkpoint_nt1000(hv):
    """cfg 4 grid (2048 x 6144, 12.9 M padded points), shot 127, probe 0, nt truncated to 1000, CHECKPOINT mode
    with k = 32 (SURVEY.md §8(d) parity sub-slice: the storage mode BJ cfg 4 mandates)."""
    wl = W.config(4).subset(shots=[127], nt=1000)
    gold = _gold("cfg4_s127_nt1000_hv_k0.npz").astype(np.float64)
    s = hv.Solver.from_workload(wl, store="checkpoint", ckpt_interval=32)
    out = s.hessvec(wl.model, wl.probes([0]))
    st = s.stats()
    assert st["store"] == hv.STORE["checkpoint"] and st["ckpt_interval"] == 32
    assert rel_l2(out[0], gold) <= TOL, rel_l2(out[0], gold)
