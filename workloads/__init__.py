"""Seeded synthetic inputs for the Gauss-Newton H·v hot path.

This module is shared DATA plumbing: it builds velocity models, acquisition geometry, the
source wavelet and probe vectors for BASELINE.json configs 0-4 (and small custom cases).
It holds none of the method's arithmetic (no stencil, no sponge, no Born / adjoint /
imaging), so both the fp64 oracle (`oracle/`) and the CUDA path
(`paper_2507_10804_b200/`) consume it without sharing any method code.

Every array is generated in float64 and rounded ONCE to float32;
the oracle casts those float32 values back to float64.

Reading notes (DESIGN.md §3 lists every reading):
- "round" below is round-half-up, floor(x + 0.5), never numpy's banker's rounding.
- The source function s(t) is the Ricker wavelet with delay t0 = 1/f_peak (C9);
  it is an input of the forward map (Eq. equ:pde: "s(t) denotes the
  source function"), not part of the discretised operator.
- Sources/receivers sit on grid nodes at iz = round(depth / h) (C7, C8, C19).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional

import numpy as np
from scipy.ndimage import gaussian_filter

F32 = np.float32

# Sponge width on all four sides, cells (BJ cfg 0: "plus a 20-cell sponge"; C10 extends it
# to every config).
SPONGE_W = 20


def _round_half_up(x):
    return np.floor(np.asarray(x, dtype=np.float64) + 0.5).astype(np.int64)


def _smooth(a: np.ndarray, sigma: float) -> np.ndarray:
    """Gaussian smoothing used by every recipe: scipy gaussian_filter, mode='nearest', truncate=4."""
    return gaussian_filter(np.asarray(a, dtype=np.float64), sigma, mode="nearest", truncate=4.0)


def ricker(nt: int, dt: float, f_peak: float, t0: Optional[float] = None) -> np.ndarray:
    """Ricker wavelet s[n] = (1 - 2 pi^2 f^2 (t_n - t0)^2) exp(-pi^2 f^2 (t_n - t0)^2),
    t_n = n dt, t0 = 1/f. Returned as float32."""
    if t0 is None:
        t0 = 1.0 / f_peak
    t = np.arange(nt, dtype=np.float64) * dt - t0
    a = (math.pi * f_peak * t) ** 2
    return ((1.0 - 2.0 * a) * np.exp(-a)).astype(F32)


@dataclasses.dataclass
class Workload:
    """One synthetic problem. Arrays are float32 / int32, layout [nz][nx] z-major row-major."""

    name: str
    nz: int
    nx: int
    h: float            # grid spacing [m]
    dt: float           # time step [s]
    nt: int             # number of time levels t_n = n dt, n = 0..nt-1
    W: int              # sponge cells per side
    v_ref: float        # fixed sponge reference speed [m/s] (C10)
    f_peak: float
    src: np.ndarray     # int32 [Ns][2] (iz, ix) interior indices
    rec: np.ndarray     # int32 [nrec][2] (iz, ix)
    wavelet: np.ndarray  # float32 [nt]
    model: np.ndarray   # float32 [nz][nx]: where forward / H·v / gradient are evaluated
    model_true: Optional[np.ndarray]  # float32 [nz][nx]: generates d_obs for gradient tests
    n_probes: int
    probe_fn: Callable[[int], np.ndarray]  # k -> float32 [nz][nx]
    notes: str = ""

    @property
    def ns(self) -> int:
        return int(self.src.shape[0])

    @property
    def nrec(self) -> int:
        return int(self.rec.shape[0])

    def probes(self, ks=None) -> np.ndarray:
        ks = range(self.n_probes) if ks is None else ks
        return np.stack([self.probe_fn(int(k)) for k in ks]).astype(F32)

    def subset(self, shots=None, nt=None) -> "Workload":
        """Same problem restricted to some shots and/or a truncated time axis."""
        w = dataclasses.replace(self)
        if shots is not None:
            w.src = np.ascontiguousarray(self.src[list(shots)])
        if nt is not None:
            w.nt = int(nt)
            w.wavelet = np.ascontiguousarray(self.wavelet[: int(nt)])
        return w


# --------------------------------------------------------------------------- models


def gaussian_probe(shape, seed: int, sigma: float) -> np.ndarray:
    """gaussian_filter(default_rng(seed).standard_normal(shape), sigma) (BJ cfg 0/2, §8(d))."""
    z = np.random.default_rng(seed).standard_normal(shape)
    return _smooth(z, sigma).astype(F32)


def rademacher_probe(shape, seed: int) -> np.ndarray:
    """default_rng(seed).integers(0, 2, shape) * 2 - 1 (BJ cfg 3, §8(d))."""
    return (np.random.default_rng(seed).integers(0, 2, shape) * 2 - 1).astype(F32)


def cosine_probe(shape, kz: float, kx: float) -> np.ndarray:
    """cos(2 pi (kx ix + kz iz)), wavenumbers in cycles per cell (BJ cfg 3, §8(d))."""
    iz = np.arange(shape[0], dtype=np.float64)[:, None]
    ix = np.arange(shape[1], dtype=np.float64)[None, :]
    return np.cos(2.0 * math.pi * (kx * ix + kz * iz)).astype(F32)


def spike_probe(shape, iz: int, ix: int) -> np.ndarray:
    """Unit spike 1.0 at one interior cell (C22)."""
    p = np.zeros(shape, dtype=F32)
    p[iz, ix] = 1.0
    return p


def marmousi_like(nz: int, nx: int, h: float, seed: int = 0, water: float = 60.0,
                  throw_scale: float = 1.0) -> np.ndarray:
    """Seeded layered 'Marmousi-like' model (BJ cfg 2; SURVEY.md §8(d) cfg 2; design choice, not
    the paper's data, which is external: PAPER.md:570-572).

    - water z < `water` m -> 1500 m/s;
    - 11 dipping interfaces z_i(x) = water + (i + U(0.2, 0.8)) (Z - water)/12 + tan(theta_i)(x - X/2),
      theta_i ~ U(-10, 10) deg, sorted in z at every x -> 12 layers;
    - v_l = 1600 + 3900 (l/11)^0.8 + U(-150, 150), clipped to [1500, 5500];
    - 3 normal faults: top x_j ~ U(0.2 X, 0.8 X) at the seafloor, dip 60 deg toward a random side,
      throw U(80, 250) m * throw_scale; the hanging wall is downthrown (layer index evaluated at z - throw).
    Returns float64 [nz][nx].
    """
    rng = np.random.default_rng(seed)
    Z = (nz - 1) * h
    X = (nx - 1) * h
    offs = rng.uniform(0.2, 0.8, 11)
    thetas = np.deg2rad(rng.uniform(-10.0, 10.0, 11))
    vnoise = rng.uniform(-150.0, 150.0, 12)
    fx = rng.uniform(0.2, 0.8, 3) * X
    fdir = rng.choice(np.array([-1.0, 1.0]), 3)
    throws = rng.uniform(80.0, 250.0, 3) * throw_scale

    z = np.arange(nz, dtype=np.float64)[:, None] * h
    x = np.arange(nx, dtype=np.float64)[None, :] * h
    zz = np.broadcast_to(z, (nz, nx)).copy()
    xx = np.broadcast_to(x, (nz, nx))
    # fault displacement: hanging wall (above the dipping plane) is downthrown
    z_eff = zz.copy()
    below = zz >= water
    for j in range(3):
        xf = fx[j] + fdir[j] * (zz - water) / math.tan(math.radians(60.0))
        hanging = (xx - xf) * fdir[j] > 0.0
        z_eff = np.where(hanging & below, z_eff - throws[j], z_eff)
    dz = (Z - water) / 12.0
    iface = np.stack([water + (i + offs[i]) * dz + math.tan(thetas[i]) * (x[0] - X / 2.0)
                      for i in range(11)])          # [11][nx]
    iface = np.sort(iface, axis=0)
    layer = np.zeros((nz, nx), dtype=np.int64)
    for i in range(11):
        layer += (z_eff >= iface[i][None, :]).astype(np.int64)
    vl = np.clip(1600.0 + 3900.0 * (np.arange(12) / 11.0) ** 0.8 + vnoise, 1500.0, 5500.0)
    v = vl[layer]
    v[zz < water] = 1500.0
    return v


# --------------------------------------------------------------------------- configs


def _surface_line(nx: int, iz: int) -> np.ndarray:
    return np.stack([np.full(nx, iz), np.arange(nx)], axis=1).astype(np.int32)


def config(k: int) -> Workload:
    """BASELINE.json configs[k] as concrete seeded inputs."""
    if k == 0:
        nz = nx = 64
        h, dt, nt, f = 10.0, 1e-3, 500, 10.0
        z = np.arange(nz)[:, None] * h
        x = np.arange(nx)[None, :] * h
        base = 1500.0 + 0.25 * z + 0.0 * x
        anomaly = 200.0 * np.exp(-((z - 315.0) ** 2 + (x - 315.0) ** 2) / (2.0 * 60.0 ** 2))
        model = (base + anomaly).astype(F32)
        return Workload(
            name="cfg0", nz=nz, nx=nx, h=h, dt=dt, nt=nt, W=SPONGE_W, v_ref=1857.5, f_peak=f,
            src=np.array([[2, 16], [2, 48]], dtype=np.int32), rec=_surface_line(nx, 2),
            wavelet=ricker(nt, dt, f), model=model, model_true=model,
            n_probes=1, probe_fn=lambda kk: gaussian_probe((64, 64), kk, 3.0),
            notes="H·v at the anomaly model; gradient at m0 = 1500 + 0.25 z with d_obs = F(model)")
    if k == 1:
        nz, nx = 201, 401
        h, dt, nt, f, ns = 10.0, 1e-3, 2000, 8.0, 16
        z = np.arange(nz)[:, None] * h
        zmax = (nz - 1) * h
        model = np.broadcast_to(1500.0 + 2000.0 * (z / zmax) ** 2, (nz, nx)).astype(F32)
        src = np.stack([np.full(ns, 2), _round_half_up((np.arange(ns) + 0.5) * nx / ns)],
                       axis=1).astype(np.int32)
        lat = [(int(_round_half_up((i + 1) * nz / 9)), int(_round_half_up((j + 1) * nx / 9)))
               for i in range(8) for j in range(8)]
        return Workload(
            name="cfg1", nz=nz, nx=nx, h=h, dt=dt, nt=nt, W=SPONGE_W, v_ref=3500.0, f_peak=f,
            src=src, rec=_surface_line(nx, 2), wavelet=ricker(nt, dt, f), model=np.ascontiguousarray(model),
            model_true=None, n_probes=64,
            probe_fn=lambda kk: spike_probe((nz, nx), *lat[kk]),
            notes="64 PSF unit spikes on a regular 8x8 lattice")
    if k in (2, 3):
        nz, nx = 384, 1152
        h, dt, nt, f, ns = 8.0, 0.6e-3, 4000, 5.0, 64
        vt = marmousi_like(nz, nx, h, seed=0)
        m = _smooth(vt, 12.5)
        m[np.arange(nz) * h < 60.0, :] = 1500.0
        src = np.stack([np.full(ns, 2), 18 * np.arange(ns) + 9], axis=1).astype(np.int32)
        if k == 2:
            probe_fn = lambda kk: gaussian_probe((nz, nx), kk, 5.0)
            K, notes = 8, "one gradient + 8 H·v (smoothed N(0,1) directions, sigma = 5 cells)"
        else:
            def probe_fn(kk):
                if kk < 16:
                    return rademacher_probe((nz, nx), kk)
                q = kk - 16
                return cosine_probe((nz, nx), (q // 4 + 1) / 16.0, (q % 4 + 1) / 16.0)
            K, notes = 32, "16 Rademacher + 16 cosine probes (4x4 lattice, 1..4/16 cycles/cell)"
        return Workload(
            name=f"cfg{k}", nz=nz, nx=nx, h=h, dt=dt, nt=nt, W=SPONGE_W, v_ref=5500.0, f_peak=f,
            src=src, rec=_surface_line(nx, 2), wavelet=ricker(nt, dt, f), model=m.astype(F32),
            model_true=vt.astype(F32), n_probes=K, probe_fn=probe_fn, notes=notes)
    if k == 4:
        nz, nx = 2048, 6144
        h, dt, nt, f, ns = 4.0, 0.35e-3, 8000, 10.0, 256
        vt = marmousi_like(nz, nx, h, seed=0, throw_scale=((nz - 1) * h) / (383 * 8.0))
        m = _smooth(vt, 25.0)
        m[np.arange(nz) * h < 60.0, :] = 1500.0
        src = np.stack([np.full(ns, 4), 24 * np.arange(ns) + 12], axis=1).astype(np.int32)
        return Workload(
            name="cfg4", nz=nz, nx=nx, h=h, dt=dt, nt=nt, W=SPONGE_W, v_ref=5500.0, f_peak=f,
            src=src, rec=_surface_line(nx, 4), wavelet=ricker(nt, dt, f), model=m.astype(F32),
            model_true=vt.astype(F32), n_probes=64,
            probe_fn=lambda kk: gaussian_probe((nz, nx), kk, 5.0),
            notes="stress test; in-HBM checkpointing")
    raise ValueError(f"unknown config {k}")


def m0_cfg0() -> np.ndarray:
    """cfg 0 gradient evaluation point: the anomaly removed, 1500 + 0.25 z (§8(d) cfg 0)."""
    z = np.arange(64)[:, None] * 10.0
    return np.broadcast_to(1500.0 + 0.25 * z, (64, 64)).astype(F32).copy()


def custom(nz: int, nx: int, *, h: float = 10.0, dt: float = 1e-3, nt: int = 120, W: int = 20,
           ns: int = 2, nrec: Optional[int] = None, src_depth: int = 2, rec_depth: int = 2,
           f_peak: float = 15.0, v_ref: Optional[float] = None, n_probes: int = 3, seed: int = 7,
           model_kind: str = "smooth", probe_sigma: float = 2.0) -> Workload:
    """A small seeded case (tests): heterogeneous smooth model, surface acquisition, smoothed
    Gaussian probes. Shapes can be chosen to span several CUDA tiles with a ragged tail."""
    rng = np.random.default_rng(seed)
    z = np.arange(nz)[:, None] * h
    x = np.arange(nx)[None, :] * h
    if model_kind == "homogeneous":
        v = np.full((nz, nx), 2000.0)
    elif model_kind == "layered":
        v = marmousi_like(nz, nx, h, seed=seed)
    else:
        v = 1600.0 + 1.2 * z + 150.0 * np.sin(2 * math.pi * x / max(nx * h, 1.0)) \
            + 80.0 * _smooth(rng.standard_normal((nz, nx)), 3.0)
    vmax = float(np.max(v))
    if v_ref is None:
        v_ref = vmax
    sx = _round_half_up((np.arange(ns) + 0.5) * nx / ns)
    src = np.stack([np.full(ns, src_depth), sx], axis=1).astype(np.int32)
    if nrec is None:
        rx = np.arange(nx)
    else:
        rx = _round_half_up(np.linspace(0, nx - 1, nrec))
    rec = np.stack([np.full(len(rx), rec_depth), rx], axis=1).astype(np.int32)
    base_seed = seed * 1000
    return Workload(
        name=f"custom{nz}x{nx}", nz=nz, nx=nx, h=h, dt=dt, nt=nt, W=W, v_ref=float(v_ref),
        f_peak=f_peak, src=src, rec=rec, wavelet=ricker(nt, dt, f_peak), model=v.astype(F32),
        model_true=(v * (1.0 + 0.02 * np.exp(-((z - nz * h / 2) ** 2 + (x - nx * h / 2) ** 2)
                                              / (2 * (0.15 * nz * h) ** 2)))).astype(F32),
        n_probes=n_probes, probe_fn=lambda kk: gaussian_probe((nz, nx), base_seed + kk, probe_sigma),
        notes="custom seeded test case")
