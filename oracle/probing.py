"""fp64 oracle of probe -> symbol assembly, SURVEY.md §8(f) N1 (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PSF method (§3.2; §3.5):
  p_k(x) = H_d delta_{x_k}(x_k + x)                          (PSF centred at x_k, Eq. after)
  s(x_k, xi) = (2 pi)^2 conj(p^_k(xi))                        (symbol row, §3.5)
  s(x, xi) ~ sum_k w_k(x) s(x_k, xi)                          (PSF method as a PsiDO, §3.5)
PDO method (§3.4; Appendix A):
  s(., xi) = H_d phi_xi / phi_xi,  phi_xi = e^{i x.xi}        (Eq. equ:symbol)
  v_p = sum_k phi_{xi_k}                                       (Eq. equ:pdo-vp; antipodal pairs -> real)
  w_k(rho, theta) = (rho / rho0) w^circle_k(theta)             (Eq. equ:pdo-w; angular FFT interpolation)
  s(x, xi) ~ sum_k s(x, xi_k) w_k(xi)                          (Eq. equ:pdo-symbol)

Discrete readings (R-probe): transforms are the unnormalised DFT / 1/N IDFT of oracle/psido.py, on
the interior grid, periodic; with a unit spike probe (C22) the (2 pi)^2 and cell-area factors of the continuous
convention cancel, so the symbol row is conj(DFT(p_k)) with p_k the window of the response around x_k rolled to
the origin (hard square window of half-width `radius`); PSF weights are bilinear hats on the sample lattice with
constant extension outside it (a partition of unity everywhere); PDO masks are discs of radius `mask_radius`
frequency cells with a 2-cell raised-cosine roll-off; angular weights use the even-r trigonometric (Dirichlet)
interpolation kernel t(phi) = sin(r phi / 2) cot(phi / 2) / r.
"""
from __future__ import annotations

import math
from typing import Sequence, Tuple

import numpy as np


# ----------------------------------------------------------------------------------------------- PSF


def delta_probes(nz: int, nx: int, points: Sequence[Tuple[int, int]], batch_of: Sequence[int]) -> np.ndarray:
    """One probe per batch: the sum of unit spikes (C22) at the batch's points."""
    nb = max(batch_of) + 1
    P = np.zeros((nb, nz, nx))
    for (iz, ix), b in zip(points, batch_of):
        P[b, iz, ix] += 1.0
    return P


def extract_psfs(responses: np.ndarray, points, batch_of, radius: int) -> np.ndarray:
    """p_k[z, x] = R_b[(iz_k + z) mod nz, (ix_k + x) mod nx] for |z|, |x| <= radius (signed offsets), else 0."""
    _, nz, nx = responses.shape
    out = np.zeros((len(points), nz, nx))
    for k, ((iz, ix), b) in enumerate(zip(points, batch_of)):
        for dz in range(-radius, radius + 1):
            for dx in range(-radius, radius + 1):
                out[k, dz % nz, dx % nx] = responses[b, (iz + dz) % nz, (ix + dx) % nx]
    return out


def psf_symbol_rows(psfs: np.ndarray) -> np.ndarray:
    """s(x_k, xi) = conj(DFT(p_k))(xi) (the paper's (2 pi)^2 conj(p^_k) in the discrete unit-spike convention)."""
    return np.conj(np.fft.fft2(psfs))


def _hat_1d(coords: Sequence[float], n: int) -> np.ndarray:
    """Piecewise-linear interpolation basis on sorted lattice coordinates, constant outside: [len(coords)][n]."""
    c = np.asarray(coords, dtype=np.float64)
    x = np.arange(n, dtype=np.float64)
    H = np.zeros((len(c), n))
    for j in range(len(c)):
        e = np.zeros(len(c))
        e[j] = 1.0
        H[j] = np.interp(x, c, e)          # numpy.interp extends with the end values
    return H


def psf_weights(nz: int, nx: int, lat_z: Sequence[int], lat_x: Sequence[int]) -> np.ndarray:
    """Bilinear hat weights w_{ij}(z, x) = hat_i(z) hat_j(x) for the lattice points (lat_z[i], lat_x[j]),
    ordered k = i * len(lat_x) + j. Partition of unity, w_k(x_j) = delta_kj."""
    hz = _hat_1d(lat_z, nz)
    hx = _hat_1d(lat_x, nx)
    return np.einsum("iz,jx->ijzx", hz, hx).reshape(len(lat_z) * len(lat_x), nz, nx)


# ----------------------------------------------------------------------------------------------- PDO


def freq_index_to_xi(kz: int, kx: int, nz: int, nx: int, h: float) -> Tuple[float, float]:
    """Angular frequency (xi_z, xi_x) of DFT index (kz, kx), unshifted order, range [-n/2, n/2)."""
    fz = kz - nz if kz >= (nz + 1) // 2 else kz
    fx = kx - nx if kx >= (nx + 1) // 2 else kx
    return 2 * math.pi * fz / (nz * h), 2 * math.pi * fx / (nx * h)


def pdo_plan(nz: int, nx: int, h: float, rho0: float, r: int = 8):
    """r equally spaced angles theta_k = 2 pi k / r (k = 1..r), xi_k = rho0 (cos theta_k, sin theta_k) as
    (xi_x, xi_z), snapped to the nearest DFT index; antipodal pairs are exact negatives."""
    assert r % 2 == 0
    idx = []
    for k in range(1, r // 2 + 1):
        th = 2 * math.pi * k / r
        fx = rho0 * math.cos(th) * nx * h / (2 * math.pi)
        fz = rho0 * math.sin(th) * nz * h / (2 * math.pi)
        idx.append((int(round(fz)), int(round(fx))))
    full = []
    for k in range(1, r + 1):
        if k <= r // 2:
            fz, fx = idx[k - 1]
        else:
            fz, fx = idx[k - r // 2 - 1]
            fz, fx = -fz, -fx
        full.append((fz % nz, fx % nx))
    thetas = [2 * math.pi * k / r for k in range(1, r + 1)]
    return full, thetas


def sinusoid_probe(nz: int, nx: int, freq_idx) -> np.ndarray:
    """v_p(x) = sum_k exp(i x . xi_k) on grid indices: exp(2 pi i (kz iz / nz + kx ix / nx)); real part."""
    iz = np.arange(nz)[:, None]
    ix = np.arange(nx)[None, :]
    v = np.zeros((nz, nx), dtype=complex)
    for kz, kx in freq_idx:
        v += np.exp(2j * math.pi * (kz * iz / nz + kx * ix / nx))
    return v


def disc_mask(nz: int, nx: int, kz: int, kx: int, radius: float, rolloff: float = 2.0) -> np.ndarray:
    """1 within `radius` frequency cells of index (kz, kx) (periodic index distance), raised-cosine to 0 over
    `rolloff` cells."""
    dz = (np.arange(nz)[:, None] - kz + nz // 2) % nz - nz // 2
    dx = (np.arange(nx)[None, :] - kx + nx // 2) % nx - nx // 2
    d = np.sqrt(dz.astype(np.float64) ** 2 + dx.astype(np.float64) ** 2)
    m = np.where(d <= radius, 1.0, 0.0)
    band = (d > radius) & (d < radius + rolloff)
    m[band] = 0.5 * (1.0 + np.cos(math.pi * (d[band] - radius) / rolloff))
    return m


def extract_symbol_columns(response: np.ndarray, freq_idx, mask_radius: float) -> np.ndarray:
    """col_k = IDFT(M_k . DFT(R)) / phi_{xi_k} (Eq. equ:symbol after spectral separation)."""
    nz, nx = response.shape
    Rh = np.fft.fft2(response)
    iz = np.arange(nz)[:, None]
    ix = np.arange(nx)[None, :]
    cols = np.zeros((len(freq_idx), nz, nx), dtype=complex)
    for k, (kz, kx) in enumerate(freq_idx):
        part = np.fft.ifft2(disc_mask(nz, nx, kz, kx, mask_radius) * Rh)
        phi = np.exp(2j * math.pi * (kz * iz / nz + kx * ix / nx))
        cols[k] = part / phi
    return cols


def dirichlet_kernel(phi: np.ndarray, r: int) -> np.ndarray:
    """Even-r trigonometric interpolation basis t(phi) = sin(r phi / 2) cot(phi / 2) / r, t(0) = 1."""
    phi = np.asarray(phi, dtype=np.float64)
    s = np.sin(phi / 2.0)
    small = np.abs(s) < 1e-12
    out = np.empty_like(phi)
    out[~small] = np.sin(r * phi[~small] / 2.0) * np.cos(phi[~small] / 2.0) / (r * s[~small])
    out[small] = np.cos(r * phi[small] / 2.0)          # limit at phi = 2 pi m: cos(r pi m) = 1 for even r
    return out


def pdo_weights(nz: int, nx: int, h: float, rho0: float, thetas: Sequence[float]) -> np.ndarray:
    """w_k(xi) = (|xi| / rho0) t(theta(xi) - theta_k) on the DFT frequency grid; theta = atan2(xi_z, xi_x)."""
    r = len(thetas)
    fz = np.fft.fftfreq(nz, d=h) * 2 * math.pi
    fx = np.fft.fftfreq(nx, d=h) * 2 * math.pi
    XZ, XX = np.meshgrid(fz, fx, indexing="ij")
    rho = np.sqrt(XZ ** 2 + XX ** 2)
    th = np.arctan2(XZ, XX)
    return np.stack([(rho / rho0) * dirichlet_kernel(th - t, r) for t in thetas])
