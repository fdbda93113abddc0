"""fp64 oracle of the randomized low-rank generalized eigensolver, SURVEY.md §8(f) N2
(TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md:168-195 (§3.1, Eq. equ:eig): H_d v_i = lambda_i R v_i, lambda_1 >= ... >= lambda_r, V_r^T R V_r = I,
computed matrix-free "via ... randomized SVD" (hIPPYlib's double-pass algorithm). Here:
  Y = R^{-1} H_d Omega;  repeat power_iters times: Q = R-orth(Y), Y = R^{-1} H_d Q;
  Q = R-orth(Y) (Q^T R Q = I);  T = Q^T H_d Q;  T = U diag(lambda) U^T;  V = Q U  (leading r).
R-orth is Cholesky-QR in the R inner product, done twice. R = Gamma_pr^{-1} = (delta I - gamma Delta)^2 applied as
the periodic spectral multiplier (delta + gamma |xi|^2)^2 (SPEC.md:107-115 reading; PAPER.md:73-85 prior).
The random probes Omega are an input (drawn by workloads/, shared with the GPU side).
"""
from __future__ import annotations

import math
from typing import Callable

import numpy as np


def prior_symbol(nz: int, nx: int, h: float, delta: float, gamma: float) -> np.ndarray:
    fz = 2 * math.pi * np.fft.fftfreq(nz, d=h)
    fx = 2 * math.pi * np.fft.fftfreq(nx, d=h)
    return (delta + gamma * (fz[:, None] ** 2 + fx[None, :] ** 2)) ** 2


def prior_apply(V: np.ndarray, h: float, delta: float, gamma: float, power: float = 1.0) -> np.ndarray:
    """R^power V for V [K][nz][nx]: the spectral multiplier (delta + gamma |xi|^2)^(2 power)."""
    s = prior_symbol(V.shape[-2], V.shape[-1], h, delta, gamma) ** power
    return np.real(np.fft.ifft2(s * np.fft.fft2(V)))


def r_orth(Y: np.ndarray, RY: Callable[[np.ndarray], np.ndarray]) -> np.ndarray:
    """Cholesky-QR in the R inner product, twice: returns Q [K][N] with Q R Q^T = I."""
    for _ in range(2):
        G = Y @ RY(Y).T
        G = 0.5 * (G + G.T)
        L = np.linalg.cholesky(G)
        Y = np.linalg.solve(L, Y)
    return Y


def randomized_gen_eig(Hd, Omega, r, power_iters, h, delta, gamma):
    """Hd: [K][nz][nx] -> [K][nz][nx]; Omega [K][nz][nx]. Returns (lambda [r] descending, V [r][nz][nx])."""
    K, nz, nx = Omega.shape
    N = nz * nx
    flat = lambda A: A.reshape(A.shape[0], N)
    grid = lambda A: A.reshape(A.shape[0], nz, nx)
    RY = lambda A: flat(prior_apply(grid(A), h, delta, gamma, 1.0))
    Rinv = lambda A: prior_apply(A, h, delta, gamma, -1.0)
    Y = flat(Rinv(Hd(np.asarray(Omega, dtype=np.float64))))
    for _ in range(power_iters):
        Q = r_orth(Y, RY)
        Y = flat(Rinv(Hd(grid(Q))))
    Q = r_orth(Y, RY)
    T = Q @ flat(Hd(grid(Q))).T
    T = 0.5 * (T + T.T)
    lam, U = np.linalg.eigh(T)
    order = np.argsort(lam)[::-1][:r]
    return lam[order], grid(U[:, order].T @ Q)
