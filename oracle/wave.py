"""fp64 numpy oracle of the discrete FWI operators (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Follows SURVEY.md §8(c) O1-O11 step by step, in the paper's notation where it has one:
- forward map f: m -> d, "values of u(x,t) at receiver locations"     PAPER.md:49 (§2)
- wave equation (1/m^2) u_tt - lap u = s(t) delta(x - x_s)            PAPER.md:44-47 (Eq. equ:pde),
  read as u_tt = v^2 lap u + f (BASELINE.json cfg 0; reading C1)
- gradient  F* Gamma^-1 (f(m) - d), F = Born, F* = migration         PAPER.md:108-112 (Eq. equ:grad)
- misfit Hessian H_d = F*F ("normal operator"), accessed via matrix-vector products
  by adjoint methods, "two wave equations per source"                PAPER.md:9, 157-164 (§3)
The discretisation itself is not in the paper (it is "proprietary"); every
discrete choice is the DESIGN.md §3 reading (C1-C24 of SURVEY.md §8(c)).

Notation: padded grid Nz x Nx = (nz + 2W) x (nx + 2W); padded index (I, J) = (iz + W, ix + W).
P restricts padded -> interior, P^T zero-extends. Everything is float64.
"""
from __future__ import annotations

import math
from typing import Callable, List, Optional, Sequence

import numpy as np

F64 = np.float64

# O3: standard 8th-order central second-derivative weights a_0..a_4.
A8 = (-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0)
RING = 4  # stencil radius = width of the boundary ring saved in BOUNDARY mode


# ----------------------------------------------------------------------------- O1 - O5


def pad_edge(v: np.ndarray, W: int) -> np.ndarray:
    """O1: v_pad = edge-replicate(v, W). Sponge speeds are not parameters (C13)."""
    return np.pad(np.asarray(v, dtype=F64), W, mode="edge")


def sponge_c(nz: int, nx: int, W: int, h: float, dt: float, v_ref: float) -> np.ndarray:
    """O2: c = eta dt / 2 with eta = eta_max [(d_z/W)^2 + (d_x/W)^2],
    d_z(I) = max(0, W - I, I - (W + nz - 1)) (likewise d_x), eta_max = 3 v_ref ln(10^3) / (2 W h).
    Zero on the interior (C10)."""
    Nz, Nx = nz + 2 * W, nx + 2 * W
    I = np.arange(Nz)
    J = np.arange(Nx)
    dz = np.maximum(0, np.maximum(W - I, I - (W + nz - 1))).astype(F64)
    dx = np.maximum(0, np.maximum(W - J, J - (W + nx - 1))).astype(F64)
    if W == 0:
        return np.zeros((Nz, Nx))
    eta_max = 3.0 * v_ref * math.log(1000.0) / (2.0 * W * h)
    eta = eta_max * ((dz / W) ** 2)[:, None] + eta_max * ((dx / W) ** 2)[None, :]
    return eta * dt / 2.0


def laplacian(u: np.ndarray, h: float) -> np.ndarray:
    """O3: (Lu)[I,J] = h^-2 [2 a0 u[I,J] + sum_{k=1..4} a_k (u[I,J+-k] + u[I+-k,J])],
    u = 0 outside the padded grid (so L is symmetric)."""
    out = 2.0 * A8[0] * u
    for k in range(1, 5):
        a = A8[k]
        out[:, k:] += a * u[:, :-k]
        out[:, :-k] += a * u[:, k:]
        out[k:, :] += a * u[:-k, :]
        out[:-k, :] += a * u[k:, :]
    return out / (h * h)


class Problem:
    """The discrete operators of one model / acquisition (O1-O5)."""

    def __init__(self, wl, model: Optional[np.ndarray] = None):
        self.wl = wl
        self.nz, self.nx, self.W = wl.nz, wl.nx, wl.W
        self.h, self.dt, self.nt = float(wl.h), float(wl.dt), int(wl.nt)
        m = wl.model if model is None else model
        self.m = np.asarray(m, dtype=F64)                     # C17: fp32 inputs -> fp64
        self.v = pad_edge(self.m, self.W)                     # O1
        self.w = self.dt ** 2 * self.v ** 2                   # O2
        self.c = sponge_c(self.nz, self.nx, self.W, self.h, self.dt, float(wl.v_ref))
        self.src = np.asarray(wl.src, dtype=np.int64) + self.W  # padded (I, J)
        self.rec = np.asarray(wl.rec, dtype=np.int64) + self.W
        self.wavelet = np.asarray(wl.wavelet, dtype=F64)[: self.nt]
        self.shape = self.v.shape

    # -- helpers (plain restatements of P, P^T, R, R^T)
    def P(self, a: np.ndarray) -> np.ndarray:
        W = self.W
        return a[W:W + self.nz, W:W + self.nx]

    def PT(self, a: np.ndarray) -> np.ndarray:
        out = np.zeros(self.shape)
        W = self.W
        out[W:W + self.nz, W:W + self.nx] = a
        return out

    def sample(self, u: np.ndarray) -> np.ndarray:
        """R: values at the receiver nodes (C8)."""
        return u[self.rec[:, 0], self.rec[:, 1]]

    def RT(self, r: np.ndarray) -> np.ndarray:
        """R^T: scatter-add receiver values into their cells."""
        out = np.zeros(self.shape)
        np.add.at(out, (self.rec[:, 0], self.rec[:, 1]), r)
        return out

    def force(self, shot: int, n: int) -> np.ndarray:
        """O5: f^n = s[n] / h^2 at the source cell, 0 elsewhere (C7)."""
        f = np.zeros(self.shape)
        I, J = self.src[shot]
        f[I, J] = self.wavelet[n] / (self.h * self.h)
        return f

    def step(self, un: np.ndarray, unm1: np.ndarray, rhs: np.ndarray) -> np.ndarray:
        """One leapfrog step with centred damping (C4):
        u^{n+1} = [2 u^n - (1 - c) u^{n-1} + w L u^n + rhs] / (1 + c)."""
        return (2.0 * un - (1.0 - self.c) * unm1 + self.w * laplacian(un, self.h) + rhs) / (1.0 + self.c)

    # ------------------------------------------------------------------------- O6

    def forward(self, shot: int, keep_history: bool = False):
        """O6: u^{-1} = u^0 = 0; for n = 0..nt-2:
        u^{n+1} = [2u^n - (1-c)u^{n-1} + w L u^n + dt^2 f^n] / (1+c); d[n, r] = u^n[rec_r].
        Returns d [nt][nrec] (and the list u^0..u^{nt-1} if keep_history)."""
        nt = self.nt
        d = np.zeros((nt, len(self.rec)))
        um1 = np.zeros(self.shape)
        u = np.zeros(self.shape)
        hist = [u] if keep_history else None
        for n in range(nt - 1):
            up1 = self.step(u, um1, self.dt ** 2 * self.force(shot, n))
            um1, u = u, up1
            d[n + 1] = self.sample(u)
            if keep_history:
                hist.append(u)
        return (d, hist) if keep_history else d

    # ------------------------------------------------------------------------- O7

    def born(self, shot: int, dv: Sequence[np.ndarray]) -> np.ndarray:
        """O7 (J): q = 2 dt^2 v_pad P^T dv; du^{-1} = du^0 = 0;
        du^{n+1} = [2du^n - (1-c)du^{n-1} + w L du^n + q L u^n] / (1+c); (J dv)[n, r] = du^n[rec_r].
        dv: K interior directions. Returns [K][nt][nrec]."""
        nt = self.nt
        K = len(dv)
        q = [2.0 * self.dt ** 2 * self.v * self.PT(np.asarray(x, dtype=F64)) for x in dv]
        out = np.zeros((K, nt, len(self.rec)))
        um1 = np.zeros(self.shape)
        u = np.zeros(self.shape)
        dum1 = [np.zeros(self.shape) for _ in range(K)]
        du = [np.zeros(self.shape) for _ in range(K)]
        for n in range(nt - 1):
            Lu = laplacian(u, self.h)
            for k in range(K):
                dup1 = self.step(du[k], dum1[k], q[k] * Lu)
                dum1[k], du[k] = du[k], dup1
                out[k, n + 1] = self.sample(du[k])
            up1 = self.step(u, um1, self.dt ** 2 * self.force(shot, n))
            um1, u = u, up1
        return out

    # ------------------------------------------------------------------------- O8 + O9

    def adjoint_image(self, rho: np.ndarray, history: Callable[[int], np.ndarray]) -> np.ndarray:
        """O8 + O9 (J^T): lambda^{nt} = lambda^{nt+1} = 0; for j = nt-1 .. 1:
        lambda^j = [2 lambda^{j+1} - (1-c) lambda^{j+2} + w L lambda^{j+1} + v^2 R^T rho[j]] / (1+c);
        J^T rho = P[ sum_{n=1}^{nt-2} (2 dt^2 / v) (L u^n) lambda^{n+1} ].
        rho: [nt][nrec] (rho[0] unused). history(n) returns u^n, called for n = nt-2 .. 1
        in decreasing order. Returns the interior image [nz][nx]."""
        nt = self.nt
        lam_p2 = np.zeros(self.shape)  # lambda^{j+2}
        lam_p1 = np.zeros(self.shape)  # lambda^{j+1}
        img = np.zeros(self.shape)
        for j in range(nt - 1, 0, -1):
            if j <= nt - 2:  # imaging term n = j pairs L u^j with lambda^{j+1}
                img += (2.0 * self.dt ** 2 / self.v) * laplacian(history(j), self.h) * lam_p1
            lam = self.step(lam_p1, lam_p2, self.v ** 2 * self.RT(rho[j]))
            lam_p2, lam_p1 = lam_p1, lam
        return self.P(img)

    # ------------------------------------------------------------------------- storage (a4)

    def history(self, shot: int, mode: str = "full", ckpt: int = 0):
        """Forward-history store for the reverse pass (not in the paper).
        Returns (d, history_fn). All three modes give u^n exactly in exact arithmetic (P8)."""
        if mode == "full":
            d, hist = self.forward(shot, keep_history=True)
            return d, (lambda n: hist[n])
        if mode == "checkpoint":
            return self._checkpoint_history(shot, ckpt or int(round(math.sqrt(self.nt))))
        if mode == "boundary":
            return self._boundary_history(shot)
        raise ValueError(mode)

    def _checkpoint_history(self, shot: int, k: int):
        """CHECKPOINT: keep (u^n, u^{n-1}) at n = 0, k, 2k, ...; replay a segment forward when
        the reverse pass first needs one of its levels."""
        nt = self.nt
        d = np.zeros((nt, len(self.rec)))
        ck = {}
        um1 = np.zeros(self.shape)
        u = np.zeros(self.shape)
        for n in range(nt - 1):
            if n % k == 0:
                ck[n] = (u.copy(), um1.copy())
            up1 = self.step(u, um1, self.dt ** 2 * self.force(shot, n))
            um1, u = u, up1
            d[n + 1] = self.sample(u)
        cache = {}

        def get(n: int) -> np.ndarray:
            base = (n // k) * k
            if base not in cache:
                cache.clear()
                a, b = ck[base]                     # u^base, u^{base-1}
                seg = {base: a}
                for m in range(base, min(base + k - 1, nt - 1)):  # -> u^{base+1} .. u^{base+k-1}
                    nxt = self.step(a, b, self.dt ** 2 * self.force(shot, m))
                    b, a = a, nxt
                    seg[m + 1] = a
                cache[base] = seg
            return cache[base][n]

        return d, get

    def _boundary_history(self, shot: int):
        """BOUNDARY: save the RING-cell ring of sponge cells around the interior at every level
        plus the last two levels; rebuild u^{n-1} = 2u^n - u^{n+1} + w L u^n + dt^2 f^n on the
        interior (c = 0 there) and restore the ring from the store."""
        nt, W, nz, nx = self.nt, self.W, self.nz, self.nx
        assert W >= RING
        lo_z, hi_z, lo_x, hi_x = W - RING, W + nz + RING, W - RING, W + nx + RING
        ring_mask = np.zeros(self.shape, dtype=bool)
        ring_mask[lo_z:hi_z, lo_x:hi_x] = True
        ring_mask[W:W + nz, W:W + nx] = False
        d = np.zeros((nt, len(self.rec)))
        rings = [None] * nt
        um1 = np.zeros(self.shape)
        u = np.zeros(self.shape)
        rings[0] = u[ring_mask].copy()
        for n in range(nt - 1):
            up1 = self.step(u, um1, self.dt ** 2 * self.force(shot, n))
            um1, u = u, up1
            d[n + 1] = self.sample(u)
            rings[n + 1] = u[ring_mask].copy()
        state = {"n": nt - 1, "u": u.copy(), "up1": None, "um1": um1.copy()}
        interior = np.zeros(self.shape, dtype=bool)
        interior[W:W + nz, W:W + nx] = True

        def rebuild(u_n, u_np1, n):
            """u^{n-1} from u^n, u^{n+1} on the interior + stored ring."""
            prev = np.zeros(self.shape)
            full = 2.0 * u_n - u_np1 + self.w * laplacian(u_n, self.h) + self.dt ** 2 * self.force(shot, n)
            prev[interior] = full[interior]
            prev[ring_mask] = rings[n - 1]
            return prev

        def get(n: int) -> np.ndarray:
            # levels are requested in decreasing order starting at nt-2
            while state["n"] > n:
                cur = state["n"]
                if cur == nt - 1:
                    newer, older = state["u"], state["um1"]  # u^{nt-1}, u^{nt-2}: stored levels
                    state.update(n=nt - 2, u=older, up1=newer)
                    continue
                prev = rebuild(state["u"], state["up1"], cur)
                state.update(n=cur - 1, u=prev, up1=state["u"])
            return state["u"]

        return d, get

    # ------------------------------------------------------------------------- O10 / O11

    def hessvec_shot(self, shot: int, V: Sequence[np.ndarray], mode: str = "full", ckpt: int = 0):
        """H_s [v_1..v_K] = J_s^T (J_s v_k) for one shot, background shared (O10, O11)."""
        dd = self.born(shot, V)
        _, hist = self.history(shot, mode, ckpt)
        return np.stack([self.adjoint_image(dd[k], hist) for k in range(len(V))])

    def hessvec(self, V: Sequence[np.ndarray], shots: Optional[Sequence[int]] = None,
                mode: str = "full", ckpt: int = 0) -> np.ndarray:
        """O10: H v = sum_s J_s^T (J_s v). V: [K][nz][nx]. Returns [K][nz][nx]."""
        shots = range(len(self.src)) if shots is None else shots
        out = np.zeros((len(V), self.nz, self.nx))
        for s in shots:
            out += self.hessvec_shot(s, V, mode, ckpt)
        return out

    def forward_all(self, shots: Optional[Sequence[int]] = None) -> np.ndarray:
        shots = range(len(self.src)) if shots is None else shots
        return np.stack([self.forward(s) for s in shots])

    def gradient(self, d_obs: np.ndarray, shots: Optional[Sequence[int]] = None,
                 mode: str = "full", ckpt: int = 0):
        """O10: phi = 1/2 sum_s sum_{n,r} (d_s - d_obs,s)^2 (Gamma_noise = I, C11);
        g = sum_s J_s^T (d_s - d_obs,s) (Eq. equ:grad, misfit term).
        d_obs: [len(shots)][nt][nrec]. Returns (phi, g [nz][nx])."""
        shots = list(range(len(self.src))) if shots is None else list(shots)
        phi = 0.0
        g = np.zeros((self.nz, self.nx))
        for i, s in enumerate(shots):
            d, hist = self.history(s, mode, ckpt)
            res = d - np.asarray(d_obs[i], dtype=F64)
            phi += 0.5 * float(np.sum(res * res))
            g += self.adjoint_image(res, hist)
        return phi, g
