"""fp64 oracle of PSF+ (the paper's unified method), SURVEY.md §8(f) N3 (TEST INFRASTRUCTURE ONLY — see
oracle/__init__.py).

PAPER.md:330-357 (§3.6, Eq. equ:psfplus):
 (i)   S_psf = W S~[I_r, :]                                   (PSF weights times the computed symbol rows)
 (ii)  SVD of S~[I_r, :] -> basis B of its row space (leading `rank` right singular vectors); S_psf = A_0 B
 (iii) A = argmin ||A B[:, I_c] - S~[:, I_c]||_F^2 + alpha ||A - A_0||_F^2, alpha = ||B[:, I_c]||_F^2 / ||B||_F^2
       -> closed form A = (S~[:, I_c] B[:, I_c]^H + alpha A_0)(B[:, I_c] B[:, I_c]^H + alpha I)^{-1}
 The low-rank symbol is s(x, xi) ~ sum_k A[x, k] B[k, xi] (Eq. equ:lr_symbol_matrix), applied as
 out = Re sum_k A[:, k] . IDFT(B[k] . DFT(v)).
Discrete reading (DESIGN.md §3 R-psfplus): rows [nr][N] complex (the N1 symbol rows), W [nr][N] real (N1 hat
weights), columns S~[:, I_c] [nc][N] complex (N1 symbol columns) at DFT indices I_c = (kz, kx).
"""
from __future__ import annotations

import numpy as np


def psf_plus(rows, W, cols, col_idx, rank, alpha=None):
    """Returns (A [N][rank] complex, B [rank][N] complex, alpha). Arrays may be [k][nz][nx] shaped."""
    nr = rows.shape[0]
    shape = rows.shape[1:]
    N = int(np.prod(shape))
    Sr = np.asarray(rows, dtype=np.complex128).reshape(nr, N)
    Wm = np.asarray(W, dtype=np.float64).reshape(nr, N).T                  # N x nr
    Sc = np.asarray(cols, dtype=np.complex128).reshape(len(cols), N).T     # N x nc
    nx = shape[-1]
    ic = [kz * nx + kx for kz, kx in col_idx]
    U, sig, Vh = np.linalg.svd(Sr, full_matrices=False)                    # (ii)
    B = Vh[:rank]                                                          # rank x N, orthonormal rows
    A0 = Wm @ (U[:, :rank] * sig[:rank])                                   # S_psf = W Sr = A0 B (+ tail)
    Bc = B[:, ic]
    if alpha is None:
        alpha = float(np.linalg.norm(Bc) ** 2 / np.linalg.norm(B) ** 2)
    M = Bc @ Bc.conj().T + alpha * np.eye(rank)                             # (iii)
    A = (Sc @ Bc.conj().T + alpha * A0) @ np.linalg.inv(M)
    return A, B, alpha


def apply(A, B, v):
    """out = Re sum_k A[:, k] . IDFT(B[k] . DFT(v)) for v [nz][nx]."""
    nz, nx = v.shape
    vh = np.fft.fft2(np.asarray(v, dtype=np.float64))
    out = np.zeros((nz, nx))
    for k in range(B.shape[0]):
        out += np.real(A[:, k].reshape(nz, nx) * np.fft.ifft2(B[k].reshape(nz, nx) * vh))
    return out
