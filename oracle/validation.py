"""Validation-battery statistics -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may use this module;
the product path (libp2s) never does.

The paper builds the sampler so that the Zernike coefficient fields reproduce the spatial
auto-correlation of the coefficients between pixels: homogeneous kernels A_jj(s)
(P:234-238), mixed per pixel by L (block-diagonal model, Eq.10), so that

    E[a_j(x) a_j(x + s)] = sum_k L_jk^2 c_k(s),

with c_k the unit-variance kernel of mode k that the sampler actually realises on the
periodic P x Q grid, c_k = IDFT(S_k) / (P Q) with S_k the clamped, renormalised PSD
(reading Q7).  The tilt statistics follow from modes 2 and 3: the differential tilt
variance along a lag is D_t(s) = 2 (A_22(0) - A_22(s)).
"""
from __future__ import annotations

import numpy as np


def empirical_autocorr(fields: np.ndarray, L: int) -> np.ndarray:
    """Plain definition of the estimator the GPU computes (periodic lags):

        R[j, 0, l] = mean_{f,y,x} a[f, j, y, x] a[f, j, y, (x + l) mod W]
        R[j, 1, l] = mean_{f,y,x} a[f, j, y, x] a[f, j, (y + l) mod H, x]

    fields: [F][Z][H][W].  Returns float64 [Z][2][L]."""
    a = np.asarray(fields, dtype=np.float64)
    F, Z, H, W = a.shape
    out = np.empty((Z, 2, L))
    for l in range(L):
        out[:, 0, l] = (a * np.roll(a, -l, axis=3)).mean(axis=(0, 2, 3))
        out[:, 1, l] = (a * np.roll(a, -l, axis=2)).mean(axis=(0, 2, 3))
    return out


def realised_kernels(sqrtS: np.ndarray, L: int) -> np.ndarray:
    """c_k along the x and y axes at lags 0..L-1 for the unit-variance sampler tables:
    c_k = IDFT(S_k)/(P Q), S_k = sqrtS_k^2.  sqrtS [Z-1][P][Q] (modes 2..Z).
    Returns float64 [Z-1][2][L]."""
    S = np.asarray(sqrtS, dtype=np.float64) ** 2
    c = np.real(np.fft.ifft2(S, axes=(-2, -1)))  # numpy ifft2 includes the 1/(P Q)
    return np.stack([c[:, 0, :L], c[:, :L, 0]], axis=1)


def model_autocorr(chol: np.ndarray, kernels: np.ndarray) -> np.ndarray:
    """Eq.10 (block-diagonal model): R_j(l) = sum_k L_jk^2 c_k(l).

    chol: L with L L^T = A_0 ([Z][Z] with a zero piston row/column, as
    optics.noll_cholesky returns, or its [Z-1][Z-1] block of modes 2..Z); kernels:
    [Z-1][2][L].  Returns [Z][2][L] with a zero piston row (slot 0 = Noll j = 1),
    matching the p2s_sample_zernike plane order."""
    Lm = np.asarray(chol, dtype=np.float64)
    if Lm.shape[0] == kernels.shape[0] + 1:
        Lm = Lm[1:, 1:]
    n = Lm.shape[0]
    out = np.zeros((n + 1,) + kernels.shape[1:])
    out[1:] = np.einsum("jk,kdl->jdl", Lm ** 2, kernels)
    return out


def differential_tilt_variance(R: np.ndarray) -> np.ndarray:
    """D_t(l) = 2 (R_t(0) - R_t(l)) for the two tilt modes (Noll 2, 3).
    R: [Z][2][L] auto-correlations.  Returns [2 modes][2 dirs][L]."""
    t = np.asarray(R)[1:3]
    return 2.0 * (t[:, :, :1] - t)
