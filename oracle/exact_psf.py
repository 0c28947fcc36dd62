"""Exact-PSF path (partial) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may use this module.

Eq.2: h_x(u) = |F{P(xi) e^{-j phi_x(xi)}}|^2 with the pupil phase
phi_x = sum_j a_j(x) Z_j on the unit disk, and Eq.1: the image is the gather of
every output pixel's own PSF with the input neighbourhood (only the centre pixel's PSF is
used for I(x)).  The paper leaves the sampling constants out ("withholding some constants
that determine the size of the PSF"); reading Q24:

* pupil: PUPIL_D = 32 samples across the aperture diameter (sample centres, rho <= 1),
  zero-padded to an FFT_N = 64 grid: padding 2, so one PSF pixel is lambda/(2D), the
  Nyquist IFOV of the image grid (reading Q5) -- a pure tilt a_2 then moves the PSF by
  4 a_2 / pi pixels, the warp constant of reading Q12;
* forward DFT (e^{-2 pi i}), |.|^2, the T x T window of displacements u in [-T/2, T/2]^2
  taken as h(u) = I[u mod N] (a positive x tilt puts the peak at u_x = -kappa a_2, i.e.
  the content moves to +kappa a_2 exactly as the warp's gather I(x + d)), normalised to
  unit sum;
* the render convolves like the blur (true convolution, whole-sample mirror boundary):
  out_c(x) = sum_u h_x(u) I_c(x - u).
"""
from __future__ import annotations

import numpy as np

from .optics import zernike
from .pipeline import reflect_index

PUPIL_D = 32
FFT_N = 64


def pupil_grid(Dp: int = PUPIL_D):
    """(rho, theta, mask) at the Dp x Dp sample centres, rho in units of the radius,
    theta from the column (x) axis (reading Q4)."""
    c = (np.arange(Dp) + 0.5 - Dp / 2.0) / (Dp / 2.0)
    Y, X = np.meshgrid(c, c, indexing="ij")
    rho = np.hypot(X, Y)
    return rho, np.arctan2(Y, X), rho <= 1.0


def pupil_phase(a: np.ndarray, Dp: int = PUPIL_D, include_tilt: bool = True) -> np.ndarray:
    """phi = sum_{j >= 2} a_j Z_j on the pupil samples (a: Noll 1..Z, a[0] = piston)."""
    rho, theta, mask = pupil_grid(Dp)
    phi = np.zeros((Dp, Dp))
    for j in range(2, len(a) + 1):
        if not include_tilt and j in (2, 3):
            continue
        phi += a[j - 1] * zernike(j, rho, theta)
    return phi * mask


def exact_psf(a: np.ndarray, T: int, include_tilt: bool = True, Dp: int = PUPIL_D, N: int = FFT_N) -> np.ndarray:
    """Eq.2 on the tap grid: [T][T], tap (c + uy, c + ux) = h(uy, ux), unit sum."""
    rho, theta, mask = pupil_grid(Dp)
    field = np.zeros((N, N), dtype=np.complex128)
    field[:Dp, :Dp] = mask * np.exp(-1j * pupil_phase(a, Dp, include_tilt))
    inten = np.abs(np.fft.fft2(field)) ** 2
    c = T // 2
    u = np.arange(-c, c + 1) % N
    h = inten[np.ix_(u, u)]
    return h / h.sum()


def render_exact(img: np.ndarray, a: np.ndarray, T: int, include_tilt: bool = True) -> np.ndarray:
    """Eq.1 gather: img [C][H][W], a [Z][H][W] -> [C][H][W]; each pixel uses its own PSF."""
    C, H, W = img.shape
    c = T // 2
    u = np.arange(T) - c
    out = np.empty((C, H, W))
    for y in range(H):
        py = reflect_index(y - u, H)
        for x in range(W):
            h = exact_psf(a[:, y, x], T, include_tilt)
            px = reflect_index(x - u, W)
            patch = img[:, py[:, None], px[None, :]]
            out[:, y, x] = np.einsum("tu,ctu->c", h, patch)
    return out


def pca_basis(psfs: np.ndarray, M: int):
    """Eq.7: mean PSF + the M leading principal components of a PSF database
    (plain definition: eigen-decomposition of the sample covariance).  psfs [n][T][T] ->
    (basis [M+1][T][T] with row 0 the mean, components unit-norm, largest entry positive;
    residual = fraction of the centred energy not captured)."""
    X = np.asarray(psfs, dtype=np.float64).reshape(psfs.shape[0], -1)
    mu = X.mean(0)
    Xc = X - mu
    C = Xc.T @ Xc
    evals, evecs = np.linalg.eigh(C)
    idx = np.argsort(evals)[::-1][:M]
    V = evecs[:, idx].T
    for r in range(M):
        if V[r, np.argmax(np.abs(V[r]))] < 0:
            V[r] = -V[r]
    T = psfs.shape[1]
    basis = np.concatenate([mu[None], V]).reshape(M + 1, T, T)
    res = max(0.0, 1.0 - evals[idx].sum() / np.trace(C)) if np.trace(C) > 0 else 0.0
    return basis, res


def fit_readout(layers, a: np.ndarray, beta: np.ndarray, lam: float):
    """Ridge regression of the MLP output layer (NEXT-1 readout training), plain definition:
    X = [relu(W2 relu(W1 a + b1) + b2), 1]; Theta = argmin ||X Theta - beta||^2 +
    lam ||Theta[:-1]||^2, solved by lstsq on the stacked system.  layers = unpack_mlp(...)
    (W3, b3 are replaced).  Returns (W3 [K][h2], b3 [K], relative residual)."""
    (W1, b1), (W2, b2), _ = layers
    h = np.maximum(np.asarray(a, np.float64) @ W1.T + b1, 0.0)
    h = np.maximum(h @ W2.T + b2, 0.0)
    X = np.concatenate([h, np.ones((h.shape[0], 1))], axis=1)
    d = X.shape[1]
    reg = np.sqrt(lam) * np.eye(d)[:-1]  # bias not shrunk
    A = np.concatenate([X, reg])
    B = np.concatenate([np.asarray(beta, np.float64), np.zeros((d - 1, beta.shape[1]))])
    Th = np.linalg.lstsq(A, B, rcond=None)[0]
    res = np.linalg.norm(X @ Th - beta) / np.linalg.norm(beta)
    return Th[:-1].T, Th[-1], res
