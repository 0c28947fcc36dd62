"""Optics core of the oracle (test infrastructure; see oracle/__init__.py).

* Noll indexing and Zernike polynomials Z_j(rho) -- P:129-135 (Eq.5), Noll 1976.
* Kolmogorov constants: structure function D_phi(r) = C_D (r/r0)^{5/3}
  (Eq.4; C_D = 2[(24/5)Gamma(6/5)]^{5/6} = 6.8839, printed 6.88 in
  the paper -- reading Q1) and the phase PSD W(f) = C_W r0^{-5/3} f^{-11/3}
   with C_W fixed by D_phi(r) = 2 Int (1 - cos 2pi f.r) W(f) d^2f.
* Noll matrix A_0 = [A]_{0,i,j}: Noll's Gamma-function closed form,
  written with K_N = C_W 2^{-5/3} pi^{8/3} Gamma(14/3) (reading Q1); piston row
  and column are zero (Q2).
* Cholesky factor L with L L^T = A_0 over j = 2..N (Eq.10).
"""
from __future__ import annotations

from math import factorial

import numpy as np
from scipy.special import gamma

# ---------------------------------------------------------------- constants
C_D = 2.0 * ((24.0 / 5.0) * gamma(6.0 / 5.0)) ** (5.0 / 6.0)  # Eq.4 coefficient (6.8839)
# Int_0^inf (1 - J0(x)) x^{-8/3} dx = 2^{-5/3} Gamma(1/6) / ((5/3) Gamma(11/6))
_I_SF = 2.0 ** (-5.0 / 3.0) * gamma(1.0 / 6.0) / ((5.0 / 3.0) * gamma(11.0 / 6.0))
# D(r) = 4 pi C_W r0^{-5/3} (2 pi r)^{5/3} _I_SF  =>
C_W = C_D / (4.0 * np.pi * (2.0 * np.pi) ** (5.0 / 3.0) * _I_SF)  # 0.0228956
K_NOLL = C_W * 2.0 ** (-5.0 / 3.0) * np.pi ** (8.0 / 3.0) * gamma(14.0 / 3.0)  # 2.246065


def structure_function(r, r0):
    """D_phi(r) = C_D (r/r0)^{5/3} -- P:112-115 (Eq.4)."""
    if r0 <= 0:
        raise ValueError("r0 must be > 0")
    return C_D * (np.asarray(r, dtype=np.float64) / r0) ** (5.0 / 3.0)


# ---------------------------------------------------------------- Noll index
def noll_nm(j: int):
    """Noll index j >= 1 -> (n, m, kind) with kind in {'cos','sin','rot'}.

    n = min{n : (n+1)(n+2)/2 >= j}; within a radial order the azimuthal orders
    run 0,2,2,4,4,.. (n even) or 1,1,3,3,.. (n odd); for m != 0 even j is the
    cos branch and odd j the sin branch (Noll 1976 convention).
    """
    if j < 1:
        raise ValueError("Noll index must be >= 1")
    n = 0
    while (n + 1) * (n + 2) // 2 < j:
        n += 1
    p = j - n * (n + 1) // 2 - 1  # position inside the radial order
    if n % 2 == 0:
        m = 2 * ((p + 1) // 2)
    else:
        m = 2 * (p // 2) + 1
    if m == 0:
        kind = "rot"
    else:
        kind = "cos" if j % 2 == 0 else "sin"
    return n, m, kind


def zernike_radial(n: int, m: int, rho):
    rho = np.asarray(rho, dtype=np.float64)
    out = np.zeros_like(rho)
    for s in range((n - m) // 2 + 1):
        c = (-1) ** s * factorial(n - s) / (
            factorial(s) * factorial((n + m) // 2 - s) * factorial((n - m) // 2 - s))
        out = out + c * rho ** (n - 2 * s)
    return out


def zernike(j: int, rho, theta):
    """Noll-normalised Z_j(rho, theta) on the unit disk (unit mean square for j >= 2)."""
    n, m, kind = noll_nm(j)
    R = zernike_radial(n, m, rho)
    if kind == "rot":
        return np.sqrt(n + 1.0) * R
    ang = np.cos(m * np.asarray(theta)) if kind == "cos" else np.sin(m * np.asarray(theta))
    return np.sqrt(2.0 * (n + 1.0)) * R * ang


# ---------------------------------------------------------------- Noll matrix
def noll_covariance(N: int, d_over_r0: float) -> np.ndarray:
    """A_0[i-1][j-1] = E[a_i a_j] for i, j = 1..N ("covariance matrix given by Noll").

    Closed form (Noll 1976 Eq.25 with the exact Kolmogorov constant K_NOLL):
      K_N (-1)^{(n_i+n_j-2m)/2} sqrt((n_i+1)(n_j+1)) Gamma((n_i+n_j-5/3)/2) (D/r0)^{5/3}
      / [Gamma((n_i-n_j+17/3)/2) Gamma((n_j-n_i+17/3)/2) Gamma((n_i+n_j+23/3)/2)]
    when m_i == m_j and (m == 0 or same cos/sin branch), else 0.  Piston is 0 (Q2).
    """
    if N < 3:
        raise ValueError("N must be >= 3")
    if d_over_r0 < 0:
        raise ValueError("D/r0 must be >= 0")
    A = np.zeros((N, N))
    scale = d_over_r0 ** (5.0 / 3.0)
    for i in range(2, N + 1):
        ni, mi, ki = noll_nm(i)
        for j in range(2, N + 1):
            nj, mj, kj = noll_nm(j)
            if mi != mj:
                continue
            if mi != 0 and ki != kj:
                continue
            sign = (-1.0) ** ((ni + nj - 2 * mi) // 2)
            num = K_NOLL * sign * np.sqrt((ni + 1.0) * (nj + 1.0)) * gamma((ni + nj - 5.0 / 3.0) / 2.0)
            den = (gamma((ni - nj + 17.0 / 3.0) / 2.0) * gamma((nj - ni + 17.0 / 3.0) / 2.0)
                   * gamma((ni + nj + 23.0 / 3.0) / 2.0))
            A[i - 1, j - 1] = num / den * scale
    return A


def noll_cholesky(A0: np.ndarray) -> np.ndarray:
    """Lower-triangular L (N x N) with L L^T = A0, L row/col 0 (piston) = 0.

    Factorises A0[1:, 1:]; if that fails, adds 1e-12 trace/N to the diagonal
     and retries; D/r0 = 0 gives L = 0.
    """
    N = A0.shape[0]
    L = np.zeros_like(A0)
    B = A0[1:, 1:]
    if not np.any(B):
        return L
    try:
        L[1:, 1:] = np.linalg.cholesky(B)
    except np.linalg.LinAlgError:
        reg = 1e-12 * np.trace(B) / B.shape[0]
        L[1:, 1:] = np.linalg.cholesky(B + reg * np.eye(B.shape[0]))
    return L


# ---------------------------------------------------------------- geometry
def geometry(aperture_m=0.1, wavelength_m=525e-9, L_m=1000.0, s_per_px=0.0, tilt_px_per_rad=0.0):
    """(s_px, kappa_t) -- readings Q5 and Q12.

    s_px = L * IFOV / D with the default Nyquist IFOV = lambda/(2D) (P:263 footnote
    s = L(theta - theta')/D).  kappa_t = 4/pi pixels per unit a_2 at Nyquist
    sampling (Z_2 = 2 rho cos theta => tilt angle (2/pi)(lambda/D) a_2).
    """
    ifov = wavelength_m / (2.0 * aperture_m)
    s_px = s_per_px if s_per_px > 0 else L_m * ifov / aperture_m
    kappa = tilt_px_per_rad if tilt_px_per_rad > 0 else 4.0 / np.pi
    return s_px, kappa
