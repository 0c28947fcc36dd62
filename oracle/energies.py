"""Zernike cross-correlation kernels and the approximation energies of P:369-397
 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may use this module.

Cross-correlation A_ij(s, phi) = E[a_i(x) a_j(x + s)] of the single-screen model (the
general form of reading Q4, pinned against the independent 4-D structure-function
quadrature `correlation.brute_force_Ajj` for cos/sin and mixed-m pairs):

  A_ij = 2 pi C_W sqrt((n_i+1)(n_j+1)) Int nu^{-8/3} [2 J_{n_i+1}(pi nu)/(pi nu)]
         [2 J_{n_j+1}(pi nu)/(pi nu)] Re{ conj(c_i) c_j G_ij(2 pi nu s, phi) } d nu,

  c_j = (-1)^{(n_j - m_j)/2} i^{m_j},
  G_ij(x, phi) = (1/2pi) Int_0^{2pi} A_i(t) A_j(t) e^{i x cos(t - phi)} dt,

with A_j(t) = 1 (m = 0), sqrt(2) cos(m t) (cos branch) or sqrt(2) sin(m t) (sin branch);
every product of two angular factors is a sum of cos/sin(M t), and
(1/2pi) Int trig(M t) e^{i x cos(t - phi)} dt = i^M J_M(x) trig(M phi).

Energies:  E(s) = Int_0^s Int_0^{2pi} tr(A_s'^T A_s') s' dphi ds',
E~(s) the same with the model A~_s = L diag(c_k(s)) L^T (c_k = A_kk / A_kk(0), the kernels
the sampler realises before mixing, Eq.10), and E^-(s) with |tr(A^T A - A~^T A~)|; the
paper plots modes 4..36 (piston and tilts excluded).
"""
from __future__ import annotations

import numpy as np
from scipy.special import jv

from .correlation import C_W, quad_nodes
from .optics import noll_cholesky, noll_covariance, noll_nm


def _angular_terms(i: int, j: int):
    """[(coef, M, trig)] with A_i(t) A_j(t) = sum coef * trig(M t)."""
    _, a, ki = noll_nm(i)
    _, b, kj = noll_nm(j)
    if a == 0 and b == 0:
        return [(1.0, 0, "c")]
    if a == 0:
        return [(np.sqrt(2.0), b, "c" if kj == "cos" else "s")]
    if b == 0:
        return [(np.sqrt(2.0), a, "c" if ki == "cos" else "s")]
    if ki == "cos" and kj == "cos":
        return [(1.0, a - b, "c"), (1.0, a + b, "c")]
    if ki == "sin" and kj == "sin":
        return [(1.0, a - b, "c"), (-1.0, a + b, "c")]
    if ki == "cos" and kj == "sin":
        return [(1.0, a + b, "s"), (-1.0, a - b, "s")]
    return [(1.0, a + b, "s"), (1.0, a - b, "s")]


def cross_kernel(i: int, j: int, s: np.ndarray, phi: np.ndarray, d_over_r0: float = 1.0,
                 nu_max: float = 200.0) -> np.ndarray:
    """A_ij at lags (s, phi) (arrays of the same shape), s in units of D."""
    s = np.asarray(s, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    ni, mi, _ = noll_nm(i)
    nj, mj, _ = noll_nm(j)
    nu, w = quad_nodes(max(float(np.max(s)), 0.05), nu_max)
    x = np.pi * nu
    rad = w * 2 * np.pi * C_W * np.sqrt((ni + 1.0) * (nj + 1.0)) * nu ** (-8.0 / 3.0) \
        * (2 * jv(ni + 1, x) / x) * (2 * jv(nj + 1, x) / x)
    cc = np.conj((-1) ** ((ni - mi) // 2) * 1j ** mi) * ((-1) ** ((nj - mj) // 2) * 1j ** mj)
    out = np.zeros(s.shape)
    arg = 2 * np.pi * np.outer(s.ravel(), nu)
    for coef, M, trig in _angular_terms(i, j):
        t = (np.cos if trig == "c" else np.sin)(M * phi.ravel())
        val = np.real(cc * coef * 1j ** M) * (jv(M, arg) @ rad) * t
        out += val.reshape(s.shape)
    return out * d_over_r0 ** (5.0 / 3.0)


def energies(s_max: float, n_s: int = 24, modes=(4, 36), N: int = 36, d_over_r0: float = 1.0, n_phi: int = 32,
             angle_mean: bool = False):
    """(s, E, E~, E-) on a uniform grid of n_s points per unit of s over [0, s_max]; radial
    integral by the cumulative trapezoid.

    angle_mean=False: the formulas as printed -- tr(A^T A) at every (s', phi), the angular
    integral as the exact mean over n_phi uniform angles (trigonometric polynomials of
    degree < n_phi).  angle_mean=True (reading Q25, "we integrate over the angular
    components"): the correlation functions are averaged over the angle first (only the
    M = 0 harmonics survive), then squared -- the reading that reproduces the paper's
    conclusions (E ~ E~, E- << E)."""
    lo, hi = modes
    idx = list(range(lo, hi + 1))
    A0 = noll_covariance(N, d_over_r0)
    L = noll_cholesky(A0)
    ns = max(2, int(round(n_s * s_max)))
    sg = np.linspace(0.0, s_max, ns + 1)
    if angle_mean:
        n_phi = 1
    ph = 2 * np.pi * np.arange(n_phi) / n_phi
    nu, w = quad_nodes(max(s_max, 0.05), 200.0)
    x = np.pi * nu
    arg = 2 * np.pi * np.outer(sg, nu)
    JM = {}
    R = {}

    def radial(ni, nj, M):
        key = (min(ni, nj), max(ni, nj), M)
        if key not in R:
            if M not in JM:
                JM[M] = jv(M, arg)
            rad = w * 2 * np.pi * C_W * np.sqrt((ni + 1.0) * (nj + 1.0)) * nu ** (-8.0 / 3.0) \
                * (2 * jv(ni + 1, x) / x) * (2 * jv(nj + 1, x) / x)
            R[key] = JM[M] @ rad
        return R[key]

    def kernel(a, b):
        na, ma, _ = noll_nm(a)
        nb, mb, _ = noll_nm(b)
        cc = np.conj((-1) ** ((na - ma) // 2) * 1j ** ma) * ((-1) ** ((nb - mb) // 2) * 1j ** mb)
        out = np.zeros((sg.size, n_phi))
        for coef, M, trig in _angular_terms(a, b):
            if angle_mean and (M != 0 or trig != "c"):
                continue  # zero angular mean
            t = (np.cos if trig == "c" else np.sin)(M * ph)
            out += np.real(cc * coef * 1j ** M) * np.outer(radial(na, nb, abs(M)) * (1 if M >= 0 else (-1) ** M), t)
        return out * d_over_r0 ** (5.0 / 3.0)

    c = {k: kernel(k, k) / A0[k - 1, k - 1] for k in range(2, N + 1)}
    full = np.zeros((sg.size, n_phi))
    model = np.zeros_like(full)
    diff = np.zeros_like(full)
    for a in idx:
        for b in idx:
            if b < a:
                continue
            Aab = kernel(a, b)
            # A_ba(s, phi) = A_ab(s, phi + pi); the angular mean is symmetric
            Aba = Aab if angle_mean else np.roll(Aab, -n_phi // 2, axis=1)
            Mab = sum(L[a - 1, k - 1] * L[b - 1, k - 1] * c[k] for k in range(2, N + 1))
            for A_ in ((Aab,) if a == b else (Aab, Aba)):
                full += A_ ** 2
                model += Mab ** 2
                diff += A_ ** 2 - Mab ** 2
    f_full = full.mean(axis=1) * 2 * np.pi * sg
    f_model = model.mean(axis=1) * 2 * np.pi * sg
    f_diff = np.abs(diff).mean(axis=1) * 2 * np.pi * sg

    def cum(f):
        return np.concatenate([[0.0], np.cumsum(0.5 * (f[1:] + f[:-1]) * np.diff(sg))])
    return sg, cum(f_full), cum(f_model), cum(f_diff)
