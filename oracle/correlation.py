"""Homogeneous Zernike auto-correlation slices and their PSDs (test infrastructure).

Paper: for a fixed mode pair the slice A_{i,j} of the correlation tensor is a
function of the lag s = (x - x')/D only (P:254-274 and footnote P:263), so
A_{i,i} is circulant on a periodic grid and is diagonalised by the DFT
(P:234-238): sigma^{1/2} e = F^{-1}(S^{1/2} F(e)) with S "the Fourier spectrum of
one row ... of the correlation matrix".  DF-P2S draws N unit-variance fields from
the A_{i,i} alone (step 1).

The paper cites [Chimitt2020] for the form of A_{i,i}(s) without restating it
(reading Q4): collapsed single-screen model, i.e. the Zernike coefficients of one
Kolmogorov screen seen through an aperture translated by D s.  With nu in cycles
per aperture diameter and W(nu) = C_W (D/r0)^{5/3} nu^{-11/3}:

  A_jj(s, phi) = 2 pi C_W (n+1) Int_0^inf nu^{-8/3} [2 J_{n+1}(pi nu)/(pi nu)]^2
                 [ J_0(2 pi nu s) +/- (-1)^m J_{2m}(2 pi nu s) cos(2 m phi) ] d nu
                 * (D/r0)^{5/3}

(+ for the cos branch, - for the sin branch, no J_{2m} term for m = 0; phi is the
angle of the lag from the x (column) axis).  Pinned in tests against (i) the Noll
closed form at s = 0 and (ii) a brute-force 4-D double-aperture quadrature of the
structure function (``brute_force_Ajj``).

Numerics (the paper gives none): radial tables R_{n,q}(s) by composite 8-point
Gauss-Legendre on nu in [0, 50] (nu = u^3 substitution on [0,1] for the
nu^{-2/3} end-point behaviour of the tilt modes), panel width <= 1/(2 s_max);
then a cubic spline in |s| on a 0.01-spaced grid.
"""
from __future__ import annotations

import numpy as np
from scipy import integrate
from scipy.interpolate import CubicSpline
from scipy.special import jv

from .optics import C_D, C_W, noll_nm, zernike

NU_MAX = 50.0
H_S = 0.01


def _radial_weight(n: int, nu):
    """2 pi C_W (n+1) nu^{-8/3} [2 J_{n+1}(pi nu)/(pi nu)]^2 (unit (D/r0))."""
    x = np.pi * nu
    return 2.0 * np.pi * C_W * (n + 1.0) * nu ** (-8.0 / 3.0) * (2.0 * jv(n + 1, x) / x) ** 2


def quad_nodes(s_max: float, nu_max: float = NU_MAX, npan_pts: int = 8):
    """Composite Gauss-Legendre nodes/weights on nu in (0, nu_max]."""
    w_nu = min(0.25, 1.0 / (2.0 * max(s_max, 1e-6)))
    xg, wg = np.polynomial.legendre.leggauss(npan_pts)
    nodes, weights = [], []
    # region A: nu = u^3, u in [0,1]; d nu = 3u^2 du
    npa = int(np.ceil(3.0 / w_nu))
    ub = np.linspace(0.0, 1.0, npa + 1)
    for a, b in zip(ub[:-1], ub[1:]):
        u = 0.5 * (b - a) * xg + 0.5 * (a + b)
        nodes.append(u ** 3)
        weights.append(0.5 * (b - a) * wg * 3.0 * u ** 2)
    # region B: nu in [1, nu_max]
    npb = int(np.ceil((nu_max - 1.0) / w_nu))
    vb = np.linspace(1.0, nu_max, npb + 1)
    for a, b in zip(vb[:-1], vb[1:]):
        nodes.append(0.5 * (b - a) * xg + 0.5 * (a + b))
        weights.append(0.5 * (b - a) * wg)
    return np.concatenate(nodes), np.concatenate(weights)


def radial_pairs(N: int = 36):
    """The (n, q) radial integrals needed for modes 2..N: q = 0 and q = 2m (m > 0)."""
    pairs = set()
    for j in range(2, N + 1):
        n, m, _ = noll_nm(j)
        pairs.add((n, 0))
        if m > 0:
            pairs.add((n, 2 * m))
    return sorted(pairs)


def radial_tables(s_max: float, N: int = 36, h: float = H_S, nu_max: float = NU_MAX, chunk: int = 64):
    """s grid and {(n,q): R_{n,q}(s_grid)} per unit (D/r0)^{5/3}."""
    ns = int(np.ceil(s_max / h)) + 4
    s = h * np.arange(ns)
    nu, wq = quad_nodes(s[-1], nu_max)
    pairs = radial_pairs(N)
    ns_needed = sorted({n for n, _ in pairs})
    gw = {n: _radial_weight(n, nu) * wq for n in ns_needed}
    R = {p: np.empty(ns) for p in pairs}
    qs = sorted({q for _, q in pairs})
    for i0 in range(0, ns, chunk):
        sc = s[i0:i0 + chunk]
        arg = 2.0 * np.pi * np.outer(sc, nu)
        for q in qs:
            Jq = jv(q, arg)
            for (n, qq) in pairs:
                if qq == q:
                    R[(n, q)][i0:i0 + chunk] = Jq @ gw[n]
    return s, R


def radial_tables_cached(s_max: float, N: int = 36):
    """radial_tables() with s_max rounded up to an integer and an on-disk cache.

    The cache (default /tmp/p2s_oracle_cache, env P2S_ORACLE_CACHE) only ever
    holds values this module computed; delete it to recompute.
    """
    import os
    s_r = float(np.ceil(max(s_max, 1e-3)))
    d = os.environ.get("P2S_ORACLE_CACHE", "/tmp/p2s_oracle_cache")
    fn = os.path.join(d, f"radial_s{s_r:.0f}_N{N}_h{H_S}_nu{NU_MAX}.npz")
    if os.path.exists(fn):
        z = np.load(fn)
        s = z["s"]
        R = {tuple(int(t) for t in k.split("_")): z[k] for k in z.files if k != "s"}
        return s, R
    s, R = radial_tables(s_r, N)
    os.makedirs(d, exist_ok=True)
    tmp = fn + f".{os.getpid()}.tmp.npz"
    np.savez(tmp, s=s, **{f"{n}_{q}": v for (n, q), v in R.items()})
    os.replace(tmp, fn)
    return s, R


def Ajj_quad(j: int, s: float, phi: float, d_over_r0: float = 1.0) -> float:
    """A_jj(s, phi) by adaptive scipy.quad (slow; pins and spot checks only)."""
    n, m, kind = noll_nm(j)
    sgn = 1.0 if kind == "cos" else -1.0

    def f(nu):
        val = jv(0, 2 * np.pi * nu * s)
        if m > 0:
            val = val + sgn * (-1.0) ** m * jv(2 * m, 2 * np.pi * nu * s) * np.cos(2 * m * phi)
        return _radial_weight(n, nu) * val

    def fu(u):  # nu = u^3 on [0, 1]
        return f(u ** 3) * 3.0 * u ** 2

    lim = 400
    a = integrate.quad(fu, 0.0, 1.0, limit=lim, epsabs=1e-13, epsrel=1e-11)[0]
    b = integrate.quad(f, 1.0, 8.0, limit=lim, epsabs=1e-13, epsrel=1e-11)[0]
    c = integrate.quad(f, 8.0, 200.0, limit=2000, epsabs=1e-14, epsrel=1e-10)[0]
    return (a + b + c) * d_over_r0 ** (5.0 / 3.0)


def brute_force_Ajj(i: int, j: int, sx: float, sy: float, d_over_r0: float = 1.0,
                    nr: int = 24, nt: int = 48) -> float:
    """E[a_i(0) a_j(s)] by 4-D quadrature of the structure function (independent route).

    a_j(x) = (1/pi) Int_disk Z_j(rho) phi(x + R rho) d^2rho; for zero-mean modes
    (j >= 2) E[phi phi'] may be replaced by -D_phi/2, so
      A_ij(s) = -(C_D/(2 pi^2)) Int Int Z_i(rho) Z_j(rho') |s + (rho' - rho)/2|^{5/3}
    in units of (D/r0)^{5/3}, lag s in units of D.
    """
    xr, wr = np.polynomial.legendre.leggauss(nr)
    r = 0.5 * (xr + 1.0)
    wr = 0.5 * wr * r  # polar Jacobian
    th = 2 * np.pi * (np.arange(nt) + 0.5) / nt
    wt = np.full(nt, 2 * np.pi / nt)
    R, TH = np.meshgrid(r, th, indexing="ij")
    Wgt = np.outer(wr, wt).ravel()
    X, Y = (R * np.cos(TH)).ravel(), (R * np.sin(TH)).ravel()
    Zi = zernike(i, R.ravel(), TH.ravel()) * Wgt
    Zj = zernike(j, R.ravel(), TH.ravel()) * Wgt
    dx = sx + 0.5 * (X[None, :] - X[:, None])
    dy = sy + 0.5 * (Y[None, :] - Y[:, None])
    Dm = (dx * dx + dy * dy) ** (5.0 / 6.0)
    val = -(C_D / (2.0 * np.pi ** 2)) * (Zi @ Dm @ Zj)
    return val * d_over_r0 ** (5.0 / 3.0)


def lag_grid(P: int, Q: int, s_px: float):
    """Minimum-image signed lags (dy, dx) in pixels, |s| (units of D) and angle phi."""
    iy = np.arange(P)
    ix = np.arange(Q)
    dy = np.where(iy <= P // 2, iy, iy - P).astype(np.float64)
    dx = np.where(ix <= Q // 2, ix, ix - Q).astype(np.float64)
    DY, DX = np.meshgrid(dy, dx, indexing="ij")
    s = s_px * np.hypot(DY, DX)
    phi = np.arctan2(DY, DX)
    return s, phi


def autocorrelation_kernels(P: int, Q: int, s_px: float, N: int = 36, tables=None):
    """c_j(dy, dx) = A_jj(s)/A_jj(0) on the periodic P x Q lag grid, j = 2..N.

    Returns float64 [N-1][P][Q] (slot j-2).  Unit variance at zero lag.
    """
    s, phi = lag_grid(P, Q, s_px)
    if tables is None:
        tables = radial_tables_cached(float(s.max()), N)
    sg, R = tables
    spl = {p: CubicSpline(sg, v) for p, v in R.items()}
    out = np.empty((N - 1, P, Q))
    cache = {}
    for j in range(2, N + 1):
        n, m, kind = noll_nm(j)
        if (n, 0) not in cache:
            cache[(n, 0)] = spl[(n, 0)](s)
        val = cache[(n, 0)].copy()
        if m > 0:
            if (n, 2 * m) not in cache:
                cache[(n, 2 * m)] = spl[(n, 2 * m)](s)
            sgn = 1.0 if kind == "cos" else -1.0
            val += sgn * (-1.0) ** m * cache[(n, 2 * m)] * np.cos(2 * m * phi)
        out[j - 2] = val / R[(n, 0)][0]
    return out


def psd_from_kernel(c: np.ndarray):
    """S = DFT(c) (real: c is real and even), clamp S >= 0, renormalise sum S = PQ.

    Reading Q7 (circulant embedding can produce negative eigenvalues): clamp to
    zero and renormalise so the field keeps unit variance.  Returns
    (S, sqrt(S), clamped_fraction) where clamped_fraction = negative mass / sum|S|.
    """
    P, Q = c.shape[-2:]
    F = np.fft.fft2(c)
    S = F.real
    neg = -S[S < 0].sum()
    frac = neg / np.abs(S).sum()
    S = np.maximum(S, 0.0)
    S = S * (P * Q) / S.sum()
    return S, np.sqrt(S), frac


def sqrt_psd_tables(P: int, Q: int, s_px: float, N: int = 36, tables=None):
    """sqrt(S_j) for j = 2..N as float64 [N-1][P][Q] plus the clamped fractions."""
    c = autocorrelation_kernels(P, Q, s_px, N, tables)
    out = np.empty_like(c)
    fr = np.empty(N - 1)
    for k in range(N - 1):
        _, out[k], fr[k] = psd_from_kernel(c[k])
    return out, fr
