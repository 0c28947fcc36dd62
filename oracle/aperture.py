"""Aperture statistics of the validation battery --
TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may use this module.

The paper validates the sampled Zernike vectors on the aperture by (a) the phase
structure function against Eq.4 (Fig. struct_fun) and (b) the long- and
short-exposure OTFs:

    H(xi)    = (P e^{-j phi}) (*) (P(-xi) e^{j phi(-xi)})      (pupil autocorrelation)
    H_LE     = E[H],   H_SE = E[H] with the tilt-corrected phase phi - alpha^T xi
               (alpha^T xi the plane of best fit over the pupil).

Discretisation (the pupil of reading Q24): Dp = 32 samples across the aperture, sample
centres with rho <= 1; lags xi = (dy, dx), dy in [0, Dp), dx in (-Dp, Dp) samples.  Per
Zernike vector (one pixel of one frame) and lag, with M the pupil mask and
Delta(x) = phi(x) - phi(x + xi):

    cnt(xi) = sum_x M(x) M(x+xi)
    SF(xi)  = sum_x M M' Delta^2 / cnt(xi)             (0 where cnt = 0)
    LE(xi)  = sum_x M M' cos(Delta) / cnt(0)            (Re H / H(0))
    SE(xi)  = the same with phi replaced by the residual of the least-squares plane fit

and the battery averages the three over all vectors.  `aperture_stats` is that definition
written out (the real part of H: its imaginary part is odd in the phase and averages to 0).

Reference curves:
  * model (the sampler's own law, exact for Gaussian a ~ N(0, A_0)):
    Var Delta = dZ^T A_0 dZ with dZ_j = Z_j(x) - Z_j(x + xi), so E[SF] = mean of
    Var Delta and E[cos Delta] = exp(-Var Delta / 2); for SE, Z_j is replaced by its
    residual after the plane fit (a linear projection of the phase);
  * theory ([Roggemann 1996]): D(r) = C_D (r/r0)^{5/3} (Eq.4),
    H_LE = H_diff(u) exp(-D(r)/2), H_SE = H_diff(u) exp(-D(r)/2 (1 - u^{1/3})) with
    u = r/D and H_diff the diffraction OTF of the disc -- the untruncated Kolmogorov
    phase, which a 36-mode phase only approaches.
"""
from __future__ import annotations

import numpy as np

from .optics import C_D, zernike

PUPIL_D = 32


def pupil_coords(Dp: int = PUPIL_D):
    """(X, Y, mask): sample-centre coordinates in radius units and the disc mask."""
    c = (np.arange(Dp) + 0.5 - Dp / 2.0) / (Dp / 2.0)
    Y, X = np.meshgrid(c, c, indexing="ij")
    return X, Y, np.hypot(X, Y) <= 1.0


def zernike_planes(Z: int, Dp: int = PUPIL_D) -> np.ndarray:
    """Z_j (j = 1..Z) at the pupil samples, zero outside the disc: [Z][Dp][Dp]."""
    X, Y, m = pupil_coords(Dp)
    rho, th = np.hypot(X, Y), np.arctan2(Y, X)
    return np.stack([zernike(j, rho, th) * m for j in range(1, Z + 1)])


def plane_residual(phi: np.ndarray, Dp: int = PUPIL_D) -> np.ndarray:
    """phi - (c + alpha_x X + alpha_y Y), least squares over the disc samples;
    phi [..][Dp][Dp].  Zero outside the disc."""
    X, Y, m = pupil_coords(Dp)
    A = np.stack([np.ones(m.sum()), X[m], Y[m]], axis=1)
    flat = phi.reshape(-1, Dp, Dp)[:, m]  # [n][npts]
    coef, *_ = np.linalg.lstsq(A, flat.T, rcond=None)
    res = np.zeros((flat.shape[0], Dp, Dp))
    res[:, m] = flat - (A @ coef).T
    return res.reshape(phi.shape)


def lag_overlap(Dp: int = PUPIL_D) -> np.ndarray:
    """cnt(xi) = sum_x M(x) M(x + xi) on the lag grid [Dp][2Dp-1]."""
    _, _, m = pupil_coords(Dp)
    out = np.zeros((Dp, 2 * Dp - 1))
    for dy in range(Dp):
        for i, dx in enumerate(range(-(Dp - 1), Dp)):
            a, b = _overlap(m[None].astype(float), dy, dx)
            out[dy, i] = (a * b).sum()
    return out


def _overlap(f: np.ndarray, dy: int, dx: int):
    """(f(x), f(x + xi)) over the positions where both lie on the grid; f [n][Dp][Dp]."""
    Dp = f.shape[-1]
    y0, y1 = 0, Dp - dy
    x0, x1 = max(0, -dx), min(Dp, Dp - dx)
    return f[:, y0:y1, x0:x1], f[:, y0 + dy:y1 + dy, x0 + dx:x1 + dx]


def aperture_stats(a: np.ndarray, Dp: int = PUPIL_D):
    """The definition above for Zernike vectors a [n][Z] (Noll 1..Z, a[:, 0] = piston,
    ignored): returns (SF, LE, SE), each [Dp][2Dp-1] averaged over the n vectors."""
    a = np.asarray(a, dtype=np.float64)
    Z = a.shape[1]
    zp = zernike_planes(Z, Dp)
    phi = np.einsum("nj,jyx->nyx", a[:, 1:], zp[1:])
    vphi = plane_residual(phi, Dp)
    _, _, m = pupil_coords(Dp)
    mk = np.broadcast_to(m.astype(float), phi.shape)
    cnt = lag_overlap(Dp)
    n0 = cnt[0, Dp - 1]
    SF = np.zeros((Dp, 2 * Dp - 1))
    LE = np.zeros_like(SF)
    SE = np.zeros_like(SF)
    for dy in range(Dp):
        for i, dx in enumerate(range(-(Dp - 1), Dp)):
            if cnt[dy, i] == 0:
                continue
            m1, m2 = _overlap(mk, dy, dx)
            w = m1 * m2
            p1, p2 = _overlap(phi, dy, dx)
            q1, q2 = _overlap(vphi, dy, dx)
            SF[dy, i] = np.mean((w * (p1 - p2) ** 2).sum(axis=(1, 2))) / cnt[dy, i]
            LE[dy, i] = np.mean((w * np.cos(p1 - p2)).sum(axis=(1, 2))) / n0
            SE[dy, i] = np.mean((w * np.cos(q1 - q2)).sum(axis=(1, 2))) / n0
    return SF, LE, SE


def model_stats(A0: np.ndarray, Dp: int = PUPIL_D):
    """E[SF], E[LE], E[SE] for a ~ N(0, A0) (A0 [Z][Z], Noll 1..Z): the Gaussian identities
    E[Delta^2] = dZ^T A0 dZ and E[cos Delta] = exp(-E[Delta^2] / 2)."""
    A0 = np.asarray(A0, dtype=np.float64)
    Z = A0.shape[0]
    zp = zernike_planes(Z, Dp)
    zr = plane_residual(zp, Dp)
    _, _, m = pupil_coords(Dp)
    mk = m[None].astype(float)
    cnt = lag_overlap(Dp)
    n0 = cnt[0, Dp - 1]
    SF = np.zeros((Dp, 2 * Dp - 1))
    LE = np.zeros_like(SF)
    SE = np.zeros_like(SF)
    for dy in range(Dp):
        for i, dx in enumerate(range(-(Dp - 1), Dp)):
            if cnt[dy, i] == 0:
                continue
            m1, m2 = _overlap(mk, dy, dx)
            w = (m1 * m2)[0]
            z1, z2 = _overlap(zp, dy, dx)
            r1, r2 = _overlap(zr, dy, dx)
            dz, dr = z1 - z2, r1 - r2
            v = (dz * np.tensordot(A0, dz, axes=(1, 0))).sum(axis=0)  # dZ^T A0 dZ per position
            vr = (dr * np.tensordot(A0, dr, axes=(1, 0))).sum(axis=0)
            SF[dy, i] = (w * v).sum() / cnt[dy, i]
            LE[dy, i] = (w * np.exp(-0.5 * v)).sum() / n0
            SE[dy, i] = (w * np.exp(-0.5 * vr)).sum() / n0
    return SF, LE, SE


def lag_radius(Dp: int = PUPIL_D) -> np.ndarray:
    """|xi| / Dp = r / D on the lag grid."""
    dy = np.arange(Dp)[:, None]
    dx = np.arange(-(Dp - 1), Dp)[None, :]
    return np.hypot(dy, dx) / Dp


def diffraction_otf(u):
    """Diffraction OTF of a circular aperture at u = r/D (0 beyond u = 1)."""
    u = np.clip(np.asarray(u, dtype=np.float64), 0.0, 1.0)
    return (2.0 / np.pi) * (np.arccos(u) - u * np.sqrt(1.0 - u * u))


def theory_curves(u, d_over_r0: float):
    """(D(r), H_LE, H_SE) of the untruncated Kolmogorov phase at u = r/D."""
    u = np.asarray(u, dtype=np.float64)
    D = C_D * (u * d_over_r0) ** (5.0 / 3.0)
    Hd = diffraction_otf(u)
    return D, Hd * np.exp(-0.5 * D), Hd * np.exp(-0.5 * D * (1.0 - np.cbrt(np.clip(u, 0.0, 1.0))))
