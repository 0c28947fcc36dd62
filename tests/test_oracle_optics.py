"""Pins for oracle/optics.py and oracle/philox.py (CPU, -m "not gpu").

Each assertion compares the oracle with something other than itself: values
printed in Noll 1976 (the paper's source for A_0), closed forms, the
paper's Eq.4, quadrature of the definitions, or the Random123 KAT vectors.
"""
import os

import numpy as np
import pytest
from scipy import integrate
from scipy.special import jv

from oracle import optics, philox

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ Philox
def test_philox_known_answers():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = philox.philox4x32_10(*v[:6])
        assert [int(o) for o in out] == v[6:]


def test_box_muller_moments():
    idx = np.arange(200000)
    (g1, g2), (g3, g4) = philox.gaussians(idx, 3, 0, 7, 2210)
    for g in (g1, g2, g3, g4):
        assert abs(g.mean()) < 0.01
        assert abs(g.var() - 1.0) < 0.01
        k = ((g - g.mean()) ** 4).mean() / g.var() ** 2
        assert 2.95 < k < 3.05
    assert abs(np.corrcoef(g1, g3)[0, 1]) < 0.01


# ------------------------------------------------------------------ Noll / Zernike
def test_noll_index_table():
    # Noll 1976 Table I (first 22 terms)
    expect = {1: (0, 0), 2: (1, 1), 3: (1, 1), 4: (2, 0), 5: (2, 2), 6: (2, 2), 7: (3, 1), 8: (3, 1),
              9: (3, 3), 10: (3, 3), 11: (4, 0), 12: (4, 2), 13: (4, 2), 14: (4, 4), 15: (4, 4),
              16: (5, 1), 21: (5, 5), 22: (6, 0), 29: (7, 1), 36: (7, 7)}
    for j, nm in expect.items():
        assert optics.noll_nm(j)[:2] == nm
    assert optics.noll_nm(2)[2] == "cos" and optics.noll_nm(3)[2] == "sin"
    assert optics.noll_nm(7)[2] == "sin" and optics.noll_nm(8)[2] == "cos"


def test_zernike_values_and_orthonormality():
    # SPEC S:53 Z4(0) = -sqrt(3); Z2 = 2 rho cos theta
    assert optics.zernike(4, 0.0, 0.0) == pytest.approx(-np.sqrt(3.0), abs=1e-14)
    assert optics.zernike(2, 0.5, 0.3) == pytest.approx(2 * 0.5 * np.cos(0.3), abs=1e-14)
    # Gauss-polar quadrature is exact for these polynomials: (1/pi) Int Z_i Z_j = delta_ij
    xr, wr = np.polynomial.legendre.leggauss(24)
    r = 0.5 * (xr + 1)
    wr = 0.5 * wr * r
    nt = 64
    th = 2 * np.pi * np.arange(nt) / nt
    R, TH = np.meshgrid(r, th, indexing="ij")
    wgt = np.outer(wr, np.full(nt, 2 * np.pi / nt)) / np.pi
    Z = np.stack([optics.zernike(j, R, TH) for j in range(1, 37)])
    G = np.einsum("ihw,jhw,hw->ij", Z, Z, wgt)
    assert np.abs(G - np.eye(36)).max() < 1e-10


def test_kolmogorov_constants():
    # Eq.4 prints 6.88; exact 2[(24/5)Gamma(6/5)]^{5/6}
    assert optics.C_D == pytest.approx(6.88, abs=0.005)
    # C_W from D(r) = 2 Int (1 - J0(2 pi f r)) W(f) 2 pi f df (r = r0 = 1): with x = 2 pi f,
    # D = 4 pi C_W (2 pi)^{5/3} Int_0^inf (1 - J0(x)) x^{-8/3} dx; integral by quadrature
    g = lambda x: (1 - jv(0, x)) * x ** (-8.0 / 3.0)
    X = 400.0
    edges = np.linspace(0, X, 401)
    val = sum(integrate.quad(g, a, b, limit=200, epsabs=1e-14)[0] for a, b in zip(edges[:-1], edges[1:]))
    val += 0.6 * X ** (-5.0 / 3.0)  # tail of x^{-8/3}; the J0 tail is O(X^{-19/6})
    D = 4 * np.pi * optics.C_W * (2 * np.pi) ** (5.0 / 3.0) * val
    assert D == pytest.approx(optics.C_D, rel=1e-6)
    # literature value of the Kolmogorov phase-PSD coefficient 0.023
    assert optics.C_W == pytest.approx(0.023, abs=2e-4)


def test_noll_matrix_vs_noll1976_table():
    """Noll 1976 Table IV residuals Delta_J (D/r0 = 1): <a_J^2> = Delta_{J-1} - Delta_J.

    Noll's constant differs from the exact Kolmogorov one by 0.25% (reading Q1)
    and the table is printed to 3-4 digits, hence 2% on each difference.
    """
    delta = [1.0299, 0.582, 0.134, 0.111, 0.0880, 0.0648, 0.0587, 0.0525, 0.0463, 0.0401,
             0.0377, 0.0352, 0.0328, 0.0304, 0.0279, 0.0267, 0.0255, 0.0243, 0.0232, 0.0220, 0.0208]
    A = optics.noll_covariance(36, 1.0)
    for J in range(2, 22):
        assert A[J - 1, J - 1] == pytest.approx(delta[J - 2] - delta[J - 1], rel=0.03, abs=1.05e-4), J  # table printed to 4 decimals
    # total piston-removed variance ~ Delta_1 (1.0299), remainder after 36 terms
    # ~ 0.2944 J^{-sqrt(3)/2} (Noll's asymptote)
    rem = 0.2944 * 36 ** (-np.sqrt(3) / 2)
    assert np.trace(A) + rem == pytest.approx(1.0299, rel=0.01)


def test_noll_matrix_structure():
    A1 = optics.noll_covariance(36, 1.0)
    A2 = optics.noll_covariance(36, 2.0)
    assert np.allclose(A2, A1 * 2 ** (5 / 3), rtol=1e-13, atol=0)
    assert A1[1, 2] == 0.0 and A1[0].max() == 0 and A1[:, 0].max() == 0  # S:79, Q2
    assert np.allclose(A1, A1.T, atol=0)
    assert np.linalg.eigvalsh(A1[1:, 1:]).min() > 0
    for i in range(2, 37):
        for j in range(2, 37):
            ni, mi, ki = optics.noll_nm(i)
            nj, mj, kj = optics.noll_nm(j)
            if mi != mj or (mi and ki != kj):
                assert A1[i - 1, j - 1] == 0.0
    # the 35x35 lower triangle has 31 nonzero off-diagonal entries
    assert int(np.count_nonzero(np.tril(A1[1:, 1:], -1))) == 31


def test_noll_diagonal_vs_weber_schafheitlin_integral():
    """<a_j^2> = 2 (n+1) C_W 2^{-5/3} (2 pi)^{11/3}/pi Int J_{n+1}(x)^2 x^{-14/3} dx -- the
    spectral route (Noll 1976 Eq.9 with W(f) = C_W r0^{-5/3} f^{-11/3}), by quadrature."""
    A = optics.noll_covariance(36, 1.0)
    for j in (2, 4, 7, 11, 16, 22, 29):
        n = optics.noll_nm(j)[0]
        g = lambda x: jv(n + 1, x) ** 2 * x ** (-14.0 / 3.0)
        I = sum(integrate.quad(g, a, b, limit=1000, epsabs=1e-15)[0]
                for a, b in [(0, 1), (1, 10), (10, 100), (100, 1e4)])
        v = 2 * (n + 1) * optics.C_W * 2 ** (-5 / 3) * (2 * np.pi) ** (11 / 3) / np.pi * I
        assert v == pytest.approx(A[j - 1, j - 1], rel=1e-6), j


def test_cholesky_factor():
    A = optics.noll_covariance(36, 3.0)
    L = optics.noll_cholesky(A)
    assert np.abs(L @ L.T - A).max() < 1e-12
    assert np.all(np.triu(L, 1) == 0)
    assert L[2, 1] == 0.0  # A0[2][3] = 0 => L_32 = 0 (tilt planes decouple)
    assert np.all(optics.noll_cholesky(optics.noll_covariance(36, 0.0)) == 0)


@pytest.mark.parametrize("d_over_r0", [1.0, 2.0, 4.0])
def test_structure_function_from_noll_matrix(d_over_r0):
    """Eq.4: D_phi over the aperture from the 36-term Noll matrix,
    E[(phi(p)-phi(p'))^2] = sum_ij A_ij dZ_i dZ_j, against 6.88 (r/r0)^{5/3}.

    Truncation at N = 36 removes small-scale power, so the ratio depends on r/D
    only, is < 1 and rises towards 1 with r; within 10% for
    r >= D/4 (SPEC's 10% acceptance)."""
    A = optics.noll_covariance(36, d_over_r0)
    rng = np.random.default_rng(1)
    ratios = []
    for r_over_D in (0.25, 0.5, 0.75):
        r = 2.0 * r_over_D  # separation in units of the aperture radius
        vals = []
        for _ in range(600):
            ang = rng.uniform(0, 2 * np.pi)
            while True:
                c = rng.uniform(-1, 1, 2)
                p1 = c - 0.5 * r * np.array([np.cos(ang), np.sin(ang)])
                p2 = c + 0.5 * r * np.array([np.cos(ang), np.sin(ang)])
                if np.hypot(*p1) <= 1 and np.hypot(*p2) <= 1:
                    break
            z1 = np.array([optics.zernike(j, np.hypot(*p1), np.arctan2(p1[1], p1[0])) for j in range(1, 37)])
            z2 = np.array([optics.zernike(j, np.hypot(*p2), np.arctan2(p2[1], p2[0])) for j in range(1, 37)])
            d = z1 - z2
            vals.append(d @ A @ d)
        th = optics.structure_function(r_over_D * d_over_r0, 1.0)
        ratios.append(np.mean(vals) / th)
    ratios = np.array(ratios)
    assert np.all(np.abs(ratios - 1) < 0.10), ratios
    assert np.all(ratios < 1.0) and np.all(np.diff(ratios) > -0.01), ratios


def test_geometry_defaults():
    s_px, kappa = optics.geometry()
    assert s_px == pytest.approx(0.02625, rel=1e-12)  # Q5
    assert kappa == pytest.approx(4 / np.pi)  # Q12
