"""Pins of the cross-correlation kernels and approximation energies (oracle/energies.py,
P:369-397):
  * A_ij(s) equals the independent 4-D structure-function quadrature (brute_force_Ajj) for
    same-m, cross-m, cos/sin-mixed and odd-harmonic pairs;
  * A_ij(0) is Noll's matrix (closed form) for every pair of modes 2..15;
  * A_ji(s) = A_ij(-s);
  * the energies vanish at s = 0 and the model is exact at zero lag; under reading Q25
    (angle-averaged correlation functions) E and E~ agree and E- << E, the paper's claims.
"""
import numpy as np
import pytest

from oracle import correlation, energies, optics


@pytest.mark.parametrize("i,j", [(2, 8), (3, 4), (2, 5), (4, 11), (5, 6), (6, 13), (7, 11), (9, 10)])
def test_cross_kernel_matches_brute_force(i, j):
    for sx, sy in ((0.6, 0.35), (1.3, -0.8)):
        bf = correlation.brute_force_Ajj(i, j, sx, sy, nr=20, nt=40)
        k = energies.cross_kernel(i, j, np.array([np.hypot(sx, sy)]), np.array([np.arctan2(sy, sx)]))[0]
        assert abs(k - bf) < 2e-3 * max(abs(bf), 1e-3) + 5e-7


def test_cross_kernel_zero_lag_is_noll_matrix():
    A0 = optics.noll_covariance(36, 2.0)
    for i in range(2, 16):
        for j in range(i, 16):
            k = energies.cross_kernel(i, j, np.array([0.0]), np.array([0.0]), 2.0)[0]
            assert abs(k - A0[i - 1, j - 1]) < 1e-4 * A0[1, 1]


def test_cross_kernel_transpose_is_reversed_lag():
    s, phi = np.array([0.7]), np.array([0.4])
    for i, j in ((2, 4), (5, 13), (7, 12)):
        a = energies.cross_kernel(i, j, s, phi)[0]
        b = energies.cross_kernel(j, i, s, phi + np.pi)[0]
        assert abs(a - b) < 1e-12 + 1e-9 * abs(a)


def test_energies_zero_at_origin_and_paper_claims_under_angle_mean():
    s, E, Et, Em = energies.energies(6.0, n_s=6, angle_mean=True)
    assert E[0] == Et[0] == Em[0] == 0.0
    assert abs(E[-1] - Et[-1]) / E[-1] < 0.1 and Em[-1] / E[-1] < 0.1
    # most of the residual is incurred at small separations
    k1 = int(np.searchsorted(s, 1.0))
    assert Em[k1] > 0.5 * Em[-1]
