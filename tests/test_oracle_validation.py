"""Pins of the validation-battery oracle (oracle/validation.py).

Each pin is fixed by mathematics, not by re-running the oracle's own formula:
  * the estimator of a pure sinusoid is (A^2/2) cos(2 pi k l / W) exactly (periodic lags);
  * on random arrays it equals an explicit quadruple loop (brute force, tiny sizes);
  * the realised kernels of a delta PSD (white field) are delta functions; of a single
    Fourier mode, a cosine;
  * the model at zero lag is diag(L L^T) = diag(A_0) (Noll matrix), because every
    realised kernel has unit variance (sum S = P Q);
  * the differential tilt variance vanishes at zero lag and equals 2(R(0) - R(l)).
"""
import numpy as np

from oracle import correlation, optics, validation


def test_sinusoid_autocorr_closed_form():
    F, Z, H, W, L = 2, 3, 12, 40, 9
    y, x = np.mgrid[0:H, 0:W]
    f = np.zeros((F, Z, H, W))
    f[:, 1] = 1.7 * np.cos(2 * np.pi * 3 * x / W + 0.3)  # along x
    f[:, 2] = 0.9 * np.cos(2 * np.pi * 2 * y / H - 1.1)  # along y
    R = validation.empirical_autocorr(f, L)
    l = np.arange(L)
    assert np.allclose(R[1, 0], 0.5 * 1.7 ** 2 * np.cos(2 * np.pi * 3 * l / W), atol=1e-12)
    assert np.allclose(R[1, 1], 0.5 * 1.7 ** 2, atol=1e-12)  # constant along y
    assert np.allclose(R[2, 1], 0.5 * 0.9 ** 2 * np.cos(2 * np.pi * 2 * l / H), atol=1e-12)
    assert np.allclose(R[0], 0.0)


def test_autocorr_equals_brute_force_loops():
    rng = np.random.default_rng(5)
    F, Z, H, W, L = 2, 2, 5, 7, 4
    a = rng.standard_normal((F, Z, H, W))
    R = validation.empirical_autocorr(a, L)
    for j in range(Z):
        for l in range(L):
            sx = sy = 0.0
            for f in range(F):
                for yy in range(H):
                    for xx in range(W):
                        sx += a[f, j, yy, xx] * a[f, j, yy, (xx + l) % W]
                        sy += a[f, j, yy, xx] * a[f, j, (yy + l) % H, xx]
            n = F * H * W
            assert abs(R[j, 0, l] - sx / n) < 1e-12 and abs(R[j, 1, l] - sy / n) < 1e-12


def test_realised_kernels_delta_and_cosine():
    P, Q, L = 8, 10, 5
    white = np.ones((1, P, Q))  # S = 1 everywhere: white field, c = delta
    c = validation.realised_kernels(white, L)
    assert np.allclose(c[0, :, 0], 1.0) and np.allclose(c[0, :, 1:], 0.0, atol=1e-15)
    S = np.zeros((1, P, Q))
    S[0, 0, 3] = S[0, 0, Q - 3] = P * Q / 2  # one real Fourier mode along x, unit variance
    c = validation.realised_kernels(np.sqrt(S), L)
    l = np.arange(L)
    assert np.allclose(c[0, 0], np.cos(2 * np.pi * 3 * l / Q), atol=1e-12)
    assert np.allclose(c[0, 1], 1.0, atol=1e-12)


def test_model_zero_lag_is_noll_diagonal():
    Z = 36
    A0 = optics.noll_covariance(Z, 3.0)
    Lc = optics.noll_cholesky(A0)
    sq, _ = correlation.sqrt_psd_tables(16, 16, optics.geometry()[0], Z)
    kern = validation.realised_kernels(sq, 4)
    assert np.allclose(kern[:, :, 0], 1.0, atol=1e-12)
    R = validation.model_autocorr(Lc, kern)
    assert np.allclose(R[1:, 0, 0], np.diag(A0)[1:], rtol=1e-10)
    assert np.allclose(R[1:, 1, 0], np.diag(A0)[1:], rtol=1e-10)
    assert np.all(R[0] == 0)


def test_differential_tilt_variance_identity():
    rng = np.random.default_rng(1)
    R = rng.standard_normal((36, 2, 6))
    D = validation.differential_tilt_variance(R)
    assert np.allclose(D[:, :, 0], 0.0)
    assert np.allclose(D, 2 * (R[1:3, :, :1] - R[1:3]))
