"""Pins for oracle/correlation.py and the step-1 sampler of oracle/pipeline.py.

Routes that are independent of the code under test:
* Noll closed form (A_jj(0) = A_0[j][j]) for the Hankel radial integral;
* brute-force 4-D double-aperture quadrature of the structure function (Eq.4)
  for A_jj(s) at s != 0 (x and y lags, cos and sin branches);
* explicit DFT sums (not numpy.fft) for the circulant-eigenvalue identity of
  P:234-238 and the covariance of the sampled fields;
* the dense covariance tensor A~ = L blkdiag(A_11..A_NN) L^T of Eq.10
  assembled explicitly on a 16x16 crop ("dense Cholesky" oracle).
"""
import numpy as np
import pytest

from oracle import correlation as corr
from oracle import optics, pipeline


def test_hankel_zero_lag_equals_noll_diagonal():
    A = optics.noll_covariance(36, 1.0)
    for j in range(2, 37):
        assert corr.Ajj_quad(j, 0.0, 0.0) == pytest.approx(A[j - 1, j - 1], rel=1e-8), j


@pytest.mark.parametrize("j,sx,sy", [(2, 1.0, 0.0), (2, 0.0, 0.5), (3, 1.0, 0.0), (3, 0.4, 0.3),
                                     (4, 0.3, 0.0), (7, 0.45, 0.45), (8, 1.5, 0.0), (11, 0.0, 0.8),
                                     (12, 0.6, 0.2)])
def test_hankel_vs_brute_force_double_aperture(j, sx, sy):
    A = optics.noll_covariance(36, 1.0)
    s, phi = np.hypot(sx, sy), np.arctan2(sy, sx)
    h = corr.Ajj_quad(j, s, phi)
    bf = corr.brute_force_Ajj(j, j, sx, sy, nr=28, nt=56)
    assert abs(h - bf) < 2e-4 * A[j - 1, j - 1] + 1e-9, (h, bf)


def test_tilt_longitudinal_transverse_orientation():
    """x-tilt (Z2, cos) correlates less along x (longitudinal) than along y."""
    A22 = optics.noll_covariance(36, 1.0)[1, 1]
    cx = corr.Ajj_quad(2, 1.0, 0.0) / A22
    cy = corr.Ajj_quad(2, 1.0, np.pi / 2) / A22
    assert cx < cy
    # y-tilt is the 90-degree rotation of x-tilt
    assert corr.Ajj_quad(3, 1.0, np.pi / 2) / A22 == pytest.approx(cx, rel=1e-9)
    # i = 4, |s| = 8 -> |value| < 0.02 ("vanish for s > 4")
    A44 = optics.noll_covariance(36, 1.0)[3, 3]
    assert abs(corr.Ajj_quad(4, 8.0, 0.0) / A44) < 0.02


def test_radial_table_spline_vs_quad():
    A = optics.noll_covariance(36, 1.0)
    tab = corr.radial_tables_cached(3.0)
    sg, R = tab
    from scipy.interpolate import CubicSpline
    rng = np.random.default_rng(0)
    for _ in range(12):
        j = int(rng.integers(2, 37))
        s = float(rng.uniform(0, 2.9))
        phi = float(rng.uniform(-np.pi, np.pi))
        n, m, kind = optics.noll_nm(j)
        v = CubicSpline(sg, R[(n, 0)])(s)
        if m:
            sgn = 1 if kind == "cos" else -1
            v += sgn * (-1) ** m * CubicSpline(sg, R[(n, 2 * m)])(s) * np.cos(2 * m * phi)
        assert abs(v - corr.Ajj_quad(j, s, phi)) < 2e-6 * A[j - 1, j - 1], (j, s, phi)


def test_kernel_grid_properties():
    P, Q, s_px = 24, 30, 0.07
    c = corr.autocorrelation_kernels(P, Q, s_px, N=36)
    assert np.allclose(c[:, 0, 0], 1.0, atol=1e-12)
    assert np.abs(c).max() <= 1.0 + 1e-9
    # evenness in each axis separately (cos(2 m phi) is even under dx -> -dx and dy -> -dy)
    iy = (-np.arange(P)) % P
    ix = (-np.arange(Q)) % Q
    assert np.allclose(c, c[:, iy, :], atol=1e-12)
    assert np.allclose(c, c[:, :, ix], atol=1e-12)
    # direct evaluation at a few lags
    A = optics.noll_covariance(36, 1.0)
    for (j, y, x) in [(2, 0, 3), (3, 2, 0), (9, 5, 7), (36, 1, 1)]:
        s = s_px * np.hypot(y, x)
        v = corr.Ajj_quad(j, s, np.arctan2(y, x)) / A[j - 1, j - 1]
        assert c[j - 2, y, x] == pytest.approx(v, abs=2e-6)


def _explicit_dft2(c):
    P, Q = c.shape
    ky = np.arange(P)
    kx = np.arange(Q)
    Ey = np.exp(-2j * np.pi * np.outer(ky, ky) / P)
    Ex = np.exp(-2j * np.pi * np.outer(kx, kx) / Q)
    return Ey @ c @ Ex.T


def test_psd_is_dft_of_kernel_and_renormalised():
    P, Q = 16, 20
    c = corr.autocorrelation_kernels(P, Q, 0.1, N=6)
    for k in range(c.shape[0]):
        S, sq, frac = corr.psd_from_kernel(c[k])
        E = _explicit_dft2(c[k])
        assert np.abs(E.imag).max() < 1e-10 * np.abs(E.real).max()
        Sc = np.maximum(E.real, 0)
        Sc *= P * Q / Sc.sum()
        assert np.allclose(S, Sc, atol=1e-10)
        assert S.sum() == pytest.approx(P * Q, rel=1e-12)
        assert np.allclose(sq ** 2, S)


def _field_linear_map(sqrtS_pair, P, Q, H, W):
    """Columns = fields (f_a, f_b) produced by each independent unit Gaussian."""
    canon, is_canon, is_self = pipeline.bin_symmetry(P, Q)
    cols = []
    M = sqrtS_pair.shape[0]
    for c in np.unique(canon):
        sel = (canon == c)
        selfc = bool(is_self[sel].all())
        for which in range(M):
            for comp in ((0,) if selfc else (0, 1)):
                g1 = np.where(sel, 1.0 if comp == 0 else 0.0, 0.0)
                g2 = np.where(sel, 1.0 if comp == 1 else 0.0, 0.0)
                eta = np.zeros((M, P, Q), dtype=complex)
                eta[which] = pipeline.eta_from_gaussians(g1, g2)
                f = pipeline.fields_from_noise(eta, sqrtS_pair, H, W)
                cols.append(f.reshape(-1))
    return np.array(cols).T


def test_sampler_exact_covariance_tiny_grid():
    """C4: Cov(f_a) = circ(IDFT S_a), Cov(f_b) = circ(IDFT S_b), Cov(f_a, f_b) = 0 (8 x 6)."""
    P, Q = 8, 6
    c = corr.autocorrelation_kernels(P, Q, 0.15, N=3)  # modes 2, 3 -> one complex pair
    sq = np.stack([corr.psd_from_kernel(c[k])[1] for k in range(2)])
    Mlin = _field_linear_map(sq, P, Q, P, Q)
    Cov = Mlin @ Mlin.T
    n = P * Q
    for k in range(2):
        S = sq[k] ** 2
        # circulant from explicit inverse-DFT sums
        ky, kx = np.meshgrid(np.arange(P), np.arange(Q), indexing="ij")
        r = np.empty((P, Q))
        for y in range(P):
            for x in range(Q):
                r[y, x] = (S * np.cos(2 * np.pi * (ky * y / P + kx * x / Q))).sum() / n
        Cexp = np.empty((n, n))
        for i in range(n):
            for jj in range(n):
                Cexp[i, jj] = r[(i // Q - jj // Q) % P, (i % Q - jj % Q) % Q]
        blk = Cov[k * n:(k + 1) * n, k * n:(k + 1) * n]
        assert np.abs(blk - Cexp).max() < 1e-12
    assert np.abs(Cov[:n, n:]).max() < 1e-12


def test_sampler_vs_dense_eq10_tensor():
    """C5 / SPEC S:214: 12x12 crop of a 24x24 periodic grid (pad 2), modes 2..7.

    The exact covariance of the sampler output after mixing equals Eq.10's
    A~ = (L x I) blkdiag(C_2..C_7) (L x I)^T, C_j[x,x'] = A_jj(x-x')/A_jj(0) evaluated
    directly (scipy quad), up to the clamp/renormalise step (reading Q7)."""
    N, H, W, P, Q, s_px = 7, 12, 12, 24, 24, 0.12
    A0 = optics.noll_covariance(N, 2.0)
    L = optics.noll_cholesky(A0)
    c = corr.autocorrelation_kernels(P, Q, s_px, N=N)
    S_list = [corr.psd_from_kernel(c[k]) for k in range(N - 1)]
    # exact per-mode crop covariance from the (clamped) PSD: IDFT(S) at crop lags
    n = H * W
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    yy, xx = yy.ravel(), xx.ravel()
    dY = (yy[:, None] - yy[None, :]) % P
    dX = (xx[:, None] - xx[None, :]) % Q
    blk_s, blk_d = [], []
    A1 = optics.noll_covariance(N, 1.0)  # Ajj_quad is evaluated at D/r0 = 1
    DYs = yy[:, None] - yy[None, :]
    DXs = xx[:, None] - xx[None, :]
    for k in range(N - 1):
        r = np.fft.ifft2(S_list[k][0]).real
        blk_s.append(r[dY, dX])
        j = k + 2
        # direct quad on the quadrant of lags; c_j is even in each axis
        T = np.empty((H, W))
        for y in range(H):
            for x in range(W):
                T[y, x] = corr.Ajj_quad(j, s_px * np.hypot(y, x), np.arctan2(y, x)) / A1[j - 1, j - 1]
        blk_d.append(T[np.abs(DYs), np.abs(DXs)])

    def mixed(blks):
        Lm = L[1:, 1:]
        out = np.zeros(((N - 1) * n, (N - 1) * n))
        for a in range(N - 1):
            for b in range(N - 1):
                acc = np.zeros((n, n))
                for k in range(N - 1):
                    if Lm[a, k] and Lm[b, k]:
                        acc += Lm[a, k] * Lm[b, k] * blks[k]
                out[a * n:(a + 1) * n, b * n:(b + 1) * n] = acc
        return out

    As, Ad = mixed(blk_s), mixed(blk_d)
    rel = np.linalg.norm(As - Ad) / np.linalg.norm(Ad)
    assert rel < 0.05, rel  # SPEC's 5% Frobenius; exact up to the clamp
    # at zero lag Eq.10 reproduces the Noll matrix exactly ("no loss at s = 0")
    for a in range(N - 1):
        for b in range(N - 1):
            assert Ad[a * n, b * n] == pytest.approx(A0[a + 1, b + 1], abs=1e-12)


def test_sampler_monte_carlo_statistics():
    """Philox noise path end-to-end: per-pixel Noll covariance and the sampled
    spatial autocovariance vs IDFT(S), 1500 frames on a 24 x 20 grid."""
    N, P, Q, s_px = 7, 24, 20, 0.12
    A0 = optics.noll_covariance(N, 3.0)
    L = optics.noll_cholesky(A0)
    c = corr.autocorrelation_kernels(P, Q, s_px, N=N)
    sq = np.stack([corr.psd_from_kernel(c[k])[1] for k in range(N - 1)])
    a = pipeline.sample_zernike(2210, 0, 1500, sq, L, P, Q)
    # pixel-wise covariance across modes (pooled over pixels)
    X = a[:, 1:].transpose(1, 0, 2, 3).reshape(N - 1, -1)
    C = X @ X.T / X.shape[1]
    ref = A0[1:, 1:]
    assert np.linalg.norm(C - ref) / np.linalg.norm(ref) < 0.05
    # 4-sigma bound on the tilt variance (SURVEY C6 with n_eff = (PQ)^2 / sum S^2)
    S2 = sq[0] ** 2
    sig = ref[0, 0] * np.sqrt(2 * (S2 ** 2).sum()) / (P * Q * np.sqrt(a.shape[0]))
    assert abs(C[0, 0] - ref[0, 0]) < 4 * sig
    # spatial autocorrelation of the unmixed field f_4 at lag (0, 1) vs IDFT(S_4)
    f = np.stack([pipeline.fields_from_noise(e, sq, P, Q)
                  for e in pipeline.spectral_noise_sequence(7, 0, 600, P, Q, 0.0, N)])
    r_emp = (f[:, 2] * np.roll(f[:, 2], -1, axis=2)).mean()
    r_th = np.fft.ifft2(sq[2] ** 2).real[0, 1]
    assert abs(r_emp - r_th) < 0.03
    kurt = ((f[:, 2] ** 4).mean() / (f[:, 2] ** 2).mean() ** 2)
    assert 2.8 < kurt < 3.2


def test_ar1_replay_and_correlation():
    P, Q, N = 8, 8, 5
    seq = list(pipeline.spectral_noise_sequence(11, 0, 9, P, Q, 0.9, N))
    part = list(pipeline.spectral_noise_sequence(11, 5, 4, P, Q, 0.9, N))
    for x, y in zip(seq[5:], part):
        assert np.array_equal(x, y)
    white = list(pipeline.spectral_noise_sequence(11, 0, 3, P, Q, 0.0, N))
    assert np.array_equal(white[0], seq[0])
    # lag-1 correlation of eta ~ alpha
    long = np.stack(list(pipeline.spectral_noise_sequence(3, 0, 400, P, Q, 0.8, N)))
    x, y = long[:-1].real.ravel(), long[1:].real.ravel()
    assert np.corrcoef(x, y)[0, 1] == pytest.approx(0.8, abs=0.03)
    _, _, is_self = pipeline.bin_symmetry(P, Q)
    expect = (P * Q / 2 * (1 + is_self)).mean()  # self-conjugate bins carry sqrt(PQ) g1
    assert (long.real ** 2).mean() == pytest.approx(expect, rel=0.05)


def test_clamped_psd_fraction_reported():
    """Reading Q7: the negative mass of the circulant embedding shrinks with grid size."""
    s_px = 0.02625
    f64 = corr.psd_from_kernel(corr.autocorrelation_kernels(64, 64, s_px, N=3)[0])[2]
    f256 = corr.psd_from_kernel(corr.autocorrelation_kernels(256, 256, s_px, N=3)[0])[2]
    assert 0 < f256 < f64 < 0.1


# ------------------------------------------------------------------ frozen flow (NEXT-3)
def test_frozen_flow_integer_velocity_is_a_periodic_roll():
    """frame t is the frame-0 field translated by v t; for integer v t the
    spectral shift factors reproduce np.roll exactly (the Nyquist cos(pi s) = (-1)^s)."""
    from oracle import pipeline, optics, correlation
    P, Q, N = 12, 16, 36
    sq, _ = correlation.sqrt_psd_tables(P, Q, optics.geometry()[0], N)
    L = optics.noll_cholesky(optics.noll_covariance(N, 2.0))
    a = pipeline.sample_zernike(7, 0, 4, sq, L, P, Q, flow=(2.0, -1.0))
    for t in range(4):
        assert np.allclose(a[t], np.roll(a[0], (-1 * t, 2 * t), axis=(1, 2)), atol=1e-12)


def test_frozen_flow_fractional_shifts_compose_and_stay_real():
    from oracle import pipeline
    n = 10
    for s1, s2 in ((0.3, 0.45), (1.25, -0.7)):
        p = pipeline.flow_phase_1d(n, s1) * pipeline.flow_phase_1d(n, s2)
        q = pipeline.flow_phase_1d(n, s1 + s2)
        assert np.allclose(p[np.arange(n) != n // 2], q[np.arange(n) != n // 2], atol=1e-12)
        ph = pipeline.flow_phase_1d(n, s1)
        k = np.arange(n)
        assert np.allclose(ph[(n - k) % n], np.conj(ph), atol=1e-15)  # Hermitian: real fields
    # band-limited translation of a pure tone is exact at any sub-pixel shift
    x = np.arange(n)
    f = np.cos(2 * np.pi * 3 * x / n + 0.4)
    g = np.real(np.fft.ifft(np.fft.fft(f) * pipeline.flow_phase_1d(n, 0.37)))
    assert np.allclose(g, np.cos(2 * np.pi * 3 * (x - 0.37) / n + 0.4), atol=1e-12)
