"""Pins of the aperture-statistics oracle (oracle/aperture.py, SURVEY 8(f) NEXT-2,
P:477-500), each fixed by mathematics rather than by the oracle's own formulas:

  * zero phase: SF = 0 and LE = SE = cnt(xi)/cnt(0), with cnt the overlap of the
    discrete disc counted by explicit loops (brute force);
  * the discrete pupil's overlap approaches the analytic diffraction OTF of the disc;
  * a pure tilt phi = 2 a_2 X is a plane: Delta = -2 a_2 (2 dx / Dp) exactly, so
    SF = Delta^2, LE = cnt cos(Delta) / cnt(0) and SE (tilt removed) = diffraction;
    adding any plane to a phase leaves SE unchanged;
  * Monte Carlo: Gaussian vectors a ~ N(0, A_0) drawn with numpy reproduce the model
    E[Delta^2] = dZ^T A_0 dZ, E[cos Delta] = exp(-E[Delta^2]/2) within 5 standard errors;
  * the Kolmogorov curves: D(r0) = C_D = 6.88 at r = r0 and H_LE = H_diff e^{-D/2}.
"""
import numpy as np

from oracle import aperture as ap
from oracle import optics


def test_zero_phase_is_diffraction_by_brute_force():
    Dp = 8
    X, Y, m = ap.pupil_coords(Dp)
    cnt = np.zeros((Dp, 2 * Dp - 1))
    for dy in range(Dp):
        for i, dx in enumerate(range(-(Dp - 1), Dp)):
            for y in range(Dp):
                for x in range(Dp):
                    y2, x2 = y + dy, x + dx
                    if 0 <= y2 < Dp and 0 <= x2 < Dp and m[y, x] and m[y2, x2]:
                        cnt[dy, i] += 1
    assert np.array_equal(ap.lag_overlap(Dp), cnt)
    SF, LE, SE = ap.aperture_stats(np.zeros((3, 10)), Dp)
    assert np.all(SF == 0)
    assert np.allclose(LE, cnt / cnt[0, Dp - 1]) and np.allclose(SE, cnt / cnt[0, Dp - 1])


def test_discrete_pupil_overlap_approaches_disc_otf():
    cnt = ap.lag_overlap(32)
    H = cnt / cnt[0, 31]
    assert np.max(np.abs(H - ap.diffraction_otf(ap.lag_radius(32)))) < 0.03


def test_pure_tilt_closed_form_and_plane_invariance():
    Dp, a2 = 16, 0.7
    a = np.zeros((1, 6))
    a[0, 1] = a2
    SF, LE, SE = ap.aperture_stats(a, Dp)
    cnt = ap.lag_overlap(Dp)
    dx = np.arange(-(Dp - 1), Dp)[None, :] * np.ones((Dp, 1))
    delta = 2 * a2 * 2 * dx / Dp
    on = cnt > 0
    assert np.allclose(SF[on], (delta ** 2)[on], rtol=1e-12, atol=1e-14)
    assert np.allclose(LE, cnt * np.cos(delta) / cnt[0, Dp - 1], atol=1e-12)
    assert np.allclose(SE, cnt / cnt[0, Dp - 1], atol=1e-12)
    # defocus + coma with and without an added plane: SE identical
    b = np.zeros((1, 8))
    b[0, 3], b[0, 6] = 0.9, -0.4
    c = b.copy()
    c[0, 1], c[0, 2] = 1.3, -0.8
    assert np.allclose(ap.aperture_stats(b, Dp)[2], ap.aperture_stats(c, Dp)[2], atol=1e-12)


def test_monte_carlo_matches_gaussian_model():
    Dp, Z, dr0 = 12, 10, 2.0
    A0 = optics.noll_covariance(Z, dr0)
    rng = np.random.default_rng(7)
    a = np.zeros((4000, Z))
    a[:, 1:] = rng.multivariate_normal(np.zeros(Z - 1), A0[1:, 1:], size=4000)
    batches = [ap.aperture_stats(b, Dp) for b in np.split(a, 10)]
    emp = np.mean(batches, axis=0)
    se = np.std(batches, axis=0, ddof=1) / np.sqrt(10)
    model = np.array(ap.model_stats(A0, Dp))
    on = ap.lag_overlap(Dp) > 0
    for k in range(3):
        z = np.abs(emp[k] - model[k])[on] / (se[k][on] + 1e-12)
        assert z.max() < 5.0, (k, z.max())


def test_kolmogorov_curves():
    D, LE, SE = ap.theory_curves(np.array([0.0, 0.25, 1.0]), 4.0)
    assert abs(D[1] - optics.C_D) < 1e-12  # r = D/4 = r0
    assert LE[0] == 1.0 and SE[0] == 1.0 and LE[2] == 0.0
    assert abs(LE[1] - ap.diffraction_otf(0.25) * np.exp(-optics.C_D / 2)) < 1e-15
    assert SE[1] > LE[1]
