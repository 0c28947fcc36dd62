"""Pins of the exact-PSF oracle (oracle/exact_psf.py; Eq.1-2, SURVEY NEXT-1 partial).

* zero phase gives the Airy pattern of a circular pupil: the sampled PSF follows
  [2 J1(pi r / 2) / (pi r / 2)]^2 (pixel = lambda/(2D)) and its first dark ring sits at
  2 * 3.8317 / pi = 2.44 px (textbook 1.22 lambda/D);
* a pure tilt shifts the PSF by -kappa a_2 with kappa = 4/pi (reading Q12 derived from the
  optics, not from the oracle's own constant), linearly for small a_2;
* unit sum and non-negativity; a defocus (Z_4) PSF is symmetric under u -> -u;
* the exact render of a constant image is that constant; with zero aberration it equals the
  plain convolution with the Airy PSF (brute-force loop).
"""
import numpy as np
from scipy.special import j1

from oracle import exact_psf, optics, pipeline


def test_zero_phase_is_airy():
    T = 15
    h = exact_psf.exact_psf(np.zeros(36), T)
    c = T // 2
    yy, xx = np.mgrid[-c:c + 1, -c:c + 1]
    r = np.hypot(yy, xx)
    v = np.pi * r / 2.0
    airy = np.where(r == 0, 1.0, (2 * j1(np.maximum(v, 1e-12)) / np.maximum(v, 1e-12)) ** 2)
    hn = h / h[c, c]
    assert np.max(np.abs(hn - airy)) < 0.03
    # the core ends at the first dark ring (2.44 px): half power near 1 px, < 5% at 2 px
    assert hn[c, c + 1] > 0.4 and hn[c, c + 2] < 0.05 and hn[c + 2, c] < 0.05


def test_tilt_shift_is_four_over_pi():
    T = 21
    c = T // 2
    for a2 in (0.05, 0.1, 0.2):
        a = np.zeros(36)
        a[1] = a2
        h = exact_psf.exact_psf(a, T)
        u = np.arange(T) - c
        cx = (h.sum(0) * u).sum()
        cy = (h.sum(1) * u).sum()
        assert abs(cx + 4.0 / np.pi * a2) < 0.02 * 4.0 / np.pi * a2 + 2e-3
        assert abs(cy) < 1e-9
        assert abs(optics.geometry()[1] - 4.0 / np.pi) < 1e-15


def test_unit_sum_nonnegative_and_defocus_symmetry():
    rng = np.random.default_rng(4)
    a = np.zeros(36)
    a[1:] = 0.3 * rng.standard_normal(35)
    h = exact_psf.exact_psf(a, 17)
    assert abs(h.sum() - 1) < 1e-12 and h.min() >= 0
    d = np.zeros(36)
    d[3] = 0.8  # Noll 4, defocus: rotationally symmetric phase
    hd = exact_psf.exact_psf(d, 17)
    assert np.allclose(hd, hd[::-1, ::-1], atol=1e-14)


def test_render_exact_constant_and_diffraction_limit():
    rng = np.random.default_rng(8)
    H, W, T = 9, 11, 7
    a = 0.2 * rng.standard_normal((36, H, W))
    a[0] = 0
    const = np.full((2, H, W), 0.37)
    assert np.allclose(exact_psf.render_exact(const, a, T), 0.37, atol=1e-12)
    img = rng.uniform(size=(1, H, W))
    zero = np.zeros((36, H, W))
    got = exact_psf.render_exact(img, zero, T)
    h = exact_psf.exact_psf(np.zeros(36), T)
    c = T // 2
    ref = np.zeros_like(img)
    for y in range(H):
        for x in range(W):
            s = 0.0
            for ty in range(T):
                for tx in range(T):
                    yy = pipeline.reflect_index(np.array([y - (ty - c)]), H)[0]
                    xx = pipeline.reflect_index(np.array([x - (tx - c)]), W)[0]
                    s += h[ty, tx] * img[0, yy, xx]
            ref[0, y, x] = s
    assert np.allclose(got, ref, atol=1e-12)
