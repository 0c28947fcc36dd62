"""Pins for steps 2-5 of oracle/pipeline.py (warp, P2S MLP, Eq.9 blur, step 5).

Independent routes: closed forms (identity, integer shift, bilinear exactness on
affine images, constant images), scipy.ndimage.convolve(mode='mirror') for the
spatially invariant special case of Eq.9, torch.nn.functional for
the MLP, and the D/r0 = 0 end-to-end special case.
"""
import numpy as np
import pytest
import scipy.ndimage as ndi

import synth
from oracle import optics, pipeline
from oracle import correlation as corr


# ------------------------------------------------------------------ warp (step 2)
def test_warp_zero_displacement_identity():
    img = synth.image(20, 24, 2, seed=1).astype(np.float64)
    z = np.zeros((20, 24))
    assert np.array_equal(pipeline.warp(img, z, z, 4 / np.pi), img)


def test_warp_integer_shift_and_clamp():
    img = synth.image(16, 18, 1, seed=2).astype(np.float64)
    out = pipeline.warp(img, np.full((16, 18), 3.0), np.full((16, 18), -2.0), 1.0)
    # out(y, x) = I(y - 2, x + 3), clamped to the border
    ys = np.clip(np.arange(16) - 2, 0, 15)
    xs = np.clip(np.arange(18) + 3, 0, 17)
    assert np.array_equal(out[0], img[0][ys][:, xs])


def test_warp_bilinear_exact_on_affine_image():
    H, W = 30, 40
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    img = (0.3 * xx - 0.7 * yy + 2.0)[None].astype(np.float64)
    rng = np.random.default_rng(0)
    a2 = rng.uniform(-2, 2, (H, W))
    a3 = rng.uniform(-2, 2, (H, W))
    kappa = 1.3
    out = pipeline.warp(img, a2, a3, kappa)
    X, Y = xx + kappa * a2, yy + kappa * a3
    inside = (X >= 0) & (X <= W - 1) & (Y >= 0) & (Y <= H - 1)
    assert np.abs(out[0] - (0.3 * X - 0.7 * Y + 2.0))[inside].max() < 1e-12
    assert inside.mean() > 0.8


# ------------------------------------------------------------------ MLP (step 3)
def test_mlp_degenerate_cases():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(33, 5, 7))
    K = 16
    layers = [(np.zeros((100, 33)), rng.normal(size=100)), (np.zeros((100, 100)), rng.normal(size=100)),
              (np.zeros((K, 100)), rng.normal(size=K))]
    out = pipeline.mlp(x, layers)
    assert np.allclose(out, layers[2][1][:, None, None])
    # identity layers with non-negative input pass the input through the ReLUs
    xp = np.abs(x)
    ident = [(np.eye(33), np.zeros(33))] * 3
    assert np.allclose(pipeline.mlp(xp, ident), xp)


def test_mlp_vs_torch_functional():
    torch = pytest.importorskip("torch")
    K = 100
    layers = synth.unpack_mlp(synth.mlp_weights(K, seed=3), K)
    rng = np.random.default_rng(2)
    x = rng.normal(size=(33, 6, 9)) * 0.2
    h = torch.tensor(x.reshape(33, -1).T)
    for i, (Wm, b) in enumerate(layers):
        h = torch.nn.functional.linear(h, torch.tensor(Wm), torch.tensor(b))
        if i < 2:
            h = torch.relu(h)
    ref = h.numpy().T.reshape(K, 6, 9)
    assert np.abs(pipeline.mlp(x, layers) - ref).max() < 1e-12


# ------------------------------------------------------------------ blur (step 4)
def test_blur_delta_basis_is_identity():
    Iw = synth.image(21, 17, 3, seed=4).astype(np.float64)
    T = 9
    h = np.zeros((1, T, T))
    h[0, T // 2, T // 2] = 1.0
    w = np.ones((1, 21, 17))
    assert np.allclose(pipeline.blur(Iw, w, h), Iw, atol=0, rtol=0)


def test_blur_shifted_delta_pins_convolution_orientation():
    Iw = synth.image(15, 19, 1, seed=5).astype(np.float64)
    T = 5
    h = np.zeros((1, T, T))
    h[0, T // 2 + 1, T // 2 - 2] = 1.0  # tap u = (+1, -2)
    out = pipeline.blur(Iw, np.ones((1, 15, 19)), h)
    # true convolution: out(y, x) = Iw(refl(y - 1), refl(x + 2))
    ys = pipeline.reflect_index(np.arange(15) - 1, 15)
    xs = pipeline.reflect_index(np.arange(19) + 2, 19)
    assert np.array_equal(out[0], Iw[0][ys][:, xs])


def test_blur_single_basis_vs_scipy_mirror_convolve():
    Iw = synth.image(23, 29, 2, seed=6).astype(np.float64)
    h = synth.basis(1, 11, seed=7).astype(np.float64)
    h[0] += 0.01 * np.arange(121).reshape(11, 11) / 121  # break symmetry
    w = np.full((1, 23, 29), 2.5)
    out = pipeline.blur(Iw, w, h)
    for c in range(2):
        ref = 2.5 * ndi.convolve(Iw[c], h[0], mode="mirror")
        assert np.abs(out[c] - ref).max() < 1e-12


def test_blur_linear_in_weights_and_constant_image():
    rng = np.random.default_rng(8)
    K, T, H, W = 5, 7, 12, 13
    h = synth.basis(K, T, seed=9).astype(np.float64)
    Iw = synth.image(H, W, 1, seed=10).astype(np.float64)
    w1 = rng.normal(size=(K, H, W))
    w2 = rng.normal(size=(K, H, W))
    o = pipeline.blur(Iw, w1 + w2, h)
    assert np.allclose(o, pipeline.blur(Iw, w1, h) + pipeline.blur(Iw, w2, h), atol=1e-12)
    # constant image c0: out = c0 * sum_k w_k sum_u h_k (unit-sum basis)
    const = np.full((1, H, W), 0.37)
    assert np.allclose(pipeline.blur(const, w1, h)[0], 0.37 * w1.sum(0), atol=1e-12)
    # sampled evaluation agrees with the full one
    ys, xs = rng.integers(0, H, 20), rng.integers(0, W, 20)
    sub = pipeline.blur_at(Iw, w1[:, ys, xs].T, h, ys, xs)
    assert np.allclose(sub[0], o[0][ys, xs] - pipeline.blur(Iw, w2, h)[0][ys, xs], atol=1e-12)


# ------------------------------------------------------------------ step 5
def test_step5_normalise_noise_clamp():
    K, T, H, W = 4, 5, 40, 50
    h = synth.basis(K, T, seed=11).astype(np.float64)
    rng = np.random.default_rng(3)
    w = rng.uniform(0.1, 1.0, (K, H, W))
    const = np.full((2, H, W), 0.6)
    out = pipeline.blur(const, w, h)
    norm = pipeline.step5(out, w, h, 5, 0, normalize=True)
    assert np.allclose(norm, 0.6, atol=1e-12)
    noisy = pipeline.step5(norm, w, h, 5, 3, sigma=0.1)
    z = (noisy - norm) / 0.1
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1) < 0.03
    assert not np.allclose(z[0], z[1])  # channels draw distinct noise
    again = pipeline.step5(norm, w, h, 5, 3, sigma=0.1)
    assert np.array_equal(noisy, again)
    cl = pipeline.step5(out * 3 - 1, w, h, 5, 3, clamp01=True)
    assert cl.min() >= 0 and cl.max() <= 1


def test_step5_at_sampled_pixels_equals_full_frame():
    """step5_at (used at full sizes) evaluated at sample pixels equals step5 on the frame."""
    K, T, H, W = 4, 5, 30, 44
    h = synth.basis(K, T, seed=2).astype(np.float64)
    rng = np.random.default_rng(9)
    w = rng.uniform(-0.2, 1.0, (K, H, W))
    out = rng.uniform(-0.5, 1.5, (3, H, W))
    ys, xs = rng.integers(0, H, 50), rng.integers(0, W, 50)
    for kw in (dict(sigma=0.05), dict(normalize=True, clamp01=True), dict(sigma=0.1, normalize=True, clamp01=True)):
        full = pipeline.step5(out, w, h, 17, 4, **kw)
        at = pipeline.step5_at(out[:, ys, xs], w[:, ys, xs].T, h, 17, 4, ys, xs, W, **kw)
        assert np.allclose(at, full[:, ys, xs], rtol=0, atol=1e-12)


# ------------------------------------------------------------------ end to end
def _small_plan(H, W, N=36, d_over_r0=2.0, s_px=0.02625):
    A0 = optics.noll_covariance(N, d_over_r0)
    L = optics.noll_cholesky(A0)
    sq, _ = corr.sqrt_psd_tables(H, W, s_px, N)
    return A0, L, sq


def test_end_to_end_zero_turbulence_is_invariant_blur():
    """D/r0 = 0 => a = 0 => Iw = I => w = MLP(0) everywhere =>
    out = I (*) sum_k w_k(0) h_k, a spatially invariant blur."""
    H, W, C, K, T = 32, 40, 2, 16, 9
    _, L, sq = _small_plan(H, W, d_over_r0=0.0)
    img = synth.image(H, W, C, seed=12)[None]
    h = synth.basis(K, T, seed=13)
    layers = synth.unpack_mlp(synth.mlp_weights(K, seed=14), K)
    out = pipeline.simulate(img, True, 2210, 0, 2, sq, L, h, layers, 4 / np.pi)
    w0 = pipeline.mlp(np.zeros((33, 1, 1)), layers)[:, 0, 0]
    heff = np.einsum("k,ktu->tu", w0, h.astype(np.float64))
    for f in range(2):
        for c in range(C):
            ref = ndi.convolve(img[0, c].astype(np.float64), heff, mode="mirror")
            assert np.abs(out[f, c] - ref).max() < 1e-12


def test_end_to_end_deterministic_and_seed_dependent():
    H, W, K, T = 24, 20, 8, 7
    _, L, sq = _small_plan(H, W)
    img = synth.image(H, W, 1, seed=15)[None]
    h = synth.basis(K, T, seed=16)
    layers = synth.unpack_mlp(synth.mlp_weights(K, seed=17), K)
    a = pipeline.simulate(img, True, 1, 0, 2, sq, L, h, layers, 4 / np.pi)
    b = pipeline.simulate(img, True, 1, 0, 2, sq, L, h, layers, 4 / np.pi)
    c = pipeline.simulate(img, True, 2, 0, 2, sq, L, h, layers, 4 / np.pi)
    assert np.array_equal(a, b)
    assert not np.allclose(a, c)
    # frame f of a batch equals the same frame run alone (counter-based noise)
    d = pipeline.simulate(img, True, 1, 1, 1, sq, L, h, layers, 4 / np.pi)
    assert np.array_equal(a[1], d[0])
