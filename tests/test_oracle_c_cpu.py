"""Pins of the C oracle (oracle/p2s_oracle.c: naive DFT, scalar MLP, direct Eq.9).

It inherits the numpy oracle's pins by agreeing with it function by function (1e-12,
tests/test_oracle_*.py pin the numpy oracle against the paper and the mathematics), and
has its own: the Random123 Philox known-answer vectors, the IDFT sign on a single tone
(a spectrum with one canonical bin k0 and its conjugate mirror is 2 Re(c e^{+2 pi i k0.x})/PQ,
so y(x) and y(-x) -- equal in distribution -- are told apart), and the full frame against
the numpy pipeline.
"""
import os

import numpy as np
import pytest

import synth
from oracle import c_oracle, correlation, optics, pipeline

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.skipif(not os.path.exists(c_oracle.LIB), reason="libp2s_oracle.so not built")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300)


def test_philox_known_answers():
    for line in open(os.path.join(ROOT, "tests", "golden", "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        assert list(c_oracle.philox(v[0:4], v[4:6])) == v[6:10]


@pytest.mark.parametrize("P,Q", [(8, 6), (9, 10), (16, 15)])
def test_white_noise_equals_numpy_oracle(P, Q):
    for frame in (0, 3, (1 << 33) + 5):
        assert rel(c_oracle.white_noise(2210, frame, P, Q), pipeline.white_spectral_noise(2210, frame, P, Q)) < 1e-13


def test_ar_update_equals_numpy_recursion():
    seq = list(pipeline.spectral_noise_sequence(7, 0, 3, 10, 12, 0.9))
    eta = c_oracle.white_noise(7, 0, 10, 12)
    for t in (1, 2):
        eta = c_oracle.ar_update(eta, c_oracle.white_noise(7, t, 10, 12), 0.9)
        assert rel(eta, seq[t]) < 1e-13


def test_idft_sign_single_tone():
    """Y = delta at the canonical bin (ky0, kx0) and the conjugate at its mirror, mode a
    only: y(x) = (2/PQ) Re(e^{+2 pi i (ky0 y / P + kx0 x / Q)}) for f_a; with an imaginary
    amplitude i the field is -(2/PQ) sin(...), whose sign flips under x -> -x."""
    P, Q, H, W = 12, 10, 12, 10
    ky0, kx0 = 2, 3
    eta = np.zeros((35, P, Q), np.complex128)
    eta[0, ky0, kx0] = 1j
    eta[0, (P - ky0) % P, (Q - kx0) % Q] = -1j
    sq = np.ones((35, P, Q))
    f = c_oracle.fields(eta, sq, H, W)
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    ph = 2 * np.pi * (ky0 * yy / P + kx0 * xx / Q)
    assert np.abs(f[0] - (-2.0 / (P * Q)) * np.sin(ph)).max() < 1e-15
    assert np.abs(f[1:]).max() < 1e-15  # f_b = Im y: the conjugate pair cancels to rounding
    assert rel(f, pipeline.fields_from_noise(eta, sq, H, W)) < 1e-12


@pytest.mark.parametrize("P,Q,H,W", [(16, 15, 16, 15), (18, 20, 13, 17)])
def test_fields_and_mix_equal_numpy_oracle(P, Q, H, W):
    s_px = optics.geometry()[0]
    sq, _ = correlation.sqrt_psd_tables(P, Q, s_px, 36)
    eta = pipeline.white_spectral_noise(5, 2, P, Q)
    f = c_oracle.fields(eta, sq, H, W)
    fr = pipeline.fields_from_noise(eta, sq, H, W)
    assert rel(f, fr) < 1e-12
    L = optics.noll_cholesky(optics.noll_covariance(36, 3.0))
    assert rel(c_oracle.mix(f, L), pipeline.mix(fr, L)) < 1e-12


def test_warp_mlp_blur_step5_equal_numpy_oracle():
    H, W, C, K, T = 21, 26, 2, 7, 9
    rng = np.random.default_rng(0)
    img = synth.image(H, W, C, seed=2).astype(np.float64)
    a2, a3 = 3.0 * rng.standard_normal((2, H, W))
    kappa = optics.geometry()[1]
    Iw = c_oracle.warp(img, a2, a3, kappa)
    assert rel(Iw, pipeline.warp(img, a2, a3, kappa)) < 1e-13
    packed = synth.mlp_weights(K, hidden=(12, 10), n_in=33, seed=4).astype(np.float64)
    x = rng.standard_normal((33, H, W))
    w = c_oracle.mlp(x, packed, K, hidden=(12, 10))
    wr = pipeline.mlp(x, synth.unpack_mlp(packed, K, hidden=(12, 10)))
    assert rel(w, wr) < 1e-13
    basis = synth.basis(K, T, seed=3).astype(np.float64)
    out = c_oracle.blur(Iw, w, basis)
    ref = pipeline.blur(Iw, w, basis)
    assert rel(out, ref) < 1e-12
    ys = np.array([0, 5, H - 1, 20])
    xs = np.array([0, W - 1, 7, 25])
    assert rel(c_oracle.blur(Iw, w, basis, ys, xs), pipeline.blur_at(Iw, w[:, ys, xs].T, basis, ys, xs)) < 1e-12
    for sigma, norm, clamp in [(0.05, False, True), (0.0, True, False), (0.02, True, True)]:
        got = c_oracle.step5(out, w, basis, 11, 4, sigma, norm, clamp)
        exp = pipeline.step5(out, w, basis, 11, 4, sigma=sigma, normalize=norm, clamp01=clamp)
        assert rel(got, exp) < 1e-12


def test_simulate_frame_equals_numpy_pipeline():
    H, W, C, K, T, dr0 = 20, 24, 3, 6, 7, 2.0
    s_px, kappa = optics.geometry()
    sq, _ = correlation.sqrt_psd_tables(H, W, s_px, 36)
    L = optics.noll_cholesky(optics.noll_covariance(36, dr0))
    packed = synth.mlp_weights(K, seed=1).astype(np.float64)
    basis = synth.basis(K, T, seed=1).astype(np.float64)
    img = synth.image(H, W, C, seed=1).astype(np.float64)
    got = c_oracle.simulate_frame(img, 2210, 6, sq, L, packed, basis, kappa, sigma=0.01, clamp01=True)
    ref = pipeline.simulate(img[None], True, 2210, 6, 1, sq, L, basis, synth.unpack_mlp(packed, K), kappa,
                            sigma=0.01, clamp01=True)[0]
    assert rel(got, ref) < 1e-12
