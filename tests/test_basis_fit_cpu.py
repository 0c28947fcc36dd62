"""PCA PSF basis (Eq.7, NEXT-1 part): the library's host fit (p2s_fit_basis, C++) against
the oracle's plain eigen-decomposition, and the oracle against a known low-rank database."""
import numpy as np
import pytest

from oracle import exact_psf


def test_oracle_pca_recovers_known_low_rank_structure():
    rng = np.random.default_rng(1)
    T, n = 7, 400
    d = T * T
    Q, _ = np.linalg.qr(rng.standard_normal((d, 3)))
    mu = rng.uniform(size=d)
    coeff = rng.standard_normal((n, 3)) * np.array([3.0, 2.0, 1.0])
    X = mu + coeff @ Q.T
    basis, res = exact_psf.pca_basis(X.reshape(n, T, T), 3)
    assert res < 1e-12
    assert np.allclose(basis[0].ravel(), X.mean(0), atol=1e-12)
    P = basis[1:].reshape(3, d)
    assert np.allclose(P @ P.T, np.eye(3), atol=1e-10)
    # same subspace as the generating one
    assert np.allclose(np.linalg.svd(P @ Q, compute_uv=False), 1.0, atol=1e-8)


def test_library_fit_matches_oracle_on_exact_psfs():
    from paper_2210_06713_b200 import fit_basis
    rng = np.random.default_rng(2)
    T, n, M = 9, 300, 6
    psfs = []
    for _ in range(n):
        a = np.zeros(36)
        a[3:15] = 0.3 * rng.standard_normal(12)  # higher-order aberrations, Noll 4..15
        psfs.append(exact_psf.exact_psf(a, T, include_tilt=False))
    psfs = np.asarray(psfs)
    got, res = fit_basis(psfs.astype(np.float32), M)
    ref, res_ref = exact_psf.pca_basis(psfs.astype(np.float32).astype(np.float64), M)
    assert np.allclose(got[0], ref[0], atol=1e-7)
    G, R = got[1:].reshape(M, -1).astype(np.float64), ref[1:].reshape(M, -1)
    assert np.allclose(G @ G.T, np.eye(M), atol=1e-5)
    # component by component (well-separated leading eigenvalues): same direction
    assert np.all(np.abs(np.sum(G * R, axis=1)) > 1 - 1e-4)
    assert abs(res - res_ref) < 1e-6


def test_fit_basis_rejects_bad_arguments():
    from paper_2210_06713_b200 import P2SError, fit_basis
    with pytest.raises(P2SError):
        fit_basis(np.zeros((3, 5, 5), np.float32), 3)  # M >= n


def test_readout_fit_recovers_an_exact_linear_readout():
    """Targets that ARE a linear readout of the hidden features are fitted exactly (lam = 0),
    and the library's Cholesky solve equals the oracle's lstsq on general targets."""
    import synth
    from paper_2210_06713_b200 import fit_readout
    K = 7
    mlp = synth.mlp_weights(K, seed=4)
    layers = synth.unpack_mlp(mlp, K)
    rng = np.random.default_rng(7)
    a = 0.5 * rng.standard_normal((600, 33))
    (W1, b1), (W2, b2), (W3, b3) = layers
    h = np.maximum(np.maximum(a @ W1.T + b1, 0) @ W2.T + b2, 0)
    target = h @ W3.T + b3
    out, res = fit_readout(mlp, a, target, lam=0.0)
    assert res < 1e-4
    l2 = synth.unpack_mlp(out, K)
    assert np.allclose(l2[2][0], W3, atol=1e-3) and np.allclose(l2[2][1], b3, atol=1e-3)
    assert np.array_equal(out[: mlp.size - K * 100 - K], mlp[: mlp.size - K * 100 - K])  # hidden layers kept
    beta = rng.standard_normal((600, K))
    out, res = fit_readout(mlp, a, beta, lam=0.1)
    W3o, b3o, res_o = exact_psf.fit_readout(layers, a.astype(np.float32), beta.astype(np.float32), 0.1)
    l2 = synth.unpack_mlp(out, K)
    assert np.allclose(l2[2][0], W3o, atol=2e-4) and np.allclose(l2[2][1], b3o, atol=2e-4)
    assert abs(res - res_o) < 1e-6


def test_train_mlp_matches_oracle_training():
    """p2s_train_mlp (host fp64) follows the oracle's training loop (oracle/train.py,
    reading Q26) step by step: same sample order, batches, Adam updates -> same weights and
    loss curve up to summation order."""
    import synth
    from oracle import train
    from paper_2210_06713_b200 import train_mlp
    K = 5
    mlp = synth.mlp_weights(K, hidden=(16, 12), seed=6)
    layers = synth.unpack_mlp(mlp, K, hidden=(16, 12))
    rng = np.random.default_rng(9)
    a = (0.5 * rng.standard_normal((300, 33))).astype(np.float32)
    beta = rng.standard_normal((300, K)).astype(np.float32)
    order = np.stack([rng.permutation(300) for _ in range(4)]).astype(np.int32)
    out, curve = train_mlp(mlp, a, beta, order, batch=32, lr=2e-3, hidden=(16, 12))
    ref, ref_curve = train.train(layers, a.astype(np.float64), beta.astype(np.float64), order, 4, 32, 2e-3)
    got = synth.unpack_mlp(out, K, hidden=(16, 12))
    for (Wg, bg), (Wr, br) in zip(got, ref):
        assert np.allclose(Wg, Wr, rtol=0, atol=1e-6) and np.allclose(bg, br, rtol=0, atol=1e-6)
    assert np.allclose(curve, ref_curve, rtol=1e-9)
    assert curve[-1] < curve[0]


def test_train_mlp_rejects_bad_order():
    import synth
    from paper_2210_06713_b200 import P2SError, train_mlp
    mlp = synth.mlp_weights(3, seed=1)
    a = np.zeros((4, 33), np.float32)
    beta = np.zeros((4, 3), np.float32)
    with pytest.raises(P2SError):
        train_mlp(mlp, a, beta, np.array([[0, 1, 2, 4]], np.int32))
