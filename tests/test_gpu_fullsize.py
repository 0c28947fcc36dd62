"""GPU checks at BASELINE.json's full sizes, in bench.py's launch configuration.

* 512x512 RGB, K = 100, T = 33 (the bench workload): the step-1 fields are compared with
  the oracle on every pixel (its IDFT is cheap), the final output on sampled pixels
  (oracle Eq.9 evaluated pixel by pixel, `pipeline.blur_at`).
* 1080p: every pixel of all 35 mode planes against the oracle, sampled output pixels
  (tests/test_gpu_geometry_parity.py does the same at 4K).
* 1080p and 4K: properties that hold at any size -- the sampled fields reproduce the
  Noll matrix A_0 (Eq.10 at zero lag), the closed-form tilt variance within a
  4-sigma bound, unit-variance unmixed fields, Gaussian kurtosis; bit-identical
  frames for any batch split (counter-based noise).
"""
import numpy as np
import pytest

import oracle_fast
import synth
from oracle import correlation, optics, pipeline

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SEED = 2210


def rel_l2(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b)


def _plan(H, W, C, dr0, K, T, **kw):
    from paper_2210_06713_b200 import Plan, PlanConfig
    basis = synth.basis(K, T, seed=0)
    mlp = synth.mlp_weights(K, seed=0)
    return Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, K=K, taps=T, **kw), basis, mlp), basis, mlp


def test_512_rgb_bench_config_vs_oracle_sampled():
    """bench.py's workload and step-5 configuration (noise sigma, clamp)."""
    import bench
    H = W = 512
    C, K, T, dr0, F = 3, 100, 33, 3.0, 2
    st5 = bench.STEP5
    plan, basis, mlp = _plan(H, W, C, dr0, K, T, max_batch=64, **st5)
    s_px, kappa = optics.geometry()
    sq, _ = correlation.sqrt_psd_tables(H, W, s_px, 36, tables=oracle_fast.radial_tables_golden())
    plan.import_sqrtS(sq)
    img = synth.image(H, W, C, seed=0)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, 7, F, out)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 7, F, z)
    torch.cuda.synchronize()
    got, zg = out.cpu().numpy(), z.cpu().numpy()
    A0 = optics.noll_covariance(36, dr0)
    L = optics.noll_cholesky(A0)
    layers = synth.unpack_mlp(mlp, K)
    rng = np.random.default_rng(0)
    ys = np.concatenate([rng.integers(0, H, 600), [0, 0, H - 1, H - 1, 255, 17]])
    xs = np.concatenate([rng.integers(0, W, 600), [0, W - 1, 0, W - 1, 128, 500]])
    for f, eta in enumerate(pipeline.spectral_noise_sequence(SEED, 7, F, H, W, 0.0, 36)):
        a = pipeline.mix(pipeline.fields_from_noise(eta, sq, H, W), L)
        worst = max(rel_l2(zg[f, j], a[j]) for j in range(1, 36))
        assert worst <= 1e-4, worst
        Iw = pipeline.warp(img, a[1], a[2], kappa)
        w_at = pipeline.mlp(a[3:, ys, xs][:, :, None], layers)[:, :, 0].T
        ref = pipeline.step5_at(pipeline.blur_at(Iw, w_at, basis, ys, xs), w_at, basis, SEED, 7 + f, ys, xs, W,
                                sigma=st5["noise_sigma"], normalize=st5["normalize_psf_sum"],
                                clamp01=st5["clamp01"])
        for c in range(C):
            assert rel_l2(got[f, c, ys, xs], ref[c]) <= 2e-2


def test_1080p_rgb_vs_oracle_sampled():
    """cfg4's geometry (1080 x 1920 RGB, D/r0 = 4, K = 100, T = 33: generic mixed-radix FFTs,
    separate warp kernel, 15 x-tiles with a ragged last one): step-1 fields on every pixel
    of all 35 modes, the final output on sampled pixels, one frame."""
    import bench
    H, W, C, K, T, dr0, F = 1080, 1920, 3, 100, 33, 4.0, 1
    st5 = bench.STEP5
    plan, basis, mlp = _plan(H, W, C, dr0, K, T, max_batch=8, **st5)
    s_px, kappa = optics.geometry()
    sq, _ = correlation.sqrt_psd_tables(plan.P, plan.Q, s_px, 36, tables=oracle_fast.radial_tables_golden())
    plan.import_sqrtS(sq)
    img = synth.image(H, W, C, seed=3)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, 11, F, out)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 11, F, z)
    torch.cuda.synchronize()
    got, zg = out.cpu().numpy(), z.cpu().numpy()
    L = optics.noll_cholesky(optics.noll_covariance(36, dr0))
    layers = synth.unpack_mlp(mlp, K)
    rng = np.random.default_rng(1)
    ys = np.concatenate([rng.integers(0, H, 400), [0, H - 1, 0, H - 1, 540]])
    xs = np.concatenate([rng.integers(0, W, 400), [0, W - 1, W - 1, 0, 1919]])
    eta = oracle_fast.white_spectral_noise(SEED, 11, plan.P, plan.Q)
    a = pipeline.mix(pipeline.fields_from_noise(eta, sq, H, W), L)
    for j in range(1, 36):
        assert rel_l2(zg[0, j], a[j]) <= 1e-4, j
    Iw = pipeline.warp(img, a[1], a[2], kappa)
    w_at = pipeline.mlp(a[3:, ys, xs][:, :, None], layers)[:, :, 0].T
    ref = pipeline.step5_at(pipeline.blur_at(Iw, w_at, basis, ys, xs), w_at, basis, SEED, 11, ys, xs, W,
                            sigma=st5["noise_sigma"], normalize=st5["normalize_psf_sum"], clamp01=st5["clamp01"])
    for c in range(C):
        assert rel_l2(got[0, c, ys, xs], ref[c]) <= 2e-2


@pytest.mark.parametrize("H,W,dr0,F", [(1080, 1920, 4.0, 8), (2160, 3840, 5.0, 2)])
def test_fullsize_field_statistics(H, W, dr0, F):
    plan, *_ = _plan(H, W, 3, dr0, 100, 33, max_batch=F)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, F, z)
    torch.cuda.synchronize()
    A0, Lc, sq = plan.export_tables()
    Ao = optics.noll_covariance(36, dr0)
    assert np.abs(A0 - Ao).max() < 1e-12
    a = z.double()
    n = a.shape[0] * a.shape[2] * a.shape[3]
    X = a[:, 1:].permute(1, 0, 2, 3).reshape(35, -1)
    Cov = (X @ X.T / n).cpu().numpy()
    ref = Ao[1:, 1:]
    # tilt variance: 4-sigma bound from the exact per-frame variance of the periodic field
    S2 = sq[0].astype(np.float64) ** 2
    sig = ref[0, 0] * np.sqrt(2 * (S2 ** 2).sum()) / (plan.P * plan.Q * np.sqrt(F))
    assert abs(Cov[0, 0] - ref[0, 0]) < 4 * sig + 1e-3 * ref[0, 0]
    # the whole per-pixel Noll matrix (Eq.10 at zero lag), high-order modes decorrelate fast
    hi = np.arange(2, 35)
    assert np.linalg.norm(Cov[np.ix_(hi, hi)] - ref[np.ix_(hi, hi)]) / np.linalg.norm(ref[np.ix_(hi, hi)]) < 0.05
    x4 = X[2].cpu().numpy() / np.sqrt(ref[2, 2])
    k = (x4 ** 4).mean() / (x4 ** 2).mean() ** 2
    assert 2.8 < k < 3.2


def test_bench_config_batch_split_and_rerun_bit_identical():
    H = W = 512
    plan, *_ = _plan(H, W, 3, 3.0, 100, 33, max_batch=8)
    img = torch.from_numpy(synth.image(H, W, 3, seed=1)).cuda()
    a = torch.empty((8, 3, H, W), device="cuda")
    b = torch.empty_like(a)
    plan.simulate_frames(img, 0, SEED, 100, 8, a)
    plan.simulate_frames(img, 0, SEED, 100, 3, b[:3])
    plan.simulate_frames(img, 0, SEED, 103, 5, b[3:])
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_per_frame_images_stride():
    """img_frame_stride != 0: frame i reads image i."""
    H = W = 64
    plan, *_ = _plan(H, W, 1, 2.0, 16, 17)
    imgs = np.stack([synth.image(H, W, 1, seed=s) for s in range(3)])
    d = torch.from_numpy(imgs).cuda()
    out = torch.empty((3, 1, H, W), device="cuda")
    plan.simulate_frames(d, H * W, SEED, 0, 3, out)
    one = torch.empty((1, 1, H, W), device="cuda")
    plan.simulate_frames(d[2], 0, SEED, 2, 1, one)
    torch.cuda.synchronize()
    assert torch.equal(out[2], one[0])


@pytest.mark.parametrize("H,W,F,max_batch", [(512, 512, 3, 0), (1080, 1920, 2, 2), (2160, 3840, 1, 1)])
def test_host_entry_split_tail_bit_identical(H, W, F, max_batch):
    """p2s_simulate_frames_host at BASELINE geometries: a one-frame last sub-batch runs its
    blur as two row-band halves (the top half's device->host copy overlaps the bottom half);
    the host output equals the device entry point's bit for bit."""
    plan, *_ = _plan(H, W, 3, 4.0, 100, 33, max_batch=max_batch)
    img = synth.image(H, W, 3, seed=6)
    dev = torch.empty((F, 3, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, 40, F, dev)
    torch.cuda.synchronize()
    img_h = torch.from_numpy(img).pin_memory().numpy()
    out_h = torch.full((F, 3, H, W), float("nan")).pin_memory().numpy()
    plan.simulate_frames_host(img_h, 0, SEED, 40, F, out_h)
    assert np.array_equal(out_h, dev.cpu().numpy())
