"""GPU parity against the fp64 oracle at BASELINE.json's own geometries and edge cases.

* cfg5 (2160 x 3840 RGB, D/r0 = 5, K = 100, T = 33): the 4K kernels (rows 3840 = 16·16·15
  in place, columns 2160 = 16·15·9 in place, octet-pair MLP inputs) against
  `pipeline.sample_zernike` on all 35 mode planes of a frame, and steps 1-5 on sampled
  pixels (corners and edges included) against Eq.9 evaluated pixel by pixel.
* cfg4 / cfg5 as AR(0.95) sequences (reading Q18): fresh start, stored-state
  continuation and a replayed start against the oracle's AR recursion; the
  one-CTA-per-row AR kernel forced once.
* D/r0 = 0: A_0 = 0, so a = 0, no warp, and the frame is one spatially
  invariant blur with the kernel sum_k w_k(0) h_k -- against scipy's mirror convolution.
* Row length 4096 (16·16·16 in place; the AR pass falls back to the row kernel) and a row
  length no row kernel fits (4050: P2S_ERR_UNSUPPORTED at plan creation).
* The MLP input layouts where each is used: tile-major at 512^2 (k_cols512 with step 2 fused)
  against the oracle, planes vs tiles at 1080p (k_cols_p) and 4K, bit for bit.

Tolerances as everywhere (north_star): rel-L2 <= 1e-4 per mode plane (fp32 step 1),
<= 2e-2 per channel for the bf16 tensor-core steps 3-5.  The oracle's sqrt(S) tables are
built from the golden radial tables (tests/oracle_fast.py) and imported into the plans.
"""
import numpy as np
import pytest

import oracle_fast
import synth
from oracle import correlation, optics, pipeline

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SEED = 2210

_SQ = {}


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def oracle_sqrtS(P, Q):
    if (P, Q) not in _SQ:
        _SQ.clear()  # 4K tables are 2.3 GB in fp64: keep one geometry
        _SQ[(P, Q)] = correlation.sqrt_psd_tables(P, Q, optics.geometry()[0], 36,
                                                  tables=oracle_fast.radial_tables_golden())[0]
    return _SQ[(P, Q)]


def plan_for(H, W, C, dr0, K=100, T=33, **kw):
    from paper_2210_06713_b200 import Plan, PlanConfig
    basis = synth.basis(K, T, seed=0)
    mlp = synth.mlp_weights(K, seed=0)
    plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, K=K, taps=T, **kw), basis, mlp)
    plan.import_sqrtS(oracle_sqrtS(plan.P, plan.Q))
    L = optics.noll_cholesky(optics.noll_covariance(36, dr0))
    return plan, basis, mlp, L


def fields_of(eta, sq, L, H, W):
    return pipeline.mix(pipeline.fields_from_noise(eta, sq, H, W), L)


def assert_planes(got, ref, tol=1e-4):
    """got: device/host [36][H][W] float32, ref [36][H][W] fp64; every mode plane j = 2..36."""
    g = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert np.all(g[0] == 0)
    worst = max((rel_l2(g[j], ref[j]), j) for j in range(1, 36))
    assert worst[0] <= tol, worst


def sample_pixels(H, W, n, seed):
    rng = np.random.default_rng(seed)
    ys = np.concatenate([rng.integers(0, H, n), [0, 0, H - 1, H - 1, H // 2, 1, H - 2, 16, H - 17]])
    xs = np.concatenate([rng.integers(0, W, n), [0, W - 1, 0, W - 1, W // 2, W - 2, 1, W - 17, 16]])
    return ys, xs


def check_sampled_output(got, img, a, layers, basis, frame, ys, xs, st5):
    """got [C][H][W] (device frame) vs Eq.9 + step 5 at (ys, xs) on the oracle fields a."""
    C, H, W = img.shape
    Iw = pipeline.warp(img, a[1], a[2], optics.geometry()[1])
    w_at = pipeline.mlp(a[3:, ys, xs][:, :, None], layers)[:, :, 0].T
    ref = pipeline.step5_at(pipeline.blur_at(Iw, w_at, basis, ys, xs), w_at, basis, SEED, frame, ys, xs, W,
                            sigma=st5["noise_sigma"], normalize=st5["normalize_psf_sum"], clamp01=st5["clamp01"])
    g = got.cpu().numpy()[:, ys, xs]
    for c in range(C):
        assert rel_l2(g[c], ref[c]) <= 2e-2, (c, rel_l2(g[c], ref[c]))


# ------------------------------------------------------------------ cfg5: 2160 x 3840 RGB
def test_4k_fields_all_planes_and_sampled_output_vs_oracle():
    import bench
    H, W, C, dr0, frame = 2160, 3840, 3, 5.0, 5
    st5 = bench.STEP5
    plan, basis, mlp, L = plan_for(H, W, C, dr0, max_batch=2, **st5)
    assert (plan.P, plan.Q) == (H, W)
    img = synth.image(H, W, C, seed=0)
    z = torch.empty((1, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, frame, 1, z)
    out = torch.empty((1, C, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, frame, 1, out)
    torch.cuda.synchronize()
    sq = oracle_sqrtS(H, W)
    eta = oracle_fast.white_spectral_noise(SEED, frame, H, W)
    a = fields_of(eta, sq, L, H, W)
    del eta
    assert_planes(z[0], a)
    del z
    ys, xs = sample_pixels(H, W, 600, 4)
    check_sampled_output(out[0], img, a, synth.unpack_mlp(mlp, 100), basis, frame, ys, xs, st5)


def test_4k_mlp_input_layouts_bit_identical():
    """cfg5's default octet-pair MLP inputs against the plane layout (P2S_FORCE_X_PLANES):
    the same values in another order, so the simulated frames are bit-identical."""
    from paper_2210_06713_b200 import FORCE_X_PLANES
    H, W, C = 2160, 3840, 3
    img = torch.from_numpy(synth.image(H, W, C, seed=1)).cuda()
    outs = []
    for force in (0, FORCE_X_PLANES):
        plan, *_ = plan_for(H, W, C, 5.0, max_batch=2, force=force)
        o = torch.empty((2, C, H, W), device="cuda")
        plan.simulate_frames(img, 0, SEED, 3, 2, o)
        torch.cuda.synchronize()
        outs.append(o)
        del plan
    assert torch.equal(outs[0], outs[1])


# ------------------------------------------------------------------ AR(0.95) at cfg4 / cfg5
@pytest.mark.parametrize("H,W,dr0,force", [(1080, 1920, 4.0, 0), (1080, 1920, 4.0, 0x004), (2160, 3840, 5.0, 0)])
def test_ar_long_rows_vs_oracle(H, W, dr0, force):
    """AR(0.95) sequences at the cfg4 / cfg5 geometries (default dispatch: the Hermitian
    row-pair kernel with register state; 0x004 forces k_rows_ar) directly against the oracle:
    frames 0-1 fresh, frame 2 from the stored state, frame 1 again from a replayed start."""
    alpha = 0.95
    plan, basis, mlp, L = plan_for(H, W, 1, dr0, K=16, T=17, ar_alpha=alpha, max_batch=2, force=force)
    z = torch.empty((4, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 2, z[0:2])  # fresh sequence
    plan.sample_zernike(SEED, 2, 1, z[2:3])  # continuation from the stored AR state
    plan.sample_zernike(SEED, 1, 1, z[3:4])  # replays frame 0 on the device, then frame 1
    torch.cuda.synchronize()
    assert torch.equal(z[3], z[1])
    zc = z.cpu().numpy()
    del z
    sq = oracle_sqrtS(plan.P, plan.Q)
    for t, eta in enumerate(oracle_fast.spectral_noise_sequence(SEED, 0, 3, plan.P, plan.Q, alpha)):
        if t == 1 and H > 1080:
            continue  # frame 1 at 4K: covered by the bit-identical replay and frame 2's state
        assert_planes(zc[t], fields_of(eta, sq, L, H, W))


# ------------------------------------------------------------------ MLP input layouts
def test_1080p_mlp_input_layouts_bit_identical():
    """The long-column kernel writing its default octet-pair MLP inputs, tile-major
    (P2S_FORCE_X_TILES) and planes (P2S_FORCE_X_PLANES) at 1080p: bit-identical frames."""
    from paper_2210_06713_b200 import FORCE_X_PLANES, FORCE_X_TILES
    H, W, C = 1080, 1920, 3
    img = torch.from_numpy(synth.image(H, W, C, seed=2)).cuda()
    outs = []
    for force in (0, FORCE_X_TILES, FORCE_X_PLANES):
        plan, *_ = plan_for(H, W, C, 4.0, max_batch=3, force=force)
        o = torch.empty((3, C, H, W), device="cuda")
        plan.simulate_frames(img, 0, SEED, 0, 3, o)
        torch.cuda.synchronize()
        outs.append(o)
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


@pytest.mark.parametrize("force", [0x080, 0x1000])
def test_512_rgb_tile_layout_fused_warp_vs_oracle(force):
    """512^2 RGB with tile-major / octet-pair MLP inputs forced: k_cols512 runs its fused
    warp and writes the tiled layout; sampled output pixels against the oracle."""
    import bench
    H = W = 512
    C, frame = 3, 9
    st5 = bench.STEP5
    plan, basis, mlp, L = plan_for(H, W, C, 3.0, max_batch=4, force=force | 0x100, **st5)
    img = synth.image(H, W, C, seed=0)
    out = torch.empty((1, C, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, frame, 1, out)
    torch.cuda.synchronize()
    eta = pipeline.white_spectral_noise(SEED, frame, H, W)
    a = fields_of(eta, oracle_sqrtS(H, W), L, H, W)
    ys, xs = sample_pixels(H, W, 600, 5)
    check_sampled_output(out[0], img, a, synth.unpack_mlp(mlp, 100), basis, frame, ys, xs, st5)


# ------------------------------------------------------------------ D/r0 = 0
def test_diffraction_limited_is_one_invariant_blur():
    """D/r0 = 0: A_0 = 0 and L = 0, so every Zernike plane is exactly 0, the warp is the
    identity and w(x) = w(0) = MLP(0) everywhere: the frame is I convolved (true convolution,
    whole-sample mirror boundary, Q14) with sum_k w_k(0) h_k -- scipy.ndimage.convolve."""
    from scipy import ndimage
    H = W = 512
    C, K, T = 3, 100, 33
    plan, basis, mlp, L = plan_for(H, W, C, 0.0)
    assert np.all(L == 0)
    A0, Lc, _ = plan.export_tables()
    assert np.all(A0 == 0) and np.all(Lc == 0)
    z = torch.empty((2, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 2, z)
    img = synth.image(H, W, C, seed=7)
    out = torch.empty((2, C, H, W), device="cuda")
    plan.simulate_frames(torch.from_numpy(img).cuda(), 0, SEED, 0, 2, out)
    torch.cuda.synchronize()
    assert torch.count_nonzero(z).item() == 0
    w0 = pipeline.mlp(np.zeros((33, 1)), synth.unpack_mlp(mlp, K))[:, 0]
    h = np.einsum("k,ktu->tu", w0, basis.astype(np.float64))
    got = out.cpu().numpy()
    assert np.array_equal(got[0], got[1])  # no field, no noise: every frame is the same
    for c in range(C):
        ref = ndimage.convolve(img[c].astype(np.float64), h, mode="mirror")
        assert rel_l2(got[0, c], ref) <= 2e-2, c


# ------------------------------------------------------------------ row lengths at the limit
def test_row_length_4096_vs_oracle():
    """Q = 4096: the row plan is 16·16·16 so the in-place row kernel fits (the ping-pong one
    would need 237 KB); AR(1) rows fall back to the one-CTA-per-row kernel."""
    H, W = 24, 4096
    for alpha in (0.0, 0.9):
        plan, basis, mlp, L = plan_for(H, W, 1, 2.0, K=16, T=17, ar_alpha=alpha)
        assert plan.Q == 4096
        z = torch.empty((2, 36, H, W), device="cuda")
        plan.sample_zernike(SEED, 0, 2, z)
        torch.cuda.synchronize()
        sq = oracle_sqrtS(plan.P, plan.Q)
        for f, eta in enumerate(pipeline.spectral_noise_sequence(SEED, 0, 2, plan.P, plan.Q, alpha)):
            assert_planes(z[f], fields_of(eta, sq, L, H, W))


def test_row_length_without_a_fitting_kernel_is_unsupported():
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    with pytest.raises(P2SError) as e:
        Plan(PlanConfig(H=20, W=4050, C=1, d_over_r0=1.0, K=16, taps=17), synth.basis(16, 17), synth.mlp_weights(16))
    assert e.value.status == 5  # P2S_ERR_UNSUPPORTED


@pytest.mark.parametrize("H,W,C,img_frames", [(1080, 1920, 3, 1), (200, 328, 2, 3)])
def test_tma_window_warp_matches_gather_warp(H, W, C, img_frames):
    """Step 2 with the TMA-staged image window (default at long columns) against the plain
    gather kernel (P2S_FORCE_WARP_GATHER): the same arithmetic on the same values, so the
    frames are bit-identical -- broadcast image and per-frame images."""
    from paper_2210_06713_b200 import FORCE_WARP_GATHER
    imgs = np.stack([synth.image(H, W, C, seed=s) for s in range(img_frames)])
    img = torch.from_numpy(imgs if img_frames > 1 else imgs[0]).cuda()
    stride = C * H * W if img_frames > 1 else 0
    F = img_frames if img_frames > 1 else 2
    outs = []
    for force in (0, FORCE_WARP_GATHER):
        plan, *_ = plan_for(H, W, C, 5.0, K=16, T=17, max_batch=F, force=force)
        o = torch.empty((F, C, H, W), device="cuda")
        plan.simulate_frames(img, stride, SEED, 4, F, o)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("W,force", [(2400, 0), (2400, 0x004), (1200, 0)])
def test_ar_generic_long_rows_vs_oracle(W, force):
    """AR(0.9) on long rows outside the compile-time plans: 2400 = 16·15·10 takes the generic
    512-thread row-pair kernel (0x004: the one-CTA-per-row kernel), 1200 (512 < Q <= 1024 is
    not it; 1200 > 1024) the pair kernel with four bins per thread -- fresh start, continuation
    and replayed start against the oracle's recursion."""
    H, alpha = 20, 0.9
    plan, basis, mlp, L = plan_for(H, W, 1, 2.0, K=16, T=17, ar_alpha=alpha, force=force)
    z = torch.empty((4, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 2, z[0:2])
    plan.sample_zernike(SEED, 2, 1, z[2:3])
    plan.sample_zernike(SEED, 1, 1, z[3:4])
    torch.cuda.synchronize()
    assert torch.equal(z[3], z[1])
    zc = z.cpu().numpy()
    sq = oracle_sqrtS(plan.P, plan.Q)
    for t, eta in enumerate(pipeline.spectral_noise_sequence(SEED, 0, 3, plan.P, plan.Q, alpha)):
        assert_planes(zc[t], fields_of(eta, sq, L, H, W))
