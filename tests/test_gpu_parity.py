"""GPU parity: libp2s (sm_100a) vs the fp64 CPU oracle, element by element.

Every call goes through the C ABI (paper_2210_06713_b200.p2s, ctypes).  Inputs are
seeded and synthetic (synth/).  Tolerances (BASELINE north_star): rel-L2 <= 1e-4 for
fp32 stages (step 1 per mode plane, step 2 per channel) and <= 2e-2 for the bf16
tensor-core stages (steps 3-5, per channel).  Unless a test says otherwise the plan
imports the oracle's sqrt(S) tables so per-frame parity is isolated from the
(separately tested) plan-time quadrature.
"""
import numpy as np
import pytest

import synth
from oracle import correlation, optics, philox, pipeline

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 2210


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


_TABLES = {}


def oracle_tables(P, Q, Z=36, s_px=None):
    s_px = s_px or optics.geometry()[0]
    key = (P, Q, Z, s_px)
    if key not in _TABLES:
        _TABLES[key] = correlation.sqrt_psd_tables(P, Q, s_px, Z)[0]
    return _TABLES[key]


def make_plan(H, W, C, dr0, K, T, Z=36, basis=None, mlp=None, import_tables=True, **kw):
    from paper_2210_06713_b200 import Plan, PlanConfig
    basis = synth.basis(K, T, seed=1) if basis is None else basis
    mlp = synth.mlp_weights(K, n_in=Z - 3, seed=1) if mlp is None else mlp
    cfg = PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, Z=Z, K=K, taps=T, **kw)
    plan = Plan(cfg, basis, mlp)
    sq = oracle_tables(plan.P, plan.Q, Z)
    if import_tables:
        plan.import_sqrtS(sq)
    A0 = optics.noll_covariance(Z, dr0)
    L = optics.noll_cholesky(A0)
    return plan, basis, mlp, sq, L


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


# ------------------------------------------------------------------ Philox
def test_device_philox_bit_exact():
    from paper_2210_06713_b200 import philox_fill
    n = 4096
    out = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    philox_fill(7 | (1 << 16), 123, 4, 0xDEADBEEF, 0x1234, n, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    ref = philox.philox4x32_10(np.arange(n), 7 | (1 << 16), 123, 4, 0xDEADBEEF, 0x1234)
    for w in range(4):
        assert np.array_equal(got[:, w], np.asarray(ref[w], dtype=np.uint32))


# ------------------------------------------------------------------ step 1
@pytest.mark.parametrize("H,W,dr0,frame0,F", [(64, 64, 2.0, 0, 2), (60, 90, 3.0, 5, 2), (96, 160, 1.0, 0, 1)])
def test_sample_zernike_vs_oracle(H, W, dr0, frame0, F):
    plan, _, _, sq, L = make_plan(H, W, 1, dr0, 16, 17)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, frame0, F, z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    ref = pipeline.sample_zernike(SEED, frame0, F, sq, L, H, W)
    assert np.all(got[:, 0] == 0)
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-4, worst


@pytest.mark.parametrize("H,W,dr0,F", [(64, 64, 2.0, 2), (60, 90, 3.0, 1), (512, 96, 1.0, 1)])
def test_sample_zernike_from_host_noise_vs_oracle(H, W, dr0, F):
    """North_star parity on identical host-generated noise: the oracle's spectral noise
    (reading Q8, its own Philox) is handed to p2s_sample_zernike_from_noise; the fields match
    the oracle's IDFT + mixing of the same noise, and the library's own Philox path."""
    plan, _, _, sq, L = make_plan(H, W, 1, dr0, 16, 17)
    etas = list(pipeline.spectral_noise_sequence(SEED, 4, F, plan.P, plan.Q, 0.0, 36))
    eta = torch.from_numpy(np.stack(etas).astype(np.complex64)).cuda()
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike_from_noise(eta, F, z)
    z2 = torch.empty_like(z)
    plan.sample_zernike(SEED, 4, F, z2)
    torch.cuda.synchronize()
    got, own = z.cpu().numpy(), z2.cpu().numpy()
    for f in range(F):
        ref = pipeline.mix(pipeline.fields_from_noise(etas[f], sq, H, W), L)
        assert np.all(got[f, 0] == 0)
        assert max(rel_l2(got[f, j], ref[j]) for j in range(1, 36)) <= 1e-4
        assert max(rel_l2(got[f, j], own[f, j]) for j in range(1, 36)) <= 1e-5


@pytest.mark.parametrize("H,W,F", [(512, 96, 2), (96, 512, 3), (512, 512, 1)])
def test_sample_zernike_register_fft_path_vs_oracle(H, W, F):
    """512-point axes take the register-resident radix-8 kernels (rows: Q = 512, columns:
    P = 512); each combination with the generic shared-memory path on the other axis."""
    plan, _, _, sq, L = make_plan(H, W, 1, 3.0, 16, 17)
    assert (plan.P == 512) or (plan.Q == 512)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 3, F, z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    ref = pipeline.sample_zernike(SEED, 3, F, sq, L, H, W)
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-4, worst


def test_register_fft_matches_generic_fft():
    """The 512-point register kernels and the generic shared-memory Stockham kernels run
    the same radix-8 passes: their fields agree to fp32 rounding."""
    from paper_2210_06713_b200 import FORCE_FFT_GENERIC
    H = W = 512
    plan, _, _, _, _ = make_plan(H, W, 1, 3.0, 16, 17)
    zf = torch.empty((2, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 2, zf)
    plan_g, _, _, _, _ = make_plan(H, W, 1, 3.0, 16, 17, force=FORCE_FFT_GENERIC)
    zg = torch.empty_like(zf)
    plan_g.sample_zernike(SEED, 0, 2, zg)
    torch.cuda.synchronize()
    a, b = zf.cpu().numpy(), zg.cpu().numpy()
    worst = max(rel_l2(a[f, j], b[f, j]) for f in range(2) for j in range(1, 36))
    assert worst <= 1e-6, worst


def test_sample_zernike_own_tables_vs_oracle():
    """Library plan tables (C++ quadrature/FFT) instead of the oracle's: the sampled
    fields still agree to the table tolerance."""
    H = W = 64
    plan, _, _, sq, L = make_plan(H, W, 1, 2.0, 16, 17, import_tables=False)
    z = torch.empty((1, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 1, z)
    torch.cuda.synchronize()
    ref = pipeline.sample_zernike(SEED, 0, 1, sq, L, H, W)
    worst = max(rel_l2(z.cpu().numpy()[0, j], ref[0, j]) for j in range(1, 36))
    assert worst <= 1e-3, worst


@pytest.mark.parametrize("force", [0, 0x008, 0x004])  # default, row-pair (k_rows_ar_pair), row kernel (k_rows_ar)
def test_sample_zernike_ar_sequence_and_replay(force):
    H = W = 64
    alpha = 0.95
    plan, _, _, sq, L = make_plan(H, W, 1, 3.0, 16, 17, ar_alpha=alpha, force=force)
    ref = pipeline.sample_zernike(SEED, 0, 6, sq, L, H, W, alpha=alpha)
    z = torch.empty((6, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 4, z[:4])      # fresh sequence
    plan.sample_zernike(SEED, 4, 2, z[4:])      # continuation from the stored state
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(6) for j in range(1, 36))
    assert worst <= 1e-4, worst
    z2 = torch.empty((2, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 2, 2, z2)         # replay frames 0..1 on the device
    torch.cuda.synchronize()
    assert torch.equal(z2, z[2:4])              # bit-identical to the sequential run


@pytest.mark.parametrize("force", [0, 0x400])  # 0x400: the persistent kernel (k_cols_p)
def test_persistent_column_kernel_vs_oracle(force):
    """P = 1000 (radices 10 x 10 x 10) takes the in-place two-CTAs-per-SM column kernel
    (k_cols_ip, 4 columns per block) or, forced, the persistent one (k_cols_p, 8 columns
    per block); fields against the oracle."""
    H, W, F = 1000, 42, 1
    plan, _, _, sq, L = make_plan(H, W, 1, 3.0, 16, 17, force=force)
    assert plan.P == 1000
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 2, F, z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    ref = pipeline.sample_zernike(SEED, 2, F, sq, L, H, W)
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-4, worst


def test_inplace_row_kernel_vs_oracle():
    """Q = 2400 (radices 16 x 15 x 10, two interleaved rows, <= 512 butterflies per pass;
    the ping-pong kernel would need 165 KB) takes the in-place row kernel (k_rows_pair_ip,
    sqrt(S) read from global); fields against the oracle."""
    H, W, F = 20, 2400, 2
    plan, _, _, sq, L = make_plan(H, W, 1, 2.0, 16, 17)
    assert plan.Q == 2400
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 5, F, z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    ref = pipeline.sample_zernike(SEED, 5, F, sq, L, H, W)
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-4, worst


@pytest.mark.parametrize("H,W,F", [(1080, 1920, 2), (2160, 3840, 1)])
def test_inplace_row_kernel_matches_pingpong_kernel(H, W, F):
    """k_rows_pair_ip against k_rows_pair (P2S_FORCE_ROWS_PINGPONG) at the cfg4/cfg5
    geometries: same draws and butterflies, fields equal to fp32 rounding."""
    from paper_2210_06713_b200 import FORCE_ROWS_PINGPONG, Plan, PlanConfig
    outs = []
    for force in (0, FORCE_ROWS_PINGPONG):
        plan = Plan(PlanConfig(H=H, W=W, C=1, d_over_r0=3.0, Z=36, K=16, taps=17, force=force),
                    synth.basis(16, 17, seed=1), synth.mlp_weights(16, n_in=33, seed=1))
        z = torch.empty((F, 36, H, W), device="cuda")
        plan.sample_zernike(SEED, 3, F, z)
        torch.cuda.synchronize()
        outs.append(z.cpu().numpy())
    a, b = outs
    worst = max(rel_l2(a[f, j], b[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-6, worst


@pytest.mark.parametrize("H,W,F", [(1080, 1920, 2), (2160, 3840, 1)])
def test_persistent_column_kernel_matches_per_block_kernel(H, W, F):
    """The three long-column kernels at the cfg4/cfg5 geometries: k_cols_ip (default: in
    place, two CTAs per SM), k_cols (P2S_FORCE_COLS_PER_BLOCK: ping-pong) and k_cols_p
    (P2S_FORCE_COLS_PERSISTENT: persistent, cp.async prefetch): the same butterflies, so the
    fields agree to fp32 rounding; both the fp32 field output and the fused bf16 path."""
    from paper_2210_06713_b200 import FORCE_COLS_PER_BLOCK, FORCE_COLS_PERSISTENT, Plan, PlanConfig
    plans = [Plan(PlanConfig(H=H, W=W, C=1, d_over_r0=3.0, Z=36, K=16, taps=17, force=force),
                  synth.basis(16, 17, seed=1), synth.mlp_weights(16, n_in=33, seed=1))
             for force in (0, FORCE_COLS_PER_BLOCK, FORCE_COLS_PERSISTENT)]
    outs = []
    for plan in plans:
        z = torch.empty((F, 36, H, W), device="cuda")
        plan.sample_zernike(SEED, 1, F, z)
        torch.cuda.synchronize()
        outs.append(z.cpu().numpy())
    for b in outs[1:]:
        worst = max(rel_l2(outs[0][f, j], b[f, j]) for f in range(F) for j in range(1, 36))
        assert worst <= 1e-6, worst
    img = torch.from_numpy(synth.image(H, W, 1, seed=4)).cuda()
    sims = []
    for plan in plans:
        out = torch.empty((F, 1, H, W), device="cuda")
        plan.simulate_frames(img, 0, SEED, 1, F, out)
        torch.cuda.synchronize()
        sims.append(out.cpu().numpy())
    for b in sims[1:]:
        assert rel_l2(sims[0], b) <= 1e-4


@pytest.mark.parametrize("H,W", [(45, 75), (64, 96), (256, 256), (1080, 1920)])
def test_ar_row_pair_kernel_matches_row_kernel(H, W):
    """The AR(1) row-pair kernel (k_rows_ar_pair: mirror state = conjugate, one draw per bin
    pair, P2S_FORCE_AR_PAIR_KERNEL) against the one-CTA-per-row kernel (P2S_FORCE_AR_ROW_KERNEL):
    the same draws and state, so the fields agree to the FFT's fp32 rounding, for a fresh start,
    a stored-state continuation and a replayed start; odd P and Q included."""
    from paper_2210_06713_b200 import FORCE_AR_PAIR_KERNEL, FORCE_AR_ROW_KERNEL, Plan, PlanConfig
    F = 2 if H > 512 else 3
    outs = []
    # default dispatch (128-thread pair CTAs for Q <= 512), forced pair, row kernel
    for force in (0, FORCE_AR_PAIR_KERNEL, FORCE_AR_ROW_KERNEL):
        plan = Plan(PlanConfig(H=H, W=W, C=1, d_over_r0=3.0, Z=36, K=16, taps=17, ar_alpha=0.95, force=force),
                    synth.basis(16, 17, seed=1), synth.mlp_weights(16, n_in=33, seed=1))
        z = torch.empty((2 * F + 1, 36, H, W), device="cuda")
        plan.sample_zernike(SEED, 0, F, z[:F])
        plan.sample_zernike(SEED, F, F, z[F:2 * F])
        plan.sample_zernike(SEED, 2 * F + 2, 1, z[2 * F:])   # replays frames 0..2F+1
        torch.cuda.synchronize()
        outs.append(z.cpu().numpy())
    for a in outs[:2]:
        b = outs[2]
        worst = max(rel_l2(a[f, j], b[f, j]) for f in range(2 * F + 1) for j in range(1, 36))
        assert worst <= 1e-6, worst


# ------------------------------------------------------------------ step 2
@pytest.mark.parametrize("H,W,C", [(64, 64, 1), (60, 90, 3)])
def test_warp_vs_oracle(H, W, C):
    plan, _, _, sq, L = make_plan(H, W, C, 5.0, 16, 17)
    a = pipeline.sample_zernike(SEED, 0, 2, sq, L, H, W)
    img = synth.image(H, W, C, seed=3)
    kappa = optics.geometry()[1]
    out = torch.empty((2, C, H, W), device="cuda")
    plan.warp(cuda(img), 0, cuda(a), out, 2)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for f in range(2):
        ref = pipeline.warp(img, a[f, 1].astype(np.float32).astype(np.float64),
                            a[f, 2].astype(np.float32).astype(np.float64), kappa)
        for c in range(C):
            assert rel_l2(got[f, c], ref[c]) <= 1e-5


# ------------------------------------------------------------------ steps 3-5 (p2s_blur)
def _onehot_mlp(K, k0, Z=36, hidden=(100, 100)):
    sizes = synth.mlp_sizes(Z - 3, hidden, K)
    parts = []
    for li, (o, i) in enumerate(sizes):
        parts.append(np.zeros(o * i))
        b = np.zeros(o)
        if li == len(sizes) - 1:
            b[k0] = 1.0
        parts.append(b)
    return np.concatenate(parts).astype(np.float32)


def test_blur_delta_basis_identity():
    """Delta basis, w = e_0 => out = Iw (BASELINE north_star pin), up to bf16 rounding of Iw."""
    H, W, C, T = 64, 64, 2, 3
    basis = np.zeros((1, T, T), dtype=np.float32)
    basis[0, 1, 1] = 1.0
    plan, *_ = make_plan(H, W, C, 2.0, 1, T, basis=basis, mlp=_onehot_mlp(1, 0))
    Iw = synth.image(H, W, C, seed=4)[None]
    zern = np.zeros((1, 36, H, W), dtype=np.float32)
    out = torch.empty((1, C, H, W), device="cuda")
    plan.blur(cuda(Iw), cuda(zern), SEED, 0, out, 1)
    torch.cuda.synchronize()
    assert rel_l2(out.cpu().numpy(), Iw) <= 4e-3


@pytest.mark.parametrize("H,W,K,T,k0", [(64, 64, 16, 17, 0), (64, 64, 16, 17, 9), (96, 160, 100, 33, 57)])
def test_blur_single_basis_vs_oracle(H, W, K, T, k0):
    """w = e_k0 isolates one spatially invariant convolution (Eq.9 term) of the tap GEMM."""
    plan, basis, *_ = make_plan(H, W, 1, 2.0, K, T, mlp=_onehot_mlp(K, k0))
    Iw = synth.image(H, W, 1, seed=5)[None]
    zern = np.zeros((1, 36, H, W), dtype=np.float32)
    out = torch.empty((1, 1, H, W), device="cuda")
    plan.blur(cuda(Iw), cuda(zern), SEED, 0, out, 1)
    torch.cuda.synchronize()
    w = np.zeros((K, H, W))
    w[k0] = 1.0
    ref = pipeline.blur(Iw[0].astype(np.float64), w, basis)
    assert rel_l2(out.cpu().numpy()[0, 0], ref[0]) <= 1e-2


# forced tile-major / octet-pair MLP input layouts; per-thread A1 copies instead of the TMA box
@pytest.mark.parametrize("force", [0, 0x080, 0x1000, 0x2000, 0x3000])
@pytest.mark.parametrize("H,W,C,K,T", [(64, 64, 1, 16, 17), (96, 160, 3, 100, 33), (40, 90, 1, 16, 17)])
def test_blur_api_vs_oracle(H, W, C, K, T, force):
    plan, basis, mlp, sq, L = make_plan(H, W, C, 3.0, K, T, force=force)
    a = pipeline.sample_zernike(SEED, 0, 1, sq, L, H, W).astype(np.float32)
    Iw = synth.image(H, W, C, seed=6)[None]
    out = torch.empty((1, C, H, W), device="cuda")
    plan.blur(cuda(Iw), cuda(a), SEED, 0, out, 1)
    torch.cuda.synchronize()
    layers = synth.unpack_mlp(mlp, K)
    w = pipeline.mlp(a[0, 3:].astype(np.float64), layers)
    ref = pipeline.blur(Iw[0].astype(np.float64), w, basis)
    got = out.cpu().numpy()[0]
    for c in range(C):
        assert rel_l2(got[c], ref[c]) <= 2e-2


@pytest.mark.parametrize("C,T", [(1, 5), (2, 7), (3, 9), (1, 15), (3, 25), (2, 63)])
def test_blur_tap_sizes_vs_oracle(C, T):
    """Every tap-group shape of the blur's K-step schedule: T < 8 (transposed rows only),
    T % 8 = 1 (one leftover row), T % 8 = 7 (seven leftover rows), up to T = 63."""
    H = W = 64
    K = 16
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T)
    a = pipeline.sample_zernike(SEED, 0, 1, sq, L, H, W).astype(np.float32)
    Iw = synth.image(H, W, C, seed=8)[None]
    out = torch.empty((1, C, H, W), device="cuda")
    plan.blur(cuda(Iw), cuda(a), SEED, 0, out, 1)
    torch.cuda.synchronize()
    w = pipeline.mlp(a[0, 3:].astype(np.float64), synth.unpack_mlp(mlp, K))
    ref = pipeline.blur(Iw[0].astype(np.float64), w, basis)
    got = out.cpu().numpy()[0]
    for c in range(C):
        assert rel_l2(got[c], ref[c]) <= 2e-2, (C, T, c)


@pytest.mark.parametrize("C,K,T", [(4, 128, 33), (1, 1, 3), (2, 100, 17), (4, 100, 33), (3, 128, 33), (4, 64, 17)])
@pytest.mark.parametrize("pair", [True, False])
def test_blur_extreme_shapes_vs_oracle(C, K, T, pair):
    """Edges of the accepted shapes (C = 4, K = 128 = the widest accumulator, K = 1) in both
    blur modes: CTA pairs (cta_group::2, M = 256) and single CTAs (P2S_FORCE_BLUR_SINGLE)."""
    from paper_2210_06713_b200 import FORCE_BLUR_SINGLE
    H, W = 72, 136
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T, force=0 if pair else FORCE_BLUR_SINGLE)
    a = pipeline.sample_zernike(SEED, 0, 1, sq, L, H, W).astype(np.float32)
    Iw = synth.image(H, W, C, seed=9)[None]
    out = torch.empty((1, C, H, W), device="cuda")
    plan.blur(cuda(Iw), cuda(a), SEED, 0, out, 1)
    torch.cuda.synchronize()
    w = pipeline.mlp(a[0, 3:].astype(np.float64), synth.unpack_mlp(mlp, K))
    ref = pipeline.blur(Iw[0].astype(np.float64), w, basis)
    got = out.cpu().numpy()[0]
    for c in range(C):
        assert rel_l2(got[c], ref[c]) <= 2e-2, (C, K, T, pair, c)


# ------------------------------------------------------------------ steps 1-5 fused
@pytest.mark.parametrize("H,W,C,K,T,dr0,F", [(64, 64, 1, 16, 17, 2.0, 1), (96, 160, 3, 100, 33, 3.0, 2)])
def test_simulate_vs_oracle(H, W, C, K, T, dr0, F):
    plan, basis, mlp, sq, L = make_plan(H, W, C, dr0, K, T)
    img = synth.image(H, W, C, seed=7)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 0, F, out)
    torch.cuda.synchronize()
    ref = pipeline.simulate(img[None], True, SEED, 0, F, sq, L, basis, synth.unpack_mlp(mlp, K),
                            optics.geometry()[1])
    got = out.cpu().numpy()
    for f in range(F):
        for c in range(C):
            assert rel_l2(got[f, c], ref[f, c]) <= 2e-2, (f, c, rel_l2(got[f, c], ref[f, c]))


@pytest.mark.parametrize("H,W,C,K,T,Z,hidden,max_batch,F", [
    (37, 41, 4, 128, 33, 66, (128, 128), 0, 1),   # maxima; odd, non-5-smooth image sizes
    (40, 48, 1, 1, 3, 4, (8, 8), 0, 2),           # minima
    (64, 64, 2, 16, 17, 36, (100, 100), 3, 7),    # more frames than the workspace holds
])
def test_simulate_shape_limits_vs_oracle(H, W, C, K, T, Z, hidden, max_batch, F):
    mlp = synth.mlp_weights(K, hidden=hidden, n_in=Z - 3, seed=3)
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.5, K, T, Z=Z, mlp=mlp, mlp_hidden=hidden, max_batch=max_batch)
    img = synth.image(H, W, C, seed=12)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 2, F, out)
    torch.cuda.synchronize()
    ref = pipeline.simulate(img[None], True, SEED, 2, F, sq, L, basis,
                            synth.unpack_mlp(mlp, K, hidden=hidden, n_in=Z - 3), optics.geometry()[1])
    got = out.cpu().numpy()
    for f in range(F):
        for c in range(C):
            assert rel_l2(got[f, c], ref[f, c]) <= 2e-2, (f, c, rel_l2(got[f, c], ref[f, c]))


def test_oversized_mlp_is_unsupported():
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    with pytest.raises(P2SError) as e:
        Plan(PlanConfig(H=64, W=64, C=1, d_over_r0=1.0, Z=66, K=128, taps=17, mlp_hidden=(256, 256)),
             synth.basis(128, 17), synth.mlp_weights(128, hidden=(256, 256), n_in=63))
    assert e.value.status == 5  # P2S_ERR_UNSUPPORTED


@pytest.mark.parametrize("force", [0, 0x080, 0x1000, 0x2000])  # MLP input layouts / A1 load paths
def test_simulate_ar_sequence_vs_oracle(force):
    """Steps 1-5 on an AR(1) sequence (reading Q18): a fresh start and the stored-state
    continuation both follow the oracle's replayed sequence."""
    H, W, C, K, T, alpha = 64, 96, 2, 16, 17, 0.9
    plan, basis, mlp, sq, L = make_plan(H, W, C, 3.0, K, T, ar_alpha=alpha, force=force)
    img = synth.image(H, W, C, seed=13)
    out = torch.empty((5, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 0, 3, out[:3])
    plan.simulate_frames(cuda(img), 0, SEED, 3, 2, out[3:])  # continues from the stored state
    torch.cuda.synchronize()
    ref = pipeline.simulate(img[None], True, SEED, 0, 5, sq, L, basis, synth.unpack_mlp(mlp, K),
                            optics.geometry()[1], alpha=alpha)
    got = out.cpu().numpy()
    for f in range(5):
        for c in range(C):
            assert rel_l2(got[f, c], ref[f, c]) <= 2e-2, (f, c)


def test_simulate_psf_sum_normalisation_vs_oracle():
    """Step 5 normalisation (reading Q16): out / sum_k w_k sum_u h_k(u), with a network whose
    weights are positive everywhere (W3 >= 0, b3 > 0 after ReLU features) so the divisor is
    well conditioned."""
    H, W, C, K, T = 64, 64, 3, 16, 17
    layers = synth.unpack_mlp(synth.mlp_weights(K, seed=5), K)
    rng = np.random.default_rng(3)
    (W1, b1), (W2, b2), (W3, b3) = layers
    W3 = 0.1 * np.abs(W3)
    b3 = rng.uniform(0.5, 1.5, K) / K
    mlp = np.concatenate([W1.ravel(), b1, W2.ravel(), b2, W3.ravel(), b3]).astype(np.float32)
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T, mlp=mlp, normalize_psf_sum=True, clamp01=True)
    img = synth.image(H, W, C, seed=14)
    out = torch.empty((1, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 1, 1, out)
    torch.cuda.synchronize()
    ref = pipeline.simulate(img[None], True, SEED, 1, 1, sq, L, basis, synth.unpack_mlp(mlp, K),
                            optics.geometry()[1], normalize=True, clamp01=True)
    for c in range(C):
        assert rel_l2(out.cpu().numpy()[0, c], ref[0, c]) <= 2e-2, c


def test_simulate_step5_vs_oracle():
    H, W, C, K, T = 64, 96, 2, 16, 17
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T, noise_sigma=0.05, clamp01=True)
    img = synth.image(H, W, C, seed=8)
    out = torch.empty((1, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 3, 1, out)
    torch.cuda.synchronize()
    ref = pipeline.simulate(img[None], True, SEED, 3, 1, sq, L, basis, synth.unpack_mlp(mlp, K),
                            optics.geometry()[1], sigma=0.05, clamp01=True)
    assert rel_l2(out.cpu().numpy(), ref) <= 2e-2


def test_simulate_batch_split_bit_identical():
    H, W, C, K, T = 64, 64, 1, 16, 17
    plan, *_ = make_plan(H, W, C, 3.0, K, T)
    img = cuda(synth.image(H, W, C, seed=9))
    a = torch.empty((4, C, H, W), device="cuda")
    b = torch.empty((4, C, H, W), device="cuda")
    plan.simulate_frames(img, 0, SEED, 10, 4, a)
    for i in range(4):
        plan.simulate_frames(img, 0, SEED, 10 + i, 1, b[i:i + 1])
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    c = torch.empty_like(a)
    plan.simulate_frames(img, 0, SEED, 10, 4, c)
    torch.cuda.synchronize()
    assert torch.equal(a, c)


def test_simulate_host_entry_matches_device_entry():
    H, W, C, K, T = 64, 64, 2, 16, 17
    plan, *_ = make_plan(H, W, C, 3.0, K, T)
    img = synth.image(H, W, C, seed=10)
    dev = torch.empty((2, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 0, 2, dev)
    host = np.empty((2, C, H, W), dtype=np.float32)
    plan.simulate_frames_host(img, 0, SEED, 0, 2, host)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), host)


@pytest.mark.parametrize("F,per_frame_img,max_batch", [(29, False, 0), (11, True, 0), (11, True, 4)])
def test_simulate_host_entry_tapered_sub_batches(F, per_frame_img, max_batch):
    """The host entry point splits a batch into tapered sub-batches (wave-aligned blur
    launches, copies overlapped): results are bit-identical to one device launch, with a
    broadcast image and with one image per frame."""
    H, W, C, K, T = 128, 256, 3, 16, 17
    plan, *_ = make_plan(H, W, C, 2.0, K, T, max_batch=max_batch)  # max_batch 4: chunked uploads
    nimg = F if per_frame_img else 1
    img = np.stack([synth.image(H, W, C, seed=20 + i) for i in range(nimg)])
    stride = C * H * W if per_frame_img else 0
    dev = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), stride, SEED, 5, F, dev)
    host = np.empty((F, C, H, W), dtype=np.float32)
    plan.simulate_frames_host(np.ascontiguousarray(img), stride, SEED, 5, F, host)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), host)


def test_non_contiguous_tensor_is_rejected():
    plan, *_ = make_plan(32, 32, 1, 2.0, 16, 17)
    z = torch.empty((1, 36, 32, 64), device="cuda")[..., ::2]  # strided view
    with pytest.raises(ValueError):
        plan.sample_zernike(SEED, 0, 1, z)


def test_invalid_arguments_fail_loudly():
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    with pytest.raises(P2SError):
        Plan(PlanConfig(H=64, W=64, C=1, d_over_r0=1.0, K=16, taps=16), synth.basis(16, 17), synth.mlp_weights(16))
    with pytest.raises(P2SError):
        Plan(PlanConfig(H=8, W=64, C=1, d_over_r0=1.0, K=16, taps=17), synth.basis(16, 17), synth.mlp_weights(16))
    with pytest.raises(P2SError):
        Plan(PlanConfig(H=64, W=64, C=1, d_over_r0=-1.0, K=16, taps=17), synth.basis(16, 17),
             synth.mlp_weights(16))


# ------------------------------------------------------------------ frozen flow (NEXT-3)
@pytest.mark.parametrize("H,W,flow,frame0", [(64, 96, (1.5, -0.75), 3), (96, 512, (-2.25, 0.5), 0),
                                              (512, 96, (0.3, 1.0), 7)])
def test_frozen_flow_sample_zernike_vs_oracle(H, W, flow, frame0):
    """frame t = frame 0 translated by t v (spectral shift factors, reading Q23);
    covers the generic and the register-resident 512-point row kernels."""
    F = 3
    plan, _, _, sq, L = make_plan(H, W, 1, 2.0, 16, 17, flow=flow)
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, frame0, F, z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    ref = pipeline.sample_zernike(SEED, frame0, F, sq, L, H, W, flow=flow)
    worst = max(rel_l2(got[f, j], ref[f, j]) for f in range(F) for j in range(1, 36))
    assert worst <= 1e-4, worst


def test_frozen_flow_integer_velocity_rolls_frame0():
    H, W = 48, 64
    plan, *_ = make_plan(H, W, 1, 3.0, 16, 17, flow=(3.0, -2.0))
    z = torch.empty((4, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 4, z)
    torch.cuda.synchronize()
    a = z.cpu().numpy()
    for t in range(1, 4):
        assert rel_l2(a[t], np.roll(a[0], (-2 * t, 3 * t), axis=(1, 2))) < 1e-5


def test_frozen_flow_simulate_vs_oracle():
    H, W, C, K, T, F = 64, 64, 3, 16, 17, 2
    flow = (0.5, 1.25)
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T, flow=flow)
    img = synth.image(H, W, C, seed=3)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 5, F, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    s_px, kappa = optics.geometry()
    layers = synth.unpack_mlp(mlp, K)
    a = pipeline.sample_zernike(SEED, 5, F, sq, L, H, W, flow=flow)
    for f in range(F):
        Iw = pipeline.warp(img, a[f, 1], a[f, 2], kappa)
        ref = pipeline.blur(Iw, pipeline.mlp(a[f, 3:], layers), basis)
        for c in range(C):
            assert rel_l2(got[f, c], ref[c]) <= 2e-2


def test_frozen_flow_with_ar_is_rejected():
    from paper_2210_06713_b200 import P2SError
    with pytest.raises(P2SError):
        make_plan(32, 32, 1, 2.0, 16, 17, flow=(1.0, 0.0), ar_alpha=0.5)


@pytest.mark.parametrize("force", [0, 0x100])  # 0x100: step 2 fused into the column kernel
def test_simulate_fused_warp_ragged_columns_vs_oracle(force):
    """512-point columns with W not a multiple of the 16-column block: the separate TMA
    warp and the fused step-2 path (mode-pair-0 column CTAs warp the image), the ragged last
    block, checked against the oracle on sampled pixels (full-frame Eq.9 is too slow)."""
    H, W, C, K, T, F = 512, 200, 3, 16, 17, 1
    plan, basis, mlp, sq, L = make_plan(H, W, C, 2.0, K, T, force=force)
    assert plan.P == 512
    img = synth.image(H, W, C, seed=4)
    out = torch.empty((F, C, H, W), device="cuda")
    plan.simulate_frames(cuda(img), 0, SEED, 2, F, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()[0]
    s_px, kappa = optics.geometry()
    layers = synth.unpack_mlp(mlp, K)
    a = pipeline.sample_zernike(SEED, 2, 1, sq, L, H, W)[0]
    Iw = pipeline.warp(img, a[1], a[2], kappa)
    rng = np.random.default_rng(3)
    ys = np.concatenate([rng.integers(0, H, 400), [0, H - 1, 511, 100]])
    xs = np.concatenate([rng.integers(0, W, 400), [W - 1, 0, 199, 192]])
    w_at = pipeline.mlp(a[3:, ys, xs][:, :, None], layers)[:, :, 0].T
    ref = pipeline.blur_at(Iw, w_at, basis, ys, xs)
    for c in range(C):
        assert rel_l2(got[c, ys, xs], ref[c]) <= 2e-2


# ------------------------------------------------------------------ ABI misuse / edge paths
def test_from_noise_non_hermitian_spectrum_is_the_re_im_split():
    """p2s_sample_zernike_from_noise does not require Hermitian noise: for arbitrary complex
    spectra it returns Re / Im of the same inverse DFT, mixed (documented in p2s.h) -- the
    oracle's fields_from_noise computes exactly that for any input."""
    H, W, F = 48, 40, 1
    plan, _, _, sq, L = make_plan(H, W, 1, 2.0, 16, 17)
    rng = np.random.default_rng(11)
    eta = (rng.standard_normal((35, plan.P, plan.Q)) + 1j * rng.standard_normal((35, plan.P, plan.Q))) * 40.0
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike_from_noise(torch.from_numpy(eta[None].astype(np.complex64)).cuda(), F, z)
    torch.cuda.synchronize()
    ref = pipeline.mix(pipeline.fields_from_noise(eta, sq, H, W), L)
    got = z.cpu().numpy()[0]
    assert max(rel_l2(got[j], ref[j]) for j in range(1, 36)) <= 1e-4


def test_legacy_default_stream_and_side_stream():
    """stream = NULL (the legacy default stream) and a caller-created stream give the same bits."""
    H = W = 64
    plan, *_ = make_plan(H, W, 1, 2.0, 16, 17)
    img = cuda(synth.image(H, W, 1, seed=3))
    a = torch.empty((2, 1, H, W), device="cuda")
    b = torch.empty_like(a)
    plan.simulate_frames(img, 0, SEED, 5, 2, a, stream=0)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.simulate_frames(img, 0, SEED, 5, 2, b, stream=s)
    s.synchronize()
    assert torch.equal(a, b)


def test_calls_on_a_destroyed_or_slab_plan_fail_loudly():
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    H = W = 64
    p = Plan(PlanConfig(H=H, W=W, C=1, d_over_r0=2.0, K=16, taps=17, slab_count=2, slab_rank=0),
             synth.basis(16, 17), synth.mlp_weights(16))
    z = torch.empty((1, 36, H, W), device="cuda")
    with pytest.raises(P2SError) as e:
        p.sample_zernike(SEED, 0, 1, z)  # a slab plan runs only through p2s_slab_*
    assert e.value.status == 1
    q, *_ = make_plan(H, W, 1, 2.0, 16, 17)
    q.close()
    with pytest.raises(P2SError) as e:
        q.sample_zernike(SEED, 0, 1, z)  # NULL plan after destroy
    assert e.value.status == 1


@pytest.mark.parametrize("H,W", [(64, 160), (48, 200)])
@pytest.mark.parametrize("layout", [0x040, 0x1000])
def test_mlp_a1_tma_box_matches_thread_copies(H, W, layout):
    """k_mlp's A1 operand by one TMA box per tile (the default for planes and octet-pair X)
    equals the per-thread copies bit for bit, ragged last tile and partial rows included."""
    outs = []
    for extra in (0, 0x2000):
        plan, basis, mlp, sq, L = make_plan(H, W, 3, 3.0, 16, 17, force=layout | extra)
        img = synth.image(H, W, 3, seed=21)
        out = torch.empty((2, 3, H, W), device="cuda")
        plan.simulate_frames(cuda(img), 0, SEED, 0, 2, out)
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])
