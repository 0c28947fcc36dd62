"""GPU exact-PSF path (NEXT-1 partial): p2s_exact_psf / p2s_render_exact vs the oracle
(oracle/exact_psf.py, Eq.1-2 with reading Q24).  fp32 phase/FFT against fp64: the PSFs
agree to ~1e-5 relative; tolerance 1e-4 (the fp32-stage bar)."""
import numpy as np
import pytest

import synth
from oracle import exact_psf, optics, correlation, pipeline

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SEED = 2210


def _plan(H, W, C, T, dr0=3.0):
    from paper_2210_06713_b200 import Plan, PlanConfig
    plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, K=16, taps=T), synth.basis(16, T, seed=1),
                synth.mlp_weights(16, seed=1))
    sq, _ = correlation.sqrt_psd_tables(plan.P, plan.Q, optics.geometry()[0], 36)
    plan.import_sqrtS(sq)
    return plan


def rel_l2(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b)


@pytest.mark.parametrize("T,include_tilt", [(33, True), (17, False)])
def test_exact_psf_vs_oracle(T, include_tilt):
    H, W = 40, 48
    plan = _plan(H, W, 1, T)
    z = torch.empty((1, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 4, 1, z)
    rng = np.random.default_rng(0)
    pix = rng.integers(0, H * W, 24).astype(np.int32)
    out = torch.empty((pix.size, T, T), device="cuda")
    plan.exact_psf(z[0], torch.from_numpy(pix).cuda(), pix.size, include_tilt, out)
    torch.cuda.synchronize()
    a = z[0].cpu().numpy().reshape(36, -1)
    got = out.cpu().numpy()
    for i, p in enumerate(pix):
        ref = exact_psf.exact_psf(a[:, p].astype(np.float64), T, include_tilt)
        assert rel_l2(got[i], ref) < 1e-4
        assert abs(got[i].sum() - 1) < 1e-5


def test_render_exact_vs_oracle():
    H, W, C, T = 20, 22, 3, 17
    plan = _plan(H, W, C, T)
    z = torch.empty((1, 36, H, W), device="cuda")
    plan.sample_zernike(SEED, 0, 1, z)
    img = synth.image(H, W, C, seed=2)
    out = torch.empty((C, H, W), device="cuda")
    plan.render_exact(torch.from_numpy(img).cuda(), z[0], True, out)
    torch.cuda.synchronize()
    ref = exact_psf.render_exact(img.astype(np.float64), z[0].cpu().numpy().astype(np.float64), T)
    for c in range(C):
        assert rel_l2(out.cpu().numpy()[c], ref[c]) < 1e-4


def test_exact_tilt_reproduces_the_warp():
    """Reading Q12 vs Q24: with only tilt, the exact render equals the bilinear warp of the
    diffraction-blurred image to first order: compare centroid-level agreement via a delta."""
    H = W = 33
    T = 21
    plan = _plan(H, W, 1, T)
    a = np.zeros((36, H, W), np.float32)
    a[1] = 0.3  # uniform x tilt
    pix = np.array([16 * W + 16], np.int32)
    out = torch.empty((1, T, T), device="cuda")
    plan.exact_psf(torch.from_numpy(a).cuda(), torch.from_numpy(pix).cuda(), 1, True, out)
    torch.cuda.synchronize()
    h = out.cpu().numpy()[0]
    u = np.arange(T) - T // 2
    cx = (h.sum(0) * u).sum()
    assert abs(cx + optics.geometry()[1] * 0.3) < 0.02
