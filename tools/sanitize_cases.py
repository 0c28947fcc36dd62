#!/usr/bin/env python
"""Small invocations of every libp2s kernel for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck --target-processes all \
        python tools/sanitize_cases.py

Each case is a plan at a small geometry that selects one kernel variant (the dispatch is
fixed per plan; P2S_FORCE_* bits pin the alternatives): the generic and 512-point
register FFT passes, the persistent / in-place long-axis kernels, the AR(1) row kernels,
the MLP, the blur in CTA-pair and single-CTA mode (with and without the transposed
leftover tap rows), the exact-PSF / render kernels and the statistics kernels.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2210_06713_b200 import (FORCE_AR_PAIR_KERNEL, FORCE_AR_ROW_KERNEL, FORCE_BLUR_SINGLE,  # noqa: E402
                                   FORCE_COLS_PER_BLOCK, FORCE_FFT_GENERIC, FORCE_X_TILES, Plan, PlanConfig)

SEED = 2210


def plan(H, W, C=1, K=16, T=17, **kw):
    return Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=2.0, K=K, taps=T, **kw), synth.basis(K, T, seed=1),
                synth.mlp_weights(K, seed=1))


def simulate(p, F=2, frame0=0):
    H, W, C = p.cfg.H, p.cfg.W, p.cfg.C
    img = torch.from_numpy(synth.image(H, W, C, seed=0)).cuda()
    out = torch.empty((F, C, H, W), device="cuda")
    p.simulate_frames(img, 0, SEED, frame0, F, out)
    z = torch.empty((F, 36, H, W), device="cuda")
    p.sample_zernike(SEED, frame0, F, z)
    torch.cuda.synchronize()
    return z


CASES = {
    "generic_fft_blur_pair": lambda: simulate(plan(64, 96, C=2)),
    "reg512_cols_fused_warp": lambda: simulate(plan(512, 64, C=3, K=100, T=33, force=0x100), F=1),
    "reg512_rows": lambda: simulate(plan(48, 512), F=1),
    "reg512_generic_forced": lambda: simulate(plan(512, 512, force=FORCE_FFT_GENERIC), F=1),
    "x_tiles": lambda: simulate(plan(64, 160, C=3, force=FORCE_X_TILES)),
    "cols_persistent": lambda: simulate(plan(1000, 40), F=1),
    "cols_per_block": lambda: simulate(plan(1000, 40, force=FORCE_COLS_PER_BLOCK), F=1),
    "rows_in_place": lambda: simulate(plan(20, 2400), F=1),
    "ar_pair_short": lambda: simulate(plan(64, 64, ar_alpha=0.9), F=3),
    "ar_pair_forced": lambda: simulate(plan(45, 75, ar_alpha=0.9, force=FORCE_AR_PAIR_KERNEL), F=2),
    "ar_row_kernel": lambda: simulate(plan(40, 64, ar_alpha=0.9, force=FORCE_AR_ROW_KERNEL), F=2),
    "ar_pair_long": lambda: simulate(plan(20, 2400, ar_alpha=0.9), F=1),
    "blur_single": lambda: simulate(plan(72, 136, C=4, K=128, T=33, force=FORCE_BLUR_SINGLE), F=1),
    "blur_padded_taps": lambda: simulate(plan(64, 64, C=1, K=16, T=15), F=1),
    "blur_small_taps": lambda: simulate(plan(40, 48, C=1, K=1, T=3), F=1),
}


def stats_cases():
    p = plan(64, 64, C=1, T=17)
    z = simulate(p, F=2)
    ac = torch.empty((36, 2, 8), dtype=torch.float64, device="cuda")
    p.field_autocorr(z, 2, 8, ac)
    pix = torch.tensor([0, 100, 2000, 4095], dtype=torch.int32, device="cuda")
    ap = torch.empty((3, 32, 63), dtype=torch.float64, device="cuda")
    p.aperture_stats(z, 2, pix, ap)
    psf = torch.empty((4, 17, 17), device="cuda")
    p.exact_psf(z[0], pix, 4, True, psf)
    img = torch.from_numpy(synth.image(64, 64, 1, seed=2)).cuda()
    out = torch.empty((1, 64, 64), device="cuda")
    p.render_exact(img, z[0], True, out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["stats"]
    for n in names:
        if n == "stats":
            stats_cases()
        else:
            CASES[n]()
        print("case ok:", n, flush=True)
    print("all cases ok")
