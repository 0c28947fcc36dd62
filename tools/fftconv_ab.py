#!/usr/bin/env python
"""A/B of the two blur formulations north_star names for Eq.9:

  (a) implicit GEMM over the PSF taps on tcgen05 (libp2s k_blur, steps 4+5), and
  (b) batched FFT convolution: per frame and channel one forward transform of the
      mirror-padded warped image, K products with the basis spectra, K inverse
      transforms, then sum_k w_k(x) conv_k(x).

(b) is run with cuFFT (torch.fft, the vendor FFT) and cuBLAS-free elementwise torch ops
on the same workload (512x512 RGB, K = 100, T = 33), so its number is what the FFT route
costs with a production FFT before any fusion; the byte model in DESIGN.md bounds what a
fused version could save.  (a) is timed through p2s_blur_weights (steps 4+5 with given
per-pixel weights, the same blur kernel the simulator runs).  Both with CUDA events after
warm-up.  Prints one JSON line.

    python tools/fftconv_ab.py [--frames 8] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    H = W = 512
    C, K, T, F = 3, 100, 33, args.frames
    c = T // 2
    dev = torch.device("cuda")
    basis = torch.from_numpy(synth.basis(K, T, seed=0)).to(dev)
    Iw = torch.from_numpy(np.stack([synth.image(H, W, C, seed=s) for s in range(F)])).to(dev)
    w = torch.randn(F, K, H, W, device=dev) * 0.1

    # (b) FFT convolution with cuFFT: mirror pad by c (whole-sample reflect = Q14), grid
    # S = 576 (5-smooth >= 512 + 32), true convolution via the product of spectra
    S = 576
    hp = torch.zeros(K, S, S, device=dev)
    hp[:, :T, :T] = basis
    Hs = torch.fft.rfft2(hp)  # [K][S][S/2+1], off the clock (plan time)

    def fftconv():
        xp = torch.nn.functional.pad(Iw, (c, c, c, c), mode="reflect")  # [F][C][H+2c][W+2c]
        xs = torch.fft.rfft2(xp, s=(S, S))                              # [F][C][S][S/2+1]
        out = torch.zeros(F, C, H, W, device=dev)
        for k0 in range(0, K, 10):  # 10 bases per batch (memory)
            y = torch.fft.irfft2(xs[:, :, None] * Hs[None, None, k0:k0 + 10], s=(S, S))  # [F][C][10][S][S]
            conv = y[..., 2 * c:2 * c + H, 2 * c:2 * c + W]                                # valid part
            out += (conv * w[:, None, k0:k0 + 10]).sum(2)
        return out

    ms_fft = timed(fftconv, args.reps)

    # (a) libp2s: the tcgen05 implicit-GEMM blur with the same per-pixel weights
    from paper_2210_06713_b200 import Plan, PlanConfig
    plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=3.0, K=K, taps=T, max_batch=F), synth.basis(K, T, seed=0),
                synth.mlp_weights(K, seed=0))
    out = torch.empty(F, C, H, W, device=dev)
    ms_gemm = timed(lambda: plan.blur_weights(Iw, w, 2210, 0, out, F), args.reps)
    # agreement of the two formulations on these inputs (bf16 operands in (a))
    ref = fftconv()
    rel = float((out - ref).norm() / ref.norm())
    print(json.dumps({"workload": f"512x512 RGB, K={K}, T={T}, {F} frames", "fft_conv_cufft_ms_per_frame": ms_fft / F,
                      "implicit_gemm_tcgen05_ms_per_frame": ms_gemm / F, "speedup_gemm_over_fft": ms_fft / ms_gemm,
                      "rel_l2_between_formulations": rel,
                      "note": "(b) = torch.fft (cuFFT) rfft2/irfft2 at 576^2 + elementwise weighting; "
                              "(a) = p2s_blur_weights (k_pack_weights + k_blur)"}))


if __name__ == "__main__":
    main()
