#!/usr/bin/env python
"""k_blur / k_mlp phase cycle counters (development tool): run with libp2s built with
EXTRA=-DP2S_BLUR_PROBE and/or -DP2S_MLP_PROBE; each blur / MLP launch prints per-CTA
(blur) or per-tile (MLP) phase averages to stderr.

    make -C paper_2210_06713_b200/csrc clean && make -C paper_2210_06713_b200/csrc EXTRA=-DP2S_BLUR_PROBE
    python tools/blur_probe.py [--workload cfg3_512] [--reps 3] [--force 0x2000]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2210_06713_b200 import Plan, PlanConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3_512")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--force", type=lambda s: int(s, 0), default=0)
    args = ap.parse_args()
    w = bench.WORKLOADS[args.workload]
    H, W, C, K, T, F = w["H"], w["W"], w["C"], w["K"], w["T"], w["F"]
    plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=w["d_over_r0"], K=K, taps=T, max_batch=F, force=args.force,
                           **bench.STEP5), synth.basis(K, T, seed=0), synth.mlp_weights(K, seed=0))
    img = torch.from_numpy(synth.image(H, W, C, seed=0)).cuda()
    out = torch.empty((F, C, H, W), device="cuda")
    for r in range(args.reps):
        plan.simulate_frames(img, 0, 2210, r * F, F, out)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
