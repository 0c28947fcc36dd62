"""Debug helper: one sample_zernike call at a given size (run under CUDA_LAUNCH_BLOCKING=1)."""
import sys
import numpy as np
import torch
import synth
from paper_2210_06713_b200 import Plan, PlanConfig

H, W, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "zern"
plan = Plan(PlanConfig(H=H, W=W, C=3, d_over_r0=3.0, K=16, taps=17, max_batch=F), synth.basis(16, 17, seed=1),
            synth.mlp_weights(16, seed=1))
if mode == "zern":
    z = torch.empty((F, 36, H, W), device="cuda")
    plan.sample_zernike(2210, 0, F, z)
    torch.cuda.synchronize()
    print("ok", H, W, float(z.abs().max()))
else:
    out = torch.empty((F, 3, H, W), device="cuda")
    img = torch.rand((3, H, W), device="cuda")
    plan.simulate_frames(img, 0, 2210, 0, F, out)
    torch.cuda.synchronize()
    print("ok sim", H, W, float(out.abs().max()))
