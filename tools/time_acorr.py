"""Times p2s_field_autocorr (development helper)."""
import sys
import torch
import synth
from paper_2210_06713_b200 import Plan, PlanConfig

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
F, L = 64, 24
plan = Plan(PlanConfig(H=H, W=W, C=1, d_over_r0=3.0, K=16, taps=17, max_batch=F), synth.basis(16, 17, seed=1),
            synth.mlp_weights(16, seed=1))
z = torch.empty((F, 36, H, W), device="cuda")
out = torch.empty((36, 2, L), dtype=torch.float64, device="cuda")
plan.sample_zernike(2210, 0, F, z)
for _ in range(3):
    plan.field_autocorr(z, F, L, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    plan.field_autocorr(z, F, L, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{H}x{W} F={F} L={L}: {ms:.3f} ms/call, {36 * H * W * 4 * F / ms / 1e6:.1f} GB/s")
