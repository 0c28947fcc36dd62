"""Times the exact-PSF path against the P2S frame (development helper; no oracle)."""
import sys
import torch
import synth
from paper_2210_06713_b200 import Plan, PlanConfig

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 256
C, K, T = 3, 100, 33
plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=3.0, K=K, taps=T, max_batch=8), synth.basis(K, T, seed=0),
            synth.mlp_weights(K, seed=0))
img = torch.from_numpy(synth.image(H, W, C, seed=0)).cuda()
z = torch.empty((1, 36, H, W), device="cuda")
plan.sample_zernike(2210, 0, 1, z)
out = torch.empty((C, H, W), device="cuda")
plan.render_exact(img, z[0], True, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.render_exact(img, z[0], True, out)
e1.record()
torch.cuda.synchronize()
t_exact = e0.elapsed_time(e1)
o8 = torch.empty((8, C, H, W), device="cuda")
plan.simulate_frames(img, 0, 2210, 0, 8, o8)
torch.cuda.synchronize()
e0.record()
plan.simulate_frames(img, 0, 2210, 0, 8, o8)
e1.record()
torch.cuda.synchronize()
t_p2s = e0.elapsed_time(e1) / 8
print(f"{H}x{W} RGB T={T}: exact render {t_exact:.2f} ms/frame ({H * W / t_exact / 1e3:.2f} M PSF/s), "
      f"P2S simulate {t_p2s:.3f} ms/frame, ratio {t_exact / t_p2s:.0f}x")
