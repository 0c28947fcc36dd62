"""Single-frame slab mode emulated on one GPU: the G ranks' row passes
run in turn, the all-to-all is emulated by device copies of the send blocks (exactly the
split sizes NCCL's all_to_all_single would use), every rank's strip pass follows, and the
assembled frame must be bit-identical to p2s_simulate_frames of the unsharded frame (the
same kernels on the same per-bin / per-pixel arithmetic; the T/2-column halo makes the
mirror boundary exact; the step-5 noise is keyed by frame coordinates)."""
import numpy as np
import pytest

import synth
from paper_2210_06713_b200 import runner

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SEED = 2210


def emulate(H, W, C, K, T, dr0, G, frame, **kw):
    from paper_2210_06713_b200 import Plan, PlanConfig, slab_geometry
    basis = synth.basis(K, T, seed=0)
    mlp = synth.mlp_weights(K, seed=0)
    img = torch.from_numpy(synth.image(H, W, C, seed=5)).cuda()
    ref_plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, K=K, taps=T, max_batch=1, **kw), basis, mlp)
    ref = torch.empty((1, C, H, W), device="cuda")
    ref_plan.simulate_frames(img, 0, SEED, frame, 1, ref)
    torch.cuda.synchronize()
    del ref_plan
    plans = [Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=dr0, K=K, taps=T, slab_count=G, slab_rank=r, **kw), basis, mlp)
             for r in range(G)]
    counts = [p.slab_counts() for p in plans]
    for r in range(G):  # the plan's split sizes are the host geometry's
        s_h, r_h = runner.slab_counts_host(H, W, T, G, r)
        assert list(counts[r][0]) == s_h and list(counts[r][1]) == r_h
    sends = []
    for r, p in enumerate(plans):
        snd = torch.empty(int(counts[r][0].sum()), device="cuda")
        p.slab_rows(SEED, frame, snd)
        sends.append(snd)
    torch.cuda.synchronize()
    out = torch.full((C, H, W), float("nan"), device="cuda")
    for r, p in enumerate(plans):
        # recv of rank r = concat over sources s of block (s -> r) of s's send buffer
        parts = []
        for s in range(G):
            off = int(counts[s][0][:r].sum())
            parts.append(sends[s][off:off + int(counts[s][0][r])])
        recv = torch.cat(parts).contiguous()
        assert recv.numel() == int(counts[r][1].sum())
        g = slab_geometry(H, W, T, G, r)
        strip = torch.empty((C, H, g["x1"] - g["x0"]), device="cuda")
        p.slab_finish(recv, img, SEED, frame, strip)
        torch.cuda.synchronize()
        out[:, :, g["x0"]:g["x1"]] = strip
    return out, ref[0]


@pytest.mark.parametrize("H,W,C,K,T,G", [(96, 160, 3, 16, 17, 3), (512, 512, 3, 100, 33, 4)])
def test_slab_emulation_bit_identical(H, W, C, K, T, G):
    import bench
    out, ref = emulate(H, W, C, K, T, 3.0, G, 7, **bench.STEP5)
    assert torch.isfinite(out).all()
    assert torch.equal(out, ref)


def test_slab_emulation_4k_eight_ranks_bit_identical():
    """The BASELINE cfg5 geometry (2160 x 3840 RGB, K = 100, T = 33) over 8 ranks: strips of
    480 columns (+16 halo), 269-271 spectral rows per rank."""
    import bench
    out, ref = emulate(2160, 3840, 3, 100, 33, 5.0, 8, 3, **bench.STEP5)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("H,W,G,kw", [(2160, 3840, 8, {"ar_alpha": 0.95}), (96, 160, 3, {"ar_alpha": 0.9}),
                                       (256, 320, 4, {"flow": (1.25, -0.5)}),
                                       (90, 700, 2, {"ar_alpha": 0.9, "force": 0x008})])
def test_slab_sequences_bit_identical(H, W, G, kw):
    """AR(1) sequences (each rank evolves the state of its own spectral rows; frame 2 of the
    sequence after frames 0-1, and frame 4 from a replayed start) and frozen flow in slab
    mode against the unsharded plan.  700-point rows take the one-CTA-per-row AR kernel by
    default; slab plans take the row-pair kernel there, so both sides force it (0x008) for
    an exact comparison (the two AR kernels agree to fp32 rounding, tests/test_gpu_parity)."""
    from paper_2210_06713_b200 import Plan, PlanConfig, slab_geometry
    C, K, T = 3, 16, 17
    basis, mlp = synth.basis(K, T, seed=0), synth.mlp_weights(K, seed=0)
    img = torch.from_numpy(synth.image(H, W, C, seed=5)).cuda()
    ref_plan = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=4.0, K=K, taps=T, max_batch=1, **kw), basis, mlp)
    plans = [Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=4.0, K=K, taps=T, slab_count=G, slab_rank=r, **kw), basis, mlp)
             for r in range(G)]
    counts = [p.slab_counts() for p in plans]
    for frame in (0, 1, 2, 4):
        ref = torch.empty((1, C, H, W), device="cuda")
        ref_plan.simulate_frames(img, 0, SEED, frame, 1, ref)
        sends = []
        for r, p in enumerate(plans):
            snd = torch.empty(int(counts[r][0].sum()), device="cuda")
            p.slab_rows(SEED, frame, snd)
            sends.append(snd)
        out = torch.empty((C, H, W), device="cuda")
        for r, p in enumerate(plans):
            recv = torch.cat([sends[s][int(counts[s][0][:r].sum()):int(counts[s][0][:r + 1].sum())]
                              for s in range(G)]).contiguous()
            g = slab_geometry(H, W, T, G, r)
            strip = torch.empty((C, H, g["x1"] - g["x0"]), device="cuda")
            p.slab_finish(recv, img, SEED, frame, strip)
            torch.cuda.synchronize()
            out[:, :, g["x0"]:g["x1"]] = strip
        assert torch.equal(out, ref[0]), frame


def test_slab_plan_rejects_frame_batches():
    from paper_2210_06713_b200 import P2SError, Plan, PlanConfig
    basis, mlp = synth.basis(16, 17), synth.mlp_weights(16)
    with pytest.raises(P2SError):
        Plan(PlanConfig(H=64, W=96, C=1, d_over_r0=2.0, K=16, taps=17, slab_count=2, slab_rank=2), basis, mlp)
    p = Plan(PlanConfig(H=64, W=96, C=1, d_over_r0=2.0, K=16, taps=17, slab_count=2, slab_rank=1), basis, mlp)
    with pytest.raises(P2SError):
        p.simulate_frames(torch.zeros((1, 64, 96), device="cuda"), 0, SEED, 0, 1, torch.empty((1, 1, 64, 96),
                                                                                               device="cuda"))
