#!/usr/bin/env python
"""Single-frame 4K latency in slab mode, per-rank compute measured on
one GPU: for G ranks, each rank's two phases (row pass + pack; unpack + column pass + warp
+ MLP + blur + strip copy) are timed alone with CUDA events (as each would run on its own
GPU), the all-to-all is emulated by device copies (not timed) and estimated from its bytes
at NVLink 5's 900 GB/s per direction.  Latency estimate = max_r(phase 1) + exchange +
max_r(phase 2), against the unsharded single-GPU frame timed the same way.

    python tools/slab_latency_emulated.py [--ranks 2,4,8] [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2210_06713_b200 import Plan, PlanConfig, slab_geometry  # noqa: E402

SEED = 2210


def ev_time(fn, reps):
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
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    w = bench.WORKLOADS["cfg5_4k"]
    H, W, C, K, T = w["H"], w["W"], w["C"], w["K"], w["T"]
    basis, mlp = synth.basis(K, T, seed=0), synth.mlp_weights(K, seed=0)
    img = torch.from_numpy(synth.image(H, W, C, seed=0)).cuda()
    base = Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=w["d_over_r0"], K=K, taps=T, max_batch=1, **bench.STEP5), basis,
                mlp)
    out = torch.empty((1, C, H, W), device="cuda")
    ms_single = ev_time(lambda: base.simulate_frames(img, 0, SEED, 0, 1, out), args.reps)
    del base
    res = {"workload": "cfg5_4k one frame (2160x3840 RGB, K=100, T=33)", "single_gpu_ms": ms_single, "sharded": {}}
    for G in [int(g) for g in args.ranks.split(",")]:
        plans = [Plan(PlanConfig(H=H, W=W, C=C, d_over_r0=w["d_over_r0"], K=K, taps=T, slab_count=G, slab_rank=r,
                                 **bench.STEP5), basis, mlp) for r in range(G)]
        counts = [p.slab_counts() for p in plans]
        sends = [torch.empty(int(c[0].sum()), device="cuda") for c in counts]
        t1 = [ev_time(lambda p=p, s=s: p.slab_rows(SEED, 0, s), args.reps) for p, s in zip(plans, sends)]
        t2, xbytes = [], []
        for r, p in enumerate(plans):
            parts = []
            for s in range(G):
                off = int(counts[s][0][:r].sum())
                parts.append(sends[s][off:off + int(counts[s][0][r])])
            recv = torch.cat(parts).contiguous()
            g = slab_geometry(H, W, T, G, r)
            strip = torch.empty((C, H, g["x1"] - g["x0"]), device="cuda")
            t2.append(ev_time(lambda p=p, recv=recv, strip=strip: p.slab_finish(recv, img, SEED, 0, strip), args.reps))
            sent = int(counts[r][0].sum() - counts[r][0][r]) * 4
            got = int(counts[r][1].sum() - counts[r][1][r]) * 4
            xbytes.append(max(sent, got))
        x_ms = max(xbytes) / 900e9 * 1e3
        lat = max(t1) + x_ms + max(t2)
        res["sharded"][G] = {"phase1_ms_max": max(t1), "phase2_ms_max": max(t2), "exchange_bytes_per_rank_max": max(xbytes),
                             "exchange_ms_at_900GBps": x_ms, "latency_ms_estimate": lat,
                             "speedup_vs_single_gpu": ms_single / lat}
        del plans, sends
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
