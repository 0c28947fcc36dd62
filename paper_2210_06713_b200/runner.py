"""Frame-parallel multi-GPU execution.

Frames are independent given (seed, global frame index): the spectral noise is
counter-based, so every GPU simulates its own disjoint frame range with a plan
replica and no data-path collective ("scaling": "weak").  An AR(1) sequence split
across GPUs needs no communication either: a plan asked for frames starting at
frame0 > 0 rebuilds eta_{frame0-1} on the device by carry replay.  torch.distributed
(NCCL on GPUs, gloo in the CPU tests) is used only for barriers and max-over-ranks
timing.
"""
from __future__ import annotations


def frame_partition(total_frames: int, world: int, rank: int):
    """Contiguous balanced split of [0, total_frames): (first frame, count) of this rank."""
    if world < 1 or not (0 <= rank < world) or total_frames < 0:
        raise ValueError("bad partition arguments")
    base, extra = divmod(total_frames, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def step_frame0(step: int, rank: int, world: int, frames_per_rank: int) -> int:
    """First global frame of `rank` in benchmark step `step` (weak scaling: every step
    simulates world * frames_per_rank new frames, rank r owns a contiguous block)."""
    return (step * world + rank) * frames_per_rank


def bench_frames(step: int, rank: int, frames_per_step: int, total_steps: int, ar: bool):
    """(seed offset, first frame) of `rank` in benchmark step `step` of `total_steps`.

    White-noise frames are independent: rank r owns the contiguous global block
    [r * total_steps * F, (r + 1) * total_steps * F) of the one sequence, step by step.
    AR(1) workloads give every rank a whole sequence of its own (seed + r, frames 0, F,
    2F, ... in step order), so each call continues from the stored AR state and no rank
    ever replays frames (whole sequences per rank when there are >= G)."""
    if not (0 <= step < total_steps) or rank < 0 or frames_per_step < 1:
        raise ValueError("bad bench step arguments")
    if ar:
        return rank, step * frames_per_step
    return 0, (rank * total_steps + step) * frames_per_step


def sequence_assignment(n_sequences: int, world: int, rank: int):
    """Whole sequences per rank when there are at least as many sequences as ranks."""
    return list(range(rank, n_sequences, world))


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class FrameShardedRunner:
    """Runs this rank's share of a frame range through one plan (device buffers)."""

    def __init__(self, plan, rank: int = 0, world: int = 1):
        self.plan, self.rank, self.world = plan, rank, world

    def local_range(self, total_frames: int, frame_base: int = 0):
        s, n = frame_partition(total_frames, self.world, self.rank)
        return frame_base + s, n

    def run(self, img, img_frame_stride, seed, total_frames, out_local, frame_base=0, stream=None):
        """Simulate this rank's frames of [frame_base, frame_base + total_frames) into out_local."""
        f0, n = self.local_range(total_frames, frame_base)
        if n:
            img_local = img if img_frame_stride == 0 else img[f0 - frame_base:]
            self.plan.simulate_frames(img_local, img_frame_stride, seed, f0, n, out_local, stream)
        return f0, n


# ---------------------------------------------------------------- single-frame slab mode (NEXT-4)
def slab_counts_host(H: int, W: int, T: int, G: int, rank: int, npairs: int = 18, pad: int = 1):
    """Per-peer float counts of rank `rank`'s all-to-all (send[d], recv[s]), from the host
    geometry alone: block (s -> d) = rows_s x npairs x strip width of d, complex as 2 floats."""
    from .p2s import slab_geometry
    geo = [slab_geometry(H, W, T, G, r, pad) for r in range(G)]
    me = geo[rank]
    send = [2 * me["rows"] * npairs * (g["hx1"] - g["hx0"]) for g in geo]
    recv = [2 * g["rows"] * npairs * (me["hx1"] - me["hx0"]) for g in geo]
    return send, recv


def slab_exchange(send, recv, send_counts, recv_counts, group=None):
    """The transpose of SURVEY 8(e) NEXT-4: one all_to_all_single (NCCL over NVLink on GPUs,
    gloo in the CPU tests) with the per-peer split sizes of p2s_slab_counts."""
    import torch.distributed as dist
    dist.all_to_all_single(recv, send, [int(c) for c in recv_counts], [int(c) for c in send_counts], group=group)


def slab_simulate_frame(plan, img, seed, frame, send, recv, out_strip, group=None):
    """One frame on this rank in slab mode: row pass -> all-to-all -> strip pass."""
    snd, rcv = plan.slab_counts()
    plan.slab_rows(seed, frame, send)
    slab_exchange(send, recv, snd, rcv, group)
    plan.slab_finish(recv, img, seed, frame, out_strip)
