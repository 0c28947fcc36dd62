"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: frame partitioning,
weak-scaling step numbering, max-over-ranks timing and the sequence assignment.
The GPU data path has no collective (frames are independent), so these cover
everything bench.py does across ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2210_06713_b200 import runner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        res["part"] = runner.frame_partition(10, world, rank)
        res["max"] = runner.max_over_ranks(1.5 + rank)
        res["sum"] = runner.sum_over_ranks(2.0)
        res["f0"] = [runner.step_frame0(s, rank, world, 64) for s in range(3)]
        res["seq"] = runner.sequence_assignment(5, world, rank)
        t = torch.tensor([rank])
        dist.all_reduce(t)
        res["allreduce"] = int(t.item())
        dist.barrier()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_and_timing_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # partition: disjoint, contiguous, covering [0, 10)
    frames = []
    for r in range(world):
        s, n = out[r]["part"]
        frames.extend(range(s, s + n))
    assert frames == list(range(10))
    assert all(out[r]["max"] == 2.5 for r in range(world))
    assert all(out[r]["sum"] == 4.0 for r in range(world))
    # weak scaling: every (step, rank) block of 64 frames is distinct
    blocks = sorted(f for r in range(world) for f in out[r]["f0"])
    assert blocks == [64 * i for i in range(6)]
    assert sorted(out[0]["seq"] + out[1]["seq"]) == list(range(5))
    assert out[0]["allreduce"] == 1


def test_partition_edge_cases():
    assert runner.frame_partition(0, 4, 3) == (0, 0)
    assert runner.frame_partition(3, 4, 3) == (3, 0)
    assert [runner.frame_partition(7, 3, r) for r in range(3)] == [(0, 3), (3, 2), (5, 2)]
    with pytest.raises(ValueError):
        runner.frame_partition(5, 2, 2)
