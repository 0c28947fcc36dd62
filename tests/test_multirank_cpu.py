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


def test_bench_frames_disjoint_and_ar_sequences_continue():
    total, F = 7, 4
    for world in (1, 2, 8):
        seen = set()
        for r in range(world):
            prev = None
            for s in range(total):
                so, f0 = runner.bench_frames(s, r, F, total, False)
                assert so == 0
                if prev is not None:
                    assert f0 == prev + F  # contiguous per rank
                prev = f0
                seen.update(range(f0, f0 + F))
        assert seen == set(range(world * total * F))
    for r in range(3):  # AR: a sequence per rank, frames 0, F, 2F, ... (never a replay)
        assert [runner.bench_frames(s, r, F, total, True) for s in range(total)] == [(r, s * F) for s in range(total)]


@pytest.mark.parametrize("workload", ["cfg3_512", "cfg4_1080p_ar"])
def test_bench_gpus2_dry_run_launches_two_ranks(workload):
    """`bench.py --gpus 2` without torchrun re-launches itself with two ranks (gloo in the
    dry run): both ranks join the communicator and the frame blocks of all steps are
    distinct."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1", "--workload", workload], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"]
    assert d["comm"]["world_size"] == 2 and d["comm"]["allreduce_ranks"] == 2
    assert d["distinct_frames"] == d["frames_expected"]


def _slab_worker(rank, world, port, q):
    """Ranks exchange synthetic row blocks laid out as p2s_slab_rows packs them; every
    received row must be the right (source row, pair, column) of the frame."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_06713_b200 import slab_geometry
        H, W, T, npairs = 40, 70, 9, 3
        geo = [slab_geometry(H, W, T, world, r) for r in range(world)]
        P = geo[0]["P"]

        def rows(g):
            out = []
            for kp in range(g["kp0"], g["kp1"]):
                out.append(kp)
                if kp != 0 and 2 * kp != P:
                    out.append(P - kp)
            return out

        me = geo[rank]
        snd_c, rcv_c = runner.slab_counts_host(H, W, T, world, rank, npairs)
        # value of (row ky, pair p, column x) of the row-transformed spectrum: a unique tag
        tag = lambda ky, p, x: float(ky * 1000 + p * 100000 + x)  # noqa: E731
        blocks = []
        for g in geo:
            blk = [[tag(ky, p, x), 0.5] for ky in rows(me) for p in range(npairs) for x in range(g["hx0"], g["hx1"])]
            blocks.append(torch.tensor(blk, dtype=torch.float32).reshape(-1))
        send = torch.cat(blocks)
        assert [b.numel() for b in blocks] == snd_c
        recv = torch.empty(sum(rcv_c))
        runner.slab_exchange(send, recv, snd_c, rcv_c)
        exp = [[tag(ky, p, x), 0.5] for g in geo for ky in rows(g) for p in range(npairs)
               for x in range(me["hx0"], me["hx1"])]
        ok = torch.equal(recv, torch.tensor(exp, dtype=torch.float32).reshape(-1))
        covered = sorted(ky for g in geo for ky in rows(g)) == list(range(P))
        q.put((rank, ok and covered))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_slab_exchange_transposes_rows_to_strips():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(out.values())
