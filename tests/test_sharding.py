"""Multi-process host logic of the view-sharded path, on CPU with gloo
(world_size 2, 127.0.0.1 rendezvous): shard partitioning, max-over-ranks timing
and the optional final image gather, plus the bench's reference arm under a
non-zero rank (must exit without work)."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18707_b200.sharding import gather_images, max_over_ranks, shard_views

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,world", [(256, 1), (256, 2), (256, 8), (255, 8), (3, 4)])
def test_shards_partition_views(n, world):
    seen = []
    for r in range(world):
        s = shard_views(n, world, r)
        seen.extend(s)
        assert abs(len(s) - n / world) < 1
    assert seen == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 7
        views = shard_views(n, world, rank)
        # stand-in per-view "images": value = view index
        imgs = torch.stack([torch.full((2, 3, 4), float(v)) for v in views])
        full = gather_images(imgs, n, dist)
        m = max_over_ranks(10.0 * (rank + 1), dist)
        if rank == 0:
            q.put(([float(full[v, 0, 0, 0]) for v in range(n)], m))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals, m = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert vals == [float(v) for v in range(7)]
    assert m == 20.0


def test_reference_arm_nonzero_rank_exits_clean():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "1"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""
