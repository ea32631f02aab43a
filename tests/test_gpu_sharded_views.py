"""View sharding end to end with real renders: two processes (one context each,
on the one GPU a gpurun box has; on an 8-GPU node each would own a device)
render disjoint contiguous shards of a 9-view C1 batch through ps_render_views,
the shards are gathered on rank 0 over gloo (sharding.gather_images), and the
gathered batch must equal a single-process render of the whole batch bit for
bit, and the reference within 1e-5 (images bit-identical for any
GPU count / views-per-GPU split)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18707_b200 import api
from paper_2603_18707_b200.sharding import gather_images, shard_views
from tests.helpers import config, max_abs, scene

pytestmark = pytest.mark.gpu

N_VIEWS = 9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    splats, deg = scene("g", 1, 10000)
    cams = api.orbit_cameras(N_VIEWS, 160, 120)
    return splats, cams, config("poly1", api.CullingMode.OpacityAware, deg)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        splats, cams, cfg = _inputs()
        mine = list(shard_views(N_VIEWS, world, rank))
        with api.Rasterizer(0) as r:
            ds = r.upload_splat3d(splats)
            out = r.render_views(ds, [cams[v] for v in mine], cfg, counters=False)
            ds.close()
        rgb = torch.from_numpy(np.stack([fb.rgb for fb, _ in out]))
        tr = torch.from_numpy(np.stack([fb.transmittance for fb, _ in out]))
        g_rgb = gather_images(rgb, N_VIEWS, dist)
        g_t = gather_images(tr, N_VIEWS, dist)
        if rank == 0:
            q.put((g_rgb.numpy(), g_t.numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_process_shards_equal_one_batch(gpu, reference):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_rgb, g_t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    splats, cams, cfg = _inputs()
    one = gpu.render_views(splats, cams, cfg, counters=False)
    for v in range(N_VIEWS):
        fb = one[v][0]
        assert np.array_equal(g_rgb[v].view(np.uint32), fb.rgb.view(np.uint32)), v
        assert np.array_equal(g_t[v].view(np.uint32), fb.transmittance.view(np.uint32)), v
        rgb_r, t_r, _ = reference.render(splats, cams[v].to_struct(), cfg.to_struct())
        assert max_abs(fb.rgb, rgb_r) <= 1e-5 and max_abs(fb.transmittance, t_r) <= 1e-5
