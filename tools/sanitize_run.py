"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): C1 (G(10k, seed 1), 256x256) through every blend variant the
bench and tests use — poly1 / exp / poly3 / a non-monotone kernel, 16x16 and
8x8 and 48x48 tiles, a sized then a speculative frame, counter-free frames, a
view batch, a crowded tile with equal depths, low-opacity crowded tiles (the
blend's prefix sort completed mid-walk and before the replay), the TMA-staged
K1, and the device metrics."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_18707_b200 import api  # noqa: E402
from tests.helpers import crowded_scene  # noqa: E402

splats, deg = api.synthetic_splat3d(3, 1, 10000)
cams = api.orbit_cameras(4, 256, 256)
cells = [("poly1", api.CullingMode.OpacityAware, 16), ("exp", api.CullingMode.StopThePop, 16),
         ("poly3", api.CullingMode.OpacityAware, 16), ("poly1", api.CullingMode.OpacityAware, 8)]
with api.Rasterizer(0) as r:
    ds = r.upload_splat3d(splats)
    for kname, mode, tile in cells:
        cfg = api.RasterConfig(kernel=api.fitted_kernel(kname), culling_mode=mode, sh_degree=deg, tile_size=tile)
        for _ in range(2):
            fb, ctr = r.render(ds, cams[0], cfg)
        print(kname, tile, ctr.tile_pairs_after_tight_test, flush=True)
    k = api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, (0.5, 0.1, -0.05))
    r.render(ds, cams[0], api.RasterConfig(kernel=k, culling_mode=api.CullingMode.ZeroCrossing, sh_degree=deg))
    cfg = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware, sh_degree=deg)
    out = r.render_views(ds, cams, cfg)
    a, b = out[0][0], out[1][0]
    print("metrics", r.image_metrics(a, b).psnr_db, flush=True)
    cs, cdeg, ccam = crowded_scene(1300, 16, True)
    r.render(cs, ccam, cfg)
    r.render(cs, ccam, cfg)
    # low opacities: the blend sorts past its ranked prefix mid-walk / before the replay
    ls, ldeg, lcam = crowded_scene(700, 21, False, opacity=(0.04, 0.12))
    for kname, mode in (("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop)):
        lc = api.RasterConfig(kernel=api.fitted_kernel(kname), culling_mode=mode, sh_degree=ldeg)
        r.render(ls, lcam, lc)
        r.render(ls, lcam, lc, counters=False)
    r.render(ds, cams[1], cfg, counters=False)  # the counter-free blend the bench times
    r.render(ds, cams[1], api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware,
                                           sh_degree=deg, tile_size=48))
    ds.close()
print("sanitize workload done")
