"""Times ps_render_views on a C4-like batch (64 views of G(3M, seed 5) at
1080p, poly1 / opacity-aware): device time per view, for A/B runs."""
import os
import sys
import ctypes as C
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_18707_b200 import api  # noqa: E402

scene = api.Scene.synthetic("g", 5, 3_000_000)
cams = api.orbit_cameras(64, 1920, 1080)
cfg = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware,
                       sh_degree=scene.sh_degree)
lib = api.lib()
with api.Rasterizer(0) as r:
    ds = r.upload(scene)
    cs = [c.to_struct() for c in cams]
    cam_arr = (type(cs[0]) * len(cs))(*cs)
    cfg_s = cfg.to_struct()
    rgb = torch.empty((len(cs), 1080, 1920, 3), device="cuda")
    t = torch.empty((len(cs), 1080, 1920), device="cuda")

    def run():
        st = lib.ps_render_views(r.handle, ds.handle, cam_arr, len(cs), C.byref(cfg_s), rgb.data_ptr(),
                                 t.data_ptr(), 1, None)
        assert st == 0, api.last_error(r.handle)
    run()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"ps_render_views (device outputs): {best / len(cs) * 1e3:.3f} ms/view")
    ds.close()
