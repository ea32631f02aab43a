"""Host-side cost of one ps_render call: wall time per call on a tiny scene (GPU
work ~ nothing) vs a C2 frame's wall and device (event) time."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_18707_b200 import api  # noqa: E402

lib = api.lib()
for kind, n, w, h in (("g", 1000, 64, 64), ("g", 1_000_000, 1920, 1080)):
    sc = api.Scene.synthetic(kind, 2, n)
    r = api.Rasterizer(0)
    ds = r.upload(sc)
    cam = api.orbit_cameras(256, w, h)[0].to_struct()
    cfg = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware,
                           sh_degree=3).to_struct()
    rgb = torch.empty((h, w, 3), device="cuda")
    t = torch.empty((h, w), device="cuda")
    stream = torch.cuda.ExternalStream(lib.ps_ctx_stream(r.handle))

    def one():
        assert lib.ps_render(r.handle, ds.handle, C.byref(cam), C.byref(cfg), rgb.data_ptr(), t.data_ptr(), 1, None) == 0
    for _ in range(10):
        one()
    torch.cuda.synchronize()
    K = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(K):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / K * 1e6
    dev = e0.elapsed_time(e1) / K * 1e3
    print(f"n={n}: wall {wall:.1f} us/call, device span {dev:.1f} us/call")
    ds.close()
    r.close()
