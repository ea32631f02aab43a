"""CUPTI trace (torch.profiler) of a few ps_render calls on a tiny scene: the
host-side CUDA API calls of one frame and the device timeline, to see where a
frame's fixed overhead goes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2603_18707_b200 import api  # noqa: E402

n, w, h = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (1000, 64, 64)))
lib = api.lib()
sc = api.Scene.synthetic("g", 2, n)
r = api.Rasterizer(0)
ds = r.upload(sc)
cam = api.orbit_cameras(256, w, h)[0].to_struct()
cfg = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware,
                       sh_degree=3).to_struct()
rgb = torch.empty((h, w, 3), device="cuda")
t = torch.empty((h, w), device="cuda")


def one():
    assert lib.ps_render(r.handle, ds.handle, C.byref(cam), C.byref(cfg), rgb.data_ptr(), t.data_ptr(), 1, None) == 0


for _ in range(20):
    one()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        one()
    torch.cuda.synchronize()
evs = sorted(prof.events(), key=lambda e: e.time_range.start)
t0 = None
for e in evs:
    if t0 is None:
        t0 = e.time_range.start
    dev = "GPU" if e.device_type == torch.autograd.DeviceType.CUDA else "cpu"
    print(f"{(e.time_range.start - t0):10.1f} {e.time_range.elapsed_us():8.1f} {dev} {e.name[:70]}")
