"""Phase times of the literal drop-in path (ps_render_splats) at C2: run with
PS_TRACE_DROPIN=1 (and PS_DROPIN_RAW=1 for the raw-record A/B)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_18707_b200 import api  # noqa: E402

splats, deg = api.synthetic_splat3d(3, 2, 1_000_000)
cam = api.orbit_cameras(256, 1920, 1080)[0]
cfg = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.OpacityAware, sh_degree=deg)
r = api.Rasterizer(0)
lib = api.lib()
cs, gs = cam.to_struct(), cfg.to_struct()
rgb = np.zeros((1080, 1920, 3))
tr = np.zeros((1080, 1920))
dp = C.POINTER(C.c_double)
ts = []
for k in range(8):
    t0 = time.perf_counter()
    st = lib.ps_render_splats(r.handle, splats.ctypes.data_as(dp), len(splats), C.byref(cs), C.byref(gs),
                              rgb.ctypes.data_as(dp), tr.ctypes.data_as(dp), None)
    ts.append((time.perf_counter() - t0) * 1e3)
    assert st == 0, api.last_error(r.handle)
print("wall ms per call:", " ".join(f"{t:.2f}" for t in ts), file=sys.stderr)
