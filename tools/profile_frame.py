"""Renders one workload a few times on cuda:0 (for ncu launch lists / captures).

    python tools/profile_frame.py [--workload c2] [--kernel poly1] [--mode OpacityAware] [--frames 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_18707_b200 import api  # noqa: E402

W = {"c1": ("g", 1, 10_000, 256, 256), "c2": ("g", 2, 1_000_000, 1920, 1080),
     "c3": ("g", 4, 6_000_000, 3840, 2160), "c4": ("g", 5, 3_000_000, 1920, 1080),
     "c5": ("skewed", 3, 1_000_000, 1920, 1080), "g2m": ("g", 6, 2_000_000, 1920, 1080)}

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--kernel", default="poly1")
ap.add_argument("--mode", default="OpacityAware")
ap.add_argument("--frames", type=int, default=3)
a = ap.parse_args()
kind, seed, n, w, h = W[a.workload]
scene = api.Scene.synthetic(kind, seed, n)
cam = api.orbit_cameras(256, w, h)[0]
cfg = api.RasterConfig(kernel=api.fitted_kernel(a.kernel), culling_mode=getattr(api.CullingMode, a.mode),
                       sh_degree=scene.sh_degree)
with api.Rasterizer(0) as r:
    ds = r.upload(scene)
    r.set_timing(True)
    stages = []
    for _ in range(a.frames):
        fb, ctr = r.render(ds, cam, cfg, counters=False)
        st = r.stats()
        stages.append(st["stage_ms"])
        print(st, flush=True)
    ds.close()
    if a.frames >= 3:
        import statistics
        med = {k: round(1000 * statistics.median(s[k] for s in stages[1:]), 1) for k in stages[0]}
        print("median stage us:", med, "sum", round(sum(med.values()), 1), flush=True)
