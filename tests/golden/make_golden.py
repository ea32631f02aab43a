"""Generates tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each case stores the input splats (Splat3D rows), the ps_camera / ps_config
bytes, and the reference's fp64 framebuffer, counters and per-tile lists.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2603_18707_b200 import abi  # noqa: E402

NOMINAL_POLY1 = (0.773, -0.176)  # test_raster.cpp:18-20


def main() -> None:
    ref = Reference()
    out = {}
    cases = []
    grid, _ = ref.synth_scene(0, 1)
    sky, _ = ref.synth_scene(2, 5)
    rnd, _ = ref.synth_scene(1, 3)
    cam3 = ref.orbit_cameras(3, 96, 80)[1]
    p1 = ref.make_polynomial_kernel(abi.PS_KERNEL_POLY_RELU, NOMINAL_POLY1)
    for sname, splats, deg in (("grid", grid, 0), ("sky", sky, 0)):
        for mname, kern, mode in (("exp_stp", abi.kernel_struct(abi.PS_KERNEL_EXPONENTIAL), 0),
                                  ("poly1_zero", p1, 1), ("poly1_opacity", p1, 2)):
            cases.append((f"{sname}_{mname}", splats, cam3, kern, mode, deg))
    cases.append(("random300_poly1_opacity", rnd[:300], ref.orbit_cameras(1, 128, 96)[0], p1, 2, 3))
    for name, splats, cam, kern, mode, deg in cases:
        cfg = abi.default_config()
        cfg.kernel = kern
        cfg.culling_mode = mode
        cfg.sh_degree = deg
        rgb, tr, ctr = ref.render(splats, cam, cfg)
        off, idx, _ = ref.tile_lists(splats, cam, cfg)
        out[name + "_splats"] = np.ascontiguousarray(splats)
        out[name + "_cam"] = np.frombuffer(bytes(cam), dtype=np.uint8)
        out[name + "_cfg"] = np.frombuffer(bytes(cfg), dtype=np.uint8)
        out[name + "_rgb"] = rgb
        out[name + "_t"] = tr
        out[name + "_ctr"] = np.array([ctr[k] for k in sorted(ctr)], dtype=np.uint64)
        out[name + "_off"] = off
        out[name + "_idx"] = idx
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(cases), "cases")


if __name__ == "__main__":
    main()
