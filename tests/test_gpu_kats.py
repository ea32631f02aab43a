"""The reference's known-answer tests for this path (test_raster.cpp,
acceptance.cpp, the C1 probe counters of SURVEY §8c) and the committed golden
fixtures (tests/golden/golden.npz, made from the reference by
tests/golden/make_golden.py), run through the GPU path. Counters, tile lists and
pair counts are exact; images use the fp32 blend's 1e-5 contract (the
reference's own 1e-12 image tolerances are for its fp64 renderer)."""
import math
import os

import numpy as np
import pytest

from paper_2603_18707_b200 import abi, api
from tests.test_oracle import GOLDEN, _cam, _cfg, _single_splat

pytestmark = pytest.mark.gpu

IMAGE_TOL = 1e-5


class GpuImpl:
    """The oracle's calling convention (ctypes structs in, fp64 arrays and a
    counter dict out) over the device rasterizer."""

    def __init__(self, r: api.Rasterizer):
        self.r = r

    def render(self, splats, cam, cfg):
        fb, ctr = self.r.render(np.asarray(splats), api.Camera.from_struct(cam), _config(cfg))
        return fb.rgb.astype(np.float64), fb.transmittance.astype(np.float64), ctr.as_dict()

    def count_pairs(self, splats, cam, cfg):
        return self.r.count_pairs(np.asarray(splats), api.Camera.from_struct(cam), _config(cfg)).as_dict()

    def tile_lists(self, splats, cam, cfg):
        return self.r.tile_lists(np.asarray(splats), api.Camera.from_struct(cam), _config(cfg))


def _config(c: abi.ps_config) -> api.RasterConfig:
    return api.RasterConfig(tile_size=c.tile_size, epsilon=c.epsilon, transmittance_floor=c.transmittance_floor,
                            culling_mode=api.CullingMode(c.culling_mode), kernel=api.KernelSpec.from_struct(c.kernel),
                            culling_kernel=api.KernelSpec.from_struct(c.culling_kernel) if c.has_culling_kernel
                            else None, v_dilation=c.v_dilation, sh_degree=c.sh_degree,
                            clamp_before_blend=bool(c.clamp_before_blend), thread_count=c.thread_count)


@pytest.fixture(scope="module")
def dev(gpu):
    return GpuImpl(gpu)


def test_empty_scene_is_background(dev, reference):
    """test_raster.cpp:124-132"""
    rgb, tr, ctr = dev.render(_single_splat(0.05, 1.0)[:0], _cam(40, 30, 30.0, 20.0), _cfg(reference, "exp", 0))
    assert np.all(rgb == 0.0) and np.all(tr == 1.0) and ctr["fragments_blended"] == 0


def test_single_splat_centre_pixel(dev, reference):
    """test_raster.cpp:134-160: a white splat's centre pixel has colour
    opacity_eff and transmittance 1 - opacity_eff."""
    s = _single_splat(0.05, 1.0, 1.0)
    cam = _cam(65, 65, 60.0, 32.5)
    rgb, tr, ctr = dev.render(s, cam, _cfg(reference, "exp", 0))
    o = reference.project_splat(s[0], cam, 0.3, 3)[9]
    assert abs(rgb[32, 32, 0] - o) <= IMAGE_TOL and abs(tr[32, 32] - (1 - o)) <= IMAGE_TOL
    assert 0 < ctr["fragments_blended"] <= ctr["kernel_evaluations"]


def test_one_small_splat_one_pair(dev, reference):
    """test_raster.cpp:162-179"""
    s = _single_splat(0.01, 0.9)
    assert dev.count_pairs(s, _cam(64, 64, 50.0, 24.0), _cfg(reference, "nominal", 2))[
        "tile_pairs_after_tight_test"] == 1


def test_culling_safety_and_pair_order(dev, reference):
    """test_raster.cpp:231-263: opacity-aware and StopThePop give the same poly1
    image (bitwise on the reference; here the same counters and images within
    the contract), and pairs(opacity) <= pairs(zero) <= pairs(stp)."""
    grid, _ = reference.synth_scene(0, 1)
    cam = reference.orbit_cameras(1, 128, 96)[0]
    a = dev.render(grid, cam, _cfg(reference, "nominal", 2, 0))
    b = dev.render(grid, cam, _cfg(reference, "nominal", 0, 0))
    assert np.abs(a[0] - b[0]).max() <= IMAGE_TOL and np.abs(a[1] - b[1]).max() <= IMAGE_TOL
    assert a[2]["tile_pairs_after_tight_test"] <= b[2]["tile_pairs_after_tight_test"]
    assert a[2]["fragments_blended"] == b[2]["fragments_blended"]
    rnd, _ = reference.synth_scene(1, 3)
    cam = reference.orbit_cameras(1, 256, 192)[0]
    pairs = [dev.count_pairs(rnd, cam, _cfg(reference, "nominal", m))["tile_pairs_after_tight_test"]
             for m in (2, 1, 0)]
    assert pairs[0] <= pairs[1] <= pairs[2]


def test_c1_counters_match_survey_probe(dev, reference):
    """C1 = G(10k, seed 1), 256x256, poly1/opacity: 24,725 pairs,
    5,628,075 evaluations, 775,924 fragments blended."""
    splats, deg = api.synthetic_splat3d(3, 1, 10000)
    cam = reference.orbit_cameras(1, 256, 256)[0]
    c = dev.count_pairs(splats, cam, _cfg(reference, "poly1", 2, deg))
    assert c["tile_pairs_after_tight_test"] == 24725
    _, _, ctr = dev.render(splats, cam, _cfg(reference, "poly1", 2, deg))
    assert ctr["kernel_evaluations"] == 5628075 and ctr["fragments_blended"] == 775924


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden fixtures not generated")
def test_golden_fixtures_on_gpu(dev):
    """Every committed golden case (reference images, counters, tile lists)."""
    g = np.load(GOLDEN)
    keys = sorted(k[:-4] for k in g.files if k.endswith("_rgb"))
    assert keys
    for key in keys:
        splats = g[key + "_splats"]
        cam = abi.ps_camera.from_buffer_copy(g[key + "_cam"].tobytes())
        cfg = abi.ps_config.from_buffer_copy(g[key + "_cfg"].tobytes())
        rgb, tr, ctr = dev.render(splats, cam, cfg)
        assert np.abs(rgb - g[key + "_rgb"]).max(initial=0) <= IMAGE_TOL, key
        assert np.abs(tr - g[key + "_t"]).max(initial=0) <= IMAGE_TOL, key
        assert [ctr[k] for k in sorted(ctr)] == list(g[key + "_ctr"]), key
        off, idx, _ = dev.tile_lists(splats, cam, cfg)
        assert np.array_equal(off, g[key + "_off"]) and np.array_equal(idx, g[key + "_idx"]), key
        assert math.isfinite(float(rgb.sum()))
