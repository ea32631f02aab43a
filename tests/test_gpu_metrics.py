"""Device image metrics, compare() and the ablation grid against the reference
(metrics.cpp:13-157, tools/main.cpp:300-345).

Per-pixel terms are computed in the reference's fp64 operation order; only the
sums over pixels are reduced in a different (fixed) order, so psnr / ssim agree
to ~1e-12 relative on identical inputs, are bit-reproducible from call to call,
and max_abs_diff is exact. compare() renders
with our rasterizer, whose images are within 1e-5 of the reference's, so its
psnr / ssim are held to the tolerance that image error implies.
"""
import math

import numpy as np
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import camera, config, scene

pytestmark = pytest.mark.gpu


def _fb(rgb, t):
    h, w = t.shape
    return api.Framebuffer(w, h, rgb, t)


@pytest.fixture(scope="module")
def c1():
    splats, deg = scene("g", 1, 10000)
    return splats, deg, camera(1, 256, 256, 0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("bg", [(1.0, 1.0, 1.0), (0.0, 0.25, 0.5)])
def test_image_metrics_match_reference(gpu, reference, c1, dtype, bg):
    splats, deg, cam = c1
    a, _ = gpu.render(splats, cam, config("exp", api.CullingMode.StopThePop, deg))
    b, _ = gpu.render(splats, cam, config("poly1", api.CullingMode.OpacityAware, deg))
    fa = _fb(a.rgb.astype(dtype), a.transmittance.astype(dtype))
    fb = _fb(b.rgb.astype(dtype), b.transmittance.astype(dtype))
    got = gpu.image_metrics(fa, fb, bg)
    p, m, s = reference.compare_images(fa.rgb, fa.transmittance, fb.rgb, fb.transmittance, bg, with_ssim=True)
    assert got.max_abs_diff == m
    assert math.isclose(got.psnr_db, p, rel_tol=1e-12)
    assert math.isclose(got.ssim, s, rel_tol=1e-12)


def test_metrics_bit_reproducible(gpu, c1):
    """The pixel sums are reduced in a fixed order: repeated calls (and a 1080p
    image, whose SSIM tiles outnumber the grid) give the same bits."""
    splats, deg, cam = c1
    for w, h in ((256, 256), (1920, 1080)):
        cam = camera(1, w, h, 0)
        a, _ = gpu.render(splats, cam, config("exp", api.CullingMode.StopThePop, deg))
        b, _ = gpu.render(splats, cam, config("poly1", api.CullingMode.OpacityAware, deg))
        runs = [gpu.image_metrics(a, b) for _ in range(3)]
        assert all((r.psnr_db, r.ssim, r.max_abs_diff) == (runs[0].psnr_db, runs[0].ssim, runs[0].max_abs_diff)
                   for r in runs)


def test_identical_images(gpu, c1):
    splats, deg, cam = c1
    a, _ = gpu.render(splats, cam, config("poly1", api.CullingMode.OpacityAware, deg))
    got = gpu.image_metrics(a, a)
    assert got.psnr_db == math.inf and got.max_abs_diff == 0.0
    assert got.ssim == pytest.approx(1.0, abs=1e-12)


def test_small_image_has_no_ssim(gpu):
    splats, deg = scene("grid", 1)
    cam = camera(3, 10, 8, 1)
    a, _ = gpu.render(splats, cam, config("poly1", api.CullingMode.OpacityAware, deg))
    b, _ = gpu.render(splats, cam, config("exp", api.CullingMode.StopThePop, deg))
    got = gpu.image_metrics(a, b)
    assert got.ssim is None and got.max_abs_diff > 0.0


def test_dimension_mismatch(gpu):
    a = api.Framebuffer(2, 2, np.zeros((2, 2, 3), np.float32), np.ones((2, 2), np.float32))
    b = api.Framebuffer(3, 2, np.zeros((2, 3, 3), np.float32), np.ones((2, 3), np.float32))
    with pytest.raises(api.Error):
        gpu.image_metrics(a, b)


def test_compare_matches_reference(gpu, reference, c1):
    splats, deg, cam = c1
    ca = config("exp", api.CullingMode.StopThePop, deg)
    cb = config("poly1", api.CullingMode.OpacityAware, deg)
    r = gpu.compare(splats, cam, ca, cb)
    ra, ta, ctr_a = reference.render(splats, cam.to_struct(), ca.to_struct())
    rb, tb, ctr_b = reference.render(splats, cam.to_struct(), cb.to_struct())
    p, m, s = reference.compare_images(ra, ta, rb, tb, with_ssim=True)
    assert r.counters_a.as_dict() == ctr_a and r.counters_b.as_dict() == ctr_b
    assert r.pair_ratio == ctr_b["tile_pairs_after_tight_test"] / ctr_a["tile_pairs_after_tight_test"]
    # our images are within 1e-5 of the reference's: max_abs moves by <= 2e-5,
    # the MSE by <= 2 * 2e-5 * sqrt(mse) + (2e-5)^2
    assert abs(r.max_abs_diff - m) <= 2e-5
    mse_ref = 10.0 ** (-p / 10.0)
    dmse = 4e-5 * math.sqrt(mse_ref) + 4e-10
    assert abs(10.0 ** (-r.psnr_db / 10.0) - mse_ref) <= dmse
    assert abs(r.ssim - s) <= 1e-4


def test_ablation_grid_counts_match_reference(gpu, reference, c1):
    splats, deg, cam = c1
    reports, csv = api.ablation_grid(gpu, splats, cam, api.RasterConfig(sh_degree=deg))
    lines = csv.strip().split("\n")
    assert lines[0] == "label_a,label_b,psnr_db,ssim,max_abs_diff,pairs_a,pairs_b,pair_ratio"
    assert [ln.split(",")[1] for ln in lines[1:]] == [c[0] for c in api.ABLATION_CELLS]
    for label, kname, mode in api.ABLATION_CELLS:
        want = reference.count_pairs(splats, cam.to_struct(), config(kname, mode, deg).to_struct())
        assert reports[label].counters_b.tile_pairs_after_tight_test == want["tile_pairs_after_tight_test"]
    # the reference row compared with itself
    assert reports["exp/stp"].psnr_db == math.inf and reports["exp/stp"].pair_ratio == 1.0
    # measured device times for every cell (the paper's Table 3 with times)
    for label, _, _ in api.ABLATION_CELLS:
        r = reports[label]
        assert r.frame_ms_a > 0.0 and r.frame_ms_b > 0.0 and 0.0 < r.blend_ms_b <= r.frame_ms_b
