"""RasterConfig corners the reference accepts, on the GPU path, against the
reference (raster.hpp:19-35, raster.cpp:13-23 validation):

* the mismatched culling kernel of acceptance criterion #5's "unsafety" half
  (acceptance.cpp:176-178): exp blending with a poly1 `culling_kernel`
  (raster.hpp:25-27), for every culling mode that consults it;
* `clamp_before_blend = true` (raster.cpp:256-260);
* non-default epsilon and transmittance floor (the fp32 certification margins
  of the blend and of the blend record are derived from them);
* v_dilation other than 0.3;
* SH degrees below the scene's, negative included (eval_sh_color keeps the DC
  term for any degree < 1, projection.cpp:93-95).

Each case is checked in both blend instantiations: with counters (all six
equal to the reference's) and without (the timed one), two frames per context
(sized, then speculative). Images within 1e-5 max-abs."""
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import camera, config, kernel, max_abs, scene
from tests.test_gpu_timed_path import render_device_nocount

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _check_both(gpu, reference, splats, cam, cfg):
    rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
    ds = gpu.upload_splat3d(splats)
    try:
        for _ in range(2):
            fb, ctr = gpu.render(ds, cam, cfg)
            assert ctr.as_dict() == ctr_r
            assert max_abs(fb.rgb, rgb_r) <= TOL and max_abs(fb.transmittance, t_r) <= TOL
            rgb, tr = render_device_nocount(gpu, ds, cam, cfg)
            assert max_abs(rgb, rgb_r) <= TOL and max_abs(tr, t_r) <= TOL
        off, idx, _ = gpu.tile_lists(ds, cam, cfg)
        r_off, r_idx, _ = reference.tile_lists(splats, cam.to_struct(), cfg.to_struct())
        assert (off == r_off).all() and (idx == r_idx).all()
    finally:
        ds.close()
    return rgb_r, t_r


@pytest.mark.parametrize("mode", [api.CullingMode.OpacityAware, api.CullingMode.ZeroCrossing,
                                  api.CullingMode.StopThePop])
@pytest.mark.parametrize("bound", ["poly1", "nominal", "poly3"])
def test_exp_blend_with_poly_culling_kernel(gpu, reference, mode, bound):
    """acceptance.cpp:176-178: exp blended inside poly bounds (visible blocky
    artefacts in the reference, reproduced here to 1e-5)."""
    splats, deg = scene("random", 0)
    cfg = config("exp", mode, deg)
    cfg.culling_kernel = kernel(bound)
    _check_both(gpu, reference, splats, camera(3, 256, 192, 0), cfg)


@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop),
                                        ("poly2p", api.CullingMode.OpacityAware)])
def test_clamp_before_blend(gpu, reference, kname, mode):
    splats, deg = scene("sky", 3)  # colours near 3: the clamp binds
    cfg = config(kname, mode, deg, clamp_before_blend=True)
    _check_both(gpu, reference, splats, camera(3, 200, 160, 1), cfg)
    splats, deg = scene("random", 2)
    _check_both(gpu, reference, splats, camera(3, 200, 160, 2), config(kname, mode, deg, clamp_before_blend=True))


@pytest.mark.parametrize("eps", [1e-3, 0.02, 0.2])
@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop),
                                        ("poly3", api.CullingMode.ZeroCrossing)])
def test_epsilon(gpu, reference, eps, kname, mode):
    splats, deg = scene("g", 1, 10000)
    _check_both(gpu, reference, splats, camera(1, 256, 256, 0), config(kname, mode, deg, epsilon=eps))


@pytest.mark.parametrize("floor", [0.0, 1e-2, 0.3])
@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop)])
def test_transmittance_floor(gpu, reference, floor, kname, mode):
    splats, deg = scene("g", 1, 10000)
    _check_both(gpu, reference, splats, camera(1, 256, 256, 0),
                config(kname, mode, deg, transmittance_floor=floor))


@pytest.mark.parametrize("v", [0.0, 0.1, 1.0])
def test_v_dilation(gpu, reference, v):
    splats, deg = scene("g", 1, 10000)
    _check_both(gpu, reference, splats, camera(1, 256, 256, 0),
                config("poly1", api.CullingMode.OpacityAware, deg, v_dilation=v))


@pytest.mark.parametrize("sh", [-2, -1, 0, 1, 2, 3, 7])
def test_sh_degree(gpu, reference, sh):
    splats, _ = scene("random", 1)
    _check_both(gpu, reference, splats, camera(2, 160, 128, 1), config("poly1", api.CullingMode.OpacityAware, sh))


def test_combined_corners(gpu, reference):
    """Everything non-default at once."""
    splats, deg = scene("g", 3, 20000)
    cfg = config("exp", api.CullingMode.OpacityAware, 1, epsilon=0.01, transmittance_floor=3e-3, v_dilation=0.2,
                 clamp_before_blend=True)
    cfg.culling_kernel = kernel("poly2p")
    _check_both(gpu, reference, splats, camera(5, 320, 200, 3), cfg)
