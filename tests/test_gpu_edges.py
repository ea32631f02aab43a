"""Edge cases against the reference on the GPU path: tile sizes other than 16
(the generic blend kernel), ragged and tiny images, empty and fully culled
scenes, a single splat, and the error convention for bad cameras and
degenerate covariances (raster.cpp:13-23, projection.cpp:10-22,67)."""
import numpy as np
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import camera, config, max_abs, scene

pytestmark = pytest.mark.gpu

IMAGE_TOL = 1e-5


def _check(gpu, reference, splats, cam, cfg):
    rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
    fb, ctr = gpu.render(splats, cam, cfg)
    assert ctr.as_dict() == ctr_r
    assert max_abs(fb.rgb, rgb_r) <= IMAGE_TOL and max_abs(fb.transmittance, t_r) <= IMAGE_TOL
    return fb, ctr


@pytest.mark.parametrize("tile", [1, 8, 12, 32, 33, 48, 64, 100])
@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop)])
def test_other_tile_sizes(gpu, reference, tile, kname, mode):
    splats, deg = scene("random", 3)
    cfg = config(kname, mode, deg, tile_size=tile)
    _check(gpu, reference, splats, camera(1, 256, 192, 0), cfg)
    off, idx, _ = gpu.tile_lists(splats, camera(1, 256, 192, 0), cfg)
    r_off, r_idx, _ = reference.tile_lists(splats, camera(1, 256, 192, 0).to_struct(), cfg.to_struct())
    assert np.array_equal(off, r_off) and np.array_equal(idx, r_idx)


@pytest.mark.parametrize("w,h", [(1, 1), (17, 9), (100, 37), (16, 16), (33, 250)])
def test_ragged_images(gpu, reference, w, h):
    splats, deg = scene("g", 1, 10000)
    _check(gpu, reference, splats, camera(1, w, h, 0), config("poly1", api.CullingMode.OpacityAware, deg))


def test_empty_scene(gpu, reference):
    splats, deg = scene("g", 1, 100)
    empty = splats[:0]
    fb, ctr = _check(gpu, reference, empty, camera(1, 64, 48, 0), config("poly1", api.CullingMode.OpacityAware, deg))
    assert np.all(fb.rgb == 0.0) and np.all(fb.transmittance == 1.0)
    assert ctr.tile_pairs_after_tight_test == 0


def test_fully_culled_scene(gpu, reference):
    splats, deg = scene("g", 1, 1000)
    behind = splats.copy()
    cam = camera(1, 64, 48, 0)
    # move every splat behind the camera: mean = camera position - 5 * forward
    R = np.array(cam.rotation).reshape(3, 3)
    fwd = R[2]
    behind[:, 0:3] = cam.position() - 5.0 * fwd
    fb, ctr = _check(gpu, reference, behind, cam, config("exp", api.CullingMode.StopThePop, deg))
    assert ctr.splats_frustum_culled == len(behind) and np.all(fb.transmittance == 1.0)


def test_single_splat(gpu, reference):
    splats, deg = scene("g", 1, 1000)
    _check(gpu, reference, splats[:1], camera(1, 128, 128, 0), config("poly3", api.CullingMode.OpacityAware, deg))


def test_views_of_empty_scene(gpu):
    splats, deg = scene("g", 1, 100)
    out = gpu.render_views(splats[:0], api.orbit_cameras(3, 32, 32), config("poly1", api.CullingMode.OpacityAware, deg))
    assert len(out) == 3 and all(np.all(fb.transmittance == 1.0) for fb, _ in out)


def test_non_orthonormal_camera_raises(gpu):
    splats, deg = scene("g", 1, 100)
    cam = camera(1, 64, 48, 0)
    cam.rotation = [2.0 * v if i == 0 else v for i, v in enumerate(cam.rotation)]
    with pytest.raises(api.NonOrthonormalRotation):
        gpu.render(splats, cam, config("poly1", api.CullingMode.OpacityAware, deg))


def test_invalid_config_raises(gpu):
    splats, deg = scene("g", 1, 100)
    for bad in (dict(tile_size=0), dict(epsilon=0.0), dict(transmittance_floor=1.0)):
        with pytest.raises(api.InvalidArgument):
            gpu.render(splats, camera(1, 64, 48, 0), config("poly1", api.CullingMode.OpacityAware, deg, **bad))


def test_degenerate_covariance_raises_like_reference(gpu, reference):
    """No dilation and a zero-scale splat: det(cov_aa) <= 1e-12 (projection.cpp:67).
    The reference throws DegenerateCovariance (inside its OpenMP region the
    process would terminate; the shim calls it where it can be caught)."""
    splats, deg = scene("g", 1, 100)
    bad = splats.copy()
    bad[7, 3:6] = 0.0  # scale
    cfg = config("poly1", api.CullingMode.OpacityAware, deg, v_dilation=0.0)
    with pytest.raises(api.DegenerateCovariance):
        gpu.render(bad, camera(1, 64, 48, 0), cfg)
