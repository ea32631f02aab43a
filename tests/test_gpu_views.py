"""View batches (ps_render_views): K1 fused over up to 4 views (each splat's
inputs read once), each view's binning and blend on its own
stream. Every view must equal the single-view render bit for bit (same
kernels, same arithmetic) and so match the reference as ps_render does."""
import numpy as np
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import config, scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware),
                                        ("exp", api.CullingMode.StopThePop),
                                        ("poly3", api.CullingMode.OpacityAware)])
@pytest.mark.parametrize("n_views", [1, 3, 6])
def test_views_equal_single_renders(gpu, kname, mode, n_views):
    splats, deg = scene("g", 1, 10000)
    cams = api.orbit_cameras(8, 256, 192)[:n_views]
    cfg = config(kname, mode, deg)
    ds = gpu.upload_splat3d(splats)
    for _ in range(2):  # the second pass takes the speculative (no mid-frame sync) path
        got = gpu.render_views(ds, cams, cfg)
        for cam, (fb, ctr) in zip(cams, got):
            want, wctr = gpu.render(ds, cam, cfg)
            assert ctr.as_dict() == wctr.as_dict()
            assert np.array_equal(fb.rgb, want.rgb) and np.array_equal(fb.transmittance, want.transmittance)
    ds.close()


def test_views_match_reference(gpu, reference):
    splats, deg = scene("g", 1, 10000)
    cams = api.orbit_cameras(5, 256, 256)
    cfg = config("poly1", api.CullingMode.OpacityAware, deg)
    got = gpu.render_views(splats, cams, cfg)
    for cam, (fb, ctr) in zip(cams, got):
        rgb, tr, ctr_ref = reference.render(splats, cam.to_struct(), cfg.to_struct())
        assert ctr.as_dict() == ctr_ref
        assert max(np.abs(fb.rgb - rgb).max(), np.abs(fb.transmittance - tr).max()) <= 1e-5


def test_views_reject_mixed_sizes(gpu):
    splats, deg = scene("g", 1, 1000)
    cams = [api.orbit_cameras(2, 64, 64)[0], api.orbit_cameras(2, 64, 32)[1]]
    with pytest.raises(api.InvalidArgument):
        gpu.render_views(splats, cams, config("poly1", api.CullingMode.OpacityAware, deg))
