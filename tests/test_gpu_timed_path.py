"""The instantiation bench.py times, checked against the reference.

bench.py renders through ps_render / ps_render_views with NO counters
(k_blend16<..., COUNT=false>) into DEVICE buffers, on a context whose first
frame was sized and whose later frames are speculative (no mid-frame host
sync). These tests call exactly that: the same C-ABI entry points, counters
NULL, PS_MEM_DEVICE outputs (torch tensors), several frames per context,
against oracle/_ref's polysplat::render (images within 1e-5 max-abs; the
counters of the same frame come from a separate counting render and must equal
the reference's)."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_18707_b200 import abi, api
from paper_2603_18707_b200._native import lib
from tests.helpers import CELLS, camera, config, crowded_scene, max_abs, scene

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _torch():
    import torch
    return torch


def render_device_nocount(gpu, ds, cam, cfg):
    """ps_render(..., PS_MEM_DEVICE, counters=NULL), the bench's call."""
    torch = _torch()
    rgb = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda")
    tr = torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda")
    c, g = cam.to_struct(), cfg.to_struct()
    st = lib().ps_render(gpu.handle, ds.handle, C.byref(c), C.byref(g), rgb.data_ptr(), tr.data_ptr(),
                         abi.PS_MEM_DEVICE, None)
    api._check(st, gpu.handle)
    gpu.synchronize()
    return rgb.cpu().numpy(), tr.cpu().numpy()


def render_views_device_nocount(gpu, ds, cams, cfg):
    torch = _torch()
    n, h, w = len(cams), cams[0].height, cams[0].width
    rgb = torch.empty((n, h, w, 3), dtype=torch.float32, device="cuda")
    tr = torch.empty((n, h, w), dtype=torch.float32, device="cuda")
    cs = (abi.ps_camera * n)(*[c.to_struct() for c in cams])
    g = cfg.to_struct()
    api._check(lib().ps_render_views(gpu.handle, ds.handle, cs, n, C.byref(g), rgb.data_ptr(), tr.data_ptr(),
                                     abi.PS_MEM_DEVICE, None), gpu.handle)
    gpu.synchronize()
    return rgb.cpu().numpy(), tr.cpu().numpy()


@pytest.mark.parametrize("label,kname,mode", CELLS, ids=[c[0] for c in CELLS])
def test_c1_nocount_device_frames(gpu, reference, label, kname, mode):
    """C1 (G(10k, seed 1), 256x256): three frames on one context (sized, then
    speculative), counters NULL, device outputs — the timed instantiation."""
    splats, deg = scene("g", 1, 10000)
    cam = camera(1, 256, 256, 0)
    cfg = config(kname, mode, deg)
    rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
    ds = gpu.upload_splat3d(splats)
    for _ in range(3):
        rgb, tr = render_device_nocount(gpu, ds, cam, cfg)
        assert max_abs(rgb, rgb_r) <= TOL and max_abs(tr, t_r) <= TOL
    # the counting instantiation of the same frame, on the same context
    fb, ctr = gpu.render(ds, cam, cfg)
    assert ctr.as_dict() == ctr_r
    ds.close()


@pytest.mark.parametrize("kind,seed,w,h", [("random", 0, 320, 240), ("grid", 0, 200, 150), ("sky", 3, 256, 192)])
@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop),
                                        ("poly3", api.CullingMode.OpacityAware)])
def test_reference_scenes_nocount(gpu, reference, kind, seed, w, h, kname, mode):
    splats, deg = scene(kind, seed)
    cam = camera(4, w, h, 1)
    cfg = config(kname, mode, deg)
    rgb_r, t_r, _ = reference.render(splats, cam.to_struct(), cfg.to_struct())
    ds = gpu.upload_splat3d(splats)
    for _ in range(2):
        rgb, tr = render_device_nocount(gpu, ds, cam, cfg)
        assert max_abs(rgb, rgb_r) <= TOL and max_abs(tr, t_r) <= TOL
    ds.close()


@pytest.mark.parametrize("n,seed,same", [(1300, 16, True), (3000, 12, False), (10000, 18, True)])
def test_crowded_nocount(gpu, reference, n, seed, same):
    """Long buckets (list-kernel sorts, the prologue's re-run path) through the
    counter-free blend."""
    splats, deg, cam = crowded_scene(n, seed, same)
    cfg = config("poly1", api.CullingMode.OpacityAware, deg)
    rgb_r, t_r, _ = reference.render(splats, cam.to_struct(), cfg.to_struct())
    ds = gpu.upload_splat3d(splats)
    for _ in range(2):
        rgb, tr = render_device_nocount(gpu, ds, cam, cfg)
        assert max_abs(rgb, rgb_r) <= TOL and max_abs(tr, t_r) <= TOL
    ds.close()


def test_sequence_nocount(gpu, reference):
    """A changing frame sequence on one context (cameras and configs alternate,
    so speculation meets pair-count growth and re-runs)."""
    splats, deg = scene("g", 1, 10000)
    cams = api.orbit_cameras(6, 256, 256)
    cfgs = [config("poly1", api.CullingMode.OpacityAware, deg), config("exp", api.CullingMode.StopThePop, deg)]
    ds = gpu.upload_splat3d(splats)
    for k in range(8):
        cam, cfg = cams[k % 6], cfgs[(k // 3) % 2]
        rgb_r, t_r, _ = reference.render(splats, cam.to_struct(), cfg.to_struct())
        rgb, tr = render_device_nocount(gpu, ds, cam, cfg)
        assert max_abs(rgb, rgb_r) <= TOL and max_abs(tr, t_r) <= TOL
    ds.close()


@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop)])
def test_views_nocount_device(gpu, reference, kname, mode):
    """ps_render_views with counters NULL into device buffers (the C4 bench call)."""
    splats, deg = scene("g", 1, 10000)
    cams = api.orbit_cameras(9, 192, 128)
    cfg = config(kname, mode, deg)
    ds = gpu.upload_splat3d(splats)
    rgb, tr = render_views_device_nocount(gpu, ds, cams, cfg)
    for k, cam in enumerate(cams):
        rgb_r, t_r, _ = reference.render(splats, cam.to_struct(), cfg.to_struct())
        assert max_abs(rgb[k], rgb_r) <= TOL and max_abs(tr[k], t_r) <= TOL
    ds.close()


def test_golden_fixtures_nocount(gpu):
    """The committed golden images (tests/golden, generated from oracle/_ref)
    through the counter-free blend into device buffers."""
    import os
    torch = _torch()
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    cases = sorted(k[: -len("_rgb")] for k in gold.files if k.endswith("_rgb"))
    assert len(cases) >= 7
    for case in cases:
        cam = abi.ps_camera.from_buffer_copy(gold[case + "_cam"].tobytes())
        cfg = abi.ps_config.from_buffer_copy(gold[case + "_cfg"].tobytes())
        ds = gpu.upload_splat3d(gold[case + "_splats"])
        rgb = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda")
        tr = torch.empty((cam.height, cam.width), dtype=torch.float32, device="cuda")
        for _ in range(2):
            api._check(lib().ps_render(gpu.handle, ds.handle, C.byref(cam), C.byref(cfg), rgb.data_ptr(),
                                       tr.data_ptr(), abi.PS_MEM_DEVICE, None), gpu.handle)
            gpu.synchronize()
            assert max_abs(rgb.cpu().numpy(), gold[case + "_rgb"]) <= TOL, case
            assert max_abs(tr.cpu().numpy(), gold[case + "_t"]) <= TOL, case
        ds.close()
