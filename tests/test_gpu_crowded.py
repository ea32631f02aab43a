"""GPU parity on crowded tiles (tests/helpers.crowded_scene): buckets longer than
the blend prologue's shared-memory sort (1536), the 512-thread list sort (4096),
the 1024-thread list sort (16384, beyond which the global radix path runs), and
all-equal depths (tie order by splat index, bitonic path; a prologue bucket of
1024-1536 equal depths cannot be padded to 2048 in shared memory, so the frame
is re-run with every bucket presorted). Each scene is rendered twice: the
first frame of a context is sized, the second speculative. Same bar as
test_gpu_parity: bit-exact tile lists and counters, images within 1e-5."""
import numpy as np
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import config, crowded_scene, max_abs

pytestmark = pytest.mark.gpu

CASES = [(700, 11, True), (1300, 16, True), (1500, 17, False), (3000, 12, False), (6000, 13, False),
         (20000, 14, False), (2500, 15, True), (10000, 18, True), (15000, 19, False), (15000, 20, True)]
CELLS = [("poly1/opacity", "poly1", api.CullingMode.OpacityAware), ("exp/stp", "exp", api.CullingMode.StopThePop)]


@pytest.mark.parametrize("n,seed,same", CASES, ids=[f"n{c[0]}{'-eqz' if c[2] else ''}" for c in CASES])
@pytest.mark.parametrize("label,kname,mode", CELLS, ids=[c[0] for c in CELLS])
def test_crowded_tiles(gpu, reference, n, seed, same, label, kname, mode):
    splats, deg, cam = crowded_scene(n, seed, same)
    cfg = config(kname, mode, deg)
    r_off, r_idx, _ = reference.tile_lists(splats, cam.to_struct(), cfg.to_struct())
    g_off, g_idx, _ = gpu.tile_lists(splats, cam, cfg)
    assert int(np.diff(r_off).max()) > 0.9 * n  # one really crowded tile
    assert np.array_equal(g_off, r_off)
    assert np.array_equal(g_idx, r_idx)
    rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
    ds = gpu.upload_splat3d(splats)
    for _ in range(2):
        fb, ctr = gpu.render(ds, cam, cfg)
        assert ctr.as_dict() == ctr_r
        assert max_abs(fb.rgb, rgb_r) <= 1e-5
        assert max_abs(fb.transmittance, t_r) <= 1e-5
    ds.close()


LOW = [(700, 21, False), (1300, 22, False), (1000, 23, True), (1500, 24, False)]


@pytest.mark.parametrize("n,seed,same", LOW, ids=[f"n{c[0]}{'-eqz' if c[2] else ''}" for c in LOW])
@pytest.mark.parametrize("label,kname,mode", CELLS, ids=[c[0] for c in CELLS])
def test_crowded_low_opacity(gpu, reference, n, seed, same, label, kname, mode):
    """Low opacities: pixels stay live past the first kSortPrefix (256) entries
    of the crowded tile's list, so the blend ranks the rest of the bucket
    mid-walk (blend.cu sort_all) — and before the exact replay."""
    splats, deg, cam = crowded_scene(n, seed, same, opacity=(0.04, 0.12))
    cfg = config(kname, mode, deg)
    rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
    assert ctr_r["kernel_evaluations"] > 300 * 256  # pixels walk past the ranked prefix
    ds = gpu.upload_splat3d(splats)
    for counters in (True, False, True):
        fb, ctr = gpu.render(ds, cam, cfg, counters=counters)
        if counters:
            assert ctr.as_dict() == ctr_r
        assert max_abs(fb.rgb, rgb_r) <= 1e-5
        assert max_abs(fb.transmittance, t_r) <= 1e-5
    ds.close()
