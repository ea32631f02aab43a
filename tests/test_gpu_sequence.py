"""One context over a sequence of frames whose sizes change, as a viewer or a
training loop would drive it. Frames after the first run speculatively (no
mid-frame host sync, dependent launches, heavy-first tile order); the sequence
makes them outgrow the previous frame's pair buffers (sized re-run), meet a
bucket longer than the previous frame announced (re-run), an all-equal-depth
bucket the prologue sort cannot pad (presorted re-run), and change the tile grid
(buffers and tile order rebuilt) before shrinking again. Every frame against the
reference: counters identical, images within 1e-5."""
import pytest

from paper_2603_18707_b200 import api
from tests.helpers import camera, config, crowded_scene, max_abs, scene

pytestmark = pytest.mark.gpu

IMAGE_TOL = 1e-5

# (kind, seed, n, width, height) or ("crowded", n, seed, same_depth)
SEQUENCE = [
    ("g", 1, 2000, 128, 96),
    ("g", 1, 10000, 256, 256),   # more pairs than the first frame's buffers
    ("crowded", 1500, 17, False),  # a bucket past the prologue sort, unannounced
    ("g", 2, 50000, 640, 360),   # a larger tile grid
    ("g", 1, 2000, 128, 96),
    ("crowded", 1300, 16, True),   # equal depths: the presorted re-run
    ("g", 2, 50000, 640, 360),
    ("g", 1, 10000, 256, 256),
]


def _frame(item):
    if item[0] == "crowded":
        _, n, seed, same = item
        return crowded_scene(n, seed, same)
    kind, seed, n, w, h = item
    splats, deg = scene(kind, seed, n)
    return splats, deg, camera(1, w, h, 0)


@pytest.mark.parametrize("kname,mode", [("poly1", api.CullingMode.OpacityAware), ("exp", api.CullingMode.StopThePop)])
def test_changing_frame_sequence(reference, kname, mode):
    with api.Rasterizer(0) as r:
        for step, item in enumerate(SEQUENCE + SEQUENCE[::-1]):
            splats, deg, cam = _frame(item)
            cfg = config(kname, mode, deg)
            rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
            fb, ctr = r.render(splats, cam, cfg)
            assert ctr.as_dict() == ctr_r, (step, item)
            assert max_abs(fb.rgb, rgb_r) <= IMAGE_TOL, (step, item)
            assert max_abs(fb.transmittance, t_r) <= IMAGE_TOL, (step, item)


def test_query_modes_interleaved_with_renders(reference):
    """A context alternates renders (speculative after the first; each leaves the
    counters and per-tile counts zeroed for the next frame) with pair counts,
    tile lists, prepare_splats and view batches on different image sizes: every
    result against the reference."""
    splats, deg = scene("g", 1, 10000)
    cfg = config("poly1", api.CullingMode.OpacityAware, deg)
    big, small = camera(1, 256, 256, 0), camera(1, 96, 64, 0)

    def check_render(r, cam):
        rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
        fb, ctr = r.render(splats, cam, cfg)
        assert ctr.as_dict() == ctr_r
        assert max_abs(fb.rgb, rgb_r) <= IMAGE_TOL and max_abs(fb.transmittance, t_r) <= IMAGE_TOL

    with api.Rasterizer(0) as r:
        for cam in (big, big, small, big):
            check_render(r, cam)
            c = r.count_pairs(splats, cam, cfg).as_dict()
            c_r = reference.count_pairs(splats, cam.to_struct(), cfg.to_struct())
            assert c["tile_pairs_after_tight_test"] == c_r["tile_pairs_after_tight_test"]
            assert c["tile_pairs_coarse"] == c_r["tile_pairs_coarse"]
            check_render(r, cam)
            off, idx, _ = r.tile_lists(splats, cam, cfg)
            r_off, r_idx, _ = reference.tile_lists(splats, cam.to_struct(), cfg.to_struct())
            assert (off == r_off).all() and (idx == r_idx).all()
            check_render(r, cam)
            got = r.prepare_splats(splats, cam, cfg)
            ref = reference.prepare(splats, cam.to_struct(), cfg.to_struct())
            assert (got.index == ref.index).all() and (got.depth == ref.depth).all()
            check_render(r, cam)
            cams = api.orbit_cameras(3, cam.width, cam.height)
            for (fb, ctr), cv in zip(r.render_views(splats, cams, cfg), cams):
                rgb_r, t_r, ctr_r = reference.render(splats, cv.to_struct(), cfg.to_struct())
                assert ctr.as_dict() == ctr_r
                assert max_abs(fb.rgb, rgb_r) <= IMAGE_TOL


def test_sort_prefix_adapts_across_frames(reference):
    """The blend's prologue sort prefix is chosen per context from the previous
    frame (context.cu adapt_sort_prefix): low-opacity crowded tiles whose walks
    run past 256 / 512 entries grow it (whole lists), ordinary frames shrink it
    back to 256, and kernel cells with many replayed pixels keep whole lists.
    Every frame of the alternation stays exact against the reference."""
    dense = crowded_scene(1300, 22, False, opacity=(0.04, 0.12))
    plain = (*scene("g", 1, 100000), camera(1, 256, 256, 0))  # lists of up to ~2,400 entries
    seq = [(plain, "poly1", api.CullingMode.OpacityAware), (dense, "poly1", api.CullingMode.OpacityAware),
           (dense, "exp", api.CullingMode.StopThePop), (plain, "poly1", api.CullingMode.OpacityAware),
           (plain, "exp", api.CullingMode.StopThePop), (plain, "poly1", api.CullingMode.OpacityAware),
           (dense, "poly1", api.CullingMode.OpacityAware)]
    prefixes = []
    with api.Rasterizer(0) as r:
        for (splats, deg, cam), kname, mode in seq:
            cfg = config(kname, mode, deg)
            rgb_r, t_r, ctr_r = reference.render(splats, cam.to_struct(), cfg.to_struct())
            for counters in (True, False):
                fb, ctr = r.render(splats, cam, cfg, counters=counters)
                if counters:
                    assert ctr.as_dict() == ctr_r
                assert max_abs(fb.rgb, rgb_r) <= IMAGE_TOL
                assert max_abs(fb.transmittance, t_r) <= IMAGE_TOL
                prefixes.append(r.stats()["sort_prefix"])
    # the crowded low-opacity tile (~650 entries, never terminating) outgrows
    # the smallest prefix, so the state did change along the sequence
    assert max(prefixes) > 256 and len(set(prefixes)) > 1, prefixes
