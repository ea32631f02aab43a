"""Pins the parity oracle (CPU, no GPU).

1. The C restatement (oracle/ps_oracle.c) equals the UNMODIFIED reference
   (oracle/_ref, built from /root/reference) bit for bit: images, counters,
   prepared lists and per-tile lists, on the reference's own test scenes.
2. The reference's known-answer tests for this path hold for both
   (test_raster.cpp, test_projection.cpp, test_kernel.cpp, acceptance.cpp), and
   the C1 counters match the survey's probe of the reference.
3. Both agree with the committed golden fixtures (tests/golden/make_golden.py).
"""
import math
import os

import numpy as np
import pytest

from paper_2603_18707_b200 import abi
from tests.helpers import CELLS, NOMINAL_POLY1

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def _kernel(ref, name):
    from paper_2603_18707_b200 import api
    if name == "exp":
        return abi.kernel_struct(abi.PS_KERNEL_EXPONENTIAL)
    if name == "nominal":
        return ref.make_polynomial_kernel(abi.PS_KERNEL_POLY_RELU, NOMINAL_POLY1)
    if name == "poly2p":
        return ref.make_polynomial_kernel(abi.PS_KERNEL_POLY_PIECEWISE, api.FITTED["poly2"])
    return ref.make_polynomial_kernel(abi.PS_KERNEL_POLY_RELU, api.FITTED[name])


def _cfg(ref, kname, mode, sh=3, **kw):
    c = abi.default_config()
    c.kernel = _kernel(ref, kname)
    c.culling_mode = int(mode)
    c.sh_degree = sh
    for k, v in kw.items():
        setattr(c, k, v)
    return c


SCENES = [("grid", 0, 1, (3, 96, 80, 1)), ("sky", 2, 5, (3, 96, 80, 1)), ("random", 1, 3, (1, 256, 192, 0))]


@pytest.mark.parametrize("sname,kind,seed,camspec", SCENES, ids=[s[0] for s in SCENES])
@pytest.mark.parametrize("label,kname,mode", CELLS, ids=[c[0] for c in CELLS])
def test_restatement_matches_reference(reference, restatement, sname, kind, seed, camspec, label, kname, mode):
    splats, deg = reference.synth_scene(kind, seed)
    cnt, w, h, i = camspec
    cam = reference.orbit_cameras(cnt, w, h)[i]
    cfg = _cfg(reference, kname, mode, deg)
    a = reference.render(splats, cam, cfg)
    b = restatement.render(splats, cam, cfg)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2] == b[2]
    pa, pb = reference.prepare(splats, cam, cfg), restatement.prepare(splats, cam, cfg)
    for f in ("index", "depth", "mean2d", "conic", "cov_aa", "opacity_eff", "color", "radius_sigma", "quadric_root"):
        assert np.array_equal(getattr(pa, f), getattr(pb, f)), f
    ta, tb = reference.tile_lists(splats, cam, cfg), restatement.tile_lists(splats, cam, cfg)
    assert np.array_equal(ta[0], tb[0]) and np.array_equal(ta[1], tb[1])
    assert reference.count_pairs(splats, cam, cfg) == restatement.count_pairs(splats, cam, cfg)


def test_serial_renderers_agree(reference, restatement):
    """reference::render_serial (reference.cpp:8-59) in both, and == render (test_raster.cpp:208-229)."""
    splats, _ = reference.synth_scene(1, 3)
    splats = splats[:300]
    cam = reference.orbit_cameras(1, 64, 48)[0]
    for kname, mode in (("exp", 0), ("nominal", 1), ("nominal", 2)):
        cfg = _cfg(reference, kname, mode, 3)
        ra = reference.render_serial(splats, cam, cfg)
        rb = restatement.render_serial(splats, cam, cfg)
        assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
        rr = reference.render(splats, cam, cfg)
        assert np.array_equal(ra[0], rr[0]) and np.array_equal(ra[1], rr[1])


# ---------------------------------------------------------------- reference KATs
@pytest.fixture(params=["reference", "restatement"])
def impl(request, reference, restatement):
    return reference if request.param == "reference" else restatement


def test_tile_rect_kats(reference):
    """test_raster.cpp:50-70"""
    assert reference.tile_rect(24.0, 24.0, [1, 0, 1], 2.094, 16, 320, 320) == (1, 1, 1, 1)
    r = reference.tile_rect(160.0, 160.0, [100, 0, 1], 3.0, 16, 320, 320)
    hx, hy = 30.0, 3.0
    assert r == (math.floor((160 - hx) / 16), math.floor((160 - hy) / 16), math.floor((160 + hx) / 16),
                 math.floor((160 + hy) / 16))
    assert reference.tile_rect(5000.0, 5000.0, [1, 0, 1], 2.0, 16, 320, 320) is None


def test_empty_scene_is_background(impl, reference):
    """test_raster.cpp:124-132"""
    cam = reference.orbit_cameras(1, 64, 48)[0]
    rgb, tr, ctr = impl.render(np.zeros((0, abi.SPLAT3D_DOUBLES)), cam, _cfg(reference, "exp", 0))
    assert np.all(tr == 1.0) and np.all(rgb == 0.0)
    assert ctr["splats_submitted"] == 0 and ctr["tile_pairs_coarse"] == 0 and ctr["kernel_evaluations"] == 0


def _single_splat(scale=0.05, opacity=1.0, color=1.0):
    s = np.zeros(abi.SPLAT3D_DOUBLES)
    s[3:6] = scale
    s[6] = 1.0
    s[10] = opacity
    s[11:14] = (color - 0.5) / 0.28209479177387814
    return s[None, :]


def _cam(w, h, f, c, tz=1.0):
    cam = abi.ps_camera()
    cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy = w, h, f, f, c, c
    for k in range(9):
        cam.rotation[k] = 1.0 if k in (0, 4, 8) else 0.0
    cam.translation[2] = tz
    return cam


def test_single_splat_centre_pixel(impl, reference):
    """test_raster.cpp:134-160: centre pixel = opacity_eff to 1e-12."""
    s = _single_splat(0.05, 1.0, 1.0)
    cam = _cam(65, 65, 60.0, 32.5)
    rgb, tr, ctr = impl.render(s, cam, _cfg(reference, "exp", 0))
    o = impl.project_splat(s[0], cam, 0.3, 3)[9]
    assert abs(rgb[32, 32, 0] - o) <= 1e-12 * o
    assert abs(tr[32, 32] - (1 - o)) <= 1e-12
    assert 0 < ctr["fragments_blended"] <= ctr["kernel_evaluations"]


def test_one_small_splat_one_pair(impl, reference):
    """test_raster.cpp:162-179"""
    s = _single_splat(0.01, 0.9)
    cam = _cam(64, 64, 50.0, 24.0)
    assert impl.count_pairs(s, cam, _cfg(reference, "nominal", 2))["tile_pairs_after_tight_test"] == 1


def test_culling_safety_and_pair_order(impl, reference):
    """test_raster.cpp:231-263: opacity-aware == StopThePop image for poly1; oa <= zero <= stp pairs."""
    grid, _ = reference.synth_scene(0, 1)
    cam = reference.orbit_cameras(1, 128, 96)[0]
    a = impl.render(grid, cam, _cfg(reference, "nominal", 2, 0))
    b = impl.render(grid, cam, _cfg(reference, "nominal", 0, 0))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2]["tile_pairs_after_tight_test"] <= b[2]["tile_pairs_after_tight_test"]
    assert a[2]["fragments_blended"] == b[2]["fragments_blended"]
    rnd, _ = reference.synth_scene(1, 3)
    cam = reference.orbit_cameras(1, 256, 192)[0]
    pairs = [impl.count_pairs(rnd, cam, _cfg(reference, "nominal", m))["tile_pairs_after_tight_test"]
             for m in (2, 1, 0)]
    assert pairs[0] <= pairs[1] <= pairs[2]


def test_projection_kats(impl):
    """test_projection.cpp:69-102"""
    cam = _cam(100, 100, 1.0, 0.0, tz=0.0)
    s = np.zeros(abi.SPLAT3D_DOUBLES)
    s[2] = 1.0
    s[3:6] = 1.0
    s[6] = 1.0
    s[10] = 1.0
    p = impl.project_splat(s, cam, 0.0, 3)
    assert np.allclose(p[5:8], [1.0, 0.0, 1.0]) and abs(p[8] - 1.0) < 1e-12 and abs(p[9] - 1.0) < 1e-12
    p = impl.project_splat(s, cam, 0.3, 3)
    assert np.allclose(p[5:8], [1.3, 0.0, 1.3]) and abs(p[9] - math.sqrt(1 / 1.69)) < 1e-12
    for z, vis in ((0.1, False), (0.2, False), (0.21, True)):
        s[2] = z
        assert (impl.project_splat(s, cam, 0.3, 3) is not None) == vis


def test_culling_radius_kats(impl, reference):
    """test_kernel.cpp:182-208"""
    e = abi.kernel_struct(abi.PS_KERNEL_EXPONENTIAL)
    r, q, _ = impl.culling_radius(e, 1.0, 1 / 255)
    assert abs(r - 3.3291) < 1e-4 * 3.3291 and abs(q - r * r) < 1e-9
    p1 = _kernel(reference, "nominal")
    z1 = impl.culling_radius(p1, 1.0, 0.0)
    z2 = impl.culling_radius(p1, 0.123, 0.0)
    assert z1[0] == z2[0] and not z1[2] and abs(z1[0] - math.sqrt(4.392)) < 1e-4 * z1[0]
    t = impl.culling_radius(p1, 1.0, 1 / 255)
    assert abs(t[0] - 2.0904) < 1e-4 * 2.0904 and t[2]
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as ei:
        impl.culling_radius(e, 0.5, 0.0)
    assert ei.value.status == abi.PS_EPSILON_ZERO_UNBOUNDED
    for k, o in ((e, 1 / 300), (p1, 0.004)):
        with pytest.raises(OracleError) as ei:
            impl.culling_radius(k, o, 1 / 255)
        assert ei.value.status == abi.PS_FULLY_CULLED


def test_c1_counters_match_survey_probe(impl, reference):
    """SURVEY §8c / BASELINE.md §5: C1 = G(10k, seed 1), 256x256, poly1/opacity."""
    from paper_2603_18707_b200 import api
    splats, deg = api.synthetic_splat3d(3, 1, 10000)
    cam = reference.orbit_cameras(1, 256, 256)[0]
    c = impl.count_pairs(splats, cam, _cfg(reference, "poly1", 2, deg))
    assert c["tile_pairs_after_tight_test"] == 24725
    _, _, ctr = impl.render(splats, cam, _cfg(reference, "poly1", 2, deg))
    assert ctr["kernel_evaluations"] == 5628075 and ctr["fragments_blended"] == 775924


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden fixtures not generated")
def test_golden_fixtures(restatement):
    g = np.load(GOLDEN)
    for key in sorted(k[:-4] for k in g.files if k.endswith("_rgb")):
        splats = g[key + "_splats"]
        cam = abi.ps_camera.from_buffer_copy(g[key + "_cam"].tobytes())
        cfg = abi.ps_config.from_buffer_copy(g[key + "_cfg"].tobytes())
        rgb, tr, ctr = restatement.render(splats, cam, cfg)
        assert np.array_equal(rgb, g[key + "_rgb"]) and np.array_equal(tr, g[key + "_t"]), key
        assert [ctr[k] for k in sorted(ctr)] == list(g[key + "_ctr"]), key
        off, idx, _ = restatement.tile_lists(splats, cam, cfg)
        assert np.array_equal(off, g[key + "_off"]) and np.array_equal(idx, g[key + "_idx"]), key


@pytest.mark.parametrize("skewed", [False, True], ids=["g", "skewed"])
def test_reference_side_generator_matches_product(reference, skewed):
    """G(n, seed) generated inside the reference library (the bench's reference
    arm uses it, so that arm maps no product code) is bit-identical to the
    product's synth.cpp generator."""
    from paper_2603_18707_b200 import api
    a, _ = reference.synth_g(5000, 11, skewed)
    b, _ = api.synthetic_splat3d(4 if skewed else 3, 11, 5000)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    cams_r = reference.orbit_cameras(8, 1920, 1080)
    cams_p = api.orbit_cameras(8, 1920, 1080)
    for cr, cp in zip(cams_r, cams_p):
        s = cp.to_struct()
        assert list(cr.rotation) == list(s.rotation) and list(cr.translation) == list(s.translation)
        assert (cr.fx, cr.fy, cr.cx, cr.cy) == (s.fx, s.fy, s.cx, s.cy)
