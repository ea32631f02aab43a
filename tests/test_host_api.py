"""Host-side product logic (CPU, no GPU): the exact fp64 kernel math the device
preprocess uses (compiled for the host from the same source) against the
reference library, the synthetic-input generator, config/camera validation and
the no-fallback guarantee."""
import ctypes as C
import math

import numpy as np
import pytest

from paper_2603_18707_b200 import abi, api
from tests.helpers import NOMINAL_POLY1


def test_make_polynomial_kernel_bitwise(reference):
    for kind, coeffs in ((abi.PS_KERNEL_POLY_RELU, NOMINAL_POLY1), (abi.PS_KERNEL_POLY_RELU, api.FITTED["poly1"]),
                         (abi.PS_KERNEL_POLY_RELU, api.FITTED["poly2"]),
                         (abi.PS_KERNEL_POLY_PIECEWISE, api.FITTED["poly2"]),
                         (abi.PS_KERNEL_POLY_RELU, api.FITTED["poly3"])):
        got = api.make_polynomial_kernel(api.KernelKind(kind), coeffs)
        ref = reference.make_polynomial_kernel(kind, coeffs)
        assert got.first_root == ref.first_root
        assert got.order == ref.order


def test_make_polynomial_kernel_errors():
    """kernel.cpp:141-160 validation"""
    with pytest.raises(api.InvalidArgument):
        api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, [0.5, 0.1])   # order 1 must decay
    with pytest.raises(api.InvalidArgument):
        api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, [-0.5, -0.1])  # positive at 0
    with pytest.raises(api.InvalidArgument):
        api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, [1.0])         # order 0
    with pytest.raises(api.NoPositiveRoot):
        api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, [1.0, 0.0, 1.0])


def test_first_positive_root_vs_reference(reference):
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = rng.integers(2, 5)
        c = rng.uniform(-1, 1, n)
        c[0] = abs(c[0]) + 0.05
        try:
            want = reference.first_positive_root(c)
        except Exception as e:  # noqa: BLE001
            with pytest.raises(api.Error):
                api.first_positive_root(c)
            continue
        got = api.first_positive_root(c)
        # linear/quadratic are arithmetic-only: bitwise; cubic uses cbrt/acos/cos
        if n <= 3:
            assert got == want
        else:
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want))


def test_culling_radius_vs_reference(reference):
    """kernel.cpp:335-358 for the fitted kernels over random (opacity, epsilon)."""
    rng = np.random.default_rng(7)
    kernels = [api.fitted_kernel(n) for n in ("poly1", "poly2", "poly3")] + [api.make_exponential_kernel()]
    for t in range(2000):
        k = kernels[t % 4]
        o = float(rng.uniform(0.02, 1.0))
        eps = float(rng.uniform(1e-4, 0.5))
        try:
            want = reference.culling_radius(k.to_struct(), o, eps)
        except Exception as e:  # noqa: BLE001
            with pytest.raises((api.Error, api.InvalidArgument)):
                api.culling_radius(k, o, eps)
            continue
        got = api.culling_radius(k, o, eps)
        if k.kind == api.KernelKind.PolynomialRelu and k.order <= 2:
            assert (got.radius_sigma, got.quadric_root) == want[:2]
        else:  # log (exp) and cbrt/acos/cos (cubic) come from libm
            assert abs(got.quadric_root - want[1]) <= 1e-13 * want[1]
        assert got.opacity_aware == want[2]


def test_eval_kernel_vs_reference(reference):
    for k in (api.fitted_kernel("poly1"), api.fitted_kernel("poly2p"), api.fitted_kernel("poly3"),
              api.make_exponential_kernel()):
        for x in np.linspace(0.0, 12.0, 97):
            assert api.eval_kernel(k, float(x)) == pytest.approx(reference.eval_kernel(k.to_struct(), float(x)),
                                                                 rel=1e-15, abs=1e-300)


def test_validation_matches_reference(reference):
    """raster.cpp:13-23, projection.cpp:10-22"""
    good = api.RasterConfig(kernel=api.fitted_kernel("poly1"), culling_mode=api.CullingMode.ZeroCrossing)
    good.validate()
    bad = [api.RasterConfig(tile_size=0), api.RasterConfig(epsilon=0.0), api.RasterConfig(epsilon=1.0),
           api.RasterConfig(transmittance_floor=1.0), api.RasterConfig(v_dilation=-1.0),
           api.RasterConfig(thread_count=-1), api.RasterConfig(culling_mode=api.CullingMode.ZeroCrossing)]
    for cfg in bad:
        with pytest.raises(api.InvalidArgument):
            cfg.validate()
        from oracle.oracle import OracleError
        with pytest.raises(OracleError):
            reference.validate_config(cfg.to_struct())
    cam = api.orbit_cameras(1, 64, 48)[0]
    cam.validate()
    cam2 = api.Camera(**{**cam.__dict__, "rotation": cam.rotation * 1.1})
    with pytest.raises(api.NonOrthonormalRotation):
        cam2.validate()
    cam3 = api.Camera(**{**cam.__dict__, "rotation": -cam.rotation})
    with pytest.raises(api.NonOrthonormalRotation):
        cam3.validate()
    with pytest.raises(api.InvalidArgument):
        api.Camera(**{**cam.__dict__, "width": 0}).validate()


@pytest.mark.parametrize("kind,seed", [(0, 1), (1, 3), (2, 5), (1, 11)])
def test_synthetic_scene_matches_reference(reference, kind, seed):
    """scene_io.cpp:304-402: identical Splat3D arrays."""
    a, da = api.synthetic_splat3d(kind, seed)
    b, db = reference.synth_scene(kind, seed)
    assert da == db and np.array_equal(a, b)


def test_parametric_scene_extends_reference():
    """G(5000, seed) is the reference's random scene (k = (5000/n)^(1/3) = 1)."""
    g, _ = api.synthetic_splat3d(3, 3, 5000)
    r, _ = api.synthetic_splat3d(1, 3)
    assert np.array_equal(g, r)
    s = api.Scene.synthetic("g", 2, 20000)
    assert len(s) == 20000 and s.sh.shape == (20000, 16, 3)
    k = (5000 / 20000) ** (1 / 3)
    assert s.scales.min() >= 0.008 * k * (1 - 1e-12) and s.scales.max() <= 0.045 * k * (1 + 1e-12)
    sk = api.Scene.synthetic("skewed", 3, 20000)
    assert sk.opacities.min() >= 0.005 and np.median(sk.opacities) < 0.2


@pytest.mark.parametrize("args", [(1, 64, 48), (3, 96, 80), (256, 1920, 1080)])
def test_orbit_cameras_match_reference(reference, args):
    for a, b in zip(api.orbit_cameras(*args), reference.orbit_cameras(*args)):
        sa = a.to_struct()
        assert bytes(sa) == bytes(b)


def test_no_cpu_fallback_without_gpu():
    """The render path must fail loudly (never fall back to CPU) without a B200."""
    if api.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(api.DeviceError, match="no CUDA device"):
        api.Rasterizer(0)


def test_default_config_matches_reference_defaults():
    c = api.lib().ps_default_config()
    d = abi.default_config()
    assert bytes(c) == bytes(d)
    assert c.tile_size == 16 and abs(c.epsilon - 1 / 255) == 0 and c.transmittance_floor == 1e-4


def test_csv_rows_match_reference_format():
    """metrics.cpp csv_header / csv_row / fmt17 (%.17g, inf spelled out)."""
    ctr_a = api.PerfCounters(**{k: 0 for k in api.PerfCounters.__dataclass_fields__})
    ctr_b = api.PerfCounters(**{k: 0 for k in api.PerfCounters.__dataclass_fields__})
    ctr_a.tile_pairs_after_tight_test, ctr_b.tile_pairs_after_tight_test = 24725, 20000
    r = api.CompareReport(api.ImageMetrics(math.inf, 0.1, 1.0 / 3.0), ctr_a, ctr_b, 20000 / 24725)
    assert api.csv_header() == "label_a,label_b,psnr_db,ssim,max_abs_diff,pairs_a,pairs_b,pair_ratio\n"
    row = api.csv_row("exp/stp", "poly1/opacity", r)
    assert row == ("exp/stp,poly1/opacity,inf,0.10000000000000001,0.33333333333333331,24725,20000,"
                   "0.80889787664307378\n")
    assert float(row.split(",")[4]) == 1.0 / 3.0  # round-trips exactly


def test_reference_ssim_of_identical_images(reference):
    rgb = np.random.default_rng(0).uniform(0, 1, (16, 20, 3))
    t = np.zeros((16, 20))
    p, m, s = reference.compare_images(rgb, t, rgb, t, with_ssim=True)
    assert p == math.inf and m == 0.0 and s == pytest.approx(1.0, abs=1e-12)
