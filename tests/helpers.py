"""Test helpers: configs, scenes and comparison utilities shared by the suites."""
from __future__ import annotations

import numpy as np

from paper_2603_18707_b200 import abi, api

# (label, kernel name, culling mode)
CELLS = [
    ("exp/stp", "exp", api.CullingMode.StopThePop),
    ("poly1/stp", "poly1", api.CullingMode.StopThePop),
    ("poly1/zero", "poly1", api.CullingMode.ZeroCrossing),
    ("poly1/opacity", "poly1", api.CullingMode.OpacityAware),
    ("poly2p/opacity", "poly2p", api.CullingMode.OpacityAware),
    ("poly3/stp", "poly3", api.CullingMode.StopThePop),
    ("poly3/opacity", "poly3", api.CullingMode.OpacityAware),
]

# the reference tests' nominal kernel (test_raster.cpp:18-20)
NOMINAL_POLY1 = (0.773, -0.176)


def kernel(name: str) -> api.KernelSpec:
    if name == "nominal":
        return api.make_polynomial_kernel(api.KernelKind.PolynomialRelu, NOMINAL_POLY1)
    return api.fitted_kernel(name)


def config(kname: str, mode, sh_degree: int = 3, **kw) -> api.RasterConfig:
    cfg = api.RasterConfig(kernel=kernel(kname), culling_mode=mode, sh_degree=sh_degree)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def scene(kind: str, seed: int = 0, n: int = 0):
    """(Splat3D array (n, 59), sh_degree) from the product generator."""
    kinds = {"grid": 0, "random": 1, "sky": 2, "g": 3, "skewed": 4}
    return api.synthetic_splat3d(kinds[kind], seed, n)


def camera(count: int, w: int, h: int, i: int = 0) -> api.Camera:
    return api.orbit_cameras(count, w, h)[i]


def max_abs(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def psnr(rgb_a, t_a, rgb_b, t_b, bg=(1.0, 1.0, 1.0)) -> float:
    """metrics.cpp:13-44 composite + PSNR (peak 1)."""
    ca = np.asarray(rgb_a, np.float64) + np.asarray(t_a, np.float64)[..., None] * np.asarray(bg)
    cb = np.asarray(rgb_b, np.float64) + np.asarray(t_b, np.float64)[..., None] * np.asarray(bg)
    mse = float(np.mean((ca - cb) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)


def ulp_diff(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|ULP distance| between float64 arrays of the same sign."""
    ai = np.asarray(a, np.float64).view(np.int64)
    bi = np.asarray(b, np.float64).view(np.int64)
    return np.abs(ai - bi)
