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


def crowded_scene(n: int, seed: int, same_depth: bool = False, opacity=(0.3, 0.95)):
    """n small splats crowded into one 16x16 tile (pixels 32-47) of a 64x64 view
    (identity camera rotation, so depth == mean z exactly): per-tile buckets of
    ~n entries exercise the long-bucket sort kernels and the global fallback;
    same_depth puts every splat at z = 5 (all sort keys equal: the tie order by
    splat index and the bitonic path); a low `opacity` range keeps pixels live
    deep into the list (the blend sorts past its ranked prefix)."""
    rng = np.random.default_rng(seed)
    sp = np.zeros((n, 59), dtype=np.float64)
    z = np.full(n, 5.0) if same_depth else rng.uniform(4.0, 6.0, n)
    sp[:, 0] = rng.uniform(0.02, 0.23, n) * z
    sp[:, 1] = rng.uniform(0.02, 0.23, n) * z
    sp[:, 2] = z
    sp[:, 3:6] = rng.uniform(0.004, 0.02, (n, 3))
    q = rng.normal(size=(n, 4))
    sp[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    sp[:, 10] = rng.uniform(opacity[0], opacity[1], n)
    sp[:, 11:14] = rng.uniform(-1.0, 1.0, (n, 3))  # SH DC (degree 0)
    cam = api.Camera(0, 64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(3), np.zeros(3))
    return sp, 0, cam
