"""Loads libpolysplat_b200.so (the CUDA rasterizer behind the C ABI) via ctypes.

There is no fallback: if the library is missing, or no sm_100 device is present
when a context is created, calls raise. Build with
``python -m paper_2603_18707_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os

from . import abi

# PS_B200_LIB: alternative build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("PS_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpolysplat_b200.so")

# Every function include/polysplat_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ps_version", "ps_abi_version", "ps_device_count", "ps_ctx_create", "ps_ctx_destroy",
    "ps_last_error", "ps_ctx_set_timing", "ps_last_stats", "ps_ctx_synchronize", "ps_ctx_stream",
    "ps_measure_fp32_peak", "ps_measure_fp64_peak",
    "ps_scene_create_aos", "ps_scene_create_soa", "ps_scene_update_soa", "ps_scene_size",
    "ps_scene_destroy", "ps_render", "ps_render_views", "ps_render_splats", "ps_count_pairs",
    "ps_prepare", "ps_tile_lists", "ps_make_polynomial_kernel", "ps_make_exponential_kernel",
    "ps_first_positive_root", "ps_culling_radius", "ps_eval_kernel", "ps_validate_config",
    "ps_validate_camera", "ps_default_config", "ps_synth_scene", "ps_synth_scene_soa",
    "ps_orbit_cameras", "ps_image_metrics_compute", "ps_compare",
    "ps_ply_info", "ps_ply_load_soa", "ps_ply_load_splat3d", "ps_scene_load_ply",
)

_lib = None


def _declare(L) -> None:
    P = C.POINTER
    vp, dp, fp, i64 = C.c_void_p, P(C.c_double), P(C.c_float), C.c_int64
    cam_p, cfg_p, ctr_p = P(abi.ps_camera), P(abi.ps_config), P(abi.ps_counters)
    sig = {
        "ps_version": (C.c_char_p, []),
        "ps_abi_version": (C.c_int, []),
        "ps_device_count": (C.c_int, []),
        "ps_ctx_create": (C.c_int, [C.c_int, P(vp)]),
        "ps_ctx_destroy": (None, [vp]),
        "ps_last_error": (C.c_char_p, [vp]),
        "ps_ctx_set_timing": (C.c_int, [vp, C.c_int]),
        "ps_last_stats": (C.c_int, [vp, P(abi.ps_stats)]),
        "ps_ctx_synchronize": (C.c_int, [vp]),
        "ps_ctx_stream": (vp, [vp]),
        "ps_measure_fp32_peak": (C.c_int, [vp, dp]),
        "ps_measure_fp64_peak": (C.c_int, [vp, dp]),
        "ps_scene_create_aos": (C.c_int, [vp, dp, i64, P(vp)]),
        "ps_scene_create_soa": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, C.c_int, P(vp)]),
        "ps_scene_update_soa": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int]),
        "ps_scene_size": (i64, [vp]),
        "ps_scene_destroy": (None, [vp]),
        "ps_render": (C.c_int, [vp, vp, cam_p, cfg_p, vp, vp, C.c_int, ctr_p]),
        "ps_render_views": (C.c_int, [vp, vp, cam_p, C.c_int, cfg_p, vp, vp, C.c_int, ctr_p]),
        "ps_render_splats": (C.c_int, [vp, dp, i64, cam_p, cfg_p, dp, dp, ctr_p]),
        "ps_count_pairs": (C.c_int, [vp, vp, cam_p, cfg_p, ctr_p]),
        "ps_prepare": (C.c_int, [vp, vp, cam_p, cfg_p, i64, P(abi.ps_prepared), P(i64), ctr_p]),
        "ps_tile_lists": (C.c_int, [vp, vp, cam_p, cfg_p, i64, P(C.c_uint32), P(C.c_uint32), P(i64), ctr_p]),
        "ps_image_metrics_compute": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, dp,
                                              P(abi.ps_image_metrics)]),
        "ps_compare": (C.c_int, [vp, vp, cam_p, cfg_p, cfg_p, dp, P(abi.ps_compare_report)]),
        "ps_ply_info": (C.c_int, [C.c_char_p, P(i64), P(C.c_int)]),
        "ps_ply_load_soa": (C.c_int, [C.c_char_p, dp, dp, dp, dp, fp, i64, P(i64), P(C.c_int)]),
        "ps_ply_load_splat3d": (C.c_int, [C.c_char_p, dp, i64, P(i64), P(C.c_int)]),
        "ps_scene_load_ply": (C.c_int, [vp, C.c_char_p, P(vp), P(C.c_int)]),
        "ps_make_polynomial_kernel": (C.c_int, [C.c_int, dp, C.c_int, P(abi.ps_kernel)]),
        "ps_make_exponential_kernel": (abi.ps_kernel, []),
        "ps_first_positive_root": (C.c_int, [dp, C.c_int, dp]),
        "ps_culling_radius": (C.c_int, [P(abi.ps_kernel), C.c_double, C.c_double, dp, dp, P(C.c_int)]),
        "ps_eval_kernel": (C.c_double, [P(abi.ps_kernel), C.c_double]),
        "ps_validate_config": (C.c_int, [cfg_p]),
        "ps_validate_camera": (C.c_int, [cam_p]),
        "ps_default_config": (abi.ps_config, []),
        "ps_synth_scene": (C.c_int, [C.c_int, C.c_uint64, i64, dp, i64, P(i64), P(C.c_int)]),
        "ps_synth_scene_soa": (C.c_int, [C.c_int, C.c_uint64, i64, dp, dp, dp, dp, fp]),
        "ps_orbit_cameras": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, cam_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib():
    """The loaded native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2603_18707_b200.build` "
                "(there is no CPU fallback for the render path)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def last_error(ctx=None) -> str:
    msg = lib().ps_last_error(ctx)
    return msg.decode() if msg else ""
