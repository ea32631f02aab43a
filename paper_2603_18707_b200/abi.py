"""ctypes mirror of the C ABI in include/polysplat_b200.h (structs, enums, status codes).

Pure data definitions: importing this module loads no native code. The structs
mirror the reference's value types (citations relative to /root/reference/proj):
ps_kernel <- KernelSpec (include/polysplat/kernel.hpp:19-26), ps_config <-
RasterConfig (raster.hpp:19-35), ps_camera <- Camera (projection.hpp:22-31),
ps_counters <- PerfCounters (raster.hpp:37-54).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

SPLAT3D_DOUBLES = 59  # sizeof(polysplat::Splat3D) / 8 (projection.hpp:13-19)
SH_COEFFS = 16

# ps_status
PS_OK = 0
PS_INVALID_ARGUMENT = 1
PS_NON_ORTHONORMAL_ROTATION = 2
PS_DEGENERATE_COVARIANCE = 3
PS_NO_POSITIVE_ROOT = 4
PS_EPSILON_ZERO_UNBOUNDED = 5
PS_FULLY_CULLED = 6
PS_ERROR = 7
PS_CUDA_ERROR = 8
PS_OUT_OF_MEMORY = 9
PS_IO_ERROR, PS_MALFORMED_HEADER, PS_UNSUPPORTED_FORMAT, PS_MISSING_PROPERTY, PS_TRUNCATED_DATA = 10, 11, 12, 13, 14

# KernelKind (kernel.hpp:12-17)
PS_KERNEL_EXPONENTIAL = 0
PS_KERNEL_POLY_RELU = 1
PS_KERNEL_POLY_PIECEWISE = 2

# CullingMode (raster.hpp:13-17)
PS_CULL_STOP_THE_POP = 0
PS_CULL_ZERO_CROSSING = 1
PS_CULL_OPACITY_AWARE = 2

PS_MEM_HOST = 0
PS_MEM_DEVICE = 1

STAGES = ("preprocess", "tile_scan", "host_sync", "duplicate", "tile_sort", "blend", "replay")


class ps_kernel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("order", C.c_int32),
        ("coeffs", C.c_double * 4),
        ("first_root", C.c_double),
    ]


class ps_config(C.Structure):
    _fields_ = [
        ("tile_size", C.c_int32),
        ("culling_mode", C.c_int32),
        ("epsilon", C.c_double),
        ("transmittance_floor", C.c_double),
        ("kernel", ps_kernel),
        ("has_culling_kernel", C.c_int32),
        ("sh_degree", C.c_int32),
        ("culling_kernel", ps_kernel),
        ("v_dilation", C.c_double),
        ("clamp_before_blend", C.c_int32),
        ("thread_count", C.c_int32),
    ]


class ps_camera(C.Structure):
    _fields_ = [
        ("id", C.c_int32),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("reserved", C.c_int32),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("rotation", C.c_double * 9),
        ("translation", C.c_double * 3),
    ]


class ps_counters(C.Structure):
    _fields_ = [
        ("splats_submitted", C.c_uint64),
        ("splats_frustum_culled", C.c_uint64),
        ("tile_pairs_coarse", C.c_uint64),
        ("tile_pairs_after_tight_test", C.c_uint64),
        ("kernel_evaluations", C.c_uint64),
        ("fragments_blended", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class ps_image_metrics(C.Structure):
    """metrics.hpp:18-30 results (ps_image_metrics_compute)."""
    _fields_ = [
        ("psnr_db", C.c_double),
        ("ssim", C.c_double),
        ("max_abs_diff", C.c_double),
        ("ssim_valid", C.c_int32),
        ("sort_prefix", C.c_int32),
    ]


class ps_compare_report(C.Structure):
    """CompareReport (metrics.hpp:32-38)."""
    _fields_ = [
        ("metrics", ps_image_metrics),
        ("counters_a", ps_counters),
        ("counters_b", ps_counters),
        ("pair_ratio", C.c_double),
    ]


PS_DTYPE_F32, PS_DTYPE_F64 = 0, 1


class ps_stats(C.Structure):
    _fields_ = [
        ("visible", C.c_uint64),
        ("pairs", C.c_uint64),
        ("replay_pixels", C.c_uint64),
        ("exact_alpha_evals", C.c_uint64),
        ("stage_ms", C.c_float * 7),
        ("kernel_launches", C.c_int32),
        ("sort_prefix", C.c_int32),
    ]


class ps_prepared(C.Structure):
    _fields_ = [
        ("index", C.POINTER(C.c_uint32)),
        ("depth", C.POINTER(C.c_double)),
        ("mean2d", C.POINTER(C.c_double)),
        ("conic", C.POINTER(C.c_double)),
        ("cov_aa", C.POINTER(C.c_double)),
        ("opacity_eff", C.POINTER(C.c_double)),
        ("color", C.POINTER(C.c_float)),
        ("radius_sigma", C.POINTER(C.c_double)),
        ("quadric_root", C.POINTER(C.c_double)),
    ]


def dptr(a: np.ndarray | None):
    """double* of a C-contiguous float64 array (or NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def fptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


def u32ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def kernel_struct(kind: int, coeffs=(), first_root: float = float("inf")) -> ps_kernel:
    k = ps_kernel()
    k.kind = kind
    k.order = 0 if kind == PS_KERNEL_EXPONENTIAL else len(coeffs) - 1
    for i, c in enumerate(coeffs):
        k.coeffs[i] = c
    k.first_root = first_root
    return k


def default_config() -> ps_config:
    """RasterConfig{} defaults (raster.hpp:19-35)."""
    c = ps_config()
    c.tile_size = 16
    c.culling_mode = PS_CULL_STOP_THE_POP
    c.epsilon = 1.0 / 255.0
    c.transmittance_floor = 1e-4
    c.kernel = kernel_struct(PS_KERNEL_EXPONENTIAL)
    c.has_culling_kernel = 0
    c.sh_degree = 3
    c.culling_kernel = kernel_struct(PS_KERNEL_EXPONENTIAL)
    c.v_dilation = 0.3
    c.clamp_before_blend = 0
    c.thread_count = 0
    return c
