"""Reference-shaped host API over the C ABI (include/polysplat_b200.h).

Mirrors the reference's public rasterizer interface (paths relative to
/root/reference/proj): ``render`` / ``count_pairs`` / ``prepare_splats``
(include/polysplat/raster.hpp:103-113), ``KernelSpec`` / ``make_*_kernel`` /
``first_positive_root`` / ``culling_radius`` / ``eval_kernel`` (kernel.hpp:12-104),
``RasterConfig`` / ``CullingMode`` / ``PerfCounters`` / ``Framebuffer``
(raster.hpp:13-64), ``Camera`` (projection.hpp:22-31), the typed errors
(errors.hpp:9-39), and the synthetic scenes / orbit cameras the reference's
tests use (scene_io.hpp:30-40). Same argument meaning and error behaviour:
config/camera problems raise ``InvalidArgument`` (a ``ValueError``, the
std::invalid_argument analogue), data problems raise the ``Error`` subclasses.

Every render runs on the GPU through libpolysplat_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import abi
from ._native import last_error, lib


# ---------------------------------------------------------------- errors (errors.hpp:9-39)
class Error(RuntimeError):
    """polysplat::Error"""


class NoPositiveRoot(Error):
    pass


class FullyCulled(Error):
    pass


class EpsilonZeroUnbounded(Error):
    pass


class DegenerateCovariance(Error):
    pass


class NonOrthonormalRotation(Error):
    pass


class IoError(Error):
    pass


class MalformedHeader(Error):
    pass


class UnsupportedFormat(Error):
    pass


class MissingProperty(Error):
    pass


class TruncatedData(Error):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DeviceError(RuntimeError):
    """CUDA failure / out of memory (no reference analogue)."""


_STATUS = {
    abi.PS_INVALID_ARGUMENT: InvalidArgument,
    abi.PS_NON_ORTHONORMAL_ROTATION: NonOrthonormalRotation,
    abi.PS_DEGENERATE_COVARIANCE: DegenerateCovariance,
    abi.PS_NO_POSITIVE_ROOT: NoPositiveRoot,
    abi.PS_EPSILON_ZERO_UNBOUNDED: EpsilonZeroUnbounded,
    abi.PS_FULLY_CULLED: FullyCulled,
    abi.PS_ERROR: Error,
    abi.PS_CUDA_ERROR: DeviceError,
    abi.PS_OUT_OF_MEMORY: DeviceError,
    abi.PS_IO_ERROR: IoError,
    abi.PS_MALFORMED_HEADER: MalformedHeader,
    abi.PS_UNSUPPORTED_FORMAT: UnsupportedFormat,
    abi.PS_MISSING_PROPERTY: MissingProperty,
    abi.PS_TRUNCATED_DATA: TruncatedData,
}


def _check(status: int, ctx=None) -> None:
    if status != abi.PS_OK:
        raise _STATUS.get(status, Error)(last_error(ctx) or f"status {status}")


# ---------------------------------------------------------------- kernels (kernel.hpp)
class KernelKind(IntEnum):
    Exponential = abi.PS_KERNEL_EXPONENTIAL
    PolynomialRelu = abi.PS_KERNEL_POLY_RELU
    PolynomialPiecewise = abi.PS_KERNEL_POLY_PIECEWISE


@dataclass(frozen=True)
class KernelSpec:
    kind: KernelKind = KernelKind.Exponential
    order: int = 0
    coeffs: tuple = ()
    first_root: float = math.inf

    def is_polynomial(self) -> bool:
        return self.kind != KernelKind.Exponential

    def to_struct(self) -> abi.ps_kernel:
        return abi.kernel_struct(int(self.kind), self.coeffs, self.first_root)

    @staticmethod
    def from_struct(k: abi.ps_kernel) -> "KernelSpec":
        kind = KernelKind(k.kind)
        coeffs = tuple(k.coeffs[i] for i in range(k.order + 1)) if kind != KernelKind.Exponential else ()
        return KernelSpec(kind, int(k.order), coeffs, float(k.first_root))


# Fitted coefficients (reference fit_polynomial with defaults).
FITTED = {
    "poly1": (0.77007333317642512, -0.17527402122331368),
    "poly2": (0.8082182210258585, -0.22859470326756573, 0.014202796808880376),
    "poly3": (0.96130510295806615, -0.40924216692744086, 0.064908288782897464, -0.0036418092719824146),
}


def make_exponential_kernel() -> KernelSpec:
    return KernelSpec()


def make_polynomial_kernel(kind: KernelKind, coeffs: Sequence[float]) -> KernelSpec:
    """kernel.cpp:141-160: validates and caches the first positive root."""
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    k = abi.ps_kernel()
    _check(lib().ps_make_polynomial_kernel(int(kind), abi.dptr(c), len(c), C.byref(k)))
    return KernelSpec.from_struct(k)


def fitted_kernel(name: str) -> KernelSpec:
    """'poly1' | 'poly2p' (piecewise order 2) | 'poly2' (ReLU order 2) | 'poly3' | 'exp'."""
    if name == "exp":
        return make_exponential_kernel()
    if name == "poly2p":
        return make_polynomial_kernel(KernelKind.PolynomialPiecewise, FITTED["poly2"])
    return make_polynomial_kernel(KernelKind.PolynomialRelu, FITTED[name])


def first_positive_root(coeffs: Sequence[float]) -> float:
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = C.c_double(0)
    _check(lib().ps_first_positive_root(abi.dptr(c), len(c), C.byref(out)))
    return out.value


@dataclass(frozen=True)
class CullingBound:
    radius_sigma: float
    quadric_root: float
    opacity_aware: bool


def culling_radius(spec: KernelSpec, opacity: float, epsilon: float) -> CullingBound:
    """kernel.cpp:335-358; raises FullyCulled / EpsilonZeroUnbounded like the reference."""
    k = spec.to_struct()
    r, q, a = C.c_double(0), C.c_double(0), C.c_int(0)
    _check(lib().ps_culling_radius(C.byref(k), opacity, epsilon, C.byref(r), C.byref(q), C.byref(a)))
    return CullingBound(r.value, q.value, bool(a.value))


def try_culling_radius(spec: KernelSpec, opacity: float, epsilon: float) -> Optional[CullingBound]:
    """kernel.cpp:360-369"""
    if spec.kind == KernelKind.Exponential and epsilon == 0.0:
        raise EpsilonZeroUnbounded("exponential kernel has unbounded support at epsilon 0")
    try:
        return culling_radius(spec, opacity, epsilon)
    except FullyCulled:
        return None


def eval_kernel(spec: KernelSpec, x: float) -> float:
    k = spec.to_struct()
    return lib().ps_eval_kernel(C.byref(k), x)


# ---------------------------------------------------------------- config (raster.hpp)
class CullingMode(IntEnum):
    StopThePop = abi.PS_CULL_STOP_THE_POP
    ZeroCrossing = abi.PS_CULL_ZERO_CROSSING
    OpacityAware = abi.PS_CULL_OPACITY_AWARE


@dataclass
class RasterConfig:
    tile_size: int = 16
    epsilon: float = 1.0 / 255.0
    transmittance_floor: float = 1e-4
    culling_mode: CullingMode = CullingMode.StopThePop
    kernel: KernelSpec = field(default_factory=make_exponential_kernel)
    culling_kernel: Optional[KernelSpec] = None
    v_dilation: float = 0.3
    sh_degree: int = 3
    clamp_before_blend: bool = False
    thread_count: int = 0

    def bound_kernel(self) -> KernelSpec:
        return self.culling_kernel if self.culling_kernel is not None else self.kernel

    def to_struct(self) -> abi.ps_config:
        c = abi.ps_config()
        c.tile_size = self.tile_size
        c.culling_mode = int(self.culling_mode)
        c.epsilon = self.epsilon
        c.transmittance_floor = self.transmittance_floor
        c.kernel = self.kernel.to_struct()
        c.has_culling_kernel = 1 if self.culling_kernel is not None else 0
        c.culling_kernel = (self.culling_kernel or make_exponential_kernel()).to_struct()
        c.sh_degree = self.sh_degree
        c.v_dilation = self.v_dilation
        c.clamp_before_blend = 1 if self.clamp_before_blend else 0
        c.thread_count = self.thread_count
        return c

    def validate(self) -> None:
        """raster.cpp:13-23"""
        c = self.to_struct()
        _check(lib().ps_validate_config(C.byref(c)))


@dataclass
class Camera:
    id: int = 0
    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_struct(self) -> abi.ps_camera:
        c = abi.ps_camera()
        c.id, c.width, c.height = self.id, self.width, self.height
        c.fx, c.fy, c.cx, c.cy = self.fx, self.fy, self.cx, self.cy
        r = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        for i in range(9):
            c.rotation[i] = r[i]
        for i in range(3):
            c.translation[i] = t[i]
        return c

    @staticmethod
    def from_struct(c: abi.ps_camera) -> "Camera":
        return Camera(c.id, c.width, c.height, c.fx, c.fy, c.cx, c.cy,
                      np.array(c.rotation[:], dtype=np.float64).reshape(3, 3),
                      np.array(c.translation[:], dtype=np.float64))

    def position(self) -> np.ndarray:
        return -(self.rotation.T @ self.translation)

    def validate(self) -> None:
        """projection.cpp:10-22"""
        c = self.to_struct()
        _check(lib().ps_validate_camera(C.byref(c)))


@dataclass
class PerfCounters:
    splats_submitted: int = 0
    splats_frustum_culled: int = 0
    tile_pairs_coarse: int = 0
    tile_pairs_after_tight_test: int = 0
    kernel_evaluations: int = 0
    fragments_blended: int = 0

    @staticmethod
    def from_struct(c: abi.ps_counters) -> "PerfCounters":
        return PerfCounters(**c.as_dict())

    def as_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class Framebuffer:
    """raster.hpp:56-64 (rgb as (H, W, 3), transmittance as (H, W))."""
    width: int
    height: int
    rgb: np.ndarray
    transmittance: np.ndarray


# ---------------------------------------------------------------- scenes
@dataclass
class Scene:
    """Splats as SoA arrays (Splat3D, projection.hpp:13-19): means (n,3) f64,
    scales (n,3) f64, rotations (n,4) f64 (w,x,y,z), opacities (n,) f64, sh (n,16,3) f32."""
    means: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray
    sh_degree: int = 3

    def __len__(self) -> int:
        return len(self.opacities)

    @staticmethod
    def from_splat3d(arr: np.ndarray, sh_degree: int = 3) -> "Scene":
        a = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1, abi.SPLAT3D_DOUBLES)
        return Scene(np.ascontiguousarray(a[:, 0:3]), np.ascontiguousarray(a[:, 3:6]),
                     np.ascontiguousarray(a[:, 6:10]), np.ascontiguousarray(a[:, 10]),
                     np.ascontiguousarray(a[:, 11:59].reshape(-1, 16, 3).astype(np.float32)), sh_degree)

    @staticmethod
    def synthetic(kind: int | str, seed: int = 0, n: int = 0) -> "Scene":
        """kind: grid | random | sky (reference scenes) | g (parametric G(n, seed)) | skewed (C5)."""
        kinds = {"grid": 0, "random": 1, "sky": 2, "g": 3, "skewed": 4}
        k = kinds[kind] if isinstance(kind, str) else int(kind)
        cnt = C.c_int64(0)
        deg = C.c_int(0)
        _check(lib().ps_synth_scene(k, seed, n, None, 0, C.byref(cnt), C.byref(deg)))
        m = cnt.value
        means, scales = np.zeros((m, 3)), np.zeros((m, 3))
        rots, opac = np.zeros((m, 4)), np.zeros(m)
        sh = np.zeros((m, 16, 3), np.float32)
        _check(lib().ps_synth_scene_soa(k, seed, n, abi.dptr(means), abi.dptr(scales), abi.dptr(rots),
                                        abi.dptr(opac), sh.ctypes.data_as(C.POINTER(C.c_float))))
        return Scene(means, scales, rots, opac, sh, deg.value)


def load_ply(path: str) -> Scene:
    """load_ply (scene_io.cpp:53-199): a 3DGS checkpoint as a Scene (SoA), with
    the reference's activations applied in fp64 (bit-identical fields)."""
    n, deg = C.c_int64(0), C.c_int(0)
    p = str(path).encode()
    _check(lib().ps_ply_info(p, C.byref(n), C.byref(deg)))
    m = n.value
    means, scales = np.zeros((m, 3)), np.zeros((m, 3))
    rots, opac = np.zeros((m, 4)), np.zeros(m)
    sh = np.zeros((m, 16, 3), np.float32)
    _check(lib().ps_ply_load_soa(p, abi.dptr(means), abi.dptr(scales), abi.dptr(rots), abi.dptr(opac),
                                 sh.ctypes.data_as(C.POINTER(C.c_float)), m, C.byref(n), C.byref(deg)))
    return Scene(means, scales, rots, opac, sh, deg.value)


def load_ply_splat3d(path: str):
    """load_ply as the reference's SceneFile: (Splat3D array (n, 59) f64, sh_degree)."""
    n, deg = C.c_int64(0), C.c_int(0)
    p = str(path).encode()
    _check(lib().ps_ply_info(p, C.byref(n), C.byref(deg)))
    out = np.zeros((n.value, abi.SPLAT3D_DOUBLES))
    _check(lib().ps_ply_load_splat3d(p, abi.dptr(out), n.value, C.byref(n), C.byref(deg)))
    return out, deg.value


def synthetic_splat3d(kind: int, seed: int = 0, n: int = 0):
    """The scene as a reference Splat3D array (n, 59) f64 plus its SH degree."""
    cnt = C.c_int64(0)
    deg = C.c_int(0)
    _check(lib().ps_synth_scene(kind, seed, n, None, 0, C.byref(cnt), C.byref(deg)))
    out = np.zeros((cnt.value, abi.SPLAT3D_DOUBLES))
    _check(lib().ps_synth_scene(kind, seed, n, abi.dptr(out), cnt.value, C.byref(cnt), C.byref(deg)))
    return out, deg.value


def orbit_cameras(count: int, width: int, height: int, fov_deg: float = 50.0, radius: float = 2.0,
                  elevation: float = 0.3) -> list[Camera]:
    """scene_io.cpp:415-441"""
    cams = (abi.ps_camera * count)()
    _check(lib().ps_orbit_cameras(count, width, height, fov_deg, radius, elevation, cams))
    return [Camera.from_struct(c) for c in cams]


# ---------------------------------------------------------------- device context
class DeviceScene:
    """A scene resident in HBM (ps_scene); render it from any number of cameras."""

    def __init__(self, ctx: "Rasterizer", handle, n: int):
        self._ctx = ctx
        self.handle = handle
        self.n = n

    def close(self) -> None:
        if self.handle:
            lib().ps_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Prepared:
    """prepare_splats output (raster.hpp:103-104) as SoA arrays in depth order."""
    index: np.ndarray
    depth: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    cov_aa: np.ndarray
    opacity_eff: np.ndarray
    color: np.ndarray
    radius_sigma: np.ndarray
    quadric_root: np.ndarray
    counters: PerfCounters


class Rasterizer:
    """One CUDA device context (ps_ctx): stream, scratch, events."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().ps_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().ps_ctx_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- scenes
    def upload(self, scene: Scene) -> DeviceScene:
        h = C.c_void_p()
        n = len(scene)
        arrs = [np.ascontiguousarray(scene.means, np.float64), np.ascontiguousarray(scene.scales, np.float64),
                np.ascontiguousarray(scene.rotations, np.float64), np.ascontiguousarray(scene.opacities, np.float64),
                np.ascontiguousarray(scene.sh, np.float32)]
        _check(lib().ps_scene_create_soa(self.handle, *[a.ctypes.data for a in arrs], n, abi.PS_MEM_HOST,
                                         C.byref(h)), self.handle)
        return DeviceScene(self, h, n)

    def upload_ply(self, path: str) -> DeviceScene:
        """ps_scene_load_ply: a 3DGS checkpoint straight into a device scene."""
        h, deg = C.c_void_p(), C.c_int(0)
        _check(lib().ps_scene_load_ply(self.handle, str(path).encode(), C.byref(h), C.byref(deg)), self.handle)
        ds = DeviceScene(self, h, lib().ps_scene_size(h))
        ds.sh_degree = deg.value
        return ds

    def upload_splat3d(self, splats: np.ndarray) -> DeviceScene:
        a = np.ascontiguousarray(splats, dtype=np.float64)
        h = C.c_void_p()
        _check(lib().ps_scene_create_aos(self.handle, abi.dptr(a), len(a), C.byref(h)), self.handle)
        return DeviceScene(self, h, len(a))

    def _scene(self, scene) -> tuple[DeviceScene, bool]:
        if isinstance(scene, DeviceScene):
            return scene, False
        if isinstance(scene, Scene):
            return self.upload(scene), True
        return self.upload_splat3d(np.asarray(scene)), True

    # -- the reference API
    def render(self, scene, cam: Camera, cfg: RasterConfig, counters: bool = True):
        """polysplat::render -> (Framebuffer (fp32 arrays), PerfCounters)."""
        ds, tmp = self._scene(scene)
        try:
            c, g = cam.to_struct(), cfg.to_struct()
            rgb = np.zeros((cam.height, cam.width, 3), np.float32)
            tr = np.zeros((cam.height, cam.width), np.float32)
            ctr = abi.ps_counters()
            _check(lib().ps_render(self.handle, ds.handle, C.byref(c), C.byref(g), rgb.ctypes.data,
                                   tr.ctypes.data, abi.PS_MEM_HOST, C.byref(ctr) if counters else None),
                   self.handle)
            return Framebuffer(cam.width, cam.height, rgb, tr), PerfCounters.from_struct(ctr)
        finally:
            if tmp:
                ds.close()

    def render_views(self, scene, cams: Sequence[Camera], cfg: RasterConfig, counters: bool = True):
        """ps_render_views: a batch of views of one scene (K1 fused over up to 4
        views at a time). Returns a list of (Framebuffer, PerfCounters)."""
        ds, tmp = self._scene(scene)
        try:
            n = len(cams)
            if n == 0:
                return []
            w, h = cams[0].width, cams[0].height
            cs = (abi.ps_camera * n)(*[c.to_struct() for c in cams])
            g = cfg.to_struct()
            rgb = np.zeros((n, h, w, 3), np.float32)
            tr = np.zeros((n, h, w), np.float32)
            ctr = (abi.ps_counters * n)()
            _check(lib().ps_render_views(self.handle, ds.handle, cs, n, C.byref(g), rgb.ctypes.data, tr.ctypes.data,
                                         abi.PS_MEM_HOST, ctr if counters else None), self.handle)
            return [(Framebuffer(w, h, rgb[k], tr[k]), PerfCounters.from_struct(ctr[k])) for k in range(n)]
        finally:
            if tmp:
                ds.close()

    def render_splat3d(self, splats: np.ndarray, cam: Camera, cfg: RasterConfig):
        """One-shot drop-in (ps_render_splats): fp64 framebuffer with exact replayed pixels."""
        a = np.ascontiguousarray(splats, dtype=np.float64)
        c, g = cam.to_struct(), cfg.to_struct()
        rgb = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        ctr = abi.ps_counters()
        _check(lib().ps_render_splats(self.handle, abi.dptr(a), len(a), C.byref(c), C.byref(g), abi.dptr(rgb),
                                      abi.dptr(tr), C.byref(ctr)), self.handle)
        return Framebuffer(cam.width, cam.height, rgb, tr), PerfCounters.from_struct(ctr)

    def count_pairs(self, scene, cam: Camera, cfg: RasterConfig) -> PerfCounters:
        ds, tmp = self._scene(scene)
        try:
            c, g = cam.to_struct(), cfg.to_struct()
            ctr = abi.ps_counters()
            _check(lib().ps_count_pairs(self.handle, ds.handle, C.byref(c), C.byref(g), C.byref(ctr)), self.handle)
            return PerfCounters.from_struct(ctr)
        finally:
            if tmp:
                ds.close()

    def prepare_splats(self, scene, cam: Camera, cfg: RasterConfig) -> Prepared:
        ds, tmp = self._scene(scene)
        try:
            c, g = cam.to_struct(), cfg.to_struct()
            n = max(ds.n, 1)
            out = Prepared(np.zeros(n, np.uint32), np.zeros(n), np.zeros((n, 2)), np.zeros((n, 3)),
                           np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3), np.float32), np.zeros(n),
                           np.zeros(n), PerfCounters())
            p = abi.ps_prepared(abi.u32ptr(out.index), abi.dptr(out.depth), abi.dptr(out.mean2d),
                                abi.dptr(out.conic), abi.dptr(out.cov_aa), abi.dptr(out.opacity_eff),
                                abi.fptr(out.color), abi.dptr(out.radius_sigma), abi.dptr(out.quadric_root))
            nv = C.c_int64(0)
            ctr = abi.ps_counters()
            _check(lib().ps_prepare(self.handle, ds.handle, C.byref(c), C.byref(g), n, C.byref(p), C.byref(nv),
                                    C.byref(ctr)), self.handle)
            v = nv.value
            for f in ("index", "depth", "mean2d", "conic", "cov_aa", "opacity_eff", "color", "radius_sigma",
                      "quadric_root"):
                setattr(out, f, getattr(out, f)[:v].copy())
            out.counters = PerfCounters.from_struct(ctr)
            return out
        finally:
            if tmp:
                ds.close()

    def tile_lists(self, scene, cam: Camera, cfg: RasterConfig):
        """Per-tile splat lists as CSR (offsets[n_tiles+1], original splat indices), + counters."""
        ds, tmp = self._scene(scene)
        try:
            c, g = cam.to_struct(), cfg.to_struct()
            ts = cfg.tile_size
            nt = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
            npairs = C.c_int64(0)
            ctr = abi.ps_counters()
            _check(lib().ps_tile_lists(self.handle, ds.handle, C.byref(c), C.byref(g), 0, None, None,
                                       C.byref(npairs), C.byref(ctr)), self.handle)
            offsets = np.zeros(nt + 1, np.uint32)
            idx = np.zeros(max(npairs.value, 1), np.uint32)
            _check(lib().ps_tile_lists(self.handle, ds.handle, C.byref(c), C.byref(g), len(idx),
                                       abi.u32ptr(offsets), abi.u32ptr(idx), C.byref(npairs), C.byref(ctr)),
                   self.handle)
            return offsets, idx[: npairs.value].copy(), PerfCounters.from_struct(ctr)
        finally:
            if tmp:
                ds.close()

    # -- quality metrics (metrics.hpp:18-38)
    def image_metrics(self, a: "Framebuffer", b: "Framebuffer", background=(1.0, 1.0, 1.0)) -> "ImageMetrics":
        """composite + psnr / ssim / max_abs_diff of two host framebuffers, on the device."""
        if (a.width, a.height) != (b.width, b.height):
            raise Error("image dimensions differ")  # DimensionMismatch (metrics.cpp:28-31)
        f64 = a.rgb.dtype == np.float64 or b.rgb.dtype == np.float64
        dt = np.float64 if f64 else np.float32
        arrs = [np.ascontiguousarray(x, dtype=dt) for x in (a.rgb, a.transmittance, b.rgb, b.transmittance)]
        bg = np.ascontiguousarray(background, dtype=np.float64)
        out = abi.ps_image_metrics()
        _check(lib().ps_image_metrics_compute(self.handle, a.width, a.height, *[x.ctypes.data for x in arrs],
                                              abi.PS_DTYPE_F64 if f64 else abi.PS_DTYPE_F32, abi.PS_MEM_HOST,
                                              abi.dptr(bg), C.byref(out)), self.handle)
        return ImageMetrics.from_struct(out)

    def compare(self, scene, cam: Camera, cfg_a: RasterConfig, cfg_b: RasterConfig,
                background=(1.0, 1.0, 1.0)) -> "CompareReport":
        """polysplat::compare (metrics.cpp:138-157): renders both configs on the device and compares."""
        ds, tmp = self._scene(scene)
        try:
            c, ga, gb = cam.to_struct(), cfg_a.to_struct(), cfg_b.to_struct()
            bg = np.ascontiguousarray(background, dtype=np.float64)
            out = abi.ps_compare_report()
            _check(lib().ps_compare(self.handle, ds.handle, C.byref(c), C.byref(ga), C.byref(gb), abi.dptr(bg),
                                    C.byref(out)), self.handle)
            return CompareReport(ImageMetrics.from_struct(out.metrics), PerfCounters.from_struct(out.counters_a),
                                 PerfCounters.from_struct(out.counters_b), float(out.pair_ratio))
        finally:
            if tmp:
                ds.close()

    # -- instrumentation
    def set_timing(self, on: bool = True) -> None:
        _check(lib().ps_ctx_set_timing(self.handle, 1 if on else 0), self.handle)

    def stats(self) -> dict:
        s = abi.ps_stats()
        _check(lib().ps_last_stats(self.handle, C.byref(s)), self.handle)
        return {"visible": s.visible, "pairs": s.pairs, "replay_pixels": s.replay_pixels,
                "exact_alpha_evals": s.exact_alpha_evals, "kernel_launches": s.kernel_launches,
                "sort_prefix": s.sort_prefix,
                "stage_ms": {name: float(s.stage_ms[i]) for i, name in enumerate(abi.STAGES)}}

    def synchronize(self) -> None:
        _check(lib().ps_ctx_synchronize(self.handle), self.handle)


_default: Optional[Rasterizer] = None


def default_rasterizer() -> Rasterizer:
    global _default
    if _default is None:
        _default = Rasterizer(0)
    return _default


def render(splats, cam: Camera, cfg: RasterConfig):
    """polysplat::render(span<const Splat3D>, const Camera&, const RasterConfig&) on the default device."""
    return default_rasterizer().render(splats, cam, cfg)


def count_pairs(splats, cam: Camera, cfg: RasterConfig) -> PerfCounters:
    return default_rasterizer().count_pairs(splats, cam, cfg)


def prepare_splats(splats, cam: Camera, cfg: RasterConfig) -> Prepared:
    return default_rasterizer().prepare_splats(splats, cam, cfg)


def device_count() -> int:
    return lib().ps_device_count()


# ---------------------------------------------------------------- metrics / ablation (metrics.hpp, main.cpp)
@dataclass
class ImageMetrics:
    """psnr / ssim / max_abs_diff of two composited images (metrics.hpp:18-30).
    ssim is None where the reference throws TooSmall (images under 11x11)."""
    psnr_db: float
    ssim: Optional[float]
    max_abs_diff: float

    @staticmethod
    def from_struct(m: abi.ps_image_metrics) -> "ImageMetrics":
        return ImageMetrics(float(m.psnr_db), float(m.ssim) if m.ssim_valid else None, float(m.max_abs_diff))


@dataclass
class CompareReport:
    """CompareReport (metrics.hpp:32-38)."""
    metrics: ImageMetrics
    counters_a: PerfCounters
    counters_b: PerfCounters
    pair_ratio: float
    # device frame times (ms, median of timed frames; ablation_grid fills them):
    # config a (the exp / StopThePop reference cell) and config b, and b's blend stage
    frame_ms_a: Optional[float] = None
    frame_ms_b: Optional[float] = None
    blend_ms_b: Optional[float] = None

    @property
    def psnr_db(self) -> float:
        return self.metrics.psnr_db

    @property
    def ssim(self) -> Optional[float]:
        return self.metrics.ssim

    @property
    def max_abs_diff(self) -> float:
        return self.metrics.max_abs_diff


def _fmt17(v: float) -> str:
    """metrics.cpp fmt17: %.17g, with inf / -inf spelled out."""
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def csv_header() -> str:
    """metrics.cpp csv_header."""
    return "label_a,label_b,psnr_db,ssim,max_abs_diff,pairs_a,pairs_b,pair_ratio\n"


def csv_row(label_a: str, label_b: str, r: CompareReport) -> str:
    """metrics.cpp csv_row (values round-trip exactly)."""
    return (f"{label_a},{label_b},{_fmt17(r.psnr_db)},{_fmt17(r.ssim if r.ssim is not None else 0.0)},"
            f"{_fmt17(r.max_abs_diff)},{r.counters_a.tile_pairs_after_tight_test},"
            f"{r.counters_b.tile_pairs_after_tight_test},{_fmt17(r.pair_ratio)}\n")


# The reference CLI's ablation cells (tools/main.cpp:315-323): kernel x culling,
# each compared against exp / StopThePop.
ABLATION_CELLS = (
    ("exp/stp", "exp", CullingMode.StopThePop),
    ("poly1/stp", "poly1", CullingMode.StopThePop),
    ("poly1/zero", "poly1", CullingMode.ZeroCrossing),
    ("poly1/opacity", "poly1", CullingMode.OpacityAware),
    ("poly2p/opacity", "poly2p", CullingMode.OpacityAware),
    ("poly3/stp", "poly3", CullingMode.StopThePop),
    ("poly3/opacity", "poly3", CullingMode.OpacityAware),
)


def frame_times(rasterizer: "Rasterizer", scene, cam: Camera, cfg: RasterConfig, frames: int = 5) -> dict:
    """Device time of one frame (ms; median over `frames` frames after one
    warm-up, stage events on the rasterizer's stream, counters off) and its
    stage split."""
    ds, tmp = rasterizer._scene(scene)
    try:
        rasterizer.render(ds, cam, cfg, counters=False)
        rasterizer.set_timing(True)
        runs = []
        for _ in range(max(1, frames)):
            rasterizer.render(ds, cam, cfg, counters=False)
            runs.append(rasterizer.stats()["stage_ms"])
        rasterizer.set_timing(False)
        order = sorted(range(len(runs)), key=lambda k: sum(runs[k].values()))
        med = runs[order[len(runs) // 2]]
        return {"frame_ms": sum(med.values()), "stage_ms": med}
    finally:
        if tmp:
            ds.close()


def ablation_grid(rasterizer: "Rasterizer", scene, cam: Camera, base: Optional[RasterConfig] = None,
                  background=(1.0, 1.0, 1.0), cells=ABLATION_CELLS, time_frames: int = 5):
    """The reference's ablation grid (tools/main.cpp:300-345) on the device:
    every cell compared against exp / StopThePop with the fitted kernels, and
    (time_frames > 0) each cell's device frame time (the paper's Table 3 with
    measured times instead of pair counts): frame_ms_b /
    blend_ms_b of every report, frame_ms_a = the exp / StopThePop frame.
    Returns (reports by label, csv text in the reference's format)."""
    base = base or RasterConfig()
    ds, tmp = rasterizer._scene(scene)
    try:
        def cfg(kname, mode):
            return RasterConfig(tile_size=base.tile_size, epsilon=base.epsilon,
                                transmittance_floor=base.transmittance_floor, culling_mode=mode,
                                kernel=fitted_kernel(kname), v_dilation=base.v_dilation,
                                sh_degree=base.sh_degree, clamp_before_blend=base.clamp_before_blend)
        ref = cfg("exp", CullingMode.StopThePop)
        ref_t = frame_times(rasterizer, ds, cam, ref, time_frames) if time_frames > 0 else None
        reports, csv = {}, csv_header()
        for label, kname, mode in cells:
            c = cfg(kname, mode)
            r = rasterizer.compare(ds, cam, ref, c, background)
            if ref_t is not None:
                t = frame_times(rasterizer, ds, cam, c, time_frames)
                r.frame_ms_a = ref_t["frame_ms"]
                r.frame_ms_b = t["frame_ms"]
                r.blend_ms_b = t["stage_ms"].get("blend")
            reports[label] = r
            csv += csv_row("exp/stp", label, r)
        return reports, csv
    finally:
        if tmp:
            ds.close()
