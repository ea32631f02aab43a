"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the parity checkers.

* ``Restatement`` wraps oracle/libps_oracle.so (ps_oracle.c, the plain-C fp64
  restatement of the reference's hot path).
* ``Reference`` wraps oracle/_ref/libpolysplat_ref.so (the UNMODIFIED reference
  library compiled from /root/reference by oracle/Makefile, plus ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module; the product (paper_2603_18707_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2603_18707_b200 import abi
from paper_2603_18707_b200.abi import dptr, u32ptr

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "libps_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libpolysplat_ref.so")


def build() -> None:
    """Builds the checkers (the reference only where /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "-s", "all"], check=True)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


@dataclass
class Prepared:
    index: np.ndarray
    depth: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    cov_aa: np.ndarray
    opacity_eff: np.ndarray
    color: np.ndarray
    radius_sigma: np.ndarray
    quadric_root: np.ndarray
    counters: dict


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        cam_p, cfg_p, ctr_p = C.POINTER(abi.ps_camera), C.POINTER(abi.ps_config), C.POINTER(abi.ps_counters)
        dp, u32p, i64 = C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.c_int64
        getattr(L, p + "last_error").restype = C.c_char_p
        self._fn("render", [dp, i64, cam_p, cfg_p, dp, dp, ctr_p])
        self._fn("render_serial", [dp, i64, cam_p, cfg_p, dp, dp])
        self._fn("count_pairs", [dp, i64, cam_p, cfg_p, ctr_p])
        self._fn("prepare", [dp, i64, cam_p, cfg_p, i64, u32p, dp, dp, dp, dp, dp, dp, dp, dp,
                             C.POINTER(C.c_int64), ctr_p])
        self._fn("tile_lists", [dp, i64, cam_p, cfg_p, i64, u32p, u32p, C.POINTER(C.c_int64), ctr_p])
        self._fn("first_positive_root", [dp, C.c_int, dp])
        self._fn("make_polynomial_kernel", [C.c_int, dp, C.c_int, C.POINTER(abi.ps_kernel)])
        self._fn("culling_radius", [C.POINTER(abi.ps_kernel), C.c_double, C.c_double, dp, dp,
                                    C.POINTER(C.c_int)])
        getattr(L, p + "eval_kernel").argtypes = [C.POINTER(abi.ps_kernel), C.c_double]
        getattr(L, p + "eval_kernel").restype = C.c_double
        self._fn("validate_config", [cfg_p])
        self._fn("validate_camera", [cam_p])
        self._fn("project_splat", [dp, cam_p, C.c_double, C.c_int, dp])
        getattr(L, p + "min_quadric_over_box").argtypes = [dp, C.c_double, C.c_double, dp]
        getattr(L, p + "min_quadric_over_box").restype = C.c_double

    def _fn(self, name, argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = C.c_int

    def _call(self, name, *args) -> int:
        st = getattr(self.lib, self.prefix + name)(*args)
        if st != abi.PS_OK:
            raise OracleError(st, getattr(self.lib, self.prefix + "last_error")().decode())
        return st

    # -- hot path ---------------------------------------------------------
    def render(self, splats: np.ndarray, cam: abi.ps_camera, cfg: abi.ps_config):
        """polysplat::render -> (rgb[H,W,3] f64, transmittance[H,W] f64, counters dict)."""
        splats = np.ascontiguousarray(splats, dtype=np.float64)
        rgb = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        ctr = abi.ps_counters()
        self._call("render", dptr(splats), len(splats), C.byref(cam), C.byref(cfg), dptr(rgb),
                   dptr(tr), C.byref(ctr))
        return rgb, tr, ctr.as_dict()

    def render_serial(self, splats, cam, cfg):
        splats = np.ascontiguousarray(splats, dtype=np.float64)
        rgb = np.zeros((cam.height, cam.width, 3))
        tr = np.zeros((cam.height, cam.width))
        self._call("render_serial", dptr(splats), len(splats), C.byref(cam), C.byref(cfg),
                   dptr(rgb), dptr(tr))
        return rgb, tr

    def count_pairs(self, splats, cam, cfg) -> dict:
        splats = np.ascontiguousarray(splats, dtype=np.float64)
        ctr = abi.ps_counters()
        self._call("count_pairs", dptr(splats), len(splats), C.byref(cam), C.byref(cfg), C.byref(ctr))
        return ctr.as_dict()

    def prepare(self, splats, cam, cfg) -> Prepared:
        splats = np.ascontiguousarray(splats, dtype=np.float64)
        n = len(splats)
        cap = max(n, 1)
        out = Prepared(np.zeros(cap, np.uint32), np.zeros(cap), np.zeros((cap, 2)), np.zeros((cap, 3)),
                       np.zeros((cap, 3)), np.zeros(cap), np.zeros((cap, 3)), np.zeros(cap),
                       np.zeros(cap), {})
        nv = C.c_int64(0)
        ctr = abi.ps_counters()
        self._call("prepare", dptr(splats), n, C.byref(cam), C.byref(cfg), cap, u32ptr(out.index),
                   dptr(out.depth), dptr(out.mean2d), dptr(out.conic), dptr(out.cov_aa),
                   dptr(out.opacity_eff), dptr(out.color), dptr(out.radius_sigma),
                   dptr(out.quadric_root), C.byref(nv), C.byref(ctr))
        v = nv.value
        for f in ("index", "depth", "mean2d", "conic", "cov_aa", "opacity_eff", "color",
                  "radius_sigma", "quadric_root"):
            setattr(out, f, getattr(out, f)[:v].copy())
        out.counters = ctr.as_dict()
        return out

    def tile_lists(self, splats, cam, cfg):
        """Per-tile lists as CSR (offsets[n_tiles+1], original splat indices)."""
        splats = np.ascontiguousarray(splats, dtype=np.float64)
        ts = cfg.tile_size
        nt = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
        npairs = C.c_int64(0)
        ctr = abi.ps_counters()
        self._call("tile_lists", dptr(splats), len(splats), C.byref(cam), C.byref(cfg), 0, None, None,
                   C.byref(npairs), C.byref(ctr))
        offsets = np.zeros(nt + 1, np.uint32)
        idx = np.zeros(max(npairs.value, 1), np.uint32)
        self._call("tile_lists", dptr(splats), len(splats), C.byref(cam), C.byref(cfg), len(idx),
                   u32ptr(offsets), u32ptr(idx), C.byref(npairs), C.byref(ctr))
        return offsets, idx[: npairs.value].copy(), ctr.as_dict()

    # -- kernel math ------------------------------------------------------
    def first_positive_root(self, coeffs) -> float:
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = C.c_double(0)
        self._call("first_positive_root", dptr(c), len(c), C.byref(out))
        return out.value

    def make_polynomial_kernel(self, kind: int, coeffs) -> abi.ps_kernel:
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        k = abi.ps_kernel()
        self._call("make_polynomial_kernel", kind, dptr(c), len(c), C.byref(k))
        return k

    def culling_radius(self, kernel: abi.ps_kernel, o: float, eps: float):
        r, q, a = C.c_double(0), C.c_double(0), C.c_int(0)
        self._call("culling_radius", C.byref(kernel), o, eps, C.byref(r), C.byref(q), C.byref(a))
        return r.value, q.value, bool(a.value)

    def eval_kernel(self, kernel: abi.ps_kernel, x: float) -> float:
        return getattr(self.lib, self.prefix + "eval_kernel")(C.byref(kernel), x)

    def validate_config(self, cfg):
        return self._call("validate_config", C.byref(cfg))

    def validate_camera(self, cam):
        return self._call("validate_camera", C.byref(cam))

    def project_splat(self, splat, cam, v, sh_degree):
        s = np.ascontiguousarray(splat, dtype=np.float64)
        out = np.zeros(14)
        st = getattr(self.lib, self.prefix + "project_splat")(dptr(s), C.byref(cam), v, sh_degree, dptr(out))
        if st < 0:
            raise OracleError(-st, getattr(self.lib, self.prefix + "last_error")().decode())
        return out if st == 1 else None

    def min_quadric_over_box(self, conic, mx, my, box) -> float:
        c = np.ascontiguousarray(conic, dtype=np.float64)
        b = np.ascontiguousarray(box, dtype=np.float64)
        return getattr(self.lib, self.prefix + "min_quadric_over_box")(dptr(c), mx, my, dptr(b))


class Restatement(_Lib):
    prefix = "or_"

    def __init__(self, path: str = RESTATEMENT_SO):
        super().__init__(path)


class Reference(_Lib):
    """The unmodified reference (oracle/_ref), via ref_shim.cpp."""

    prefix = "ref_"

    def __init__(self, path: str = REFERENCE_SO):
        super().__init__(path)
        L = self.lib
        L.ref_synth_scene.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_int64,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.ref_synth_scene.restype = C.c_int
        L.ref_synth_g.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.POINTER(C.c_double), C.c_int64]
        L.ref_synth_g.restype = C.c_int
        L.ref_orbit_cameras.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.POINTER(abi.ps_camera)]
        L.ref_orbit_cameras.restype = C.c_int
        L.ref_fit_polynomial.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                         C.POINTER(abi.ps_kernel), C.POINTER(C.c_double)]
        L.ref_fit_polynomial.restype = C.c_int
        L.ref_tile_rect.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double), C.c_double,
                                    C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_tile_rect.restype = C.c_int
        L.ref_compare_images.argtypes = [C.c_int, C.c_int] + [C.POINTER(C.c_double)] * 5 + [
            C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_compare_images.restype = C.c_int
        L.ref_load_ply.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int)]
        L.ref_load_ply.restype = C.c_int
        L.ref_write_ply.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int, C.c_char_p]
        L.ref_write_ply.restype = C.c_int
        L.ref_resolve_thread_count.argtypes = [C.c_int]
        L.ref_resolve_thread_count.restype = C.c_int

    def synth_scene(self, kind: int, seed: int = 0):
        n = C.c_int64(0)
        deg = C.c_int(0)
        self._call("synth_scene", kind, seed, None, 0, C.byref(n), C.byref(deg))
        out = np.zeros((n.value, abi.SPLAT3D_DOUBLES))
        self._call("synth_scene", kind, seed, dptr(out), n.value, C.byref(n), C.byref(deg))
        return out, deg.value

    def synth_g(self, n: int, seed: int, skewed: bool = False):
        """G(n, seed) (skewed: the C5 opacity law) as a Splat3D
        array (n, 59), generated inside the reference library (ref_shim.cpp)."""
        out = np.zeros((n, abi.SPLAT3D_DOUBLES))
        self._call("synth_g", 4 if skewed else 3, seed, n, dptr(out), n)
        return out, 3

    def orbit_cameras(self, count, width, height, fov_deg=50.0, radius=2.0, elevation=0.3):
        cams = (abi.ps_camera * count)()
        self._call("orbit_cameras", count, width, height, fov_deg, radius, elevation, cams)
        return list(cams)

    def fit_polynomial(self, order, epsilon=1.0 / 255.0, iterations=30000, samples=4096, step=0.01):
        k = abi.ps_kernel()
        loss = C.c_double(0)
        self._call("fit_polynomial", order, epsilon, iterations, samples, step, C.byref(k), C.byref(loss))
        return k, loss.value

    def tile_rect(self, mx, my, cov_aa, radius, tile_size, width, height):
        cv = np.ascontiguousarray(cov_aa, dtype=np.float64)
        r = (C.c_int * 4)()
        ok = self.lib.ref_tile_rect(mx, my, dptr(cv), radius, tile_size, width, height, r)
        return tuple(r) if ok else None

    def compare_images(self, rgb_a, t_a, rgb_b, t_b, bg=(1.0, 1.0, 1.0), with_ssim=False):
        """composite + psnr / max_abs_diff (+ ssim) of the reference (metrics.cpp:13-134)."""
        h, w = t_a.shape
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (rgb_a, t_a, rgb_b, t_b, bg)]
        p, m, s = C.c_double(0), C.c_double(0), C.c_double(0)
        self._call("compare_images", w, h, *[dptr(a) for a in arrs], C.byref(p), C.byref(m),
                   C.byref(s) if with_ssim else None)
        return (p.value, m.value, s.value) if with_ssim else (p.value, m.value)

    def load_ply(self, path):
        """load_ply -> (Splat3D array (n, 59), sh_degree); raises OracleError(status, msg)."""
        n, deg = C.c_int64(0), C.c_int(0)
        self._call("load_ply", str(path).encode(), None, 0, C.byref(n), C.byref(deg))
        out = np.zeros((n.value, abi.SPLAT3D_DOUBLES))
        self._call("load_ply", str(path).encode(), dptr(out), n.value, C.byref(n), C.byref(deg))
        return out, deg.value

    def write_ply(self, splats, sh_degree, path):
        a = np.ascontiguousarray(splats, dtype=np.float64)
        self._call("write_ply", dptr(a), len(a), sh_degree, str(path).encode())

    def resolve_thread_count(self, requested: int = 0) -> int:
        return self.lib.ref_resolve_thread_count(requested)


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
