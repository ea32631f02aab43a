// exact_math.cuh — the reference's fp64 geometry, kernel and culling math,
// restated for device (and host) with the reference's operation order.
//
// BIT-EXACTNESS CONTRACT: include this header only from translation units
// compiled with `-fmad=false` (device) and `-ffp-contract=off` (host). fp64
// add/mul/div/sqrt are then IEEE round-to-nearest on both sides, so every
// arithmetic-only result (depth, mean2d, conic, cov_aa, opacity_eff, culling
// roots of order 1/2, tile rects, tight tests) is bit-identical to the
// reference compiled without FMA (SURVEY finding 2). The libm transcendentals
// (log for StopThePop/exp bounds, cbrt/acos/cos for cubic roots) come from
// libdevice and may differ from glibc by <= 1-2 ulp; the reference's
// kBoundSlack (raster.cpp:36-46) keeps such differences from changing any tile
// decision, and tests/ measure the bit agreement of those bounds.
//
// Citations are relative to /root/reference/proj.
#pragma once

#include <cmath>
#include <cstdint>
#include <climits>

#include "polysplat_b200.h"

#ifdef __CUDACC__
#define PS_HD __host__ __device__ __forceinline__
#else
#define PS_HD inline
#endif

namespace ps {

constexpr double kNearPlane = 0.2;   // projection.hpp:44
constexpr double kBoundSlack = 1e-7; // raster.cpp:40

// std::max / std::min / std::clamp argument-order semantics (NaN handling).
PS_HD double std_max(double a, double b) { return (a < b) ? b : a; }
PS_HD double std_min(double a, double b) { return (b < a) ? b : a; }
PS_HD double std_clamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }
PS_HD int imax(int a, int b) { return (a < b) ? b : a; }
PS_HD int imin(int a, int b) { return (b < a) ? b : a; }

// static_cast<int>(double) as the x86-64 reference build executes it
// (cvttsd2si): NaN or out-of-range gives INT_MIN. CUDA's conversion saturates
// instead, so the device must not use a plain cast for tile_rect.
PS_HD int x86_cvtt_int(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
    return static_cast<int>(v);
}

struct Sym2 { double xx, xy, yy; };
PS_HD double det(const Sym2& s) { return s.xx * s.yy - s.xy * s.xy; }   // geometry.hpp:45
PS_HD Sym2 inverse(const Sym2& s) {                                       // geometry.hpp:47-50
    double d = det(s);
    return {s.yy / d, -s.xy / d, s.xx / d};
}
PS_HD double quadric(const Sym2& s, double dx, double dy) {               // geometry.hpp:53-55
    return s.xx * dx * dx + 2.0 * s.xy * dx * dy + s.yy * dy * dy;
}

// geometry.hpp:97-111 (with Quat::normalized, geometry.hpp:33-38)
PS_HD void rotation_from_quat(double w, double x, double y, double z, double r[9]) {
    double n = sqrt(w * w + x * x + y * y + z * z);
    if (n < 1e-12) { w = 1.0; x = 0.0; y = 0.0; z = 0.0; }
    else { w = w / n; x = x / n; y = y / n; z = z / n; }
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}

// projection.cpp:24-34 + Mat3::operator* (geometry.hpp:70-79); symmetric, so
// only the 6 distinct entries are produced (each with the reference's sum order).
PS_HD void covariance3d(const double s[3], const double q[4], double c[9]) {
    double rs[9];
    rotation_from_quat(q[0], q[1], q[2], q[3], rs);
    for (int i = 0; i < 3; ++i) {
        rs[i * 3 + 0] *= s[0];
        rs[i * 3 + 1] *= s[1];
        rs[i * 3 + 2] *= s[2];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += rs[i * 3 + k] * rs[j * 3 + k];
            c[i * 3 + j] = acc;
        }
}

struct Projected {
    double mx, my;
    Sym2 conic, cov_aa;
    double depth, opacity_eff;
};

// projection.cpp:36-79 project_splat (geometry part; the SH colour of :77 is
// evaluated separately in fp32). Returns 1 visible, 0 behind the near plane,
// -PS_DEGENERATE_COVARIANCE when det(cov_aa) <= 1e-12.
// cov3d: the 3D covariance of covariance3d(scale, quat) as its 6 distinct
// entries (xx, xy, xz, yy, yz, zz). It does not depend on the camera, so the
// scene stores it (computed once per upload with this same arithmetic).
PS_HD int project(const double mean[3], const double c6[6], double opacity, const ps_camera& cam, double v,
                  Projected& out) {
    const double* R = cam.rotation;
    const double* t = cam.translation;
    double px = R[0] * mean[0] + R[1] * mean[1] + R[2] * mean[2];
    double py = R[3] * mean[0] + R[4] * mean[1] + R[5] * mean[2];
    double pz = R[6] * mean[0] + R[7] * mean[1] + R[8] * mean[2];
    px = px + t[0];
    py = py + t[1];
    pz = pz + t[2];
    if (pz <= kNearPlane) return 0;

    double inv_z = 1.0 / pz;
    out.mx = cam.fx * px * inv_z + cam.cx;
    out.my = cam.fy * py * inv_z + cam.cy;
    double jr0[3] = {cam.fx * inv_z, 0.0, -cam.fx * px * inv_z * inv_z};
    double jr1[3] = {0.0, cam.fy * inv_z, -cam.fy * py * inv_z * inv_z};
    double m0[3], m1[3];
    for (int j = 0; j < 3; ++j) {
        m0[j] = jr0[0] * R[0 * 3 + j] + jr0[1] * R[1 * 3 + j] + jr0[2] * R[2 * 3 + j];
        m1[j] = jr1[0] * R[0 * 3 + j] + jr1[1] * R[1 * 3 + j] + jr1[2] * R[2 * 3 + j];
    }
    const double cov3d[9] = {c6[0], c6[1], c6[2], c6[1], c6[3], c6[4], c6[2], c6[4], c6[5]};
    double t0[3], t1[3];
    for (int j = 0; j < 3; ++j) {
        t0[j] = m0[0] * cov3d[0 * 3 + j] + m0[1] * cov3d[1 * 3 + j] + m0[2] * cov3d[2 * 3 + j];
        t1[j] = m1[0] * cov3d[0 * 3 + j] + m1[1] * cov3d[1 * 3 + j] + m1[2] * cov3d[2 * 3 + j];
    }
    Sym2 cov;
    cov.xx = t0[0] * m0[0] + t0[1] * m0[1] + t0[2] * m0[2];
    cov.xy = t0[0] * m1[0] + t0[1] * m1[1] + t0[2] * m1[2];
    cov.yy = t1[0] * m1[0] + t1[1] * m1[1] + t1[2] * m1[2];
    Sym2 cov_aa{cov.xx + v, cov.xy, cov.yy + v};
    double det_aa = det(cov_aa);
    if (det_aa <= 1e-12) return -PS_DEGENERATE_COVARIANCE;
    double d = det(cov);
    double ratio = d > 0.0 ? sqrt(d / det_aa) : 0.0;
    out.cov_aa = cov_aa;
    out.conic = inverse(cov_aa);
    out.depth = pz;
    out.opacity_eff = opacity * ratio;
    return 1;
}

// ------------------------------------------------------------ polynomial roots
// kernel.cpp:16-20
PS_HD double horner(const double* c, int n, double x) {
    double p = c[n - 1];
    for (int i = n - 2; i >= 0; --i) p = p * x + c[i];
    return p;
}
// kernel.cpp:22-27
PS_HD double horner_derivative(const double* c, int n, double x) {
    int d = n - 1;
    double p = c[d] * d;
    for (int i = d - 1; i >= 1; --i) p = p * x + c[i] * i;
    return p;
}
// kernel.cpp:30-41
PS_HD double polish_root(const double* c, int n, double x) {
    for (int it = 0; it < 2; ++it) {
        double f = horner(c, n, x);
        double d = horner_derivative(c, n, x);
        if (d == 0.0) break;
        double nx = x - f / d;
        if (!(nx > 0.0) || !isfinite(nx)) break;
        if (fabs(horner(c, n, nx)) >= fabs(f)) break;
        x = nx;
    }
    return x;
}
// kernel.cpp:43-48
PS_HD int root_linear(double c0, double c1, double& out) {
    if (c1 == 0.0) return PS_NO_POSITIVE_ROOT;
    double x = -c0 / c1;
    if (!(x > 0.0)) return PS_NO_POSITIVE_ROOT;
    out = x;
    return PS_OK;
}
// kernel.cpp:50-68
PS_HD int root_quadratic(const double* c, double& out) {
    double c0 = c[0], c1 = c[1], c2 = c[2];
    double disc = c1 * c1 - 4.0 * c2 * c0;
    if (disc < 0.0) return PS_NO_POSITIVE_ROOT;
    double s = sqrt(disc);
    double q = -0.5 * (c1 + copysign(s, c1));
    double best = INFINITY;
    if (q != 0.0) {
        double r = q / c2;
        if (r > 0.0 && isfinite(r)) best = std_min(best, r);
        r = c0 / q;
        if (r > 0.0 && isfinite(r)) best = std_min(best, r);
    } else {
        return PS_NO_POSITIVE_ROOT;
    }
    if (!isfinite(best)) return PS_NO_POSITIVE_ROOT;
    out = best;
    return PS_OK;
}
// kernel.cpp:70-109
PS_HD int root_cubic(const double* c, double& out) {
    const double pi = 3.141592653589793; // std::numbers::pi
    double c0 = c[0], c1 = c[1], c2 = c[2], c3 = c[3];
    double d0 = c2 * c2 - 3.0 * c3 * c1;
    double d1 = 2.0 * c2 * c2 * c2 - 9.0 * c3 * c2 * c1 + 27.0 * c3 * c3 * c0;
    double disc = d1 * d1 - 4.0 * d0 * d0 * d0;
    double best = INFINITY;
    if (disc > 0.0) {
        double sq = sqrt(disc);
        double n = (d1 >= 0.0) ? 0.5 * (d1 + sq) : 0.5 * (d1 - sq);
        double C = cbrt(n);
        double x;
        if (C == 0.0) x = -c2 / (3.0 * c3);
        else x = -(c2 + C + d0 / C) / (3.0 * c3);
        if (x > 0.0) best = x;
    } else {
        double p = (3.0 * c3 * c1 - c2 * c2) / (3.0 * c3 * c3);
        double q = (2.0 * c2 * c2 * c2 - 9.0 * c3 * c2 * c1 + 27.0 * c3 * c3 * c0) /
                   (27.0 * c3 * c3 * c3);
        double mp3 = -p / 3.0;
        double m = 2.0 * sqrt(std_max(mp3, 0.0));
        double arg = 0.0;
        if (m > 0.0) arg = 3.0 * q / (p * m);
        arg = std_clamp(arg, -1.0, 1.0);
        double theta = acos(arg) / 3.0;
        double shift = -c2 / (3.0 * c3);
        for (int k = 0; k < 3; ++k) {
            double t = m * cos(theta - 2.0 * pi * k / 3.0);
            double x = t + shift;
            if (x > 0.0) best = std_min(best, x);
        }
    }
    if (!isfinite(best)) return PS_NO_POSITIVE_ROOT;
    out = best;
    return PS_OK;
}
// kernel.cpp:117-135 first_positive_root
PS_HD int first_positive_root(const double* coeffs, int n, double& out) {
    if (n < 1 || !(coeffs[0] > 0.0)) return PS_INVALID_ARGUMENT;
    if (n > 4) return PS_INVALID_ARGUMENT;
    while (n > 1 && fabs(coeffs[n - 1]) < 1e-12) --n;
    double x = 0.0;
    int st;
    switch (n) {
        case 1: return PS_NO_POSITIVE_ROOT;
        case 2: st = root_linear(coeffs[0], coeffs[1], x); break;
        case 3: st = root_quadratic(coeffs, x); break;
        default: st = root_cubic(coeffs, x); break;
    }
    if (st != PS_OK) return st;
    out = polish_root(coeffs, n, x);
    return PS_OK;
}

// kernel.cpp:162-172 eval_kernel
PS_HD double eval_kernel(const ps_kernel& k, double x) {
    switch (k.kind) {
        case PS_KERNEL_EXPONENTIAL: return exp(-0.5 * x);
        case PS_KERNEL_POLY_RELU: return std_max(horner(k.coeffs, k.order + 1, x), 0.0);
        case PS_KERNEL_POLY_PIECEWISE: return x < k.first_root ? horner(k.coeffs, k.order + 1, x) : 0.0;
    }
    return 0.0;
}

// kernel.cpp:335-358 culling_radius (quadric root only; radius = sqrt(root)).
PS_HD int culling_root(const ps_kernel& k, double o, double eps, double& x) {
    if (!(o > 0.0) || o > 1.0) return PS_INVALID_ARGUMENT;
    if (eps < 0.0) return PS_INVALID_ARGUMENT;
    if (k.kind == PS_KERNEL_EXPONENTIAL) {
        if (eps == 0.0) return PS_EPSILON_ZERO_UNBOUNDED;
        if (!(o > eps)) return PS_FULLY_CULLED;
        x = 2.0 * log(o / eps);
        return PS_OK;
    }
    if (!(o * k.coeffs[0] > eps)) return PS_FULLY_CULLED;
    if (eps == 0.0) {
        x = k.first_root;
        return PS_OK;
    }
    double shifted[4] = {k.coeffs[0], k.coeffs[1], k.coeffs[2], k.coeffs[3]};
    shifted[0] -= eps / o;
    return first_positive_root(shifted, k.order + 1, x);
}

// raster.cpp:50-69 culling_bound_for + widen (raster.cpp:42-46).
// Returns 1 (bound set), 0 (nullopt: below epsilon, dropped uncounted) or -status.
PS_HD int culling_bound_for(const ps_config& cfg, double o, double& radius, double& qroot) {
    if (!(o > 0.0)) return 0;
    const ps_kernel& bk = cfg.has_culling_kernel ? cfg.culling_kernel : cfg.kernel;
    double x = 0.0;
    switch (cfg.culling_mode) {
        case PS_CULL_STOP_THE_POP:
            if (!(o > cfg.epsilon)) return 0;
            x = 2.0 * log(o / cfg.epsilon);
            break;
        case PS_CULL_ZERO_CROSSING:
            x = bk.first_root;
            break;
        case PS_CULL_OPACITY_AWARE: {
            // kernel.cpp:360-369 try_culling_radius: FullyCulled -> nullopt, others propagate
            if (bk.kind == PS_KERNEL_EXPONENTIAL && cfg.epsilon == 0.0) return -PS_EPSILON_ZERO_UNBOUNDED;
            int st = culling_root(bk, o, cfg.epsilon, x);
            if (st == PS_FULLY_CULLED) return 0;
            if (st != PS_OK) return -st;
            break;
        }
        default: return 0;
    }
    qroot = x + kBoundSlack;
    radius = sqrt(qroot);
    return 1;
}

// raster.cpp:71-86 tile_rect. Returns false when the rect misses the image.
PS_HD bool tile_rect(double mx, double my, double cov_xx, double cov_yy, double radius, int ts,
                     int width, int height, int r[4]) {
    double hx = radius * sqrt(std_max(cov_xx, 0.0));
    double hy = radius * sqrt(std_max(cov_yy, 0.0));
    int tiles_x = (width + ts - 1) / ts;
    int tiles_y = (height + ts - 1) / ts;
    int x0 = x86_cvtt_int(floor((mx - hx) / ts));
    int x1 = x86_cvtt_int(floor((mx + hx) / ts));
    int y0 = x86_cvtt_int(floor((my - hy) / ts));
    int y1 = x86_cvtt_int(floor((my + hy) / ts));
    x0 = imax(x0, 0);
    y0 = imax(y0, 0);
    x1 = imin(x1, tiles_x - 1);
    y1 = imin(y1, tiles_y - 1);
    if (x0 > x1 || y0 > y1) return false;
    r[0] = x0; r[1] = y0; r[2] = x1; r[3] = y1;
    return true;
}

// raster.cpp:103-124 min_quadric_over_box with the box of tile_pixel_box
// (raster.cpp:97-101): pixel centres, NOT clipped at the image edge.
PS_HD double min_quadric_over_box(const Sym2& cn, double mx, double my, double bx0, double by0,
                                  double bx1, double by1) {
    double lx = bx0 - mx, hx = bx1 - mx;
    double ly = by0 - my, hy = by1 - my;
    if (lx <= 0.0 && hx >= 0.0 && ly <= 0.0 && hy >= 0.0) return 0.0;
    double a = cn.xx, b = cn.xy, c = cn.yy;
    double dy = std_clamp(c != 0.0 ? -b * lx / c : ly, ly, hy);
    double m = quadric(cn, lx, dy);
    dy = std_clamp(c != 0.0 ? -b * hx / c : ly, ly, hy);
    m = std_min(m, quadric(cn, hx, dy));
    double dx = std_clamp(a != 0.0 ? -b * ly / a : lx, lx, hx);
    m = std_min(m, quadric(cn, dx, ly));
    dx = std_clamp(a != 0.0 ? -b * hy / a : lx, lx, hx);
    m = std_min(m, quadric(cn, dx, hy));
    return m;
}

// raster.cpp:126-128 tight_tile_test on tile (tx, ty)
PS_HD bool tight_tile_test(const Sym2& cn, double mx, double my, double qroot, int tx, int ty, int ts) {
    double x0 = tx * static_cast<double>(ts) + 0.5;
    double y0 = ty * static_cast<double>(ts) + 0.5;
    return min_quadric_over_box(cn, mx, my, x0, y0, x0 + ts - 1, y0 + ts - 1) <= qroot;
}

// raster.cpp:13-23 RasterConfig::validate
PS_HD int validate_config(const ps_config& c) {
    if (c.tile_size < 1) return PS_INVALID_ARGUMENT;
    if (!(c.epsilon > 0.0) || !(c.epsilon < 1.0)) return PS_INVALID_ARGUMENT;
    if (!(c.transmittance_floor >= 0.0) || !(c.transmittance_floor < 1.0)) return PS_INVALID_ARGUMENT;
    const ps_kernel& bk = c.has_culling_kernel ? c.culling_kernel : c.kernel;
    if (c.culling_mode == PS_CULL_ZERO_CROSSING && bk.kind == PS_KERNEL_EXPONENTIAL) return PS_INVALID_ARGUMENT;
    if (c.v_dilation < 0.0) return PS_INVALID_ARGUMENT;
    if (c.thread_count < 0) return PS_INVALID_ARGUMENT;
    return PS_OK;
}

// projection.cpp:10-22 Camera::validate
PS_HD int validate_camera(const ps_camera& cam) {
    if (cam.width <= 0 || cam.height <= 0) return PS_INVALID_ARGUMENT;
    if (!(cam.fx > 0.0) || !(cam.fy > 0.0)) return PS_INVALID_ARGUMENT;
    const double* m = cam.rotation;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += m[k * 3 + i] * m[k * 3 + j];
            double expect = (i == j) ? 1.0 : 0.0;
            if (fabs(s - expect) > 1e-3) return PS_NON_ORTHONORMAL_ROTATION;
        }
    double d = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
               m[2] * (m[3] * m[7] - m[4] * m[6]);
    if (d < 0.0) return PS_NON_ORTHONORMAL_ROTATION;
    return PS_OK;
}

} // namespace ps
