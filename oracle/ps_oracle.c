/*
 * ps_oracle.c — TEST INFRASTRUCTURE ONLY. A plain-C (C99, fp64) restatement of
 * the reference CPU rasterizer's hot path, used as the parity checker for the
 * B200 kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never does.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit for bit
 * against the reference itself compiled from /root/reference by
 * oracle/Makefile (oracle/_ref/libpolysplat_ref.so), and against the golden
 * fixtures in tests/golden/ generated from that build (tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Build with -ffp-contract=off: the reference's bits are
 * FMA-free (SURVEY finding 2), and the operation order below is the reference's.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <limits.h>

#include "../include/polysplat_b200.h"

static const char* g_err = "";
const char* or_last_error(void) { return g_err; }
#define FAIL(code, msg) do { g_err = (msg); return (code); } while (0)

/* ------------------------------------------------------------ value types */
/* geometry.hpp:42-56 Sym2 */
typedef struct { double xx, xy, yy; } sym2;
static double sym2_det(sym2 s) { return s.xx * s.yy - s.xy * s.xy; }
static sym2 sym2_inverse(sym2 s) {
    double d = sym2_det(s);
    sym2 r = {s.yy / d, -s.xy / d, s.xx / d};
    return r;
}
static double sym2_quadric(sym2 s, double dx, double dy) { /* geometry.hpp:53-55 */
    return s.xx * dx * dx + 2.0 * s.xy * dx * dy + s.yy * dy * dy;
}
/* std::min / std::max / std::clamp semantics (NaN-propagation order matters) */
static double std_max(double a, double b) { return (a < b) ? b : a; }
static double std_min(double a, double b) { return (b < a) ? b : a; }
static double std_clamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }
static int imax(int a, int b) { return (a < b) ? b : a; }
static int imin(int a, int b) { return (b < a) ? b : a; }
/* static_cast<int>(double) as compiled for x86-64 (cvttsd2si): out of range or
 * NaN gives INT_MIN. Written without UB. */
static int x86_cvtt_int(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
    return (int)v;
}

/* geometry.hpp:97-111 rotation_from_quat (row-major out[9]) */
static void rotation_from_quat(const double q0[4], double r[9]) {
    double w = q0[0], x = q0[1], y = q0[2], z = q0[3];
    double n = sqrt(w * w + x * x + y * y + z * z); /* geometry.hpp:33-38 */
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

/* projection.cpp:24-34 build_covariance3d: (R diag(s)) (R diag(s))^T via
 * Mat3::operator* (geometry.hpp:70-79: s = 0; s += a(i,k) b(k,j)) */
static void build_covariance3d(const double scale[3], const double quat[4], double c[9]) {
    double rs[9];
    rotation_from_quat(quat, rs);
    for (int i = 0; i < 3; ++i) {
        rs[i * 3 + 0] *= scale[0];
        rs[i * 3 + 1] *= scale[1];
        rs[i * 3 + 2] *= scale[2];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += rs[i * 3 + k] * rs[j * 3 + k];
            c[i * 3 + j] = s;
        }
}

/* ------------------------------------------------------------ kernel math */
/* kernel.cpp:16-20 */
static double horner(const double* c, int n, double x) {
    double p = c[n - 1];
    for (int i = n - 2; i >= 0; --i) p = p * x + c[i];
    return p;
}
/* kernel.cpp:22-27 */
static double horner_derivative(const double* c, int n, double x) {
    int d = n - 1;
    double p = c[d] * d;
    for (int i = d - 1; i >= 1; --i) p = p * x + c[i] * i;
    return p;
}
/* kernel.cpp:30-41 */
static double polish_root(const double* c, int n, double x) {
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
/* kernel.cpp:43-48 */
static int root_linear(double c0, double c1, double* out) {
    if (c1 == 0.0) FAIL(PS_NO_POSITIVE_ROOT, "constant polynomial has no root");
    double x = -c0 / c1;
    if (!(x > 0.0)) FAIL(PS_NO_POSITIVE_ROOT, "linear root is not positive");
    *out = x;
    return PS_OK;
}
/* kernel.cpp:50-68 */
static int root_quadratic(const double* c, double* out) {
    double c0 = c[0], c1 = c[1], c2 = c[2];
    double disc = c1 * c1 - 4.0 * c2 * c0;
    if (disc < 0.0) FAIL(PS_NO_POSITIVE_ROOT, "quadratic has no real root");
    double s = sqrt(disc);
    double q = -0.5 * (c1 + copysign(s, c1));
    double best = INFINITY;
    if (q != 0.0) {
        double r = q / c2;
        if (r > 0.0 && isfinite(r)) best = std_min(best, r);
        r = c0 / q;
        if (r > 0.0 && isfinite(r)) best = std_min(best, r);
    } else {
        FAIL(PS_NO_POSITIVE_ROOT, "quadratic touches zero only at x = 0");
    }
    if (!isfinite(best)) FAIL(PS_NO_POSITIVE_ROOT, "quadratic has no positive root");
    *out = best;
    return PS_OK;
}
/* kernel.cpp:70-109 */
static int root_cubic(const double* c, double* out) {
    const double pi = 3.141592653589793; /* std::numbers::pi */
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
    if (!isfinite(best)) FAIL(PS_NO_POSITIVE_ROOT, "cubic has no positive root");
    *out = best;
    return PS_OK;
}
/* kernel.cpp:117-135 */
int or_first_positive_root(const double* coeffs, int n, double* out) {
    if (n < 1 || !(coeffs[0] > 0.0))
        FAIL(PS_INVALID_ARGUMENT, "first_positive_root: polynomial must be positive at 0");
    if (n > 4) FAIL(PS_INVALID_ARGUMENT, "first_positive_root: order above 3 unsupported");
    while (n > 1 && fabs(coeffs[n - 1]) < 1e-12) --n;
    double x = 0.0;
    int st;
    switch (n) {
        case 1: FAIL(PS_NO_POSITIVE_ROOT, "constant polynomial has no root");
        case 2: st = root_linear(coeffs[0], coeffs[1], &x); break;
        case 3: st = root_quadratic(coeffs, &x); break;
        default: st = root_cubic(coeffs, &x); break;
    }
    if (st != PS_OK) return st;
    *out = polish_root(coeffs, n, x);
    return PS_OK;
}
/* kernel.cpp:162-172 */
double or_eval_kernel(const ps_kernel* k, double x) {
    switch (k->kind) {
        case PS_KERNEL_EXPONENTIAL: return exp(-0.5 * x);
        case PS_KERNEL_POLY_RELU: return std_max(horner(k->coeffs, k->order + 1, x), 0.0);
        case PS_KERNEL_POLY_PIECEWISE:
            return x < k->first_root ? horner(k->coeffs, k->order + 1, x) : 0.0;
    }
    return 0.0;
}
/* kernel.cpp:141-160 */
int or_make_polynomial_kernel(int kind, const double* coeffs, int n, ps_kernel* out) {
    if (kind == PS_KERNEL_EXPONENTIAL)
        FAIL(PS_INVALID_ARGUMENT, "make_polynomial_kernel: kind must be polynomial");
    int order = n - 1;
    if (order < 1 || order > 3) FAIL(PS_INVALID_ARGUMENT, "polynomial order must be in {1,2,3}");
    if (!(coeffs[0] > 0.0)) FAIL(PS_INVALID_ARGUMENT, "kernel must be positive at the splat center");
    if (order == 1 && !(coeffs[1] < 0.0))
        FAIL(PS_INVALID_ARGUMENT, "order-1 kernel must decay (c_1 < 0)");
    ps_kernel k;
    memset(&k, 0, sizeof k);
    k.kind = kind;
    k.order = order;
    int st = or_first_positive_root(coeffs, n, &k.first_root);
    if (st != PS_OK) return st;
    for (int i = 0; i < n; ++i) k.coeffs[i] = coeffs[i];
    if (fabs(horner(k.coeffs, n, k.first_root)) >= 1e-9) FAIL(PS_ERROR, "first root failed verification");
    *out = k;
    return PS_OK;
}
/* kernel.cpp:335-358 culling_radius */
int or_culling_radius(const ps_kernel* k, double o, double eps, double* radius, double* qroot,
                      int* aware) {
    if (!(o > 0.0) || o > 1.0) FAIL(PS_INVALID_ARGUMENT, "opacity must be in (0,1]");
    if (eps < 0.0) FAIL(PS_INVALID_ARGUMENT, "epsilon must be >= 0");
    if (k->kind == PS_KERNEL_EXPONENTIAL) {
        if (eps == 0.0) FAIL(PS_EPSILON_ZERO_UNBOUNDED, "exponential kernel has unbounded support at epsilon 0");
        if (!(o > eps)) FAIL(PS_FULLY_CULLED, "opacity below cutoff");
        double x = 2.0 * log(o / eps);
        *radius = sqrt(x); *qroot = x; *aware = 1;
        return PS_OK;
    }
    if (!(o * k->coeffs[0] > eps)) FAIL(PS_FULLY_CULLED, "opacity below cutoff");
    double x;
    if (eps == 0.0) {
        x = k->first_root;
    } else {
        double shifted[4];
        int n = k->order + 1;
        for (int i = 0; i < n; ++i) shifted[i] = k->coeffs[i];
        shifted[0] -= eps / o;
        int st = or_first_positive_root(shifted, n, &x);
        if (st != PS_OK) return st;
    }
    *radius = sqrt(x); *qroot = x; *aware = eps > 0.0;
    return PS_OK;
}

/* ------------------------------------------------------------ validation */
/* raster.cpp:13-23 RasterConfig::validate */
int or_validate_config(const ps_config* c) {
    if (c->tile_size < 1) FAIL(PS_INVALID_ARGUMENT, "tile_size must be >= 1");
    if (!(c->epsilon > 0.0) || !(c->epsilon < 1.0)) FAIL(PS_INVALID_ARGUMENT, "epsilon must be in (0,1)");
    if (!(c->transmittance_floor >= 0.0) || !(c->transmittance_floor < 1.0))
        FAIL(PS_INVALID_ARGUMENT, "transmittance_floor must be in [0,1)");
    const ps_kernel* bk = c->has_culling_kernel ? &c->culling_kernel : &c->kernel;
    if (c->culling_mode == PS_CULL_ZERO_CROSSING && bk->kind == PS_KERNEL_EXPONENTIAL)
        FAIL(PS_INVALID_ARGUMENT, "zero-crossing culling requires a polynomial kernel");
    if (c->v_dilation < 0.0) FAIL(PS_INVALID_ARGUMENT, "v_dilation must be >= 0");
    if (c->thread_count < 0) FAIL(PS_INVALID_ARGUMENT, "thread_count must be >= 0");
    return PS_OK;
}
/* projection.cpp:10-22 Camera::validate */
int or_validate_camera(const ps_camera* cam) {
    if (cam->width <= 0 || cam->height <= 0) FAIL(PS_INVALID_ARGUMENT, "camera size must be positive");
    if (!(cam->fx > 0.0) || !(cam->fy > 0.0)) FAIL(PS_INVALID_ARGUMENT, "focal lengths must be positive");
    const double* m = cam->rotation;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0; /* (R^T R)(i,j) = sum_k R(k,i) R(k,j) */
            for (int k = 0; k < 3; ++k) s += m[k * 3 + i] * m[k * 3 + j];
            double expect = (i == j) ? 1.0 : 0.0;
            if (fabs(s - expect) > 1e-3) FAIL(PS_NON_ORTHONORMAL_ROTATION, "camera rotation is not orthonormal");
        }
    double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                 m[2] * (m[3] * m[7] - m[4] * m[6]); /* geometry.hpp:86-89 */
    if (det < 0.0) FAIL(PS_NON_ORTHONORMAL_ROTATION, "camera rotation is a reflection");
    return PS_OK;
}

/* ------------------------------------------------------------ projection */
typedef struct {
    double mx, my;          /* mean2d */
    sym2 conic, cov_aa;
    double depth, opacity_eff;
    double color[3];
    double radius_sigma, quadric_root;
    uint32_t index;
} prepared_t;

static const double kSH0 = 0.28209479177387814;
static const double kSH1 = 0.4886025119029199;
static const double kSH2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                               -1.0925484305920792, 0.5462742152960396};
static const double kSH3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                               0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                               -0.5900435899266435};

/* projection.cpp:93-116 eval_sh_color; sh = 16 x (x,y,z) doubles */
static void eval_sh_color(const double* sh, const double d[3], int degree, double out[3]) {
    for (int ch = 0; ch < 3; ++ch) {
        const double dx = d[0], dy = d[1], dz = d[2];
#define SH(k) sh[3 * (k) + ch]
        double c = SH(0) * kSH0;
        if (degree >= 1) c = c - SH(1) * (kSH1 * dy) + SH(2) * (kSH1 * dz) - SH(3) * (kSH1 * dx);
        if (degree >= 2) {
            double xx = dx * dx, yy = dy * dy, zz = dz * dz;
            double xy = dx * dy, yz = dy * dz, xz = dx * dz;
            c = c + SH(4) * (kSH2[0] * xy) + SH(5) * (kSH2[1] * yz) +
                SH(6) * (kSH2[2] * (2.0 * zz - xx - yy)) + SH(7) * (kSH2[3] * xz) +
                SH(8) * (kSH2[4] * (xx - yy));
            if (degree >= 3) {
                c = c + SH(9) * (kSH3[0] * dy * (3.0 * xx - yy)) + SH(10) * (kSH3[1] * xy * dz) +
                    SH(11) * (kSH3[2] * dy * (4.0 * zz - xx - yy)) +
                    SH(12) * (kSH3[3] * dz * (2.0 * zz - 3.0 * xx - 3.0 * yy)) +
                    SH(13) * (kSH3[4] * dx * (4.0 * zz - xx - yy)) +
                    SH(14) * (kSH3[5] * dz * (xx - yy)) + SH(15) * (kSH3[6] * dx * (xx - yy));
            }
        }
#undef SH
        out[ch] = std_max(c + 0.5, 0.0);
    }
}

/* projection.cpp:36-79 project_splat. Returns 1 visible, 0 near-plane culled,
 * or a negative status (-PS_DEGENERATE_COVARIANCE). */
static int project_splat(const double* s, const ps_camera* cam, double v, int sh_degree,
                         prepared_t* out) {
    const double* R = cam->rotation;
    const double* t = cam->translation;
    const double mean[3] = {s[0], s[1], s[2]};
    /* Mat3 * Vec3 (geometry.hpp:65-69), then + translation */
    double px = R[0] * mean[0] + R[1] * mean[1] + R[2] * mean[2];
    double py = R[3] * mean[0] + R[4] * mean[1] + R[5] * mean[2];
    double pz = R[6] * mean[0] + R[7] * mean[1] + R[8] * mean[2];
    px = px + t[0]; py = py + t[1]; pz = pz + t[2];
    if (pz <= 0.2) return 0; /* kNearPlane, projection.hpp:44 */

    double inv_z = 1.0 / pz;
    out->mx = cam->fx * px * inv_z + cam->cx;
    out->my = cam->fy * py * inv_z + cam->cy;
    double jr0[3] = {cam->fx * inv_z, 0.0, -cam->fx * px * inv_z * inv_z};
    double jr1[3] = {0.0, cam->fy * inv_z, -cam->fy * py * inv_z * inv_z};
    double m0[3], m1[3];
    for (int j = 0; j < 3; ++j) {
        m0[j] = jr0[0] * R[0 * 3 + j] + jr0[1] * R[1 * 3 + j] + jr0[2] * R[2 * 3 + j];
        m1[j] = jr1[0] * R[0 * 3 + j] + jr1[1] * R[1 * 3 + j] + jr1[2] * R[2 * 3 + j];
    }
    double cov3d[9];
    build_covariance3d(s + 3, s + 6, cov3d);
    double t0[3], t1[3];
    for (int j = 0; j < 3; ++j) {
        t0[j] = m0[0] * cov3d[0 * 3 + j] + m0[1] * cov3d[1 * 3 + j] + m0[2] * cov3d[2 * 3 + j];
        t1[j] = m1[0] * cov3d[0 * 3 + j] + m1[1] * cov3d[1 * 3 + j] + m1[2] * cov3d[2 * 3 + j];
    }
    sym2 cov;
    cov.xx = t0[0] * m0[0] + t0[1] * m0[1] + t0[2] * m0[2];
    cov.xy = t0[0] * m1[0] + t0[1] * m1[1] + t0[2] * m1[2];
    cov.yy = t1[0] * m1[0] + t1[1] * m1[1] + t1[2] * m1[2];
    sym2 cov_aa = {cov.xx + v, cov.xy, cov.yy + v};
    double det_aa = sym2_det(cov_aa);
    if (det_aa <= 1e-12) { g_err = "dilated 2D covariance is singular"; return -PS_DEGENERATE_COVARIANCE; }
    double det = sym2_det(cov);
    double ratio = det > 0.0 ? sqrt(det / det_aa) : 0.0;
    out->cov_aa = cov_aa;
    out->conic = sym2_inverse(cov_aa);
    out->depth = pz;
    out->opacity_eff = s[10] * ratio;
    /* camera position = R^T t * -1 (projection.hpp:29, geometry.hpp:90-94) */
    double cpx = (R[0] * t[0] + R[3] * t[1] + R[6] * t[2]) * -1.0;
    double cpy = (R[1] * t[0] + R[4] * t[1] + R[7] * t[2]) * -1.0;
    double cpz = (R[2] * t[0] + R[5] * t[1] + R[8] * t[2]) * -1.0;
    double d[3] = {mean[0] - cpx, mean[1] - cpy, mean[2] - cpz};
    double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]); /* geometry.hpp:22-26 */
    if (n > 0.0) { d[0] = d[0] / n; d[1] = d[1] / n; d[2] = d[2] / n; }
    else { d[0] = 0.0; d[1] = 0.0; d[2] = 0.0; }
    eval_sh_color(s + 11, d, sh_degree, out->color);
    return 1;
}

/* ------------------------------------------------------------ raster helpers */
static const double kBoundSlack = 1e-7; /* raster.cpp:40 */

/* raster.cpp:50-69 culling_bound_for (+ widen raster.cpp:42-46).
 * Returns 1 bound set, 0 nullopt, negative status on error. */
static int culling_bound_for(const ps_config* cfg, double o, double* radius, double* qroot) {
    if (!(o > 0.0)) return 0;
    const ps_kernel* bk = cfg->has_culling_kernel ? &cfg->culling_kernel : &cfg->kernel;
    double x;
    switch (cfg->culling_mode) {
        case PS_CULL_STOP_THE_POP:
            if (!(o > cfg->epsilon)) return 0;
            x = 2.0 * log(o / cfg->epsilon);
            break;
        case PS_CULL_ZERO_CROSSING:
            x = bk->first_root;
            break;
        case PS_CULL_OPACITY_AWARE: {
            /* kernel.cpp:360-369 try_culling_radius */
            if (bk->kind == PS_KERNEL_EXPONENTIAL && cfg->epsilon == 0.0) {
                g_err = "exponential kernel has unbounded support at epsilon 0";
                return -PS_EPSILON_ZERO_UNBOUNDED;
            }
            double r; int aware;
            int st = or_culling_radius(bk, o, cfg->epsilon, &r, &x, &aware);
            if (st == PS_FULLY_CULLED) return 0;
            if (st != PS_OK) return -st;
            break;
        }
        default: return 0;
    }
    *qroot = x + kBoundSlack;
    *radius = sqrt(*qroot);
    return 1;
}

/* raster.cpp:71-86 tile_rect; returns 1 and the inclusive rect, 0 if off screen */
static int tile_rect(const prepared_t* p, int ts, int width, int height, int r[4]) {
    double hx = p->radius_sigma * sqrt(std_max(p->cov_aa.xx, 0.0));
    double hy = p->radius_sigma * sqrt(std_max(p->cov_aa.yy, 0.0));
    int tiles_x = (width + ts - 1) / ts;
    int tiles_y = (height + ts - 1) / ts;
    int x0 = x86_cvtt_int(floor((p->mx - hx) / ts));
    int x1 = x86_cvtt_int(floor((p->mx + hx) / ts));
    int y0 = x86_cvtt_int(floor((p->my - hy) / ts));
    int y1 = x86_cvtt_int(floor((p->my + hy) / ts));
    x0 = imax(x0, 0);
    y0 = imax(y0, 0);
    x1 = imin(x1, tiles_x - 1);
    y1 = imin(y1, tiles_y - 1);
    if (x0 > x1 || y0 > y1) return 0;
    r[0] = x0; r[1] = y0; r[2] = x1; r[3] = y1;
    return 1;
}

/* raster.cpp:103-124 min_quadric_over_box; box = tile_pixel_box raster.cpp:97-101 */
double or_min_quadric_over_box(const double conic[3], double mx, double my, const double box[4]) {
    sym2 cn = {conic[0], conic[1], conic[2]};
    double lx = box[0] - mx, hx = box[2] - mx;
    double ly = box[1] - my, hy = box[3] - my;
    if (lx <= 0.0 && hx >= 0.0 && ly <= 0.0 && hy >= 0.0) return 0.0;
    double a = cn.xx, b = cn.xy, c = cn.yy;
    double dy, dx, m, e;
    dy = std_clamp(c != 0.0 ? -b * lx / c : ly, ly, hy);
    m = sym2_quadric(cn, lx, dy);
    dy = std_clamp(c != 0.0 ? -b * hx / c : ly, ly, hy);
    e = sym2_quadric(cn, hx, dy);
    m = std_min(m, e);
    dx = std_clamp(a != 0.0 ? -b * ly / a : lx, lx, hx);
    e = sym2_quadric(cn, dx, ly);
    m = std_min(m, e);
    dx = std_clamp(a != 0.0 ? -b * hy / a : lx, lx, hx);
    e = sym2_quadric(cn, dx, hy);
    m = std_min(m, e);
    return m;
}
static void tile_pixel_box(int tx, int ty, int ts, double box[4]) {
    double x0 = tx * (double)ts + 0.5;
    double y0 = ty * (double)ts + 0.5;
    box[0] = x0; box[1] = y0; box[2] = x0 + ts - 1; box[3] = y0 + ts - 1;
}
/* raster.cpp:126-128 */
static int tight_tile_test(const prepared_t* p, int tx, int ty, int ts) {
    double box[4], conic[3] = {p->conic.xx, p->conic.xy, p->conic.yy};
    tile_pixel_box(tx, ty, ts, box);
    return or_min_quadric_over_box(conic, p->mx, p->my, box) <= p->quadric_root;
}

/* ------------------------------------------------------------ pipeline */
static int cmp_prepared(const void* a, const void* b) { /* raster.cpp:172-175 */
    const prepared_t* x = (const prepared_t*)a;
    const prepared_t* y = (const prepared_t*)b;
    if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
    return x->index < y->index ? -1 : (x->index > y->index ? 1 : 0);
}

/* raster.cpp:132-177 prepare_splats (serial restatement; the reference's OMP
 * loop is per-splat independent, so order of evaluation does not matter). */
static int prepare(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                   prepared_t** out, int64_t* n_out, ps_counters* ctr) {
    ctr->splats_submitted += (uint64_t)n;
    prepared_t* list = (prepared_t*)malloc(sizeof(prepared_t) * (size_t)(n > 0 ? n : 1));
    int64_t v = 0;
    for (int64_t i = 0; i < n; ++i) {
        prepared_t p;
        memset(&p, 0, sizeof p);
        int st = project_splat(splats + i * PS_SPLAT3D_DOUBLES, cam, cfg->v_dilation, cfg->sh_degree, &p);
        if (st < 0) { free(list); return -st; }
        if (st == 0) { ++ctr->splats_frustum_culled; continue; }          /* kFrustum */
        int b = culling_bound_for(cfg, p.opacity_eff, &p.radius_sigma, &p.quadric_root);
        if (b < 0) { free(list); return -b; }
        if (b == 0) continue;                                              /* kBelowEpsilon: uncounted */
        p.index = (uint32_t)i;
        int r[4];
        if (tile_rect(&p, cfg->tile_size, cam->width, cam->height, r)) list[v++] = p;
        else ++ctr->splats_frustum_culled;                                 /* off screen */
    }
    qsort(list, (size_t)v, sizeof(prepared_t), cmp_prepared);
    *out = list;
    *n_out = v;
    return PS_OK;
}

/* raster.cpp:186-208 bin_splats as CSR (counting pass, then fill in k order) */
static void bin(const prepared_t* prep, int64_t v, const ps_config* cfg, int width, int height,
                uint32_t** offsets_out, uint32_t** bins_out, ps_counters* ctr) {
    int ts = cfg->tile_size;
    int tiles_x = (width + ts - 1) / ts, tiles_y = (height + ts - 1) / ts;
    int64_t nt = (int64_t)tiles_x * tiles_y;
    uint32_t* off = (uint32_t*)calloc((size_t)nt + 1, sizeof(uint32_t));
    for (int pass = 0; pass < 2; ++pass) {
        uint32_t* bins = pass ? (uint32_t*)malloc(sizeof(uint32_t) * (off[nt] ? off[nt] : 1)) : NULL;
        uint32_t* cur = pass ? (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nt) : NULL;
        if (pass) memcpy(cur, off, sizeof(uint32_t) * (size_t)nt);
        for (int64_t k = 0; k < v; ++k) {
            int r[4];
            if (!tile_rect(&prep[k], ts, width, height, r)) continue;
            if (!pass) ctr->tile_pairs_coarse += (uint64_t)(r[2] - r[0] + 1) * (uint64_t)(r[3] - r[1] + 1);
            for (int ty = r[1]; ty <= r[3]; ++ty)
                for (int tx = r[0]; tx <= r[2]; ++tx)
                    if (tight_tile_test(&prep[k], tx, ty, ts)) {
                        int64_t t = (int64_t)ty * tiles_x + tx;
                        if (!pass) { ++off[t + 1]; ++ctr->tile_pairs_after_tight_test; }
                        else bins[cur[t]++] = (uint32_t)k;
                    }
        }
        if (!pass) { for (int64_t t = 0; t < nt; ++t) off[t + 1] += off[t]; }
        else { free(cur); *bins_out = bins; }
    }
    *offsets_out = off;
}

static int check_inputs(const ps_camera* cam, const ps_config* cfg) {
    int st = or_validate_config(cfg);
    if (st != PS_OK) return st;
    return or_validate_camera(cam);
}

/* raster.cpp:212-308 render (tile loop run serially; each tile is independent) */
int or_render(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
              double* rgb, double* trans_out, ps_counters* counters) {
    int st = check_inputs(cam, cfg);
    if (st != PS_OK) return st;
    ps_counters ctr;
    memset(&ctr, 0, sizeof ctr);
    prepared_t* prep; int64_t v;
    st = prepare(splats, n, cam, cfg, &prep, &v, &ctr);
    if (st != PS_OK) return st;
    uint32_t *off, *bins;
    bin(prep, v, cfg, cam->width, cam->height, &off, &bins, &ctr);

    const int T = cfg->tile_size, W = cam->width, H = cam->height;
    const int tiles_x = (W + T - 1) / T, tiles_y = (H + T - 1) / T;
    double* trans = (double*)malloc(sizeof(double) * (size_t)T * T);
    double* accum = (double*)malloc(sizeof(double) * 3 * (size_t)T * T);
    unsigned char* done = (unsigned char*)malloc((size_t)T * T);
    for (int tile = 0; tile < tiles_x * tiles_y; ++tile) {
        int tx = tile % tiles_x, ty = tile / tiles_x;
        int px0 = tx * T, py0 = ty * T;
        int px1 = imin(px0 + T, W), py1 = imin(py0 + T, H);
        int tw = px1 - px0, th = py1 - py0, n_px = tw * th;
        if (n_px <= 0) continue;
        for (int i = 0; i < n_px; ++i) { trans[i] = 1.0; accum[3 * i] = accum[3 * i + 1] = accum[3 * i + 2] = 0.0; done[i] = 0; }
        int remaining = n_px;
        uint64_t evals = 0, blended = 0;
        for (uint32_t j = off[tile]; j < off[tile + 1]; ++j) {
            if (remaining == 0) break;
            const prepared_t* p = &prep[bins[j]];
            double a = p->conic.xx, b = p->conic.xy, c = p->conic.yy;
            double mx = p->mx, my = p->my;
            double cr = p->color[0], cg = p->color[1], cb = p->color[2];
            if (cfg->clamp_before_blend) {
                cr = std_clamp(cr, 0.0, 1.0); cg = std_clamp(cg, 0.0, 1.0); cb = std_clamp(cb, 0.0, 1.0);
            }
            for (int iy = 0; iy < th; ++iy) {
                double dy = py0 + iy + 0.5 - my;
                for (int ix = 0; ix < tw; ++ix) {
                    int idx = iy * tw + ix;
                    if (done[idx]) continue;
                    double dx = px0 + ix + 0.5 - mx;
                    double q = a * dx * dx + 2.0 * b * dx * dy + c * dy * dy;
                    ++evals;
                    double alpha = std_min(0.999, p->opacity_eff * or_eval_kernel(&cfg->kernel, q));
                    if (alpha < cfg->epsilon) continue;
                    double test_t = trans[idx] * (1.0 - alpha);
                    if (test_t < cfg->transmittance_floor) { done[idx] = 1; --remaining; continue; }
                    double w = alpha * trans[idx];
                    accum[3 * idx + 0] += cr * w;
                    accum[3 * idx + 1] += cg * w;
                    accum[3 * idx + 2] += cb * w;
                    trans[idx] = test_t;
                    ++blended;
                }
            }
        }
        for (int iy = 0; iy < th; ++iy)
            for (int ix = 0; ix < tw; ++ix) {
                int idx = iy * tw + ix;
                size_t o = (size_t)(py0 + iy) * W + (px0 + ix);
                if (trans_out) trans_out[o] = trans[idx];
                if (rgb) { rgb[3 * o] = accum[3 * idx]; rgb[3 * o + 1] = accum[3 * idx + 1]; rgb[3 * o + 2] = accum[3 * idx + 2]; }
            }
        ctr.kernel_evaluations += evals;
        ctr.fragments_blended += blended;
    }
    free(trans); free(accum); free(done); free(off); free(bins); free(prep);
    if (counters) *counters = ctr;
    return PS_OK;
}

/* reference.cpp:8-59 render_serial: per pixel over all prepared splats,
 * re-deriving tile membership. O(pixels x V): small inputs only. */
int or_render_serial(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                     double* rgb, double* trans_out) {
    int st = check_inputs(cam, cfg);
    if (st != PS_OK) return st;
    ps_counters unused;
    memset(&unused, 0, sizeof unused);
    prepared_t* prep; int64_t v;
    st = prepare(splats, n, cam, cfg, &prep, &v, &unused);
    if (st != PS_OK) return st;
    const int T = cfg->tile_size;
    for (int py = 0; py < cam->height; ++py)
        for (int px = 0; px < cam->width; ++px) {
            int tx = px / T, ty = py / T;
            double trans = 1.0, r = 0.0, g = 0.0, b = 0.0;
            for (int64_t k = 0; k < v; ++k) {
                const prepared_t* p = &prep[k];
                int rc[4];
                if (!tile_rect(p, T, cam->width, cam->height, rc) || tx < rc[0] || tx > rc[2] ||
                    ty < rc[1] || ty > rc[3])
                    continue;
                if (!tight_tile_test(p, tx, ty, T)) continue;
                double dx = px + 0.5 - p->mx;
                double dy = py + 0.5 - p->my;
                double q = sym2_quadric(p->conic, dx, dy);
                double alpha = std_min(0.999, p->opacity_eff * or_eval_kernel(&cfg->kernel, q));
                if (alpha < cfg->epsilon) continue;
                double test_t = trans * (1.0 - alpha);
                if (test_t < cfg->transmittance_floor) break;
                double cr = p->color[0], cg = p->color[1], cb = p->color[2];
                if (cfg->clamp_before_blend) {
                    cr = std_clamp(cr, 0.0, 1.0); cg = std_clamp(cg, 0.0, 1.0); cb = std_clamp(cb, 0.0, 1.0);
                }
                double w = alpha * trans;
                r += cr * w; g += cg * w; b += cb * w;
                trans = test_t;
            }
            size_t o = (size_t)py * cam->width + px;
            trans_out[o] = trans;
            rgb[3 * o] = r; rgb[3 * o + 1] = g; rgb[3 * o + 2] = b;
        }
    free(prep);
    return PS_OK;
}

/* raster.cpp:310-318 count_pairs */
int or_count_pairs(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                   ps_counters* counters) {
    int st = check_inputs(cam, cfg);
    if (st != PS_OK) return st;
    ps_counters ctr;
    memset(&ctr, 0, sizeof ctr);
    prepared_t* prep; int64_t v;
    st = prepare(splats, n, cam, cfg, &prep, &v, &ctr);
    if (st != PS_OK) return st;
    uint32_t *off, *bins;
    bin(prep, v, cfg, cam->width, cam->height, &off, &bins, &ctr);
    free(off); free(bins); free(prep);
    *counters = ctr;
    return PS_OK;
}

/* prepare_splats as SoA (any pointer may be NULL; color is fp64 here) */
int or_prepare(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
               int64_t capacity, uint32_t* index, double* depth, double* mean2d, double* conic,
               double* cov_aa, double* opacity_eff, double* color, double* radius_sigma,
               double* quadric_root, int64_t* n_out, ps_counters* counters) {
    ps_counters ctr;
    memset(&ctr, 0, sizeof ctr);
    prepared_t* prep; int64_t v;
    int st = prepare(splats, n, cam, cfg, &prep, &v, &ctr);
    if (st != PS_OK) return st;
    *n_out = v;
    if (counters) *counters = ctr;
    if (v > capacity) { free(prep); FAIL(PS_INVALID_ARGUMENT, "capacity too small"); }
    for (int64_t k = 0; k < v; ++k) {
        const prepared_t* p = &prep[k];
        if (index) index[k] = p->index;
        if (depth) depth[k] = p->depth;
        if (mean2d) { mean2d[2 * k] = p->mx; mean2d[2 * k + 1] = p->my; }
        if (conic) { conic[3 * k] = p->conic.xx; conic[3 * k + 1] = p->conic.xy; conic[3 * k + 2] = p->conic.yy; }
        if (cov_aa) { cov_aa[3 * k] = p->cov_aa.xx; cov_aa[3 * k + 1] = p->cov_aa.xy; cov_aa[3 * k + 2] = p->cov_aa.yy; }
        if (opacity_eff) opacity_eff[k] = p->opacity_eff;
        if (color) { color[3 * k] = p->color[0]; color[3 * k + 1] = p->color[1]; color[3 * k + 2] = p->color[2]; }
        if (radius_sigma) radius_sigma[k] = p->radius_sigma;
        if (quadric_root) quadric_root[k] = p->quadric_root;
    }
    free(prep);
    return PS_OK;
}

/* per-tile lists (bins) as CSR of original splat indices */
int or_tile_lists(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                  int64_t capacity, uint32_t* tile_offsets, uint32_t* splat_index,
                  int64_t* n_pairs, ps_counters* counters) {
    int st = check_inputs(cam, cfg);
    if (st != PS_OK) return st;
    ps_counters ctr;
    memset(&ctr, 0, sizeof ctr);
    prepared_t* prep; int64_t v;
    st = prepare(splats, n, cam, cfg, &prep, &v, &ctr);
    if (st != PS_OK) return st;
    uint32_t *off, *bins;
    bin(prep, v, cfg, cam->width, cam->height, &off, &bins, &ctr);
    int ts = cfg->tile_size;
    int64_t nt = (int64_t)((cam->width + ts - 1) / ts) * ((cam->height + ts - 1) / ts);
    *n_pairs = off[nt];
    if (counters) *counters = ctr;
    if (!tile_offsets && !splat_index) { free(off); free(bins); free(prep); return PS_OK; } /* size query */
    if ((int64_t)off[nt] > capacity) { free(off); free(bins); free(prep); FAIL(PS_INVALID_ARGUMENT, "capacity too small"); }
    if (tile_offsets) memcpy(tile_offsets, off, sizeof(uint32_t) * (size_t)(nt + 1));
    if (splat_index)
        for (uint32_t j = 0; j < off[nt]; ++j) splat_index[j] = prep[bins[j]].index;
    free(off); free(bins); free(prep);
    return PS_OK;
}

/* projection.cpp:36-79 for one Splat3D (KAT helper); returns 1/0 or -status */
int or_project_splat(const double* splat, const ps_camera* cam, double v, int sh_degree,
                     double* out14) {
    prepared_t p;
    memset(&p, 0, sizeof p);
    int st = project_splat(splat, cam, v, sh_degree, &p);
    if (st == 1) {
        double o[14] = {p.mx, p.my, p.conic.xx, p.conic.xy, p.conic.yy, p.cov_aa.xx, p.cov_aa.xy,
                        p.cov_aa.yy, p.depth, p.opacity_eff, p.color[0], p.color[1], p.color[2], 0.0};
        memcpy(out14, o, sizeof o);
    }
    return st;
}
