// hostmath.cpp — the exact fp64 kernel math of exact_math.cuh compiled for the
// host (g++ -ffp-contract=off), exported through the C ABI: kernel
// construction (kernel.cpp:137-160), roots (kernel.cpp:117-135), culling radius
// (kernel.cpp:335-358), eval (kernel.cpp:162-172) and config/camera validation
// (raster.cpp:13-23, projection.cpp:10-22). These are API helpers, not a
// render path: rendering always runs on the device.
#include <cmath>
#include <cstring>
#include <string>

namespace ps {
using std::acos;
using std::cbrt;
using std::copysign;
using std::cos;
using std::exp;
using std::fabs;
using std::floor;
using std::isfinite;
using std::log;
using std::sqrt;
} // namespace ps

#include "exact_math.cuh"

namespace ps {

extern thread_local std::string g_free_error;

int host_validate_config(const ps_config& c) { return validate_config(c); }

// first_positive_root's degenerate-leading-coefficient trim (kernel.cpp:124):
// the coefficient count the root solver actually uses.
int host_effective_terms(const ps_kernel& k) {
    int n = k.order + 1;
    while (n > 1 && std::fabs(k.coeffs[n - 1]) < 1e-12) --n;
    return n;
}

// Camera::position() = R^T t * -1 (projection.hpp:29, geometry.hpp:90-94).
void host_camera_position(const ps_camera& cam, double out[3]) {
    const double* R = cam.rotation;
    const double* t = cam.translation;
    out[0] = (R[0] * t[0] + R[3] * t[1] + R[6] * t[2]) * -1.0;
    out[1] = (R[1] * t[0] + R[4] * t[1] + R[7] * t[2]) * -1.0;
    out[2] = (R[2] * t[0] + R[5] * t[1] + R[8] * t[2]) * -1.0;
}
int host_validate_camera(const ps_camera& c) { return validate_camera(c); }

// Blend-threshold mode (see blend.cu): the quadric-space skip test is exact iff
// alpha = min(.999, o k(q)) >= eps is equivalent to q <= q*(o), i.e. k is
// non-increasing in q (over [0, inf) for ReLU kernels, over [0, first_root)
// for piecewise ones). p'(q) = c1 + 2 c2 q + 3 c3 q^2 is checked analytically.
int host_kernel_threshold_mode(const ps_kernel& k) {
    if (k.kind == PS_KERNEL_EXPONENTIAL) return 0;
    const double d0 = k.order >= 1 ? k.coeffs[1] : 0.0;
    const double d1 = k.order >= 2 ? 2.0 * k.coeffs[2] : 0.0;
    const double d2 = k.order >= 3 ? 3.0 * k.coeffs[3] : 0.0;
    auto dval = [&](double q) { return d0 + d1 * q + d2 * q * q; };
    if (d0 > 0.0) return 1;
    if (k.kind == PS_KERNEL_POLY_RELU) {
        if (d2 > 0.0) return 1;
        if (d2 == 0.0) return d1 <= 0.0 ? 0 : 1;
        const double qv = -d1 / (2.0 * d2);
        return (qv > 0.0 && dval(qv) > 0.0) ? 1 : 0;
    }
    // piecewise: only [0, first_root) matters
    const double R = k.first_root;
    if (!(R > 0.0) || !std::isfinite(R)) return 1;
    if (dval(R) > 0.0) return 1;
    if (d2 != 0.0) {
        const double qv = -d1 / (2.0 * d2);
        if (qv > 0.0 && qv < R && dval(qv) > 0.0) return 1;
    }
    return 0;
}

// Quadric-threshold mode, polynomial kernel: the reference decides alpha >= eps
// from o p(q) evaluated in fp64 (Horner, order + 1 roundings, plus the eps / o
// division of the shifted root problem), so near the threshold its decision
// can differ from q <= q* by at most 8 u64 (sum |c_j| q^j + 1) / |p'(q)| in q.
// Over q in [0, R] (R: first root of p; q* < R) that is bounded by this
// constant (infinite when p' vanishes on [0, R]).
double host_root_slack(const ps_kernel& k) {
    if (k.kind == PS_KERNEL_EXPONENTIAL) return 0.0;
    const double R = k.first_root;
    if (!(R > 0.0) || !std::isfinite(R)) return INFINITY;
    const double d0 = k.order >= 1 ? k.coeffs[1] : 0.0;
    const double d1 = k.order >= 2 ? 2.0 * k.coeffs[2] : 0.0;
    const double d2 = k.order >= 3 ? 3.0 * k.coeffs[3] : 0.0;
    auto dval = [&](double q) { return d0 + d1 * q + d2 * q * q; };
    double lo = std::fmin(std::fabs(dval(0.0)), std::fabs(dval(R)));
    if (dval(0.0) * dval(R) <= 0.0) lo = 0.0;
    if (d2 != 0.0) {
        const double qv = -d1 / (2.0 * d2);
        if (qv > 0.0 && qv < R) {
            if (dval(qv) * dval(0.0) <= 0.0) lo = 0.0;
            lo = std::fmin(lo, std::fabs(dval(qv)));
        }
    }
    if (!(lo > 0.0)) return INFINITY;
    double mag = 0.0, qp = 1.0;
    for (int j = 0; j <= k.order; ++j) {
        mag += std::fabs(k.coeffs[j]) * qp;
        qp *= R;
    }
    return 1.1 * 8.0 * 1.1102230246251565e-16 * (mag + 1.0) / lo;
}

} // namespace ps

using namespace ps;

namespace {
int fail(int code, const char* msg) {
    g_free_error = msg;
    return code;
}
} // namespace

extern "C" {

ps_kernel ps_make_exponential_kernel(void) {
    ps_kernel k;
    std::memset(&k, 0, sizeof k);
    k.kind = PS_KERNEL_EXPONENTIAL;
    k.first_root = INFINITY;
    return k;
}

ps_config ps_default_config(void) {
    ps_config c;
    std::memset(&c, 0, sizeof c);
    c.tile_size = 16;
    c.culling_mode = PS_CULL_STOP_THE_POP;
    c.epsilon = 1.0 / 255.0;
    c.transmittance_floor = 1e-4;
    c.kernel = ps_make_exponential_kernel();
    c.culling_kernel = ps_make_exponential_kernel();
    c.v_dilation = 0.3;
    c.sh_degree = 3;
    return c;
}

int ps_first_positive_root(const double* coeffs, int n, double* out) {
    if (!coeffs || !out) return fail(PS_INVALID_ARGUMENT, "null argument");
    if (n < 1 || !(coeffs[0] > 0.0)) return fail(PS_INVALID_ARGUMENT, "first_positive_root: polynomial must be positive at 0");
    if (n > 4) return fail(PS_INVALID_ARGUMENT, "first_positive_root: order above 3 unsupported");
    double x = 0.0;
    int st = first_positive_root(coeffs, n, x);
    if (st != PS_OK) return fail(st, "polynomial has no positive root");
    *out = x;
    return PS_OK;
}

int ps_make_polynomial_kernel(int kind, const double* coeffs, int n, ps_kernel* out) {
    if (!out || !coeffs) return fail(PS_INVALID_ARGUMENT, "null argument");
    if (kind == PS_KERNEL_EXPONENTIAL) return fail(PS_INVALID_ARGUMENT, "make_polynomial_kernel: kind must be polynomial");
    if (kind != PS_KERNEL_POLY_RELU && kind != PS_KERNEL_POLY_PIECEWISE) return fail(PS_INVALID_ARGUMENT, "unknown kernel kind");
    const int order = n - 1;
    if (order < 1 || order > 3) return fail(PS_INVALID_ARGUMENT, "polynomial order must be in {1,2,3}");
    if (!(coeffs[0] > 0.0)) return fail(PS_INVALID_ARGUMENT, "kernel must be positive at the splat center");
    if (order == 1 && !(coeffs[1] < 0.0)) return fail(PS_INVALID_ARGUMENT, "order-1 kernel must decay (c_1 < 0)");
    ps_kernel k;
    std::memset(&k, 0, sizeof k);
    k.kind = kind;
    k.order = order;
    int st = ps_first_positive_root(coeffs, n, &k.first_root);
    if (st != PS_OK) return st;
    for (int i = 0; i < n; ++i) k.coeffs[i] = coeffs[i];
    if (std::fabs(horner(k.coeffs, n, k.first_root)) >= 1e-9) return fail(PS_ERROR, "first root failed verification");
    *out = k;
    return PS_OK;
}

int ps_culling_radius(const ps_kernel* k, double o, double eps, double* radius, double* qroot, int* aware) {
    if (!k || !radius || !qroot || !aware) return fail(PS_INVALID_ARGUMENT, "null argument");
    double x = 0.0;
    int st = culling_root(*k, o, eps, x);
    if (st != PS_OK) {
        const char* msg = st == PS_FULLY_CULLED ? "opacity below cutoff"
                          : st == PS_EPSILON_ZERO_UNBOUNDED ? "exponential kernel has unbounded support at epsilon 0"
                          : st == PS_NO_POSITIVE_ROOT ? "polynomial has no positive root"
                                                      : "opacity must be in (0,1] and epsilon >= 0";
        return fail(st, msg);
    }
    *qroot = x;
    *radius = std::sqrt(x);
    *aware = (k->kind == PS_KERNEL_EXPONENTIAL) ? 1 : (eps > 0.0 ? 1 : 0);
    return PS_OK;
}

double ps_eval_kernel(const ps_kernel* k, double x) { return k ? eval_kernel(*k, x) : NAN; }

int ps_validate_config(const ps_config* c) {
    if (!c) return fail(PS_INVALID_ARGUMENT, "null config");
    int st = validate_config(*c);
    return st == PS_OK ? st : fail(st, "RasterConfig::validate: invalid configuration");
}

int ps_validate_camera(const ps_camera* c) {
    if (!c) return fail(PS_INVALID_ARGUMENT, "null camera");
    int st = validate_camera(*c);
    return st == PS_OK ? st
                       : fail(st, st == PS_NON_ORTHONORMAL_ROTATION ? "camera rotation is not orthonormal"
                                                                    : "Camera::validate: invalid camera");
}

} // extern "C"
