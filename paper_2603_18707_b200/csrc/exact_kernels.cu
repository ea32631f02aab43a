// exact_kernels.cu — the stages that must reproduce the reference's fp64 bits.
// COMPILED WITH -fmad=false (see build.py): no FMA contraction, so fp64
// arithmetic here equals the reference's FMA-free x86-64 build bit for bit.
//
//   K1 k_preprocess : project_splat + culling_bound_for + tile_rect + tight-tile
//                     count + SH colour + fp32 blend record (raster.cpp:132-171,
//                     projection.cpp:36-116, kernel.cpp:335-369)
//   K3 k_duplicate  : duplicate-with-keys in depth order with the exact tight
//                     test (bin_splats, raster.cpp:186-208)
//   K7 k_replay     : exact fp64 re-blend of flagged pixels with the reference's
//                     per-pixel arithmetic (raster.cpp:250-283, reference.cpp:27-50)
#include <cfloat>

#include "common.cuh"
#include "exact_math.cuh"
#include "kernels.h"
#include "tile_sort.cuh"

namespace ps {

namespace {

constexpr float kSH0f = 0.28209479177387814f;
constexpr float kSH1f = 0.4886025119029199f;
__constant__ float kSH2f[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kSH3f[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                               0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

__device__ __forceinline__ void raise_error(DevCounters* ctr, int code, int64_t i) {
    if (atomicCAS(&ctr->error, 0u, static_cast<unsigned>(code)) == 0u)
        ctr->error_index = static_cast<unsigned>(i);
}

// eval_sh_color (projection.cpp:93-116) in fp32 from the fp32 SH planes. The
// colour never feeds a discrete decision; its fp32 error (~1e-7) is inside the
// image tolerance.
__device__ void sh_color(const float* v, int degree, float x, float y, float z, float out[3]) {
    // explicit fmaf: this file is compiled without FMA contraction (for the
    // fp64 stages), and the colour needs no particular rounding order
    float bs[16];
    bs[0] = kSH0f;
    bs[1] = -kSH1f * y; bs[2] = kSH1f * z; bs[3] = -kSH1f * x;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    bs[4] = kSH2f[0] * xy; bs[5] = kSH2f[1] * yz; bs[6] = kSH2f[2] * (2.0f * zz - xx - yy);
    bs[7] = kSH2f[3] * xz; bs[8] = kSH2f[4] * (xx - yy);
    bs[9] = kSH3f[0] * y * (3.0f * xx - yy); bs[10] = kSH3f[1] * xy * z;
    bs[11] = kSH3f[2] * y * (4.0f * zz - xx - yy); bs[12] = kSH3f[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    bs[13] = kSH3f[4] * x * (4.0f * zz - xx - yy); bs[14] = kSH3f[5] * z * (xx - yy);
    bs[15] = kSH3f[6] * x * (xx - yy);
    const int nb = degree >= 3 ? 16 : degree == 2 ? 9 : degree == 1 ? 4 : 1;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float c = v[ch] * bs[0];
#pragma unroll
        for (int k = 1; k < 16; ++k)
            if (k < nb) c = fmaf(v[3 * k + ch], bs[k], c);
        out[ch] = fmaxf(c + 0.5f, 0.0f);
    }
}

// Threshold q* of the BLEND kernel: alpha = min(.999, o k(q)) >= eps  <=>  q <= q*
// for kernels non-increasing in q (checked on the host). Returns 0 when alpha < eps
// everywhere, 1 with q*, 2 when alpha >= eps for every q.
__device__ int blend_threshold(const ps_kernel& k, double o, double eps, double& qs) {
    if (k.kind == PS_KERNEL_EXPONENTIAL) {
        if (!(o > eps)) return 0;
        qs = 2.0 * log(o / eps);
        return 1;
    }
    if (!(o * k.coeffs[0] > eps)) return 0;
    double shifted[4] = {k.coeffs[0] - eps / o, k.coeffs[1], k.coeffs[2], k.coeffs[3]};
    int st = first_positive_root(shifted, k.order + 1, qs);
    return st == PS_OK ? 1 : 2;
}

// fp32 blend record + decision guards (DESIGN.md §blend numerics). The blend
// evaluates q in the completed-square form  q = A (dx + beta dy)^2 + gamma dy^2
// (A = a, beta = b/a, gamma = c - b^2/a, all rounded to fp32) in tile-local
// coordinates. Gq bounds |q_fp32 - q_ref64| over the region q <= 1.25 q* + 1
// (forward error analysis with a 4x margin); decisions with q inside
// [q* - Gq, q* + Gq] are re-decided in fp64. eT bounds the per-blend relative
// error of the fp32 transmittance; pixels whose T lands within the accumulated
// bound of the floor are replayed exactly.
// Blend kernel classes for K1b: exponential, polynomial of effective order 1..3.
enum BlendClass : int { kBkExp = 0, kBkP1 = 1, kBkP2 = 2, kBkP3 = 3, kBkGeneric = 4 };

template <int BK>
__device__ int blend_threshold_t(const ps_kernel& k, double o, double eps, double& qs) {
    if (BK == kBkGeneric) return blend_threshold(k, o, eps, qs);
    if (BK == kBkExp) {
        if (!(o > eps)) return 0;
        qs = 2.0 * log(o / eps);
        return 1;
    }
    if (!(o * k.coeffs[0] > eps)) return 0;
    double c[4] = {k.coeffs[0] - eps / o, k.coeffs[1], k.coeffs[2], k.coeffs[3]};
    if (!(c[0] > 0.0)) return 2;
    double x = 0.0;
    int st;
    if (BK == kBkP1) { st = root_linear(c[0], c[1], x); if (st == PS_OK) x = polish_root(c, 2, x); }
    else if (BK == kBkP2) { st = root_quadratic(c, x); if (st == PS_OK) x = polish_root(c, 3, x); }
    else { st = root_cubic(c, x); if (st == PS_OK) x = polish_root(c, 4, x); }
    if (st != PS_OK) return 2;
    qs = x;
    return 1;
}


template <int BK>
__device__ void blend_record(double a, double b, double c, double o, const FrameParams& P, float cr, float cg,
                             float cb, float4& r0, float4& r1, float2& r2, const double* qs_known = nullptr) {
    const double e32 = 5.9604644775390625e-08; // 2^-24
    const double e64 = 1.1102230246251565e-16; // 2^-53
    const ps_kernel& k = P.cfg.kernel;
    const double eps = P.cfg.epsilon;
    const double ts = P.cfg.tile_size;
    double beta = b / a;
    double gamma = c - b * b / a;
    double qs = 0.0;
    int th;
    if (qs_known) { // the culling bound's root is this threshold (same kernel, epsilon and opacity)
        qs = *qs_known;
        th = 1;
    } else {
        th = blend_threshold_t<BK>(k, o, eps, qs);
    }
    float qhi, qlo, eT;
    bool ok = a > 0.0 && gamma > 0.0 && isfinite(beta) && isfinite(gamma);
    double amax = k.kind == PS_KERNEL_EXPONENTIAL ? o : o * k.coeffs[0];
    amax = fmin(amax, 0.999);
    if (!ok) {
        // ill-conditioned: every candidate is decided in fp64 and any pixel that
        // blends it is replayed exactly
        qhi = INFINITY; qlo = -INFINITY; eT = INFINITY;
    } else {
        // Gq(qb): bound on |q_fp32 - q_ref| over the region q <= qb
        auto gq_for = [&](double qb) -> double {
            double U = sqrt(qb / a), D = sqrt(qb / gamma);
            double ab_ = fabs(beta);
            double X = U + ab_ * D;
            double gam_rel = e32 + 4.0 * e64 * (c + b * b / a) / gamma;
            double du, ddy;
            if (P.cfg.tile_size == 16) {
                // k_blend16 (blend.cu pair_frag) works in record-local coordinates:
                // the tile-local mean m = o + m' with o = rint(m) (integer, exact)
                // and |m'| <= M = 0.5 + e32 (X + ts) held in fp32 (error e32 M);
                // dy = (yc - oy) - my' (yc - oy exact), t = fma(beta, dy, -mx'),
                // u = (x - ox) + t (x - ox exact), so no term scales with the tile
                const double Mx = 0.5 + e32 * (X + ts), My = 0.5 + e32 * (D + ts);
                const double dmx = e32 * Mx, dmy = e32 * My;
                ddy = dmy + e32 * D;
                du = ab_ * ddy + e32 * ab_ * D + dmx + e32 * (ab_ * D + Mx) + e32 * U;
            } else {
                // k_blend: tile-local fp32 mean (error e32 (X + ts))
                const double dmx = e32 * (X + ts), dmy = e32 * (D + ts);
                const double ddx = dmx + e32 * X;
                ddy = dmy + e32 * D;
                // u is formed either as (dx + beta dy) or as x - (mx - beta dy); bound both
                du = 2.0 * dmx + ddx + ab_ * ddy + 2.0 * e32 * ab_ * D + e32 * (U + X);
            }
            double dr = qb * (2.0 * e32 + gam_rel) + 2.0 * gamma * D * ddy;
            double dau = qb * 3.0 * e32 + 2.0 * a * U * du;
            double dq = e32 * qb + dau + dr;
            double ref = 8.0 * e64 * (a * X * X + 2.0 * fabs(b) * X * D + c * D * D) +
                         4.0 * e64 * (a * X + fabs(b) * D) * (X + D);
            // each term above is a first-order upper bound; 1.25 covers the
            // second-order products. The threshold q*: a polished fp64 root
            // (~1e-15 relative; 1e-9 qb) and, for polynomials, the reference's
            // fp64 rounding of o p(q) near eps in q units (P.root_slack)
            const double droot = 1e-9 * qb + (th == 1 ? P.root_slack : 0.0);
            return 1.25 * (dq + ref) + droot + 1e-12;
        };
        // quadric mode: a candidate has fp32 q <= q_hi = fl_up(q* + Gq), so its
        // true q is below q* + 2 Gq (+ one fp32 ulp) and a region just above q*
        // suffices; otherwise (or if that region turns out too tight) q <= 1.25 q* + 1
        const bool tight = th == 1 && P.threshold_mode == kQuadricThreshold;
        double qb = tight ? 1.01 * qs + 0.01 : (th == 1 ? 1.25 * qs : 25.0) + 1.0;
        double Gq = gq_for(qb);
        if (tight && !((qs + Gq) * (1.0 + 2.5e-7) + Gq <= qb)) {
            qb = 1.25 * qs + 1.0;
            Gq = gq_for(qb);
        }
        // |alpha_fp32 - alpha_ref| for accepted fragments (q <= qb):
        //   o max|k'| Gq  +  evaluation rounding  (+ ex2.approx error for exp)
        double kp = 0.5, kmag = 1.0, extra = 0.0;
        if (k.kind != PS_KERNEL_EXPONENTIAL) {
            // max |p'(q)| over [0, qb] exactly: p' = d0 + d1 q + d2 q^2
            const double d0 = k.order >= 1 ? k.coeffs[1] : 0.0;
            const double d1 = k.order >= 2 ? 2.0 * k.coeffs[2] : 0.0;
            const double d2 = k.order >= 3 ? 3.0 * k.coeffs[3] : 0.0;
            auto dp = [&](double q) { return fabs(d0 + d1 * q + d2 * q * q); };
            kp = fmax(dp(0.0), dp(qb));
            if (d2 != 0.0) {
                const double qv = -d1 / (2.0 * d2);
                if (qv > 0.0 && qv < qb) kp = fmax(kp, dp(qv));
            }
            kmag = 0.0;
            double qp = 1.0;
            for (int j = 0; j <= k.order; ++j) {
                kmag += fabs(k.coeffs[j]) * qp;
                qp *= qb;
            }
            // Horner with FMA rounds once per step, so the term a_j q^j carries
            // at most j (<= order) roundings (Higham, Accuracy and Stability,
            // 5.1), plus one for the folded coefficient o c_j in fp32 (quadric
            // mode) or for the fp32 coefficient and the final o * p (alpha
            // mode): gamma_{order+2} sum |c_j| q^j, with 10% slack
            kmag *= k.order + 2.2;
        } else {
            // ex2.approx (2^-22) + fp32 rounding of its argument (|arg| <= 0.73 qb + |log2 o|)
            extra = amax * (2.4e-7 + (0.73 * qb + fabs(log2(o)) + 1.0) * e32 * 0.7);
            kmag = 0.0;
        }
        const double Ga = 1.02 * (o * kp * Gq + e32 * o * kmag + extra) + 2.0 * e32 * amax + 1e-15;
        if (P.threshold_mode == kAlphaThreshold) {
            qhi = __double2float_ru(Ga);
            qlo = 0.0f;
        } else if (th == 0) {
            qhi = -1.0f; qlo = -1.0f;               // never reaches epsilon
        } else if (th == 2) {
            qhi = INFINITY; qlo = INFINITY;         // above epsilon everywhere
        } else {
            qhi = __double2float_ru(qs + Gq);
            qlo = __double2float_rd(qs - Gq);
        }
        eT = __double2float_ru(Ga);
    }
    float oval = k.kind == PS_KERNEL_EXPONENTIAL ? (o > 0.0 ? static_cast<float>(log2(o)) : -INFINITY)
                                                 : static_cast<float>(o);
    r0 = make_float4(static_cast<float>(a), static_cast<float>(beta), static_cast<float>(gamma), qhi);
    r1 = make_float4(qlo, oval, eT, cr);
    r2 = make_float2(cg, cb);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

} // namespace

// Tight-tile decision (raster.cpp:103-128) in three tiers, each deciding only
// what it can certify against the reference's exact fp64 result m_ref:
//  1. fp32 screen: the same box minimum in fp32 (per-splat multipliers, FMNMX
//     clamps). Its deviation from m_ref is < ~10u32 * scale, with
//     scale = a X^2 + 2|b| X Y + c Y^2 (X, Y = the box's largest |offsets|):
//     ~2u from rounding the offsets, ~5u from the products/sums, the minimiser
//     error entering only at second order. A margin of 1e-5 scale (~170u32)
//     plus the fp32 rounding of q_root decides all but a sliver of tests.
//  2. fp64 without per-test divisions: the edge minimisers use kx = -b/c,
//     ky = -b/a instead of ((-b)*d)/c, within ~40 ulp64 of scale of m_ref, so
//     decisions with |m - q_root| > 1e-12 scale are the reference's.
//  3. the reference arithmetic (min_quadric_over_box) for the rest.
struct TightSplat {
    Sym2 cn;
    double mx, my, qroot, kx, ky;
    float a32, b32, c32, kx32, ky32, q32;
    bool screen; // fp32 tier usable (finite, non-degenerate conic)
};

__device__ __forceinline__ TightSplat make_tight(const Sym2& cn, double mx, double my, double qroot) {
    TightSplat t{cn, mx, my, qroot, 0.0, 0.0, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, false};
    t.kx = cn.yy != 0.0 ? -cn.xy / cn.yy : 0.0;
    t.ky = cn.xx != 0.0 ? -cn.xy / cn.xx : 0.0;
    t.a32 = static_cast<float>(cn.xx);
    t.b32 = static_cast<float>(cn.xy);
    t.c32 = static_cast<float>(cn.yy);
    t.kx32 = static_cast<float>(t.kx);
    t.ky32 = static_cast<float>(t.ky);
    t.q32 = static_cast<float>(qroot);
    t.screen = cn.xx != 0.0 && cn.yy != 0.0 && fabs(cn.xx) < 1e30 && fabs(cn.xy) < 1e30 && fabs(cn.yy) < 1e30 &&
               fabs(t.kx) < 1e30 && fabs(t.ky) < 1e30 && fabs(qroot) < 1e30;
    return t;
}

__device__ __forceinline__ float quadric32(const TightSplat& t, float dx, float dy) {
    return fmaf(t.a32 * dx, dx, fmaf(2.0f * t.b32 * dx, dy, t.c32 * dy * dy));
}

__device__ __forceinline__ bool tight_test_fast(const TightSplat& t, int tx, int ty, int ts) {
    const double x0 = tx * static_cast<double>(ts) + 0.5;
    const double y0 = ty * static_cast<double>(ts) + 0.5;
    const double bx1 = x0 + ts - 1, by1 = y0 + ts - 1;
    const double lx = x0 - t.mx, hx = bx1 - t.mx;
    const double ly = y0 - t.my, hy = by1 - t.my;
    if (lx <= 0.0 && hx >= 0.0 && ly <= 0.0 && hy >= 0.0) return 0.0 <= t.qroot;
    if (t.screen) {
        const float flx = static_cast<float>(lx), fhx = static_cast<float>(hx);
        const float fly = static_cast<float>(ly), fhy = static_cast<float>(hy);
        float m = quadric32(t, flx, fminf(fmaxf(t.kx32 * flx, fly), fhy));
        m = fminf(m, quadric32(t, fhx, fminf(fmaxf(t.kx32 * fhx, fly), fhy)));
        m = fminf(m, quadric32(t, fminf(fmaxf(t.ky32 * fly, flx), fhx), fly));
        m = fminf(m, quadric32(t, fminf(fmaxf(t.ky32 * fhy, flx), fhx), fhy));
        const float X = fmaxf(fabsf(flx), fabsf(fhx)), Y = fmaxf(fabsf(fly), fabsf(fhy));
        const float scale = fabsf(t.a32) * X * X + 2.0f * fabsf(t.b32) * X * Y + fabsf(t.c32) * Y * Y;
        const float tol = fmaf(1e-5f, scale, fmaf(1e-6f, fabsf(t.q32), 1e-30f));
        if (scale < 1e30f) {
            if (m < t.q32 - tol) return true;
            if (m > t.q32 + tol) return false;
        }
    }
    const Sym2& c = t.cn;
    double dy = std_clamp(c.yy != 0.0 ? t.kx * lx : ly, ly, hy);
    double m = quadric(c, lx, dy);
    dy = std_clamp(c.yy != 0.0 ? t.kx * hx : ly, ly, hy);
    m = std_min(m, quadric(c, hx, dy));
    double dx = std_clamp(c.xx != 0.0 ? t.ky * ly : lx, lx, hx);
    m = std_min(m, quadric(c, dx, ly));
    dx = std_clamp(c.xx != 0.0 ? t.ky * hy : lx, lx, hx);
    m = std_min(m, quadric(c, dx, hy));
    const double X = fmax(fabs(lx), fabs(hx)), Y = fmax(fabs(ly), fabs(hy));
    const double scale = fabs(c.xx) * X * X + 2.0 * fabs(c.xy) * X * Y + fabs(c.yy) * Y * Y;
    const double tol = 1e-12 * scale;
    if (isfinite(m) && isfinite(tol)) {
        if (m < t.qroot - tol) return true;
        if (m > t.qroot + tol) return false;
    }
    return min_quadric_over_box(c, t.mx, t.my, x0, y0, bx1, by1) <= t.qroot; // exact reference path
}

// tile_rect (raster.cpp:71-86); for a power-of-two tile size x / ts is an
// exact scaling, so multiplying by 1/ts gives the same bits as the division.
__device__ __forceinline__ bool tile_rect_fast(double mx, double my, double cov_xx, double cov_yy, double radius,
                                               int ts, int width, int height, int r[4]) {
    if (ts & (ts - 1)) return tile_rect(mx, my, cov_xx, cov_yy, radius, ts, width, height, r);
    const double inv = 1.0 / ts;
    const double hx = radius * sqrt(std_max(cov_xx, 0.0));
    const double hy = radius * sqrt(std_max(cov_yy, 0.0));
    const int tiles_x = (width + ts - 1) / ts;
    const int tiles_y = (height + ts - 1) / ts;
    int x0 = x86_cvtt_int(floor((mx - hx) * inv));
    int x1 = x86_cvtt_int(floor((mx + hx) * inv));
    int y0 = x86_cvtt_int(floor((my - hy) * inv));
    int y1 = x86_cvtt_int(floor((my + hy) * inv));
    x0 = imax(x0, 0);
    y0 = imax(y0, 0);
    x1 = imin(x1, tiles_x - 1);
    y1 = imin(y1, tiles_y - 1);
    if (x0 > x1 || y0 > y1) return false;
    r[0] = x0; r[1] = y0; r[2] = x1; r[3] = y1;
    return true;
}

// Warp-cooperative tight tests for rects of up to 8x8 tiles. Rect sizes differ
// a lot between the splats of a warp (1 to 64 tiles), so a per-thread loop runs
// at the warp's largest rect. Instead each lane publishes its splat's fp32
// screen (below) in shared memory, the warp enumerates all (splat, tile) tests
// of its lanes in rounds of 32 (test g belongs to the first lane whose
// inclusive prefix of rect sizes exceeds g), and each owner collects its
// results from the round's ballot. Tests the fp32 screen cannot certify are
// re-done by the owner with tight_test_fast's fp64 tiers.
//   The screen is tight_test_fast's tier 1 with the box offsets formed as
// fp32 fma(j, ts, fx0) (+ ts - 1) from the rect's first box offset fx0 =
// fl(x0 - mx): two more fp32 roundings of offsets (<= ~4u32 relative), inside
// the screen's ~170u32 scale margin. The centre-inside case (box minimum 0) is
// decided exactly per splat: the one tile whose pixel-centre box holds the
// centre, found with the reference's fp64 expressions.
struct ScreenRec {
    float a, b, c, kx, ky, q, fx0, fy0;
    float rcpw;     // 1 / rect width (tile index -> row)
    uint32_t meta;  // off (12 bits) | w << 12 | ix_in << 16 | iy_in << 20 | inside_pass << 24 | screen << 25
    uint32_t pad[2];
};

__device__ __forceinline__ int inside_index(double m, int t0, int t1, int ts) {
    // the tile t in [t0, t1] whose box [t ts + 0.5, t ts + ts - 0.5] holds m (else 15)
    // c = floor((m - 0.5) / ts): for a power-of-two ts the scaling is exact and
    // rounding m - 0.5 is monotone with t ts and t ts + ts - 1 representable, so
    // a centre in box t gives c == t; otherwise c +- 1 are tested too
    const int c = x86_cvtt_int(floor((m - 0.5) * (1.0 / ts)));
    const int span = (ts & (ts - 1)) == 0 ? 0 : 1;
    for (int d = -span; d <= span; ++d) {
        const int t = c + d;
        if (t < t0 || t > t1) continue;
        const double x0 = t * static_cast<double>(ts) + 0.5;
        const double bx1 = x0 + ts - 1;
        if (x0 - m <= 0.0 && bx1 - m >= 0.0) return t - t0;
    }
    return 15;
}

// The screen of a small-rect splat straight from its fp64 conic: the minimiser
// multipliers kx = -b/c, ky = -b/a in fp32 (they only place the edge points,
// so their error enters the box minimum at second order, like their rounding
// from fp64 in make_tight); the fp64 ones are formed only for undecided tests.
__device__ __forceinline__ ScreenRec make_screen(const Sym2& cn, double mx, double my, double qroot, const int r[4],
                                                 int ts) {
    ScreenRec s;
    s.a = static_cast<float>(cn.xx);
    s.b = static_cast<float>(cn.xy);
    s.c = static_cast<float>(cn.yy);
    s.kx = s.c != 0.0f ? -s.b / s.c : 0.0f;
    s.ky = s.a != 0.0f ? -s.b / s.a : 0.0f;
    s.q = static_cast<float>(qroot);
    const bool screen = s.a != 0.0f && s.c != 0.0f && fabsf(s.a) < 1e30f && fabsf(s.b) < 1e30f &&
                        fabsf(s.c) < 1e30f && fabsf(s.kx) < 1e30f && fabsf(s.ky) < 1e30f && fabsf(s.q) < 1e30f;
    s.fx0 = static_cast<float>((r[0] * static_cast<double>(ts) + 0.5) - mx);
    s.fy0 = static_cast<float>((r[1] * static_cast<double>(ts) + 0.5) - my);
    const int w = r[2] - r[0] + 1;
    s.rcpw = 1.0f / static_cast<float>(w);
    const int ixin = inside_index(mx, r[0], r[2], ts), iyin = inside_index(my, r[1], r[3], ts);
    s.meta = (static_cast<uint32_t>(w) << 12) | (static_cast<uint32_t>(ixin) << 16) |
             (static_cast<uint32_t>(iyin) << 20) | ((0.0 <= qroot ? 1u : 0u) << 24) | ((screen ? 1u : 0u) << 25);
    s.pad[0] = s.pad[1] = 0u;
    return s;
}

// 1 = passes, 0 = fails, 2 = undecided (fp64 tiers)
__device__ __forceinline__ int screen_test(const ScreenRec& s, int j, float tsf) {
    const int w = static_cast<int>((s.meta >> 12) & 15u);
    const int jy = static_cast<int>((static_cast<float>(j) + 0.5f) * s.rcpw);
    const int jx = j - jy * w;
    if (jx == static_cast<int>((s.meta >> 16) & 15u) && jy == static_cast<int>((s.meta >> 20) & 15u))
        return (s.meta >> 24) & 1u;
    if (!((s.meta >> 25) & 1u)) return 2;
    const float flx = fmaf(static_cast<float>(jx), tsf, s.fx0), fhx = flx + (tsf - 1.0f);
    const float fly = fmaf(static_cast<float>(jy), tsf, s.fy0), fhy = fly + (tsf - 1.0f);
    auto q32 = [&](float dx, float dy) { return fmaf(s.a * dx, dx, fmaf(2.0f * s.b * dx, dy, s.c * dy * dy)); };
    float m = q32(flx, fminf(fmaxf(s.kx * flx, fly), fhy));
    m = fminf(m, q32(fhx, fminf(fmaxf(s.kx * fhx, fly), fhy)));
    m = fminf(m, q32(fminf(fmaxf(s.ky * fly, flx), fhx), fly));
    m = fminf(m, q32(fminf(fmaxf(s.ky * fhy, flx), fhx), fhy));
    const float X = fmaxf(fabsf(flx), fabsf(fhx)), Y = fmaxf(fabsf(fly), fabsf(fhy));
    const float scale = fabsf(s.a) * X * X + 2.0f * fabsf(s.b) * X * Y + fabsf(s.c) * Y * Y;
    const float tol = fmaf(1e-5f, scale, fmaf(1e-6f, fabsf(s.q), 1e-30f));
    if (scale < 1e30f) {
        if (m < s.q - tol) return 1;
        if (m > s.q + tol) return 0;
    }
    return 2;
}

// All lanes of the warp call this (converged). cand = this lane's rect size
// (0: nothing to test), its screen already in srec[threadIdx.x] (offset field
// 0; set here). Returns the
// lane's pass bits in the stride-8 rect layout (bit 8 jy + jx) and, in *und,
// the bits left undecided (same layout).
__device__ __forceinline__ unsigned long long warp_tight_tests(ScreenRec* srec, int cand, int w, int h, float tsf,
                                                               unsigned long long* und) {
    const int lane = threadIdx.x & 31;
    ScreenRec* wrec = srec + (threadIdx.x & ~31);
    int inc = cand;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const int total = __shfl_sync(0xffffffffu, inc, 31);
    const int off = inc - cand;
    if (cand) wrec[lane].meta |= static_cast<uint32_t>(off);
    __syncwarp();
    unsigned long long pc = 0ull, uc = 0ull; // compact order (bit j)
    for (int base = 0; base < total; base += 32) {
        const int g = base + lane;
        int owner = 0; // lanes whose inclusive prefix <= g
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, inc, owner + step - 1);
            if (v <= g) owner += step;
        }
        int res = 0;
        if (g < total) {
            const ScreenRec& s = wrec[owner];
            res = screen_test(s, g - static_cast<int>(s.meta & 0xfffu), tsf);
        }
        const uint32_t pb = __ballot_sync(0xffffffffu, res == 1);
        const uint32_t ub = __ballot_sync(0xffffffffu, res == 2);
        const int sh = off - base; // this lane's first test relative to the round
        if (cand && sh < 32 && sh + cand > 0) {
            if (sh >= 0) {
                pc |= static_cast<unsigned long long>(pb >> sh);
                uc |= static_cast<unsigned long long>(ub >> sh);
            } else {
                pc |= static_cast<unsigned long long>(pb) << (-sh);
                uc |= static_cast<unsigned long long>(ub) << (-sh);
            }
        }
    }
    unsigned long long pm = 0ull, um = 0ull;
    if (cand) {
        const unsigned long long keep = cand == 64 ? ~0ull : ((1ull << cand) - 1ull);
        pc &= keep;
        uc &= keep;
        const unsigned long long row = (1ull << w) - 1ull;
        for (int jy = 0; jy < h; ++jy) {
            pm |= ((pc >> (jy * w)) & row) << (8 * jy);
            um |= ((uc >> (jy * w)) & row) << (8 * jy);
        }
    }
    *und = um;
    return pm;
}

// Block-level tile aggregation. Splats are Morton-ordered, so one CTA's splats
// cover a compact screen region: per-tile counts / bucket slots are gathered
// in a shared-memory window over the union of the CTA's tile rects, and only
// one global atomic per distinct tile per CTA is issued. Rects of > 64 tiles
// (or a window larger than kWinCap) fall back to direct global atomics.

struct Window {
    int x0, y0, w, h;
    bool ok;
};

__device__ __forceinline__ Window block_window(bool has, const int r[4], int* wb) {
    if (threadIdx.x == 0) { wb[0] = INT_MAX; wb[1] = INT_MAX; wb[2] = -1; wb[3] = -1; }
    // warp-reduce first: one shared atomic per warp instead of one per thread
    const int x0 = __reduce_min_sync(0xffffffffu, has ? r[0] : INT_MAX);
    const int y0 = __reduce_min_sync(0xffffffffu, has ? r[1] : INT_MAX);
    const int x1 = __reduce_max_sync(0xffffffffu, has ? r[2] : -1);
    const int y1 = __reduce_max_sync(0xffffffffu, has ? r[3] : -1);
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && x1 >= 0) {
        atomicMin(&wb[0], x0);
        atomicMin(&wb[1], y0);
        atomicMax(&wb[2], x1);
        atomicMax(&wb[3], y1);
    }
    __syncthreads();
    Window w;
    w.x0 = wb[0];
    w.y0 = wb[1];
    w.w = wb[2] - wb[0] + 1;
    w.h = wb[3] - wb[1] + 1;
    w.ok = wb[2] >= 0 && w.w * w.h <= kWinCap;
    return w;
}

// Tight-tile masks use a fixed row stride of 8 (bit = 8 * (ty - y0) + (tx - x0)),
// so rects of up to 8 x 8 tiles fit and bit -> tile is shifts, not divisions.
__device__ __forceinline__ bool rect_is_small(const int r[4]) { return r[2] - r[0] < 8 && r[3] - r[1] < 8; }

__device__ __forceinline__ int rect_bit_tile(const int r[4], int b, int tiles_x) {
    return (r[1] + (b >> 3)) * tiles_x + r[0] + (b & 7);
}

__device__ __forceinline__ int rect_bit_win(const int r[4], int b, const Window& W) {
    return (r[1] + (b >> 3) - W.y0) * W.w + (r[0] + (b & 7) - W.x0);
}

// ------------------------------------------------------------ K1 preprocess
// Split in two so each variant stays small (the all-modes kernel thrashed the
// instruction cache):
//   K1a k_geometry<BC>: project_splat (projection.cpp:36-79), culling_bound_for
//       specialised on the culling class (raster.cpp:50-69, kernel.cpp:335-369),
//       tile_rect (raster.cpp:71-86) and the tight-tile bitmask (raster.cpp:126-128).
//   K1b k_shade<BK>: SH colour (projection.cpp:93-116) + the fp32 blend record,
//       specialised on the blend kernel.
enum BoundClass : int { kBcStp = 0, kBcZero = 1, kBcOaExp = 2, kBcOaP1 = 3, kBcOaP2 = 4, kBcOaP3 = 5, kBcGeneric = 6 };

// culling_bound_for specialised per class. 1 = bound set, 0 = nullopt (below
// epsilon, uncounted), -status on error. Same arithmetic as exact_math.cuh.
template <int BC>
__device__ __forceinline__ int bound_for(const ps_config& cfg, double o, double& radius, double& qroot, double& xr) {
    if (BC == kBcGeneric) return culling_bound_for(cfg, o, radius, qroot);
    if (!(o > 0.0)) return 0;
    double x = 0.0;
    if (BC == kBcStp) {
        if (!(o > cfg.epsilon)) return 0;
        x = 2.0 * log(o / cfg.epsilon);
    } else if (BC == kBcZero) {
        x = (cfg.has_culling_kernel ? cfg.culling_kernel : cfg.kernel).first_root;
    } else {
        const ps_kernel& k = cfg.has_culling_kernel ? cfg.culling_kernel : cfg.kernel;
        if (o > 1.0) return -PS_INVALID_ARGUMENT; // culling_radius: opacity must be in (0,1]
        if (BC == kBcOaExp) {
            if (!(o > cfg.epsilon)) return 0;
            x = 2.0 * log(o / cfg.epsilon);
        } else {
            if (!(o * k.coeffs[0] > cfg.epsilon)) return 0;
            double c[4] = {k.coeffs[0] - cfg.epsilon / o, k.coeffs[1], k.coeffs[2], k.coeffs[3]};
            if (!(c[0] > 0.0)) return -PS_INVALID_ARGUMENT;
            int st;
            if (BC == kBcOaP1) {
                st = root_linear(c[0], c[1], x);
                if (st == PS_OK) x = polish_root(c, 2, x);
            } else if (BC == kBcOaP2) {
                st = root_quadratic(c, x);
                if (st == PS_OK) x = polish_root(c, 3, x);
            } else {
                st = root_cubic(c, x);
                if (st == PS_OK) x = polish_root(c, 4, x);
            }
            if (st != PS_OK) return -st;
        }
    }
    xr = x;
    qroot = x + kBoundSlack;
    radius = sqrt(qroot);
    return 1;
}

// The blend threshold (blend_threshold_t<BK>) of a visible splat equals the
// culling root x of bound_for<BC> when both solve the same equation: the
// opacity-aware bound of the blend kernel itself (no separate culling kernel),
// or the exponential threshold 2 ln(o / eps) (StopThePop or opacity-aware exp).
// The fused K1 then passes x on instead of solving it again.
template <int BC, int BK>
constexpr bool kThresholdIsBound = (BC == kBcOaP1 && BK == kBkP1) || (BC == kBcOaP2 && BK == kBkP2) ||
                                   (BC == kBcOaP3 && BK == kBkP3) || ((BC == kBcOaExp || BC == kBcStp) && BK == kBkExp);

// K1a for one view: splat i (in = i < n) with its camera-independent inputs
// (mean, 3D covariance, opacity) already in registers. Every thread of the CTA
// calls it (block-level tile aggregation inside).
// What the shading of a visible splat needs from K1a (the fused kernel passes it
// in registers instead of through the frame arrays).
struct GeoOut {
    bool visible = false;
    double a = 0.0, b = 0.0, c = 0.0, o = 0.0; // conic (xx, xy, yy), opacity_eff
    double x = 0.0;                             // the culling root (bound_for)
};

// Tight pairs per tile for the bucket scan (K2), aggregated in the CTA's
// shared window (block_window); every thread of the CTA calls this.
__device__ __forceinline__ void tile_window_counts(bool small, const int (&my_r)[4], unsigned long long my_mask,
                                                   const FrameDev& f, const FrameParams& P) {
    __shared__ uint32_t win[kWinCap];
    __shared__ int wb[4];
    const Window W = block_window(small, my_r, wb);
    if (W.ok) {
        for (int k = threadIdx.x; k < W.w * W.h; k += blockDim.x) win[k] = 0;
        __syncthreads();
        if (small) {
            unsigned long long m = my_mask;
            while (m) {
                const int b = __ffsll(static_cast<long long>(m)) - 1;
                m &= m - 1;
                atomicAdd(&win[rect_bit_win(my_r, b, W)], 1u);
            }
        }
        __syncthreads();
        uint32_t* wc = f.win_counts + static_cast<size_t>(blockIdx.x) * kWinCap; // for K3
        for (int k = threadIdx.x; k < W.w * W.h; k += blockDim.x) {
            const uint32_t v = win[k];
            wc[k] = v;
            if (v) atomicAdd(&f.tile_count[(W.y0 + k / W.w) * P.tiles_x + W.x0 + k % W.w], v);
        }
        if (threadIdx.x == 0) f.win_rect[blockIdx.x] = make_int4(W.x0, W.y0, W.w, W.h);
    } else {
        if (small) {
            unsigned long long m = my_mask;
            while (m) {
                const int b = __ffsll(static_cast<long long>(m)) - 1;
                m &= m - 1;
                atomicAdd(&f.tile_count[rect_bit_tile(my_r, b, P.tiles_x)], 1u);
            }
        }
        if (threadIdx.x == 0) f.win_rect[blockIdx.x] = make_int4(0, 0, 0, 0);
        // (W.ok is CTA-uniform) every thread has read wb before a next call's
        // thread 0 resets it (the multi-view kernels count view after view)
        __syncthreads();
    }
}

// The CTA's six frame counters (per-warp partials in red[k][warp], written
// before a CTA barrier) into the device counters: one atomic each per CTA.
__device__ __forceinline__ void flush_cta_counters(const unsigned long long (*red)[8], DevCounters* ctr) {
    if (threadIdx.x < 6) {
        const int k = threadIdx.x, nw = blockDim.x >> 5;
        unsigned long long v = red[k][0];
        for (int j = 1; j < nw; ++j) v = k < 2 ? max(v, red[k][j]) : v + red[k][j];
        if (v) {
            if (k == 0) atomicMax(&ctr->key_min, v);
            else if (k == 1) atomicMax(&ctr->key_max, v);
            else if (k == 2) atomicAdd(&ctr->frustum, v);
            else if (k == 3) atomicAdd(&ctr->coarse, v);
            else if (k == 4) atomicAdd(&ctr->tight, v);
            else atomicAdd(&ctr->visible, v);
        }
    }
}

// CTA_RED: the frame counters are reduced over the CTA before their atomics
// (one update per CTA instead of per warp; see the end).
template <int BC, bool CTA_RED = false>
__device__ __forceinline__ void geometry_view(int64_t i, bool in, const double (&mean)[3], const double (&c6)[6],
                                              double opacity, const FrameParams& P, const FrameDev& f,
                                              DevCounters* ctr, GeoOut* out = nullptr, ulonglong2* late = nullptr,
                                              unsigned long long (*late_red)[8] = nullptr) {
    __shared__ ScreenRec srec[256];
    unsigned long long frustum = 0, coarse = 0, tight = 0, visible = 0;
    unsigned long long kmin_inv = 0ull, kmax = 0ull; // min tracked as max of the complement
    bool small = false;
    unsigned long long my_mask = 0ull;
    int my_r[4] = {0, 0, -1, -1};
    int cand = 0; // tiles of a small rect, tested by the warp below
    const int ts = P.cfg.tile_size;
    if (in) {
        unsigned long long key = ~0ull;
        uint32_t cnt = 0;
        Projected pr;
        const int st = project(mean, c6, opacity, P.cam, P.cfg.v_dilation, pr);
        if (st < 0) {
            raise_error(ctr, -st, i);
        } else if (st == 0) {
            frustum = 1; // kFrustum (raster.cpp:144-146,162-163)
        } else {
            double radius = 0.0, qroot = 0.0, xr = 0.0;
            const int b = bound_for<BC>(P.cfg, pr.opacity_eff, radius, qroot, xr);
            if (b < 0) {
                raise_error(ctr, -b, i);
            } else if (b > 0) { // b == 0: below epsilon, dropped uncounted (raster.cpp:149-151)
                int r[4];
                if (!tile_rect_fast(pr.mx, pr.my, pr.cov_aa.xx, pr.cov_aa.yy, radius, ts, P.cam.width, P.cam.height, r)) {
                    frustum = 1; // off screen (raster.cpp:165-168)
                } else {
                    visible = 1;
                    coarse = static_cast<unsigned long long>(r[2] - r[0] + 1) *
                             static_cast<unsigned long long>(r[3] - r[1] + 1);
                    if (!rect_is_small(r)) { // big rect (rare): per-thread tests, direct atomics
                        const TightSplat tsp = make_tight(pr.conic, pr.mx, pr.my, qroot);
                        for (int ty = r[1]; ty <= r[3]; ++ty)
                            for (int tx = r[0]; tx <= r[2]; ++tx)
                                if (tight_test_fast(tsp, tx, ty, ts)) {
                                    ++cnt;
                                    if (f.tile_count) atomicAdd(&f.tile_count[ty * P.tiles_x + tx], 1u);
                                }
                        f.tmask[i] = 0ull;
                    } else {
                        cand = static_cast<int>(coarse);
                        srec[threadIdx.x] = make_screen(pr.conic, pr.mx, pr.my, qroot, r, ts);
                    }
                    for (int k = 0; k < 4; ++k) my_r[k] = r[k];
                    key = static_cast<unsigned long long>(__double_as_longlong(pr.depth));
                    kmin_inv = ~key;
                    kmax = key;
                    f.mean2d[i] = make_double2(pr.mx, pr.my);
                    f.conic_ab[i] = make_double2(pr.conic.xx, pr.conic.xy);
                    f.conic_cq[i] = make_double2(pr.conic.yy, qroot);
                    f.rect[i] = make_ushort4(static_cast<unsigned short>(r[0]), static_cast<unsigned short>(r[1]),
                                             static_cast<unsigned short>(r[2]), static_cast<unsigned short>(r[3]));
                    f.opacity_eff[i] = pr.opacity_eff;
                    if (out) {
                        out->visible = true;
                        out->a = pr.conic.xx;
                        out->b = pr.conic.xy;
                        out->c = pr.conic.yy;
                        out->o = pr.opacity_eff;
                        out->x = xr;
                    }
                    if (f.cov_aa) {
                        f.cov_aa[3 * i] = pr.cov_aa.xx;
                        f.cov_aa[3 * i + 1] = pr.cov_aa.xy;
                        f.cov_aa[3 * i + 2] = pr.cov_aa.yy;
                    }
                }
            }
        }
        f.key[i] = key;
        f.val[i] = static_cast<uint32_t>(i);
        tight = cnt; // big rects; small ones below
    }
    {   // small rects: the warp's tests together (warp_tight_tests)
        const int w = my_r[2] - my_r[0] + 1, h = my_r[3] - my_r[1] + 1;
        unsigned long long und = 0ull;
        unsigned long long mask = warp_tight_tests(srec, cand, w, h, static_cast<float>(ts), &und);
        if (cand) {
            if (und) { // the fp64 tiers for what the screen left open (rare)
                const double2 mm = f.mean2d[i], ab = f.conic_ab[i], cq = f.conic_cq[i];
                const TightSplat t = make_tight(Sym2{ab.x, ab.y, cq.x}, mm.x, mm.y, cq.y);
                do {
                    const int b = __ffsll(static_cast<long long>(und)) - 1;
                    und &= und - 1;
                    if (tight_test_fast(t, my_r[0] + (b & 7), my_r[1] + (b >> 3), ts)) mask |= 1ull << b;
                } while (und);
            }
            const uint32_t cnt = static_cast<uint32_t>(__popcll(mask));
            small = cnt > 0;
            my_mask = mask;
            f.tmask[i] = mask;
            tight = cnt;
        }
        if (in) f.tcount[i] = static_cast<uint32_t>(tight);
    }
    if (f.tile_count) { // tight pairs per tile for the bucket scan (K2)
        if (late) late[threadIdx.x] = make_ulonglong2(small ? my_mask : 0ull,
                                                      (static_cast<unsigned long long>(static_cast<uint16_t>(my_r[0]))) |
                                                      (static_cast<unsigned long long>(static_cast<uint16_t>(my_r[1])) << 16) |
                                                      (static_cast<unsigned long long>(static_cast<uint16_t>(my_r[2])) << 32) |
                                                      (static_cast<unsigned long long>(static_cast<uint16_t>(my_r[3])) << 48));
        else tile_window_counts(small, my_r, my_mask, f, P);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin_inv = max(kmin_inv, __shfl_xor_sync(0xffffffffu, kmin_inv, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    frustum = warp_sum_u64(frustum);
    coarse = warp_sum_u64(coarse);
    tight = warp_sum_u64(tight);
    visible = warp_sum_u64(visible);
    if (!CTA_RED) {
        if ((threadIdx.x & 31) == 0) {
            if (kmax) {
                atomicMax(&ctr->key_min, kmin_inv);
                atomicMax(&ctr->key_max, kmax);
            }
            if (frustum) atomicAdd(&ctr->frustum, frustum);
            if (coarse) atomicAdd(&ctr->coarse, coarse);
            if (tight) atomicAdd(&ctr->tight, tight);
            if (visible) atomicAdd(&ctr->visible, visible);
        }
        return;
    }
    // one set of counter atomics per CTA: the six counter words are single L2
    // addresses every CTA of the grid updates, and per warp (3-6M splats: up to
    // ~190k updates per address per frame) they throttled the fused K1 at scale
    // (C3 preprocess 1,437 -> 870 us, C4 707 -> 405 us with this; at 1M the
    // per-warp atomics are as fast and the split kernels slower with it)
    __shared__ unsigned long long s_red_own[6][8];
    unsigned long long (*s_red)[8] = late_red ? late_red : s_red_own;
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_red[0][w] = kmin_inv; s_red[1][w] = kmax; s_red[2][w] = frustum;
        s_red[3][w] = coarse; s_red[4][w] = tight; s_red[5][w] = visible;
    }
    if (late_red) return; // flushed by the caller after its next CTA barrier
    __syncthreads();
    flush_cta_counters(s_red, ctr);
}

template <int BC>
__global__ void __launch_bounds__(256, 2) k_geometry(SceneDev s, FrameParams P, FrameDev f, DevCounters* ctr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < s.n;
    double mean[3] = {0.0, 0.0, 0.0}, c6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, opacity = 0.0;
    if (in) {
        for (int k = 0; k < 3; ++k) mean[k] = s.mean[k][i];
        for (int k = 0; k < 6; ++k) c6[k] = s.cov[k][i];
        opacity = s.opacity[i];
    }
    geometry_view<BC>(i, in, mean, c6, opacity, P, f, ctr);
}

// Multi-view K1a: each splat's camera-independent inputs are
// read once and projected into NV views (a batch of ps_render_views), each view
// writing its own frame arrays and counters.
template <int NV>
struct MultiView {
    FrameParams P[NV];
    FrameDev f[NV];
    DevCounters* ctr[NV];
};

template <int BC, int NV>
__global__ void __launch_bounds__(256, 3) k_geometry_mv(SceneDev s, MultiView<NV> mv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < s.n;
    double mean[3] = {0.0, 0.0, 0.0}, c6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, opacity = 0.0;
    if (in) {
        for (int k = 0; k < 3; ++k) mean[k] = s.mean[k][i];
        for (int k = 0; k < 6; ++k) c6[k] = s.cov[k][i];
        opacity = s.opacity[i];
    }
#pragma unroll 1
    for (int v = 0; v < NV; ++v) geometry_view<BC>(i, in, mean, c6, opacity, mv.P[v], mv.f[v], mv.ctr[v]);
}

// K1b for one view: SH colour from the splat's coefficients (in registers) and
// the fp32 blend record of a visible splat.
template <int BK>
__device__ __forceinline__ void shade_record(int64_t i, const double (&mean)[3], const float (&v)[48],
                                             const FrameParams& P, const FrameDev& f, double ca, double cb, double cc,
                                             double o, const double* qs_known = nullptr) {
    // view direction (mean - camera position), normalised; fp32 suffices for colour
    const float dx = static_cast<float>(mean[0] - P.campos[0]);
    const float dy = static_cast<float>(mean[1] - P.campos[1]);
    const float dz = static_cast<float>(mean[2] - P.campos[2]);
    const float nrm = sqrtf(dx * dx + dy * dy + dz * dz);
    const float inv = nrm > 0.f ? 1.0f / nrm : 0.f;
    float col[3];
    sh_color(v, P.cfg.sh_degree, dx * inv, dy * inv, dz * inv, col);
    if (P.cfg.clamp_before_blend) {
        col[0] = fminf(fmaxf(col[0], 0.f), 1.f);
        col[1] = fminf(fmaxf(col[1], 0.f), 1.f);
        col[2] = fminf(fmaxf(col[2], 0.f), 1.f);
    }
    float4 r0, r1;
    float2 r2;
    blend_record<BK>(ca, cb, cc, o, P, col[0], col[1], col[2], r0, r1, r2, qs_known);
    f.bl0[i] = r0;
    f.bl1[i] = r1;
    f.bl2[i] = r2;
}

template <int BK>
__device__ __forceinline__ void shade_view(int64_t i, const double (&mean)[3], const float (&v)[48],
                                           const FrameParams& P, const FrameDev& f) {
    if (f.key[i] == ~0ull) return;
    const double2 ab = f.conic_ab[i];
    const double2 cq = f.conic_cq[i];
    shade_record<BK>(i, mean, v, P, f, ab.x, ab.y, cq.x, f.opacity_eff[i]);
}

template <int NVS>
__device__ __forceinline__ void load_sh(const SceneDev& s, int64_t i, int sh_floats4, float (&v)[48]) {
#pragma unroll
    for (int j = 0; j < kShPlanes; ++j) {
        const float4 t = j < sh_floats4 ? s.sh4[j * s.n + i] : make_float4(0.f, 0.f, 0.f, 0.f); // plane-major: coalesced
        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
    }
}

template <int BK>
__global__ void __launch_bounds__(256) k_shade(SceneDev s, FrameParams P, FrameDev f) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s.n || f.key[i] == ~0ull) return;
    const double mean[3] = {s.mean[0][i], s.mean[1][i], s.mean[2][i]};
    float v[48];
    load_sh<1>(s, i, P.sh_floats4, v);
    shade_view<BK>(i, mean, v, P, f);
}

// K1 fused (K1a + K1b in one kernel, for the common culling x blend kernel
// pairs): the SH loads and colour of a visible splat follow its projection in
// the same thread, so the HBM-bound SH traffic overlaps the fp64-latency-bound
// geometry of other warps, and the conic / opacity stay in registers.
// MINB: CTAs per SM the registers are budgeted for; CTA_RED: counters reduced
// per CTA (above kFusedWarpCounters splats)
template <int BC, int BK, int MINB, bool CTA_RED>
__global__ void __launch_bounds__(256, MINB) k_preprocess(SceneDev s, FrameParams P, FrameDev f, DevCounters* ctr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < s.n;
    double mean[3] = {0.0, 0.0, 0.0}, c6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, opacity = 0.0;
    if (in) {
        for (int k = 0; k < 3; ++k) mean[k] = s.mean[k][i];
        for (int k = 0; k < 6; ++k) c6[k] = s.cov[k][i];
        opacity = s.opacity[i];
    }
    GeoOut g;
    // The CTA-wide steps (the tile window counts for K2 / K3 and, with
    // CTA_RED, the counter flush) run after the shading: no CTA barrier between
    // a warp's fp64 geometry and its SH stream (C2 -3 us, C3 -13 us, exp -8 us
    // against counting before the shading).
    __shared__ ulonglong2 s_late[256];
    __shared__ unsigned long long s_red[6][8];
    geometry_view<BC, CTA_RED>(i, in, mean, c6, opacity, P, f, ctr, &g, s_late, CTA_RED ? s_red : nullptr);
    if (g.visible) {
        float v[48];
        load_sh<1>(s, i, P.sh_floats4, v);
        const bool same = kThresholdIsBound<BC, BK> && !P.cfg.has_culling_kernel;
        shade_record<BK>(i, mean, v, P, f, g.a, g.b, g.c, g.o, same ? &g.x : nullptr);
    }
    if (f.tile_count) {
        const ulonglong2 wm = s_late[threadIdx.x];
        // (the rect is read only for a nonzero mask, i.e. a visible small rect:
        // tile indices < 2^16 like f.rect's)
        const int r[4] = {static_cast<int>(wm.y & 0xffffu), static_cast<int>((wm.y >> 16) & 0xffffu),
                          static_cast<int>((wm.y >> 32) & 0xffffu), static_cast<int>(wm.y >> 48)};
        tile_window_counts(wm.x != 0ull, r, wm.x, f, P); // (its CTA barriers order s_red too)
    } else if (CTA_RED) {
        __syncthreads();
    }
    if (CTA_RED) flush_cta_counters(s_red, ctr);
    pdl_trigger(); // K2 may be scheduled once every CTA is past its tile counts
}

// Multi-view K1b: the splat's SH coefficients (192 B, most of K1b's traffic)
// are read once for all NV views.
template <int BK, int NV>
__global__ void __launch_bounds__(256) k_shade_mv(SceneDev s, MultiView<NV> mv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    bool any = false;
#pragma unroll
    for (int k = 0; k < NV; ++k) any |= mv.f[k].key[i] != ~0ull;
    if (!any) return;
    const double mean[3] = {s.mean[0][i], s.mean[1][i], s.mean[2][i]};
    float v[48];
    load_sh<NV>(s, i, mv.P[0].sh_floats4, v);
#pragma unroll 1
    for (int k = 0; k < NV; ++k) shade_view<BK>(i, mean, v, mv.P[k], mv.f[k]);
}

// Fused multi-view K1 (the common cells): each view's geometry, then the SH
// coefficients loaded once and every view's colour / blend record, so the SH
// stream overlaps the fp64 chains of other warps as in the single-view fused K1.
template <int BC, int BK, int NV>
__global__ void __launch_bounds__(256, 3) k_preprocess_mv(SceneDev s, MultiView<NV> mv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < s.n;
    double mean[3] = {0.0, 0.0, 0.0}, c6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, opacity = 0.0;
    if (in) {
        for (int k = 0; k < 3; ++k) mean[k] = s.mean[k][i];
        for (int k = 0; k < 6; ++k) c6[k] = s.cov[k][i];
        opacity = s.opacity[i];
    }
#pragma unroll 1
    for (int v = 0; v < NV; ++v) geometry_view<BC>(i, in, mean, c6, opacity, mv.P[v], mv.f[v], mv.ctr[v]);
    if (!in) return;
    bool any = false;
#pragma unroll
    for (int k = 0; k < NV; ++k) any |= mv.f[k].key[i] != ~0ull;
    if (!any) return;
    float v[48];
    load_sh<NV>(s, i, mv.P[0].sh_floats4, v);
#pragma unroll 1
    for (int k = 0; k < NV; ++k) shade_view<BK>(i, mean, v, mv.P[k], mv.f[k]);
}

// ------------------------------------------------------------ K3 duplicate
// One thread per depth rank r: emits (tile id, splat index) for every tile of
// the rect that passes the tight test, in the rect's row-major order, at the
// rank's exclusive-scan offset. Pairs therefore come out in (depth, index)
// order globally, so a STABLE sort by tile id alone yields the reference's
// per-tile lists (raster.cpp:193-206).
__global__ void __launch_bounds__(256) k_duplicate(FrameDev f, FrameParams P, const uint32_t* order,
                                                   int64_t n) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t i = order[r];
    if (f.tcount[i] == 0) return;
    uint32_t o = f.offset[r];
    const ushort4 rc = f.rect[i];
    const double2 m = f.mean2d[i];
    const double2 ab = f.conic_ab[i];
    const double2 cq = f.conic_cq[i];
    const Sym2 cn{ab.x, ab.y, cq.x};
    const int ts = P.cfg.tile_size;
    for (int ty = rc.y; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.z; ++tx)
            if (tight_tile_test(cn, m.x, m.y, cq.y, tx, ty, ts)) {
                f.pkey[o] = static_cast<uint32_t>(ty * P.tiles_x + tx);
                f.pval[o] = i;
                ++o;
            }
}

// K3 (bucketed): splat indices into per-tile buckets. A CTA counts its pairs
// per tile in the shared window, reserves one contiguous slot range per
// distinct tile with a single global atomic, then hands out slots with shared
// atomics. Bucket order is arbitrary; K4 sorts each bucket by the reference's
// exact key.
// Rects larger than 8x8 tiles (rare): exact tests, direct global atomics.
// Out of line with scalar arguments so the common path keeps few registers.
__device__ __noinline__ void duplicate_big(uint32_t* __restrict__ pval, uint32_t* __restrict__ pkey, uint32_t k32,
                                           uint32_t* __restrict__ tile_count,
                                           double2 mm, double2 ab, double2 cq, int ts, int tiles_x, uint32_t i,
                                           int r0, int r1, int r2, int r3) {
    const TightSplat t = make_tight(Sym2{ab.x, ab.y, cq.x}, mm.x, mm.y, cq.y);
    for (int ty = r1; ty <= r3; ++ty)
        for (int tx = r0; tx <= r2; ++tx)
            if (tight_test_fast(t, tx, ty, ts)) {
                const uint32_t o = atomicAdd(&tile_count[ty * tiles_x + tx], 1u);
                pval[o] = i;
                pkey[o] = k32;
            }
}

// Heavy-first tile order for the blend (its CTA -> tile map), so the long tiles
// start in the first waves instead of trailing the grid: a counting sort of the
// tiles by bucket length in 8-pair classes, run by one extra 256-thread CTA of
// K3 (it finishes well inside K3; the blend follows K3 on the stream). Each
// thread takes consecutive tiles as runs of equal class, one shared atomic per
// run (neighbouring tiles mostly share a class; empty sky would otherwise
// serialise on one bin).
constexpr int kOrderBins = 512;
constexpr int kOrderChunk = 16;
static_assert(kOrderBins <= kWinCap, "the order bins reuse K3's window");

__device__ __forceinline__ int order_bin(const uint2 r) {
    return kOrderBins - 1 - static_cast<int>(min((r.y - r.x) >> 3, kOrderBins - 1u));
}

__device__ __noinline__ void build_tile_order(const uint2* __restrict__ ranges, int n_tiles,
                                              uint32_t* __restrict__ order, uint32_t* obin) {
    __shared__ uint32_t wsum[8];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int b = t; b < kOrderBins; b += 256) obin[b] = 0;
    __syncthreads();
    const int per = (n_tiles + 255) / 256;
    const int t0 = min(n_tiles, t * per), t1 = min(n_tiles, t0 + per);
    int cb = -1, ks = t0;
    for (int c0 = t0; c0 < t1; c0 += kOrderChunk) {
        int bin[kOrderChunk];
#pragma unroll
        for (int q = 0; q < kOrderChunk; ++q) bin[q] = c0 + q < t1 ? order_bin(ranges[c0 + q]) : -2;
#pragma unroll
        for (int q = 0; q < kOrderChunk; ++q)
            if (bin[q] != cb && bin[q] != -2) {
                if (cb >= 0) atomicAdd(&obin[cb], static_cast<uint32_t>(c0 + q - ks));
                cb = bin[q];
                ks = c0 + q;
            }
    }
    if (cb >= 0) atomicAdd(&obin[cb], static_cast<uint32_t>(t1 - ks));
    __syncthreads();
    const uint32_t h0 = obin[2 * t], h1 = obin[2 * t + 1];
    uint32_t x = h0 + h1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t pre = x - h0 - h1;
    for (int w = 0; w < warp; ++w) pre += wsum[w];
    obin[2 * t] = pre;
    obin[2 * t + 1] = pre + h0;
    __syncthreads();
    auto flush = [&](int b, int k0, int k1) {
        const uint32_t pos = atomicAdd(&obin[b], static_cast<uint32_t>(k1 - k0));
        for (int k = k0; k < k1; ++k) order[pos + (k - k0)] = static_cast<uint32_t>(k);
    };
    cb = -1;
    ks = t0;
    for (int c0 = t0; c0 < t1; c0 += kOrderChunk) {
        int bin[kOrderChunk];
#pragma unroll
        for (int q = 0; q < kOrderChunk; ++q) bin[q] = c0 + q < t1 ? order_bin(ranges[c0 + q]) : -2;
#pragma unroll
        for (int q = 0; q < kOrderChunk; ++q)
            if (bin[q] != cb && bin[q] != -2) {
                if (cb >= 0) flush(cb, ks, c0 + q);
                cb = bin[q];
                ks = c0 + q;
            }
    }
    if (cb >= 0) flush(cb, ks, t1);
}

__global__ void __launch_bounds__(256, 6) k_duplicate_buckets(FrameDev f, FrameParams P, int64_t n,
                                                               const DevCounters* __restrict__ ctr) {
    __shared__ uint32_t win[kWinCap];
    pdl_trigger(); // the blend / long sorts may be scheduled into freed slots
    pdl_wait();    // K2's cursors and key range
    if (pairs_overflow(f)) return; // speculative frame over capacity: re-run by the host
    int blk = static_cast<int>(blockIdx.x);
    if (f.tile_order) { // CTA 0 builds the blend's tile order
        if (blk == 0) {
            build_tile_order(f.ranges, P.tiles_x * P.tiles_y, f.tile_order, win);
            return;
        }
        --blk;
    }
    const int64_t i = static_cast<int64_t>(blk) * blockDim.x + threadIdx.x;
    // all of a splat's inputs are loaded at once (one memory round trip; the
    // rect / mask / key of an inactive splat are stale and unused)
    const int64_t ic = i < n ? i : 0;
    const uint32_t tc = f.tcount[ic];
    const ushort4 rc = f.rect[ic];
    const unsigned long long tm = f.tmask[ic];
    const unsigned long long kk = f.key[ic];
    const bool active = i < n && tc != 0;
    int r[4] = {0, 0, -1, -1};
    unsigned long long m0 = 0ull;
    bool small = false;
    uint32_t k32 = 0u; // coarse depth key stored next to every bucket entry (tile_sort.cuh)
    if (active) {
        k32 = coarse_key(kk, ~ctr->key_min, ctr->key_max);
        r[0] = rc.x; r[1] = rc.y; r[2] = rc.z; r[3] = rc.w;
        if (rect_is_small(r)) {
            small = true;
            m0 = tm;
        } else { // big rect: exact tests, direct atomics (rare)
            duplicate_big(f.pval, f.pkey, k32, f.tile_count, f.mean2d[i], f.conic_ab[i], f.conic_cq[i], P.cfg.tile_size,
                          P.tiles_x, static_cast<uint32_t>(i), r[0], r[1], r[2], r[3]);
        }
    }
    // the same CTA of K1 counted this window's pairs (geometry_view): reserve
    // each cell's bucket slots from those counts (one global atomic per cell)
    const int4 wr = f.win_rect[blk];
    Window W;
    W.x0 = wr.x; W.y0 = wr.y; W.w = wr.z; W.h = wr.w;
    W.ok = wr.z > 0;
    if (W.ok) {
        const uint32_t* wc = f.win_counts + static_cast<size_t>(blk) * kWinCap;
        for (int k = threadIdx.x; k < W.w * W.h; k += blockDim.x) {
            const uint32_t v = wc[k];
            win[k] = v ? atomicAdd(&f.tile_count[(W.y0 + k / W.w) * P.tiles_x + W.x0 + k % W.w], v) : 0u;
        }
        __syncthreads();
        unsigned long long m = m0;
        while (m) {
            const int b = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
            const uint32_t o = atomicAdd(&win[rect_bit_win(r, b, W)], 1u);
            f.pval[o] = static_cast<uint32_t>(i);
            f.pkey[o] = k32;
        }
    } else if (small) {
        unsigned long long m = m0;
        while (m) {
            const int b = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
            const uint32_t o = atomicAdd(&f.tile_count[rect_bit_tile(r, b, P.tiles_x)], 1u);
            f.pval[o] = static_cast<uint32_t>(i);
            f.pkey[o] = k32;
        }
    }
}

// ------------------------------------------------------------ K7 exact replay
// One WARP per flagged pixel: the reference's per-pixel loop in fp64
// (raster.cpp:250-283) over the pixel's tile list. The 32 lanes evaluate
// alpha for 32 consecutive list entries at once (independent); the
// transmittance chain, which is sequential, then runs over the accepted
// fragments in list order with every lane holding the same (T, r, g, b), so
// each operation happens in the reference's order and rounding. Colours are
// the same fp32 SH colours the fast path blends.
__global__ void __launch_bounds__(256) k_replay(FrameDev f, FrameParams P, DevCounters* ctr,
                                                float* out_rgb, float* out_t, int count_work) {
    const unsigned long long n_flags = ctr->replay_px;
    const int W = P.cam.width;
    const int ts = P.cfg.tile_size;
    const int lane = threadIdx.x & 31;
    const unsigned long long warp0 = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    const double eps = P.cfg.epsilon, floor_t = P.cfg.transmittance_floor;
    for (unsigned long long slot = warp0; slot < n_flags; slot += nwarps) {
        const uint32_t pix = f.flags[slot];
        const int px = static_cast<int>(pix % W), py = static_cast<int>(pix / W);
        const int tile = (py / ts) * P.tiles_x + (px / ts);
        const uint2 range = f.ranges[tile];
        double trans = 1.0, r = 0.0, g = 0.0, b = 0.0;
        unsigned long long evals = 0, blended = 0;
        bool done = false;
        for (uint32_t base = range.x; base < range.y && !done; base += 32) {
            const uint32_t j = base + lane;
            const bool valid = j < range.y;
            double alpha = 0.0;
            float cr = 0.f, cg = 0.f, cb = 0.f;
            bool acc = false;
            if (valid) {
                const uint32_t i = f.pval[j];
                const double2 m = f.mean2d[i];
                const double2 ab = f.conic_ab[i];
                const double2 cq = f.conic_cq[i];
                const double o = f.opacity_eff[i];
                const double dx = px + 0.5 - m.x;
                const double dy = py + 0.5 - m.y;
                const double q = ab.x * dx * dx + 2.0 * ab.y * dx * dy + cq.x * dy * dy;
                alpha = std_min(0.999, o * eval_kernel(P.cfg.kernel, q));
                acc = !(alpha < eps);
                if (acc) {
                    const float4 b1 = f.bl1[i];
                    const float2 b2 = f.bl2[i];
                    cr = b1.w; cg = b2.x; cb = b2.y;
                }
            }
            uint32_t mask = __ballot_sync(0xffffffffu, acc);
            const uint32_t nvalid = min(32u, range.y - base);
            int stop = -1;
            while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const double a = __shfl_sync(0xffffffffu, alpha, src);
                const double test_t = trans * (1.0 - a);
                if (test_t < floor_t) { stop = src; break; }
                const double w = a * trans;
                r += static_cast<double>(__shfl_sync(0xffffffffu, cr, src)) * w;
                g += static_cast<double>(__shfl_sync(0xffffffffu, cg, src)) * w;
                b += static_cast<double>(__shfl_sync(0xffffffffu, cb, src)) * w;
                trans = test_t;
                ++blended;
            }
            if (stop >= 0) {
                evals += static_cast<unsigned long long>(stop) + 1;
                done = true;
            } else {
                evals += nvalid;
            }
        }
        if (lane == 0) {
            out_rgb[3ull * pix + 0] = static_cast<float>(r);
            out_rgb[3ull * pix + 1] = static_cast<float>(g);
            out_rgb[3ull * pix + 2] = static_cast<float>(b);
            out_t[pix] = static_cast<float>(trans);
            if (f.replay_vals) f.replay_vals[slot] = make_double4(r, g, b, trans);
            if (count_work) {
                atomicAdd(&ctr->evals, evals);
                atomicAdd(&ctr->blended, blended);
            }
        }
    }
}

// ------------------------------------------------------------ scene covariance
// build_covariance3d (projection.cpp:24-34) once per upload, in this -fmad=false
// translation unit so the bits equal the reference's per-render computation.
__global__ void __launch_bounds__(256) k_scene_cov(SceneDev s) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const double scale[3] = {s.scale[0][i], s.scale[1][i], s.scale[2][i]};
    const double quat[4] = {s.rot[0][i], s.rot[1][i], s.rot[2][i], s.rot[3][i]};
    double c[9];
    covariance3d(scale, quat, c);
    s.cov[0][i] = c[0]; s.cov[1][i] = c[1]; s.cov[2][i] = c[2];
    s.cov[3][i] = c[4]; s.cov[4][i] = c[5]; s.cov[5][i] = c[8];
}

// ------------------------------------------------------------ launchers
int launch_preprocess(const SceneDev& s, const FrameParams& P, const FrameDev& f, DevCounters* ctr,
                      cudaStream_t st) {
    if (s.n == 0) return 0;
    const int blocks = static_cast<int>((s.n + 255) / 256);
    // fused K1 for the fitted-kernel cells of the reference's grid (main.cpp:315-323)
    // (3 CTAs per SM, 80 registers): at 1M 162 us against 191 at 2 CTAs and 201
    // for the split K1a / K1b below. Above 1.5M splats its frame counters are
    // reduced per CTA (geometry_view CTA_RED): with per-warp counter atomics the
    // fused kernel lost to the split ones at scale (C3 1,437 vs 1,027 us),
    // with per-CTA ones it wins there too (870 us)
#ifndef PS_K1_MINB
#define PS_K1_MINB 3
#endif
#ifndef PS_FUSED_WARP_COUNTERS
#define PS_FUSED_WARP_COUNTERS 1500000 // (0: per-CTA counters at every size; sanitizer builds)
#endif
    constexpr int64_t kFusedWarpCounters = PS_FUSED_WARP_COUNTERS;
#define PS_FUSED(BCV, BKV)                                                                 \
    if (P.bound_class == BCV && P.blend_class == BKV) {                                  \
        if (s.n <= kFusedWarpCounters)                                                   \
            k_preprocess<BCV, BKV, PS_K1_MINB, false><<<blocks, 256, 0, st>>>(s, P, f, ctr);      \
        else                                                                             \
            k_preprocess<BCV, BKV, PS_K1_MINB, true><<<blocks, 256, 0, st>>>(s, P, f, ctr);       \
        return 1;                                                                        \
    }
    PS_FUSED(kBcStp, kBkExp)
    PS_FUSED(kBcOaExp, kBkExp)
    PS_FUSED(kBcStp, kBkP1)
    PS_FUSED(kBcZero, kBkP1)
    PS_FUSED(kBcOaP1, kBkP1)
    PS_FUSED(kBcOaP2, kBkP2)
    PS_FUSED(kBcStp, kBkP3)
    PS_FUSED(kBcOaP3, kBkP3)
#undef PS_FUSED
    switch (P.bound_class) {
        case kBcStp: k_geometry<kBcStp><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        case kBcZero: k_geometry<kBcZero><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        case kBcOaExp: k_geometry<kBcOaExp><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        case kBcOaP1: k_geometry<kBcOaP1><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        case kBcOaP2: k_geometry<kBcOaP2><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        case kBcOaP3: k_geometry<kBcOaP3><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
        default: k_geometry<kBcGeneric><<<blocks, 256, 0, st>>>(s, P, f, ctr); break;
    }
    switch (P.blend_class) {
        case kBkExp: k_shade<kBkExp><<<blocks, 256, 0, st>>>(s, P, f); break;
        case kBkP1: k_shade<kBkP1><<<blocks, 256, 0, st>>>(s, P, f); break;
        case kBkP2: k_shade<kBkP2><<<blocks, 256, 0, st>>>(s, P, f); break;
        case kBkP3: k_shade<kBkP3><<<blocks, 256, 0, st>>>(s, P, f); break;
        default: k_shade<kBkGeneric><<<blocks, 256, 0, st>>>(s, P, f); break;
    }
    return 2;
}

namespace {
template <int NV>
void launch_mv(const SceneDev& s, const FrameParams* P, const FrameDev* f, DevCounters* const* ctr, cudaStream_t st) {
    MultiView<NV> mv;
    for (int k = 0; k < NV; ++k) {
        mv.P[k] = P[k];
        mv.f[k] = f[k];
        mv.ctr[k] = ctr[k];
    }
    const int blocks = static_cast<int>((s.n + 255) / 256);
    if (P[0].bound_class == kBcOaP1 && P[0].blend_class == kBkP1) {
        k_preprocess_mv<kBcOaP1, kBkP1, NV><<<blocks, 256, 0, st>>>(s, mv);
        return;
    }
    if (P[0].bound_class == kBcStp && P[0].blend_class == kBkExp) {
        k_preprocess_mv<kBcStp, kBkExp, NV><<<blocks, 256, 0, st>>>(s, mv);
        return;
    }
    switch (P[0].bound_class) {
        case kBcStp: k_geometry_mv<kBcStp, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBcZero: k_geometry_mv<kBcZero, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBcOaExp: k_geometry_mv<kBcOaExp, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBcOaP1: k_geometry_mv<kBcOaP1, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBcOaP2: k_geometry_mv<kBcOaP2, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBcOaP3: k_geometry_mv<kBcOaP3, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        default: k_geometry_mv<kBcGeneric, NV><<<blocks, 256, 0, st>>>(s, mv); break;
    }
    switch (P[0].blend_class) {
        case kBkExp: k_shade_mv<kBkExp, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBkP1: k_shade_mv<kBkP1, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBkP2: k_shade_mv<kBkP2, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        case kBkP3: k_shade_mv<kBkP3, NV><<<blocks, 256, 0, st>>>(s, mv); break;
        default: k_shade_mv<kBkGeneric, NV><<<blocks, 256, 0, st>>>(s, mv); break;
    }
}
} // namespace

void launch_preprocess_views(const SceneDev& s, const FrameParams* P, const FrameDev* f, DevCounters* const* ctr,
                             int nv, cudaStream_t st) {
    if (s.n == 0 || nv <= 0) return;
    if (nv == 1) (void)launch_preprocess(s, P[0], f[0], ctr[0], st);
    else if (nv == 2) launch_mv<2>(s, P, f, ctr, st);
    else if (nv == 3) launch_mv<3>(s, P, f, ctr, st);
    else launch_mv<kMaxFusedViews>(s, P, f, ctr, st);
}

void launch_scene_cov(const SceneDev& s, cudaStream_t st) {
    if (s.n == 0) return;
    k_scene_cov<<<static_cast<int>((s.n + 255) / 256), 256, 0, st>>>(s);
}

void launch_duplicate(const FrameDev& f, const FrameParams& P, const uint32_t* order, int64_t n,
                      cudaStream_t st) {
    if (n == 0) return;
    const int blocks = static_cast<int>((n + 255) / 256);
    k_duplicate<<<blocks, 256, 0, st>>>(f, P, order, n);
}

int launch_duplicate_buckets(const FrameDev& f, const FrameParams& P, int64_t n, const DevCounters* ctr,
                             cudaStream_t st) {
    const int blocks = static_cast<int>((n + 255) / 256) + (f.tile_order ? 1 : 0);
    if (blocks == 0) return 0;
    launch_pdl(k_duplicate_buckets, dim3(blocks), dim3(256), 0, st, f, P, n, ctr);
    return 1;
}

void launch_replay(const FrameDev& f, const FrameParams& P, DevCounters* ctr, float* out_rgb,
                   float* out_t, bool count_work, int sm_count, cudaStream_t st) {
    k_replay<<<sm_count * 4, 256, 0, st>>>(f, P, ctr, out_rgb, out_t, count_work ? 1 : 0);
}

} // namespace ps
