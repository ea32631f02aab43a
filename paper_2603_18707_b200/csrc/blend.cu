// blend.cu — K6: front-to-back alpha blending per tile (raster.cpp:227-301).
//
// One CTA per tile, one pixel per thread (tile_size^2 <= 1024). The tile's
// splat list is staged through shared memory in batches of blockDim records
// (gathered by splat index from the fp32 blend records written by K1, with the
// fp64 mean turned into tile-local fp32 coordinates on the way in).
//
// Per (pixel, splat) the fast path is
//     u = (dx + beta dy);  q = A u^2 + gamma dy^2;  skip unless q <= q_hi
// i.e. the reference's alpha < epsilon test (raster.cpp:269-271) moved into
// quadric space: for a kernel non-increasing in q, min(.999, o k(q)) >= eps
// <=> q <= q*(o). No MUFU on the skip path for any kernel; polynomial kernels
// evaluate alpha with FFMA only. q in [q_lo, q_hi] (the certified fp32 error
// band) is re-decided with the reference's fp64 arithmetic (exact_alpha_ge_eps).
// The transmittance test (raster.cpp:272-277) carries a per-pixel absolute
// error bound on T; a pixel whose test value lands inside that band around the
// floor is flagged and replayed exactly in fp64 by K7. Early termination: the CTA stops
// when no pixel is live (__syncthreads_count), the reference's `remaining == 0`.
#include "kernels.h"
#include "tile_sort.cuh"

namespace ps {

namespace {

struct BlendArgs {
    FrameParams P;
    const uint2* ranges;
    const uint32_t* pval;
    uint32_t* pval_w;                  // buckets to sort in the prologue (null: presorted)
    const unsigned long long* key;     // fp64 depth bits (sort key)
    const uint32_t* orig;              // original splat index (tie-break)
    const double2* mean2d;
    const float4* bl0;
    const float4* bl1;
    const float2* bl2;
    const double2* conic_ab;
    const double2* conic_cq;
    const double* opacity_eff;
    uint32_t* flags;
    DevCounters* ctr;
    float* out_rgb;
    float* out_t;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Blend kernel in fp64 for the exact decisions (set per frame, stream-ordered).
__constant__ ps_kernel c_exact_kernel;
__constant__ double c_exact_eps;

// eval_kernel (kernel.cpp:162-172) with explicitly rounded ops (never contracted)
__device__ double eval_kernel_rn(double x) {
    const ps_kernel& k = c_exact_kernel;
    if (k.kind == PS_KERNEL_EXPONENTIAL) return exp(dmul(-0.5, x));
    double p = k.coeffs[k.order];
    for (int i = k.order - 1; i >= 0; --i) p = dadd(dmul(p, x), k.coeffs[i]);
    if (k.kind == PS_KERNEL_POLY_RELU) return (p < 0.0) ? 0.0 : p;
    return x < k.first_root ? p : 0.0;
}

// The reference's alpha decision for pixel (gx, gy) and splat i, in its exact
// fp64 arithmetic (raster.cpp:262-271): dx = px + 0.5 - mx, q = a dx dx +
// 2 b dx dy + c dy dy, alpha = min(0.999, o k(q)); returns !(alpha < eps).
__device__ __noinline__ bool exact_alpha_ge_eps(const double2* __restrict__ mean2d,
                                                const double2* __restrict__ conic_ab,
                                                const double2* __restrict__ conic_cq,
                                                const double* __restrict__ opacity_eff, uint32_t i,
                                                int gx, int gy) {
    const double2 m = mean2d[i];
    const double2 ab = conic_ab[i];
    const double2 cq = conic_cq[i];
    const double o = opacity_eff[i];
    const double dx = dsub(dadd(static_cast<double>(gx), 0.5), m.x);
    const double dy = dsub(dadd(static_cast<double>(gy), 0.5), m.y);
    const double q = dadd(dadd(dmul(dmul(ab.x, dx), dx), dmul(dmul(dmul(2.0, ab.y), dx), dy)),
                          dmul(dmul(cq.x, dy), dy));
    const double v = dmul(o, eval_kernel_rn(q));
    const double alpha = (v < 0.999) ? v : 0.999;
    return !(alpha < c_exact_eps);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fp32 alpha of an accepted fragment. KIND 0: exponential (oval = log2 o);
// KIND 1: polynomial (oval = o), relu/piecewise semantics.
template <int KIND>
__device__ __forceinline__ float alpha_f32(float q, float oval, const KernelF32& kf) {
    if (KIND == 0) {
        return fminf(0.999f, ex2_approx(fmaf(q, -0.72134752044448170f, oval)));
    } else {
        float p = kf.c[kf.order];
        for (int j = kf.order - 1; j >= 0; --j) p = fmaf(p, q, kf.c[j]);
        if (kf.kind == PS_KERNEL_POLY_PIECEWISE && !(q < kf.first_root)) p = 0.0f;
        return fminf(0.999f, fmaxf(oval * p, 0.0f));
    }
}

template <int KIND, int MODE, bool COUNT>
__global__ void k_blend(const BlendArgs A) {
    extern __shared__ float4 smem[];
    const int nt = blockDim.x;
    float4* s0 = smem;
    float4* s1 = s0 + nt;
    float4* s2 = s1 + nt;
    uint32_t* si = reinterpret_cast<uint32_t*>(s2 + nt);

    const FrameParams& P = A.P;
    const int tile = blockIdx.x;
    const int tx = tile % P.tiles_x, ty = tile / P.tiles_x;
    const int ts = P.cfg.tile_size;
    const int W = P.cam.width, H = P.cam.height;
    const int px0 = tx * ts, py0 = ty * ts;
    const int t = threadIdx.x;
    const int lx = t % ts, ly = t / ts;
    const int gx = px0 + lx, gy = py0 + ly;
    const bool inside = (t < ts * ts) && gx < W && gy < H;
    const float xc = lx + 0.5f, yc = ly + 0.5f;
    const float eps = P.eps_f, floor_f = P.floor_f;

    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, eT = 0.0f;
    bool done = !inside, flagged = false;
    uint32_t term = 0xffffffffu, nbl = 0, nexact = 0;

    const uint2 range = A.ranges[tile];
    const int L = static_cast<int>(range.y - range.x);
    for (int base = 0; base < L; base += nt) {
        if (__syncthreads_count(!done) == 0) break;
        const int j = base + t;
        if (j < L) {
            const uint32_t i = A.pval[range.x + j];
            const double2 m = A.mean2d[i];
            const float4 b0 = A.bl0[i];
            const float4 b1 = A.bl1[i];
            const float2 b2 = A.bl2[i];
            s0[t] = make_float4(static_cast<float>(m.x - px0), static_cast<float>(m.y - py0), b0.x, b0.y);
            s1[t] = make_float4(b0.z, b0.w, b1.x, b1.y);
            s2[t] = make_float4(b1.z, b1.w, b2.x, b2.y);
            si[t] = i;
        }
        __syncthreads();
        const int cnt = min(nt, L - base);
        if (!done) {
            for (int k = 0; k < cnt; ++k) {
                const float4 v0 = s0[k];
                const float4 v1 = s1[k];
                const float dx = xc - v0.x, dy = yc - v0.y;
                const float u = fmaf(v0.w, dy, dx);
                const float q = fmaf(v0.z * u, u, v1.x * dy * dy);
                float alpha;
                if (MODE == kQuadricThreshold) {
                    if (!(q <= v1.y)) continue; // alpha < eps certainly (or pixel/splat pair skipped)
                    if (q >= v1.z) {            // inside the fp32 error band: decide in fp64
                        ++nexact;
                        if (!exact_alpha_ge_eps(A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, si[k], gx, gy)) continue;
                    }
                    alpha = alpha_f32<KIND>(q, v1.w, P.kf);
                } else {
                    alpha = alpha_f32<KIND>(q, v1.w, P.kf);
                    if (alpha < eps - v1.y) continue;
                    if (alpha < eps + v1.y) {
                        ++nexact;
                        if (!exact_alpha_ge_eps(A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, si[k], gx, gy)) continue;
                    }
                }
                const float4 v2 = s2[k];
                // absolute error bound of the fp32 transmittance (see blend_px)
                const float om = 1.0f - alpha;
                const float test_t = T * om;
                const float en = fmaf(2.5f * 5.9604645e-08f, test_t, fmaf(eT, om, T * v2.x));
                if (test_t < floor_f + en) {
                    done = true;
                    if (test_t < floor_f - en) term = static_cast<uint32_t>(base + k);
                    else flagged = true;
                    break;
                }
                eT = en;
                const float w = alpha * T;
                cr = fmaf(v2.y, w, cr);
                cg = fmaf(v2.z, w, cg);
                cb = fmaf(v2.w, w, cb);
                T = test_t;
                ++nbl;
            }
        }
    }

    if (inside) {
        const size_t pix = static_cast<size_t>(gy) * W + gx;
        A.out_rgb[3 * pix + 0] = cr;
        A.out_rgb[3 * pix + 1] = cg;
        A.out_rgb[3 * pix + 2] = cb;
        A.out_t[pix] = T;
        if (flagged) {
            const unsigned long long slot = atomicAdd(&A.ctr->replay_px, 1ull);
            A.flags[slot] = static_cast<uint32_t>(pix);
        }
    }
    // per-CTA sums of the reference's counters (raster.cpp:268,283); flagged
    // pixels are counted by the exact replay instead
    unsigned long long ev = 0, bl = 0;
    if (COUNT && inside && !flagged) {
        ev = term != 0xffffffffu ? term + 1u : static_cast<unsigned>(L);
        bl = nbl;
    }
    unsigned long long ex = nexact;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ev += __shfl_xor_sync(0xffffffffu, ev, o);
        bl += __shfl_xor_sync(0xffffffffu, bl, o);
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
    }
    if ((t & 31) == 0) {
        if (ev) atomicAdd(&A.ctr->evals, ev);
        if (bl) atomicAdd(&A.ctr->blended, bl);
        if (ex) atomicAdd(&A.ctr->exact_evals, ex);
    }
}

// ---------------------------------------------------------------- 16x16 fast path
// tile_size == 16: 128 threads, two pixels per thread in the same row (x and
// x+8), so the per-row terms (dy, the row-shifted centre, gamma dy^2) are
// shared. Batches of 128 records live in static shared memory (immediate
// offsets in the inner loop) and the next batch is prefetched into registers
// while the current one is blended. A finished pixel gets x = NaN, which makes
// its quadric NaN and the skip test `!(q <= q_hi)` true: no per-pixel branch.
constexpr int kB16 = 128;
constexpr float kNaNf = __builtin_nanf("");

struct Px {
    float x;      // tile-local pixel-centre x (NaN once the pixel is finished)
    float T, r, g, b, eT;
    uint32_t term, nbl;
    bool flagged;
};

// Shared-memory record of one staged splat (tile-local, fp32):
//   a = {mx, my, A, beta}  b = {gamma, q_hi, q_lo, K0}  c = {g_alpha, r, g, b}
//   d = {K1, K2, K3, splat index bits}   box = {x_lo, x_hi, y_lo, y_hi}
// K_j = o c_j folds the opacity into the polynomial (K0 = log2 o for exp);
// box is the axis-aligned extent of {q <= q_hi} (+ margin) used for warp culling.
template <int KIND, int ORDER, int MODE, bool COUNT>
__device__ __forceinline__ void blend_px(Px& p, float q, const float4& sb, const float4& sc, const float4& sd,
                                         const BlendArgs& A, int gx, int gy, int jpos, uint32_t& nexact) {
    float alpha;
    if (MODE == kQuadricThreshold) {
        if (q >= sb.z) { // inside the certified fp32 error band: decide with fp64
            ++nexact;
            if (!exact_alpha_ge_eps(A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, __float_as_uint(sd.w), gx, gy))
                return;
        }
        // Accepted fragments have q < q* + Gq < first_root, where the ReLU /
        // piecewise cut-offs are inactive: alpha = min(.999, sum K_j q^j).
        if (KIND == 0) {
            alpha = fminf(0.999f, ex2_approx(fmaf(q, -0.72134752044448170f, sb.w)));
        } else {
            float pq = ORDER == 1 ? sd.x : ORDER == 2 ? sd.y : sd.z;
            if (ORDER >= 3) pq = fmaf(pq, q, sd.y);
            if (ORDER >= 2) pq = fmaf(pq, q, sd.x);
            alpha = fminf(0.999f, fmaf(pq, q, sb.w));
        }
    } else {
        // non-monotone kernel: full ReLU / piecewise semantics, guard on alpha
        const KernelF32& kf = A.P.kf;
        float pq = kf.c[kf.order];
        for (int j = kf.order - 1; j >= 0; --j) pq = fmaf(pq, q, kf.c[j]);
        if (kf.kind == PS_KERNEL_POLY_PIECEWISE && !(q < kf.first_root)) pq = 0.0f;
        alpha = KIND == 0 ? fminf(0.999f, ex2_approx(fmaf(q, -0.72134752044448170f, sb.w)))
                          : fminf(0.999f, fmaxf(sb.w * pq, 0.0f)); // K0 = o here
        if (alpha < A.P.eps_f - sb.y) return;
        if (alpha < A.P.eps_f + sb.y) {
            ++nexact;
            if (!exact_alpha_ge_eps(A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, __float_as_uint(sd.w), gx, gy))
                return;
        }
    }
    // Transmittance decision (raster.cpp:272-277) with a running ABSOLUTE error
    // bound e >= |T_fp32 - T_ref|: with g = the splat's |alpha_fp32 - alpha_ref|
    // bound (sc.x), e' = e (1 - alpha) + T g + 2.5u T' covers the error of
    // test_t = T (1 - alpha) (two fp32 roundings, u = 2^-24). The reference
    // terminates iff its test_t < floor: certain if test_t + e' < floor,
    // certainly not if test_t - e' >= floor, otherwise the pixel is replayed.
    const float om = 1.0f - alpha;
    const float test_t = p.T * om;
    const float en = fmaf(2.5f * 5.9604645e-08f, test_t, fmaf(p.eT, om, p.T * sc.x));
    const float fl = A.P.floor_f;
    if (test_t < fl + en) {
        if (test_t < fl - en) {
            if (COUNT) p.term = static_cast<uint32_t>(jpos);
        } else {
            p.flagged = true;
        }
        p.x = kNaNf; // finished
        return;
    }
    p.eT = en;
    const float w = alpha * p.T;
    p.r = fmaf(sc.y, w, p.r);
    p.g = fmaf(sc.z, w, p.g);
    p.b = fmaf(sc.w, w, p.b);
    p.T = test_t;
    if (COUNT) ++p.nbl;
}

template <int KIND, int ORDER, int MODE, bool COUNT>
__global__ void __launch_bounds__(128, 6) k_blend16(const BlendArgs A) {
    // Shared memory: the bucket sort's workspace; once the tile's list is
    // sorted (it ends in sm[0, 1024)), the staging records overlay the rest.
    using SortSm = TileSortSmem<128, 16>;
    union __align__(16) Smem {
        uint32_t sort[SortSm::WORDS];
        struct {
            uint32_t list[SortSm::CAP]; // the sorted bucket (sort_one_tile leaves it here)
            float4 a[kB16], b[kB16], c[kB16], d[kB16], e[kB16];
        } st;
    };
    __shared__ Smem S;
    uint32_t* sm = S.sort;
    float4* sA = S.st.a;
    float4* sB = S.st.b;
    float4* sC = S.st.c;
    float4* sD = S.st.d;
    float4* sE = S.st.e;

    const FrameParams& P = A.P;
    const int tile = blockIdx.x;
    const int tx = tile % P.tiles_x, ty = tile / P.tiles_x;
    const int W = P.cam.width, H = P.cam.height;
    const int px0 = tx * 16, py0 = ty * 16;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int lx = t & 7, ly = (warp << 2) + (lane >> 3);
    const int gy = py0 + ly;
    const float yc = ly + 0.5f;
    // this warp's rows of pixel centres, for the culling test
    const float wy_lo = (warp << 2) + 0.5f, wy_hi = (warp << 2) + 3.5f;
    Px p0{(gy < H && px0 + lx < W) ? lx + 0.5f : kNaNf, 1.f, 0.f, 0.f, 0.f, 0.f, 0xffffffffu, 0u, false};
    Px p1{(gy < H && px0 + lx + 8 < W) ? lx + 8.5f : kNaNf, 1.f, 0.f, 0.f, 0.f, 0.f, 0xffffffffu, 0u, false};
    const bool in0 = p0.x == p0.x, in1 = p1.x == p1.x;
    uint32_t nexact = 0;
    const float c0 = P.kf.c[0], c1 = P.kf.c[1], c2 = P.kf.c[2], c3 = P.kf.c[3];

    const uint2 range = A.ranges[tile];
    const int L = static_cast<int>(range.y - range.x);
    // the tile's list in (depth, index) order: sorted here for buckets that fit
    // one CTA, presorted in global memory otherwise
    const uint32_t* list = A.pval + range.x;
    if (A.pval_w && L > 1 && L <= SortSm::CAP) {
        list = sort_one_tile<128, 16>(range, A.pval_w, A.key, A.orig, sm);
        __syncthreads();
    }
    double2 pm = make_double2(0.0, 0.0);
    float4 pb0 = make_float4(0.f, 0.f, 0.f, -1.f), pb1 = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 pb2 = make_float2(0.f, 0.f);
    uint32_t pi = 0;
    if (t < L) {
        pi = list[t];
        pm = A.mean2d[pi];
        pb0 = A.bl0[pi];
        pb1 = A.bl1[pi];
        pb2 = A.bl2[pi];
    }
    for (int base = 0; base < L; base += kB16) {
        const bool live = (p0.x == p0.x) || (p1.x == p1.x);
        if (__syncthreads_count(live) == 0) break;
        {   // stage the record prefetched for this batch
            const float mx = static_cast<float>(pm.x - px0), my = static_cast<float>(pm.y - py0);
            const float Aq = pb0.x, beta = pb0.y, gamma = pb0.z, qhi = pb0.w;
            sA[t] = make_float4(mx, my, Aq, beta);
            const float o = pb1.y;
            float K0 = o, K1 = 0.f, K2 = 0.f, K3 = 0.f;
            if (KIND == 1 && MODE == kQuadricThreshold) {
                K0 = o * c0; K1 = o * c1; K2 = o * c2; K3 = o * c3;
            }
            sB[t] = make_float4(gamma, qhi, pb1.x, K0);
            sC[t] = make_float4(pb1.z, pb1.w, pb2.x, pb2.y);
            sD[t] = make_float4(K1, K2, K3, __uint_as_float(pi));
            // extent of {q <= q_hi}: |x - mx| <= sqrt(q_hi (beta^2/gamma + 1/A)), |y - my| <= sqrt(q_hi / gamma)
            // (evaluated at q_hi + 2 Gq, Gq = (q_hi - q_lo)/2, so a culled pixel has q_fp32 > q_hi)
            const float qb = qhi + (qhi - pb1.x);
            float hx = sqrtf(qb * (beta * beta / gamma + 1.0f / Aq));
            float hy = sqrtf(qb / gamma);
            hx = hx * 1.001f + 1e-3f;
            hy = hy * 1.001f + 1e-3f;
            if (MODE != kQuadricThreshold || !(qhi < 3.0e38f)) { hx = INFINITY; hy = INFINITY; }
            if (!(qhi >= 0.f)) { hx = -1.f; hy = -1.f; } // never reaches epsilon (or NaN)
            sE[t] = make_float4(mx - hx, mx + hx, my - hy, my + hy);
        }
        __syncthreads();
        const int nb = base + kB16;
        if (nb + t < L) { // prefetch the next batch while this one is blended
            pi = list[nb + t];
            pm = A.mean2d[pi];
            pb0 = A.bl0[pi];
            pb1 = A.bl1[pi];
            pb2 = A.bl2[pi];
        }
        const int cnt = min(kB16, L - base);
        if (!__any_sync(0xffffffffu, live)) continue;
        for (int g = 0; g < kB16 / 32; ++g) {
            const int k0 = g * 32;
            if (k0 >= cnt) break;
            // warp culling: splats whose box misses this warp's 16x4 strip
            const float4 e = sE[k0 + lane];
            const bool hit = (k0 + lane < cnt) && e.x <= 15.5f && e.y >= 0.5f && e.z <= wy_hi && e.w >= wy_lo;
            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
            // phase 1: candidate bitmasks (q <= q_hi) of both pixels over the 32
            // splats, branch-free per pixel (the per-splat skip is warp-uniform)
            uint32_t m0 = 0u, m1 = 0u;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                if (hm & (1u << k)) {
                    const float4 a = sA[k0 + k];
                    const float4 b = sB[k0 + k];
                    const float dy = yc - a.y;
                    const float mrow = fmaf(-a.w, dy, a.x);
                    const float R = b.x * dy * dy;
                    const float u0 = p0.x - mrow, u1 = p1.x - mrow;
                    const float q0 = fmaf(a.z * u0, u0, R);
                    const float q1 = fmaf(a.z * u1, u1, R);
                    if (q0 <= b.y) m0 |= 1u << k;
                    if (q1 <= b.y) m1 |= 1u << k;
                }
            }
            // phase 2: each pixel's candidates in list order
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                Px& p = side ? p1 : p0;
                uint32_t m = side ? m1 : m0;
                const int gx = px0 + lx + (side ? 8 : 0);
                while (m) {
                    const int k = k0 + __ffs(m) - 1;
                    m &= m - 1;
                    const float4 a = sA[k];
                    const float4 b = sB[k];
                    const float dy = yc - a.y;
                    const float u = p.x - fmaf(-a.w, dy, a.x);
                    const float q = fmaf(a.z * u, u, b.x * dy * dy);
                    blend_px<KIND, ORDER, MODE, COUNT>(p, q, b, sC[k], sD[k], A, gx, gy, base + k, nexact);
                    if (!(p.x == p.x)) m = 0u; // finished or flagged
                }
            }
        }
    }

    unsigned long long ev = 0, bl = 0;
    auto finish = [&](Px& p, bool inside, int gx) {
        if (!inside) return;
        const size_t pix = static_cast<size_t>(gy) * W + gx;
        A.out_rgb[3 * pix + 0] = p.r;
        A.out_rgb[3 * pix + 1] = p.g;
        A.out_rgb[3 * pix + 2] = p.b;
        A.out_t[pix] = p.T;
        if (p.flagged) {
            const unsigned long long slot = atomicAdd(&A.ctr->replay_px, 1ull);
            A.flags[slot] = static_cast<uint32_t>(pix);
        } else if (COUNT) {
            ev += p.term != 0xffffffffu ? p.term + 1u : static_cast<unsigned>(L);
            bl += p.nbl;
        }
    };
    finish(p0, in0, px0 + lx);
    finish(p1, in1, px0 + lx + 8);
    unsigned long long ex = nexact;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ev += __shfl_xor_sync(0xffffffffu, ev, o);
        bl += __shfl_xor_sync(0xffffffffu, bl, o);
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
    }
    if (lane == 0) {
        if (ev) atomicAdd(&A.ctr->evals, ev);
        if (bl) atomicAdd(&A.ctr->blended, bl);
        if (ex) atomicAdd(&A.ctr->exact_evals, ex);
    }
}

template <int KIND, int ORDER, int MODE>
void launch16(const BlendArgs& a, int n_tiles, bool count, cudaStream_t st) {
    if (count) k_blend16<KIND, ORDER, MODE, true><<<n_tiles, 128, 0, st>>>(a);
    else k_blend16<KIND, ORDER, MODE, false><<<n_tiles, 128, 0, st>>>(a);
}

template <int MODE>
void launch16_kind(const BlendArgs& a, int n_tiles, bool count, cudaStream_t st) {
    const KernelF32& kf = a.P.kf;
    if (kf.kind == PS_KERNEL_EXPONENTIAL) launch16<0, 1, MODE>(a, n_tiles, count, st);
    else if (kf.order == 1) launch16<1, 1, MODE>(a, n_tiles, count, st);
    else if (kf.order == 2) launch16<1, 2, MODE>(a, n_tiles, count, st);
    else launch16<1, 3, MODE>(a, n_tiles, count, st);
}

template <int KIND, int MODE>
void launch_t(const BlendArgs& a, int n_tiles, int nt, size_t smem, bool count, cudaStream_t st) {
    if (count) k_blend<KIND, MODE, true><<<n_tiles, nt, smem, st>>>(a);
    else k_blend<KIND, MODE, false><<<n_tiles, nt, smem, st>>>(a);
}

} // namespace

int launch_blend(const FrameDev& f, const FrameParams& P, const uint32_t* pair_vals, uint32_t* sort_in_place,
                 const uint32_t* orig, DevCounters* ctr, BlendOut out, bool count_work, cudaStream_t st) {
    BlendArgs a;
    a.P = P;
    a.ranges = f.ranges;
    a.pval = pair_vals;
    a.pval_w = sort_in_place;
    a.key = f.key;
    a.orig = orig;
    a.mean2d = f.mean2d;
    a.bl0 = f.bl0;
    a.bl1 = f.bl1;
    a.bl2 = f.bl2;
    a.conic_ab = f.conic_ab;
    a.conic_cq = f.conic_cq;
    a.opacity_eff = f.opacity_eff;
    a.flags = f.flags;
    a.ctr = ctr;
    a.out_rgb = out.rgb;
    a.out_t = out.t;
    const int ts = P.cfg.tile_size;
    const int nt = ((ts * ts + 31) / 32) * 32;
    const size_t smem = static_cast<size_t>(nt) * (3 * sizeof(float4) + sizeof(uint32_t));
    const int n_tiles = P.tiles_x * P.tiles_y;
    if (n_tiles == 0) return 0;
    cudaMemcpyToSymbolAsync(c_exact_kernel, &P.cfg.kernel, sizeof(ps_kernel), 0, cudaMemcpyHostToDevice, st);
    cudaMemcpyToSymbolAsync(c_exact_eps, &P.cfg.epsilon, sizeof(double), 0, cudaMemcpyHostToDevice, st);
    if (ts == 16) {
        if (P.threshold_mode == kQuadricThreshold) launch16_kind<kQuadricThreshold>(a, n_tiles, count_work, st);
        else launch16_kind<kAlphaThreshold>(a, n_tiles, count_work, st);
        return 1;
    }
    const bool expk = P.kf.kind == PS_KERNEL_EXPONENTIAL;
    if (P.threshold_mode == kQuadricThreshold) {
        if (expk) launch_t<0, kQuadricThreshold>(a, n_tiles, nt, smem, count_work, st);
        else launch_t<1, kQuadricThreshold>(a, n_tiles, nt, smem, count_work, st);
    } else {
        if (expk) launch_t<0, kAlphaThreshold>(a, n_tiles, nt, smem, count_work, st);
        else launch_t<1, kAlphaThreshold>(a, n_tiles, nt, smem, count_work, st);
    }
    return 1;
}

} // namespace ps
