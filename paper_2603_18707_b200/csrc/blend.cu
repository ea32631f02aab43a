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
    double4* replay_vals;              // exact (r, g, b, T) per replayed pixel (optional)
    DevCounters* ctr;
    const DevCounters* gate;           // speculative frame: skip when pairs_total > pair_cap
    unsigned long long pair_cap;
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
                // absolute error bound of the fp32 transmittance (see cand_step)
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
// tile_size == 16: 128 threads; warp w owns the 8x8 block (w & 1, w >> 1) of the
// tile, lane L the pixels (L & 7, L >> 3) and (L & 7, 4 + (L >> 3)) of it.
// Batches of 128 records live in static shared memory and the next batch is
// prefetched into registers while the current one is blended. While staging a
// record, its thread also computes a conservative coverage mask of
// {q <= q_hi} over the tile's 256 pixel centres (one x-interval per row);
// per group of 32 records a warp bit-transposes its block's masks into one
// 32-record candidate mask per pixel, then walks both pixels' candidates in
// list order, one of each per step, re-deciding q <= q_hi exactly. A finished
// pixel gets x = NaN, so its later tests fail without a branch. Pixels whose
// decisions the fp32 error bounds cannot certify are replayed at the end of the
// CTA in exact fp64 from the tile's sorted list.
constexpr int kB16 = 128;
constexpr float kNaNf = __builtin_nanf("");
// byte offsets of the record planes a, b, c, d in the staging area
constexpr uint32_t kOffB = kB16 * 16, kOffC = 2 * kB16 * 16, kOffD = 3 * kB16 * 16;

struct Px {
    float x;      // tile-local pixel-centre x (NaN once the pixel is finished)
    float T, r, g, b, eT;
    uint32_t term, nbl;
    uint32_t flagged;
};

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Warp-wide 32x32 bit-matrix transpose: lane r holds row r (bit c = element
// (r, c)); returns column `lane` (bit r = element (r, lane)). Five block-swap
// steps; keep[s] / rot[s] are the lane's select mask and rotation for step s.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, const uint32_t (&keep)[5],
                                                     const uint32_t (&rot)[5]) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16 >> s);
        const uint32_t yr = __funnelshift_l(y, y, rot[s]);
        x = (x & keep[s]) | (yr & ~keep[s]);
    }
    return x;
}

// Conservative coverage of {q <= q_hi} over the 16 pixel centres of tile row
// `row`, as a 16-bit mask. Every pixel whose fp32 quadric (cand_step's exact
// expression, same dy and row centre) is <= q_hi is included: q_hi is inflated
// by the quadric's rounding (~5u relative) and the half-width by the
// approximate rcp/sqrt error plus an absolute margin; a pixel included in
// excess only costs one re-decided candidate step.
__device__ __forceinline__ uint32_t row_cover(int row, float mx, float my, float beta, float gamma, float qpad,
                                              float ia) {
    const float dy = (row + 0.5f) - my;
    const float rhs = fmaf(-gamma * dy, dy, qpad);
    const float mr = fmaf(-beta, dy, mx);
    float h = sqrt_approx(fmaxf(rhs, 0.0f) * ia);
    h = fmaf(h, 1.00002f, fmaf(fabsf(mr), 2e-6f, 1e-3f));
    if (!(rhs >= 0.0f)) h = -1.0f; // empty row
    const int lo = min(max(__float2int_ru(mr - h - 0.5f), 0), 16);
    const int hi = max(min(__float2int_rd(mr + h - 0.5f), 15), -1);
    return (0xFFFFu << lo) & (0xFFFFu >> (15 - hi));
}

// Shared-memory record of one staged splat (tile-local, fp32):
//   a = {mx, my, A, beta}  b = {gamma, q_hi, q_lo, K0}  c = {g_alpha, r, g, b}
//   d = {K1, K2, K3, splat index bits}   e = {x_lo, x_hi, y_lo, y_hi}
// K_j = o c_j folds the opacity into the polynomial (K0 = log2 o for exp);
// e is the axis-aligned extent of {q <= q_hi} (+ margin) used for warp culling.
//
// One candidate (q <= q_hi) of pixel p, at list position jpos; v = lane has one.
template <int KIND, int ORDER, int MODE, bool COUNT>
__device__ __forceinline__ void cand_step(Px& p, bool v, uint32_t rec, float yc, const FrameParams& P, int jpos) {
    const float4 a = lds128(rec);
    const float4 b = lds128(rec + kOffB);
    const float4 c = lds128(rec + kOffC);
    const float dy = yc - a.y;
    const float u = p.x - fmaf(-a.w, dy, a.x);
    const float q = fmaf(a.z * u, u, b.x * dy * dy);
    float alpha;
    bool amb, skip = false;
    if (MODE == kQuadricThreshold) {
        // the coverage masks are a superset: q > q_hi is a certain skip
        skip = !(q <= b.y);
        // q in the certified band [q_lo, q_hi]: the reference's alpha < eps is
        // undecided in fp32 -> exact replay of the pixel
        amb = q >= b.z;
        // accepted fragments have q < q* + Gq < first_root, where the ReLU /
        // piecewise cut-offs are inactive: alpha = min(.999, sum K_j q^j)
        if (KIND == 0) {
            alpha = fminf(0.999f, ex2_approx(fmaf(q, -0.72134752044448170f, b.w)));
        } else {
            float pq;
            if (ORDER == 1) {
                pq = lds32(rec + kOffD);
            } else {
                const float4 d = lds128(rec + kOffD);
                pq = ORDER == 2 ? d.y : d.z;
                if (ORDER >= 3) pq = fmaf(pq, q, d.y);
                pq = fmaf(pq, q, d.x);
            }
            alpha = fminf(0.999f, fmaf(pq, q, b.w));
        }
    } else {
        // non-monotone kernel: full ReLU / piecewise semantics, guard on alpha
        const KernelF32& kf = P.kf;
        float pq = kf.c[kf.order];
        for (int j = kf.order - 1; j >= 0; --j) pq = fmaf(pq, q, kf.c[j]);
        if (kf.kind == PS_KERNEL_POLY_PIECEWISE && !(q < kf.first_root)) pq = 0.0f;
        alpha = KIND == 0 ? fminf(0.999f, ex2_approx(fmaf(q, -0.72134752044448170f, b.w)))
                          : fminf(0.999f, fmaxf(b.w * pq, 0.0f)); // K0 = o here
        skip = alpha < P.eps_f - b.y;
        amb = !skip && alpha < P.eps_f + b.y;
    }
    // Transmittance decision (raster.cpp:272-277) with a running ABSOLUTE error
    // bound e >= |T_fp32 - T_ref|: with g = the splat's |alpha_fp32 - alpha_ref|
    // bound (c.x), e' = e (1 - alpha) + T g + 2.5u T' covers the error of
    // test_t = T (1 - alpha) (two fp32 roundings, u = 2^-24). The reference
    // terminates iff its test_t < floor: certain if test_t + e' < floor,
    // certainly not if test_t - e' >= floor, otherwise the pixel is replayed.
    const float om = 1.0f - alpha;
    const float tt = p.T * om;
    const float en = fmaf(2.5f * 5.9604645e-08f, tt, fmaf(p.eT, om, p.T * c.x));
    const float fl = P.floor_f;
    const bool live = v && !skip;
    if (__builtin_expect(live && (amb || tt < fl + en), 0)) {
        if (!amb && tt < fl - en) {
            if (COUNT) p.term = static_cast<uint32_t>(jpos);
        } else {
            p.flagged = 1u;
        }
        p.x = kNaNf; // finished
    } else if (live) {
        p.eT = en;
        const float w = alpha * p.T;
        p.r = fmaf(c.y, w, p.r);
        p.g = fmaf(c.z, w, p.g);
        p.b = fmaf(c.w, w, p.b);
        p.T = tt;
        if (COUNT) ++p.nbl;
    }
}

// alpha of (pixel (gx, gy), splat i) in the reference's exact fp64 arithmetic
// (raster.cpp:262-271; see exact_alpha_ge_eps)
__device__ __forceinline__ double exact_alpha(const BlendArgs& A, uint32_t i, double2 m, int gx, int gy) {
    const double2 ab = A.conic_ab[i];
    const double2 cq = A.conic_cq[i];
    const double o = A.opacity_eff[i];
    const double dx = dsub(dadd(static_cast<double>(gx), 0.5), m.x);
    const double dy = dsub(dadd(static_cast<double>(gy), 0.5), m.y);
    const double q = dadd(dadd(dmul(dmul(ab.x, dx), dx), dmul(dmul(dmul(2.0, ab.y), dx), dy)),
                          dmul(dmul(cq.x, dy), dy));
    const double v = dmul(o, eval_kernel_rn(q));
    return (v < 0.999) ? v : 0.999;
}

// Exact replay of one flagged pixel by a whole warp (the reference's per-pixel
// loop, raster.cpp:250-283, in fp64 with its operation order): alpha of 32 list
// entries in parallel, then the transmittance chain serially over the accepted
// ones. In quadric mode an entry with fp32 q > q_hi is certainly skipped by the
// reference (the same certified test the fast path uses), so only candidates
// reach the fp64 kernel evaluation.
template <int MODE, bool COUNT>
__device__ __forceinline__ void replay_pixel(const BlendArgs& A, const uint32_t* list, int L, int lxy, int px0,
                                          int py0, unsigned long long& ev, unsigned long long& bl) {
    const int lane = threadIdx.x & 31;
    const int lx = lxy & 15, ly = lxy >> 4;
    const int gx = px0 + lx, gy = py0 + ly;
    const float xc = lx + 0.5f, yc = ly + 0.5f;
    const double eps = c_exact_eps, floor_t = A.P.cfg.transmittance_floor;
    double trans = 1.0, r = 0.0, g = 0.0, b = 0.0;
    unsigned long long evals = 0, blended = 0;
    bool done = false;
    for (int base = 0; base < L && !done; base += 32) {
        const int j = base + lane;
        double alpha = 0.0;
        float cr = 0.f, cg = 0.f, cb = 0.f;
        bool acc = false;
        if (j < L) {
            const uint32_t i = list[j];
            const double2 m = A.mean2d[i];
            bool cand = true;
            if (MODE == kQuadricThreshold) {
                const float4 b0 = A.bl0[i];
                const float mx = static_cast<float>(m.x - px0), my = static_cast<float>(m.y - py0);
                const float dy = yc - my;
                const float u = xc - fmaf(-b0.y, dy, mx);
                const float q = fmaf(b0.x * u, u, b0.z * dy * dy);
                cand = q <= b0.w;
            }
            if (cand) {
                alpha = exact_alpha(A, i, m, gx, gy);
                acc = !(alpha < eps);
                if (acc) {
                    const float4 b1 = A.bl1[i];
                    const float2 b2 = A.bl2[i];
                    cr = b1.w; cg = b2.x; cb = b2.y;
                }
            }
        }
        uint32_t mask = __ballot_sync(0xffffffffu, acc);
        const int nvalid = min(32, L - base);
        int stop = -1;
        while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            const double a = __shfl_sync(0xffffffffu, alpha, src);
            const double test_t = dmul(trans, dsub(1.0, a));
            if (test_t < floor_t) { stop = src; break; }
            const double w = dmul(a, trans);
            r = dadd(r, dmul(static_cast<double>(__shfl_sync(0xffffffffu, cr, src)), w));
            g = dadd(g, dmul(static_cast<double>(__shfl_sync(0xffffffffu, cg, src)), w));
            b = dadd(b, dmul(static_cast<double>(__shfl_sync(0xffffffffu, cb, src)), w));
            trans = test_t;
            ++blended;
        }
        if (stop >= 0) {
            evals += static_cast<unsigned long long>(stop) + 1;
            done = true;
        } else {
            evals += static_cast<unsigned long long>(nvalid);
        }
    }
    if (lane == 0) {
        const size_t pix = static_cast<size_t>(gy) * A.P.cam.width + gx;
        A.out_rgb[3 * pix + 0] = static_cast<float>(r);
        A.out_rgb[3 * pix + 1] = static_cast<float>(g);
        A.out_rgb[3 * pix + 2] = static_cast<float>(b);
        A.out_t[pix] = static_cast<float>(trans);
        const unsigned long long slot = atomicAdd(&A.ctr->replay_px, 1ull);
        A.flags[slot] = static_cast<uint32_t>(pix);
        if (A.replay_vals) A.replay_vals[slot] = make_double4(r, g, b, trans);
        if (COUNT) {
            ev += evals;
            bl += blended;
        }
    }
}

template <int KIND, int ORDER, int MODE, bool COUNT>
__global__ void __launch_bounds__(128, 6) k_blend16(const BlendArgs A) {
    using SortSm = TileSortSmem<128, 16>;
    // Shared memory: the bucket sort's workspace; the sorted list starts at word
    // SortSm::LIST, the staging records (a, b, c, d planes + coverage words)
    // overlay the sort's dead arrays below it.
    __shared__ __align__(16) uint32_t S[SortSm::WORDS];
    __shared__ uint32_t s_nflag;
    __shared__ uint16_t s_flag[256];
    static_assert(4 * kB16 * 16 + 8 * kB16 * 4 <= SortSm::LIST * 4, "staging overlaps the sorted list");
    float4* sA = reinterpret_cast<float4*>(S);
    float4* sB = sA + kB16;
    float4* sC = sA + 2 * kB16;
    float4* sD = sA + 3 * kB16;
    uint32_t (*cover)[kB16] = reinterpret_cast<uint32_t (*)[kB16]>(sA + 4 * kB16); // [warp * 2 + half][record]
    const uint32_t s_rec = static_cast<uint32_t>(__cvta_generic_to_shared(sA));

    if (A.gate && A.gate->pairs_total > A.pair_cap) return; // over capacity: the host re-runs
    const FrameParams& P = A.P;
    const int tile = blockIdx.x;
    const int tx = tile % P.tiles_x, ty = tile / P.tiles_x;
    const int W = P.cam.width, H = P.cam.height;
    const int px0 = tx * 16, py0 = ty * 16;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int lx = ((warp & 1) << 3) + (lane & 7);      // both pixels' column
    const int ly0 = ((warp >> 1) << 3) + (lane >> 3);   // first pixel's row; second: ly0 + 4
    const float yc0 = ly0 + 0.5f, yc1 = ly0 + 4.5f;
    const bool col_in = px0 + lx < W;
    Px p0{(col_in && py0 + ly0 < H) ? lx + 0.5f : kNaNf, 1.f, 0.f, 0.f, 0.f, 0.f, 0xffffffffu, 0u, 0u};
    Px p1{(col_in && py0 + ly0 + 4 < H) ? lx + 0.5f : kNaNf, 1.f, 0.f, 0.f, 0.f, 0.f, 0xffffffffu, 0u, 0u};
    const bool in0 = p0.x == p0.x, in1 = p1.x == p1.x;
    const float c0 = P.kf.c[0], c1 = P.kf.c[1], c2 = P.kf.c[2], c3 = P.kf.c[3];
    uint32_t tkeep[5], trot[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int j = 16 >> k;
        const uint32_t m = k == 0 ? 0x0000FFFFu : k == 1 ? 0x00FF00FFu : k == 2 ? 0x0F0F0F0Fu : k == 3 ? 0x33333333u
                                                                                                     : 0x55555555u;
        tkeep[k] = (lane & j) ? ~m : m;
        trot[k] = (lane & j) ? 32u - j : static_cast<uint32_t>(j);
    }

    const uint2 range = A.ranges[tile];
    const int L = static_cast<int>(range.y - range.x);
    // the tile's list in (depth, index) order: sorted here for buckets that fit
    // one CTA, presorted in global memory otherwise
    const uint32_t* list = A.pval + range.x;
    if (A.pval_w && L > 1 && L <= SortSm::CAP) {
        list = sort_one_tile<128, 16, false>(range, A.pval_w, A.key, A.orig, S);
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
            // coverage of {q <= q_hi}: words (warp, half) hold 4 rows x 8 columns
            uint32_t cw[8];
            const bool full = MODE != kQuadricThreshold || !(qhi < 3.0e38f) || !(Aq > 0.0f) ||
                              !(gamma > 0.0f) || !(fabsf(beta) < 3.0e38f) || !(fabsf(mx) < 1.0e30f) ||
                              !(fabsf(my) < 1.0e30f);
            if (full || !(qhi >= 0.0f)) {
                const uint32_t v = full ? 0xFFFFFFFFu : 0u; // everything / never reaches epsilon
#pragma unroll
                for (int j = 0; j < 8; ++j) cw[j] = v;
            } else {
                const float qpad = qhi * 1.000004f;
                const float ia = rcp_approx(Aq) * 1.000002f;
#pragma unroll
                for (int g = 0; g < 4; ++g) { // rows 4g .. 4g+3 -> words of warps (g>>1)*2 + {0,1}, half g&1
                    const uint32_t r0 = row_cover(4 * g + 0, mx, my, beta, gamma, qpad, ia);
                    const uint32_t r1 = row_cover(4 * g + 1, mx, my, beta, gamma, qpad, ia);
                    const uint32_t r2 = row_cover(4 * g + 2, mx, my, beta, gamma, qpad, ia);
                    const uint32_t r3 = row_cover(4 * g + 3, mx, my, beta, gamma, qpad, ia);
                    const uint32_t t01 = __byte_perm(r0, r1, 0x5140), t23 = __byte_perm(r2, r3, 0x5140);
                    const int wl = (g >> 1) * 4 + (g & 1);     // (warp (g>>1)*2) * 2 + half
                    cw[wl] = __byte_perm(t01, t23, 0x5410);     // columns 0-7
                    cw[wl + 2] = __byte_perm(t01, t23, 0x7632); // columns 8-15
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) cover[j][t] = cw[j];
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
            // candidate masks: lane s holds record k0+s's coverage of this warp's
            // block; the transpose gives lane L's pixels' masks over the 32 records
            uint32_t w0 = 0u, w1 = 0u;
            if (k0 + lane < cnt) {
                w0 = cover[warp * 2][k0 + lane];
                w1 = cover[warp * 2 + 1][k0 + lane];
            }
            if (!__any_sync(0xffffffffu, (w0 | w1) != 0u)) continue;
            uint32_t m0 = warp_transpose32(w0, tkeep, trot);
            uint32_t m1 = warp_transpose32(w1, tkeep, trot);
            if (!(p0.x == p0.x)) m0 = 0u;
            if (!(p1.x == p1.x)) m1 = 0u;
            // both pixels' candidates in list order, one of each per step
            const uint32_t rb = s_rec + static_cast<uint32_t>(k0) * 16u;
            const int jb = base + k0;
            while ((m0 | m1) != 0u) {
                const bool v0 = m0 != 0u, v1 = m1 != 0u;
                // (bit 31 forced so an empty mask still yields a valid record slot)
                const uint32_t j0 = static_cast<uint32_t>(__ffs(m0 | 0x80000000u) - 1);
                const uint32_t j1 = static_cast<uint32_t>(__ffs(m1 | 0x80000000u) - 1);
                m0 &= m0 - 1u;
                m1 &= m1 - 1u;
                cand_step<KIND, ORDER, MODE, COUNT>(p0, v0, rb + j0 * 16u, yc0, P, jb + static_cast<int>(j0));
                cand_step<KIND, ORDER, MODE, COUNT>(p1, v1, rb + j1 * 16u, yc1, P, jb + static_cast<int>(j1));
                if (!(p0.x == p0.x)) m0 = 0u; // finished or flagged
                if (!(p1.x == p1.x)) m1 = 0u;
            }
        }
    }

    unsigned long long ev = 0, bl = 0;
    if (t == 0) s_nflag = 0;
    __syncthreads();
    auto finish = [&](Px& p, bool inside, int lyp) {
        if (!inside) return;
        if (p.flagged) { // replayed below
            s_flag[atomicAdd(&s_nflag, 1u)] = static_cast<uint16_t>(lyp * 16 + lx);
            return;
        }
        const size_t pix = static_cast<size_t>(py0 + lyp) * W + px0 + lx;
        A.out_rgb[3 * pix + 0] = p.r;
        A.out_rgb[3 * pix + 1] = p.g;
        A.out_rgb[3 * pix + 2] = p.b;
        A.out_t[pix] = p.T;
        if (COUNT) {
            ev += p.term != 0xffffffffu ? p.term + 1u : static_cast<unsigned>(L);
            bl += p.nbl;
        }
    };
    finish(p0, in0, ly0);
    finish(p1, in1, ly0 + 4);
    __syncthreads();
    const int nf = static_cast<int>(s_nflag);
    for (int k = warp; k < nf; k += 4)
        replay_pixel<MODE, COUNT>(A, list, L, s_flag[k], px0, py0, ev, bl);
    if (COUNT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ev += __shfl_xor_sync(0xffffffffu, ev, o);
            bl += __shfl_xor_sync(0xffffffffu, bl, o);
        }
        if (lane == 0) {
            if (ev) atomicAdd(&A.ctr->evals, ev);
            if (bl) atomicAdd(&A.ctr->blended, bl);
        }
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
                 const uint32_t* orig, DevCounters* ctr, BlendOut out, bool count_work, cudaStream_t st,
                 bool* replay_fused) {
    *replay_fused = false;
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
    a.replay_vals = f.replay_vals;
    a.ctr = ctr;
    a.gate = f.gate;
    a.pair_cap = f.pair_cap;
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
        *replay_fused = true; // flagged pixels are replayed inside k_blend16
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
