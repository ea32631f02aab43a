// blend.cu — K6: front-to-back alpha blending per tile (raster.cpp:227-301).
//
// Two kernels. k_blend16 (tile_size 16, the reference default): 128 threads per
// tile, a pixel PAIR per thread in packed f32x2, the tile's bucket sorted in
// its prologue (only the prefix the walk needs, tile_sort.cuh), records staged
// through shared memory in record-local fp32 coordinates with per-record
// coverage masks, and the exact fp64 replay of flagged pixels fused at the end
// (see the comments above k_blend16). k_blend (other tile sizes): one pixel per
// thread, tiles above 32x32 in chunks of 1024 pixels, tile-local coordinates,
// replay by K7 (exact_kernels.cu k_replay).
//
// Per (pixel, splat) the fast path is
//     u = (dx + beta dy);  q = A u^2 + gamma dy^2;  skip unless q <= q_hi
// i.e. the reference's alpha < epsilon test (raster.cpp:269-271) moved into
// quadric space: for a kernel non-increasing in q, min(.999, o k(q)) >= eps
// <=> q <= q*(o). No MUFU on the skip path for any kernel; polynomial kernels
// evaluate alpha with FFMA only. q in [q_lo, q_hi] (the certified fp32 error
// band) is re-decided with the reference's fp64 arithmetic. The transmittance
// test (raster.cpp:272-277) carries certified bounds on the reference's T; a
// pixel whose test lands inside the band around the floor is flagged and
// replayed exactly in fp64. Early termination: the CTA stops when no pixel is
// live (__syncthreads_count), the reference's `remaining == 0`.
#include <algorithm>

#include "kernels.h"
#include "tile_sort.cuh"

namespace ps {

namespace {

struct BlendArgs {
    FrameParams P;
    const uint2* ranges;
    const uint32_t* order;             // CTA -> tile (longest bucket first; null: row-major)
    const uint32_t* pval;
    uint32_t* pval_w;                  // buckets to sort in the prologue (null: presorted)
    const uint32_t* pkey;              // coarse depth key per bucket entry (K3)
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
    DevCounters* publish;              // pinned host copy of the counters (last CTA writes it), or null
    uint32_t* zero_counts;             // with publish: per-tile counts, zeroed for the next frame
    const DevCounters* gate;           // speculative frame: skip when pairs_total > pair_cap
    unsigned long long pair_cap;
    float* out_rgb;
    float* out_t;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }


// eval_kernel (kernel.cpp:162-172) with explicitly rounded ops (never contracted)
__device__ double eval_kernel_rn(const ps_kernel& k, double x) {
    if (k.kind == PS_KERNEL_EXPONENTIAL) return exp(dmul(-0.5, x));
    double p = k.coeffs[k.order];
    for (int i = k.order - 1; i >= 0; --i) p = dadd(dmul(p, x), k.coeffs[i]);
    if (k.kind == PS_KERNEL_POLY_RELU) return (p < 0.0) ? 0.0 : p;
    return x < k.first_root ? p : 0.0;
}

// The reference's alpha decision for pixel (gx, gy) and splat i, in its exact
// fp64 arithmetic (raster.cpp:262-271): dx = px + 0.5 - mx, q = a dx dx +
// 2 b dx dy + c dy dy, alpha = min(0.999, o k(q)); returns !(alpha < eps).
__device__ __noinline__ bool exact_alpha_ge_eps(const ps_kernel& kern, double eps,
                                                const double2* __restrict__ mean2d,
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
    const double v = dmul(o, eval_kernel_rn(kern, q));
    const double alpha = (v < 0.999) ? v : 0.999;
    return !(alpha < eps);
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
__global__ void __launch_bounds__(1024) k_blend(const BlendArgs A) {
    extern __shared__ float4 smem[];
    const int nt = blockDim.x;
    float4* s0 = smem;
    float4* s1 = s0 + nt;
    float4* s2 = s1 + nt;
    uint32_t* si = reinterpret_cast<uint32_t*>(s2 + nt);

    const FrameParams& P = A.P;
    const int tile = A.order ? static_cast<int>(A.order[blockIdx.x]) : static_cast<int>(blockIdx.x);
    const int tx = tile % P.tiles_x, ty = tile / P.tiles_x;
    const int ts = P.cfg.tile_size;
    const int W = P.cam.width, H = P.cam.height;
    const int px0 = tx * ts, py0 = ty * ts;
    const int t = threadIdx.x;
    const float eps = P.eps_f, floor_f = P.floor_f;
    const uint2 range = A.ranges[tile];
    const int L = static_cast<int>(range.y - range.x);
    unsigned long long ev = 0, bl = 0, ex = 0;

    // Tiles of more than 1024 pixels (tile_size > 32, which the reference
    // accepts: raster.cpp:13-23, 212-308) are blended in chunks of blockDim
    // pixels, each walking the tile's whole list; one chunk otherwise.
    const int npix = ts * ts;
    for (int p0 = 0; p0 < npix; p0 += nt) {
        const int p = p0 + t;
        const int lx = p % ts, ly = p / ts;
        const int gx = px0 + lx, gy = py0 + ly;
        const bool inside = (p < npix) && gx < W && gy < H;
        const float xc = lx + 0.5f, yc = ly + 0.5f;

        float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, eT = 0.0f;
        bool done = !inside, flagged = false;
        uint32_t term = 0xffffffffu, nbl = 0, nexact = 0;

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
                            if (!exact_alpha_ge_eps(P.cfg.kernel, P.cfg.epsilon, A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, si[k], gx, gy)) continue;
                        }
                        alpha = alpha_f32<KIND>(q, v1.w, P.kf);
                    } else {
                        alpha = alpha_f32<KIND>(q, v1.w, P.kf);
                        if (alpha < eps - v1.y) continue;
                        if (alpha < eps + v1.y) {
                            ++nexact;
                            if (!exact_alpha_ge_eps(P.cfg.kernel, P.cfg.epsilon, A.mean2d, A.conic_ab, A.conic_cq, A.opacity_eff, si[k], gx, gy)) continue;
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
        if (COUNT && inside && !flagged) {
            ev += term != 0xffffffffu ? term + 1u : static_cast<unsigned>(L);
            bl += nbl;
        }
        ex += nexact;
    }
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
// tile, lane L the horizontal pixel PAIR (2 (L & 3), 2 (L & 3) + 1) of block row
// L >> 2. Both pixels of a pair walk the same records: one record load, one
// set of row terms (dy, row centre, gamma dy^2) per step, and the per-pixel
// arithmetic in packed f32x2 (FFMA2 / FMUL2 / FADD2 with broadcast operands).
// Batches of 128 records live in static shared memory and the next batch is
// prefetched into registers while the current one is blended. While staging a
// record, its thread also computes a conservative coverage mask of
// {q <= q_hi} over the tile's 128 pixel pairs (one x-interval per row, widened
// to whole pairs); per group of 32 records each warp bit-transposes its
// block's words into one 32-record candidate mask per pair, then walks it in
// list order, re-deciding q <= q_hi exactly for each pixel. A finished pixel
// gets x = NaN, so its later tests fail without a branch. Pixels whose
// decisions the fp32 error bounds cannot certify are replayed at the end of the
// CTA in exact fp64 from the tile's sorted list.
constexpr int kB16 = 128;

constexpr float kNaNf = __builtin_nanf("");
// byte offsets of the record planes a, b, c, d in the staging area
constexpr int kRecs = kB16;
constexpr uint32_t kOffB = kRecs * 16, kOffC = 2 * kRecs * 16, kOffD = 3 * kRecs * 16, kOffE = 4 * kRecs * 16;

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
// steps; each lane's select mask and rotation per step come from its lane bits.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = s == 0 ? 0x0000FFFFu : s == 1 ? 0x00FF00FFu : s == 2 ? 0x0F0F0F0Fu : s == 3 ? 0x33333333u
                                                                                                     : 0x55555555u;
        const bool up = (lane & j) != 0;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        const uint32_t yr = __funnelshift_l(y, y, up ? 32u - j : static_cast<uint32_t>(j));
        const uint32_t keep = up ? ~m : m;
        x = (x & keep) | (yr & ~keep);
    }
    return x;
}

// ---- packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2 via the CUDA builtins;
// a broadcast scalar becomes a .F32 operand, a negation an operand modifier)
using F2 = float2;
__device__ __forceinline__ F2 f2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ F2 f2b(float s) { return make_float2(s, s); }
__device__ __forceinline__ float f2lo(F2 a) { return a.x; }
__device__ __forceinline__ float f2hi(F2 a) { return a.y; }
__device__ __forceinline__ F2 f2add(F2 a, F2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ F2 f2sub(F2 a, F2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ F2 f2mul(F2 a, F2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ F2 f2fma(F2 a, F2 b, F2 c) { return __ffma2_rn(a, b, c); }

// Conservative coverage of {q <= q_hi} over the 16 pixel centres of tile row
// `row`, widened to the row's 8 pixel pairs (bit k = pair (2k, 2k+1)). Every
// pixel whose fp32 quadric (the walk's exact expression, same dy and row
// centre) is <= q_hi is included: q_hi is inflated by the quadric's rounding
// (~5u relative) and the half-width by the approximate rcp/sqrt error plus an
// absolute margin; a pair included in excess only costs one skipped step.
// Rows r and r + 8 at once: the per-row floating-point work in packed f32x2
// (C2 blend -3.7 us against one row at a time).
__device__ __forceinline__ void row_pairs2(int row, float mx, float my, float beta, float gamma, float qpad,
                                           float ia, uint32_t& m_lo, uint32_t& m_hi) {
    const F2 dy = f2sub(f2(row + 0.5f, row + 8.5f), f2b(my));
    const F2 rhs = f2fma(f2mul(f2b(-gamma), dy), dy, f2b(qpad));
    const F2 mr = f2fma(f2b(-beta), dy, f2b(mx));
    const F2 h2 = f2mul(f2(fmaxf(f2lo(rhs), 0.0f), fmaxf(f2hi(rhs), 0.0f)), f2b(ia));
    F2 h = f2(sqrt_approx(f2lo(h2)), sqrt_approx(f2hi(h2)));
    h = f2fma(h, f2b(1.00002f), f2fma(f2(fabsf(f2lo(mr)), fabsf(f2hi(mr))), f2b(2e-6f), f2b(1e-3f)));
    const float h0 = f2lo(rhs) >= 0.0f ? f2lo(h) : -1.0f; // empty rows
    const float h1 = f2hi(rhs) >= 0.0f ? f2hi(h) : -1.0f;
    const F2 hh = f2(h0, h1);
    const F2 l = f2sub(f2sub(mr, hh), f2b(0.5f));
    const F2 r = f2sub(f2add(mr, hh), f2b(0.5f));
    const int lo0 = min(max(__float2int_ru(f2lo(l)), 0), 16) >> 1, lo1 = min(max(__float2int_ru(f2hi(l)), 0), 16) >> 1;
    const int hi0 = max(min(__float2int_rd(f2lo(r)), 15), -2) >> 1, hi1 = max(min(__float2int_rd(f2hi(r)), 15), -2) >> 1;
    m_lo = (0xFFu << lo0) & (0xFFu >> (7 - hi0));
    m_hi = (0xFFu << lo1) & (0xFFu >> (7 - hi1));
}

// Record-local split of a tile-local coordinate v (see the record layout below).
__device__ __forceinline__ void split_local(double v, float& o, float& r) {
    o = rintf(static_cast<float>(v));
    r = static_cast<float>(v - static_cast<double>(o));
}

// Shared-memory record of one staged splat (fp32):
//   a = {mx', my', A, beta}  b = {gamma, q_hi, q_lo, g'}  c = {-K0, -r, -g, -b}
//   d = {ox, oy, -K1, -K2}   e = {-K3, -, -, -}
// Record-local coordinates: the tile-local mean is (ox + mx', oy + my') with
// (ox, oy) = rint of it (exact small integers) and |mx'|, |my'| <= 1/2, so a
// pixel's offset x - ox is exact and no rounding error scales with the
// position inside the tile (exact_kernels.cu blend_record bounds q's error
// for exactly this arithmetic: split_local / record_q).
// K_j = o c_j folds the opacity into the polynomial (c.x = log2 o for exp; -o
// in alpha-threshold mode). The walk carries NEGATED alphas (-alpha = Horner
// over the negated coefficients, exactly), so that T' = fma(-alpha, T, T) is
// one rounding and the colour update fma(-alpha T, -c, rgb) needs no negation.
// g' = 1.001 (g + 3.2u) + 4u64 widens g = the splat's |alpha_fp32 - alpha_ref|
// bound (u = 2^-24, u64 = 2^-53) for the interval update below.
//
// Per-pair state of the walk. Invariant: for each live pixel, the reference's
// fp64 transmittance lies in [Lo, Up]. A blend of a fragment with fp32 alpha a
// (so alpha_ref in [a - g, a + g]) maps it to
//     Up' = fma(Up, (-a) + g', Up),   Lo' = fma(Lo, (-a) - g', Lo)
// The sum (-a) +- g' is rounded once (absolute error <= u, as |a| + g' < 1) and
// the fma once (relative u of a result >= Up (1 - a)); g' - g covers both, and
// the reference's two fp64 roundings, so the reference's test_t < floor is
// certainly false when Lo' >= floor and certainly true when Up' < floor; only
// the band between is undecided (exact replay). T itself is the fp32 value
// blended with (T' = fma(-a, T, T)).
struct Pair {
    F2 x;                   // tile-local pixel-centre x of both pixels (NaN once finished)
    F2 T, Up, Lo, r, g, b;
    uint32_t term0, term1;  // list position of the terminating fragment (COUNT)
    uint32_t nbl0, nbl1;    // fragments blended (COUNT)
    uint32_t flag;          // bit p: pixel p needs the exact replay
};

// One record's fragments for both pixels of a pair: everything that does not
// depend on the pixels' running state (alpha, the skip / ambiguity decisions).
struct Frag {
    float n0, n1;          // -alpha (0 when skipped)
    float g0, g1;          // g' (0 when skipped)
    float cr, cg, cb;      // -colour
    bool skip0, skip1;     // certainly alpha < eps in the reference (or pixel finished)
    bool amb0, amb1;       // accepted, but the alpha < eps decision is not certified in fp32
};

// Fragments of the record staged at shared address rec for the pair's pixels
// (x = their tile-local centres) at row centre yc. CLAMP: apply min(.999, .)
// (quadric mode skips it for batches whose records cannot reach .999).
template <int KIND, int ORDER, int MODE, bool CLAMP>
__device__ __forceinline__ Frag pair_frag(F2 x, uint32_t rec, float yc, const FrameParams& P) {
    const float4 a = lds128(rec);
    const float4 b = lds128(rec + kOffB);
    const float4 c = lds128(rec + kOffC);
    const float4 d = lds128(rec + kOffD);
    // q = A u^2 + gamma dy^2 in record-local coordinates: dy = (yc - oy) - my',
    // u = (x - ox) + (beta dy - mx') (yc - oy and x - ox are exact)
    const float dy = (yc - d.y) - a.y;
    const float tt = fmaf(a.w, dy, -a.x);
    const float cr = b.x * dy * dy;
    const F2 u = f2add(f2sub(x, f2b(d.x)), f2b(tt));
    const F2 q = f2fma(f2mul(u, f2b(a.z)), u, f2b(cr));
    const float q0 = f2lo(q), q1 = f2hi(q);
    Frag f;
    if (MODE == kQuadricThreshold) {
        // the coverage masks are a superset: q > q_hi is a certain skip; q in
        // the certified band [q_lo, q_hi] leaves the reference's alpha < eps
        // undecided in fp32 -> exact replay of the pixel. Accepted fragments
        // have q < q* + Gq < first_root, where the ReLU / piecewise cut-offs
        // are inactive: alpha = min(.999, sum K_j q^j)
        f.skip0 = !(q0 <= b.y);
        f.skip1 = !(q1 <= b.y);
        f.amb0 = q0 >= b.z;
        f.amb1 = q1 >= b.z;
        F2 na;
        if (KIND == 0) {
            const F2 ar = f2fma(q, f2b(-0.72134752044448170f), f2b(c.x));
            na = f2(-ex2_approx(f2lo(ar)), -ex2_approx(f2hi(ar)));
        } else if (ORDER == 1) {
            na = f2fma(q, f2b(d.z), f2b(c.x));
        } else {
            F2 pq = f2b(ORDER == 2 ? d.w : lds32(rec + kOffE));
            if (ORDER >= 3) pq = f2fma(pq, q, f2b(d.w));
            pq = f2fma(pq, q, f2b(d.z));
            na = f2fma(pq, q, f2b(c.x));
        }
        f.n0 = CLAMP ? fmaxf(-0.999f, f2lo(na)) : f2lo(na);
        f.n1 = CLAMP ? fmaxf(-0.999f, f2hi(na)) : f2hi(na);
    } else {
        // non-monotone kernel: full ReLU / piecewise semantics, guard on alpha
        const KernelF32& kf = P.kf;
        float a0, a1;
        if (KIND == 0) {
            a0 = ex2_approx(fmaf(q0, -0.72134752044448170f, c.x));
            a1 = ex2_approx(fmaf(q1, -0.72134752044448170f, c.x));
        } else {
            F2 pq = f2b(kf.c[kf.order]);
            for (int j = kf.order - 1; j >= 0; --j) pq = f2fma(pq, q, f2b(kf.c[j]));
            a0 = f2lo(pq), a1 = f2hi(pq);
            if (kf.kind == PS_KERNEL_POLY_PIECEWISE) {
                if (!(q0 < kf.first_root)) a0 = 0.0f;
                if (!(q1 < kf.first_root)) a1 = 0.0f;
            }
            a0 = fmaxf(-c.x * a0, 0.0f);
            a1 = fmaxf(-c.x * a1, 0.0f);
        }
        const float ga = b.y; // |alpha_fp32 - alpha_ref| bound in this mode
        a0 = fminf(0.999f, a0);
        a1 = fminf(0.999f, a1);
        f.skip0 = !(a0 >= P.eps_f - ga);
        f.skip1 = !(a1 >= P.eps_f - ga);
        f.amb0 = a0 < P.eps_f + ga;
        f.amb1 = a1 < P.eps_f + ga;
        f.n0 = -a0;
        f.n1 = -a1;
    }
    f.g0 = f.g1 = b.w;
    if (f.skip0) { f.n0 = 0.0f; f.g0 = 0.0f; f.amb0 = false; }
    if (f.skip1) { f.n1 = 0.0f; f.g1 = 0.0f; f.amb1 = false; }
    f.cr = c.y; f.cg = c.z; f.cb = c.w;
    return f;
}

// Blends fragment f (list position jpos) into the pair. When a pixel finishes
// here, `next` (a following record's fragments, if already computed) is
// cancelled for it; m (the pair's remaining candidates) is cleared when both
// pixels are finished.
template <bool COUNT>
__device__ __forceinline__ void pair_blend(Pair& p, Frag f, int jpos, const FrameParams& P, uint32_t& m,
                                           Frag* next) {
    F2 na = f2(f.n0, f.n1);
    const F2 gp = f2(f.g0, f.g1);
    const F2 up = f2fma(p.Up, f2add(na, gp), p.Up);
    F2 lo = f2fma(p.Lo, f2sub(na, gp), p.Lo);
    // Transmittance decision (raster.cpp:272-277): the reference terminates iff
    // its test_t < floor; Lo' >= floor certifies it does not (the common case,
    // no branch); otherwise decide per pixel below.
    const float fl = P.floor_f;
    if (__builtin_expect((f.amb0 | f.amb1) | (fminf(f2lo(lo), f2hi(lo)) < fl), 0)) {
        float x0 = f2lo(p.x), x1 = f2hi(p.x);
        bool done0 = false, done1 = false;
        if (!f.skip0 && (f.amb0 || f2lo(lo) < fl)) {
            done0 = true;
            if (!f.amb0 && f2lo(up) < fl) { if (COUNT) p.term0 = static_cast<uint32_t>(jpos); }
            else p.flag |= 1u;
        }
        if (!f.skip1 && (f.amb1 || f2hi(lo) < fl)) {
            done1 = true;
            if (!f.amb1 && f2hi(up) < fl) { if (COUNT) p.term1 = static_cast<uint32_t>(jpos); }
            else p.flag |= 2u;
        }
        // a finished pixel does not blend this fragment (nor the next one) and
        // keeps its T (alpha = 0 below); a huge Lo keeps it out of this branch
        float l0 = f2lo(lo), l1 = f2hi(lo);
        if (done0) {
            f.n0 = 0.0f; x0 = kNaNf; f.skip0 = true; l0 = 3.0e38f;
            if (next) { next->n0 = 0.0f; next->g0 = 0.0f; next->skip0 = true; next->amb0 = false; }
        }
        if (done1) {
            f.n1 = 0.0f; x1 = kNaNf; f.skip1 = true; l1 = 3.0e38f;
            if (next) { next->n1 = 0.0f; next->g1 = 0.0f; next->skip1 = true; next->amb1 = false; }
        }
        p.x = f2(x0, x1);
        na = f2(f.n0, f.n1);
        lo = f2(l0, l1);
        if (x0 != x0 && x1 != x1) m = 0u; // both pixels finished
    }
    const F2 w = f2mul(na, p.T);  // -alpha T
    p.T = f2fma(na, p.T, p.T);    // T (1 - alpha), one rounding; == T when skipped or finished
    p.r = f2fma(w, f2b(f.cr), p.r);
    p.g = f2fma(w, f2b(f.cg), p.g);
    p.b = f2fma(w, f2b(f.cb), p.b);
    p.Up = up;
    p.Lo = lo;
    if (COUNT) {
        p.nbl0 += f.skip0 ? 0u : 1u;
        p.nbl1 += f.skip1 ? 0u : 1u;
    }
}

// One warp's walk over a group's candidate mask m (records at shared address
// rb, list positions jb + bit). Unrolled by two so the loop-carried pair state
// alternates between two register sets instead of being copied every step.
template <int KIND, int ORDER, int MODE, bool COUNT, bool CLAMP>
__device__ __forceinline__ void walk(Pair& p, uint32_t m, uint32_t rb, float yc, const FrameParams& P, int jb) {
    while (m != 0u) {
        uint32_t j = static_cast<uint32_t>(__ffs(m) - 1);
        m &= m - 1u;
        pair_blend<COUNT>(p, pair_frag<KIND, ORDER, MODE, CLAMP>(p.x, rb + j * 16u, yc, P), jb + static_cast<int>(j),
                          P, m, nullptr);
        if (m == 0u) break;
        j = static_cast<uint32_t>(__ffs(m) - 1);
        m &= m - 1u;
        pair_blend<COUNT>(p, pair_frag<KIND, ORDER, MODE, CLAMP>(p.x, rb + j * 16u, yc, P), jb + static_cast<int>(j),
                          P, m, nullptr);
    }
}

// Exact replay of one flagged pixel by a whole warp (the reference's per-pixel
// loop, raster.cpp:250-283, in fp64 with its operation order): alpha of 32 list
// entries in parallel, then the transmittance chain serially over the accepted
// ones. In quadric mode an entry with fp32 q > q_hi is certainly skipped by the
// reference (the same certified test the fast path uses), so only candidates
// reach the fp64 kernel evaluation. Each lane's records arrive in one memory
// round trip, and the next 32 entries' are in flight during the chain.
struct ReplayRec {
    double2 m, ab, cq;
    double o;
    float4 b0, b1;
    float2 b2;
};

__device__ __forceinline__ void replay_fetch(const BlendArgs& A, const uint32_t* list, int j, int L, ReplayRec& R) {
    if (j < L) {
        const uint32_t i = list[j];
        R.m = A.mean2d[i]; R.ab = A.conic_ab[i]; R.cq = A.conic_cq[i]; R.o = A.opacity_eff[i];
        R.b0 = A.bl0[i]; R.b1 = A.bl1[i]; R.b2 = A.bl2[i];
    }
}

template <int MODE, bool COUNT>
__device__ __forceinline__ void replay_pixel(const BlendArgs& A, const uint32_t* list, int L, int lxy, int px0,
                                          int py0, unsigned long long& ev, unsigned long long& bl) {
    const int lane = threadIdx.x & 31;
    const int lx = lxy & 15, ly = lxy >> 4;
    const int gx = px0 + lx, gy = py0 + ly;
    const float xc = lx + 0.5f, yc = ly + 0.5f;
    const double eps = A.P.cfg.epsilon, floor_t = A.P.cfg.transmittance_floor;
    double trans = 1.0, r = 0.0, g = 0.0, b = 0.0;
    unsigned long long evals = 0, blended = 0;
    ReplayRec R;
    R.b0 = make_float4(0.f, 0.f, 0.f, -1.f);
    replay_fetch(A, list, lane, L, R);
    for (int base = 0; base < L; base += 32) {
        const int j = base + lane;
        double alpha = 0.0;
        bool acc = false;
        if (j < L) {
            bool cand = true;
            if (MODE == kQuadricThreshold) {
                // the walk's arithmetic (pair_frag), so the same certified bound applies
                float ox, oy, mxr, myr;
                split_local(R.m.x - px0, ox, mxr);
                split_local(R.m.y - py0, oy, myr);
                const float dy = (yc - oy) - myr;
                const float tt = fmaf(R.b0.y, dy, -mxr);
                const float u = (xc - ox) + tt;
                const float q = fmaf(R.b0.x * u, u, R.b0.z * dy * dy);
                cand = q <= R.b0.w;
            }
            if (cand) {
                const double dx = dsub(dadd(static_cast<double>(gx), 0.5), R.m.x);
                const double dy = dsub(dadd(static_cast<double>(gy), 0.5), R.m.y);
                const double q = dadd(dadd(dmul(dmul(R.ab.x, dx), dx), dmul(dmul(dmul(2.0, R.ab.y), dx), dy)),
                                      dmul(dmul(R.cq.x, dy), dy));
                const double v = dmul(R.o, eval_kernel_rn(A.P.cfg.kernel, q));
                alpha = (v < 0.999) ? v : 0.999;
                acc = !(alpha < eps);
            }
        }
        const float cr = R.b1.w, cg = R.b2.x, cb = R.b2.y;
        replay_fetch(A, list, base + 32 + lane, L, R); // next 32 entries, in flight during the chain
        uint32_t mask = __ballot_sync(0xffffffffu, acc);
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
            break;
        }
        evals += static_cast<unsigned long long>(min(32, L - base));
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

// CAPR: rounds of the prologue sort (12: buckets <= 1536 in 18 KB of shared
// memory; 16: <= 2048 in 24 KB). 8 CTAs (32 warps) per SM at 64 registers:
// measured faster than 9 at 56 (-5 us at C2) and 7 at 72 (+10 us)
// The last CTA to finish copies the frame's counters to the host (mapped pinned
// memory) and zeroes them for the next frame (which then needs no memset):
// every CTA's counter atomics are fenced before it counts itself done.
__device__ __forceinline__ void publish_counters(const BlendArgs& A) {
    static_assert(sizeof(DevCounters) % 4 == 0 && sizeof(DevCounters) / 4 <= 32, "one word per lane of warp 0");
    if (!A.publish) return;
    __syncthreads(); // the CTA's counter atomics precede thread 0's release below (barrier + fence cumulativity)
    if (threadIdx.x >= 32) return;
    bool last = false;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&A.ctr->done_ctas, 1u) == gridDim.x - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last && threadIdx.x < sizeof(DevCounters) / 4) {
        __threadfence();
        volatile uint32_t* src = reinterpret_cast<volatile uint32_t*>(A.ctr);
        reinterpret_cast<volatile uint32_t*>(A.publish)[threadIdx.x] = src[threadIdx.x];
        src[threadIdx.x] = 0u;
        __threadfence_system();
    }
}

template <int KIND, int ORDER, int MODE, bool COUNT, int CAPR>
__global__ void __launch_bounds__(128, 8) k_blend16(const BlendArgs A) {
    using SortSm = TileSortSmem<128, CAPR>;
    pdl_wait(); // K3 / the long-bucket sorts
    // Shared memory: the bucket sort's workspace; the sorted list starts at word
    // SortSm::LIST, the staging records (a, b, c, d planes + coverage words)
    // overlay the sort's dead arrays below it.
    __shared__ __align__(16) uint32_t S[SortSm::WORDS];
    __shared__ uint32_t s_nflag;
    __shared__ uint16_t s_flag[256];
    static_assert(5 * kRecs * 16 + 4 * kB16 * 4 <= SortSm::LIST * 4, "staging overlaps the sorted list");
    float4* sA = reinterpret_cast<float4*>(S);
    float4* sB = sA + kRecs;
    float4* sC = sA + 2 * kRecs;
    float4* sD = sA + 3 * kRecs;
    float4* sE = sA + 4 * kRecs;
    uint32_t (*cover)[kB16] = reinterpret_cast<uint32_t (*)[kB16]>(sA + 5 * kRecs); // [warp][record]
    const uint32_t s_rec = static_cast<uint32_t>(__cvta_generic_to_shared(sA));

    if (A.zero_counts && threadIdx.x == 0) A.zero_counts[blockIdx.x] = 0u; // K3's cursors are dead
    if (A.gate && A.gate->pairs_total > A.pair_cap) { // over capacity: the host re-runs
        publish_counters(A);
        return;
    }
    const FrameParams& P = A.P;
    const int tile = A.order ? static_cast<int>(A.order[blockIdx.x]) : static_cast<int>(blockIdx.x);
    const int tx = tile % P.tiles_x, ty = tile / P.tiles_x;
    const int W = P.cam.width, H = P.cam.height;
    const int px0 = tx * 16, py0 = ty * 16;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int lx = ((warp & 1) << 3) + ((lane & 3) << 1); // left pixel's column; right: lx + 1
    const int ly = ((warp >> 1) << 3) + (lane >> 2);      // the pair's row
    const float yc = ly + 0.5f;
    const bool row_in = py0 + ly < H;
    const bool in0 = row_in && px0 + lx < W, in1 = row_in && px0 + lx + 1 < W;
    Pair p;
    p.x = f2(in0 ? lx + 0.5f : kNaNf, in1 ? lx + 1.5f : kNaNf);
    p.T = f2b(1.0f);
    p.Up = p.Lo = f2b(1.0f);
    p.r = p.g = p.b = f2b(0.0f);
    p.term0 = p.term1 = 0xffffffffu;
    p.nbl0 = p.nbl1 = 0u;
    p.flag = 0u;
    const float c0 = P.kf.c[0], c1 = P.kf.c[1], c2 = P.kf.c[2], c3 = P.kf.c[3];
    const uint2 range = A.ranges[tile];
    const int L = static_cast<int>(range.y - range.x);
    // the tile's list in (depth, index) order: sorted here for buckets that fit
    // one CTA, presorted in global memory otherwise
    // (only its first P.sort_prefix positions, exactly: tiles terminate after
    // ~200 entries at C2; the rest is sorted when a batch or the replay needs it)
    const uint32_t* list = A.pval + range.x;
    int ranked = L;
    const bool sort_here = A.pval_w && L > 1 && L <= SortSm::CAP;
    if (sort_here) {
        list = sort_one_tile<128, CAPR, false>(range, A.pval_w, A.pkey, A.key, A.orig, S, &A.ctr->unsorted,
                                               max(P.sort_prefix, kB16), &ranked);
        __syncthreads();
    }
    auto sort_all = [&]() { // the whole bucket (the staging area is dead when this runs)
        list = sort_one_tile<128, CAPR, false>(range, A.pval_w, A.pkey, A.key, A.orig, S, &A.ctr->unsorted);
        ranked = L;
        __syncthreads();
    };
    double2 pm = make_double2(0.0, 0.0);
    float4 pb0 = make_float4(0.f, 0.f, 0.f, -1.f), pb1 = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 pb2 = make_float2(0.f, 0.f);
    auto fetch = [&](int j) {
        if (j < L) {
            const uint32_t pi = list[j];
            pm = A.mean2d[pi];
            pb0 = A.bl0[pi];
            pb1 = A.bl1[pi];
            pb2 = A.bl2[pi];
        }
    };
    fetch(t); // the ranked prefix holds at least the first batch
    bool fetched = true;
    int staged = 0; // list positions staged (the tile's walk ended before them)
    for (int base = 0; base < L; base += kB16) {
        const bool live = (f2lo(p.x) == f2lo(p.x)) || (f2hi(p.x) == f2hi(p.x));
        if (__syncthreads_count(live) == 0) break;
        staged = base + kB16;
        if (!fetched) { // this batch lies beyond the sorted prefix (rare)
            sort_all();
            fetch(base + t);
        }
        bool needs_clamp;
        {   // stage the record prefetched for this batch
            const double lxd = pm.x - px0, lyd = pm.y - py0;
            const float mx = static_cast<float>(lxd), my = static_cast<float>(lyd); // coverage only
            float ox, oy, mxr, myr;
            split_local(lxd, ox, mxr);
            split_local(lyd, oy, myr);
            const float Aq = pb0.x, beta = pb0.y, gamma = pb0.z, qhi = pb0.w;
            const float o = pb1.y, ga = pb1.z;
            float K0 = o, K1 = 0.f, K2 = 0.f, K3 = 0.f;
            if (KIND == 1 && MODE == kQuadricThreshold) {
                K0 = o * c0; K1 = o * c1; K2 = o * c2; K3 = o * c3;
            }
            const float gp = fmaf(1.001f, fmaf(3.2f, 5.9604645e-08f, ga), 4.5e-16f);
            // can this record's alpha reach the .999 clamp? (quadric mode: the
            // kernel is non-increasing in q >= 0, so alpha <= alpha(0) = K0, resp.
            // 2^K0 = o for exp; the margin covers fp32 Horner rounding)
            needs_clamp = t < L - base && (MODE != kQuadricThreshold || (KIND == 0 ? pb1.y >= -1.6e-3f : K0 >= 0.9989f));
            sA[t] = make_float4(mxr, myr, Aq, beta);
            sB[t] = make_float4(gamma, qhi, pb1.x, gp);
            sC[t] = make_float4(KIND == 0 ? pb1.y : -K0, -pb1.w, -pb2.x, -pb2.y);
            sD[t] = make_float4(ox, oy, -K1, -K2);
            if (ORDER >= 3) sE[t].x = -K3;
            // coverage of {q <= q_hi}: word w = 8 rows x 4 pairs of warp w's block
            uint32_t cw[4] = {0u, 0u, 0u, 0u};
            const bool full = MODE != kQuadricThreshold || !(qhi < 3.0e38f) || !(Aq > 0.0f) ||
                              !(gamma > 0.0f) || !(fabsf(beta) < 3.0e38f) || !(fabsf(mx) < 1.0e30f) ||
                              !(fabsf(my) < 1.0e30f);
            if (full || !(qhi >= 0.0f)) {
                const uint32_t v = full ? 0xFFFFFFFFu : 0u; // everything / never reaches epsilon
#pragma unroll
                for (int j = 0; j < 4; ++j) cw[j] = v;
            } else {
                const float qpad = qhi * 1.000004f;
                const float ia = rcp_approx(Aq) * 1.000002f;
#pragma unroll
                for (int row = 0; row < 8; ++row) { // rows row and row + 8 (words 0,1 and 2,3)
                    uint32_t m0, m1;
                    row_pairs2(row, mx, my, beta, gamma, qpad, ia, m0, m1);
                    const int sh = row << 2;
                    cw[0] |= (m0 & 0xFu) << sh;
                    cw[1] |= (m0 >> 4) << sh;
                    cw[2] |= (m1 & 0xFu) << sh;
                    cw[3] |= (m1 >> 4) << sh;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) cover[j][t] = cw[j];
        }
        const bool clamp = __syncthreads_or(needs_clamp) != 0;
        const int nb = base + kB16;
        fetched = nb + kB16 <= ranked || ranked == L;
        if (fetched) fetch(nb + t); // prefetch the next batch while this one is blended
        const int cnt = min(kB16, L - base);
        if (!__any_sync(0xffffffffu, live)) continue;
        for (int g = 0; g < kB16 / 32; ++g) {
            const int k0 = g * 32;
            if (k0 >= cnt) break;
            // candidate masks: lane s holds record k0+s's coverage of this warp's
            // block; the transpose gives lane L's pair its mask over the 32 records
            const uint32_t w = k0 + lane < cnt ? cover[warp][k0 + lane] : 0u;
            if (!__any_sync(0xffffffffu, w != 0u)) continue;
            uint32_t m = warp_transpose32(w, lane);
            const uint32_t rb = s_rec + static_cast<uint32_t>(k0) * 16u;
            const int jb = base + k0;
            if (!((f2lo(p.x) == f2lo(p.x)) || (f2hi(p.x) == f2hi(p.x)))) m = 0u; // both finished
            if (clamp) walk<KIND, ORDER, MODE, COUNT, true>(p, m, rb, yc, P, jb);
            else walk<KIND, ORDER, MODE, COUNT, false>(p, m, rb, yc, P, jb);
        }
    }

    unsigned long long ev = 0, bl = 0;
    if (t == 0) s_nflag = 0;
    __syncthreads();
    auto finish = [&](bool inside, int pxl, bool flagged, float r, float g, float b, float T, uint32_t term,
                      uint32_t nbl) {
        if (!inside) return;
        if (flagged) { // replayed below
            s_flag[atomicAdd(&s_nflag, 1u)] = static_cast<uint16_t>(ly * 16 + pxl);
            return;
        }
        const size_t pix = static_cast<size_t>(py0 + ly) * W + px0 + pxl;
        A.out_rgb[3 * pix + 0] = r;
        A.out_rgb[3 * pix + 1] = g;
        A.out_rgb[3 * pix + 2] = b;
        A.out_t[pix] = T;
        if (COUNT) {
            ev += term != 0xffffffffu ? term + 1u : static_cast<unsigned>(L);
            bl += nbl;
        }
    };
    finish(in0, lx, p.flag & 1u, f2lo(p.r), f2lo(p.g), f2lo(p.b), f2lo(p.T), p.term0, p.nbl0);
    finish(in1, lx + 1, p.flag & 2u, f2hi(p.r), f2hi(p.g), f2hi(p.b), f2hi(p.T), p.term1, p.nbl1);
    __syncthreads();
    const int nf = static_cast<int>(s_nflag);
    if (nf > 0 && ranked < L) sort_all(); // the replay walks the list to the exact termination
    if (sort_here && t == 0) { // how far down its list this tile needed the exact order
        const int need = nf > 0 ? L : min(L, staged);
        if (need > 256) atomicAdd(&A.ctr->need_over[0], 1u);
        if (need > 512) atomicAdd(&A.ctr->need_over[1], 1u);
        if (need > 1024) atomicAdd(&A.ctr->need_over[2], 1u);
    }
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
    publish_counters(A);
}

template <int KIND, int ORDER, int MODE>
void launch16(const BlendArgs& a, int n_tiles, bool count, uint32_t cap, cudaStream_t st) {
    if (cap <= kBlendSortCapSmall) {
        if (count) launch_pdl(k_blend16<KIND, ORDER, MODE, true, kBlendSortCapSmall / 128>, dim3(n_tiles), dim3(128), 0, st, a);
        else launch_pdl(k_blend16<KIND, ORDER, MODE, false, kBlendSortCapSmall / 128>, dim3(n_tiles), dim3(128), 0, st, a);
    } else {
        if (count) launch_pdl(k_blend16<KIND, ORDER, MODE, true, kBlendSortCapLarge / 128>, dim3(n_tiles), dim3(128), 0, st, a);
        else launch_pdl(k_blend16<KIND, ORDER, MODE, false, kBlendSortCapLarge / 128>, dim3(n_tiles), dim3(128), 0, st, a);
    }
}

template <int MODE>
void launch16_kind(const BlendArgs& a, int n_tiles, bool count, uint32_t cap, cudaStream_t st) {
    const KernelF32& kf = a.P.kf;
    if (kf.kind == PS_KERNEL_EXPONENTIAL) launch16<0, 1, MODE>(a, n_tiles, count, cap, st);
    else if (kf.order == 1) launch16<1, 1, MODE>(a, n_tiles, count, cap, st);
    else if (kf.order == 2) launch16<1, 2, MODE>(a, n_tiles, count, cap, st);
    else launch16<1, 3, MODE>(a, n_tiles, count, cap, st);
}

template <int KIND, int MODE>
void launch_t(const BlendArgs& a, int n_tiles, int nt, size_t smem, bool count, cudaStream_t st) {
    // tile 32: 1024 threads x 52 B of staging = 52 KB of dynamic shared memory
    if (count) {
        cudaFuncSetAttribute(k_blend<KIND, MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_blend<KIND, MODE, true><<<n_tiles, nt, smem, st>>>(a);
    } else {
        cudaFuncSetAttribute(k_blend<KIND, MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_blend<KIND, MODE, false><<<n_tiles, nt, smem, st>>>(a);
    }
}

} // namespace

int launch_blend(const FrameDev& f, const FrameParams& P, const uint32_t* pair_vals, uint32_t* sort_in_place,
                 uint32_t sort_cap, const uint32_t* orig, DevCounters* ctr, BlendOut out, bool count_work,
                 cudaStream_t st, bool* replay_fused, DevCounters* publish, uint32_t* published) {
    *replay_fused = false;
    if (published) *published = 0;
    BlendArgs a;
    a.P = P;
    a.ranges = f.ranges;
    a.order = f.tile_order;
    a.pval = pair_vals;
    a.pval_w = sort_in_place;
    a.pkey = f.pkey;
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
    a.publish = nullptr;
    a.zero_counts = nullptr;
    a.gate = f.gate;
    a.pair_cap = f.pair_cap;
    a.out_rgb = out.rgb;
    a.out_t = out.t;
    const int ts = P.cfg.tile_size;
    // one pixel per thread up to 32x32 tiles; larger tiles in 1024-pixel chunks
    const int nt = std::min(((ts * ts + 31) / 32) * 32, 1024);
    const size_t smem = static_cast<size_t>(nt) * (3 * sizeof(float4) + sizeof(uint32_t));
    const int n_tiles = P.tiles_x * P.tiles_y;
    if (n_tiles == 0) return 0;
    if (ts == 16) {
        if (publish && published) {
            a.publish = publish;
            a.zero_counts = f.tile_count;
            *published = static_cast<uint32_t>(n_tiles);
        }
        if (P.threshold_mode == kQuadricThreshold) launch16_kind<kQuadricThreshold>(a, n_tiles, count_work, sort_cap, st);
        else launch16_kind<kAlphaThreshold>(a, n_tiles, count_work, sort_cap, st);
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
