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
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
#define SH(k) v[3 * (k) + ch]
        float c = SH(0) * kSH0f;
        if (degree >= 1) c = c - SH(1) * (kSH1f * y) + SH(2) * (kSH1f * z) - SH(3) * (kSH1f * x);
        if (degree >= 2) {
            float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            c = c + SH(4) * (kSH2f[0] * xy) + SH(5) * (kSH2f[1] * yz) +
                SH(6) * (kSH2f[2] * (2.0f * zz - xx - yy)) + SH(7) * (kSH2f[3] * xz) +
                SH(8) * (kSH2f[4] * (xx - yy));
            if (degree >= 3)
                c = c + SH(9) * (kSH3f[0] * y * (3.0f * xx - yy)) + SH(10) * (kSH3f[1] * xy * z) +
                    SH(11) * (kSH3f[2] * y * (4.0f * zz - xx - yy)) +
                    SH(12) * (kSH3f[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy)) +
                    SH(13) * (kSH3f[4] * x * (4.0f * zz - xx - yy)) +
                    SH(14) * (kSH3f[5] * z * (xx - yy)) + SH(15) * (kSH3f[6] * x * (xx - yy));
        }
#undef SH
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
__device__ void blend_record(double a, double b, double c, double o, double mx, double my,
                             const FrameParams& P, float cr, float cg, float cb, float4& r0,
                             float4& r1, float2& r2) {
    (void)mx; (void)my;
    const double e32 = 5.9604644775390625e-08; // 2^-24
    const double e64 = 1.1102230246251565e-16; // 2^-53
    const ps_kernel& k = P.cfg.kernel;
    const double eps = P.cfg.epsilon;
    const double ts = P.cfg.tile_size;
    double beta = b / a;
    double gamma = c - b * b / a;
    double qs = 0.0;
    int th = blend_threshold(k, o, eps, qs);
    float qhi, qlo, eT;
    bool ok = a > 0.0 && gamma > 0.0 && isfinite(beta) && isfinite(gamma);
    double amax = k.kind == PS_KERNEL_EXPONENTIAL ? o : o * k.coeffs[0];
    amax = fmin(amax, 0.999);
    if (!ok) {
        // ill-conditioned: every candidate is decided in fp64 and any pixel that
        // blends it is replayed exactly
        qhi = INFINITY; qlo = -INFINITY; eT = INFINITY;
    } else {
        double qb = (th == 1 ? 1.25 * qs : 25.0) + 1.0;
        double U = sqrt(qb / a), D = sqrt(qb / gamma);
        double ab_ = fabs(beta);
        double X = U + ab_ * D;
        double dmx = e32 * (X + ts), dmy = e32 * (D + ts);
        double ddx = dmx + e32 * X, ddy = dmy + e32 * D;
        double gam_rel = e32 + 4.0 * e64 * (c + b * b / a) / gamma;
        // u is formed either as (dx + beta dy) or as x - (mx - beta dy); bound both
        double du = 2.0 * dmx + ddx + ab_ * ddy + 2.0 * e32 * ab_ * D + e32 * (U + X);
        double dr = qb * (2.0 * e32 + gam_rel) + 2.0 * gamma * D * ddy;
        double dau = qb * 3.0 * e32 + 2.0 * a * U * du;
        double dq = e32 * qb + dau + dr;
        double ref = 8.0 * e64 * (a * X * X + 2.0 * fabs(b) * X * D + c * D * D) +
                     4.0 * e64 * (a * X + fabs(b) * D) * (X + D);
        double Gq = 4.0 * (dq + ref) + 1e-7 * qb + 1e-12;
        // alpha error bound for the transmittance guard
        double kp = 0.5, kmag = 1.0, extra = 0.0;
        if (k.kind != PS_KERNEL_EXPONENTIAL) {
            kp = 0.0; kmag = 0.0;
            double qp = 1.0;
            for (int j = 0; j <= k.order; ++j) {
                kmag += fabs(k.coeffs[j]) * qp;
                if (j + 1 <= k.order) kp += (j + 1) * fabs(k.coeffs[j + 1]) * qp;
                qp *= qb;
            }
        } else {
            extra = amax * (4.0 * 1.1920928955078125e-07 + (0.73 * qb + 16.0) * e32);
        }
        double Ga = o * kp * Gq + 8.0 * e32 * o * kmag + extra;
        double eTd = 2.0 * (Ga / (1.0 - amax) + 4.0 * e32);
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
        eT = __double2float_ru(eTd);
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

// ------------------------------------------------------------ K1 preprocess
__global__ void __launch_bounds__(256) k_preprocess(SceneDev s, FrameParams P, FrameDev f,
                                                    DevCounters* ctr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long frustum = 0, coarse = 0, tight = 0, visible = 0;
    unsigned long long kmin_inv = 0ull, kmax = 0ull; // min tracked as max of the complement
    if (i < s.n) {
        unsigned long long key = ~0ull;
        uint32_t cnt = 0;
        const double mean[3] = {s.mean[0][i], s.mean[1][i], s.mean[2][i]};
        const double scale[3] = {s.scale[0][i], s.scale[1][i], s.scale[2][i]};
        const double quat[4] = {s.rot[0][i], s.rot[1][i], s.rot[2][i], s.rot[3][i]};
        const double opacity = s.opacity[i];
        Projected pr;
        int st = project(mean, scale, quat, opacity, P.cam, P.cfg.v_dilation, pr);
        if (st < 0) {
            raise_error(ctr, -st, i);
        } else if (st == 0) {
            frustum = 1; // kFrustum (raster.cpp:144-146,162-163)
        } else {
            double radius = 0.0, qroot = 0.0;
            int b = culling_bound_for(P.cfg, pr.opacity_eff, radius, qroot);
            if (b < 0) {
                raise_error(ctr, -b, i);
            } else if (b > 0) { // b == 0: below epsilon, dropped uncounted (raster.cpp:149-151)
                int r[4];
                const int ts = P.cfg.tile_size;
                if (!tile_rect(pr.mx, pr.my, pr.cov_aa.xx, pr.cov_aa.yy, radius, ts, P.cam.width,
                               P.cam.height, r)) {
                    frustum = 1; // off screen (raster.cpp:165-168)
                } else {
                    visible = 1;
                    coarse = static_cast<unsigned long long>(r[2] - r[0] + 1) *
                             static_cast<unsigned long long>(r[3] - r[1] + 1);
                    unsigned long long mask = 0ull;
                    int bit = 0;
                    for (int ty = r[1]; ty <= r[3]; ++ty)
                        for (int tx = r[0]; tx <= r[2]; ++tx, ++bit)
                            if (tight_tile_test(pr.conic, pr.mx, pr.my, qroot, tx, ty, ts)) {
                                ++cnt;
                                if (bit < 64) mask |= 1ull << bit;
                            }
                    f.tmask[i] = mask;
                    tight = cnt;
                    key = static_cast<unsigned long long>(__double_as_longlong(pr.depth));
                    kmin_inv = ~key;
                    kmax = key;
                    f.mean2d[i] = make_double2(pr.mx, pr.my);
                    f.conic_ab[i] = make_double2(pr.conic.xx, pr.conic.xy);
                    f.conic_cq[i] = make_double2(pr.conic.yy, qroot);
                    f.rect[i] = make_ushort4(static_cast<unsigned short>(r[0]), static_cast<unsigned short>(r[1]),
                                             static_cast<unsigned short>(r[2]), static_cast<unsigned short>(r[3]));
                    f.opacity_eff[i] = pr.opacity_eff;
                    if (f.cov_aa) {
                        f.cov_aa[3 * i] = pr.cov_aa.xx;
                        f.cov_aa[3 * i + 1] = pr.cov_aa.xy;
                        f.cov_aa[3 * i + 2] = pr.cov_aa.yy;
                    }
                    float v[48];
#pragma unroll
                    for (int j = 0; j < kShPlanes; ++j) {
                        float4 t = j < P.sh_floats4 ? s.sh4[i * kShPlanes + j]
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
                    }
                    float col[3];
                    sh_color(v, P.cfg.sh_degree, static_cast<float>(pr.dir[0]),
                             static_cast<float>(pr.dir[1]), static_cast<float>(pr.dir[2]), col);
                    if (P.cfg.clamp_before_blend) {
                        col[0] = fminf(fmaxf(col[0], 0.f), 1.f);
                        col[1] = fminf(fmaxf(col[1], 0.f), 1.f);
                        col[2] = fminf(fmaxf(col[2], 0.f), 1.f);
                    }
                    float4 r0, r1;
                    float2 r2;
                    blend_record(pr.conic.xx, pr.conic.xy, pr.conic.yy, pr.opacity_eff, pr.mx, pr.my, P,
                                 col[0], col[1], col[2], r0, r1, r2);
                    f.bl0[i] = r0;
                    f.bl1[i] = r1;
                    f.bl2[i] = r2;
                }
            }
        }
        f.key[i] = key;
        f.val[i] = static_cast<uint32_t>(i);
        f.tcount[i] = cnt;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin_inv = max(kmin_inv, __shfl_xor_sync(0xffffffffu, kmin_inv, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0 && kmax) {
        atomicMax(&ctr->key_min, kmin_inv);
        atomicMax(&ctr->key_max, kmax);
    }
    frustum = warp_sum_u64(frustum);
    coarse = warp_sum_u64(coarse);
    tight = warp_sum_u64(tight);
    visible = warp_sum_u64(visible);
    if ((threadIdx.x & 31) == 0) {
        if (frustum) atomicAdd(&ctr->frustum, frustum);
        if (coarse) atomicAdd(&ctr->coarse, coarse);
        if (tight) atomicAdd(&ctr->tight, tight);
        if (visible) atomicAdd(&ctr->visible, visible);
    }
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

// Tight tiles of splat i as tile ids, from the K1 bitmask (rect <= 64 tiles) or
// by re-running the exact tight test (larger rects). Calls fn(tile) in the
// rect's row-major order.
template <class Fn>
__device__ __forceinline__ void for_each_tight_tile(const FrameDev& f, const FrameParams& P, int64_t i, Fn&& fn) {
    const ushort4 rc = f.rect[i];
    const int w = rc.z - rc.x + 1, h = rc.w - rc.y + 1;
    if (w * h <= 64) {
        unsigned long long m = f.tmask[i];
        while (m) {
            const int b = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
            fn((rc.y + b / w) * P.tiles_x + rc.x + b % w);
        }
        return;
    }
    const double2 mm = f.mean2d[i];
    const double2 ab = f.conic_ab[i];
    const double2 cq = f.conic_cq[i];
    const Sym2 cn{ab.x, ab.y, cq.x};
    const int ts = P.cfg.tile_size;
    for (int ty = rc.y; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.z; ++tx)
            if (tight_tile_test(cn, mm.x, mm.y, cq.y, tx, ty, ts)) fn(ty * P.tiles_x + tx);
}

// K1c: pairs per tile (red.add; result unused).
__global__ void __launch_bounds__(256) k_count_tiles(FrameDev f, FrameParams P, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || f.tcount[i] == 0) return;
    for_each_tight_tile(f, P, i, [&](int t) { atomicAdd(&f.tile_count[t * kCounterStride], 1u); });
}

// K3 (bucketed): splat indices into per-tile buckets at atomically claimed
// slots. The order inside a bucket is arbitrary; K4 sorts each bucket by the
// reference's exact key.
__global__ void __launch_bounds__(256) k_duplicate_buckets(FrameDev f, FrameParams P, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || f.tcount[i] == 0) return;
    for_each_tight_tile(f, P, i, [&](int t) {
        const uint32_t slot = atomicAdd(&f.tile_count[t * kCounterStride], 1u);
        f.pval[slot] = static_cast<uint32_t>(i);
    });
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

// ------------------------------------------------------------ launchers
void launch_preprocess(const SceneDev& s, const FrameParams& P, const FrameDev& f, DevCounters* ctr,
                       cudaStream_t st) {
    if (s.n == 0) return;
    const int blocks = static_cast<int>((s.n + 255) / 256);
    k_preprocess<<<blocks, 256, 0, st>>>(s, P, f, ctr);
}

void launch_duplicate(const FrameDev& f, const FrameParams& P, const uint32_t* order, int64_t n,
                      cudaStream_t st) {
    if (n == 0) return;
    const int blocks = static_cast<int>((n + 255) / 256);
    k_duplicate<<<blocks, 256, 0, st>>>(f, P, order, n);
}

void launch_count_tiles(const FrameDev& f, const FrameParams& P, int64_t n, cudaStream_t st) {
    if (n == 0) return;
    const int blocks = static_cast<int>((n + 255) / 256);
    k_count_tiles<<<blocks, 256, 0, st>>>(f, P, n);
}

void launch_duplicate_buckets(const FrameDev& f, const FrameParams& P, int64_t n, cudaStream_t st) {
    if (n == 0) return;
    const int blocks = static_cast<int>((n + 255) / 256);
    k_duplicate_buckets<<<blocks, 256, 0, st>>>(f, P, n);
}

void launch_replay(const FrameDev& f, const FrameParams& P, DevCounters* ctr, float* out_rgb,
                   float* out_t, bool count_work, int sm_count, cudaStream_t st) {
    k_replay<<<sm_count * 4, 256, 0, st>>>(f, P, ctr, out_rgb, out_t, count_work ? 1 : 0);
}

} // namespace ps
