// utils.cu — small device helpers: on-device split of uploaded Splat3D records
// and the scene's Morton reordering (so a host upload is a handful of large DMA copies), and the FP32
// issue-rate microbenchmark the bench uses as the blend roofline denominator.
#include <algorithm>

#include "kernels.h"

namespace ps {

namespace {

// Uploaded splat records -> the upload staging layout: geometry fp64
// [means 3n | scales 3n | rots 4n | opacity n] and SH fp32 [n][48].
//   RAW:  the reference's Splat3D (59 doubles: mean 3, scale 3, rotation 4,
//         opacity, sh 48; projection.hpp:13-19), SH narrowed here;
//   else: the drop-in's compact record (the same 11 doubles, then the 48 SH
//         coefficients already rounded to fp32 on the host: 280 B).
// Each thread moves one 8-byte word of the flat record array (coalesced reads).
template <bool RAW>
__global__ void k_split_records(const double* __restrict__ rec, int64_t n, double* __restrict__ st,
                                float* __restrict__ sh) {
    constexpr int W = RAW ? PS_SPLAT3D_DOUBLES : 11 + 24; // 8-byte words per record
    const uint64_t total = static_cast<uint64_t>(n) * W;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double v = rec[e];
        const uint64_t i = e / W;
        const int f = static_cast<int>(e - i * W);
        if (f < 3) st[3 * i + f] = v;
        else if (f < 6) st[3 * n + 3 * i + (f - 3)] = v;
        else if (f < 10) st[6 * n + 4 * i + (f - 6)] = v;
        else if (f == 10) st[10 * n + i] = v;
        else if (RAW) sh[48 * i + (f - 11)] = __double2float_rn(v);
        else reinterpret_cast<double*>(sh)[24 * i + (f - 11)] = v; // two fp32 coefficients
    }
}

// 8 independent FFMA chains per thread, 4096 iterations: 2 flops per FFMA.
__global__ void __launch_bounds__(256) k_ffma_peak(float* out, float a, float b, int iters) {
    float x0 = threadIdx.x * 1e-7f, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
    float x4 = x0 + 4.f, x5 = x0 + 5.f, x6 = x0 + 6.f, x7 = x0 + 7.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (r == 12345.678f) out[threadIdx.x] = r; // keep the chains live
}

// Order-preserving map of a double to u64 (for atomic min/max).
__device__ __forceinline__ unsigned long long dkey(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// bounding box of the (interleaved) means: bb[0..2] = max of ~dkey (i.e. min), bb[3..5] = max
__global__ void k_bbox(const double* __restrict__ means, int64_t n, unsigned long long* bb) {
    unsigned long long lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            const double v = means[3 * i + k];
            if (v != v) continue;
            const unsigned long long d = dkey(v);
            lo[k] = max(lo[k], ~d);
            hi[k] = max(hi[k], d);
        }
    }
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = max(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&bb[k], lo[k]);
            atomicMax(&bb[3 + k], hi[k]);
        }
    }
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// 30-bit Morton code of each mean inside the bounding box (NaNs sort last)
__global__ void k_morton(const double* __restrict__ means, int64_t n, const unsigned long long* __restrict__ bb,
                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    double lo[3], sc[3];
    for (int k = 0; k < 3; ++k) {
        lo[k] = dkey_inv(~bb[k]);
        const double hi = dkey_inv(bb[3 + k]);
        const double ext = hi - lo[k];
        sc[k] = ext > 0.0 && ext == ext ? 1023.0 / ext : 0.0;
    }
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t q[3];
        bool bad = false;
        for (int k = 0; k < 3; ++k) {
            const double t = (means[3 * i + k] - lo[k]) * sc[k];
            bad |= !(t == t);
            q[k] = t > 0.0 ? static_cast<uint32_t>(fmin(t, 1023.0)) : 0u;
        }
        keys[i] = bad ? 0x3fffffffu : (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
        vals[i] = static_cast<uint32_t>(i);
    }
}

// internal splat j <- original splat perm[j] (de-interleaving the staged arrays)
__global__ void k_gather_scene(const double* __restrict__ st, const double* __restrict__ opac,
                               const float4* __restrict__ sh, const uint32_t* __restrict__ perm, int64_t n, SceneDev s) {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = perm[j];
        const double* m = st + 3 * i;
        const double* sc = st + 3 * n + 3 * i;
        const double* r = st + 6 * n + 4 * i;
        s.mean[0][j] = m[0]; s.mean[1][j] = m[1]; s.mean[2][j] = m[2];
        s.scale[0][j] = sc[0]; s.scale[1][j] = sc[1]; s.scale[2][j] = sc[2];
        s.rot[0][j] = r[0]; s.rot[1][j] = r[1]; s.rot[2][j] = r[2]; s.rot[3][j] = r[3];
        s.opacity[j] = opac[i];
#pragma unroll
        for (int k = 0; k < kShPlanes; ++k) s.sh4[k * n + j] = sh[i * kShPlanes + k];
        s.orig[j] = static_cast<uint32_t>(i);
    }
}

} // namespace

void launch_morton_order(const double* means, int64_t n, unsigned long long* bb, uint32_t* keys, uint32_t* vals,
                         cudaStream_t st) {
    cudaMemsetAsync(bb, 0, 6 * sizeof(unsigned long long), st);
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_bbox<<<blocks, 256, 0, st>>>(means, n, bb);
    k_morton<<<blocks, 256, 0, st>>>(means, n, bb, keys, vals);
}

void launch_gather_scene(const double* staging, const double* opac, const float4* sh, const uint32_t* perm,
                         int64_t n, const SceneDev& s, cudaStream_t st) {
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_gather_scene<<<blocks, 256, 0, st>>>(staging, opac, sh, perm, n, s);
}

void launch_split_records(const double* rec, int64_t n, bool raw, double* staging, float* sh, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t total = n * (raw ? PS_SPLAT3D_DOUBLES : 35);
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (raw) k_split_records<true><<<blocks, 256, 0, st>>>(rec, n, staging, sh);
    else k_split_records<false><<<blocks, 256, 0, st>>>(rec, n, staging, sh);
}

// Returns achieved FP32 TFLOP/s (FFMA = 2 flops) over `reps` timed launches.
double measure_fp32_tflops(int sm_count, cudaStream_t st) {
    float* out = nullptr;
    cudaMalloc(&out, 256 * sizeof(float));
    const int blocks = sm_count * 8, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_ffma_peak<<<blocks, threads, 0, st>>>(out, 0.9999f, 1e-4f, iters); // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st);
        k_ffma_peak<<<blocks, threads, 0, st>>>(out, 0.9999f, 1e-4f, iters);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
        if (ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}

} // namespace ps

namespace ps {
namespace {
// fp64 DFMA issue-rate probe (diagnostic for the fp64 preprocess roofline).
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, double a, double b, int iters) {
    double x0 = threadIdx.x * 1e-7, x1 = x0 + 1., x2 = x0 + 2., x3 = x0 + 3.;
    double x4 = x0 + 4., x5 = x0 + 5., x6 = x0 + 6., x7 = x0 + 7.;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (r == 12345.678) out[threadIdx.x] = r;
}
} // namespace

double measure_fp64_tflops(int sm_count, cudaStream_t st) {
    double* out = nullptr;
    cudaMalloc(&out, 256 * sizeof(double));
    const int blocks = sm_count * 8, threads = 256, iters = 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma_peak<<<blocks, threads, 0, st>>>(out, 0.9999, 1e-4, iters);
    double best = 0.0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, st);
        k_dfma_peak<<<blocks, threads, 0, st>>>(out, 0.9999, 1e-4, iters);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
        if (ms > 0.f) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}
} // namespace ps
