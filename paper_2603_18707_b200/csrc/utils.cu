// utils.cu — small device helpers: on-device de-interleave of uploaded splat
// arrays (so a host upload is a handful of large DMA copies), and the FP32
// issue-rate microbenchmark the bench uses as the blend roofline denominator.
#include <algorithm>

#include "kernels.h"

namespace ps {

namespace {

// staging = [means n*3 | scales n*3 | rots n*4] (interleaved per splat)
__global__ void k_deinterleave(const double* __restrict__ st, int64_t n, SceneDev s) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double* m = st + 3 * i;
        const double* sc = st + 3 * n + 3 * i;
        const double* r = st + 6 * n + 4 * i;
        s.mean[0][i] = m[0]; s.mean[1][i] = m[1]; s.mean[2][i] = m[2];
        s.scale[0][i] = sc[0]; s.scale[1][i] = sc[1]; s.scale[2][i] = sc[2];
        s.rot[0][i] = r[0]; s.rot[1][i] = r[1]; s.rot[2][i] = r[2]; s.rot[3][i] = r[3];
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

} // namespace

void launch_deinterleave(const double* staging, int64_t n, const SceneDev& s, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_deinterleave<<<blocks, 256, 0, st>>>(staging, n, s);
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
