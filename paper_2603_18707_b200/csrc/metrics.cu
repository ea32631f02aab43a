// metrics.cu — image quality metrics on the device (metrics.cpp:13-134):
// composite against a background, PSNR (peak 1, MSE over all channels),
// max |a - b|, and SSIM (11x11 Gaussian window, sigma 1.5, valid mode,
// C1 = 0.01^2, C2 = 0.03^2, mean over pixels, then over channels).
//
// Every per-pixel quantity is computed in fp64 with the reference's operation
// order (composited values, the separable blur's tap order, the SSIM ratio), so
// per-pixel terms equal the reference's bits; only the final sums over pixels
// are reduced in a different order (relative differences ~1e-15). That order is
// fixed (per-warp partials in fixed slots, then one CTA's fixed tree), so the
// results are bit-reproducible from run to run.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "kernels.h"

namespace ps {

namespace {

constexpr int kWin = 11;          // metrics.cpp:60
constexpr int kTx = 32, kTy = 16; // SSIM output tile per CTA
constexpr int kInX = kTx + kWin - 1, kInY = kTy + kWin - 1;

__constant__ double c_taps[kWin];
__constant__ double c_bg[3];

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// composite (metrics.cpp:13-24): rgb + T * bg[ch]
template <typename T>
__device__ __forceinline__ double comp(const T* rgb, const T* tr, int64_t pix, int ch) {
    return dadd(static_cast<double>(rgb[3 * pix + ch]), dmul(static_cast<double>(tr[pix]), c_bg[ch]));
}

struct Acc {
    double sse;                 // sum of squared differences over all channel values
    unsigned long long maxabs;  // bits of max |a - b| (non-negative doubles order as integers)
    double ssim[3];             // per-channel sums of the SSIM map
};

constexpr int kMseBlocks = 148 * 8;   // k_mse_maxabs grid (at most)
constexpr int kSsimBlocks = 148 * 4;  // k_ssim grid (grid-stride over tiles x channels)
constexpr int kSsimWarps = kTx * kTy / 2 / 32;
// scratch: Acc | sse partials [kMseBlocks * 8] | ssim partials [3][kSsimBlocks * kSsimWarps]
constexpr size_t kPartOff = (sizeof(Acc) + 255) & ~size_t(255);
constexpr int kMseParts = kMseBlocks * 8, kSsimParts = kSsimBlocks * kSsimWarps;

template <typename T>
__global__ void __launch_bounds__(256) k_mse_maxabs(const T* __restrict__ ra, const T* __restrict__ ta,
                                                    const T* __restrict__ rb, const T* __restrict__ tb,
                                                    int64_t n_vals, Acc* acc, double* part) {
    double s = 0.0, m = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_vals;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t pix = i / 3;
        const int ch = static_cast<int>(i - 3 * pix);
        const double d = dsub(comp(ra, ta, pix, ch), comp(rb, tb, pix, ch));
        s = dadd(s, dmul(d, d));
        m = fmax(m, fabs(d));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if ((threadIdx.x & 31) == 0) {
        part[blockIdx.x * 8 + (threadIdx.x >> 5)] = s;
        atomicMax(&acc->maxabs, static_cast<unsigned long long>(__double_as_longlong(m)));
    }
}

// One CTA: a kTx x kTy tile of the valid-mode SSIM map of channel blockIdx.z.
// The composited inputs (with the 10-pixel halo) and the five horizontally
// blurred planes (a, b, aa, bb, ab; metrics.cpp:103-113) live in shared memory.
template <typename T>
__global__ void __launch_bounds__(kTx * kTy / 2) k_ssim(const T* __restrict__ ra, const T* __restrict__ ta,
                                                        const T* __restrict__ rb, const T* __restrict__ tb,
                                                        int W, int H, double* part) {
    extern __shared__ double sm[];
    double* ia = sm;                          // [kInY][kInX]
    double* ib = ia + kInY * kInX;
    double* hz = ib + kInY * kInX;            // [5][kInY][kTx]
    const int ow = W - kWin + 1, oh = H - kWin + 1;
    const int gx = (ow + kTx - 1) / kTx, gy = (oh + kTy - 1) / kTy;
    const int nt = blockDim.x, t = threadIdx.x;
    double acc3[3] = {0.0, 0.0, 0.0};
    for (int item = blockIdx.x; item < 3 * gx * gy; item += gridDim.x) {
        const int ch = item % 3, tile = item / 3;
        const int x0 = (tile % gx) * kTx, y0 = (tile / gx) * kTy;
        for (int k = t; k < kInY * kInX; k += nt) {
            const int yy = y0 + k / kInX, xx = x0 + k % kInX;
            double va = 0.0, vb = 0.0;
            if (yy < H && xx < W) {
                const int64_t pix = static_cast<int64_t>(yy) * W + xx;
                va = comp(ra, ta, pix, ch);
                vb = comp(rb, tb, pix, ch);
            }
            ia[k] = va;
            ib[k] = vb;
        }
        __syncthreads();
        // horizontal pass (blur(), first loop): s += taps[k] * src[y*w + x + k]
        for (int k = t; k < kInY * kTx; k += nt) {
            const int r = k / kTx, c = k % kTx;
            double sa = 0.0, sb = 0.0, saa = 0.0, sbb = 0.0, sab = 0.0;
#pragma unroll
            for (int j = 0; j < kWin; ++j) {
                const double va = ia[r * kInX + c + j], vb = ib[r * kInX + c + j];
                const double w = c_taps[j];
                sa = dadd(sa, dmul(w, va));
                sb = dadd(sb, dmul(w, vb));
                saa = dadd(saa, dmul(w, dmul(va, va)));
                sbb = dadd(sbb, dmul(w, dmul(vb, vb)));
                sab = dadd(sab, dmul(w, dmul(va, vb)));
            }
            hz[0 * kInY * kTx + k] = sa;
            hz[1 * kInY * kTx + k] = sb;
            hz[2 * kInY * kTx + k] = saa;
            hz[3 * kInY * kTx + k] = sbb;
            hz[4 * kInY * kTx + k] = sab;
        }
        __syncthreads();
        // vertical pass + SSIM ratio (metrics.cpp:115-126)
        const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
        double sum = 0.0;
        for (int k = t; k < kTy * kTx; k += nt) {
            const int r = k / kTx, c = k % kTx;
            const int oy = y0 + r, ox = x0 + c;
            if (oy >= oh || ox >= ow) continue;
            double v[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < kWin; ++j) s = dadd(s, dmul(c_taps[j], hz[q * kInY * kTx + (r + j) * kTx + c]));
                v[q] = s;
            }
            const double ma = v[0], mb = v[1];
            const double va = dsub(v[2], dmul(ma, ma));
            const double vb = dsub(v[3], dmul(mb, mb));
            const double cov = dsub(v[4], dmul(ma, mb));
            const double num = dmul(dadd(dmul(dmul(2.0, ma), mb), c1), dadd(dmul(2.0, cov), c2));
            const double den = dmul(dadd(dadd(dmul(ma, ma), dmul(mb, mb)), c1), dadd(dadd(va, vb), c2));
            sum = dadd(sum, __ddiv_rn(num, den));
        }
        acc3[ch] += sum;
        __syncthreads(); // the planes are reused by the next item
    }
    for (int c = 0; c < 3; ++c) {
        double v = acc3[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((t & 31) == 0) part[c * kSsimParts + blockIdx.x * kSsimWarps + (t >> 5)] = v;
    }
}

// One CTA: the partial sums in a fixed order (strided per thread, then a
// fixed shared-memory tree) into acc.
__global__ void __launch_bounds__(1024) k_metrics_final(const double* __restrict__ part, int n_mse, int n_ssim,
                                                        Acc* acc) {
    __shared__ double red[1024];
    const int t = threadIdx.x;
    for (int q = 0; q < 4; ++q) {
        const double* p = q == 0 ? part : part + kMseParts + (q - 1) * kSsimParts;
        const int n = q == 0 ? n_mse : n_ssim;
        double v = 0.0;
        for (int i = t; i < n; i += 1024) v += p[i];
        red[t] = v;
        __syncthreads();
        for (int h = 512; h > 0; h >>= 1) {
            if (t < h) red[t] += red[t + h];
            __syncthreads();
        }
        if (t == 0) {
            if (q == 0) acc->sse = red[0];
            else acc->ssim[q - 1] = red[0];
        }
        __syncthreads();
    }
}

template <typename T>
int run_metrics(const T* ra, const T* ta, const T* rb, const T* tb, int W, int H, const double bg[3],
                const double taps[kWin], void* scratch, ps_image_metrics* out, cudaStream_t st) {
    Acc* acc = static_cast<Acc*>(scratch);
    double* part = reinterpret_cast<double*>(static_cast<char*>(scratch) + kPartOff);
    cudaMemcpyToSymbolAsync(c_taps, taps, sizeof(double) * kWin, 0, cudaMemcpyHostToDevice, st);
    cudaMemcpyToSymbolAsync(c_bg, bg, sizeof(double) * 3, 0, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(scratch, 0, kPartOff + sizeof(double) * (kMseParts + 3 * kSsimParts), st);
    const int64_t n_vals = 3ll * W * H;
    int blocks = static_cast<int>(std::min<int64_t>((n_vals + 255) / 256, kMseBlocks));
    if (n_vals > 0) k_mse_maxabs<T><<<blocks, 256, 0, st>>>(ra, ta, rb, tb, n_vals, acc, part);
    const int ow = W - kWin + 1, oh = H - kWin + 1;
    const bool do_ssim = W >= kWin && H >= kWin;
    if (do_ssim) {
        const size_t smem = sizeof(double) * (2 * kInY * kInX + 5 * kInY * kTx);
        cudaFuncSetAttribute(k_ssim<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        const int items = 3 * ((ow + kTx - 1) / kTx) * ((oh + kTy - 1) / kTy);
        k_ssim<T><<<std::min(items, kSsimBlocks), kTx * kTy / 2, smem, st>>>(ra, ta, rb, tb, W, H, part + kMseParts);
    }
    k_metrics_final<<<1, 1024, 0, st>>>(part, kMseParts, kSsimParts, acc);
    Acc h{};
    cudaMemcpyAsync(&h, acc, sizeof(Acc), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return -1;
    // psnr (metrics.cpp:34-44)
    const double mse = n_vals ? h.sse / static_cast<double>(n_vals) : 0.0;
    out->psnr_db = mse == 0.0 ? INFINITY : 10.0 * std::log10(1.0 / mse);
    std::memcpy(&out->max_abs_diff, &h.maxabs, sizeof(double));
    out->ssim_valid = do_ssim ? 1 : 0;
    out->reserved = 0;
    if (do_ssim) {
        double total = 0.0;
        const double cnt = static_cast<double>(ow) * oh;
        for (int c = 0; c < 3; ++c) total += h.ssim[c] / cnt;
        out->ssim = total / 3.0;
    } else {
        out->ssim = 0.0;
    }
    return 0;
}

} // namespace

size_t metrics_scratch_bytes() { return kPartOff + sizeof(double) * (kMseParts + 3 * kSsimParts); }

int launch_image_metrics(const void* ra, const void* ta, const void* rb, const void* tb, bool f64, int W, int H,
                         const double bg[3], void* scratch, ps_image_metrics* out, cudaStream_t st) {
    // taps exactly as gaussian_taps() (metrics.cpp:62-72), on the host (same libm)
    double taps[kWin];
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        const double d = i - (kWin - 1) / 2.0;
        taps[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += taps[i];
    }
    for (double& v : taps) v /= sum;
    if (f64)
        return run_metrics(static_cast<const double*>(ra), static_cast<const double*>(ta),
                           static_cast<const double*>(rb), static_cast<const double*>(tb), W, H, bg, taps, scratch,
                           out, st);
    return run_metrics(static_cast<const float*>(ra), static_cast<const float*>(ta), static_cast<const float*>(rb),
                       static_cast<const float*>(tb), W, H, bg, taps, scratch, out, st);
}

} // namespace ps
