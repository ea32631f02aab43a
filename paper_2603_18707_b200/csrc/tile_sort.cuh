// tile_sort.cuh — exact per-tile ordering of a bucket in shared memory
// (shared by the standalone sort kernels in binning.cu and the blend prologue).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace ps {

// Exact per-tile order (the reference comparator, raster.cpp:172-175:
// fp64 depth, then splat index; positive fp64 depths order like their bits):
//  1. 16-bit key = top bits of (depth bits - tile minimum) over the tile's own
//     depth span; stable LSD radix sort, 2 x 8-bit digits. Stable ranking: each
//     warp owns a contiguous slice of the current order and ranks it 32 items
//     at a time with match.any.
//  2. every run of equal 16-bit keys is re-ordered by the full (bits, index)
//     key; runs are expected to be ~L^2/2^17 pairs, so a thread insertion-sorts
//     each. A run longer than kMaxRun (degenerate depth clusters) switches the
//     CTA to a bitonic sort on the full key, which is exact for any input.
constexpr int kMaxRun = 64;

template <int THREADS, int ROUNDS>
struct TileSortSmem {
    static constexpr int CAP = THREADS * ROUNDS;
    static constexpr int WARPS = THREADS / 32;
    // vals [2][CAP] u32 | keys16 [2][CAP] u16 | pos [CAP] u16 | per-warp digit counts [WARPS][256] u32
    static constexpr size_t WORDS = 2 * CAP + CAP + CAP / 2 + WARPS * 256;
    __host__ __device__ static constexpr size_t bytes() { return sizeof(uint32_t) * WORDS; }
};

// Returns the sorted bucket in shared memory (smem[0, L)); with WRITEBACK also
// writes it back to pval[r.x, r.y). Per-item ranks live in shared memory (not registers), so
// ROUNDS (= CAP / THREADS) can be large without register pressure.
template <int THREADS, int ROUNDS, bool WRITEBACK = true>
__device__ __forceinline__ uint32_t* sort_one_tile(const uint2 r, uint32_t* __restrict__ pval,
                                                   const unsigned long long* __restrict__ key,
                                                   const uint32_t* __restrict__ orig, uint32_t* smem) {
    constexpr int WARPS = THREADS / 32;
    constexpr int CAP = THREADS * ROUNDS;
    uint32_t* vbuf = smem;                                                  // [2][CAP]
    uint16_t* kbuf = reinterpret_cast<uint16_t*>(smem + 2 * CAP);           // [2][CAP]
    uint16_t* pos = reinterpret_cast<uint16_t*>(smem + 3 * CAP);            // [CAP]
    uint32_t* whist = smem + 3 * CAP + CAP / 2;                             // [WARPS][256]
    __shared__ uint32_t dtot[256];
    __shared__ uint32_t wsum[WARPS];
    __shared__ unsigned long long red_min[WARPS], red_max[WARPS];
    __shared__ int need_bitonic;

    const int L = static_cast<int>(r.y - r.x);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int j = threadIdx.x; j < L; j += THREADS) {
        const uint32_t v = pval[r.x + j];
        const unsigned long long k = key[v];
        vbuf[j] = v;
        lo = min(lo, k);
        hi = max(hi, k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { red_min[warp] = lo; red_max[warp] = hi; }
    if (threadIdx.x == 0) need_bitonic = 0;
    __syncthreads();
    lo = red_min[0]; hi = red_max[0];
    for (int w = 1; w < WARPS; ++w) { lo = min(lo, red_min[w]); hi = max(hi, red_max[w]); }
    const unsigned long long span = hi - lo;
    const int shift = span ? max(0, 64 - __clzll(static_cast<long long>(span)) - 16) : 0;
    for (int j = threadIdx.x; j < L; j += THREADS) kbuf[j] = static_cast<uint16_t>((key[vbuf[j]] - lo) >> shift);
    const int per_warp = ((L + WARPS * 32 - 1) / (WARPS * 32)) * 32;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    int cur = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int sh = pass * 8;
        for (int d = threadIdx.x; d < WARPS * 256; d += THREADS) whist[d] = 0;
        __syncthreads();
        const uint16_t* kin = kbuf + cur * CAP;
        const uint32_t* vin = vbuf + cur * CAP;
        uint16_t* kout = kbuf + (cur ^ 1) * CAP;
        uint32_t* vout = vbuf + (cur ^ 1) * CAP;
        for (int it = 0; it < ROUNDS && it * 32 < per_warp; ++it) {
            const int j = warp * per_warp + it * 32 + lane;
            const bool valid = j < L;
            const uint32_t d = valid ? (static_cast<uint32_t>(kin[j]) >> sh) & 0xFFu : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t cb = valid ? whist[warp * 256 + d] : 0u;
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) whist[warp * 256 + d] = cb + __popc(peers);
            __syncwarp();
            if (valid) pos[j] = static_cast<uint16_t>(cb + __popc(peers & lt));
        }
        __syncthreads();
        for (int d = threadIdx.x; d < 256; d += THREADS) {
            uint32_t acc = 0;
            for (int w = 0; w < WARPS; ++w) {
                const uint32_t c = whist[w * 256 + d];
                whist[w * 256 + d] = acc;
                acc += c;
            }
            dtot[d] = acc;
        }
        __syncthreads();
        // exclusive scan of the 256 digit totals
        constexpr int PER = 256 / THREADS > 0 ? 256 / THREADS : 1;
        uint32_t loc[PER];
        uint32_t sum = 0, x = 0;
        const bool scanner = threadIdx.x * PER < 256;
        if (scanner) {
#pragma unroll
            for (int q = 0; q < PER; ++q) { loc[q] = dtot[threadIdx.x * PER + q]; sum += loc[q]; }
            x = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
        }
        __syncthreads();
        if (scanner) {
            uint32_t base = x - sum;
            for (int w = 0; w < warp; ++w) base += wsum[w];
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int d = threadIdx.x * PER + q;
                for (int w = 0; w < WARPS; ++w) whist[w * 256 + d] += base;
                base += loc[q];
            }
        }
        __syncthreads();
        for (int it = 0; it < ROUNDS && it * 32 < per_warp; ++it) {
            const int j = warp * per_warp + it * 32 + lane;
            if (j < L) {
                const uint16_t k = kin[j];
                const uint32_t dst = whist[warp * 256 + ((static_cast<uint32_t>(k) >> sh) & 0xFFu)] + pos[j];
                kout[dst] = k;
                vout[dst] = vin[j];
            }
        }
        __syncthreads();
        cur ^= 1;
    }
    const uint16_t* ks = kbuf + cur * CAP;
    uint32_t* vs = vbuf + cur * CAP;
    // ties of the 16-bit key: order each run by the full (depth bits, original index)
    for (int j = threadIdx.x; j < L; j += THREADS) {
        if ((j == 0 || ks[j - 1] != ks[j]) && j + 1 < L && ks[j + 1] == ks[j]) {
            int e = j + 1;
            while (e < L && ks[e] == ks[j] && e - j <= kMaxRun) ++e;
            if (e - j > kMaxRun) {
                need_bitonic = 1;
                continue;
            }
            for (int a = j + 1; a < e; ++a) {
                const uint32_t va = vs[a];
                const unsigned long long ka = key[va];
                int b = a - 1;
                while (b >= j) {
                    const uint32_t vb = vs[b];
                    const unsigned long long kb = key[vb];
                    if (kb < ka || (kb == ka && orig[vb] < orig[va])) break;
                    vs[b + 1] = vb;
                    --b;
                }
                vs[b + 1] = va;
            }
        }
    }
    __syncthreads();
    if (need_bitonic) {
        // degenerate depth clusters: exact bitonic sort on (bits, original index);
        // full keys in the (now free) second value buffer + key buffers
        unsigned long long* fk = reinterpret_cast<unsigned long long*>(smem + CAP);
        int n = 1;
        while (n < L) n <<= 1;
        for (int j = threadIdx.x; j < n; j += THREADS) {
            if (j < L) fk[j] = key[vs[j]];
            else { fk[j] = ~0ull; vs[j] = 0xffffffffu; }
        }
        __syncthreads();
        for (int k = 2; k <= n; k <<= 1)
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                const int lg = __ffs(jj) - 1;
                for (int p = threadIdx.x; p < (n >> 1); p += THREADS) {
                    const int i = ((p >> lg) << (lg + 1)) + (p & (jj - 1));
                    const int ix = i + jj;
                    const unsigned long long ka = fk[i], kb = fk[ix];
                    const uint32_t va = vs[i], vb = vs[ix];
                    const uint32_t oa = va == 0xffffffffu ? 0xffffffffu : orig[va];
                    const uint32_t ob = vb == 0xffffffffu ? 0xffffffffu : orig[vb];
                    const bool gt = ka > kb || (ka == kb && oa > ob);
                    if (gt == ((i & k) == 0)) { fk[i] = kb; fk[ix] = ka; vs[i] = vb; vs[ix] = va; }
                }
                __syncthreads();
            }
    }
    if (WRITEBACK)
        for (int j = threadIdx.x; j < L; j += THREADS) pval[r.x + j] = vs[j];
    return vs; // == smem (two passes end in buffer 0)
}

} // namespace ps
