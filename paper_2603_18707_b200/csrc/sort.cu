// sort.cu — hand-written device radix sort, scan and tile ranges.
//
// Radix sort: stable LSD, 8-bit digits, three kernels per pass:
//   k_hist    : per-block digit histogram (warp-aggregated via match.any),
//               stored digit-major hist[d * nblocks + b];
//   k_scan_rows: one block per digit scans its row over blocks (exclusive) and
//               records the digit total;
//   k_scatter : each block recomputes a stable rank for its items (warps own
//               consecutive sub-chunks, match.any ranks lanes within a 32-item
//               batch), adds the block's digit base, and scatters.
// The item count may live in device memory, so a pass needs no host sync.
// Stability is what makes (a) the depth sort reproduce the reference's
// (depth, index) order (raster.cpp:172-175) from index-ordered input, and
// (b) the tile sort keep each tile's list in depth order (raster.cpp:193-206).
#include <cub/warp/warp_scan.cuh>

#include "kernels.h"

namespace ps {

namespace {

constexpr int kBins = 256;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItemsPerLane = 16;
constexpr int kTile = kThreads * kItemsPerLane; // 4096 items per block

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int64_t item_count(const uint32_t* d_n, int64_t n_cap) {
    if (!d_n) return n_cap;
    int64_t n = static_cast<int64_t>(*d_n);
    return n < n_cap ? n : n_cap;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_hist(const K* __restrict__ keys, const uint32_t* d_n,
                                                   int64_t n_cap, int shift, uint32_t* __restrict__ hist,
                                                   int nblocks) {
    __shared__ uint32_t sh[kBins];
    sh[threadIdx.x] = 0;
    __syncthreads();
    const int64_t n = item_count(d_n, n_cap);
    const int64_t start = static_cast<int64_t>(blockIdx.x) * kTile;
    const int lane = threadIdx.x & 31;
    for (int64_t j0 = start; j0 < start + kTile; j0 += kThreads) {
        const int64_t j = j0 + threadIdx.x;
        const bool valid = j < n;
        const uint32_t d = valid ? static_cast<uint32_t>((keys[j] >> shift) & 0xFF) : kBins;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid && lane == __ffs(peers) - 1) atomicAdd(&sh[d], static_cast<uint32_t>(__popc(peers)));
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * nblocks + blockIdx.x] = sh[threadIdx.x];
}

// one block per digit: exclusive scan of hist[d][0..nblocks) in place; tot[d] = row sum
__global__ void __launch_bounds__(kThreads) k_scan_rows(uint32_t* __restrict__ hist, int nblocks,
                                                        uint32_t* __restrict__ tot) {
    using WarpScan = cub::WarpScan<uint32_t>;
    __shared__ typename WarpScan::TempStorage ws[kWarps];
    __shared__ uint32_t wsum[kWarps];
    uint32_t* row = hist + static_cast<int64_t>(blockIdx.x) * nblocks;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t carry = 0;
    for (int base = 0; base < nblocks; base += kThreads) {
        const int j = base + threadIdx.x;
        const uint32_t v = j < nblocks ? row[j] : 0u;
        uint32_t ex, agg;
        WarpScan(ws[warp]).ExclusiveSum(v, ex, agg);
        if (lane == 31) wsum[warp] = ex + v;
        __syncthreads();
        uint32_t woff = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            woff += (w < warp) ? wsum[w] : 0u;
            total += wsum[w];
        }
        if (j < nblocks) row[j] = carry + woff + ex;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) k_scatter(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                      K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                      const uint32_t* d_n, int64_t n_cap, int shift,
                                                      const uint32_t* __restrict__ hist,
                                                      const uint32_t* __restrict__ tot, int nblocks) {
    __shared__ uint32_t base[kBins];
    __shared__ uint32_t whist[kWarps][kBins];
    using WarpScan = cub::WarpScan<uint32_t>;
    __shared__ typename WarpScan::TempStorage ws[kWarps];
    __shared__ uint32_t wsum[kWarps];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // digit base = exclusive scan over digit totals + this block's row offset
    {
        const uint32_t v = tot[threadIdx.x];
        uint32_t ex, agg;
        WarpScan(ws[warp]).ExclusiveSum(v, ex, agg);
        if (lane == 31) wsum[warp] = ex + v;
        __syncthreads();
        uint32_t woff = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) woff += (w < warp) ? wsum[w] : 0u;
        base[threadIdx.x] = woff + ex + hist[static_cast<int64_t>(threadIdx.x) * nblocks + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) whist[w][threadIdx.x] = 0;
    }
    __syncthreads();

    const int64_t n = item_count(d_n, n_cap);
    const int64_t wstart = static_cast<int64_t>(blockIdx.x) * kTile + static_cast<int64_t>(warp) * (kTile / kWarps);
    K kk[kItemsPerLane];
    uint32_t vv[kItemsPerLane], pos[kItemsPerLane], dig[kItemsPerLane];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int it = 0; it < kItemsPerLane; ++it) {
        const int64_t j = wstart + it * 32 + lane;
        const bool valid = j < n;
        kk[it] = valid ? keys_in[j] : K(0);
        vv[it] = valid ? vals_in[j] : 0u;
        const uint32_t d = valid ? static_cast<uint32_t>((kk[it] >> shift) & 0xFF) : kBins;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t cbase = valid ? whist[warp][d] : 0u;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) whist[warp][d] = cbase + __popc(peers);
        __syncwarp();
        pos[it] = cbase + __popc(peers & lt);
        dig[it] = d;
    }
    __syncthreads();
    {
        uint32_t acc = base[threadIdx.x];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = whist[w][threadIdx.x];
            whist[w][threadIdx.x] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItemsPerLane; ++it) {
        if (dig[it] < kBins) {
            const uint32_t dst = whist[warp][dig[it]] + pos[it];
            keys_out[dst] = kk[it];
            vals_out[dst] = vv[it];
        }
    }
}

template <typename K>
bool radix_sort_impl(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, const uint32_t* d_n,
                     int64_t n_cap, int begin_bit, int end_bit, void* scratch, cudaStream_t st,
                     int* launches) {
    if (n_cap <= 0 || end_bit <= begin_bit) return false;
    const int nblocks = static_cast<int>((n_cap + kTile - 1) / kTile);
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    uint32_t* tot = hist + static_cast<int64_t>(kBins) * nblocks;
    bool alt = false;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        const K* kin = alt ? keys_alt : keys;
        const uint32_t* vin = alt ? vals_alt : vals;
        K* kout = alt ? keys : keys_alt;
        uint32_t* vout = alt ? vals : vals_alt;
        k_hist<K><<<nblocks, kThreads, 0, st>>>(kin, d_n, n_cap, shift, hist, nblocks);
        k_scan_rows<<<kBins, kThreads, 0, st>>>(hist, nblocks, tot);
        k_scatter<K><<<nblocks, kThreads, 0, st>>>(kin, vin, kout, vout, d_n, n_cap, shift, hist, tot, nblocks);
        if (launches) *launches += 3;
        alt = !alt;
    }
    return alt;
}

// ------------------------------------------------------------ scan
constexpr int kScanItems = 16;
constexpr int kScanTile = kThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* wsum, uint32_t& total) {
    using WarpScan = cub::WarpScan<uint32_t>;
    __shared__ typename WarpScan::TempStorage ws[kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ex, agg;
    WarpScan(ws[warp]).ExclusiveSum(v, ex, agg);
    if (lane == 31) wsum[warp] = ex + v;
    __syncthreads();
    uint32_t woff = 0;
    total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        woff += (w < warp) ? wsum[w] : 0u;
        total += wsum[w];
    }
    __syncthreads();
    return woff + ex;
}

__global__ void __launch_bounds__(kThreads) k_scan_reduce(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ order,
                                                          int64_t n, uint32_t* __restrict__ bsum) {
    __shared__ uint32_t wsum[kWarps];
    const int64_t start = static_cast<int64_t>(blockIdx.x) * kScanTile;
    uint32_t s = 0;
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t j = start + static_cast<int64_t>(k) * kThreads + threadIdx.x;
        if (j < n) s += cnt[order[j]];
    }
    uint32_t total;
    block_exclusive_scan(s, wsum, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kThreads) k_scan_bsums(uint32_t* __restrict__ bsum, int nb, uint32_t* d_total) {
    __shared__ uint32_t wsum[kWarps];
    uint32_t carry = 0;
    for (int base = 0; base < nb; base += kThreads) {
        const int j = base + threadIdx.x;
        const uint32_t v = j < nb ? bsum[j] : 0u;
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, wsum, total);
        if (j < nb) bsum[j] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *d_total = carry;
}

__global__ void __launch_bounds__(kThreads) k_scan_apply(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ order,
                                                         int64_t n, const uint32_t* __restrict__ bsum,
                                                         uint32_t* __restrict__ offset) {
    __shared__ uint32_t wsum[kWarps];
    // blocked arrangement: thread t owns items [start + t*16, start + t*16 + 16)
    const int64_t start = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t j = start + k;
        v[k] = j < n ? cnt[order[j]] : 0u;
        s += v[k];
    }
    uint32_t total;
    uint32_t run = bsum[blockIdx.x] + block_exclusive_scan(s, wsum, total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t j = start + k;
        if (j < n) offset[j] = run;
        run += v[k];
    }
}

__global__ void k_ranges(const uint32_t* __restrict__ keys, const uint32_t* d_n, int64_t n_cap,
                         uint2* __restrict__ ranges) {
    const int64_t n = item_count(d_n, n_cap);
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = keys[j];
        if (j == 0 || keys[j - 1] != t) ranges[t].x = static_cast<uint32_t>(j);
        if (j == n - 1 || keys[j + 1] != t) ranges[t].y = static_cast<uint32_t>(j + 1);
    }
}

} // namespace

size_t radix_scratch_bytes(int64_t n_cap) {
    const int64_t nblocks = (n_cap + kTile - 1) / kTile;
    return sizeof(uint32_t) * static_cast<size_t>(kBins * nblocks + kBins);
}

bool radix_sort_u64(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals,
                    uint32_t* vals_alt, const uint32_t* d_n, int64_t n_cap, int begin_bit, int end_bit,
                    void* scratch, cudaStream_t st, int* launches) {
    return radix_sort_impl<unsigned long long>(keys, keys_alt, vals, vals_alt, d_n, n_cap, begin_bit,
                                               end_bit, scratch, st, launches);
}

bool radix_sort_u32(uint32_t* keys, uint32_t* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                    const uint32_t* d_n, int64_t n_cap, int begin_bit, int end_bit, void* scratch,
                    cudaStream_t st, int* launches) {
    return radix_sort_impl<uint32_t>(keys, keys_alt, vals, vals_alt, d_n, n_cap, begin_bit, end_bit,
                                     scratch, st, launches);
}

size_t scan_scratch_bytes(int64_t n) {
    return sizeof(uint32_t) * static_cast<size_t>((n + kScanTile - 1) / kScanTile + 1);
}

void scan_gathered_counts(const uint32_t* tcount, const uint32_t* order, uint32_t* offset, int64_t n,
                          uint32_t* d_total, void* scratch, cudaStream_t st, int* launches) {
    uint32_t* bsum = static_cast<uint32_t*>(scratch);
    const int nb = static_cast<int>((n + kScanTile - 1) / kScanTile);
    if (nb == 0) {
        cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st);
        return;
    }
    k_scan_reduce<<<nb, kThreads, 0, st>>>(tcount, order, n, bsum);
    k_scan_bsums<<<1, kThreads, 0, st>>>(bsum, nb, d_total);
    k_scan_apply<<<nb, kThreads, 0, st>>>(tcount, order, n, bsum, offset);
    if (launches) *launches += 3;
}

void launch_ranges(const uint32_t* keys, const uint32_t* d_n, int64_t n_cap, uint2* ranges,
                   int n_tiles, cudaStream_t st, int* launches) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * static_cast<size_t>(n_tiles), st);
    if (n_cap <= 0) return;
    int blocks = static_cast<int>((n_cap + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_ranges<<<blocks, 256, 0, st>>>(keys, d_n, n_cap, ranges);
    if (launches) *launches += 1;
}

} // namespace ps
