// binning.cu — per-tile buckets instead of global sorts.
//
// The reference bins prepared splats into per-tile lists in (depth, index)
// order (raster.cpp:172-175, 193-206). Rather than sorting all V splats by
// depth and then all P pairs by tile (two global radix sorts, launch- and
// latency-bound at these sizes), the render path
//   K1 counts tight pairs per tile (red.add),
//   K2 scans the counts into tile ranges and bucket cursors  (k_tile_scan),
//   K3 scatters splat indices into the buckets by atomic cursors,
//   K4 sorts each bucket in shared memory by the exact key (fp64 depth bits,
//      splat index) — a total order, so the arbitrary scatter order of K3 does
//      not matter and the result equals the reference's per-tile list.
#include "kernels.h"
#include "tile_sort.cuh"

namespace ps {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanPer = 8;                            // tiles per thread per round
constexpr int kScanRound = kScanThreads * kScanPer;    // 8192 tiles: a 1080p frame is one round
__host__ __device__ constexpr int scan_pad(int i) { return i + (i >> 5); } // conflict-free blocked reads

// One CTA: exclusive scan of the per-tile pair counts into ranges and K3
// cursors, the total / longest bucket, and the list of buckets > list_min (sorted
// outside the blend). Global memory is read and written in striped order (each
// warp instruction one or two whole 128-byte lines) and transposed through
// shared memory to the blocked order of the scan (thread t owns tiles
// 8t .. 8t + 7 of the round): one SM's load/store path carries the whole
// kernel, so uncoalesced per-thread runs of 16 tiles had made it
// transaction-bound (8 us at 1080p, 22 us at 4K).
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(uint32_t* __restrict__ count, uint2* __restrict__ ranges,
                                                            int n_tiles, DevCounters* ctr, uint32_t* __restrict__ big_list,
                                                            uint32_t list_min) {
    __shared__ uint32_t sc[scan_pad(kScanRound) + 1];
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t wmax[32];
    pdl_trigger(); // K3 may be scheduled now (it waits for this scan)
    pdl_wait();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t carry = 0, mx = 0;
    uint32_t nxt[kScanPer]; // this round's counts, loaded during the previous round
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) nxt[q] = q * kScanThreads + t < n_tiles ? count[q * kScanThreads + t] : 0u;
    for (int base = 0; base < n_tiles; base += kScanRound) {
        const int cnt = min(kScanRound, n_tiles - base);
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) sc[scan_pad(q * kScanThreads + t)] = nxt[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) { // the next round's loads overlap this round
            const int g = base + kScanRound + q * kScanThreads + t;
            nxt[q] = g < n_tiles ? count[g] : 0u;
        }
        uint32_t v[kScanPer];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
            v[q] = sc[scan_pad(t * kScanPer + q)];
            sum += v[q];
            mx = max(mx, v[q]);
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w; // inclusive over warps
        }
        __syncthreads();
        uint32_t excl = carry + (warp ? wsum[warp - 1] : 0u) + x - sum;
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
            const int i = t * kScanPer + q;
            if (v[q] > list_min && i < cnt) big_list[atomicAdd(&ctr->big_tiles, 1u)] = static_cast<uint32_t>(base + i);
            sc[scan_pad(i)] = excl;
            excl += v[q];
        }
        const uint32_t next = carry + wsum[31];
        if (t == 0) sc[scan_pad(kScanRound)] = next; // the round's end (padding tiles hold 0)
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
            const int i = q * kScanThreads + t;
            if (i < cnt) {
                const uint32_t e = sc[scan_pad(i)];
                ranges[base + i] = make_uint2(e, sc[scan_pad(i + 1)]);
                count[base + i] = e; // the cursors for K3
            }
        }
        carry = next;
        __syncthreads(); // sc and wsum are reused by the next round
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) m = max(m, wmax[w]);
        ctr->pairs_total = carry;
        ctr->max_tile_len = m;
    }
}

// Small buckets (length <= CAP): one CTA per tile over the whole grid.
template <int THREADS, int ROUNDS>
__global__ void __launch_bounds__(THREADS) k_tile_sort_small(const uint2* __restrict__ ranges, uint32_t* __restrict__ pval,
                                                             const uint32_t* __restrict__ pkey,
                                                             const unsigned long long* __restrict__ key,
                                                             const uint32_t* __restrict__ orig,
                                                             const DevCounters* gate, unsigned long long pair_cap) {
    extern __shared__ uint32_t smem[];
    if (gate && gate->pairs_total > pair_cap) return;
    const uint2 r = ranges[blockIdx.x];
    const int L = static_cast<int>(r.y - r.x);
    if (L <= 1 || L > THREADS * ROUNDS) return;
    sort_one_tile<THREADS, ROUNDS>(r, pval, pkey, key, orig, smem);
}

// Large buckets: grid-stride over the device-built list of long tiles.
template <int THREADS, int ROUNDS>
__global__ void __launch_bounds__(THREADS) k_tile_sort_list(const uint2* __restrict__ ranges, uint32_t* __restrict__ pval,
                                                            const uint32_t* __restrict__ pkey,
                                                            const unsigned long long* __restrict__ key,
                                                            const uint32_t* __restrict__ orig,
                                                            const uint32_t* __restrict__ list, const uint32_t* count,
                                                            int min_len_exclusive, const DevCounters* gate,
                                                            unsigned long long pair_cap) {
    extern __shared__ uint32_t smem[];
    pdl_trigger();
    pdl_wait();
    if (gate && gate->pairs_total > pair_cap) return;
    const uint32_t n = *count;
    for (uint32_t q = blockIdx.x; q < n; q += gridDim.x) {
        const uint2 r = ranges[list[q]];
        const int L = static_cast<int>(r.y - r.x);
        if (L <= min_len_exclusive || L > THREADS * ROUNDS) continue;
        sort_one_tile<THREADS, ROUNDS>(r, pval, pkey, key, orig, smem);
        __syncthreads();
    }
}

} // namespace

void launch_tile_scan(uint32_t* tile_count, uint2* ranges, int n_tiles, DevCounters* ctr, uint32_t* big_list,
                      uint32_t list_min, cudaStream_t st) {
    launch_pdl(k_tile_scan, dim3(1), dim3(kScanThreads), 0, st, tile_count, ranges, n_tiles, ctr, big_list, list_min);
}

// Bucket length <= 1024: 128 threads per tile over all tiles; longer buckets
// (listed by k_tile_scan) by 512-thread (<= 4096) and 1024-thread (<= 16384)
// CTAs (power-of-two capacities: the bitonic fallback of sort_one_tile always fits). Longer than kMaxBucketSorted: returns false (caller falls back).
bool launch_tile_sort(const FrameDev& f, const uint32_t* orig, int n_tiles, uint32_t max_len,
                      const DevCounters* d_ctr, cudaStream_t st, int* launches) {
    if (max_len <= 1 || n_tiles == 0) return true;
    if (max_len > kMaxBucketSorted) return false;
    using S1 = TileSortSmem<128, 16>;
    k_tile_sort_small<128, 16><<<n_tiles, 128, S1::bytes(), st>>>(f.ranges, f.pval, f.pkey, f.key, orig, f.gate,
                                                                  f.pair_cap);
    if (launches) *launches += 1;
    if (max_len > 2048u) {
        using S2 = TileSortSmem<512, 8>;
        cudaFuncSetAttribute(k_tile_sort_list<512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S2::bytes()));
        k_tile_sort_list<512, 8><<<148 * 4, 512, S2::bytes(), st>>>(f.ranges, f.pval, f.pkey, f.key, orig, f.big_tiles,
                                                                   &d_ctr->big_tiles, 2048, f.gate, f.pair_cap);
        if (launches) *launches += 1;
    }
    if (max_len > 4096u) {
        using S3 = TileSortSmem<1024, 16>;
        cudaFuncSetAttribute(k_tile_sort_list<1024, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S3::bytes()));
        k_tile_sort_list<1024, 16><<<148, 1024, S3::bytes(), st>>>(f.ranges, f.pval, f.pkey, f.key, orig, f.big_tiles,
                                                                   &d_ctr->big_tiles, 4096, f.gate, f.pair_cap);
        if (launches) *launches += 1;
    }
    return true;
}

// max_len == 0xffffffff: unknown on the host (speculative frame) -- launch both
// list kernels; they read the device-built list and exit when it is empty.
bool launch_tile_sort_long(const FrameDev& f, const uint32_t* orig, uint32_t max_len, uint32_t cap,
                           const DevCounters* d_ctr, cudaStream_t st, int* launches) {
    const bool unknown = max_len == 0xffffffffu;
    if (max_len <= cap) return true;
    if (max_len > kMaxBucketSorted && !unknown) return false;
    using S2 = TileSortSmem<512, 8>;
    cudaFuncSetAttribute(k_tile_sort_list<512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S2::bytes()));
    launch_pdl(k_tile_sort_list<512, 8>, dim3(148 * 4), dim3(512), S2::bytes(), st, f.ranges, f.pval,
               static_cast<const uint32_t*>(f.pkey), static_cast<const unsigned long long*>(f.key), orig,
               static_cast<const uint32_t*>(f.big_tiles), static_cast<const uint32_t*>(&d_ctr->big_tiles),
               static_cast<int>(cap), f.gate, f.pair_cap);
    if (launches) *launches += 1;
    if (max_len > 4096u) {
        using S3 = TileSortSmem<1024, 16>;
        cudaFuncSetAttribute(k_tile_sort_list<1024, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S3::bytes()));
        launch_pdl(k_tile_sort_list<1024, 16>, dim3(148), dim3(1024), S3::bytes(), st, f.ranges, f.pval,
                   static_cast<const uint32_t*>(f.pkey), static_cast<const unsigned long long*>(f.key), orig,
                   static_cast<const uint32_t*>(f.big_tiles), static_cast<const uint32_t*>(&d_ctr->big_tiles), 4096,
                   f.gate, f.pair_cap);
        if (launches) *launches += 1;
    }
    return true;
}

} // namespace ps
