// tile_sort.cuh — exact per-tile ordering of a bucket in shared memory
// (shared by the standalone sort kernels in binning.cu and the blend prologue).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace ps {

// Exact per-tile order (the reference comparator, raster.cpp:172-175:
// fp64 depth, then splat index; positive fp64 depths order like their bits):
//  0. K3 stored next to every bucket entry a 32-bit coarse depth key
//     (pkey: the frame-global, order-preserving (bits - min) >> shift; see
//     coarse_key), read here coalesced instead of gathering the 64-bit keys;
//  1. 32-bit key = (coarse key - tile minimum) scaled to the tile's own
//     span (order-preserving, injective on coarse keys); one counting-sort
//     pass on its top log2(BINS) bits (shared-memory histogram + atomic
//     cursors, so the order inside a bin is arbitrary);
//  2. every item of a bin holding n > 1 items gets its rank inside the bin by
//     counting the bin's items that precede it in (32-bit key, full depth bits,
//     original index) — n compares per item, all items in parallel; the
//     64-bit depths are gathered only for equal 32-bit keys. A bin of
//     more than kMaxRun items (a degenerate depth cluster) switches the CTA to
//     a bitonic sort on the full key, which is exact for any input.
constexpr int kMaxRun = 256;

constexpr int ilog2_c(int v) { return v <= 1 ? 0 : 1 + ilog2_c(v >> 1); }

// Frame-global coarse key of a visible splat's depth bits: order-preserving
// (monotone non-decreasing), from the frame's key range [kmin, kmax].
__device__ __forceinline__ uint32_t coarse_key(unsigned long long k, unsigned long long kmin,
                                               unsigned long long kmax) {
    const unsigned long long span = kmax - kmin;
    const int nb = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
    return static_cast<uint32_t>((k - kmin) >> (nb > 32 ? nb - 32 : 0));
}

template <int THREADS, int ROUNDS>
struct TileSortSmem {
    static constexpr int CAP = THREADS * ROUNDS;
    static constexpr int WARPS = THREADS / 32;
    static constexpr int BINS = CAP >= 8192 ? 4096 : CAP >= 2048 ? 2048 : 1024;
    static constexpr int BIN_SHIFT = 32 - ilog2_c(BINS);
    // nk [CAP] u32 | perm [CAP] u16 | dest [CAP] u16 | hist [BINS] -> sorted list [CAP]
    // (the bucket's splat indices are re-read from global memory, L2-resident,
    // rather than kept in shared memory: 12 B per slot + the list)
    static constexpr int LIST = 2 * CAP; // word offset of the sorted list
    static constexpr size_t WORDS = LIST + (CAP > BINS ? CAP : BINS);
    __host__ __device__ static constexpr size_t bytes() { return sizeof(uint32_t) * WORDS; }
};

// Returns the sorted bucket in shared memory (smem + LIST); with WRITEBACK also
// writes it to pval[r.x, r.y). The caller synchronises before reading it.
// Prefix mode (limit < L, no WRITEBACK): only the bins holding the first
// `limit` positions are ranked and written, i.e. the list is exact on
// [0, *ranked) with *ranked >= limit (the end of the bin holding position
// limit - 1); positions beyond are undefined until a full sort. The blend's
// tiles terminate after a few hundred entries (their lists are ~3x longer).
// The bitonic fallback pads the bucket to a power of two n: it needs n 64-bit
// keys over the nk / perm / dest arrays (2 CAP words) and n list slots; when
// the padded bucket does not fit (CAP not a power of two), *unsorted is set and
// the caller's frame is re-run with every bucket sorted by the list kernels.
template <int THREADS, int ROUNDS, bool WRITEBACK = true>
__device__ __forceinline__ uint32_t* sort_one_tile(const uint2 r, uint32_t* __restrict__ pval,
                                                   const uint32_t* __restrict__ pkey,
                                                   const unsigned long long* __restrict__ key,
                                                   const uint32_t* __restrict__ orig, uint32_t* smem,
                                                   unsigned int* unsorted = nullptr, int limit = 0x7fffffff,
                                                   int* ranked = nullptr) {
    using S = TileSortSmem<THREADS, ROUNDS>;
    constexpr int CAP = S::CAP, BINS = S::BINS, WARPS = S::WARPS, SH = S::BIN_SHIFT;
    constexpr int PER = BINS / THREADS;
    static_assert(BINS % (4 * THREADS) == 0 && CAP <= 65536, "tile sort shape");
    // the list kernels (WRITEBACK) have no re-run path: their bitonic fallback
    // must always fit, i.e. CAP a power of two (the blend prologue's 1536 flags
    // *unsorted and its frame is re-run with every bucket presorted)
    static_assert(!WRITEBACK || (CAP & (CAP - 1)) == 0, "list-kernel capacity must be a power of two");
    const uint32_t* vin = pval + r.x;                                 // bucket order (global)
    uint32_t* nk = smem;                                              // 32-bit key per bucket slot
    uint16_t* perm = reinterpret_cast<uint16_t*>(smem + CAP);          // bin-sorted position -> slot
    uint16_t* dest = perm + CAP;                                       // bucket slot -> final position
    uint32_t* hist = smem + S::LIST;                                  // counts -> cursors -> list
    __shared__ uint32_t red_min[WARPS], red_max[WARPS];
    __shared__ uint32_t wsum[WARPS];
    __shared__ int need_bitonic;

    const int L = static_cast<int>(r.y - r.x);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (int j = t; j < L; j += THREADS) {
        const uint32_t k = pkey[r.x + j];
        nk[j] = k;
        lo = min(lo, k);
        hi = max(hi, k);
    }
    for (int d = 4 * t; d < BINS; d += 4 * THREADS) *reinterpret_cast<uint4*>(hist + d) = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { red_min[warp] = lo; red_max[warp] = hi; }
    if (t == 0) need_bitonic = 0;
    __syncthreads();
    lo = red_min[0]; hi = red_max[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) { lo = min(lo, red_min[w]); hi = max(hi, red_max[w]); }
    const uint32_t span = hi - lo;
    const int sh = span ? __clz(static_cast<int>(span)) : 0; // (k - lo) << sh spans the full 32 bits
    for (int j = t; j < L; j += THREADS) {
        const uint32_t x = (nk[j] - lo) << sh;
        nk[j] = x;
        atomicAdd(&hist[x >> SH], 1u);
    }
    __syncthreads();
    {   // exclusive scan of the bin counts (PER consecutive bins per thread)
        uint32_t loc[PER];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) { loc[q] = hist[t * PER + q]; sum += loc[q]; }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t base = x - sum;
        for (int w = 0; w < warp; ++w) base += wsum[w];
#pragma unroll
        for (int q = 0; q < PER; ++q) { hist[t * PER + q] = base; base += loc[q]; }
    }
    // prefix mode: the ranked range ends with the bin holding position limit - 1
    // (hist is still exclusive here: the last bin starting before `limit`)
    int Lr = L;
    if (limit < L) {
        __shared__ int s_lr;
        if (t == 0) s_lr = L;
        __syncthreads();
        for (int b = t; b < BINS; b += THREADS) {
            const int s0 = static_cast<int>(hist[b]);
            const int e0 = b + 1 < BINS ? static_cast<int>(hist[b + 1]) : L;
            if (s0 < limit && e0 >= limit && e0 > s0) atomicMin(&s_lr, e0);
        }
        __syncthreads();
        Lr = s_lr;
    }
    __syncthreads();
    for (int j = t; j < L; j += THREADS) perm[atomicAdd(&hist[nk[j] >> SH], 1u)] = static_cast<uint16_t>(j);
    __syncthreads();
    // hist[b] is now the end of bin b: rank every item inside its bin
    for (int p = t; p < Lr; p += THREADS) {
        const uint32_t j = perm[p];
        const uint32_t x = nk[j];
        const uint32_t b = x >> SH;
        const int s = b ? static_cast<int>(hist[b - 1]) : 0, e = static_cast<int>(hist[b]);
        int rank = 0;
        if (e - s > kMaxRun) {
            need_bitonic = 1;
        } else if (e - s > 1) {
            for (int i = s; i < e; ++i) {
                const uint32_t ji = perm[i];
                const uint32_t xi = nk[ji];
                bool before = xi < x;
                if (xi == x && ji != j) {
                    const uint32_t v = vin[j], vi = vin[ji];
                    const unsigned long long ki = key[vi], kv = key[v];
                    before = ki < kv || (ki == kv && orig[vi] < orig[v]);
                }
                rank += before;
            }
        }
        dest[j] = static_cast<uint16_t>(s + rank);
    }
    __syncthreads();
    uint32_t* list = hist;
    const int n_pad = L > 1 ? 1 << (32 - __clz(L - 1)) : 1; // next power of two >= L
    if (need_bitonic && (n_pad > CAP || n_pad > (CAP > BINS ? CAP : BINS))) {
        // (only the blend prologue's CAP 1536 gets here; it passes `unsorted`)
        for (int j = t; j < L; j += THREADS) list[j] = vin[j];
        if (t == 0 && unsorted) atomicExch(unsorted, 1u);
        Lr = L;
    } else if (!need_bitonic && Lr == L) {
        for (int j = t; j < L; j += THREADS) list[dest[j]] = vin[j]; // coalesced read of the bucket
    } else if (!need_bitonic) {
        // prefix: the items of the ranked bins sit at perm positions [0, Lr)
        for (int p = t; p < Lr; p += THREADS) {
            const uint32_t j = perm[p];
            list[dest[j]] = vin[j];
        }
    } else {
        Lr = L;
        // degenerate depth clusters: exact bitonic sort on (bits, original index);
        // full keys over the (now dead) nk / perm / dest arrays
        for (int j = t; j < L; j += THREADS) list[j] = vin[j];
        __syncthreads();
        unsigned long long* fk = reinterpret_cast<unsigned long long*>(smem);
        const int n = n_pad;
        for (int j = t; j < n; j += THREADS) {
            if (j < L) fk[j] = key[list[j]];
            else { fk[j] = ~0ull; list[j] = 0xffffffffu; }
        }
        __syncthreads();
        for (int k = 2; k <= n; k <<= 1)
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                const int lg = __ffs(jj) - 1;
                for (int q = t; q < (n >> 1); q += THREADS) {
                    const int i = ((q >> lg) << (lg + 1)) + (q & (jj - 1));
                    const int ix = i + jj;
                    const unsigned long long ka = fk[i], kb = fk[ix];
                    const uint32_t va = list[i], vb = list[ix];
                    const uint32_t oa = va == 0xffffffffu ? 0xffffffffu : orig[va];
                    const uint32_t ob = vb == 0xffffffffu ? 0xffffffffu : orig[vb];
                    const bool gt = ka > kb || (ka == kb && oa > ob);
                    if (gt == ((i & k) == 0)) { fk[i] = kb; fk[ix] = ka; list[i] = vb; list[ix] = va; }
                }
                __syncthreads();
            }
    }
    if (WRITEBACK) {
        __syncthreads();
        for (int p = t; p < L; p += THREADS) pval[r.x + p] = list[p];
    }
    if (ranked) *ranked = Lr;
    return list;
}

} // namespace ps
