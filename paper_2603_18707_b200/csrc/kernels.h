// kernels.h — host-side launchers of the rasterizer stages (one per .cu TU).
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ps {

// Launch with programmatic stream serialization: the kernel may start while
// the previous kernel on the stream finishes (it calls pdl_wait() before
// reading that kernel's output; common.cuh).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Longest per-tile bucket sorted in shared memory (binning.cu); longer tiles
// take the global radix-sort path.
constexpr uint32_t kMaxBucketSorted = 16384u;
// Longest bucket the blend kernel sorts in its prologue (16x16 tiles), chosen
// per frame from the previous frame's longest bucket: 1536 (18 KB of shared
// memory) or 2048 (24 KB); longer buckets are
// sorted by the list kernels (binning.cu) before the blend. K2 lists every
// bucket longer than the smaller capacity.
constexpr uint32_t kBlendSortCapSmall = 1536u;
constexpr uint32_t kBlendSortCapLarge = 2048u;
inline uint32_t blend_sort_cap(uint32_t longest_bucket) {
    return longest_bucket <= kBlendSortCapSmall ? kBlendSortCapSmall : kBlendSortCapLarge;
}

// exact_kernels.cu (-fmad=false)
// returns the number of kernels launched (1 fused, or K1a + K1b)
int launch_preprocess(const SceneDev& s, const FrameParams& P, const FrameDev& f, DevCounters* ctr,
                      cudaStream_t st);
// K1 fused over a batch of 1 <= nv <= kMaxFusedViews views of one scene and
// config (same bound / blend classes): each splat's inputs read once.
constexpr int kMaxFusedViews = 4;
void launch_preprocess_views(const SceneDev& s, const FrameParams* P, const FrameDev* f, DevCounters* const* ctr,
                             int nv, cudaStream_t st);
// camera-independent 3D covariance of every splat (after each upload)
void launch_scene_cov(const SceneDev& s, cudaStream_t st);
void launch_duplicate(const FrameDev& f, const FrameParams& P, const uint32_t* order, int64_t n,
                      cudaStream_t st);
// K3 also stores each entry's coarse depth key (tile_sort.cuh coarse_key) in f.pkey
// and, when f.tile_order is set, builds the blend's heavy-first tile order
// (one extra CTA). Returns the launches issued.
int launch_duplicate_buckets(const FrameDev& f, const FrameParams& P, int64_t n, const DevCounters* ctr,
                             cudaStream_t st);
void launch_replay(const FrameDev& f, const FrameParams& P, DevCounters* ctr, float* out_rgb,
                   float* out_t, bool count_work, int sm_count, cudaStream_t st);

// sort.cu — stable LSD radix sort (8-bit digits) of (key, uint32 value) pairs.
// The item count is read from device memory (*d_n), capped at n_cap; the grid
// is sized for n_cap. Sorts bits [begin_bit, end_bit). Ping-pongs between
// (keys, vals) and (keys_alt, vals_alt); returns true when the result ends in
// the *_alt buffers. scratch must hold radix_scratch_bytes(n_cap) bytes.
size_t radix_scratch_bytes(int64_t n_cap);
bool radix_sort_u64(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals,
                    uint32_t* vals_alt, const uint32_t* d_n, int64_t n_cap, int begin_bit, int end_bit,
                    void* scratch, cudaStream_t st, int* launches);
bool radix_sort_u32(uint32_t* keys, uint32_t* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                    const uint32_t* d_n, int64_t n_cap, int begin_bit, int end_bit, void* scratch,
                    cudaStream_t st, int* launches);

// Exclusive scan of tcount[order[r]] over r < n into offset[r]; the total goes
// to *d_total. scratch: scan_scratch_bytes(n).
size_t scan_scratch_bytes(int64_t n);
void scan_gathered_counts(const uint32_t* tcount, const uint32_t* order, uint32_t* offset, int64_t n,
                          uint32_t* d_total, void* scratch, cudaStream_t st, int* launches);

// per-tile [start, end) over sorted tile keys (K5)
void launch_ranges(const uint32_t* keys, const uint32_t* d_n, int64_t n_cap, uint2* ranges,
                   int n_tiles, cudaStream_t st, int* launches);

// binning.cu — per-tile buckets (K2 tile scan, K4 per-tile exact depth sort)
// list_min: buckets longer than this go to the long-bucket list (sorted before the blend)
// K3's order CTA (one 256-thread CTA inside K3): used up to 16K tiles, or more
// when K3 itself is long enough to hide it (>= 64 splats per tile)
constexpr int kTileOrderMax = 16384;
inline bool use_tile_order(int n_tiles, int64_t n) {
    return n_tiles <= kTileOrderMax || static_cast<int64_t>(n_tiles) * 64 <= n;
}
void launch_tile_scan(uint32_t* tile_count, uint2* ranges, int n_tiles, DevCounters* ctr, uint32_t* big_list,
                      uint32_t list_min, cudaStream_t st);
// sorts every bucket with 1 < length <= max_items (shared memory); returns false
// when max_items exceeds what one CTA can hold (caller falls back)
bool launch_tile_sort(const FrameDev& f, const uint32_t* orig, int n_tiles, uint32_t max_len,
                      const DevCounters* d_ctr, cudaStream_t st, int* launches);

// blend.cu (K6)
struct BlendOut {
    float* rgb;
    float* t;
};
// sort_in_place: buckets of <= 1024 entries still unsorted (sorted in the blend
// prologue and written back); null when every bucket is already sorted.
// publish (16x16 tiles only): pinned host copy the blend's last CTA writes the
// frame's counters to (no separate device-to-host copy); returns through
// *published the CTA count it leaves in publish->done_ctas (0: not published).
int launch_blend(const FrameDev& f, const FrameParams& P, const uint32_t* pair_vals, uint32_t* sort_in_place,
                 uint32_t sort_cap, const uint32_t* orig, DevCounters* ctr, BlendOut out, bool count_work,
                 cudaStream_t st, bool* replay_fused, DevCounters* publish = nullptr, uint32_t* published = nullptr);
// sort only buckets longer than min_len (the blend prologue handles the rest)
bool launch_tile_sort_long(const FrameDev& f, const uint32_t* orig, uint32_t max_len, uint32_t cap,
                           const DevCounters* d_ctr, cudaStream_t st, int* launches);

// metrics.cu — composite + PSNR / max-abs / SSIM of two framebuffers
// (fp32 or fp64, device pointers) against background bg; synchronises st.
size_t metrics_scratch_bytes();
int launch_image_metrics(const void* rgb_a, const void* t_a, const void* rgb_b, const void* t_b, bool f64, int W,
                         int H, const double bg[3], void* scratch, ps_image_metrics* out, cudaStream_t st);

// utils.cu
// uploaded splat records (device; raw Splat3D or the drop-in's compact 280-B
// record) -> upload staging (fp64 geometry planes + fp32 SH)
void launch_split_records(const double* rec, int64_t n, bool raw, double* staging, float* sh, cudaStream_t st);
// scene reordering along a 30-bit Morton curve of the means (upload time)
void launch_morton_order(const double* means, int64_t n, unsigned long long* bb, uint32_t* keys, uint32_t* vals,
                         cudaStream_t st);
void launch_gather_scene(const double* staging, const double* opac, const float4* sh, const uint32_t* perm,
                         int64_t n, const SceneDev& s, cudaStream_t st);
double measure_fp32_tflops(int sm_count, cudaStream_t st);
double measure_fp64_tflops(int sm_count, cudaStream_t st);

} // namespace ps
