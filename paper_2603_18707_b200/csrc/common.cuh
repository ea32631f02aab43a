// common.cuh — device data layout shared by the rasterizer stages.
//
// HBM layout (all arrays indexed by the ORIGINAL splat index i unless noted):
//   scene (uploaded once, ps_scene):  splats reordered along a 3D Morton curve (so a
//                                     warp's splats are spatial neighbours; orig[]
//                                     keeps the original index for the reference's
//                                     tie-break and every output);
//                                     fp64 SoA mean_x/y/z, scale_x/y/z, rot_w/x/y/z,
//                                     opacity (88 B/splat) and the camera-independent
//                                     3D covariance (6 x fp64, computed at upload) + SH as 12 float4 planes
//                                     sh4[j*n + i] (plane j = floats 4j..4j+3 of the
//                                     Splat3D coefficient order; 192 B/splat at degree 3,
//                                     each plane read fully coalesced)
//   frame (per render, ps_ctx):       depth keys/values for the depth sort, tight tile
//                                     counts, fp64 mean2d / conic / culling root / rect
//                                     (for duplicate-with-keys and the exact fp64 paths)
//                                     and the fp32 blend record (48 B) per splat;
//                                     tile pairs (key = tile id, value = splat index)
//                                     in two ping-pong buffers; per-tile [start,end).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "polysplat_b200.h"

namespace ps {

constexpr int kK1Block = 256;  // splats per K1 / K3 CTA
constexpr int kWinCap = 1024;  // tile cells of a CTA's shared window (K1 counts, K3 scatters)
constexpr int kShPlanes = 12; // 48 floats = 16 coefficients x 3 channels, as float4


struct SceneDev {
    int64_t n = 0;
    double* mean[3] = {nullptr, nullptr, nullptr};
    double* scale[3] = {nullptr, nullptr, nullptr};
    double* rot[4] = {nullptr, nullptr, nullptr, nullptr};
    double* cov[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr}; // 3D covariance (xx xy xz yy yz zz)
    double* opacity = nullptr;
    float4* sh4 = nullptr; // [kShPlanes][n]
    uint32_t* orig = nullptr; // internal -> original splat index (Morton order at upload)
};

// Device counters / status words (one struct per context, zeroed per render).
struct DevCounters {
    unsigned long long frustum;      // splats_frustum_culled
    unsigned long long coarse;       // tile_pairs_coarse
    unsigned long long tight;        // tile_pairs_after_tight_test (== P)
    unsigned long long visible;      // V
    unsigned long long evals;        // kernel_evaluations
    unsigned long long blended;      // fragments_blended
    unsigned long long replay_px;    // flagged pixels (replayed exactly in fp64)
    unsigned long long exact_evals;  // ambiguous alpha decisions re-decided in fp64
    unsigned int error;              // first ps_status raised on device (0 = none)
    unsigned int error_index;        // splat index that raised it
    unsigned int pairs_total;        // P as computed by the count scan
    unsigned int max_tile_len;       // longest per-tile list (K2)
    unsigned long long key_min;      // complement of the min / max fp64 depth bits (visible splats)
    unsigned long long key_max;
    unsigned int big_tiles;          // tiles with > 1024 pairs (listed in FrameDev::big_tiles)
    unsigned int unsorted;           // a blend-prologue bucket sort could not run (re-run presorted)
    unsigned int need_over[3];       // prologue-sorted tiles whose blend needed more than 256 / 512 / 1024
                                     // list positions (the host's next sort prefix, context.cu)
    unsigned int done_ctas;          // blend CTAs finished (the last one publishes the counters to the host)
};

// Per-splat frame arrays (indexed by original splat index).
struct FrameDev {
    unsigned long long* key = nullptr;  // depth bits (visible) or ~0 (culled)
    unsigned long long* key_alt = nullptr;
    uint32_t* val = nullptr;            // splat index (sort payload)
    uint32_t* val_alt = nullptr;
    uint32_t* tcount = nullptr;         // tight tile count (0 when not visible)
    uint32_t* offset = nullptr;         // exclusive scan of tcount in depth order
    double2* mean2d = nullptr;          // fp64 (mx, my)
    double2* conic_ab = nullptr;        // fp64 (a, b)
    double2* conic_cq = nullptr;        // fp64 (c, culling quadric root incl. slack)
    ushort4* rect = nullptr;            // inclusive tile rect (x0, y0, x1, y1)
    unsigned long long* tmask = nullptr; // tight-test bits, bit 8*(ty-y0)+(tx-x0), rects up to 8x8 tiles
    double* opacity_eff = nullptr;      // fp64 opacity_eff
    float4* bl0 = nullptr;              // fp32 blend record: A, beta, gamma, q_hi
    float4* bl1 = nullptr;              //   q_lo, o (or log2 o), eT, color r
    float2* bl2 = nullptr;              //   color g, b
    double* cov_aa = nullptr;           // [3n] only for ps_prepare (debug); may be null
    // tile pairs (length capacity P)
    uint32_t* pkey = nullptr;
    uint32_t* pkey_alt = nullptr;
    uint32_t* pval = nullptr;
    uint32_t* pval_alt = nullptr;
    uint2* ranges = nullptr;            // per tile [start, end)
    uint32_t* big_tiles = nullptr;      // ids of tiles with > 1024 pairs
    uint32_t* tile_order = nullptr;     // tile ids, longest bucket first (K2; the blend's CTA -> tile map)
    // K1's per-CTA tile windows (kK1Block splats per CTA): window rect (x0, y0,
    // w, h; w = 0: no window) and its per-tile pair counts (stride kWinCap), so
    // K3 scatters without counting again
    int4* win_rect = nullptr;
    uint32_t* win_counts = nullptr;
    uint32_t* tile_count = nullptr;     // pairs per tile (K1a), then the K3 bucket cursors
    uint32_t* flags = nullptr;          // flagged pixel ids (capacity W*H)
    double4* replay_vals = nullptr;     // exact fp64 (r, g, b, T) per flagged pixel (optional)
    // Speculative frames (no mid-frame host sync): the pair buffers hold
    // pair_cap entries; kernels writing or reading them do nothing when the
    // scan's pairs_total (in *gate) exceeds it, and the host re-runs the frame.
    const DevCounters* gate = nullptr;
    unsigned long long pair_cap = ~0ull;
};

// Programmatic dependent launch (kernels.h launch_pdl): a dependent kernel may
// be scheduled while its predecessor drains; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible (a no-op without
// PDL), pdl_trigger() lets the dependent launch once every CTA has passed it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ bool pairs_overflow(const FrameDev& f) {
    return f.gate != nullptr && static_cast<unsigned long long>(f.gate->pairs_total) > f.pair_cap;
}

// Blend-kernel parameters derived on the host from ps_config.
enum ThresholdMode : int {
    kQuadricThreshold = 0, // alpha >= eps  <=>  q <= q*(o): skip test in quadric space
    kAlphaThreshold = 1,   // non-monotone kernel: skip test on the fp32 alpha
};

struct KernelF32 {
    int kind;
    int order;
    float c[4];
    float first_root;
};

struct FrameParams {
    ps_camera cam;
    ps_config cfg;
    int tiles_x, tiles_y;
    int sh_floats4;         // float4 planes to read for cfg.sh_degree
    int threshold_mode;     // ThresholdMode
    KernelF32 kf;           // blend kernel in fp32
    float eps_f, floor_f;
    int bound_class;        // K1a specialisation (culling mode x bound kernel)
    int blend_class;        // K1b specialisation (blend kernel)
    double campos[3];       // Camera::position() (projection.hpp:29), computed on the host
    double root_slack;      // polynomial blend kernels: the reference's alpha64 rounding near eps in
                            // q units (host_root_slack); 0 for exp
    int sort_prefix;        // 16x16 blend: list positions its prologue ranks exactly (>= 128; INT_MAX: all)
};

#define PS_CUDA_TRY(expr)                                                  \
    do {                                                                   \
        cudaError_t _e = (expr);                                           \
        if (_e != cudaSuccess) return ::ps::cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)

int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

} // namespace ps
