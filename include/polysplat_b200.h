/*
 * polysplat_b200.h — C ABI of the B200-native (sm_100a) forward rasterizer for
 * ReLU-polynomial / exponential 3D Gaussian splatting (arXiv 2603.18707).
 *
 * This is the drop-in boundary for the reference's C++ render API
 * (/root/reference/proj/include/polysplat/raster.hpp:103-113). Every entry point
 * takes plain pointers, sizes and POD structs; no C++ or torch types cross it.
 * The C++ adapter `include/polysplat_b200.hpp` maps the reference's types
 * (Splat3D / Camera / RasterConfig / Framebuffer / PerfCounters) onto it and
 * rethrows the reference's exception types from the status codes below.
 *
 * Semantics follow the reference exactly:
 *   - prepare (projection, culling bound, tile rect, depth sort) is computed in
 *     fp64 with the reference's operation order and no FMA contraction, so the
 *     visible set, depths, conics, bounds and the per-tile lists are bit-identical
 *     to polysplat::prepare_splats / bin_splats (raster.cpp:132-208);
 *   - the blend runs in fp32 (tile-local coordinates, quadric-threshold skip test)
 *     with every discrete decision (alpha < epsilon, T < floor) either certified
 *     by an error bound or re-decided in fp64 with the reference's arithmetic
 *     (raster.cpp:261-283); images agree with the fp64 reference to <= 1e-5.
 *
 * Threading: calls are synchronous per context; contexts are independent and
 * may be used from different host threads (one context per device/thread).
 */
#ifndef POLYSPLAT_B200_H
#define POLYSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 1

/* Number of doubles in one reference polysplat::Splat3D
 * (projection.hpp:13-19: Vec3 mean, Vec3 scale, Quat rotation (w,x,y,z),
 * double opacity, std::array<Vec3,16> sh) — 59 doubles = 472 bytes, standard layout. */
#define PS_SPLAT3D_DOUBLES 59
#define PS_SH_COEFFS 16

/* ---------------------------------------------------------------- status
 * Mirrors the reference's error convention (errors.hpp:9-39, raster.cpp:13-23,
 * projection.cpp:10-22,67, kernel.cpp:43-160,335-369). The adapter rethrows:
 *   PS_INVALID_ARGUMENT          -> std::invalid_argument
 *   PS_NON_ORTHONORMAL_ROTATION  -> polysplat::NonOrthonormalRotation
 *   PS_DEGENERATE_COVARIANCE     -> polysplat::DegenerateCovariance
 *   PS_NO_POSITIVE_ROOT          -> polysplat::NoPositiveRoot
 *   PS_EPSILON_ZERO_UNBOUNDED    -> polysplat::EpsilonZeroUnbounded
 *   PS_FULLY_CULLED              -> polysplat::FullyCulled (culling_radius only)
 *   PS_ERROR                     -> polysplat::Error
 *   PS_CUDA_ERROR / PS_OUT_OF_MEMORY -> std::runtime_error (no reference analogue)
 *   PS_IO_ERROR / PS_MALFORMED_HEADER / PS_UNSUPPORTED_FORMAT / PS_MISSING_PROPERTY /
 *   PS_TRUNCATED_DATA -> polysplat::IoError / MalformedHeader / UnsupportedFormat /
 *                        MissingProperty / TruncatedData (load_ply, scene_io.cpp:53-199) */
typedef enum ps_status {
    PS_OK = 0,
    PS_INVALID_ARGUMENT = 1,
    PS_NON_ORTHONORMAL_ROTATION = 2,
    PS_DEGENERATE_COVARIANCE = 3,
    PS_NO_POSITIVE_ROOT = 4,
    PS_EPSILON_ZERO_UNBOUNDED = 5,
    PS_FULLY_CULLED = 6,
    PS_ERROR = 7,
    PS_CUDA_ERROR = 8,
    PS_OUT_OF_MEMORY = 9,
    PS_IO_ERROR = 10,
    PS_MALFORMED_HEADER = 11,
    PS_UNSUPPORTED_FORMAT = 12,
    PS_MISSING_PROPERTY = 13,
    PS_TRUNCATED_DATA = 14
} ps_status;

/* kernel.hpp:12-17 KernelKind */
enum { PS_KERNEL_EXPONENTIAL = 0, PS_KERNEL_POLY_RELU = 1, PS_KERNEL_POLY_PIECEWISE = 2 };
/* raster.hpp:13-17 CullingMode */
enum { PS_CULL_STOP_THE_POP = 0, PS_CULL_ZERO_CROSSING = 1, PS_CULL_OPACITY_AWARE = 2 };
/* where a buffer lives */
enum { PS_MEM_HOST = 0, PS_MEM_DEVICE = 1 };

/* kernel.hpp:19-26 KernelSpec. coeffs[0..order] constant term first; unused
 * entries must be 0. first_root = +inf for the exponential. */
typedef struct ps_kernel {
    int32_t kind;
    int32_t order;
    double coeffs[4];
    double first_root;
} ps_kernel;

/* raster.hpp:19-35 RasterConfig. thread_count is accepted and validated
 * (>= 0) but has no effect on the device path. */
typedef struct ps_config {
    int32_t tile_size;
    int32_t culling_mode;
    double epsilon;
    double transmittance_floor;
    ps_kernel kernel;
    int32_t has_culling_kernel;
    int32_t sh_degree;
    ps_kernel culling_kernel;
    double v_dilation;
    int32_t clamp_before_blend;
    int32_t thread_count;
} ps_config;

/* projection.hpp:22-31 Camera: row-major world-to-camera rotation, translation. */
typedef struct ps_camera {
    int32_t id;
    int32_t width;
    int32_t height;
    int32_t reserved;
    double fx, fy, cx, cy;
    double rotation[9];
    double translation[3];
} ps_camera;

/* raster.hpp:37-54 PerfCounters */
typedef struct ps_counters {
    uint64_t splats_submitted;
    uint64_t splats_frustum_culled;
    uint64_t tile_pairs_coarse;
    uint64_t tile_pairs_after_tight_test;
    uint64_t kernel_evaluations;
    uint64_t fragments_blended;
} ps_counters;

/* Device-side statistics of the last render on a context (not part of the
 * reference; reported by the bench). Stage times are CUDA-event milliseconds
 * on the context stream, filled only when timing is enabled. */
enum {
    PS_STAGE_PREPROCESS = 0, /* K1: projection, bounds, tight tile counts, blend records */
    PS_STAGE_TILE_SCAN = 1,  /* K2: per-tile ranges / bucket cursors */
    PS_STAGE_HOST_SYNC = 2,  /* the one mid-frame host round trip (sizes pair buffers) */
    PS_STAGE_DUPLICATE = 3,  /* K3: splat indices into per-tile buckets */
    PS_STAGE_TILE_SORT = 4,  /* K4: exact (depth, index) order per bucket */
    PS_STAGE_BLEND = 5,      /* K6: fp32 blend with exact decisions */
    PS_STAGE_REPLAY = 6,     /* K7: fp64 replay of flagged pixels */
    PS_STAGE_COUNT = 7
};
typedef struct ps_stats {
    uint64_t visible;          /* V: prepared splats */
    uint64_t pairs;            /* P: tile pairs after the tight test */
    uint64_t replay_pixels;    /* pixels re-blended exactly in fp64 */
    uint64_t exact_alpha_evals;/* fragments whose alpha<eps decision was re-decided in fp64 */
    float stage_ms[PS_STAGE_COUNT];
    int32_t kernel_launches;   /* kernels launched by the last call */
    int32_t sort_prefix;       /* 16x16 blend: list positions its prologue sorts next frame (INT32_MAX: all) */
} ps_stats;

typedef struct ps_ctx ps_ctx;
typedef struct ps_scene ps_scene;

/* ---------------------------------------------------------------- context */
const char* ps_version(void);
int ps_abi_version(void);
/* Number of CUDA devices visible (0 when no driver / no GPU). */
int ps_device_count(void);
int ps_ctx_create(int device, ps_ctx** out);
void ps_ctx_destroy(ps_ctx* ctx);
/* Message of the last failing call on this context (or of the last failing
 * context-free call when ctx is NULL). Never NULL. */
const char* ps_last_error(const ps_ctx* ctx);
/* Enables per-stage CUDA-event timing (ps_stats.stage_ms). */
int ps_ctx_set_timing(ps_ctx* ctx, int enabled);
int ps_last_stats(const ps_ctx* ctx, ps_stats* out);
/* Blocks until all work queued on the context stream is finished. */
int ps_ctx_synchronize(ps_ctx* ctx);
/* Native CUDA stream (cudaStream_t) of the context, for event timing. */
void* ps_ctx_stream(ps_ctx* ctx);
/* FP32 FFMA issue-rate microbenchmark (TFLOP/s, FFMA = 2 flops): the measured
 * roofline denominator of the FP32-bound blend kernel. */
int ps_measure_fp32_peak(ps_ctx* ctx, double* tflops);
/* fp64 DFMA issue-rate microbenchmark (TFLOP/s): denominator for the fp64 preprocess. */
int ps_measure_fp64_peak(ps_ctx* ctx, double* tflops);

/* ---------------------------------------------------------------- scenes
 * A scene is a device-resident SoA copy of the splats (fp64 geometry, fp32 SH),
 * uploaded once and rendered from any number of cameras
 * (replaces std::span<const Splat3D>, raster.hpp:108). */

/* From an array of reference Splat3D (PS_SPLAT3D_DOUBLES doubles each) in host memory. */
int ps_scene_create_aos(ps_ctx* ctx, const double* splats, int64_t n, ps_scene** out);
/* From SoA arrays: means[n*3], scales[n*3], rotations[n*4] (w,x,y,z),
 * opacities[n], sh[n*16*3] (float, coefficient-major per splat as in Splat3D).
 * memspace: PS_MEM_HOST or PS_MEM_DEVICE (device pointers on the context device). */
int ps_scene_create_soa(ps_ctx* ctx, const double* means, const double* scales,
                        const double* rotations, const double* opacities, const float* sh,
                        int64_t n, int memspace, ps_scene** out);
/* Re-uploads a scene of the same size in place (no reallocation). */
int ps_scene_update_soa(ps_ctx* ctx, ps_scene* scene, const double* means, const double* scales,
                        const double* rotations, const double* opacities, const float* sh,
                        int memspace);
int64_t ps_scene_size(const ps_scene* scene);

/* 3DGS checkpoints (load_ply, scene_io.cpp:53-199; scene_io.hpp:23-27): binary
 * little-endian PLY with float32 x,y,z,f_dc_0..2,f_rest_*,opacity,scale_0..2,
 * rot_0..3 (other properties skipped by stride). The activations
 * (sigmoid(opacity), exp(scale), normalized quaternion) run on the host in
 * fp64 with the reference's expressions, so the fields equal the reference's
 * Splat3D bit for bit. SH degree from the f_rest count (9/24/45 -> 1/2/3).
 * ps_ply_info: header only. ps_ply_load_soa / _splat3d: host arrays of
 * `capacity` splats (SoA as ps_scene_create_soa, or Splat3D records).
 * ps_scene_load_ply: straight into a device scene. */
int ps_ply_info(const char* path, int64_t* n_out, int* sh_degree);
int ps_ply_load_soa(const char* path, double* means, double* scales, double* rotations, double* opacities,
                    float* sh, int64_t capacity, int64_t* n_out, int* sh_degree);
int ps_ply_load_splat3d(const char* path, double* splats, int64_t capacity, int64_t* n_out, int* sh_degree);
int ps_scene_load_ply(ps_ctx* ctx, const char* path, ps_scene** out, int* sh_degree);
void ps_scene_destroy(ps_scene* scene);

/* ---------------------------------------------------------------- render
 * Replaces polysplat::render (raster.hpp:108-109, raster.cpp:212-308).
 * out_rgb: width*height*3 floats (rgb[3*(y*W+x)+ch]), out_transmittance:
 * width*height floats; in out_memspace. counters may be NULL (skips the
 * kernel_evaluations / fragments_blended bookkeeping). */
int ps_render(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cam, const ps_config* cfg,
              float* out_rgb, float* out_transmittance, int out_memspace, ps_counters* counters);

/* A batch of views of one scene (the multi-view bench path). Outputs are
 * contiguous per view: out_rgb[v*W*H*3 ...], out_transmittance[v*W*H ...];
 * all cameras must share width/height. counters: n_views entries or NULL. */
int ps_render_views(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cams, int n_views,
                    const ps_config* cfg, float* out_rgb, float* out_transmittance,
                    int out_memspace, ps_counters* counters);

/* One-shot drop-in equivalent of polysplat::render: host Splat3D array in,
 * fp64 framebuffer out (exact widening of the fp32 image; replayed pixels carry
 * their exact fp64 values). */
int ps_render_splats(ps_ctx* ctx, const double* splats, int64_t n, const ps_camera* cam,
                     const ps_config* cfg, double* out_rgb, double* out_transmittance,
                     ps_counters* counters);

/* Replaces polysplat::count_pairs (raster.hpp:112-113, raster.cpp:310-318). */
int ps_count_pairs(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cam,
                   const ps_config* cfg, ps_counters* counters);

/* Replaces polysplat::prepare_splats (raster.hpp:103-104, raster.cpp:132-177):
 * the depth-sorted prepared list as host SoA arrays of capacity entries.
 * Any output pointer may be NULL. mean2d/conic/cov_aa/color are 2/3/3/3 per
 * entry (conic/cov_aa as xx,xy,yy). *n_out receives V (also when V > capacity,
 * in which case nothing is written and PS_INVALID_ARGUMENT is returned). */
typedef struct ps_prepared {
    uint32_t* index;
    double* depth;
    double* mean2d;
    double* conic;
    double* cov_aa;
    double* opacity_eff;
    float* color;
    double* radius_sigma;
    double* quadric_root;
} ps_prepared;
int ps_prepare(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cam, const ps_config* cfg,
               int64_t capacity, const ps_prepared* out, int64_t* n_out, ps_counters* counters);

/* Per-tile splat lists (the reference's TileBins, raster.cpp:181-208) as CSR:
 * tile_offsets[n_tiles+1], splat_index[P] = original splat index, in blend order.
 * *n_pairs receives P. */
int ps_tile_lists(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cam, const ps_config* cfg,
                  int64_t capacity, uint32_t* tile_offsets, uint32_t* splat_index,
                  int64_t* n_pairs, ps_counters* counters);

/* ---------------------------------------------------------------- image metrics
 * Replaces composite / psnr / ssim / max_abs_diff (metrics.hpp:18-30,
 * metrics.cpp:13-134) on the device. Both framebuffers are composited against
 * bg[3] (rgb + T * bg), then: psnr_db (peak 1, MSE over all channel values;
 * +inf for identical images), ssim (11x11 Gaussian window sigma 1.5, valid
 * mode, mean over channels; ssim_valid = 0 and ssim = 0 when the image is
 * smaller than 11x11, where the reference throws TooSmall) and max_abs_diff.
 * Per-pixel terms are computed in fp64 in the reference's operation order; the
 * sums over pixels are reduced in parallel (relative differences ~1e-15).
 * dtype: PS_DTYPE_F32 (framebuffers as ps_render writes them) or PS_DTYPE_F64
 * (the reference's Framebuffer). Buffers in memspace. */
enum { PS_DTYPE_F32 = 0, PS_DTYPE_F64 = 1 };
typedef struct ps_image_metrics {
    double psnr_db;
    double ssim;
    double max_abs_diff;
    int32_t ssim_valid;
    int32_t reserved;
} ps_image_metrics;
int ps_image_metrics_compute(ps_ctx* ctx, int width, int height, const void* rgb_a, const void* t_a,
                             const void* rgb_b, const void* t_b, int dtype, int memspace, const double* bg,
                             ps_image_metrics* out);

/* compare (metrics.cpp:138-157): renders cfg_a (the reference side) and cfg_b
 * of one scene and camera on the device and compares them with
 * ps_image_metrics_compute; counters_a / counters_b and pair_ratio =
 * pairs_b / pairs_a (0 when pairs_a == 0) as in CompareReport. */
typedef struct ps_compare_report {
    ps_image_metrics metrics;
    ps_counters counters_a;
    ps_counters counters_b;
    double pair_ratio;
} ps_compare_report;
int ps_compare(ps_ctx* ctx, const ps_scene* scene, const ps_camera* cam, const ps_config* cfg_a,
               const ps_config* cfg_b, const double* bg, ps_compare_report* out);

/* ---------------------------------------------------------------- kernel math
 * Host implementations of the exact fp64 math the device preprocess uses
 * (same source, compiled for host). Mirror kernel.cpp. */
/* make_polynomial_kernel (kernel.cpp:141-160): validates, computes first_root. */
int ps_make_polynomial_kernel(int kind, const double* coeffs, int n_coeffs, ps_kernel* out);
ps_kernel ps_make_exponential_kernel(void);
/* first_positive_root (kernel.cpp:117-135). */
int ps_first_positive_root(const double* coeffs, int n_coeffs, double* out);
/* culling_radius (kernel.cpp:335-358); PS_FULLY_CULLED when o*k(0) <= eps. */
int ps_culling_radius(const ps_kernel* kernel, double opacity, double epsilon,
                      double* radius_sigma, double* quadric_root, int* opacity_aware);
/* eval_kernel (kernel.cpp:162-172). */
double ps_eval_kernel(const ps_kernel* kernel, double x);
/* RasterConfig::validate / Camera::validate (raster.cpp:13-23, projection.cpp:10-22). */
int ps_validate_config(const ps_config* cfg);
int ps_validate_camera(const ps_camera* cam);
/* Default RasterConfig (raster.hpp:19-35): tile 16, eps 1/255, floor 1e-4,
 * StopThePop, exponential kernel, v 0.3, sh 3. */
ps_config ps_default_config(void);

/* ---------------------------------------------------------------- synthetic inputs
 * Bench/test harness (not on the render path). Same mt19937_64 uniforms and
 * draw order as the reference generator (scene_io.cpp:304-371, 415-441).
 * kind: 0 grid, 1 random (5000 splats), 2 overexposed sky,
 *       3 parametric random G(n, seed) (scales x (5000/n)^(1/3)),
 *       4 parametric random with skewed opacity 0.005 + 0.99 u^3 (C5).
 * Writes up to `capacity` Splat3D records (PS_SPLAT3D_DOUBLES each) and returns
 * the count via *n_out; with splats == NULL only the count is returned. */
int ps_synth_scene(int kind, uint64_t seed, int64_t n, double* splats, int64_t capacity,
                   int64_t* n_out, int* sh_degree);
/* The same scene straight into SoA arrays (see ps_scene_create_soa). */
int ps_synth_scene_soa(int kind, uint64_t seed, int64_t n, double* means, double* scales,
                       double* rotations, double* opacities, float* sh);
/* orbit_cameras (scene_io.cpp:415-441). */
int ps_orbit_cameras(int count, int width, int height, double fov_deg, double radius,
                     double elevation, ps_camera* out);

#ifdef __cplusplus
}
#endif

#endif /* POLYSPLAT_B200_H */
