// context.cu — host runtime behind the C ABI (include/polysplat_b200.h):
// contexts (device, stream, events, device scratch sized for the largest
// scene/frame seen), device-resident scenes, and the per-frame pipeline
//   K1 preprocess -> K2 depth sort -> K3 scan + duplicate-with-keys ->
//   K4 tile sort -> K5 ranges -> K6 blend -> K7 exact replay.
// One host sync per frame (after the count scan, to size the pair buffers and
// surface device-side errors), plus the final copy-out.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "polysplat_b200.h"

namespace ps {

thread_local std::string g_free_error;

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    g_free_error = buf;
    return e == cudaErrorMemoryAllocation ? PS_OUT_OF_MEMORY : PS_CUDA_ERROR;
}

// host restatements compiled in hostmath.cpp (same exact_math.cuh source)
int host_validate_config(const ps_config& c);
int host_validate_camera(const ps_camera& c);
int host_kernel_threshold_mode(const ps_kernel& k);
double host_root_slack(const ps_kernel& k);
int host_effective_terms(const ps_kernel& k);
void host_camera_position(const ps_camera& cam, double out[3]);

} // namespace ps

using namespace ps;

namespace {

// Persistent host worker threads for the drop-in path's host-side passes
// (copying the caller's Splat3D array into pinned chunks, widening the fp32
// image into the caller's fp64 framebuffer). run() shares ntasks among the
// workers and the calling thread and returns when all are done.
class HostPool {
public:
    explicit HostPool(int n) : n_(std::max(n, 1)) {
        for (int i = 1; i < n_; ++i) th_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return n_; }
    void run(int ntasks, const std::function<void(int)>& fn) {
        if (n_ == 1 || ntasks <= 1) {
            for (int k = 0; k < ntasks; ++k) fn(k);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            ntasks_ = ntasks;
            next_.store(0);
            pending_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [&] { return pending_ == 0; });
    }

private:
    void work() {
        for (int k; (k = next_.fetch_add(1)) < ntasks_;) (*fn_)(k);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            work();
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int ntasks_ = 0;
    std::atomic<int> next_{0};
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

int host_threads() {
    if (const char* e = std::getenv("PS_HOST_THREADS")) {
        const int v = std::atoi(e);
        if (v > 0) return std::min(v, 64);
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return static_cast<int>(std::min(std::max(hc, 1u), 32u));
}

// PS_TRACE_DROPIN=1: phase times of the drop-in path on stderr (diagnostic)
bool trace_dropin() {
    static const bool on = std::getenv("PS_TRACE_DROPIN") != nullptr;
    return on;
}
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// pinned upload ring of the drop-in path: kRing chunks of kChunk bytes
constexpr int kRing = 4;
constexpr size_t kChunk = size_t(16) << 20;

} // namespace

struct ps_scene {
    ps_ctx* ctx = nullptr;
    SceneDev dev;
    void* block = nullptr;
    int64_t n = 0;
};

struct ps_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    bool timing = false;
    cudaEvent_t ev[PS_STAGE_COUNT + 1] = {};
    ps_stats stats{};

    // frame scratch
    int64_t n_cap = 0;
    int64_t p_cap = 0;
    uint32_t last_max_len = 0; // longest bucket of the last rendered frame (speculation hint)
    int64_t clean_tiles = 0;   // the last frame's blend left the counters and this many tile counts zero
    int sort_prefix = 256;      // blend prologue sort prefix for the next frame (adapt_sort_prefix)
    int64_t frame_tiles = 0;    // tiles of the frame in flight
    int64_t pix_cap = 0;
    int64_t tiles_cap = 0;
    FrameDev f;
    void* n_block = nullptr;
    void* p_block = nullptr;
    void* radix_scratch = nullptr;
    size_t radix_scratch_size = 0;
    void* scan_scratch = nullptr;
    size_t scan_scratch_size = 0;
    float* img_rgb = nullptr;
    float* img_t = nullptr;
    double* cov_dbg = nullptr;
    int64_t cov_dbg_cap = 0;
    double4* replay_vals = nullptr;
    DevCounters* d_ctr = nullptr;
    DevCounters* h_ctr = nullptr; // pinned
    void* stage = nullptr;        // scene upload staging
    size_t stage_bytes = 0;
    // image metrics / compare: accumulators and the two framebuffers
    void* metrics_acc = nullptr;
    void* cmp_block = nullptr;
    size_t cmp_bytes = 0;
    // view batches (ps_render_views): one child context per fused view, each
    // with its own frame arrays, counters and stream
    std::vector<ps_ctx*> views;
    cudaEvent_t k1_event = nullptr;
    // drop-in path (ps_render_splats, ps_scene_create_aos): a reusable scene,
    // the raw Splat3D array on the device, a pinned chunk ring (AoS upload),
    // pinned image readback, host worker threads
    ps_scene* dropin = nullptr;
    int64_t dropin_cap = 0;
    void* aos_dev = nullptr;
    size_t aos_dev_bytes = 0;
    char* ring = nullptr;
    cudaEvent_t ring_ev[kRing] = {};
    void* pin_out = nullptr;
    size_t pin_out_bytes = 0;
    std::unique_ptr<HostPool> pool;
};

namespace {

// bytes of a context's device counters block (padded; the per-tile counts follow)
constexpr size_t kCtrBytes = (sizeof(DevCounters) + 255) & ~size_t(255);

int set_err(ps_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    g_free_error = msg;
    return code;
}

int cuda_err(ps_ctx* c, cudaError_t e, const char* what) {
    int code = cuda_fail(e, what, __FILE__, __LINE__);
    if (c) c->err = g_free_error;
    return code;
}

#define CTX_TRY(c, expr)                                  \
    do {                                                  \
        cudaError_t _e = (expr);                          \
        if (_e != cudaSuccess) return cuda_err(c, _e, #expr); \
    } while (0)

const char* status_message(int st) {
    switch (st) {
        case PS_INVALID_ARGUMENT: return "invalid argument";
        case PS_NON_ORTHONORMAL_ROTATION: return "camera rotation is not orthonormal";
        case PS_DEGENERATE_COVARIANCE: return "dilated 2D covariance is singular";
        case PS_NO_POSITIVE_ROOT: return "polynomial has no positive root";
        case PS_EPSILON_ZERO_UNBOUNDED: return "exponential kernel has unbounded support at epsilon 0";
        case PS_FULLY_CULLED: return "opacity below cutoff";
        default: return "error";
    }
}

template <typename T>
T* carve(char*& p, int64_t count) {
    T* r = reinterpret_cast<T*>(p);
    size_t bytes = sizeof(T) * static_cast<size_t>(count);
    bytes = (bytes + 255) & ~size_t(255);
    p += bytes;
    return r;
}

size_t frame_bytes(int64_t n) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    size_t s = 0;
    s += 2 * al(8 * n) + 2 * al(4 * n) + 2 * al(4 * n); // key, key_alt, val, val_alt, tcount, offset
    s += 3 * al(16 * n);                                 // mean2d, conic_ab, conic_cq
    s += al(8 * n) + al(8 * n) + al(8 * n);              // rect, opacity_eff, tmask
    s += 2 * al(16 * n) + al(8 * n);                     // bl0, bl1, bl2
    const size_t nblk = static_cast<size_t>((n + kK1Block - 1) / kK1Block);
    s += al(16 * nblk) + al(4 * nblk * kWinCap);         // win_rect, win_counts
    return s;
}

int ensure_frame(ps_ctx* c, int64_t n) {
    if (n <= c->n_cap) return PS_OK;
    int64_t cap = std::max<int64_t>(n, 1024);
    if (c->n_block) cudaFree(c->n_block);
    c->n_block = nullptr;
    c->n_cap = 0;
    CTX_TRY(c, cudaMalloc(&c->n_block, frame_bytes(cap)));
    char* p = static_cast<char*>(c->n_block);
    c->f.key = carve<unsigned long long>(p, cap);
    c->f.key_alt = carve<unsigned long long>(p, cap);
    c->f.val = carve<uint32_t>(p, cap);
    c->f.val_alt = carve<uint32_t>(p, cap);
    c->f.tcount = carve<uint32_t>(p, cap);
    c->f.offset = carve<uint32_t>(p, cap);
    c->f.mean2d = carve<double2>(p, cap);
    c->f.conic_ab = carve<double2>(p, cap);
    c->f.conic_cq = carve<double2>(p, cap);
    c->f.rect = carve<ushort4>(p, cap);
    c->f.tmask = carve<unsigned long long>(p, cap);
    c->f.opacity_eff = carve<double>(p, cap);
    c->f.bl0 = carve<float4>(p, cap);
    c->f.bl1 = carve<float4>(p, cap);
    c->f.bl2 = carve<float2>(p, cap);
    {
        const int64_t nblk = (cap + kK1Block - 1) / kK1Block;
        c->f.win_rect = carve<int4>(p, nblk);
        c->f.win_counts = carve<uint32_t>(p, nblk * kWinCap);
    }
    size_t rs = radix_scratch_bytes(cap);
    size_t ss = scan_scratch_bytes(cap);
    if (rs > c->radix_scratch_size) {
        if (c->radix_scratch) cudaFree(c->radix_scratch);
        c->radix_scratch = nullptr;
        CTX_TRY(c, cudaMalloc(&c->radix_scratch, rs));
        c->radix_scratch_size = rs;
    }
    if (ss > c->scan_scratch_size) {
        if (c->scan_scratch) cudaFree(c->scan_scratch);
        c->scan_scratch = nullptr;
        CTX_TRY(c, cudaMalloc(&c->scan_scratch, ss));
        c->scan_scratch_size = ss;
    }
    c->n_cap = cap;
    return PS_OK;
}

int ensure_pairs(ps_ctx* c, int64_t p) {
    if (p <= c->p_cap) return PS_OK;
    int64_t cap = std::max<int64_t>(p + p / 4, 1 << 16);
    if (c->p_block) cudaFree(c->p_block);
    c->p_block = nullptr;
    c->p_cap = 0;
    CTX_TRY(c, cudaMalloc(&c->p_block, 4 * ((sizeof(uint32_t) * cap + 255) & ~size_t(255))));
    char* q = static_cast<char*>(c->p_block);
    c->f.pkey = carve<uint32_t>(q, cap);
    c->f.pkey_alt = carve<uint32_t>(q, cap);
    c->f.pval = carve<uint32_t>(q, cap);
    c->f.pval_alt = carve<uint32_t>(q, cap);
    size_t rs = radix_scratch_bytes(cap);
    if (rs > c->radix_scratch_size) {
        if (c->radix_scratch) cudaFree(c->radix_scratch);
        c->radix_scratch = nullptr;
        CTX_TRY(c, cudaMalloc(&c->radix_scratch, rs));
        c->radix_scratch_size = rs;
    }
    c->p_cap = cap;
    return PS_OK;
}

int ensure_image(ps_ctx* c, int64_t pix, int n_tiles) {
    if (pix > c->pix_cap) {
        if (c->img_rgb) cudaFree(c->img_rgb);
        if (c->img_t) cudaFree(c->img_t);
        if (c->f.flags) cudaFree(c->f.flags);
        if (c->replay_vals) cudaFree(c->replay_vals);
        c->img_rgb = nullptr; c->img_t = nullptr; c->f.flags = nullptr; c->replay_vals = nullptr;
        c->pix_cap = 0;
        CTX_TRY(c, cudaMalloc(&c->img_rgb, sizeof(float) * 3 * pix));
        CTX_TRY(c, cudaMalloc(&c->img_t, sizeof(float) * pix));
        CTX_TRY(c, cudaMalloc(&c->f.flags, sizeof(uint32_t) * pix));
        CTX_TRY(c, cudaMalloc(&c->replay_vals, sizeof(double4) * pix));
        c->pix_cap = pix;
    }
    if (n_tiles > c->tiles_cap) {
        if (c->f.ranges) cudaFree(c->f.ranges);
        if (c->f.big_tiles) cudaFree(c->f.big_tiles);
        if (c->f.tile_order) cudaFree(c->f.tile_order);
        c->f.ranges = nullptr;
        c->f.big_tiles = nullptr;
        c->f.tile_order = nullptr;
        c->tiles_cap = 0;
        CTX_TRY(c, cudaMalloc(&c->f.ranges, sizeof(uint2) * n_tiles));
        CTX_TRY(c, cudaMalloc(&c->f.big_tiles, sizeof(uint32_t) * n_tiles));
        CTX_TRY(c, cudaMalloc(&c->f.tile_order, sizeof(uint32_t) * n_tiles));
        // the device counters and the per-tile counts share one block, so one
        // memset clears both at the start of a frame (frame_zero_bytes)
        void* blk = nullptr;
        CTX_TRY(c, cudaMalloc(&blk, kCtrBytes + sizeof(uint32_t) * n_tiles));
        cudaFree(c->d_ctr);
        c->d_ctr = static_cast<DevCounters*>(blk);
        c->f.tile_count = reinterpret_cast<uint32_t*>(static_cast<char*>(blk) + kCtrBytes);
        c->tiles_cap = n_tiles;
        c->clean_tiles = 0;
    }
    return PS_OK;
}

int bits_for(int64_t n_tiles) {
    int b = 0;
    while ((int64_t(1) << b) < n_tiles) ++b;
    return std::max(b, 1);
}

enum class Mode { Render, CountPairs, Prepare, TileLists };

struct FrameRequest {
    Mode mode = Mode::Render;
    float* d_rgb = nullptr; // device outputs (Render)
    float* d_t = nullptr;
    bool count_work = false;
    bool want_replay_vals = false;
    bool no_speculation = false; // force the synchronous (sized) path
    bool k1_done = false;        // K1 (and the counter / tile-count zeroing) already issued by a view batch
    bool defer = false;          // speculative path: return kPending instead of the end-of-frame sync
    bool presort_all = false;    // every bucket sorted by the list kernels before the blend
};

// run_frame status: the speculative frame is queued, finish_frame() completes it
constexpr int kPending = 1000;

struct FrameResult {
    int launches = 0;            // kernels launched so far (deferred frames)
    int64_t visible = 0;
    int64_t pairs = 0;
    bool pairs_in_alt = false;
    bool order_in_alt = false;
    uint32_t published = 0;      // blend CTAs expected in h_ctr->done_ctas (0: counters copied instead)
    DevCounters ctr{};
};

void record(ps_ctx* c, int stage) {
    if (c->timing) cudaEventRecord(c->ev[stage], c->stream);
}

// Validation and the per-frame parameter block (camera, config, kernel classes).
int make_params(ps_ctx* c, const ps_camera& cam, const ps_config& cfg_in, Mode mode, FrameParams& P) {
    int st = host_validate_config(cfg_in);
    if (st != PS_OK) return set_err(c, st, "RasterConfig::validate: invalid configuration");
    st = host_validate_camera(cam);
    if (st != PS_OK)
        return set_err(c, st, st == PS_NON_ORTHONORMAL_ROTATION ? "camera rotation is not orthonormal"
                                                                 : "Camera::validate: invalid camera");
    ps_config cfg = cfg_in;
    if (cfg.sh_degree > 3) cfg.sh_degree = 3;
    if (cfg.sh_degree < 0) cfg.sh_degree = -1;
    if (cfg.kernel.kind != PS_KERNEL_EXPONENTIAL && (cfg.kernel.order < 1 || cfg.kernel.order > 3))
        return set_err(c, PS_INVALID_ARGUMENT, "kernel order must be in {1,2,3}");
    if (cfg.has_culling_kernel && cfg.culling_kernel.kind != PS_KERNEL_EXPONENTIAL &&
        (cfg.culling_kernel.order < 1 || cfg.culling_kernel.order > 3))
        return set_err(c, PS_INVALID_ARGUMENT, "culling kernel order must be in {1,2,3}");

    std::memset(&P, 0, sizeof P);
    P.cam = cam;
    P.cfg = cfg;
    P.tiles_x = (cam.width + cfg.tile_size - 1) / cfg.tile_size;
    P.tiles_y = (cam.height + cfg.tile_size - 1) / cfg.tile_size;
    // the DC term is evaluated for every degree < 1, negative ones included
    // (eval_sh_color, projection.cpp:93-95)
    const int sh_deg = cfg.sh_degree < 0 ? 0 : cfg.sh_degree;
    const int sh_floats = 3 * (sh_deg + 1) * (sh_deg + 1);
    P.sh_floats4 = (sh_floats + 3) / 4;
    P.threshold_mode = host_kernel_threshold_mode(cfg.kernel);
    P.root_slack = host_root_slack(cfg.kernel);
    // The 16x16 blend ranks only the first positions of a tile's list in its
    // prologue (tiles terminate after ~200 entries at C2) unless the last frame
    // replayed many pixels: a tile with a replayed pixel then sorts its whole list
    P.sort_prefix = c->sort_prefix;
    c->frame_tiles = static_cast<int64_t>(P.tiles_x) * P.tiles_y;
#ifdef PS_AB_FULLSORT
    P.sort_prefix = INT_MAX;
#endif
    P.kf.kind = cfg.kernel.kind;
    P.kf.order = cfg.kernel.order;
    for (int j = 0; j < 4; ++j) P.kf.c[j] = static_cast<float>(cfg.kernel.coeffs[j]);
    P.kf.first_root = static_cast<float>(cfg.kernel.first_root);
    P.eps_f = static_cast<float>(cfg.epsilon);
    P.floor_f = static_cast<float>(cfg.transmittance_floor);
    host_camera_position(cam, P.campos);
    {   // kernel specialisations (exact_kernels.cu BoundClass / BlendClass)
        const ps_kernel& bk = cfg.has_culling_kernel ? cfg.culling_kernel : cfg.kernel;
        if (cfg.culling_mode == PS_CULL_STOP_THE_POP) P.bound_class = 0;
        else if (cfg.culling_mode == PS_CULL_ZERO_CROSSING) P.bound_class = 1;
        else if (bk.kind == PS_KERNEL_EXPONENTIAL) P.bound_class = 2;
        else {
            const int nt = host_effective_terms(bk);
            P.bound_class = nt == 2 ? 3 : nt == 3 ? 4 : nt == 4 ? 5 : 6;
        }
        if (cfg.kernel.kind == PS_KERNEL_EXPONENTIAL) P.blend_class = 0;
        else {
            const int nt = host_effective_terms(cfg.kernel);
            P.blend_class = nt == 2 ? 1 : nt == 3 ? 2 : nt == 4 ? 3 : 4;
        }
    }
    return PS_OK;
}

int run_frame(ps_ctx* c, const ps_scene* s, const ps_camera& cam, const ps_config& cfg_in,
              const FrameRequest& req, FrameResult& res);

// Counter checks after a frame's end-of-frame (or mid-frame) readback: device
// errors, and the count scan's pair total against the tight-pair count.
int check_frame_counters(ps_ctx* c, const ps_scene* s, FrameResult& res) {
    res.ctr = *c->h_ctr;
    res.visible = static_cast<int64_t>(res.ctr.visible);
    res.pairs = static_cast<int64_t>(res.ctr.pairs_total);
    if (res.ctr.error) {
        uint32_t orig_index = res.ctr.error_index;
        cudaMemcpy(&orig_index, s->dev.orig + res.ctr.error_index, sizeof(uint32_t), cudaMemcpyDeviceToHost);
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s (splat %u)", status_message(static_cast<int>(res.ctr.error)),
                      orig_index);
        return set_err(c, static_cast<int>(res.ctr.error), buf);
    }
    if (static_cast<unsigned long long>(res.pairs) != res.ctr.tight)
        return set_err(c, PS_ERROR, "internal: pair scan disagrees with tight count");
    return PS_OK;
}

// The 16x16 blend ranks only the first sort_prefix positions of a tile's list
// in its prologue and the rest when the walk (or the exact replay) gets there,
// which costs a second, whole sort. Tiles terminate after a scene-dependent
// depth (C2: ~200 entries; C4 / C5 deeper) and a tile with a replayed pixel
// needs its whole list, so each frame reports how many tiles needed more than
// 256 / 512 / 1024 positions, and the next frame of this context takes the
// prefix of least modelled sort cost: a sort's fixed half (keys, histogram,
// scan, bin scatter over the whole bucket) plus its ranking half in proportion
// to the positions ranked, plus one whole sort for every tile that outgrows the
// prefix; whole lists cost 1. Measured choices: 256 at C2 / C3, 512 at C4,
// whole lists for C5, exp and poly3. Results do not depend on it.
void adapt_sort_prefix(ps_ctx* c, const FrameResult& res) {
    const double nt = static_cast<double>(c->frame_tiles);
    if (!(nt > 0.0)) return;
    const double lavg = std::max(1.0, static_cast<double>(res.pairs) / nt);
    const int prefixes[3] = {256, 512, 1024};
    int best = INT_MAX;
    double best_cost = 1.0;
    for (int k = 0; k < 3; ++k) {
        const double cost = 0.5 + 0.5 * std::min(1.0, prefixes[k] / lavg) + res.ctr.need_over[k] / nt;
        if (cost < best_cost) { best_cost = cost; best = prefixes[k]; }
    }
    c->sort_prefix = best;
}

void frame_stats(ps_ctx* c, const FrameResult& res) {
    adapt_sort_prefix(c, res);
    c->stats.visible = res.visible;
    c->stats.pairs = res.pairs;
    c->stats.replay_pixels = res.ctr.replay_px;
    c->stats.exact_alpha_evals = res.ctr.exact_evals;
    c->stats.kernel_launches = res.launches;
    c->stats.sort_prefix = c->sort_prefix;
    if (c->timing) {
        for (int k = 0; k < PS_STAGE_COUNT; ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c->ev[k], c->ev[k + 1]);
            c->stats.stage_ms[k] = ms;
        }
    }
}

// Completes a speculative frame: one sync, the counter checks, and a sized
// re-run when the frame outgrew the pair buffers or met an unannounced long
// bucket (K1 is re-issued: K2 / K3 consumed its tile counts).
int finish_frame(ps_ctx* c, const ps_scene* s, const ps_camera& cam, const ps_config& cfg_in,
                 const FrameRequest& req, FrameResult& res) {
    CTX_TRY(c, cudaStreamSynchronize(c->stream));
    CTX_TRY(c, cudaGetLastError());
    if (res.published && c->h_ctr->done_ctas != res.published)
        return set_err(c, PS_ERROR, "internal: the blend did not publish the frame counters");
    int st = check_frame_counters(c, s, res);
    if (st != PS_OK) return st;
    const uint32_t cap = blend_sort_cap(c->last_max_len); // what the speculative frame ran with
    const bool long_sorts = c->last_max_len > cap;
    c->last_max_len = res.ctr.max_tile_len;
    if (res.pairs > c->p_cap || res.ctr.max_tile_len > kMaxBucketSorted ||
        (!long_sorts && res.ctr.max_tile_len > cap) || res.ctr.unsorted) {
        FrameRequest sized = req;
        sized.no_speculation = true;
        sized.k1_done = false;
        sized.defer = false;
        sized.presort_all = res.ctr.unsorted != 0; // a prologue sort could not run
        return run_frame(c, s, cam, cfg_in, sized, res);
    }
    frame_stats(c, res);
    // the blend's last CTA zeroed the counters, its CTAs the frame's tile counts
    const int64_t ts = cfg_in.tile_size;
    c->clean_tiles = res.published ? ((cam.width + ts - 1) / ts) * ((cam.height + ts - 1) / ts) : 0;
    return PS_OK;
}

int run_frame(ps_ctx* c, const ps_scene* s, const ps_camera& cam, const ps_config& cfg_in,
              const FrameRequest& req, FrameResult& res) {
    FrameParams P;
    int st = make_params(c, cam, cfg_in, req.mode, P);
    if (st != PS_OK) return st;
    const ps_config& cfg = P.cfg;
    const int64_t n = s->n;
    const int n_tiles = P.tiles_x * P.tiles_y;
    const int64_t pix = static_cast<int64_t>(cam.width) * cam.height;

    CTX_TRY(c, cudaSetDevice(c->device));
    if ((st = ensure_frame(c, n)) != PS_OK) return st;
    if ((st = ensure_image(c, pix, n_tiles)) != PS_OK) return st;
    FrameDev f = c->f;
    f.cov_aa = nullptr;
    f.replay_vals = req.want_replay_vals ? c->replay_vals : nullptr;
    if (req.mode == Mode::Prepare) {
        if (n * 3 > c->cov_dbg_cap) {
            if (c->cov_dbg) cudaFree(c->cov_dbg);
            c->cov_dbg = nullptr;
            c->cov_dbg_cap = 0;
            CTX_TRY(c, cudaMalloc(&c->cov_dbg, sizeof(double) * std::max<int64_t>(3 * n, 3)));
            c->cov_dbg_cap = 3 * n;
        }
        f.cov_aa = c->cov_dbg;
        P.cfg.clamp_before_blend = 0; // prepared colours are unclamped (projection.cpp:93-116)
    }

    int launches = 0;
    cudaStream_t strm = c->stream;
    if (req.mode == Mode::Prepare) f.tile_count = nullptr;
    record(c, 0);
    const bool clean = c->clean_tiles >= n_tiles && c->clean_tiles > 0;
    c->clean_tiles = 0;
    if (!req.k1_done) {
        // counters (+ the per-tile counts right after them) in one memset,
        // unless the last frame's blend left them zeroed
        if (!clean)
            CTX_TRY(c, cudaMemsetAsync(c->d_ctr, 0, kCtrBytes + (f.tile_count ? sizeof(uint32_t) * n_tiles : 0), strm));
        // K1: preprocess (+ tight pair count per tile)
        launches += launch_preprocess(s->dev, P, f, c->d_ctr, strm);
    }
    record(c, 1);
    // speculative frame: no host round trip between the count scan and the blend (below)
    const bool speculative = req.mode == Mode::Render && cfg.tile_size == 16 && c->p_cap > 0 &&
                             !req.no_speculation && !req.presort_all && c->last_max_len <= kMaxBucketSorted;
    const uint32_t* order = nullptr;
    // heavy-first tile order for the blend, built by an extra CTA of K3 (render
    // frames through the bucketed path only; row-major otherwise)
    if (req.mode != Mode::Render || !use_tile_order(n_tiles, n)) f.tile_order = nullptr;
    if (req.mode == Mode::Prepare) {
        // prepare_splats needs the global (depth, index) order: stable radix
        // sort of the fp64 depth bits (culled splats carry ~0 and sort last)
        bool oalt = radix_sort_u64(f.key, f.key_alt, f.val, f.val_alt, nullptr, n, 0, 64, c->radix_scratch,
                                   strm, &launches);
        order = oalt ? f.val_alt : f.val;
        res.order_in_alt = oalt;
        scan_gathered_counts(f.tcount, order, f.offset, n, &c->d_ctr->pairs_total, c->scan_scratch, strm,
                             &launches);
    } else {
        // K2: tile ranges + bucket cursors from the per-tile counts (K1a)
        // a speculative frame lists the buckets its prologue cannot sort; a sized
        // frame lists every bucket above the smaller capacity (its cap is chosen
        // after this scan)
        launch_tile_scan(f.tile_count, f.ranges, n_tiles, c->d_ctr, f.big_tiles,
                         speculative ? blend_sort_cap(c->last_max_len) : kBlendSortCapSmall, strm);
        launches += 1;
    }
    record(c, 2);
    if (speculative) {
        // Speculative frame: no host round trip between the count scan and the
        // blend. The pair buffers from earlier frames are used as they are;
        // K3 / the long-bucket sorts / the blend do nothing when this frame's
        // pairs_total exceeds their capacity, and the host re-runs the frame
        // (sized) after the single end-of-frame sync; likewise for a bucket
        // longer than the shared-memory sorts take (the global-sort fallback).
        record(c, 3);
        f.pkey = c->f.pkey; f.pkey_alt = c->f.pkey_alt; f.pval = c->f.pval; f.pval_alt = c->f.pval_alt;
        f.gate = c->d_ctr;
        f.pair_cap = static_cast<unsigned long long>(c->p_cap);
        launches += launch_duplicate_buckets(f, P, n, c->d_ctr, strm);
        record(c, 4);
        // buckets > kBlendSortCap (sorted outside the blend): launched when the
        // last frame had any; a frame that has them unannounced is re-run
        const uint32_t cap = blend_sort_cap(c->last_max_len);
        const bool long_sorts = c->last_max_len > cap;
        if (long_sorts) launch_tile_sort_long(f, s->dev.orig, 0xffffffffu, cap, c->d_ctr, strm, &launches);
        record(c, 5);
        BlendOut out{req.d_rgb, req.d_t};
        bool replay_fused = false;
        c->h_ctr->done_ctas = 0xffffffffu; // poisoned until the blend's last CTA publishes
#ifdef PS_AB_PRESORT
        launch_tile_sort(f, s->dev.orig, n_tiles, cap, c->d_ctr, strm, &launches);
        launches += launch_blend(f, P, f.pval, nullptr, cap, s->dev.orig, c->d_ctr, out, req.count_work, strm,
                                 &replay_fused, c->h_ctr, &res.published);
#else
        launches += launch_blend(f, P, f.pval, f.pval, cap, s->dev.orig, c->d_ctr, out, req.count_work, strm,
                                 &replay_fused, c->h_ctr, &res.published);
#endif
        record(c, 6);
        record(c, 7);
        if (!res.published)
            CTX_TRY(c, cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, strm));
        res.launches = launches;
        if (req.defer) return kPending; // finish_frame() syncs and checks
        return finish_frame(c, s, cam, cfg_in, req, res);
    }
    CTX_TRY(c, cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, strm));
    CTX_TRY(c, cudaStreamSynchronize(strm));
    CTX_TRY(c, cudaGetLastError());
    record(c, 3);
    if ((st = check_frame_counters(c, s, res)) != PS_OK) return st;
    if (req.mode == Mode::CountPairs || req.mode == Mode::Prepare) {
        c->stats.visible = res.visible;
        c->stats.pairs = res.pairs;
        c->stats.kernel_launches = launches;
        return PS_OK;
    }

    if ((st = ensure_pairs(c, res.pairs)) != PS_OK) return st;
    f.pkey = c->f.pkey; f.pkey_alt = c->f.pkey_alt; f.pval = c->f.pval; f.pval_alt = c->f.pval_alt;
    const uint32_t* svals = f.pval;
    uint32_t* sort_in_blend = nullptr;
    uint32_t sort_cap = kBlendSortCapLarge;
    if (res.ctr.max_tile_len <= kMaxBucketSorted) {
        // K3: scatter splat indices into per-tile buckets
        launches += launch_duplicate_buckets(f, P, n, c->d_ctr, strm);
        record(c, 4);
        // K4: exact (depth, index) order inside every bucket — long buckets
        // here, buckets of <= 1024 in the blend prologue (16x16 tiles), all of
        // them here for the tile-list query or other tile sizes
        if (req.mode == Mode::Render && cfg.tile_size == 16 && !req.presort_all) {
            sort_cap = blend_sort_cap(res.ctr.max_tile_len);
            launch_tile_sort_long(f, s->dev.orig, res.ctr.max_tile_len, sort_cap, c->d_ctr, strm, &launches);
            sort_in_blend = f.pval;
        } else {
            launch_tile_sort(f, s->dev.orig, n_tiles, res.ctr.max_tile_len, c->d_ctr, strm, &launches);
        }
        record(c, 5);
    } else {
        // Fallback for tiles longer than one CTA's shared memory: global stable
        // radix sort by depth, duplicate in depth order, stable sort by tile.
        f.tile_order = nullptr;
        bool oalt = radix_sort_u64(f.key, f.key_alt, f.val, f.val_alt, nullptr, n, 0, 64, c->radix_scratch,
                                   strm, &launches);
        order = oalt ? f.val_alt : f.val;
        scan_gathered_counts(f.tcount, order, f.offset, n, &c->d_ctr->pairs_total, c->scan_scratch, strm,
                             &launches);
        launch_duplicate(f, P, order, n, strm);
        launches += n > 0;
        record(c, 4);
        bool palt = radix_sort_u32(f.pkey, f.pkey_alt, f.pval, f.pval_alt, nullptr, res.pairs, 0,
                                   bits_for(n_tiles), c->radix_scratch, strm, &launches);
        res.pairs_in_alt = palt;
        const uint32_t* skeys = palt ? f.pkey_alt : f.pkey;
        svals = palt ? f.pval_alt : f.pval;
        launch_ranges(skeys, nullptr, res.pairs, f.ranges, n_tiles, strm, &launches);
        record(c, 5);
    }
    if (req.mode == Mode::TileLists) {
        CTX_TRY(c, cudaStreamSynchronize(strm));
        CTX_TRY(c, cudaGetLastError());
        c->stats.visible = res.visible;
        c->stats.pairs = res.pairs;
        c->stats.kernel_launches = launches;
        return PS_OK;
    }
    // K6: blend
    BlendOut out{req.d_rgb, req.d_t};
    bool replay_fused = false;
    launches += launch_blend(f, P, svals, sort_in_blend, sort_cap, s->dev.orig, c->d_ctr, out, req.count_work,
                             strm, &replay_fused);
    record(c, 6);
    if (!replay_fused) {
        // K7: exact replay of flagged pixels (grid-stride over the device-side count)
        FrameDev fr = f;
        fr.pval = const_cast<uint32_t*>(svals);
        launch_replay(fr, P, c->d_ctr, req.d_rgb, req.d_t, req.count_work, c->sm_count, strm);
        launches += 1;
    }
    record(c, 7);
    CTX_TRY(c, cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, strm));
    CTX_TRY(c, cudaStreamSynchronize(strm));
    CTX_TRY(c, cudaGetLastError());
    res.ctr = *c->h_ctr;
    c->last_max_len = res.ctr.max_tile_len;
    if (res.ctr.unsorted && !req.presort_all) { // a prologue sort could not run: every bucket presorted
        FrameRequest again = req;
        again.no_speculation = true;
        again.k1_done = false;
        again.defer = false;
        again.presort_all = true;
        return run_frame(c, s, cam, cfg_in, again, res);
    }
    res.launches = launches;
    frame_stats(c, res);
    return PS_OK;
}

void fill_counters(ps_counters* out, const ps_scene* s, const FrameResult& r, bool with_work) {
    if (!out) return;
    out->splats_submitted = static_cast<uint64_t>(s->n);
    out->splats_frustum_culled = r.ctr.frustum;
    out->tile_pairs_coarse = r.ctr.coarse;
    out->tile_pairs_after_tight_test = r.ctr.tight;
    out->kernel_evaluations = with_work ? r.ctr.evals : 0;
    out->fragments_blended = with_work ? r.ctr.blended : 0;
}

int render_one(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg, float* out_rgb,
               float* out_t, int memspace, ps_counters* counters, bool want_replay_vals,
               FrameResult* res_out) {
    if (!c || !s || !cam || !cfg) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    if (s->ctx != c) return set_err(c, PS_INVALID_ARGUMENT, "scene belongs to another context");
    const int64_t pix = static_cast<int64_t>(cam->width) * cam->height;
    int st = PS_OK;
    if (pix > 0 && (st = ensure_image(c, pix, 1)) != PS_OK) return st;
    FrameRequest req;
    req.mode = Mode::Render;
    const bool dev_out = memspace == PS_MEM_DEVICE;
    req.d_rgb = dev_out && out_rgb ? out_rgb : c->img_rgb;
    req.d_t = dev_out && out_t ? out_t : c->img_t;
    req.count_work = counters != nullptr;
    req.want_replay_vals = want_replay_vals;
    FrameResult r;
    st = run_frame(c, s, *cam, *cfg, req, r);
    if (st != PS_OK) return st;
    if (!dev_out) {
        if (out_rgb)
            CTX_TRY(c, cudaMemcpyAsync(out_rgb, req.d_rgb, sizeof(float) * 3 * pix, cudaMemcpyDeviceToHost, c->stream));
        if (out_t)
            CTX_TRY(c, cudaMemcpyAsync(out_t, req.d_t, sizeof(float) * pix, cudaMemcpyDeviceToHost, c->stream));
        CTX_TRY(c, cudaStreamSynchronize(c->stream));
    }
    fill_counters(counters, s, r, true);
    if (res_out) *res_out = r;
    return PS_OK;
}

// Device staging of one scene upload: the raw arrays (fp64 geometry interleaved
// per splat: means | scales | rots | opacity; SH as n x 48 fp32) and the Morton
// sort's keys / scratch.
struct Staging {
    double* st = nullptr;
    float4* sh_st = nullptr;
    uint32_t* keys = nullptr;
    unsigned long long* bb = nullptr;
    void* scratch = nullptr;
};

int stage_alloc(ps_ctx* c, int64_t n, Staging& S) {
    // (every region 256-byte aligned: an odd n leaves 88 n bytes of fp64
    // geometry, which would misalign the float4 SH staging after it)
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t geo = al(sizeof(double) * 11 * static_cast<size_t>(n));
    const size_t shb = al(sizeof(float) * 48 * static_cast<size_t>(n));
    const size_t keyb = al(sizeof(uint32_t) * 4 * static_cast<size_t>(n));
    const size_t sort_bytes = keyb + 256 + radix_scratch_bytes(n);
    const size_t stage_bytes = geo + shb + sort_bytes + 256;
    if (stage_bytes > c->stage_bytes) {
        if (c->stage) cudaFree(c->stage);
        c->stage = nullptr;
        c->stage_bytes = 0;
        CTX_TRY(c, cudaMalloc(&c->stage, stage_bytes));
        c->stage_bytes = stage_bytes;
    }
    char* p = static_cast<char*>(c->stage);
    S.st = reinterpret_cast<double*>(p);
    S.sh_st = reinterpret_cast<float4*>(p + geo);
    S.keys = reinterpret_cast<uint32_t*>(p + geo + shb);
    S.bb = reinterpret_cast<unsigned long long*>(p + geo + shb + keyb);
    S.scratch = reinterpret_cast<char*>(S.bb) + 256;
    return PS_OK;
}

// Orders the staged splats along a Morton curve of their means and gathers
// them into the scene's SoA planes in that order (+ the 3D covariances).
int finish_upload(ps_ctx* c, ps_scene* s, const Staging& S) {
    const int64_t n = s->n;
    uint32_t* keys_alt = S.keys + n;
    uint32_t* vals = S.keys + 2 * n;
    uint32_t* vals_alt = S.keys + 3 * n;
    launch_morton_order(S.st, n, S.bb, S.keys, vals, c->stream);
    const bool alt = radix_sort_u32(S.keys, keys_alt, vals, vals_alt, nullptr, n, 0, 30, S.scratch, c->stream, nullptr);
    launch_gather_scene(S.st, S.st + 10 * n, S.sh_st, alt ? vals_alt : vals, n, s->dev, c->stream);
    launch_scene_cov(s->dev, c->stream);
    CTX_TRY(c, cudaStreamSynchronize(c->stream));
    CTX_TRY(c, cudaGetLastError());
    return PS_OK;
}

int upload_soa(ps_ctx* c, ps_scene* s, const double* means, const double* scales, const double* rots,
               const double* opac, const float* sh, int memspace) {
    const int64_t n = s->n;
    if (n == 0) return PS_OK;
    const cudaMemcpyKind kind = memspace == PS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // Stage the raw arrays (a few large DMAs; full link rate when the host
    // buffers are pinned), then order and gather them on the device.
    Staging S;
    int st = stage_alloc(c, n, S);
    if (st != PS_OK) return st;
    CTX_TRY(c, cudaMemcpyAsync(S.st, means, sizeof(double) * 3 * n, kind, c->stream));
    CTX_TRY(c, cudaMemcpyAsync(S.st + 3 * n, scales, sizeof(double) * 3 * n, kind, c->stream));
    CTX_TRY(c, cudaMemcpyAsync(S.st + 6 * n, rots, sizeof(double) * 4 * n, kind, c->stream));
    CTX_TRY(c, cudaMemcpyAsync(S.st + 10 * n, opac, sizeof(double) * n, kind, c->stream));
    // exactly the caller's 48 n floats (the staging layout only pads the region)
    CTX_TRY(c, cudaMemcpyAsync(S.sh_st, sh, sizeof(float) * 48 * static_cast<size_t>(n), kind, c->stream));
    return finish_upload(c, s, S);
}

HostPool& pool_of(ps_ctx* c) {
    if (!c->pool) c->pool = std::make_unique<HostPool>(host_threads());
    return *c->pool;
}

// Host (pageable) -> device transfer through the context's pinned chunk ring:
// the host workers fill chunk k of a free ring slot while the DMA engine moves
// chunk k-1 (a pageable cudaMemcpy would bounce through the driver's small
// staging buffers at a fraction of the link rate). fill(dst, first, count)
// writes `count` records starting at record `first` (rec_bytes each) into
// pinned memory.
int h2d_chunked(ps_ctx* c, void* dst, int64_t records, size_t rec_bytes,
                const std::function<void(char*, int64_t, int64_t)>& fill) {
    if (records == 0) return PS_OK;
    if (!c->ring) {
        CTX_TRY(c, cudaMallocHost(reinterpret_cast<void**>(&c->ring), kRing * kChunk));
        for (auto& e : c->ring_ev) CTX_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    HostPool& pool = pool_of(c);
    char* d = static_cast<char*>(dst);
    const int64_t per_chunk = static_cast<int64_t>(kChunk / rec_bytes);
    double t_wait = 0.0, t_copy = 0.0;
    const bool tr = trace_dropin();
    int64_t first = 0;
    for (int k = 0; first < records; ++k) {
        const int slot = k % kRing;
        const double t0 = tr ? now_ms() : 0.0;
        if (k >= kRing) CTX_TRY(c, cudaEventSynchronize(c->ring_ev[slot]));
        const double t1 = tr ? now_ms() : 0.0;
        const int64_t cnt = std::min(per_chunk, records - first);
        char* pin = c->ring + static_cast<size_t>(slot) * kChunk;
        const int parts = cnt * rec_bytes >= (size_t(1) << 20) ? pool.size() : 1;
        pool.run(parts, [&](int q) {
            const int64_t a = cnt * q / parts, b = cnt * (q + 1) / parts;
            fill(pin + a * rec_bytes, first + a, b - a);
        });
        if (tr) { t_wait += t1 - t0; t_copy += now_ms() - t1; }
        CTX_TRY(c, cudaMemcpyAsync(d + first * rec_bytes, pin, cnt * rec_bytes, cudaMemcpyHostToDevice, c->stream));
        CTX_TRY(c, cudaEventRecord(c->ring_ev[slot], c->stream));
        first += cnt;
    }
    if (tr)
        std::fprintf(stderr, "[dropin] h2d %lld x %zu B: host fill %.3f ms, ring waits %.3f ms (%d threads)\n",
                     static_cast<long long>(records), rec_bytes, t_copy, t_wait, pool.size());
    return PS_OK;
}

// Reference Splat3D array (host) -> scene. The host workers narrow each 472-B
// record to the 280-B upload record (fp64 mean, scale, rotation, opacity; SH
// rounded to fp32 — the scene keeps fp32 SH either way) while filling the
// pinned ring, so both the host memory traffic and the PCIe bytes shrink by
// 40%; the device splits the records into the staging layout. PS_DROPIN_RAW=1
// ships the raw 472-B records instead (A/B).
constexpr size_t kCompactRec = 11 * sizeof(double) + 48 * sizeof(float);

int upload_aos(ps_ctx* c, ps_scene* s, const double* splats) {
    const int64_t n = s->n;
    if (n == 0) return PS_OK;
    Staging S;
    int st = stage_alloc(c, n, S);
    if (st != PS_OK) return st;
    static const bool raw = std::getenv("PS_DROPIN_RAW") != nullptr;
    const size_t rec = raw ? sizeof(double) * PS_SPLAT3D_DOUBLES : kCompactRec;
    const size_t bytes = rec * static_cast<size_t>(n);
    if (bytes > c->aos_dev_bytes) {
        if (c->aos_dev) cudaFree(c->aos_dev);
        c->aos_dev = nullptr;
        c->aos_dev_bytes = 0;
        CTX_TRY(c, cudaMalloc(&c->aos_dev, bytes));
        c->aos_dev_bytes = bytes;
    }
    if (raw) {
        st = h2d_chunked(c, c->aos_dev, n, rec, [&](char* dst, int64_t first, int64_t cnt) {
            std::memcpy(dst, splats + first * PS_SPLAT3D_DOUBLES, cnt * rec);
        });
    } else {
        st = h2d_chunked(c, c->aos_dev, n, rec, [&](char* dst, int64_t first, int64_t cnt) {
            for (int64_t i = 0; i < cnt; ++i) {
                const double* sp = splats + (first + i) * PS_SPLAT3D_DOUBLES;
                char* o = dst + i * kCompactRec;
                std::memcpy(o, sp, 11 * sizeof(double));
                float* f = reinterpret_cast<float*>(o + 11 * sizeof(double));
                for (int k = 0; k < 48; ++k) f[k] = static_cast<float>(sp[11 + k]);
            }
        });
    }
    if (st != PS_OK) return st;
    launch_split_records(static_cast<const double*>(c->aos_dev), n, raw, S.st, reinterpret_cast<float*>(S.sh_st),
                         c->stream);
    return finish_upload(c, s, S);
}

int alloc_scene(ps_ctx* c, int64_t n, ps_scene** out, int64_t capacity = 0) {
    auto* s = new ps_scene();
    s->ctx = c;
    s->n = n;
    s->dev.n = n;
    // planes sized for `capacity` splats: a smaller scene reuses them (the SH
    // planes are strided by the scene's own n, which only shrinks the region)
    const int64_t cap = std::max<int64_t>(std::max(n, capacity), 1);
    const size_t plane = (sizeof(double) * cap + 255) & ~size_t(255);
    const size_t shb = (sizeof(float) * 48 * cap + 255) & ~size_t(255);
    const size_t origb = (sizeof(uint32_t) * cap + 255) & ~size_t(255);
    cudaError_t e = cudaMalloc(&s->block, 17 * plane + shb + origb);
    if (e != cudaSuccess) {
        delete s;
        return cuda_err(c, e, "cudaMalloc(scene)");
    }
    char* p = static_cast<char*>(s->block);
    for (int k = 0; k < 3; ++k) { s->dev.mean[k] = reinterpret_cast<double*>(p); p += plane; }
    for (int k = 0; k < 3; ++k) { s->dev.scale[k] = reinterpret_cast<double*>(p); p += plane; }
    for (int k = 0; k < 4; ++k) { s->dev.rot[k] = reinterpret_cast<double*>(p); p += plane; }
    s->dev.opacity = reinterpret_cast<double*>(p); p += plane;
    for (int k = 0; k < 6; ++k) { s->dev.cov[k] = reinterpret_cast<double*>(p); p += plane; }
    s->dev.sh4 = reinterpret_cast<float4*>(p);
    p += shb;
    s->dev.orig = reinterpret_cast<uint32_t*>(p);
    *out = s;
    return PS_OK;
}

} // namespace

// ====================================================================== C ABI
extern "C" {

const char* ps_version(void) { return "polysplat-b200 0.1 (sm_100a)"; }
int ps_abi_version(void) { return PS_ABI_VERSION; }

int ps_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int ps_ctx_create(int device, ps_ctx** out) {
    if (!out) return set_err(nullptr, PS_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_err(nullptr, PS_CUDA_ERROR, "no CUDA device available: the B200 path has no CPU fallback");
    }
    if (device < 0 || device >= n) return set_err(nullptr, PS_INVALID_ARGUMENT, "device index out of range");
    auto* c = new ps_ctx();
    c->device = device;
    auto fail = [&](cudaError_t err, const char* what) {
        int code = cuda_err(c, err, what);
        ps_ctx_destroy(c);
        return code;
    };
    if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e, "cudaSetDevice");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return fail(e, "cudaGetDeviceProperties");
    if (prop.major < 10) {
        ps_ctx_destroy(c);
        return set_err(nullptr, PS_CUDA_ERROR, "device is not sm_100-class (Blackwell) — this build targets sm_100a");
    }
    c->sm_count = prop.multiProcessorCount;
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
    for (auto& ev : c->ev)
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaMalloc(&c->d_ctr, kCtrBytes)) != cudaSuccess) return fail(e, "counters");
    if ((e = cudaMallocHost(&c->h_ctr, sizeof(DevCounters))) != cudaSuccess) return fail(e, "pinned counters");
    *out = c;
    return PS_OK;
}

void ps_ctx_destroy(ps_ctx* c) {
    if (!c) return;
    for (ps_ctx* v : c->views) ps_ctx_destroy(v);
    c->views.clear();
    cudaSetDevice(c->device);
    if (c->dropin) ps_scene_destroy(c->dropin);
    c->dropin = nullptr;
    c->pool.reset();
    if (c->ring) cudaFreeHost(c->ring);
    if (c->pin_out) cudaFreeHost(c->pin_out);
    for (auto& e : c->ring_ev)
        if (e) cudaEventDestroy(e);
    if (c->aos_dev) cudaFree(c->aos_dev);
    if (c->k1_event) cudaEventDestroy(c->k1_event);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& ev : c->ev)
        if (ev) cudaEventDestroy(ev);
    void* bufs[] = {c->n_block, c->p_block, c->radix_scratch, c->scan_scratch, c->img_rgb, c->img_t,
                    c->f.flags, c->f.ranges, c->f.big_tiles, c->f.tile_order, c->cov_dbg, c->replay_vals, c->d_ctr, c->stage,
                    c->metrics_acc, c->cmp_block};
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* ps_last_error(const ps_ctx* c) { return c ? c->err.c_str() : g_free_error.c_str(); }

int ps_ctx_set_timing(ps_ctx* c, int enabled) {
    if (!c) return PS_INVALID_ARGUMENT;
    c->timing = enabled != 0;
    return PS_OK;
}

int ps_last_stats(const ps_ctx* c, ps_stats* out) {
    if (!c || !out) return PS_INVALID_ARGUMENT;
    *out = c->stats;
    return PS_OK;
}

int ps_ctx_synchronize(ps_ctx* c) {
    if (!c) return PS_INVALID_ARGUMENT;
    CTX_TRY(c, cudaStreamSynchronize(c->stream));
    return PS_OK;
}

void* ps_ctx_stream(ps_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int ps_measure_fp64_peak(ps_ctx* c, double* tflops) {
    if (!c || !tflops) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    CTX_TRY(c, cudaSetDevice(c->device));
    *tflops = measure_fp64_tflops(c->sm_count, c->stream);
    CTX_TRY(c, cudaGetLastError());
    return PS_OK;
}

int ps_measure_fp32_peak(ps_ctx* c, double* tflops) {
    if (!c || !tflops) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    CTX_TRY(c, cudaSetDevice(c->device));
    *tflops = measure_fp32_tflops(c->sm_count, c->stream);
    CTX_TRY(c, cudaGetLastError());
    return PS_OK;
}

int ps_scene_create_soa(ps_ctx* c, const double* means, const double* scales, const double* rotations,
                        const double* opacities, const float* sh, int64_t n, int memspace, ps_scene** out) {
    if (!c || !out || n < 0) return set_err(c, PS_INVALID_ARGUMENT, "bad scene arguments");
    if (n > 0 && (!means || !scales || !rotations || !opacities || !sh))
        return set_err(c, PS_INVALID_ARGUMENT, "null scene array");
    if (n > 0xFFFFFFFFll) return set_err(c, PS_INVALID_ARGUMENT, "scene too large (> 2^32 splats)");
    CTX_TRY(c, cudaSetDevice(c->device));
    ps_scene* s = nullptr;
    int st = alloc_scene(c, n, &s);
    if (st != PS_OK) return st;
    st = upload_soa(c, s, means, scales, rotations, opacities, sh, memspace);
    if (st != PS_OK) {
        ps_scene_destroy(s);
        return st;
    }
    *out = s;
    return PS_OK;
}

int ps_scene_update_soa(ps_ctx* c, ps_scene* s, const double* means, const double* scales,
                        const double* rotations, const double* opacities, const float* sh, int memspace) {
    if (!c || !s || s->ctx != c) return set_err(c, PS_INVALID_ARGUMENT, "bad scene");
    CTX_TRY(c, cudaSetDevice(c->device));
    return upload_soa(c, s, means, scales, rotations, opacities, sh, memspace);
}

int ps_scene_create_aos(ps_ctx* c, const double* splats, int64_t n, ps_scene** out) {
    if (!c || !out || n < 0 || (n > 0 && !splats)) return set_err(c, PS_INVALID_ARGUMENT, "bad scene arguments");
    if (n > 0xFFFFFFFFll) return set_err(c, PS_INVALID_ARGUMENT, "scene too large (> 2^32 splats)");
    CTX_TRY(c, cudaSetDevice(c->device));
    ps_scene* s = nullptr;
    int st = alloc_scene(c, n, &s);
    if (st != PS_OK) return st;
    if ((st = upload_aos(c, s, splats)) != PS_OK) {
        ps_scene_destroy(s);
        return st;
    }
    *out = s;
    return PS_OK;
}

int64_t ps_scene_size(const ps_scene* s) { return s ? s->n : -1; }

void ps_scene_destroy(ps_scene* s) {
    if (!s) return;
    if (s->block) {
        cudaSetDevice(s->ctx->device);
        cudaStreamSynchronize(s->ctx->stream);
        cudaFree(s->block);
    }
    delete s;
}

int ps_render(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg, float* out_rgb,
              float* out_t, int memspace, ps_counters* counters) {
    return render_one(c, s, cam, cfg, out_rgb, out_t, memspace, counters, false, nullptr);
}

namespace {

// One in-flight batch of ps_render_views: up to kMaxFusedViews views on one set
// of child contexts.
struct ViewBatch {
    int first = 0, nv = 0;
    FrameRequest req[ps::kMaxFusedViews];
    FrameResult res[ps::kMaxFusedViews];
    int status[ps::kMaxFusedViews];
};

// Issues batch vb on child-context set `set`: K1 fused over its views on the
// parent stream, then each view's K2..K6 queued on its child stream (deferred).
int issue_views(ps_ctx* c, const ps_scene* s, const ps_camera* cams, const ps_config* cfg, float* out_rgb,
                float* out_t, bool dev_out, bool count, int set, ViewBatch& vb, float* k1_ms) {
    const int G = ps::kMaxFusedViews;
    const int64_t pix = static_cast<int64_t>(cams[0].width) * cams[0].height;
    FrameParams P[ps::kMaxFusedViews];
    FrameDev f[ps::kMaxFusedViews];
    DevCounters* ctr[ps::kMaxFusedViews];
    for (int k = 0; k < vb.nv; ++k) {
        ps_ctx* v = c->views[set * G + k];
        v->timing = c->timing;
        int st = make_params(v, cams[vb.first + k], *cfg, Mode::Render, P[k]);
        if (st != PS_OK) return set_err(c, st, v->err);
        const int n_tiles = P[k].tiles_x * P[k].tiles_y;
        if ((st = ensure_frame(v, s->n)) != PS_OK || (st = ensure_image(v, pix, n_tiles)) != PS_OK)
            return set_err(c, st, v->err);
        f[k] = v->f;
        f[k].cov_aa = nullptr;
        f[k].replay_vals = nullptr;
        ctr[k] = v->d_ctr;
        CTX_TRY(c, cudaMemsetAsync(v->d_ctr, 0, kCtrBytes + sizeof(uint32_t) * n_tiles, c->stream));
    }
    if (c->timing) cudaEventRecord(c->ev[0], c->stream);
    launch_preprocess_views(s->dev, P, f, ctr, vb.nv, c->stream);
    if (c->timing) cudaEventRecord(c->ev[1], c->stream);
    CTX_TRY(c, cudaEventRecord(c->k1_event, c->stream));
    for (int k = 0; k < vb.nv; ++k) {
        ps_ctx* v = c->views[set * G + k];
        CTX_TRY(c, cudaStreamWaitEvent(v->stream, c->k1_event, 0));
        FrameRequest& rq = vb.req[k];
        rq = FrameRequest{};
        rq.mode = Mode::Render;
        rq.d_rgb = dev_out && out_rgb ? out_rgb + 3 * pix * (vb.first + k) : v->img_rgb;
        rq.d_t = dev_out && out_t ? out_t + pix * (vb.first + k) : v->img_t;
        rq.count_work = count;
        rq.k1_done = true;
        rq.defer = true;
        vb.res[k] = FrameResult{};
        vb.status[k] = run_frame(v, s, cams[vb.first + k], *cfg, rq, vb.res[k]);
        if (vb.status[k] != PS_OK && vb.status[k] != kPending) return set_err(c, vb.status[k], v->err);
    }
    if (c->timing) {
        float ms = 0.f;
        cudaEventSynchronize(c->ev[1]);
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        *k1_ms += ms;
    }
    return PS_OK;
}

// Completes batch vb: per-view end-of-frame checks, outputs, counters, stats.
int finish_views(ps_ctx* c, const ps_scene* s, const ps_camera* cams, const ps_config* cfg, float* out_rgb,
                 float* out_t, bool dev_out, ps_counters* counters, int set, ViewBatch& vb, ps_stats& total) {
    const int G = ps::kMaxFusedViews;
    const int64_t pix = static_cast<int64_t>(cams[0].width) * cams[0].height;
    for (int k = 0; k < vb.nv; ++k) {
        ps_ctx* v = c->views[set * G + k];
        if (vb.status[k] == kPending) {
            const int st = finish_frame(v, s, cams[vb.first + k], *cfg, vb.req[k], vb.res[k]);
            if (st != PS_OK) return set_err(c, st, v->err);
        }
        if (!dev_out) {
            if (out_rgb)
                CTX_TRY(c, cudaMemcpyAsync(out_rgb + 3 * pix * (vb.first + k), vb.req[k].d_rgb,
                                           sizeof(float) * 3 * pix, cudaMemcpyDeviceToHost, v->stream));
            if (out_t)
                CTX_TRY(c, cudaMemcpyAsync(out_t + pix * (vb.first + k), vb.req[k].d_t, sizeof(float) * pix,
                                           cudaMemcpyDeviceToHost, v->stream));
            CTX_TRY(c, cudaStreamSynchronize(v->stream));
        }
        fill_counters(counters ? counters + vb.first + k : nullptr, s, vb.res[k], true);
        total.visible += v->stats.visible;
        total.pairs += v->stats.pairs;
        total.replay_pixels += v->stats.replay_pixels;
        total.exact_alpha_evals += v->stats.exact_alpha_evals;
        total.kernel_launches += v->stats.kernel_launches;
        for (int q = 1; q < PS_STAGE_COUNT; ++q) total.stage_ms[q] += v->stats.stage_ms[q];
    }
    total.kernel_launches += 2; // the fused K1a + K1b
    return PS_OK;
}

} // namespace

int ps_render_views(ps_ctx* c, const ps_scene* s, const ps_camera* cams, int n_views, const ps_config* cfg,
                    float* out_rgb, float* out_t, int memspace, ps_counters* counters) {
    if (!c || !s || !cams || !cfg || n_views < 0) return set_err(c, PS_INVALID_ARGUMENT, "bad arguments");
    if (s->ctx != c) return set_err(c, PS_INVALID_ARGUMENT, "scene belongs to another context");
    for (int v = 0; v < n_views; ++v) {
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
            return set_err(c, PS_INVALID_ARGUMENT, "all views must share width/height");
    }
    if (n_views == 0) return PS_OK;
    const bool dev_out = memspace == PS_MEM_DEVICE;
    CTX_TRY(c, cudaSetDevice(c->device));
    // Views go in batches of up to kMaxFusedViews: K1 is issued once per batch
    // (each splat's inputs read once for all of its views) on
    // this context's stream; each view then runs K2..K6 on its own child
    // context's stream. Two sets of child contexts alternate, so batch b+1's
    // K1 overlaps batch b's binning / blend.
    const int G = ps::kMaxFusedViews;
    const int nb = (n_views + G - 1) / G;
    const int sets = nb > 1 ? 2 : 1;
    const int need = (sets - 1) * G + std::min(G, n_views);
    while (static_cast<int>(c->views.size()) < need) {
        ps_ctx* v = nullptr;
        int st = ps_ctx_create(c->device, &v);
        if (st != PS_OK) return set_err(c, st, "cannot create a view context");
        c->views.push_back(v);
    }
    if (!c->k1_event) CTX_TRY(c, cudaEventCreateWithFlags(&c->k1_event, cudaEventDisableTiming));
    ps_stats total{};
    float k1_ms = 0.f;
    ViewBatch vb[2];
    int st = PS_OK;
    for (int b = 0; b <= nb && st == PS_OK; ++b) {
        if (b < nb) {
            ViewBatch& cur = vb[b % 2];
            cur.first = b * G;
            cur.nv = std::min(G, n_views - b * G);
            st = issue_views(c, s, cams, cfg, out_rgb, out_t, dev_out, counters != nullptr, b % 2, cur, &k1_ms);
        }
        if (st == PS_OK && b > 0)
            st = finish_views(c, s, cams, cfg, out_rgb, out_t, dev_out, counters, (b - 1) % 2, vb[(b - 1) % 2],
                              total);
    }
    if (st != PS_OK) {
        for (ps_ctx* v : c->views) cudaStreamSynchronize(v->stream); // leave no batch in flight
        return st;
    }
    // per-call totals over the views (stage times: K1 per batch on this
    // stream, the rest summed over the views' streams, which overlap)
    total.stage_ms[PS_STAGE_PREPROCESS] = k1_ms;
    c->stats = total;
    return PS_OK;
}

int ps_render_splats(ps_ctx* c, const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                     double* out_rgb, double* out_t, ps_counters* counters) {
    if (!c || !cam || !cfg || n < 0 || (n > 0 && !splats)) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    if (n > 0xFFFFFFFFll) return set_err(c, PS_INVALID_ARGUMENT, "scene too large (> 2^32 splats)");
    int st = host_validate_config(*cfg);
    if (st != PS_OK) return set_err(c, st, "RasterConfig::validate: invalid configuration");
    st = host_validate_camera(*cam);
    if (st != PS_OK)
        return set_err(c, st, st == PS_NON_ORTHONORMAL_ROTATION ? "camera rotation is not orthonormal"
                                                                 : "Camera::validate: invalid camera");
    CTX_TRY(c, cudaSetDevice(c->device));
    // the context's drop-in scene, reallocated only when a call brings more splats
    if (!c->dropin || c->dropin_cap < n) {
        if (c->dropin) ps_scene_destroy(c->dropin);
        c->dropin = nullptr;
        c->dropin_cap = 0;
        if ((st = alloc_scene(c, n, &c->dropin)) != PS_OK) return st;
        c->dropin_cap = n;
    }
    ps_scene* s = c->dropin;
    s->n = n;
    s->dev.n = n;
    const bool tr = trace_dropin();
    const double t0 = tr ? now_ms() : 0.0;
    if ((st = upload_aos(c, s, splats)) != PS_OK) return st;
    const double t1 = tr ? now_ms() : 0.0;
    FrameResult r;
    if ((st = render_one(c, s, cam, cfg, nullptr, nullptr, PS_MEM_DEVICE, counters, true, &r)) != PS_OK) return st;
    const double t2 = tr ? now_ms() : 0.0;
    // read back the fp32 image and the exact fp64 values of the replayed
    // pixels into pinned memory, then widen into the caller's fp64 framebuffer
    // on the host workers and patch the replayed pixels
    const int64_t pix = static_cast<int64_t>(cam->width) * cam->height;
    const uint64_t nf = r.ctr.replay_px;
    const size_t img_b = (sizeof(float) * 4 * static_cast<size_t>(pix) + 255) & ~size_t(255);
    const size_t ids_b = (sizeof(uint32_t) * nf + 255) & ~size_t(255);
    const size_t need = img_b + ids_b + sizeof(double4) * nf;
    if (need > c->pin_out_bytes) {
        if (c->pin_out) cudaFreeHost(c->pin_out);
        c->pin_out = nullptr;
        c->pin_out_bytes = 0;
        CTX_TRY(c, cudaMallocHost(&c->pin_out, need + need / 8));
        c->pin_out_bytes = need + need / 8;
    }
    float* h_rgb = static_cast<float*>(c->pin_out);
    float* h_t = h_rgb + 3 * pix;
    uint32_t* h_ids = reinterpret_cast<uint32_t*>(static_cast<char*>(c->pin_out) + img_b);
    double4* h_vals = reinterpret_cast<double4*>(static_cast<char*>(c->pin_out) + img_b + ids_b);
    if (pix > 0) {
        if (out_rgb) CTX_TRY(c, cudaMemcpyAsync(h_rgb, c->img_rgb, sizeof(float) * 3 * pix, cudaMemcpyDeviceToHost, c->stream));
        if (out_t) CTX_TRY(c, cudaMemcpyAsync(h_t, c->img_t, sizeof(float) * pix, cudaMemcpyDeviceToHost, c->stream));
    }
    if (nf) {
        CTX_TRY(c, cudaMemcpyAsync(h_ids, c->f.flags, sizeof(uint32_t) * nf, cudaMemcpyDeviceToHost, c->stream));
        CTX_TRY(c, cudaMemcpyAsync(h_vals, c->replay_vals, sizeof(double4) * nf, cudaMemcpyDeviceToHost, c->stream));
    }
    CTX_TRY(c, cudaStreamSynchronize(c->stream));
    const double t3 = tr ? now_ms() : 0.0;
    HostPool& pool = pool_of(c);
    const int parts = pix >= (1 << 16) ? pool.size() : 1;
    pool.run(parts, [&](int q) {
        const int64_t a = pix * q / parts, b = pix * (q + 1) / parts;
        if (out_rgb)
            for (int64_t k = 3 * a; k < 3 * b; ++k) out_rgb[k] = h_rgb[k];
        if (out_t)
            for (int64_t k = a; k < b; ++k) out_t[k] = h_t[k];
    });
    for (uint64_t k = 0; k < nf; ++k) {
        const uint32_t p = h_ids[k];
        if (out_rgb) { out_rgb[3 * p] = h_vals[k].x; out_rgb[3 * p + 1] = h_vals[k].y; out_rgb[3 * p + 2] = h_vals[k].z; }
        if (out_t) out_t[p] = h_vals[k].w;
    }
    if (tr)
        std::fprintf(stderr, "[dropin] upload %.3f ms, render %.3f ms, readback %.3f ms, widen %.3f ms\n", t1 - t0,
                     t2 - t1, t3 - t2, now_ms() - t3);
    return PS_OK;
}

int ps_count_pairs(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg,
                   ps_counters* counters) {
    if (!c || !s || !cam || !cfg) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    FrameRequest req;
    req.mode = Mode::CountPairs;
    FrameResult r;
    int st = run_frame(c, s, *cam, *cfg, req, r);
    if (st != PS_OK) return st;
    fill_counters(counters, s, r, false);
    return PS_OK;
}

int ps_prepare(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg, int64_t capacity,
               const ps_prepared* out, int64_t* n_out, ps_counters* counters) {
    if (!c || !s || !cam || !cfg || !n_out) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    FrameRequest req;
    req.mode = Mode::Prepare;
    FrameResult r;
    int st = run_frame(c, s, *cam, *cfg, req, r);
    if (st != PS_OK) return st;
    fill_counters(counters, s, r, false);
    const int64_t v = r.visible;
    *n_out = v;
    if (!out || v == 0) return PS_OK; // size query
    if (v > capacity) return set_err(c, PS_INVALID_ARGUMENT, "capacity too small");
    const FrameDev& f = c->f;
    const uint32_t* order = r.order_in_alt ? f.val_alt : f.val;
    const unsigned long long* keys = r.order_in_alt ? f.key_alt : f.key;
    std::vector<uint32_t> idx(v);
    std::vector<unsigned long long> kk(v);
    CTX_TRY(c, cudaMemcpy(idx.data(), order, sizeof(uint32_t) * v, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(kk.data(), keys, sizeof(unsigned long long) * v, cudaMemcpyDeviceToHost));
    const int64_t n = s->n;
    std::vector<double2> m(n), ab(n), cq(n);
    std::vector<double> o(n), cov(3 * n);
    std::vector<float4> b1(n);
    std::vector<float2> b2(n);
    CTX_TRY(c, cudaMemcpy(m.data(), f.mean2d, sizeof(double2) * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(ab.data(), f.conic_ab, sizeof(double2) * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(cq.data(), f.conic_cq, sizeof(double2) * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(o.data(), f.opacity_eff, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(cov.data(), c->cov_dbg, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(b1.data(), f.bl1, sizeof(float4) * n, cudaMemcpyDeviceToHost));
    CTX_TRY(c, cudaMemcpy(b2.data(), f.bl2, sizeof(float2) * n, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> orig(n);
    CTX_TRY(c, cudaMemcpy(orig.data(), s->dev.orig, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
    // the device sort is stable in internal (Morton) order; the reference breaks
    // depth ties by the original index (raster.cpp:172-175)
    for (int64_t a = 0; a < v;) {
        int64_t b = a + 1;
        while (b < v && kk[b] == kk[a]) ++b;
        if (b - a > 1)
            std::sort(idx.begin() + a, idx.begin() + b, [&](uint32_t x, uint32_t y) { return orig[x] < orig[y]; });
        a = b;
    }
    for (int64_t k = 0; k < v; ++k) {
        const uint32_t i = idx[k];
        if (out->index) out->index[k] = orig[i];
        if (out->depth) { double d; std::memcpy(&d, &kk[k], 8); out->depth[k] = d; }
        if (out->mean2d) { out->mean2d[2 * k] = m[i].x; out->mean2d[2 * k + 1] = m[i].y; }
        if (out->conic) { out->conic[3 * k] = ab[i].x; out->conic[3 * k + 1] = ab[i].y; out->conic[3 * k + 2] = cq[i].x; }
        if (out->cov_aa) for (int j = 0; j < 3; ++j) out->cov_aa[3 * k + j] = cov[3 * i + j];
        if (out->opacity_eff) out->opacity_eff[k] = o[i];
        if (out->color) { out->color[3 * k] = b1[i].w; out->color[3 * k + 1] = b2[i].x; out->color[3 * k + 2] = b2[i].y; }
        if (out->quadric_root) out->quadric_root[k] = cq[i].y;
        if (out->radius_sigma) out->radius_sigma[k] = std::sqrt(cq[i].y);
    }
    return PS_OK;
}

int ps_tile_lists(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg, int64_t capacity,
                  uint32_t* tile_offsets, uint32_t* splat_index, int64_t* n_pairs, ps_counters* counters) {
    if (!c || !s || !cam || !cfg || !n_pairs) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    FrameRequest req;
    req.mode = Mode::TileLists;
    FrameResult r;
    int st = run_frame(c, s, *cam, *cfg, req, r);
    if (st != PS_OK) return st;
    fill_counters(counters, s, r, false);
    *n_pairs = r.pairs;
    if (!tile_offsets && !splat_index) return PS_OK; // size query
    if (r.pairs > capacity) return set_err(c, PS_INVALID_ARGUMENT, "capacity too small");
    const int ts = cfg->tile_size;
    const int n_tiles = ((cam->width + ts - 1) / ts) * ((cam->height + ts - 1) / ts);
    std::vector<uint2> rng(n_tiles);
    CTX_TRY(c, cudaMemcpy(rng.data(), c->f.ranges, sizeof(uint2) * n_tiles, cudaMemcpyDeviceToHost));
    if (tile_offsets) {
        // tiles without pairs carry [0,0); rebuild a monotone CSR
        uint32_t run = 0;
        for (int t = 0; t < n_tiles; ++t) {
            if (rng[t].y > rng[t].x) { tile_offsets[t] = rng[t].x; run = rng[t].y; }
            else tile_offsets[t] = run;
        }
        tile_offsets[n_tiles] = static_cast<uint32_t>(r.pairs);
    }
    if (splat_index && r.pairs) {
        CTX_TRY(c, cudaMemcpy(splat_index, r.pairs_in_alt ? c->f.pval_alt : c->f.pval,
                              sizeof(uint32_t) * r.pairs, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> orig(s->n);
        CTX_TRY(c, cudaMemcpy(orig.data(), s->dev.orig, sizeof(uint32_t) * s->n, cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < r.pairs; ++k) splat_index[k] = orig[splat_index[k]];
    }
    return PS_OK;
}

namespace {

// device buffers for two framebuffers (rgb + T) of `bytes_per_elem`-sized values
int ensure_cmp(ps_ctx* c, int64_t pix, size_t elem) {
    // four 256-byte aligned regions (rgb a, T a, rgb b, T b; ps_image_metrics_compute)
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t need = 2 * al(3 * static_cast<size_t>(pix) * elem) + 2 * al(static_cast<size_t>(pix) * elem);
    if (!c->metrics_acc) CTX_TRY(c, cudaMalloc(&c->metrics_acc, ps::metrics_scratch_bytes()));
    if (need > c->cmp_bytes) {
        if (c->cmp_block) cudaFree(c->cmp_block);
        c->cmp_block = nullptr;
        c->cmp_bytes = 0;
        CTX_TRY(c, cudaMalloc(&c->cmp_block, need));
        c->cmp_bytes = need;
    }
    return PS_OK;
}

} // namespace

int ps_image_metrics_compute(ps_ctx* c, int width, int height, const void* rgb_a, const void* t_a,
                             const void* rgb_b, const void* t_b, int dtype, int memspace, const double* bg,
                             ps_image_metrics* out) {
    if (!c || !out || !rgb_a || !t_a || !rgb_b || !t_b) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    if (width < 0 || height < 0 || (dtype != PS_DTYPE_F32 && dtype != PS_DTYPE_F64))
        return set_err(c, PS_INVALID_ARGUMENT, "bad image size or dtype");
    CTX_TRY(c, cudaSetDevice(c->device));
    const int64_t pix = static_cast<int64_t>(width) * height;
    const size_t elem = dtype == PS_DTYPE_F64 ? sizeof(double) : sizeof(float);
    int st = ensure_cmp(c, pix, elem);
    if (st != PS_OK) return st;
    const void* p[4] = {rgb_a, t_a, rgb_b, t_b};
    if (memspace == PS_MEM_HOST) {
        char* q = static_cast<char*>(c->cmp_block);
        const size_t sz[4] = {3 * pix * elem, pix * elem, 3 * pix * elem, pix * elem};
        for (int k = 0; k < 4; ++k) {
            CTX_TRY(c, cudaMemcpyAsync(q, p[k], sz[k], cudaMemcpyHostToDevice, c->stream));
            p[k] = q;
            q += (sz[k] + 255) & ~size_t(255);
        }
    }
    const double white[3] = {1.0, 1.0, 1.0};
    if (ps::launch_image_metrics(p[0], p[1], p[2], p[3], dtype == PS_DTYPE_F64, width, height, bg ? bg : white,
                                 c->metrics_acc, out, c->stream) != 0)
        CTX_TRY(c, cudaGetLastError());
    CTX_TRY(c, cudaGetLastError());
    return PS_OK;
}

int ps_compare(ps_ctx* c, const ps_scene* s, const ps_camera* cam, const ps_config* cfg_a, const ps_config* cfg_b,
               const double* bg, ps_compare_report* out) {
    if (!c || !s || !cam || !cfg_a || !cfg_b || !out) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    const int64_t pix = static_cast<int64_t>(cam->width) * cam->height;
    int st = ensure_cmp(c, pix, sizeof(float));
    if (st != PS_OK) return st;
    float* a_rgb = static_cast<float*>(c->cmp_block);
    float* a_t = a_rgb + 3 * pix;
    float* b_rgb = a_t + pix;
    float* b_t = b_rgb + 3 * pix;
    if ((st = render_one(c, s, cam, cfg_a, a_rgb, a_t, PS_MEM_DEVICE, &out->counters_a, false, nullptr)) != PS_OK)
        return st;
    if ((st = render_one(c, s, cam, cfg_b, b_rgb, b_t, PS_MEM_DEVICE, &out->counters_b, false, nullptr)) != PS_OK)
        return st;
    if ((st = ps_image_metrics_compute(c, cam->width, cam->height, a_rgb, a_t, b_rgb, b_t, PS_DTYPE_F32,
                                       PS_MEM_DEVICE, bg, &out->metrics)) != PS_OK)
        return st;
    const uint64_t pa = out->counters_a.tile_pairs_after_tight_test;
    out->pair_ratio = pa ? static_cast<double>(out->counters_b.tile_pairs_after_tight_test) / static_cast<double>(pa)
                         : 0.0;
    return PS_OK;
}

int ps_scene_load_ply(ps_ctx* c, const char* path, ps_scene** out, int* sh_degree) {
    if (!c || !out) return set_err(c, PS_INVALID_ARGUMENT, "null argument");
    int64_t n = 0;
    int deg = 0;
    int st = ps_ply_info(path, &n, &deg);
    if (st != PS_OK) return set_err(c, st, g_free_error);
    std::vector<double> means(3 * n), scales(3 * n), rots(4 * n), opac(n);
    std::vector<float> sh(48 * n);
    st = ps_ply_load_soa(path, means.data(), scales.data(), rots.data(), opac.data(), sh.data(), n, &n, &deg);
    if (st != PS_OK) return set_err(c, st, g_free_error);
    if (sh_degree) *sh_degree = deg;
    return ps_scene_create_soa(c, means.data(), scales.data(), rots.data(), opac.data(), sh.data(), n, PS_MEM_HOST,
                               out);
}

} // extern "C"
