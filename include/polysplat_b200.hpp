// polysplat_b200.hpp — header-only C++ adapter: the reference's rasterizer API
// (include/polysplat/raster.hpp:103-113 in /root/reference/proj) implemented on
// the B200 C ABI (polysplat_b200.h). A reference user swaps
//     polysplat::render(splats, cam, cfg)            ->  polysplat::b200::render(splats, cam, cfg)
//     polysplat::count_pairs / prepare_splats         ->  polysplat::b200::count_pairs / prepare_splats
// with the same argument types, the same results (bit-exact prepared data,
// per-tile lists and counters; images within 1e-5 of the fp64 reference) and
// the same exception types (std::invalid_argument, polysplat::Error subclasses).
//
// Include after the reference headers are on the include path; link
// libpolysplat_b200.so. Nothing here depends on the reference library itself.
#pragma once

#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "polysplat/errors.hpp"
#include "polysplat/metrics.hpp"
#include "polysplat/projection.hpp"
#include "polysplat/raster.hpp"
#include "polysplat/scene_io.hpp"
#include "polysplat_b200.h"

namespace polysplat::b200 {

static_assert(sizeof(Splat3D) == PS_SPLAT3D_DOUBLES * sizeof(double), "Splat3D layout changed");

// Status -> the reference's exception types (errors.hpp:9-39).
[[noreturn]] inline void throw_status(int st, const char* msg) {
    const std::string m = msg ? msg : "polysplat_b200 error";
    switch (st) {
        case PS_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case PS_NON_ORTHONORMAL_ROTATION: throw NonOrthonormalRotation(m);
        case PS_DEGENERATE_COVARIANCE: throw DegenerateCovariance(m);
        case PS_NO_POSITIVE_ROOT: throw NoPositiveRoot(m);
        case PS_EPSILON_ZERO_UNBOUNDED: throw EpsilonZeroUnbounded(m);
        case PS_FULLY_CULLED: throw FullyCulled(m);
        case PS_ERROR: throw Error(m);
        case PS_IO_ERROR: throw IoError(m);
        case PS_MALFORMED_HEADER: throw MalformedHeader(m);
        case PS_UNSUPPORTED_FORMAT: throw UnsupportedFormat(m);
        case PS_MISSING_PROPERTY: throw MissingProperty(m);
        case PS_TRUNCATED_DATA: throw TruncatedData(m);
        default: throw std::runtime_error(m);
    }
}

inline ps_kernel to_ps(const KernelSpec& k) {
    ps_kernel o;
    std::memset(&o, 0, sizeof o);
    o.kind = static_cast<int32_t>(k.kind);
    o.order = k.order;
    for (std::size_t i = 0; i < k.coeffs.size() && i < 4; ++i) o.coeffs[i] = k.coeffs[i];
    o.first_root = k.first_root;
    return o;
}

inline ps_config to_ps(const RasterConfig& c) {
    ps_config o;
    std::memset(&o, 0, sizeof o);
    o.tile_size = c.tile_size;
    o.culling_mode = static_cast<int32_t>(c.culling_mode);
    o.epsilon = c.epsilon;
    o.transmittance_floor = c.transmittance_floor;
    o.kernel = to_ps(c.kernel);
    o.has_culling_kernel = c.culling_kernel ? 1 : 0;
    o.culling_kernel = to_ps(c.culling_kernel ? *c.culling_kernel : c.kernel);
    o.v_dilation = c.v_dilation;
    o.sh_degree = c.sh_degree;
    o.clamp_before_blend = c.clamp_before_blend ? 1 : 0;
    o.thread_count = c.thread_count;
    return o;
}

inline ps_camera to_ps(const Camera& c) {
    ps_camera o;
    std::memset(&o, 0, sizeof o);
    o.id = c.id;
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    for (int i = 0; i < 9; ++i) o.rotation[i] = c.rotation.m[i];
    o.translation[0] = c.translation.x;
    o.translation[1] = c.translation.y;
    o.translation[2] = c.translation.z;
    return o;
}

inline PerfCounters from_ps(const ps_counters& c) {
    PerfCounters o;
    o.splats_submitted = c.splats_submitted;
    o.splats_frustum_culled = c.splats_frustum_culled;
    o.tile_pairs_coarse = c.tile_pairs_coarse;
    o.tile_pairs_after_tight_test = c.tile_pairs_after_tight_test;
    o.kernel_evaluations = c.kernel_evaluations;
    o.fragments_blended = c.fragments_blended;
    return o;
}

// One device context (stream + scratch) per host thread, as the C ABI requires.
class Device {
public:
    explicit Device(int device = 0) {
        ps_ctx* c = nullptr;
        const int st = ps_ctx_create(device, &c);
        if (st != PS_OK) throw_status(st, ps_last_error(nullptr));
        ctx_.reset(c);
    }
    ps_ctx* get() const { return ctx_.get(); }
    void check(int st) const {
        if (st != PS_OK) throw_status(st, ps_last_error(ctx_.get()));
    }

private:
    struct Del {
        void operator()(ps_ctx* c) const { ps_ctx_destroy(c); }
    };
    std::unique_ptr<ps_ctx, Del> ctx_;
};

inline Device& default_device() {
    thread_local Device d(0);
    return d;
}

// A scene resident in HBM: upload once, render many cameras (the multi-view path).
class Scene {
public:
    Scene(Device& dev, std::span<const Splat3D> splats) : dev_(&dev) {
        ps_scene* s = nullptr;
        dev.check(ps_scene_create_aos(dev.get(), reinterpret_cast<const double*>(splats.data()),
                                      static_cast<int64_t>(splats.size()), &s));
        scene_.reset(s);
    }
    ps_scene* get() const { return scene_.get(); }
    Device& device() const { return *dev_; }

private:
    struct Del {
        void operator()(ps_scene* s) const { ps_scene_destroy(s); }
    };
    Device* dev_;
    std::unique_ptr<ps_scene, Del> scene_;
};

// polysplat::render (raster.hpp:108-109)
inline std::pair<Framebuffer, PerfCounters> render(std::span<const Splat3D> splats, const Camera& cam,
                                                   const RasterConfig& cfg, Device& dev = default_device()) {
    const ps_camera c = to_ps(cam);
    const ps_config g = to_ps(cfg);
    dev.check(ps_validate_config(&g));
    dev.check(ps_validate_camera(&c));
    Framebuffer fb(cam.width, cam.height);
    ps_counters ctr;
    dev.check(ps_render_splats(dev.get(), reinterpret_cast<const double*>(splats.data()),
                               static_cast<int64_t>(splats.size()), &c, &g, fb.rgb.data(), fb.transmittance.data(),
                               &ctr));
    return {std::move(fb), from_ps(ctr)};
}

// Render from a resident scene (fp32 device image widened to the fp64 Framebuffer).
inline std::pair<Framebuffer, PerfCounters> render(const Scene& scene, const Camera& cam, const RasterConfig& cfg) {
    const ps_camera c = to_ps(cam);
    const ps_config g = to_ps(cfg);
    const std::size_t pix = static_cast<std::size_t>(cam.width) * cam.height;
    std::vector<float> rgb(3 * pix), tr(pix);
    ps_counters ctr;
    scene.device().check(ps_render(scene.device().get(), scene.get(), &c, &g, rgb.data(), tr.data(), PS_MEM_HOST, &ctr));
    Framebuffer fb(cam.width, cam.height);
    for (std::size_t k = 0; k < 3 * pix; ++k) fb.rgb[k] = rgb[k];
    for (std::size_t k = 0; k < pix; ++k) fb.transmittance[k] = tr[k];
    return {std::move(fb), from_ps(ctr)};
}

// polysplat::count_pairs (raster.hpp:112-113)
inline PerfCounters count_pairs(std::span<const Splat3D> splats, const Camera& cam, const RasterConfig& cfg,
                                Device& dev = default_device()) {
    Scene s(dev, splats);
    const ps_camera c = to_ps(cam);
    const ps_config g = to_ps(cfg);
    ps_counters ctr;
    dev.check(ps_count_pairs(dev.get(), s.get(), &c, &g, &ctr));
    return from_ps(ctr);
}

// polysplat::prepare_splats (raster.hpp:103-104). Colours come from the fp32
// SH evaluation (|error| ~1e-7); every other field is bit-identical.
inline std::vector<ProjectedSplat> prepare_splats(std::span<const Splat3D> splats, const Camera& cam,
                                                  const RasterConfig& cfg, PerfCounters& counters,
                                                  Device& dev = default_device()) {
    Scene s(dev, splats);
    const ps_camera c = to_ps(cam);
    const ps_config g = to_ps(cfg);
    const std::size_t n = splats.size();
    std::vector<uint32_t> index(n);
    std::vector<double> depth(n), mean2d(2 * n), conic(3 * n), cov(3 * n), op(n), rad(n), qr(n);
    std::vector<float> color(3 * n);
    ps_prepared out{index.data(), depth.data(), mean2d.data(), conic.data(), cov.data(), op.data(), color.data(),
                    rad.data(), qr.data()};
    int64_t v = 0;
    ps_counters ctr;
    dev.check(ps_prepare(dev.get(), s.get(), &c, &g, static_cast<int64_t>(n), &out, &v, &ctr));
    PerfCounters pc = from_ps(ctr);
    counters.splats_submitted += pc.splats_submitted;
    counters.splats_frustum_culled += pc.splats_frustum_culled;
    std::vector<ProjectedSplat> res(static_cast<std::size_t>(v));
    const bool aware_mode = cfg.culling_mode != CullingMode::ZeroCrossing;
    for (int64_t k = 0; k < v; ++k) {
        ProjectedSplat& p = res[static_cast<std::size_t>(k)];
        p.mean2d = {mean2d[2 * k], mean2d[2 * k + 1]};
        p.conic = {conic[3 * k], conic[3 * k + 1], conic[3 * k + 2]};
        p.cov_aa = {cov[3 * k], cov[3 * k + 1], cov[3 * k + 2]};
        p.depth = depth[k];
        p.opacity_eff = op[k];
        p.color = {color[3 * k], color[3 * k + 1], color[3 * k + 2]};
        p.bound = {rad[k], qr[k], aware_mode};
        p.index = index[k];
    }
    return res;
}

// Many views of one resident scene (K1 fused over batches of views; each
// view's binning / blend on its own stream). All cameras share width / height.
inline std::vector<std::pair<Framebuffer, PerfCounters>> render_views(const Scene& scene,
                                                                      std::span<const Camera> cams,
                                                                      const RasterConfig& cfg) {
    std::vector<std::pair<Framebuffer, PerfCounters>> out;
    if (cams.empty()) return out;
    std::vector<ps_camera> c(cams.size());
    for (std::size_t k = 0; k < cams.size(); ++k) c[k] = to_ps(cams[k]);
    const ps_config g = to_ps(cfg);
    const std::size_t pix = static_cast<std::size_t>(cams[0].width) * cams[0].height;
    std::vector<float> rgb(3 * pix * cams.size()), tr(pix * cams.size());
    std::vector<ps_counters> ctr(cams.size());
    scene.device().check(ps_render_views(scene.device().get(), scene.get(), c.data(), static_cast<int>(c.size()), &g,
                                         rgb.data(), tr.data(), PS_MEM_HOST, ctr.data()));
    for (std::size_t v = 0; v < cams.size(); ++v) {
        Framebuffer fb(cams[v].width, cams[v].height);
        for (std::size_t k = 0; k < 3 * pix; ++k) fb.rgb[k] = rgb[3 * pix * v + k];
        for (std::size_t k = 0; k < pix; ++k) fb.transmittance[k] = tr[pix * v + k];
        out.emplace_back(std::move(fb), from_ps(ctr[v]));
    }
    return out;
}

// polysplat::compare (metrics.hpp:40-42): both configs rendered and compared
// on the device (composite, psnr, ssim, max_abs_diff; counters; pair ratio).
inline CompareReport compare(std::span<const Splat3D> splats, const Camera& cam, const RasterConfig& cfg_a,
                             const RasterConfig& cfg_b, const Vec3& background = {1.0, 1.0, 1.0},
                             Device& dev = default_device()) {
    Scene s(dev, splats);
    const ps_camera c = to_ps(cam);
    const ps_config ga = to_ps(cfg_a), gb = to_ps(cfg_b);
    const double bg[3] = {background.x, background.y, background.z};
    ps_compare_report r;
    dev.check(ps_compare(dev.get(), s.get(), &c, &ga, &gb, bg, &r));
    if (!r.metrics.ssim_valid) throw TooSmall("ssim needs images at least 11x11");
    CompareReport out;
    out.psnr_db = r.metrics.psnr_db;
    out.ssim = r.metrics.ssim;
    out.max_abs_diff = r.metrics.max_abs_diff;
    out.counters_a = from_ps(r.counters_a);
    out.counters_b = from_ps(r.counters_b);
    out.pair_ratio = r.pair_ratio;
    return out;
}

// psnr / ssim / max_abs_diff of two framebuffers on the device (composite +
// metrics.cpp:34-134), in one pass.
inline ps_image_metrics image_metrics(const Framebuffer& a, const Framebuffer& b,
                                      const Vec3& background = {1.0, 1.0, 1.0}, Device& dev = default_device()) {
    if (a.width != b.width || a.height != b.height) throw DimensionMismatch("image dimensions differ");
    const double bg[3] = {background.x, background.y, background.z};
    ps_image_metrics m;
    dev.check(ps_image_metrics_compute(dev.get(), a.width, a.height, a.rgb.data(), a.transmittance.data(),
                                       b.rgb.data(), b.transmittance.data(), PS_DTYPE_F64, PS_MEM_HOST, bg, &m));
    return m;
}

// polysplat::load_ply (scene_io.hpp:23-27): same fields to the bit, same errors.
inline SceneFile load_ply(const std::string& path) {
    int64_t n = 0;
    int deg = 0;
    int st = ps_ply_info(path.c_str(), &n, &deg);
    if (st != PS_OK) throw_status(st, ps_last_error(nullptr));
    SceneFile sf;
    sf.source_path = path;
    sf.splats.resize(static_cast<std::size_t>(n));
    st = ps_ply_load_splat3d(path.c_str(), reinterpret_cast<double*>(sf.splats.data()), n, &n, &deg);
    if (st != PS_OK) throw_status(st, ps_last_error(nullptr));
    sf.sh_degree = deg;
    return sf;
}

} // namespace polysplat::b200
