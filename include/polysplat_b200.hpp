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
#include "polysplat/projection.hpp"
#include "polysplat/raster.hpp"
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

} // namespace polysplat::b200
