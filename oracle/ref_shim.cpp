// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. extern "C" entry points over the
// UNMODIFIED reference library (polysplat, compiled out of tree from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py's CPU-baseline leg call the reference's own
// polysplat::render / count_pairs / prepare_splats / reference::render_serial
// and its synthetic scene / orbit-camera generators through ctypes.
// This file is original glue; it contains no reference source.

#include "polysplat_b200.h"

#include "polysplat/errors.hpp"
#include "polysplat/kernel.hpp"
#include "polysplat/metrics.hpp"
#include "polysplat/projection.hpp"
#include "polysplat/raster.hpp"
#include "polysplat/reference.hpp"
#include "polysplat/scene_io.hpp"

#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

using namespace polysplat;

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const NonOrthonormalRotation& e) {
        return fail(PS_NON_ORTHONORMAL_ROTATION, e.what());
    } catch (const DegenerateCovariance& e) {
        return fail(PS_DEGENERATE_COVARIANCE, e.what());
    } catch (const NoPositiveRoot& e) {
        return fail(PS_NO_POSITIVE_ROOT, e.what());
    } catch (const EpsilonZeroUnbounded& e) {
        return fail(PS_EPSILON_ZERO_UNBOUNDED, e.what());
    } catch (const FullyCulled& e) {
        return fail(PS_FULLY_CULLED, e.what());
    } catch (const IoError& e) {
        return fail(PS_IO_ERROR, e.what());
    } catch (const MalformedHeader& e) {
        return fail(PS_MALFORMED_HEADER, e.what());
    } catch (const UnsupportedFormat& e) {
        return fail(PS_UNSUPPORTED_FORMAT, e.what());
    } catch (const MissingProperty& e) {
        return fail(PS_MISSING_PROPERTY, e.what());
    } catch (const TruncatedData& e) {
        return fail(PS_TRUNCATED_DATA, e.what());
    } catch (const Error& e) {
        return fail(PS_ERROR, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(PS_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return fail(PS_ERROR, e.what());
    }
}

KernelSpec to_kernel(const ps_kernel& k) {
    KernelSpec s;
    s.kind = static_cast<KernelKind>(k.kind);
    s.order = k.order;
    if (k.kind != PS_KERNEL_EXPONENTIAL) s.coeffs.assign(k.coeffs, k.coeffs + k.order + 1);
    s.first_root = k.first_root;
    return s;
}

ps_kernel from_kernel(const KernelSpec& s) {
    ps_kernel k;
    std::memset(&k, 0, sizeof k);
    k.kind = static_cast<int32_t>(s.kind);
    k.order = s.order;
    for (std::size_t i = 0; i < s.coeffs.size() && i < 4; ++i) k.coeffs[i] = s.coeffs[i];
    k.first_root = s.first_root;
    return k;
}

RasterConfig to_config(const ps_config& c) {
    RasterConfig r;
    r.tile_size = c.tile_size;
    r.epsilon = c.epsilon;
    r.transmittance_floor = c.transmittance_floor;
    r.culling_mode = static_cast<CullingMode>(c.culling_mode);
    r.kernel = to_kernel(c.kernel);
    if (c.has_culling_kernel) r.culling_kernel = to_kernel(c.culling_kernel);
    r.v_dilation = c.v_dilation;
    r.sh_degree = c.sh_degree;
    r.clamp_before_blend = c.clamp_before_blend != 0;
    r.thread_count = c.thread_count;
    return r;
}

Camera to_camera(const ps_camera& c) {
    Camera cam;
    cam.id = c.id;
    cam.width = c.width;
    cam.height = c.height;
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    for (int i = 0; i < 9; ++i) cam.rotation.m[i] = c.rotation[i];
    cam.translation = {c.translation[0], c.translation[1], c.translation[2]};
    return cam;
}

ps_camera from_camera(const Camera& cam) {
    ps_camera c;
    std::memset(&c, 0, sizeof c);
    c.id = cam.id;
    c.width = cam.width;
    c.height = cam.height;
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    for (int i = 0; i < 9; ++i) c.rotation[i] = cam.rotation.m[i];
    c.translation[0] = cam.translation.x;
    c.translation[1] = cam.translation.y;
    c.translation[2] = cam.translation.z;
    return c;
}

static_assert(sizeof(Splat3D) == PS_SPLAT3D_DOUBLES * sizeof(double), "Splat3D layout");

std::span<const Splat3D> as_splats(const double* p, int64_t n) {
    return {reinterpret_cast<const Splat3D*>(p), static_cast<std::size_t>(n)};
}

void put_counters(ps_counters* out, const PerfCounters& c) {
    if (!out) return;
    out->splats_submitted = c.splats_submitted;
    out->splats_frustum_culled = c.splats_frustum_culled;
    out->tile_pairs_coarse = c.tile_pairs_coarse;
    out->tile_pairs_after_tight_test = c.tile_pairs_after_tight_test;
    out->kernel_evaluations = c.kernel_evaluations;
    out->fragments_blended = c.fragments_blended;
}

void put_fb(const Framebuffer& fb, double* rgb, double* trans) {
    if (rgb) std::memcpy(rgb, fb.rgb.data(), fb.rgb.size() * sizeof(double));
    if (trans) std::memcpy(trans, fb.transmittance.data(), fb.transmittance.size() * sizeof(double));
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_splat3d_size(void) { return static_cast<int>(sizeof(Splat3D)); }
int ref_resolve_thread_count(int requested) { return resolve_thread_count(requested); }

int ref_render(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
               double* rgb, double* trans, ps_counters* counters) {
    return guarded([&]() -> int {
        auto [fb, c] = render(as_splats(splats, n), to_camera(*cam), to_config(*cfg));
        put_fb(fb, rgb, trans);
        put_counters(counters, c);
        return PS_OK;
    });
}

int ref_render_serial(const double* splats, int64_t n, const ps_camera* cam,
                      const ps_config* cfg, double* rgb, double* trans) {
    return guarded([&]() -> int {
        Framebuffer fb = reference::render_serial(as_splats(splats, n), to_camera(*cam),
                                                  to_config(*cfg));
        put_fb(fb, rgb, trans);
        return PS_OK;
    });
}

int ref_count_pairs(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                    ps_counters* counters) {
    return guarded([&]() -> int {
        put_counters(counters, count_pairs(as_splats(splats, n), to_camera(*cam), to_config(*cfg)));
        return PS_OK;
    });
}

// prepare_splats (raster.hpp:103-104); color in fp64
int ref_prepare(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                int64_t capacity, uint32_t* index, double* depth, double* mean2d, double* conic,
                double* cov_aa, double* opacity_eff, double* color, double* radius_sigma,
                double* quadric_root, int64_t* n_out, ps_counters* counters) {
    return guarded([&]() -> int {
        PerfCounters c;
        RasterConfig rc = to_config(*cfg);
        std::vector<ProjectedSplat> prep = prepare_splats(as_splats(splats, n), to_camera(*cam), rc, c);
        *n_out = static_cast<int64_t>(prep.size());
        put_counters(counters, c);
        if (static_cast<int64_t>(prep.size()) > capacity) return fail(PS_INVALID_ARGUMENT, "capacity too small");
        for (std::size_t k = 0; k < prep.size(); ++k) {
            const ProjectedSplat& p = prep[k];
            if (index) index[k] = p.index;
            if (depth) depth[k] = p.depth;
            if (mean2d) { mean2d[2 * k] = p.mean2d.x; mean2d[2 * k + 1] = p.mean2d.y; }
            if (conic) { conic[3 * k] = p.conic.xx; conic[3 * k + 1] = p.conic.xy; conic[3 * k + 2] = p.conic.yy; }
            if (cov_aa) { cov_aa[3 * k] = p.cov_aa.xx; cov_aa[3 * k + 1] = p.cov_aa.xy; cov_aa[3 * k + 2] = p.cov_aa.yy; }
            if (opacity_eff) opacity_eff[k] = p.opacity_eff;
            if (color) { color[3 * k] = p.color.x; color[3 * k + 1] = p.color.y; color[3 * k + 2] = p.color.z; }
            if (radius_sigma) radius_sigma[k] = p.bound.radius_sigma;
            if (quadric_root) quadric_root[k] = p.bound.quadric_root;
        }
        return PS_OK;
    });
}

// Per-tile lists rebuilt through the public tile_rect / tight_tile_test /
// tile_pixel_box in the exact loop order of bin_splats (raster.cpp:193-206),
// which is not itself exported. Values are original splat indices.
int ref_tile_lists(const double* splats, int64_t n, const ps_camera* cam, const ps_config* cfg,
                   int64_t capacity, uint32_t* tile_offsets, uint32_t* splat_index,
                   int64_t* n_pairs, ps_counters* counters) {
    return guarded([&]() -> int {
        RasterConfig rc = to_config(*cfg);
        rc.validate();
        Camera c = to_camera(*cam);
        c.validate();
        PerfCounters pc;
        std::vector<ProjectedSplat> prep = prepare_splats(as_splats(splats, n), c, rc, pc);
        int ts = rc.tile_size;
        int tiles_x = (c.width + ts - 1) / ts, tiles_y = (c.height + ts - 1) / ts;
        std::vector<std::vector<uint32_t>> bins(static_cast<std::size_t>(tiles_x) * tiles_y);
        for (const ProjectedSplat& p : prep) {
            auto rect = tile_rect(p, ts, c.width, c.height);
            if (!rect) continue;
            pc.tile_pairs_coarse += rect->count();
            for (int ty = rect->y0; ty <= rect->y1; ++ty)
                for (int tx = rect->x0; tx <= rect->x1; ++tx)
                    if (tight_tile_test(p, tile_pixel_box(tx, ty, ts))) {
                        bins[static_cast<std::size_t>(ty) * tiles_x + tx].push_back(p.index);
                        ++pc.tile_pairs_after_tight_test;
                    }
        }
        uint64_t total = 0;
        for (auto& b : bins) total += b.size();
        *n_pairs = static_cast<int64_t>(total);
        put_counters(counters, pc);
        if (!tile_offsets && !splat_index) return PS_OK; // size query
        if (static_cast<int64_t>(total) > capacity) return fail(PS_INVALID_ARGUMENT, "capacity too small");
        uint32_t off = 0;
        for (std::size_t t = 0; t < bins.size(); ++t) {
            if (tile_offsets) tile_offsets[t] = off;
            if (splat_index) std::memcpy(splat_index + off, bins[t].data(), bins[t].size() * sizeof(uint32_t));
            off += static_cast<uint32_t>(bins[t].size());
        }
        if (tile_offsets) tile_offsets[bins.size()] = off;
        return PS_OK;
    });
}

int ref_synth_scene(int kind, uint64_t seed, double* out, int64_t capacity, int64_t* n_out,
                    int* sh_degree) {
    return guarded([&]() -> int {
        SceneFile s = generate_synthetic_scene(static_cast<SyntheticKind>(kind), seed);
        *n_out = static_cast<int64_t>(s.splats.size());
        if (sh_degree) *sh_degree = s.sh_degree;
        if (out) {
            if (static_cast<int64_t>(s.splats.size()) > capacity) return fail(PS_INVALID_ARGUMENT, "capacity too small");
            std::memcpy(out, s.splats.data(), s.splats.size() * sizeof(Splat3D));
        }
        return PS_OK;
    });
}

// The parametric scene G(n, seed) of SURVEY §8d (kind 3) and its skewed-
// opacity variant (kind 4, C5), written against the reference's Splat3D type
// so the reference arm of bench.py needs no product code: the random-scene
// distribution of scene_io.cpp:354-371 (same mt19937_64 uniform stream, same
// draw order) with scales log-U(0.008 k, 0.045 k), k = (5000/n)^(1/3), and for
// kind 4 opacity = 0.005 + 0.99 u^3. tests/test_oracle.py pins it bit for bit
// against the product's generator (synth.cpp).
int ref_synth_g(int kind, uint64_t seed, int64_t n, double* out, int64_t capacity) {
    return guarded([&]() -> int {
        if ((kind != 3 && kind != 4) || n <= 0) return fail(PS_INVALID_ARGUMENT, "kind must be 3 or 4, n > 0");
        if (capacity < n) return fail(PS_INVALID_ARGUMENT, "capacity too small");
        std::mt19937_64 gen(seed);
        auto uni = [&]() { return double(gen() >> 11) * 0x1.0p-53; };
        auto uab = [&](double a, double b) { return a + (b - a) * uni(); };
        auto logu = [&](double a, double b) { return std::exp(uab(std::log(a), std::log(b))); };
        const double pi = 3.141592653589793, sh0 = 0.28209479177387814;
        const double k = std::cbrt(5000.0 / static_cast<double>(n));
        const double lo = 0.008 * k, hi = 0.045 * k;
        Splat3D* sp = reinterpret_cast<Splat3D*>(out);
        for (int64_t i = 0; i < n; ++i) {
            Splat3D s;
            const double mx = uab(-0.5, 0.5), my = uab(-0.5, 0.5), mz = uab(-0.5, 0.5);
            s.mean = {mx, my, mz};
            const double sx = logu(lo, hi), sy = logu(lo, hi), sz = logu(lo, hi);
            s.scale = {sx, sy, sz};
            const double u1 = uni(), u2 = uni(), u3 = uni();
            const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
            const double t2 = 2.0 * pi * u2, t3 = 2.0 * pi * u3;
            s.rotation = Quat{b * std::cos(t3), a * std::sin(t2), a * std::cos(t2), b * std::sin(t3)};
            if (kind == 4) {
                const double u = uni();
                s.opacity = 0.005 + 0.99 * u * u * u;
            } else {
                s.opacity = uab(0.05, 0.995);
            }
            const double r = uni(), g = uni(), bb = uni();
            s.sh[0] = {(r - 0.5) / sh0, (g - 0.5) / sh0, (bb - 0.5) / sh0};
            for (int j = 1; j < 16; ++j) {
                const double x = uab(-0.04, 0.04), y = uab(-0.04, 0.04), z = uab(-0.04, 0.04);
                s.sh[j] = {x, y, z};
            }
            sp[i] = s;
        }
        return PS_OK;
    });
}

int ref_orbit_cameras(int count, int width, int height, double fov_deg, double radius,
                      double elevation, ps_camera* out) {
    return guarded([&]() -> int {
        auto cams = orbit_cameras(count, width, height, fov_deg, radius, elevation);
        for (std::size_t i = 0; i < cams.size(); ++i) out[i] = from_camera(cams[i]);
        return PS_OK;
    });
}

int ref_fit_polynomial(int order, double epsilon, int iterations, int samples, double step,
                       ps_kernel* out, double* loss) {
    return guarded([&]() -> int {
        FitConfig fc;
        fc.order = order;
        fc.epsilon = epsilon;
        fc.iterations = iterations;
        fc.sample_count = samples;
        fc.step_size = step;
        FitResult r = fit_polynomial(fc);
        *out = from_kernel(r.kernel);
        if (loss) *loss = r.final_l1_loss;
        return PS_OK;
    });
}

int ref_make_polynomial_kernel(int kind, const double* coeffs, int n, ps_kernel* out) {
    return guarded([&]() -> int {
        *out = from_kernel(make_polynomial_kernel(static_cast<KernelKind>(kind),
                                                  std::vector<double>(coeffs, coeffs + n)));
        return PS_OK;
    });
}

int ref_first_positive_root(const double* coeffs, int n, double* out) {
    return guarded([&]() -> int {
        *out = first_positive_root(std::span<const double>(coeffs, static_cast<std::size_t>(n)));
        return PS_OK;
    });
}

int ref_culling_radius(const ps_kernel* k, double o, double eps, double* radius, double* qroot,
                       int* aware) {
    return guarded([&]() -> int {
        CullingBound b = culling_radius(to_kernel(*k), o, eps);
        *radius = b.radius_sigma;
        *qroot = b.quadric_root;
        *aware = b.opacity_aware ? 1 : 0;
        return PS_OK;
    });
}

double ref_eval_kernel(const ps_kernel* k, double x) { return eval_kernel(to_kernel(*k), x); }

int ref_validate_config(const ps_config* cfg) {
    return guarded([&]() -> int { to_config(*cfg).validate(); return PS_OK; });
}

int ref_validate_camera(const ps_camera* cam) {
    return guarded([&]() -> int { to_camera(*cam).validate(); return PS_OK; });
}

// project_splat (projection.cpp:36-79): out14 = mean2d(2) conic(3) cov_aa(3)
// depth opacity_eff color(3) 0; returns 1 visible / 0 near-culled / -status
int ref_project_splat(const double* splat, const ps_camera* cam, double v, int sh_degree,
                      double* out14) {
    int vis = 0;
    int st = guarded([&]() -> int {
        auto p = project_splat(*reinterpret_cast<const Splat3D*>(splat), to_camera(*cam), v, sh_degree);
        if (!p) return PS_OK;
        vis = 1;
        double o[14] = {p->mean2d.x, p->mean2d.y, p->conic.xx, p->conic.xy, p->conic.yy,
                        p->cov_aa.xx, p->cov_aa.xy, p->cov_aa.yy, p->depth, p->opacity_eff,
                        p->color.x, p->color.y, p->color.z, 0.0};
        std::memcpy(out14, o, sizeof o);
        return PS_OK;
    });
    return st == PS_OK ? vis : -st;
}

// tile_rect on a manual ProjectedSplat (KATs of test_raster.cpp:50-70)
int ref_tile_rect(double mx, double my, const double cov_aa[3], double radius_sigma, int tile_size,
                  int width, int height, int* rect4) {
    ProjectedSplat p;
    p.mean2d = {mx, my};
    p.cov_aa = {cov_aa[0], cov_aa[1], cov_aa[2]};
    p.bound.radius_sigma = radius_sigma;
    p.bound.quadric_root = radius_sigma * radius_sigma;
    auto r = tile_rect(p, tile_size, width, height);
    if (!r) return 0;
    rect4[0] = r->x0; rect4[1] = r->y0; rect4[2] = r->x1; rect4[3] = r->y1;
    return 1;
}

double ref_min_quadric_over_box(const double conic[3], double mx, double my, const double box[4]) {
    return min_quadric_over_box(Sym2{conic[0], conic[1], conic[2]}, Vec2{mx, my},
                                PixelBox{box[0], box[1], box[2], box[3]});
}

// load_ply (scene_io.cpp:53-199): Splat3D records; with splats == NULL only n / degree
int ref_load_ply(const char* path, double* splats, int64_t capacity, int64_t* n_out, int* sh_degree) {
    return guarded([&]() -> int {
        SceneFile sf = load_ply(path);
        *n_out = static_cast<int64_t>(sf.splats.size());
        *sh_degree = sf.sh_degree;
        if (splats) {
            if (*n_out > capacity) return fail(PS_INVALID_ARGUMENT, "capacity too small");
            std::memcpy(splats, sf.splats.data(), sizeof(Splat3D) * sf.splats.size());
        }
        return PS_OK;
    });
}

// write_ply (scene_io.cpp:201-238)
int ref_write_ply(const double* splats, int64_t n, int sh_degree, const char* path) {
    return guarded([&]() -> int {
        SceneFile sf;
        sf.splats.assign(reinterpret_cast<const Splat3D*>(splats), reinterpret_cast<const Splat3D*>(splats) + n);
        sf.sh_degree = sh_degree;
        write_ply(sf, path);
        return PS_OK;
    });
}

// composite + psnr / max_abs_diff / ssim (metrics.cpp:13-134), background (bg[3]); ssim_out may be NULL
int ref_compare_images(int w, int h, const double* rgb_a, const double* t_a, const double* rgb_b,
                       const double* t_b, const double* bg, double* psnr_db, double* max_abs, double* ssim_out) {
    return guarded([&]() -> int {
        Framebuffer a(w, h), b(w, h);
        std::memcpy(a.rgb.data(), rgb_a, a.rgb.size() * sizeof(double));
        std::memcpy(a.transmittance.data(), t_a, a.transmittance.size() * sizeof(double));
        std::memcpy(b.rgb.data(), rgb_b, b.rgb.size() * sizeof(double));
        std::memcpy(b.transmittance.data(), t_b, b.transmittance.size() * sizeof(double));
        Vec3 background{bg[0], bg[1], bg[2]};
        Image ia = composite(a, background), ib = composite(b, background);
        *psnr_db = psnr(ia, ib);
        *max_abs = max_abs_diff(ia, ib);
        if (ssim_out) *ssim_out = ssim(ia, ib); // throws TooSmall below 11x11
        return PS_OK;
    });
}

} // extern "C"
