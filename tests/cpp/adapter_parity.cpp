// Drop-in parity harness (test infrastructure): the reference's own API
// (polysplat::render / count_pairs / prepare_splats from the UNMODIFIED
// reference library, oracle/_ref) against polysplat::b200 (the adapter in
// include/polysplat_b200.hpp over the C ABI), on the reference's synthetic
// scenes, with the reference's own types. Exit code 0 = all checks pass.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "polysplat/kernel.hpp"
#include "polysplat/metrics.hpp"
#include "polysplat/raster.hpp"
#include "polysplat/scene_io.hpp"
#include "polysplat_b200.hpp"

using namespace polysplat;

static int failures = 0;
static void check(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}

int main() {
    const KernelSpec poly1 = make_polynomial_kernel(KernelKind::PolynomialRelu, {0.773, -0.176});
    struct Cell { const char* name; KernelSpec k; CullingMode m; };
    const Cell cells[] = {{"exp/stp", make_exponential_kernel(), CullingMode::StopThePop},
                          {"poly1/zero", poly1, CullingMode::ZeroCrossing},
                          {"poly1/opacity", poly1, CullingMode::OpacityAware}};
    const SceneFile scenes[] = {generate_synthetic_scene(SyntheticKind::Grid, 1),
                                generate_synthetic_scene(SyntheticKind::Random, 3),
                                generate_synthetic_scene(SyntheticKind::OverexposedSky, 5)};
    const Camera cams[] = {orbit_cameras(3, 96, 80)[1], orbit_cameras(1, 256, 192)[0], orbit_cameras(3, 96, 80)[1]};
    char buf[256];
    for (int si = 0; si < 3; ++si) {
        for (const Cell& c : cells) {
            RasterConfig cfg;
            cfg.kernel = c.k;
            cfg.culling_mode = c.m;
            cfg.sh_degree = scenes[si].sh_degree;
            auto [fr, cr] = polysplat::render(scenes[si].splats, cams[si], cfg);
            auto [fg, cg] = polysplat::b200::render(scenes[si].splats, cams[si], cfg);
            double err = 0.0;
            for (std::size_t k = 0; k < fr.rgb.size(); ++k) err = std::fmax(err, std::fabs(fr.rgb[k] - fg.rgb[k]));
            for (std::size_t k = 0; k < fr.transmittance.size(); ++k)
                err = std::fmax(err, std::fabs(fr.transmittance[k] - fg.transmittance[k]));
            std::snprintf(buf, sizeof buf, "render scene %d %s: max|d| %.2e", si, c.name, err);
            check(err <= 1e-5, buf);
            const bool same = cr.splats_submitted == cg.splats_submitted &&
                              cr.splats_frustum_culled == cg.splats_frustum_culled &&
                              cr.tile_pairs_coarse == cg.tile_pairs_coarse &&
                              cr.tile_pairs_after_tight_test == cg.tile_pairs_after_tight_test &&
                              cr.kernel_evaluations == cg.kernel_evaluations &&
                              cr.fragments_blended == cg.fragments_blended;
            std::snprintf(buf, sizeof buf, "counters scene %d %s", si, c.name);
            check(same, buf);
            PerfCounters pr, pg;
            auto a = polysplat::prepare_splats(scenes[si].splats, cams[si], cfg, pr);
            auto b = polysplat::b200::prepare_splats(scenes[si].splats, cams[si], cfg, pg);
            bool eq = a.size() == b.size();
            for (std::size_t k = 0; eq && k < a.size(); ++k)
                eq = a[k].index == b[k].index && a[k].depth == b[k].depth && a[k].mean2d.x == b[k].mean2d.x &&
                     a[k].mean2d.y == b[k].mean2d.y && a[k].conic.xx == b[k].conic.xx &&
                     a[k].conic.xy == b[k].conic.xy && a[k].conic.yy == b[k].conic.yy &&
                     a[k].opacity_eff == b[k].opacity_eff &&
                     std::fabs(a[k].bound.quadric_root - b[k].bound.quadric_root) <= 1e-13 * a[k].bound.quadric_root;
            std::snprintf(buf, sizeof buf, "prepare_splats scene %d %s (%zu)", si, c.name, a.size());
            check(eq, buf);
        }
    }
    // compare (metrics.cpp:138-157): same counters; quality within the 1e-5 image tolerance
    {
        RasterConfig ca, cb;
        ca.sh_degree = cb.sh_degree = scenes[1].sh_degree;
        cb.kernel = poly1;
        cb.culling_mode = CullingMode::OpacityAware;
        CompareReport r = polysplat::compare(scenes[1].splats, cams[1], ca, cb);
        CompareReport g = polysplat::b200::compare(scenes[1].splats, cams[1], ca, cb);
        const bool ok = r.counters_b.tile_pairs_after_tight_test == g.counters_b.tile_pairs_after_tight_test &&
                        r.pair_ratio == g.pair_ratio && std::fabs(r.psnr_db - g.psnr_db) < 1e-2 &&
                        std::fabs(r.ssim - g.ssim) < 1e-4 && std::fabs(r.max_abs_diff - g.max_abs_diff) <= 2e-5;
        std::snprintf(buf, sizeof buf, "compare: psnr %.6f vs %.6f, ssim %.6f vs %.6f", r.psnr_db, g.psnr_db, r.ssim,
                      g.ssim);
        check(ok, buf);
    }
    // load_ply (scene_io.cpp:53-199): the reference's writer, both loaders, bitwise
    {
        const char* path = "/tmp/adapter_parity.ply";
        write_ply(scenes[1], path);
        SceneFile a = polysplat::load_ply(path), b = polysplat::b200::load_ply(path);
        const bool ok = a.sh_degree == b.sh_degree && a.splats.size() == b.splats.size() &&
                        std::memcmp(a.splats.data(), b.splats.data(), sizeof(Splat3D) * a.splats.size()) == 0;
        check(ok, "load_ply bitwise");
        try {
            polysplat::b200::load_ply("/nonexistent/x.ply");
            check(false, "missing file throws IoError");
        } catch (const IoError&) {
            check(true, "missing file throws IoError");
        }
    }
    // error convention: invalid config -> std::invalid_argument
    try {
        RasterConfig bad;
        bad.tile_size = 0;
        polysplat::b200::render(scenes[0].splats, cams[0], bad);
        check(false, "invalid config throws std::invalid_argument");
    } catch (const std::invalid_argument&) {
        check(true, "invalid config throws std::invalid_argument");
    }
    try {
        Camera bad = cams[0];
        bad.rotation.m[0] = 2.0;
        polysplat::b200::render(scenes[0].splats, bad, RasterConfig{});
        check(false, "non-orthonormal camera throws NonOrthonormalRotation");
    } catch (const NonOrthonormalRotation&) {
        check(true, "non-orthonormal camera throws NonOrthonormalRotation");
    }
    std::printf("%d failures\n", failures);
    return failures ? 1 : 0;
}
