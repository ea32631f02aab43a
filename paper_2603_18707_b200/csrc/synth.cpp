// synth.cpp — deterministic synthetic inputs for the bench and the parity
// tests (harness, not the render path). Draws the same std::mt19937_64
// uniforms, in the same order, as the reference generator
// (scene_io.cpp:304-371), so a scene generated here is the exact
// Splat3D array the reference renders; orbit cameras follow scene_io.cpp:415-441.
// Compiled with -ffp-contract=off so the arithmetic matches the reference build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "polysplat_b200.h"

namespace ps {
extern thread_local std::string g_free_error;
}

namespace {

constexpr double kPi = 3.141592653589793;
constexpr double kSH0 = 0.28209479177387814;

class Rng {
public:
    explicit Rng(uint64_t seed) : gen_(seed) {}
    double uniform() { return double(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double log_uniform(double lo, double hi) { return std::exp(uniform(std::log(lo), std::log(hi))); }
    void rotation(double q[4]) {
        double u1 = uniform(), u2 = uniform(), u3 = uniform();
        double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
        double t2 = 2.0 * kPi * u2, t3 = 2.0 * kPi * u3;
        q[0] = b * std::cos(t3);
        q[1] = a * std::sin(t2);
        q[2] = a * std::cos(t2);
        q[3] = b * std::sin(t3);
    }

private:
    std::mt19937_64 gen_;
};

// One splat in reference Splat3D layout (59 doubles).
struct SplatOut {
    double* p;
    void mean(double x, double y, double z) { p[0] = x; p[1] = y; p[2] = z; }
    void scale(double x, double y, double z) { p[3] = x; p[4] = y; p[5] = z; }
    void rot(const double q[4]) { for (int k = 0; k < 4; ++k) p[6 + k] = q[k]; }
    void identity_rot() { p[6] = 1.0; p[7] = 0.0; p[8] = 0.0; p[9] = 0.0; }
    void opacity(double o) { p[10] = o; }
    void dc(double r, double g, double b) {
        p[11] = (r - 0.5) / kSH0;
        p[12] = (g - 0.5) / kSH0;
        p[13] = (b - 0.5) / kSH0;
    }
    void sh(int k, double x, double y, double z) { p[11 + 3 * k] = x; p[12 + 3 * k] = y; p[13 + 3 * k] = z; }
};

int64_t scene_count(int kind, int64_t n) {
    switch (kind) {
        case 0: return 100;
        case 1: return 5000;
        case 2: return 190;
        case 3:
        case 4: return n;
    }
    return -1;
}

// Writes the scene into `out` (count x 59 doubles, zero-initialised by caller).
void generate(int kind, uint64_t seed, int64_t n, double* out, int* sh_degree) {
    auto at = [&](int64_t i) { return SplatOut{out + i * PS_SPLAT3D_DOUBLES}; };
    if (kind == 0) { // grid (scene_io.cpp:334-352)
        *sh_degree = 0;
        const double spacing = 0.22, sigma = 0.09;
        const double opacities[3] = {0.35, 0.65, 0.95};
        int64_t k = 0;
        for (int i = 0; i < 10; ++i)
            for (int j = 0; j < 10; ++j) {
                SplatOut s = at(k++);
                s.mean((i - 4.5) * spacing, (j - 4.5) * spacing, 0.0);
                s.scale(sigma, sigma, sigma);
                s.identity_rot();
                s.opacity(opacities[(i + j) % 3]);
                s.dc(i / 9.0, j / 9.0, 1.0 - (i + j) / 18.0);
            }
        return;
    }
    if (kind == 2) { // overexposed sky (scene_io.cpp:373-402)
        *sh_degree = 0;
        Rng rng(seed);
        int64_t k = 0;
        for (int i = 0; i < 40; ++i) {
            SplatOut s = at(k++);
            double mx = rng.uniform(-0.6, 0.6);
            double my = rng.uniform(-0.6, 0.6);
            double mz = rng.uniform(0.25, 0.45);
            s.mean(mx, my, mz);
            double sc = rng.uniform(0.35, 0.75);
            s.scale(sc, sc, 0.05);
            s.identity_rot();
            s.opacity(rng.uniform(0.03, 0.12));
            double intensity = rng.uniform(2.6, 3.2);
            double blue = rng.uniform(2.2, 2.8);
            s.dc(intensity, intensity, blue);
        }
        for (int i = 0; i < 150; ++i) {
            SplatOut s = at(k++);
            double mx = rng.uniform(-0.45, 0.45);
            double my = rng.uniform(-0.45, 0.45);
            double mz = rng.uniform(-0.4, 0.0);
            s.mean(mx, my, mz);
            double sx = rng.log_uniform(0.02, 0.06);
            double sy = rng.log_uniform(0.02, 0.06);
            double sz = rng.log_uniform(0.02, 0.06);
            s.scale(sx, sy, sz);
            double q[4];
            rng.rotation(q);
            s.rot(q);
            s.opacity(rng.uniform(0.3, 0.9));
            double r = rng.uniform(), g = rng.uniform(), b = rng.uniform();
            s.dc(r, g, b);
        }
        return;
    }
    // random (scene_io.cpp:354-371) and the parametric G(n, seed) of SURVEY §8d:
    // scales log-U(0.008 k, 0.045 k), k = (5000/n)^(1/3) (k = 1 reproduces the
    // reference's 5000-splat scene); kind 4 skews opacity to 0.005 + 0.99 u^3 (C5).
    *sh_degree = 3;
    Rng rng(seed);
    const double k = (kind == 1) ? 1.0 : std::cbrt(5000.0 / static_cast<double>(n));
    const double lo = 0.008 * k, hi = 0.045 * k;
    for (int64_t i = 0; i < n; ++i) {
        SplatOut s = at(i);
        double mx = rng.uniform(-0.5, 0.5);
        double my = rng.uniform(-0.5, 0.5);
        double mz = rng.uniform(-0.5, 0.5);
        s.mean(mx, my, mz);
        double sx = rng.log_uniform(lo, hi);
        double sy = rng.log_uniform(lo, hi);
        double sz = rng.log_uniform(lo, hi);
        s.scale(sx, sy, sz);
        double q[4];
        rng.rotation(q);
        s.rot(q);
        if (kind == 4) {
            double u = rng.uniform();
            s.opacity(0.005 + 0.99 * u * u * u);
        } else {
            s.opacity(rng.uniform(0.05, 0.995));
        }
        double r = rng.uniform(), g = rng.uniform(), b = rng.uniform();
        s.dc(r, g, b);
        for (int j = 1; j < 16; ++j) {
            double x = rng.uniform(-0.04, 0.04);
            double y = rng.uniform(-0.04, 0.04);
            double z = rng.uniform(-0.04, 0.04);
            s.sh(j, x, y, z);
        }
    }
}

} // namespace

extern "C" {

int ps_synth_scene(int kind, uint64_t seed, int64_t n, double* splats, int64_t capacity, int64_t* n_out,
                   int* sh_degree) {
    const int64_t count = scene_count(kind, n);
    if (count < 0 || (kind >= 3 && n <= 0)) {
        ps::g_free_error = "unknown synthetic scene kind or size";
        return PS_INVALID_ARGUMENT;
    }
    if (n_out) *n_out = count;
    int deg = 0;
    if (!splats) {
        if (sh_degree) *sh_degree = (kind == 0 || kind == 2) ? 0 : 3;
        return PS_OK;
    }
    if (capacity < count) {
        ps::g_free_error = "capacity too small";
        return PS_INVALID_ARGUMENT;
    }
    std::memset(splats, 0, sizeof(double) * PS_SPLAT3D_DOUBLES * static_cast<size_t>(count));
    generate(kind, seed, count, splats, &deg);
    if (sh_degree) *sh_degree = deg;
    return PS_OK;
}

int ps_synth_scene_soa(int kind, uint64_t seed, int64_t n, double* means, double* scales, double* rotations,
                       double* opacities, float* sh) {
    const int64_t count = scene_count(kind, n);
    if (count < 0 || (kind >= 3 && n <= 0)) {
        ps::g_free_error = "unknown synthetic scene kind or size";
        return PS_INVALID_ARGUMENT;
    }
    // the generator draws the whole scene in the reference's order (one
    // mt19937_64 stream), into a full AoS temporary (472 B per splat)
    int deg = 0;
    std::vector<double> tmp(static_cast<size_t>(PS_SPLAT3D_DOUBLES) * count);
    generate(kind, seed, count, tmp.data(), &deg);
    for (int64_t i = 0; i < count; ++i) {
        const double* p = tmp.data() + i * PS_SPLAT3D_DOUBLES;
        for (int k = 0; k < 3; ++k) means[3 * i + k] = p[k];
        for (int k = 0; k < 3; ++k) scales[3 * i + k] = p[3 + k];
        for (int k = 0; k < 4; ++k) rotations[4 * i + k] = p[6 + k];
        opacities[i] = p[10];
        for (int k = 0; k < 48; ++k) sh[48 * i + k] = static_cast<float>(p[11 + k]);
    }
    return PS_OK;
}

int ps_orbit_cameras(int count, int width, int height, double fov_deg, double radius, double elevation,
                     ps_camera* out) {
    if (count < 0 || !out) {
        ps::g_free_error = "bad orbit camera arguments";
        return PS_INVALID_ARGUMENT;
    }
    const double focal = 0.5 * width / std::tan(0.5 * fov_deg * kPi / 180.0);
    for (int i = 0; i < count; ++i) {
        const double theta = 2.0 * kPi * i / std::max(count, 1) - 0.5 * kPi;
        const double pos[3] = {radius * std::cos(theta), elevation, radius * std::sin(theta)};
        // fwd = (0 - pos).normalized()
        double f[3] = {0.0 - pos[0], 0.0 - pos[1], 0.0 - pos[2]};
        double fn = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
        if (fn > 0.0) { f[0] = f[0] / fn; f[1] = f[1] / fn; f[2] = f[2] / fn; }
        else { f[0] = 0.0; f[1] = 0.0; f[2] = 0.0; }
        // right = (0,1,0) x fwd, normalized
        const double up0[3] = {0.0, 1.0, 0.0};
        double r[3] = {up0[1] * f[2] - up0[2] * f[1], up0[2] * f[0] - up0[0] * f[2],
                       up0[0] * f[1] - up0[1] * f[0]};
        double rn = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        if (rn > 0.0) { r[0] = r[0] / rn; r[1] = r[1] / rn; r[2] = r[2] / rn; }
        else { r[0] = 0.0; r[1] = 0.0; r[2] = 0.0; }
        // up = fwd x right
        const double u[3] = {f[1] * r[2] - f[2] * r[1], f[2] * r[0] - f[0] * r[2], f[0] * r[1] - f[1] * r[0]};
        ps_camera c;
        std::memset(&c, 0, sizeof c);
        c.id = i;
        c.width = width;
        c.height = height;
        c.fx = c.fy = focal;
        c.cx = width / 2.0;
        c.cy = height / 2.0;
        for (int k = 0; k < 3; ++k) {
            c.rotation[0 * 3 + k] = r[k];
            c.rotation[1 * 3 + k] = u[k];
            c.rotation[2 * 3 + k] = f[k];
        }
        // translation = (R * pos) * -1
        for (int row = 0; row < 3; ++row) {
            const double* m = c.rotation + 3 * row;
            c.translation[row] = (m[0] * pos[0] + m[1] * pos[1] + m[2] * pos[2]) * -1.0;
        }
        out[i] = c;
    }
    return PS_OK;
}

} // extern "C"
