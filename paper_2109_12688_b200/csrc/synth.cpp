// Seeded synthetic image pairs for the BASELINE.json configs.
// Input generation only (host, not on the registration path).  The paper's cardiac
// MRI set is private; these phantoms stand in with the configs' shapes, intensity
// ranges and displacement magnitudes.  Generated once, fed byte-identically to the
// GPU path and to the CPU reference.
//
// RNG: std::mt19937(seed), U = raw / 2^32 (the reference tests' mapping,
// tests/oracles.hpp:19-27); normals by Box-Muller on (1 - U1, U2).
// Draw order per pair: rng(seed) for the phantom geometry, rng(seed + 1) for the
// three displacement noise volumes, rng(seed + 101) / rng(seed + 202) for the
// fixed / moving image noise.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Rng {
    std::mt19937 g;
    explicit Rng(uint32_t s) : g(s) {}
    double u() { return g() * (1.0 / 4294967296.0); }
    double u(double lo, double hi) { return lo + (hi - lo) * u(); }
    double normal() {
        const double u1 = 1.0 - u(), u2 = u();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    }
};

struct Grid {
    int nx, ny, nz;
    size_t n() const { return (size_t)nx * ny * nz; }
    size_t at(int x, int y, int z) const { return (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z); }
};

// separable Gaussian, radius ceil(3 sigma), normalised, clamp-to-edge, fp64
void gauss(const Grid& g, std::vector<double>& v, double sigma) {
    if (sigma <= 0) return;
    const int r = (int)std::ceil(3.0 * sigma);
    std::vector<double> k(2 * r + 1);
    double s = 0;
    for (int i = -r; i <= r; ++i) s += (k[i + r] = std::exp(-0.5 * i * i / (sigma * sigma)));
    for (auto& x : k) x /= s;
    std::vector<double> tmp(v.size());
    const int dims[3] = {g.nx, g.ny, g.nz};
    const size_t strides[3] = {1, (size_t)g.nx, (size_t)g.nx * g.ny};
    for (int ax = 0; ax < 3; ++ax) {
        const int n = dims[ax];
        const size_t st = strides[ax];
        for (int z = 0; z < g.nz; ++z)
            for (int y = 0; y < g.ny; ++y)
                for (int x = 0; x < g.nx; ++x) {
                    const int pos = ax == 0 ? x : (ax == 1 ? y : z);
                    const size_t i = g.at(x, y, z);
                    const size_t base = i - (size_t)pos * st;
                    double acc = 0;
                    for (int t = -r; t <= r; ++t) {
                        const int q = std::min(std::max(pos + t, 0), n - 1);
                        acc += k[t + r] * v[base + (size_t)q * st];
                    }
                    tmp[i] = acc;
                }
        v.swap(tmp);
    }
}

// clamp-trilinear in fp64 with the reference semantics (volume.cpp:36-76)
double trilinear(const Grid& g, const std::vector<double>& f, double px, double py, double pz) {
    auto ax = [](double c, int n, int& lo, int& hi, double& fr) {
        c = std::clamp(c, 0.0, (double)(n - 1));
        const double fl = std::floor(c);
        lo = (int)fl;
        hi = std::min(lo + 1, n - 1);
        fr = c - fl;
    };
    int x0, x1, y0, y1, z0, z1;
    double fx, fy, fz;
    ax(px, g.nx, x0, x1, fx);
    ax(py, g.ny, y0, y1, fy);
    ax(pz, g.nz, z0, z1, fz);
    const double c00 = f[g.at(x0, y0, z0)] + (f[g.at(x1, y0, z0)] - f[g.at(x0, y0, z0)]) * fx;
    const double c10 = f[g.at(x0, y1, z0)] + (f[g.at(x1, y1, z0)] - f[g.at(x0, y1, z0)]) * fx;
    const double c01 = f[g.at(x0, y0, z1)] + (f[g.at(x1, y0, z1)] - f[g.at(x0, y0, z1)]) * fx;
    const double c11 = f[g.at(x0, y1, z1)] + (f[g.at(x1, y1, z1)] - f[g.at(x0, y1, z1)]) * fx;
    const double c0 = c00 + (c10 - c00) * fy;
    const double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// "smooth random displacement (sigma, max A)": three i.i.d. N(0,1) volumes filtered
// by G_sigma, scaled so max |u| = A.
void smooth_disp(const Grid& g, uint32_t seed, double sigma, double amax, std::vector<double> u[3]) {
    Rng r(seed);
    for (int c = 0; c < 3; ++c) {
        u[c].resize(g.n());
        for (auto& x : u[c]) x = r.normal();
        gauss(g, u[c], sigma);
    }
    double m = 0;
    for (size_t i = 0; i < g.n(); ++i)
        m = std::max(m, std::sqrt(u[0][i] * u[0][i] + u[1][i] * u[1][i] + u[2][i] * u[2][i]));
    const double s = m > 0 ? amax / m : 0.0;
    for (int c = 0; c < 3; ++c)
        for (auto& x : u[c]) x *= s;
}

void warp_into(const Grid& g, const std::vector<double>& img, const std::vector<double> u[3],
               std::vector<double>& out) {
    out.resize(g.n());
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x) {
                const size_t i = g.at(x, y, z);
                out[i] = trilinear(g, img, x + u[0][i], y + u[1][i], z + u[2][i]);
            }
}

void add_noise(std::vector<double>& v, uint32_t seed, double sd) {
    Rng r(seed);
    for (auto& x : v) x += sd * r.normal();
}

void rician(std::vector<double>& v, uint32_t seed, double sd) {
    Rng r(seed);
    for (auto& x : v) {
        const double a = x + sd * r.normal(), b = sd * r.normal();
        x = std::sqrt(a * a + b * b);
    }
}

void store(const std::vector<double>& v, float* out) {
    for (size_t i = 0; i < v.size(); ++i) out[i] = (float)v[i];
}

// config 1: three smoothed ellipsoids + N(0, 0.01); moving by smooth disp (4, 3)
void config1(const Grid& g, uint32_t seed, float* fixed, float* moving) {
    Rng r(seed);
    std::vector<double> f(g.n(), 0.0);
    const int dims[3] = {g.nx, g.ny, g.nz};
    for (int e = 0; e < 3; ++e) {
        double c[3], a[3];
        for (int d = 0; d < 3; ++d) c[d] = r.u(0.3, 0.7) * (dims[d] - 1);
        for (int d = 0; d < 3; ++d) a[d] = r.u(0.12, 0.25) * dims[d];
        const double amp = r.u(0.3, 0.6);
        for (int z = 0; z < g.nz; ++z)
            for (int y = 0; y < g.ny; ++y)
                for (int x = 0; x < g.nx; ++x) {
                    const double q = (x - c[0]) * (x - c[0]) / (a[0] * a[0]) + (y - c[1]) * (y - c[1]) / (a[1] * a[1]) +
                                     (z - c[2]) * (z - c[2]) / (a[2] * a[2]);
                    if (q <= 1.0) f[g.at(x, y, z)] += amp;
                }
    }
    gauss(g, f, 1.5);
    for (auto& x : f) x = std::clamp(x, 0.0, 1.0);
    std::vector<double> u[3], m;
    smooth_disp(g, seed + 1, 4.0, 3.0, u);
    warp_into(g, f, u, m);
    add_noise(f, seed + 101, 0.01);
    add_noise(m, seed + 202, 0.01);
    store(f, fixed);
    store(m, moving);
}

// config 2/3: nested-ellipsoid ventricle, Rician noise; moving by radial contraction
// of the myocardium plus smooth disp (6, 5)
void config2(const Grid& g, uint32_t seed, float* fixed, float* moving) {
    Rng r(seed);
    const double c[3] = {(g.nx - 1) / 2.0 + r.u(-2, 2), (g.ny - 1) / 2.0 + r.u(-2, 2), (g.nz - 1) / 2.0 + r.u(-2, 2)};
    const double a[3] = {0.28 * g.nx * r.u(0.9, 1.1), 0.24 * g.ny * r.u(0.9, 1.1), 0.30 * g.nz * r.u(0.9, 1.1)};
    const double kappa = r.u(0.10, 0.20);
    std::vector<double> f(g.n());
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x) {
                const double dx = (x - c[0]) / a[0], dy = (y - c[1]) / a[1], dz = (z - c[2]) / a[2];
                const double re = std::sqrt(dx * dx + dy * dy + dz * dz);
                f[g.at(x, y, z)] = re <= 0.6 ? 0.9 : (re <= 1.0 ? 0.4 : 0.1);
            }
    gauss(g, f, 1.0);
    std::vector<double> u[3], m;
    smooth_disp(g, seed + 1, 6.0, 5.0, u);
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x) {
                const size_t i = g.at(x, y, z);
                const double d[3] = {x - c[0], y - c[1], z - c[2]};
                const double re2 = (d[0] / a[0]) * (d[0] / a[0]) + (d[1] / a[1]) * (d[1] / a[1]) + (d[2] / a[2]) * (d[2] / a[2]);
                const double w = -kappa * std::exp(-re2 / (2.0 * 1.5 * 1.5));
                for (int k = 0; k < 3; ++k) u[k][i] += w * d[k];
            }
    warp_into(g, f, u, m);
    rician(f, seed + 101, 0.02);
    rician(m, seed + 202, 0.02);
    store(f, fixed);
    store(m, moving);
}

// config 4: six Gaussian blobs; swirl about z through the centre, |u| <= 12
void config4(const Grid& g, uint32_t seed, float* fixed, float* moving) {
    Rng r(seed);
    std::vector<double> f(g.n(), 0.0);
    const int dims[3] = {g.nx, g.ny, g.nz};
    for (int b = 0; b < 6; ++b) {
        double c[3];
        for (int d = 0; d < 3; ++d) c[d] = r.u(0.25, 0.75) * (dims[d] - 1);
        const double s = r.u(0.06, 0.12) * dims[0];
        const double amp = r.u(0.4, 0.8);
        for (int z = 0; z < g.nz; ++z)
            for (int y = 0; y < g.ny; ++y)
                for (int x = 0; x < g.nx; ++x) {
                    const double q = (x - c[0]) * (x - c[0]) + (y - c[1]) * (y - c[1]) + (z - c[2]) * (z - c[2]);
                    f[g.at(x, y, z)] += amp * std::exp(-q / (2 * s * s));
                }
    }
    for (auto& x : f) x = std::clamp(x, 0.0, 1.0);
    const double tmax = r.u(0.7, 1.0) * 30.0 * kPi / 180.0;
    const double cx = (g.nx - 1) / 2.0, cy = (g.ny - 1) / 2.0;
    const double rs = 32.0 * g.nx / 128.0;
    std::vector<double> u[3];
    for (auto& v : u) v.assign(g.n(), 0.0);
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x) {
                const size_t i = g.at(x, y, z);
                const double dx = x - cx, dy = y - cy;
                const double th = tmax * std::exp(-(dx * dx + dy * dy) / (2 * rs * rs));
                double ux = std::cos(th) * dx - std::sin(th) * dy - dx;
                double uy = std::sin(th) * dx + std::cos(th) * dy - dy;
                const double n = std::sqrt(ux * ux + uy * uy);
                if (n > 12.0) {
                    ux *= 12.0 / n;
                    uy *= 12.0 / n;
                }
                u[0][i] = ux;
                u[1][i] = uy;
            }
    std::vector<double> m;
    warp_into(g, f, u, m);
    store(f, fixed);
    store(m, moving);
}

// config 5: smoothed uniform texture rescaled to [0,1]; smooth disp (8, 6), no noise
void config5(const Grid& g, uint32_t seed, float* fixed, float* moving) {
    Rng r(seed);
    std::vector<double> f(g.n());
    for (auto& x : f) x = r.u();
    gauss(g, f, 3.0);
    double lo = 1e300, hi = -1e300;
    for (double x : f) {
        lo = std::min(lo, x);
        hi = std::max(hi, x);
    }
    for (auto& x : f) x = hi > lo ? (x - lo) / (hi - lo) : 0.0;
    std::vector<double> u[3], m;
    smooth_disp(g, seed + 1, 8.0, 6.0, u);
    warp_into(g, f, u, m);
    store(f, fixed);
    store(m, moving);
}

}  // namespace

extern "C" {

// Generates one pair for `config` (1..5; 3 = same phantom as 2) on an (nx, ny, nz)
// x-fastest grid.  Returns 0 on success, 2 on a bad argument.
int dreg_synth_pair(int config, uint32_t seed, int nx, int ny, int nz, float* fixed, float* moving) {
    if (nx < 2 || ny < 2 || nz < 2 || !fixed || !moving) return 2;
    const Grid g{nx, ny, nz};
    switch (config) {
        case 1: config1(g, seed, fixed, moving); return 0;
        case 2:
        case 3: config2(g, seed, fixed, moving); return 0;
        case 4: config4(g, seed, fixed, moving); return 0;
        case 5: config5(g, seed, fixed, moving); return 0;
        default: return 2;
    }
}

// n pairs with seeds seed0 + i, generated on `threads` host threads;
// fixed / moving are [n][voxels].
int dreg_synth_batch(int config, uint32_t seed0, int n, int nx, int ny, int nz, float* fixed, float* moving,
                     int threads) {
    if (n < 0) return 2;
    const size_t N = (size_t)nx * ny * nz;
    threads = std::max(1, std::min(threads, n));
    std::vector<std::thread> pool;
    std::vector<int> rc(threads, 0);
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (int i = t; i < n; i += threads) {
                const int r = dreg_synth_pair(config, seed0 + (uint32_t)i, nx, ny, nz, fixed + i * N, moving + i * N);
                if (r) rc[t] = r;
            }
        });
    for (auto& th : pool) th.join();
    for (int r : rc)
        if (r) return r;
    return 0;
}

}  // extern "C"
