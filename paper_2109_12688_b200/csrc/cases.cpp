// The reference's synthetic registration cases (synth.hpp / synth.cpp), restated for
// the `dreg synth` subcommand of the CLI drop-in (tools/dreg.cpp:207-226).  Host-side
// input generation, not on the registration path.  Built with -ffp-contract=off so
// every value is the reference's fp64 expression rounded the same way, and the
// outputs are byte-identical to the reference's (tests/test_cli.py pins this).
//
// Uniform draws: std::mt19937 raw / 2^32 (synth.cpp:15-25); lo + (hi - lo) * u.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "dreg_synth.h"

namespace {

struct P3 {
    double x, y, z;
};
P3 operator+(P3 a, P3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
P3 operator-(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double sq(P3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }  // Vec3::dot order (volume.hpp:46)
double len(P3 a) { return std::sqrt(sq(a)); }

struct Draw {
    std::mt19937 g;
    explicit Draw(uint32_t s) : g(s) {}
    double u() { return g() * (1.0 / 4294967296.0); }
    double u(double lo, double hi) { return lo + (hi - lo) * u(); }
};

struct Grid {
    int nx, ny, nz;
    int min_extent() const { return std::min(nx, std::min(ny, nz)); }
    P3 centre() const { return {0.5 * (nx - 1), 0.5 * (ny - 1), 0.5 * (nz - 1)}; }
};

double bump(P3 p, P3 c, double sigma) { return std::exp(-sq(p - c) / (2.0 * sigma * sigma)); }

// synth.cpp:40-108: coarse lattice (max(2, n/8) per axis) of uniform vectors in
// [-amp, amp], trilinearly interpolated at fine positions.
class Lattice {
  public:
    Lattice(const Grid& g, uint32_t seed, double amp) : g_(g) {
        c_[0] = std::max(2, g.nx / 8);
        c_[1] = std::max(2, g.ny / 8);
        c_[2] = std::max(2, g.nz / 8);
        vals_.resize(3 * (size_t)c_[0] * c_[1] * c_[2]);
        Draw r(seed);
        for (double& v : vals_) v = r.u(-amp, amp);
    }
    P3 at(P3 p) const {
        const double gx = map(p.x, g_.nx, c_[0]), gy = map(p.y, g_.ny, c_[1]), gz = map(p.z, g_.nz, c_[2]);
        return {lerp3(gx, gy, gz, 0), lerp3(gx, gy, gz, 1), lerp3(gx, gy, gz, 2)};
    }

  private:
    static double map(double x, int fine, int coarse) {
        if (fine <= 1) return 0.0;
        return std::clamp(x, 0.0, fine - 1.0) * (coarse - 1.0) / (fine - 1.0);
    }
    double v(int x, int y, int z, int c) const {
        return vals_[3 * ((size_t)x + (size_t)c_[0] * ((size_t)y + (size_t)c_[1] * (size_t)z)) + (size_t)c];
    }
    double lerp3(double gx, double gy, double gz, int c) const {
        const int x0 = std::min((int)gx, c_[0] - 1), y0 = std::min((int)gy, c_[1] - 1),
                  z0 = std::min((int)gz, c_[2] - 1);
        const int x1 = std::min(x0 + 1, c_[0] - 1), y1 = std::min(y0 + 1, c_[1] - 1), z1 = std::min(z0 + 1, c_[2] - 1);
        const double fx = gx - x0, fy = gy - y0, fz = gz - z0;
        const double a00 = v(x0, y0, z0, c) + (v(x1, y0, z0, c) - v(x0, y0, z0, c)) * fx;
        const double a10 = v(x0, y1, z0, c) + (v(x1, y1, z0, c) - v(x0, y1, z0, c)) * fx;
        const double a01 = v(x0, y0, z1, c) + (v(x1, y0, z1, c) - v(x0, y0, z1, c)) * fx;
        const double a11 = v(x0, y1, z1, c) + (v(x1, y1, z1, c) - v(x0, y1, z1, c)) * fx;
        const double b0 = a00 + (a10 - a00) * fy;
        const double b1 = a01 + (a11 - a01) * fy;
        return b0 + (b1 - b0) * fz;
    }
    Grid g_;
    int c_[3];
    std::vector<double> vals_;
};

// synth.cpp:110-127: evaluate the four volumes voxel by voxel, x fastest.
template <class I, class L>
void fill(const Grid& g, I&& intensity, L&& label, float* t, float* s, uint16_t* tl, uint16_t* sl) {
    size_t i = 0;
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x, ++i) {
                const P3 p{(double)x, (double)y, (double)z};
                t[i] = (float)intensity(p, false);
                s[i] = (float)intensity(p, true);
                if (tl) tl[i] = label(p, false);
                if (sl) sl[i] = label(p, true);
            }
}

// synth.cpp:131-145: Gaussian blob; the source is the target sampled at x + shift,
// labels = the half-maximum ball.
void translate_case(const Grid& g, P3 shift, float* t, float* s, uint16_t* tl, uint16_t* sl) {
    const P3 c = g.centre();
    const double sigma = std::max(2.0, g.min_extent() * 6.0 / 64.0);
    const double radius = sigma * std::sqrt(2.0 * std::log(2.0));
    fill(
        g, [&](P3 p, bool src) { return bump(src ? p + shift : p, c, sigma); },
        [&](P3 p, bool src) -> uint16_t { return len((src ? p + shift : p) - c) <= radius ? 1 : 0; }, t, s, tl, sl);
}

// synth.cpp:147-169: logistic-edged sphere (target) vs ellipsoid (source).
void sphere_ellipsoid_case(const Grid& g, float* t, float* s, uint16_t* tl, uint16_t* sl) {
    const P3 c = g.centre();
    const double r = 0.22 * g.min_extent();
    const P3 sphere{r, r, r}, ellipsoid{1.25 * r, 0.8 * r, 1.05 * r};
    const double edge = 1.5;
    auto level = [&](P3 p, P3 ax) {
        const P3 d = p - c;
        return std::sqrt((d.x / ax.x) * (d.x / ax.x) + (d.y / ax.y) * (d.y / ax.y) + (d.z / ax.z) * (d.z / ax.z));
    };
    fill(
        g,
        [&](P3 p, bool src) {
            const double depth = (1.0 - level(p, src ? ellipsoid : sphere)) * r;
            return 1.0 / (1.0 + std::exp(-depth / edge));
        },
        [&](P3 p, bool src) -> uint16_t { return level(p, src ? ellipsoid : sphere) <= 1.0 ? 1 : 0; }, t, s, tl, sl);
}

// synth.cpp:171-210: three seeded blobs; the source is sampled through a smooth
// lattice displacement (amplitude min(1.5, extent / 16)).
void random_smooth_case(const Grid& g, uint32_t seed, float* t, float* s, uint16_t* tl, uint16_t* sl) {
    Draw r(seed);
    const double extent = g.min_extent();
    struct Blob {
        P3 c;
        double sigma, amp;
    } blobs[3];
    for (Blob& b : blobs) {
        const double cx = r.u(0.3, 0.7) * (g.nx - 1);
        const double cy = r.u(0.3, 0.7) * (g.ny - 1);
        const double cz = r.u(0.3, 0.7) * (g.nz - 1);
        b.c = {cx, cy, cz};
        b.sigma = r.u(0.08, 0.14) * extent;
        b.amp = r.u(0.5, 1.0);
    }
    const Lattice warp(g, seed + 1, std::min(1.5, extent / 16.0));
    auto base = [&](P3 p) {
        double v = 0.0;
        for (const Blob& b : blobs) v += b.amp * bump(p, b.c, b.sigma);
        return std::min(v, 1.0);
    };
    auto inside = [&](P3 p) -> uint16_t {
        for (const Blob& b : blobs)
            if (len(p - b.c) <= b.sigma * std::sqrt(2.0 * std::log(2.0))) return 1;
        return 0;
    };
    fill(
        g, [&](P3 p, bool src) { return src ? base(p + warp.at(p)) : base(p); },
        [&](P3 p, bool src) -> uint16_t { return src ? inside(p + warp.at(p)) : inside(p); }, t, s, tl, sl);
}

}  // namespace

extern "C" {

int dreg_synth_case(int kind, int nx, int ny, int nz, const double* shift, uint32_t seed, float* target,
                    float* source, uint16_t* target_labels, uint16_t* source_labels) {
    if (nx < 1 || ny < 1 || nz < 1 || !target || !source) return 2;
    const Grid g{nx, ny, nz};
    switch (kind) {
        case DREG_CASE_TRANSLATE: {
            const P3 sh = shift ? P3{shift[0], shift[1], shift[2]} : P3{3.0, 0.0, 0.0};
            translate_case(g, sh, target, source, target_labels, source_labels);
            return 0;
        }
        case DREG_CASE_SPHERE_ELLIPSOID: sphere_ellipsoid_case(g, target, source, target_labels, source_labels); return 0;
        case DREG_CASE_RANDOM_SMOOTH: random_smooth_case(g, seed, target, source, target_labels, source_labels); return 0;
        default: return 2;
    }
}

// synth.cpp:212-219: each voxel with probability `fraction` becomes 0 or 1.
int dreg_synth_salt_pepper(float* vol, size_t voxels, double fraction, uint32_t seed) {
    if (!vol) return 2;
    Draw r(seed);
    for (size_t i = 0; i < voxels; ++i)
        if (r.u() < fraction) vol[i] = r.u() < 0.5 ? 0.0f : 1.0f;
    return 0;
}

}  // extern "C"
