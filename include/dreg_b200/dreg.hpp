// dreg_b200/dreg.hpp -- header-only C++ drop-in for the reference `dreg` hot path.
//
// Same namespace, type names, fields, defaults and function signatures as the
// reference headers (proj/core/include/dreg/{volume,admm,regularizer,registration,
// metrics,errors}.hpp); every numerical call is forwarded to the sm_100a library
// through the C ABI (include/dreg_cuda.h) and its status codes are rethrown as the
// reference's exceptions (std::invalid_argument, dreg::numeric_error,
// std::runtime_error).  Switching a reference user over is:
//     #include "dreg/registration.hpp"   ->  #include "dreg_b200/dreg.hpp"
//     -ldreg                             ->  -ldreg_cuda
// Each host thread gets its own device context on dreg::cuda_device() (default 0).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "dreg_cuda.h"

namespace dreg {

// ---- errors.hpp ------------------------------------------------------------------
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- volume.hpp ------------------------------------------------------------------
struct Dims3 {
    int x = 0;
    int y = 0;
    int z = 0;
    [[nodiscard]] std::size_t voxels() const {
        return static_cast<std::size_t>(x) * static_cast<std::size_t>(y) * static_cast<std::size_t>(z);
    }
    friend bool operator==(const Dims3& a, const Dims3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
};

struct Spacing3 {
    double x = 1.0;
    double y = 1.0;
    double z = 1.0;
    friend bool operator==(const Spacing3& a, const Spacing3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
    friend bool operator!=(const Spacing3& a, const Spacing3& b) { return !(a == b); }
};

// volume.hpp:32-49: fp64 3-vector with the reference's operators (value type; host math)
struct Vec3 {
    double x = 0.0;
    double y = 0.0;
    double z = 0.0;

    Vec3& operator+=(const Vec3& o) {
        x += o.x;
        y += o.y;
        z += o.z;
        return *this;
    }
    Vec3& operator-=(const Vec3& o) {
        x -= o.x;
        y -= o.y;
        z -= o.z;
        return *this;
    }
    Vec3& operator*=(double s) {
        x *= s;
        y *= s;
        z *= s;
        return *this;
    }
    friend Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
    friend Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
    friend Vec3 operator*(Vec3 a, double s) { return a *= s; }
    friend Vec3 operator*(double s, Vec3 a) { return a *= s; }
    [[nodiscard]] double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
    [[nodiscard]] double squared_norm() const { return dot(*this); }
    [[nodiscard]] double norm() const { return std::sqrt(squared_norm()); }
};

namespace b200_detail {
// volume.cpp:15-22 (check_geometry)
inline void check_geometry(const Dims3& d, const Spacing3& s) {
    if (d.x < 1 || d.y < 1 || d.z < 1) throw std::invalid_argument("volume dims must be positive");
    if (!(s.x > 0.0) || !(s.y > 0.0) || !(s.z > 0.0)) throw std::invalid_argument("voxel spacing must be positive");
}
}  // namespace b200_detail

struct ScalarVolume {
    Dims3 dims;
    Spacing3 spacing;
    std::vector<float> data;
    ScalarVolume() = default;
    ScalarVolume(Dims3 d, Spacing3 s, float fill = 0.0f) : dims(d), spacing(s) {
        b200_detail::check_geometry(d, s);
        data.assign(d.voxels(), fill);
    }
    [[nodiscard]] std::size_t index(int x, int y, int z) const {
        return static_cast<std::size_t>(x) + static_cast<std::size_t>(dims.x) *
                                                 (static_cast<std::size_t>(y) + static_cast<std::size_t>(dims.y) *
                                                                                    static_cast<std::size_t>(z));
    }
    [[nodiscard]] float at(int x, int y, int z) const { return data[index(x, y, z)]; }
    float& at(int x, int y, int z) { return data[index(x, y, z)]; }
};

struct VectorField {
    Dims3 dims;
    Spacing3 spacing;
    std::vector<float> data;  // 3 * voxels, interleaved (vx, vy, vz)
    VectorField() = default;
    VectorField(Dims3 d, Spacing3 s) : dims(d), spacing(s) {
        b200_detail::check_geometry(d, s);
        data.assign(3 * d.voxels(), 0.0f);
    }
    [[nodiscard]] std::size_t index(int x, int y, int z) const {
        return static_cast<std::size_t>(x) + static_cast<std::size_t>(dims.x) *
                                                 (static_cast<std::size_t>(y) + static_cast<std::size_t>(dims.y) *
                                                                                    static_cast<std::size_t>(z));
    }
    [[nodiscard]] Vec3 get(std::size_t v) const { return {data[3 * v], data[3 * v + 1], data[3 * v + 2]}; }
    void set(std::size_t v, const Vec3& val) {
        data[3 * v] = static_cast<float>(val.x);
        data[3 * v + 1] = static_cast<float>(val.y);
        data[3 * v + 2] = static_cast<float>(val.z);
    }
    [[nodiscard]] Vec3 at(int x, int y, int z) const { return get(index(x, y, z)); }
};

struct DeformationField {
    VectorField disp;
    static DeformationField identity(Dims3 d, Spacing3 s) { return {VectorField(d, s)}; }
};

inline DeformationField make_deformation(VectorField v) { return {std::move(v)}; }

inline bool all_finite(const ScalarVolume& v) {
    for (float x : v.data)
        if (!std::isfinite(x)) return false;
    return true;
}
inline bool all_finite(const VectorField& v) {
    for (float x : v.data)
        if (!std::isfinite(x)) return false;
    return true;
}

// ---- admm.hpp ----------------------------------------------------------------------
struct SolverConfig {
    int data_term = 1;
    int order = 2;
    double lambda = 0.0;
    double theta = 0.1;
    double epsilon = 1e-6;
    int max_iters = 100;
    double tol = 0.0;
    bool accelerate = true;
    bool log_objective = true;
};

struct SolverDiagnostics {
    int iterations = 0;
    double final_change = 0.0;
    bool converged = false;
    std::vector<double> objective;
    std::vector<double> constraint_residual;
};

struct SolveResult {
    VectorField velocity;
    SolverDiagnostics diagnostics;
};

// ---- regularizer.hpp ---------------------------------------------------------------
struct SpectralKernel {
    int order = 0;
    Dims3 dims;
    std::vector<double> values;
    [[nodiscard]] double at(int p, int q, int r) const {
        return values[static_cast<std::size_t>(p) +
                      static_cast<std::size_t>(dims.x) *
                          (static_cast<std::size_t>(q) + static_cast<std::size_t>(dims.y) * static_cast<std::size_t>(r))];
    }
};

// ---- registration.hpp --------------------------------------------------------------
enum class Profile { capped, converged };

struct RegistrationConfig {
    SolverConfig solver;
    int levels = 3;
    std::vector<int> max_warps_per_level;
    std::vector<int> max_admm_iters_per_level;
    double warp_improvement_threshold = 0.02;
    Profile profile = Profile::capped;
    bool smooth_levels = true;
};

struct LevelLog {
    Dims3 dims;
    int warps = 0;
    std::vector<double> mean_sad;
    std::vector<int> solver_iterations;
};

struct RegistrationResult {
    DeformationField phi;
    ScalarVolume warped;
    int velocity_count = 0;
    std::vector<LevelLog> per_level;
    double elapsed_seconds = 0.0;
};

// ---- metrics.hpp -------------------------------------------------------------------
struct JacobianStats {
    double pct_nonpositive = 0.0;
    double min_det = 0.0;
};

/// Integer segmentation labels, x-fastest, 0 = background (metrics.hpp:12-29).
struct LabelVolume {
    Dims3 dims;
    Spacing3 spacing;
    std::vector<std::uint16_t> labels;
    LabelVolume() = default;
    LabelVolume(Dims3 d, Spacing3 s, std::uint16_t fill = 0) : dims(d), spacing(s) {
        if (d.x < 1 || d.y < 1 || d.z < 1) throw std::invalid_argument("label volume dims must be positive");
        if (!(s.x > 0.0) || !(s.y > 0.0) || !(s.z > 0.0))
            throw std::invalid_argument("label volume spacing must be positive");
        labels.assign(d.voxels(), fill);
    }
    [[nodiscard]] std::size_t index(int x, int y, int z) const {
        return static_cast<std::size_t>(x) + static_cast<std::size_t>(dims.x) *
                                                 (static_cast<std::size_t>(y) + static_cast<std::size_t>(dims.y) *
                                                                                    static_cast<std::size_t>(z));
    }
    [[nodiscard]] std::uint16_t at(int x, int y, int z) const { return labels[index(x, y, z)]; }
    std::uint16_t& at(int x, int y, int z) { return labels[index(x, y, z)]; }
};

// ---- io.hpp --------------------------------------------------------------------------
enum class VolumeKind : std::uint8_t { scalar = 0, vector = 1, label = 2 };
using AnyVolume = std::variant<ScalarVolume, VectorField, LabelVolume>;

struct ReportConfig {
    std::string data_term;
    int order = 0;
    double lambda = 0.0;
    double theta = 0.0;
    int levels = 0;
    std::string profile;
    double tol = 0.0;
    double warp_improvement_threshold = 0.0;
    double epsilon = 0.0;
    int threads = 1;
};

struct RunReport {
    std::map<int, double> dice;
    std::map<int, double> hausdorff_mm;
    double jacobian_pct_nonpositive = 0.0;
    double runtime_seconds = 0.0;
    int velocity_count = 0;
    ReportConfig config;
};

// ---- parallel.hpp ---------------------------------------------------------------------
// The reference's CPU worker count.  The GPU path's results never depend on it; it is
// kept so callers (and the run report's config echo) see the value they set.
inline int& b200_thread_slot() {
    static int n = 1;
    return n;
}
inline void set_thread_count(int n) {
    if (n < 1) throw std::invalid_argument("thread count must be >= 1");
    b200_thread_slot() = n;
}
inline int thread_count() { return b200_thread_slot(); }

// =================================== implementation ==================================
namespace b200_detail {

struct Ctx {
    dreg_cuda_ctx* h = nullptr;
    explicit Ctx(int dev) {
        const int st = dreg_cuda_ctx_create(dev, &h);
        if (st != DREG_OK) throw std::runtime_error("dreg_cuda_ctx_create failed (no sm_100 device?)");
    }
    ~Ctx() { dreg_cuda_ctx_destroy(h); }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
};

inline int& device_slot() {
    static int d = 0;
    return d;
}

inline dreg_cuda_ctx* ctx() {
    thread_local std::unique_ptr<Ctx> c;
    thread_local int dev = -1;
    if (!c || dev != device_slot()) {
        c.reset();
        c = std::make_unique<Ctx>(device_slot());
        dev = device_slot();
    }
    return c->h;
}

inline void check(int st) {
    if (st == DREG_OK) return;
    const std::string msg = dreg_cuda_last_error(ctx());
    if (st == DREG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == DREG_NUMERIC) throw numeric_error(msg);
    throw std::runtime_error(msg);
}

inline dreg_dims3 D(Dims3 d) { return {d.x, d.y, d.z}; }

inline dreg_solver_cfg S(const SolverConfig& s) {
    dreg_solver_cfg c;
    c.data_term = s.data_term;
    c.order = s.order;
    c.lambda = s.lambda;
    c.theta = s.theta;
    c.epsilon = s.epsilon;
    c.max_iters = s.max_iters;
    c.tol = s.tol;
    c.accelerate = s.accelerate ? 1 : 0;
    c.log_objective = s.log_objective ? 1 : 0;
    return c;
}

inline void same(Dims3 a, Dims3 b, const char* what) {
    if (!(a == b)) throw std::invalid_argument(std::string(what) + ": dimension mismatch");
}

}  // namespace b200_detail

/// Device used by this thread's implicit context (default 0).
inline void set_cuda_device(int device) { b200_detail::device_slot() = device; }
inline int cuda_device() { return b200_detail::device_slot(); }

inline void validate(const SolverConfig& cfg) {
    const dreg_solver_cfg c = b200_detail::S(cfg);
    if (dreg_validate_solver_cfg(&c) != DREG_OK) {
        if (cfg.data_term != 1 && cfg.data_term != 2) throw std::invalid_argument("solver: data term exponent must be 1 or 2");
        if (cfg.order < 1 || cfg.order > 6) throw std::invalid_argument("solver: regulariser order must be in [1, 6]");
        if (!(cfg.lambda >= 0.0)) throw std::invalid_argument("solver: lambda must be >= 0");
        if (!(cfg.theta > 0.0)) throw std::invalid_argument("solver: theta must be > 0");
        if (!(cfg.epsilon > 0.0)) throw std::invalid_argument("solver: epsilon must be > 0");
        if (cfg.max_iters < 1) throw std::invalid_argument("solver: max_iters must be >= 1");
        throw std::invalid_argument("solver: tol must be >= 0");
    }
}

inline double nesterov_next_alpha(double alpha) { return dreg_nesterov_next_alpha(alpha); }

inline SpectralKernel laplacian_symbol(int n, Dims3 dims) {
    SpectralKernel k{n, dims, std::vector<double>(dims.voxels())};
    if (dreg_laplacian_symbol(n, b200_detail::D(dims), k.values.data()) != DREG_OK)
        throw std::invalid_argument("laplacian_symbol: order must be in [1, 6] and every axis >= 2");
    return k;
}

inline double regulariser_energy(const VectorField& w, int n) {
    double e = 0.0;
    b200_detail::check(dreg_cuda_regulariser_energy(b200_detail::ctx(), w.data.data(), b200_detail::D(w.dims), n, &e));
    return e;
}

inline VectorField v_update_l1(const ScalarVolume& target, const ScalarVolume& warped_source, const VectorField& grad,
                               const VectorField& w_hat, const VectorField& b_hat, const SolverConfig& cfg) {
    b200_detail::same(target.dims, warped_source.dims, "v_update_l1");
    b200_detail::same(target.dims, grad.dims, "v_update_l1");
    b200_detail::same(target.dims, w_hat.dims, "v_update_l1");
    b200_detail::same(target.dims, b_hat.dims, "v_update_l1");
    SolverConfig c = cfg;
    c.data_term = 1;
    const dreg_solver_cfg s = b200_detail::S(c);
    VectorField out(target.dims, target.spacing);
    b200_detail::check(dreg_cuda_v_update(b200_detail::ctx(), target.data.data(), warped_source.data.data(),
                                          grad.data.data(), w_hat.data.data(), b_hat.data.data(),
                                          b200_detail::D(target.dims), &s, out.data.data()));
    return out;
}

inline VectorField v_update_l2(const ScalarVolume& target, const ScalarVolume& warped_source, const VectorField& grad,
                               const VectorField& w_hat, const VectorField& b_hat, const SolverConfig& cfg) {
    b200_detail::same(target.dims, warped_source.dims, "v_update_l2");
    b200_detail::same(target.dims, grad.dims, "v_update_l2");
    b200_detail::same(target.dims, w_hat.dims, "v_update_l2");
    b200_detail::same(target.dims, b_hat.dims, "v_update_l2");
    SolverConfig c = cfg;
    c.data_term = 2;
    const dreg_solver_cfg s = b200_detail::S(c);
    VectorField out(target.dims, target.spacing);
    b200_detail::check(dreg_cuda_v_update(b200_detail::ctx(), target.data.data(), warped_source.data.data(),
                                          grad.data.data(), w_hat.data.data(), b_hat.data.data(),
                                          b200_detail::D(target.dims), &s, out.data.data()));
    return out;
}

inline VectorField w_update(const VectorField& v, const VectorField& b_hat, const SpectralKernel& kernel,
                            const SolverConfig& cfg) {
    b200_detail::same(v.dims, b_hat.dims, "w_update");
    b200_detail::same(v.dims, kernel.dims, "w_update: kernel");
    // The device builds (-Delta_h)^n's symbol on the fly from 1-D tables, so it can only
    // apply kernels laplacian_symbol(order, dims) returns -- the only ones the reference
    // ever passes (admm.cpp:260).  Anything else is refused rather than ignored.
    if (kernel.values.size() != v.dims.voxels() || kernel.values != laplacian_symbol(kernel.order, kernel.dims).values)
        throw std::invalid_argument("w_update: kernel is not laplacian_symbol(order, dims); arbitrary spectral "
                                    "kernels are not supported by the device path");
    SolverConfig c = cfg;
    c.order = kernel.order;
    const dreg_solver_cfg s = b200_detail::S(c);
    VectorField out(v.dims, v.spacing);
    b200_detail::check(dreg_cuda_w_update(b200_detail::ctx(), v.data.data(), b_hat.data.data(), b200_detail::D(v.dims),
                                          &s, out.data.data()));
    return out;
}

// admm.hpp:68
inline double data_term_value(const ScalarVolume& target, const ScalarVolume& warped_source, const VectorField& grad,
                              const VectorField& v, int s) {
    b200_detail::same(target.dims, warped_source.dims, "data_term_value");
    b200_detail::same(target.dims, grad.dims, "data_term_value");
    b200_detail::same(target.dims, v.dims, "data_term_value");
    double out = 0.0;
    b200_detail::check(dreg_cuda_data_term_value(b200_detail::ctx(), target.data.data(), warped_source.data.data(),
                                                 grad.data.data(), v.data.data(), b200_detail::D(target.dims), s,
                                                 &out));
    return out;
}

// volume.hpp:107,110 -- evaluated on the device (one round trip per call: sample many
// points at once with the vector overloads below)
inline std::vector<double> trilinear_sample(const ScalarVolume& vol, const std::vector<Vec3>& points) {
    std::vector<double> out(points.size());
    static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
    b200_detail::check(dreg_cuda_trilinear_sample(b200_detail::ctx(), vol.data.data(), 1, b200_detail::D(vol.dims),
                                                  reinterpret_cast<const double*>(points.data()),
                                                  static_cast<int64_t>(points.size()), out.data()));
    return out;
}
inline std::vector<Vec3> trilinear_sample(const VectorField& field, const std::vector<Vec3>& points) {
    std::vector<Vec3> out(points.size());
    b200_detail::check(dreg_cuda_trilinear_sample(b200_detail::ctx(), field.data.data(), 3,
                                                  b200_detail::D(field.dims),
                                                  reinterpret_cast<const double*>(points.data()),
                                                  static_cast<int64_t>(points.size()),
                                                  reinterpret_cast<double*>(out.data())));
    return out;
}
inline double trilinear_sample(const ScalarVolume& vol, const Vec3& p) { return trilinear_sample(vol, std::vector<Vec3>{p})[0]; }
inline Vec3 trilinear_sample(const VectorField& field, const Vec3& p) {
    return trilinear_sample(field, std::vector<Vec3>{p})[0];
}

inline SolveResult solve_velocity(const ScalarVolume& target, const ScalarVolume& warped_source,
                                  const SolverConfig& cfg) {
    validate(cfg);
    b200_detail::same(target.dims, warped_source.dims, "solve_velocity");
    const dreg_solver_cfg s = b200_detail::S(cfg);
    SolveResult r{VectorField(target.dims, target.spacing), {}};
    std::vector<double> obj(static_cast<std::size_t>(cfg.max_iters)), res(static_cast<std::size_t>(cfg.max_iters));
    dreg_solver_diag d{0, 0.0, 0, obj.data(), res.data()};
    b200_detail::check(dreg_cuda_solve_velocity(b200_detail::ctx(), target.data.data(), warped_source.data.data(),
                                                b200_detail::D(target.dims), &s, r.velocity.data.data(), &d));
    r.diagnostics.iterations = d.iterations;
    r.diagnostics.final_change = d.final_change;
    r.diagnostics.converged = d.converged != 0;
    if (cfg.log_objective) r.diagnostics.objective.assign(obj.begin(), obj.begin() + d.iterations);
    r.diagnostics.constraint_residual.assign(res.begin(), res.begin() + d.iterations);
    return r;
}

inline RegistrationConfig make_registration_config(Profile profile, SolverConfig solver, int levels = 3) {
    if (levels < 1) throw std::invalid_argument("registration: levels must be >= 1");
    dreg_reg_cfg c;
    const dreg_solver_cfg s = b200_detail::S(solver);
    if (dreg_make_registration_config(profile == Profile::converged ? DREG_PROFILE_CONVERGED : DREG_PROFILE_CAPPED,
                                      &s, levels, &c) != DREG_OK)
        throw std::invalid_argument("registration: levels must be >= 1");
    RegistrationConfig r;
    r.solver = solver;
    r.solver.tol = c.solver.tol;
    r.levels = levels;
    r.max_warps_per_level.assign(c.max_warps_per_level, c.max_warps_per_level + levels);
    r.max_admm_iters_per_level.assign(c.max_admm_iters_per_level, c.max_admm_iters_per_level + levels);
    r.warp_improvement_threshold = c.warp_improvement_threshold;
    r.profile = profile;
    r.smooth_levels = true;
    return r;
}

inline dreg_reg_cfg to_c(const RegistrationConfig& cfg) {
    validate(cfg.solver);  // registration.cpp:183, before the level checks
    if (cfg.levels < 1) throw std::invalid_argument("register_pair: levels must be >= 1");
    if (cfg.max_warps_per_level.size() != static_cast<std::size_t>(cfg.levels) ||
        cfg.max_admm_iters_per_level.size() != static_cast<std::size_t>(cfg.levels))
        throw std::invalid_argument("register_pair: per-level caps must list one entry per level");
    if (!(cfg.warp_improvement_threshold > 0.0 && cfg.warp_improvement_threshold < 1.0))
        throw std::invalid_argument("register_pair: warp improvement threshold must be in (0,1)");
    if (cfg.levels > DREG_MAX_LEVELS)  // needs axes >= 4 << 10: registration.cpp:195 rejects any smaller grid
        throw std::invalid_argument("register_pair: dims too small for the level count");
    dreg_reg_cfg c;
    std::memset(&c, 0, sizeof c);
    c.solver = b200_detail::S(cfg.solver);
    c.levels = cfg.levels;
    for (int l = 0; l < cfg.levels; ++l) {
        c.max_warps_per_level[l] = cfg.max_warps_per_level[static_cast<std::size_t>(l)];
        c.max_admm_iters_per_level[l] = cfg.max_admm_iters_per_level[static_cast<std::size_t>(l)];
    }
    c.warp_improvement_threshold = cfg.warp_improvement_threshold;
    c.profile = cfg.profile == Profile::converged ? DREG_PROFILE_CONVERGED : DREG_PROFILE_CAPPED;
    c.smooth_levels = cfg.smooth_levels ? 1 : 0;
    return c;
}

inline RegistrationResult register_pair(const ScalarVolume& target, const ScalarVolume& source,
                                        const RegistrationConfig& cfg) {
    b200_detail::same(target.dims, source.dims, "register_pair");
    const dreg_reg_cfg c = to_c(cfg);
    RegistrationResult r;
    r.phi = DeformationField::identity(target.dims, target.spacing);
    r.warped = ScalarVolume(target.dims, target.spacing);
    dreg_pair_result pr;
    b200_detail::check(dreg_cuda_register_pair(b200_detail::ctx(), target.data.data(), source.data.data(),
                                               b200_detail::D(target.dims),
                                               {target.spacing.x, target.spacing.y, target.spacing.z}, &c,
                                               r.phi.disp.data.data(), r.warped.data.data(), &pr));
    r.velocity_count = pr.velocity_count;
    for (int l = 0; l < pr.levels; ++l) {
        const dreg_level_log& lg = pr.per_level[l];
        LevelLog o;
        o.dims = {lg.dims.x, lg.dims.y, lg.dims.z};
        o.warps = lg.warps;
        o.mean_sad.assign(lg.mean_sad, lg.mean_sad + lg.warps + 1);
        o.solver_iterations.assign(lg.solver_iterations, lg.solver_iterations + lg.warps);
        r.per_level.push_back(std::move(o));
    }
    r.elapsed_seconds = pr.elapsed_seconds;
    return r;
}

// ---- B200 extension: independent pairs sharded over the GPUs of one box ----------
// (no reference counterpart).  One host thread and context per
// device, one NCCL all-gather of the per-pair records.  Each result equals
// register_pair's for the same pair.
class MultiDevice {
public:
    explicit MultiDevice(const std::vector<int>& devices) {
        if (devices.empty()) throw std::invalid_argument("MultiDevice: no devices");
        const int st = dreg_cuda_multi_create(devices.data(), static_cast<int>(devices.size()), &m_);
        if (st == DREG_INVALID_ARGUMENT) throw std::invalid_argument("MultiDevice: bad or repeated device index");
        if (st != DREG_OK) throw std::runtime_error("MultiDevice: CUDA / NCCL initialisation failed");
    }
    MultiDevice(const MultiDevice&) = delete;
    MultiDevice& operator=(const MultiDevice&) = delete;
    ~MultiDevice() { dreg_cuda_multi_destroy(m_); }
    int device_count() const { return dreg_cuda_multi_device_count(m_); }

    std::vector<RegistrationResult> register_batch(const std::vector<ScalarVolume>& targets,
                                                   const std::vector<ScalarVolume>& sources,
                                                   const RegistrationConfig& cfg,
                                                   std::vector<dreg_pair_record>* records = nullptr) {
        if (targets.size() != sources.size()) throw std::invalid_argument("register_batch: pair count mismatch");
        const std::size_t n = targets.size();
        std::vector<RegistrationResult> out(n);
        if (n == 0) return out;
        const Dims3 d = targets[0].dims;
        for (std::size_t i = 0; i < n; ++i) {
            b200_detail::same(d, targets[i].dims, "register_batch");
            b200_detail::same(d, sources[i].dims, "register_batch");
        }
        const dreg_reg_cfg c = to_c(cfg);
        std::vector<const float*> tp(n), sp(n);
        std::vector<float*> pp(n), wp(n);
        for (std::size_t i = 0; i < n; ++i) {
            out[i].phi = DeformationField::identity(d, targets[i].spacing);
            out[i].warped = ScalarVolume(d, targets[i].spacing);
            tp[i] = targets[i].data.data();
            sp[i] = sources[i].data.data();
            pp[i] = out[i].phi.disp.data.data();
            wp[i] = out[i].warped.data.data();
        }
        std::vector<dreg_pair_result> pr(n);
        std::vector<dreg_pair_record> rec(n);
        const int st = dreg_cuda_multi_register_batch(
            m_, static_cast<int>(n), tp.data(), sp.data(), b200_detail::D(d),
            {targets[0].spacing.x, targets[0].spacing.y, targets[0].spacing.z}, &c, pp.data(), wp.data(), pr.data(),
            rec.data());
        if (st == DREG_INVALID_ARGUMENT) throw std::invalid_argument(dreg_cuda_multi_last_error(m_));
        if (st == DREG_NUMERIC) throw numeric_error(dreg_cuda_multi_last_error(m_));
        if (st != DREG_OK) throw std::runtime_error(dreg_cuda_multi_last_error(m_));
        for (std::size_t i = 0; i < n; ++i) {
            out[i].velocity_count = pr[i].velocity_count;
            for (int l = 0; l < pr[i].levels; ++l) {
                const dreg_level_log& lg = pr[i].per_level[l];
                LevelLog o;
                o.dims = {lg.dims.x, lg.dims.y, lg.dims.z};
                o.warps = lg.warps;
                o.mean_sad.assign(lg.mean_sad, lg.mean_sad + lg.warps + 1);
                o.solver_iterations.assign(lg.solver_iterations, lg.solver_iterations + lg.warps);
                out[i].per_level.push_back(std::move(o));
            }
            out[i].elapsed_seconds = pr[i].elapsed_seconds;
        }
        if (records) *records = std::move(rec);
        return out;
    }

private:
    dreg_cuda_multi* m_ = nullptr;
};

inline ScalarVolume warp_image(const ScalarVolume& img, const DeformationField& phi) {
    b200_detail::same(img.dims, phi.disp.dims, "warp_image");
    ScalarVolume out(img.dims, img.spacing);
    b200_detail::check(dreg_cuda_warp_image(b200_detail::ctx(), img.data.data(), phi.disp.data.data(),
                                            b200_detail::D(img.dims), out.data.data()));
    return out;
}

inline VectorField image_gradient(const ScalarVolume& img) {
    VectorField out(img.dims, img.spacing);
    b200_detail::check(dreg_cuda_image_gradient(b200_detail::ctx(), img.data.data(), b200_detail::D(img.dims),
                                                out.data.data()));
    return out;
}

inline DeformationField compose_deformation(const DeformationField& phi, const VectorField& v) {
    b200_detail::same(phi.disp.dims, v.dims, "compose_deformation");
    DeformationField out{VectorField(v.dims, phi.disp.spacing)};
    b200_detail::check(dreg_cuda_compose_deformation(b200_detail::ctx(), phi.disp.data.data(), v.data.data(),
                                                     b200_detail::D(v.dims), out.disp.data.data()));
    return out;
}

inline ScalarVolume jacobian_determinant(const DeformationField& phi) {
    ScalarVolume out(phi.disp.dims, phi.disp.spacing);
    b200_detail::check(dreg_cuda_jacobian(b200_detail::ctx(), phi.disp.data.data(), b200_detail::D(phi.disp.dims),
                                          out.data.data(), nullptr));
    return out;
}

inline JacobianStats jacobian_stats(const DeformationField& phi) {
    dreg_jacobian_stats st;
    b200_detail::check(dreg_cuda_jacobian(b200_detail::ctx(), phi.disp.data.data(), b200_detail::D(phi.disp.dims),
                                          nullptr, &st));
    return {st.pct_nonpositive, st.min_det};
}

inline std::pair<ScalarVolume, ScalarVolume> normalize_intensity_pair(const ScalarVolume& a, const ScalarVolume& b) {
    b200_detail::same(a.dims, b.dims, "normalize_intensity_pair");
    ScalarVolume oa(a.dims, a.spacing), ob(b.dims, b.spacing);
    b200_detail::check(dreg_cuda_normalize_intensity_pair(b200_detail::ctx(), a.data.data(), b.data.data(),
                                                          b200_detail::D(a.dims), oa.data.data(), ob.data.data()));
    return {std::move(oa), std::move(ob)};
}

inline ScalarVolume binomial_smooth(const ScalarVolume& img) {
    ScalarVolume out(img.dims, img.spacing);
    b200_detail::check(dreg_cuda_binomial_smooth(b200_detail::ctx(), img.data.data(), b200_detail::D(img.dims),
                                                 out.data.data()));
    return out;
}

inline double mean_sad(const ScalarVolume& a, const ScalarVolume& b) {
    b200_detail::same(a.dims, b.dims, "mean_sad");
    double m = 0.0;
    b200_detail::check(dreg_cuda_mean_sad(b200_detail::ctx(), a.data.data(), b.data.data(), b200_detail::D(a.dims), &m));
    return m;
}

inline ScalarVolume downsample(const ScalarVolume& img) {
    const Dims3 o{(img.dims.x + 1) / 2, (img.dims.y + 1) / 2, (img.dims.z + 1) / 2};
    ScalarVolume out(o, {img.spacing.x * 2.0, img.spacing.y * 2.0, img.spacing.z * 2.0});
    b200_detail::check(dreg_cuda_downsample(b200_detail::ctx(), img.data.data(), b200_detail::D(img.dims),
                                            out.data.data()));
    return out;
}

inline VectorField upsample_velocity(const VectorField& v, Dims3 target_dims) {
    VectorField out(target_dims, {v.spacing.x / 2.0, v.spacing.y / 2.0, v.spacing.z / 2.0});
    b200_detail::check(dreg_cuda_upsample_velocity(b200_detail::ctx(), v.data.data(), b200_detail::D(v.dims),
                                                   b200_detail::D(target_dims), out.data.data()));
    return out;
}

inline DeformationField upsample_deformation(const DeformationField& phi, Dims3 target_dims) {
    return {upsample_velocity(phi.disp, target_dims)};
}

// ---- io.hpp (host file I/O through the C ABI; byte-compatible) -------------------------
namespace b200_detail {
inline void io_check(int st, const char* err) {
    if (st == DREG_OK) return;
    if (st == DREG_IO_ERROR) throw io_error(err);
    if (st == DREG_INVALID_ARGUMENT) throw std::invalid_argument(err);
    throw std::runtime_error(err);
}
inline AnyVolume read_any(const std::filesystem::path& path, int expected_kind) {
    char err[1024];
    dreg_volume_info info;
    const std::string p = path.string();
    io_check(dreg_volume_read(p.c_str(), expected_kind, &info, nullptr, 0, err, sizeof err), err);
    const Dims3 d{info.dims.x, info.dims.y, info.dims.z};
    const Spacing3 sp{info.spacing.x, info.spacing.y, info.spacing.z};
    if (info.kind == DREG_KIND_LABEL) {
        LabelVolume v(d, sp);
        io_check(dreg_volume_read(p.c_str(), expected_kind, &info, v.labels.data(), 2 * v.labels.size(), err,
                                  sizeof err), err);
        return v;
    }
    if (info.kind == DREG_KIND_VECTOR) {
        VectorField v(d, sp);
        io_check(dreg_volume_read(p.c_str(), expected_kind, &info, v.data.data(), 4 * v.data.size(), err, sizeof err),
                 err);
        return v;
    }
    ScalarVolume v(d, sp);
    io_check(dreg_volume_read(p.c_str(), expected_kind, &info, v.data.data(), 4 * v.data.size(), err, sizeof err),
             err);
    return v;
}
inline void write_any(const std::filesystem::path& path, int kind, Dims3 d, Spacing3 s, const void* payload) {
    char err[1024];
    io_check(dreg_volume_write(path.string().c_str(), kind, D(d), {s.x, s.y, s.z}, payload, err, sizeof err), err);
}
}  // namespace b200_detail

inline AnyVolume read_volume(const std::filesystem::path& path) { return b200_detail::read_any(path, -1); }
inline ScalarVolume read_scalar(const std::filesystem::path& path) {
    return std::get<ScalarVolume>(b200_detail::read_any(path, DREG_KIND_SCALAR));
}
inline VectorField read_vector(const std::filesystem::path& path) {
    return std::get<VectorField>(b200_detail::read_any(path, DREG_KIND_VECTOR));
}
inline LabelVolume read_label(const std::filesystem::path& path) {
    return std::get<LabelVolume>(b200_detail::read_any(path, DREG_KIND_LABEL));
}
inline DeformationField read_deformation(const std::filesystem::path& path) { return {read_vector(path)}; }

inline void write_volume(const std::filesystem::path& path, const ScalarVolume& v) {
    b200_detail::write_any(path, DREG_KIND_SCALAR, v.dims, v.spacing, v.data.data());
}
inline void write_volume(const std::filesystem::path& path, const VectorField& v) {
    b200_detail::write_any(path, DREG_KIND_VECTOR, v.dims, v.spacing, v.data.data());
}
inline void write_volume(const std::filesystem::path& path, const LabelVolume& v) {
    b200_detail::write_any(path, DREG_KIND_LABEL, v.dims, v.spacing, v.labels.data());
}
inline void write_volume(const std::filesystem::path& path, const DeformationField& phi) {
    write_volume(path, phi.disp);
}

inline void write_report(const std::filesystem::path& path, const RunReport& r) {
    std::vector<int> dl, hl;
    std::vector<double> dv, hv;
    for (const auto& [k, v] : r.dice) dl.push_back(k), dv.push_back(v);
    for (const auto& [k, v] : r.hausdorff_mm) hl.push_back(k), hv.push_back(v);
    const ReportConfig& c = r.config;
    dreg_run_report rep{static_cast<int>(dl.size()), dl.data(), dv.data(), static_cast<int>(hl.size()), hl.data(),
                        hv.data(), r.jacobian_pct_nonpositive, r.runtime_seconds, r.velocity_count,
                        {c.data_term.c_str(), c.order, c.lambda, c.theta, c.levels, c.profile.c_str(), c.tol,
                         c.warp_improvement_threshold, c.epsilon, c.threads}};
    char err[1024];
    b200_detail::io_check(dreg_report_write(path.string().c_str(), &rep, err, sizeof err), err);
}

// ---- metrics.hpp label metrics (GPU) --------------------------------------------------
inline double dice(const LabelVolume& a, const LabelVolume& b, int label) {
    b200_detail::same(a.dims, b.dims, "dice");
    double out = 0.0;
    b200_detail::check(dreg_cuda_dice(b200_detail::ctx(), a.labels.data(), b.labels.data(), b200_detail::D(a.dims),
                                      label, &out));
    return out;
}

inline double hausdorff_slice_avg(const LabelVolume& a, const LabelVolume& b, int label) {
    b200_detail::same(a.dims, b.dims, "hausdorff_slice_avg");
    double out = 0.0;
    b200_detail::check(dreg_cuda_hausdorff_slice_avg(b200_detail::ctx(), a.labels.data(), b.labels.data(),
                                                     b200_detail::D(a.dims),
                                                     {a.spacing.x, a.spacing.y, a.spacing.z}, label, &out));
    return out;
}

inline LabelVolume warp_labels(const LabelVolume& lbl, const DeformationField& phi) {
    b200_detail::same(lbl.dims, phi.disp.dims, "warp_labels");
    LabelVolume out(lbl.dims, lbl.spacing);
    b200_detail::check(dreg_cuda_warp_labels(b200_detail::ctx(), lbl.labels.data(), phi.disp.data.data(),
                                             b200_detail::D(lbl.dims), out.labels.data()));
    return out;
}

}  // namespace dreg
