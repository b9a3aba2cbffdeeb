// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" wrappers around the UNMODIFIED reference library (`dreg::` in
// /root/reference/proj/core), compiled from its own sources by oracle/Makefile into
// oracle/_ref/libdreg_ref.so.  Used by tests/ to pin the C restatement
// (oracle/dreg_oracle.c) and by bench.py --impl reference as the CPU baseline.
// Every entry mirrors one reference function; exceptions become status codes
// (2 invalid_argument, 4 numeric_error, 5 other) with the message in ref_last_error().
#include <algorithm>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <variant>
#include <vector>

#include "dreg/admm.hpp"
#include "dreg/errors.hpp"
#include "dreg/io.hpp"
#include "dreg/metrics.hpp"
#include "dreg/parallel.hpp"
#include "dreg/registration.hpp"
#include "dreg/regularizer.hpp"
#include "dreg/synth.hpp"
#include "dreg/volume.hpp"
#include "dreg_cuda.h"

namespace {

thread_local std::string g_err;

dreg::Dims3 D(dreg_dims3 d) { return {d.x, d.y, d.z}; }

dreg::ScalarVolume scalar(const float* p, dreg_dims3 d) {
    dreg::ScalarVolume v(D(d), {1.0, 1.0, 1.0});
    std::memcpy(v.data.data(), p, sizeof(float) * v.data.size());
    return v;
}

dreg::VectorField vec(const float* p, dreg_dims3 d) {
    dreg::VectorField v(D(d), {1.0, 1.0, 1.0});
    std::memcpy(v.data.data(), p, sizeof(float) * v.data.size());
    return v;
}

dreg::SolverConfig solver(const dreg_solver_cfg* c) {
    dreg::SolverConfig s;
    s.data_term = c->data_term;
    s.order = c->order;
    s.lambda = c->lambda;
    s.theta = c->theta;
    s.epsilon = c->epsilon;
    s.max_iters = c->max_iters;
    s.tol = c->tol;
    s.accelerate = c->accelerate != 0;
    s.log_objective = c->log_objective != 0;
    return s;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return DREG_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return DREG_INVALID_ARGUMENT;
    } catch (const dreg::numeric_error& e) {
        g_err = e.what();
        return DREG_NUMERIC;
    } catch (const dreg::io_error& e) {
        g_err = e.what();
        return DREG_IO_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DREG_RUNTIME;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_thread_count(int n) { dreg::set_thread_count(n); }
int ref_hardware_threads(void) { return static_cast<int>(std::thread::hardware_concurrency()); }
double ref_nesterov_next_alpha(double a) { return dreg::nesterov_next_alpha(a); }

int ref_validate(const dreg_solver_cfg* c) {
    return guard([&] { dreg::validate(solver(c)); });
}

int ref_make_registration_config(int profile, const dreg_solver_cfg* c, int levels,
                                 dreg_reg_cfg* out) {
    return guard([&] {
        const auto cfg = dreg::make_registration_config(
            profile == DREG_PROFILE_CONVERGED ? dreg::Profile::converged : dreg::Profile::capped,
            solver(c), levels);
        std::memset(out, 0, sizeof(*out));
        out->solver = *c;
        out->solver.tol = cfg.solver.tol;
        out->levels = cfg.levels;
        for (int l = 0; l < cfg.levels && l < DREG_MAX_LEVELS; ++l) {
            out->max_warps_per_level[l] = cfg.max_warps_per_level[static_cast<size_t>(l)];
            out->max_admm_iters_per_level[l] = cfg.max_admm_iters_per_level[static_cast<size_t>(l)];
        }
        out->warp_improvement_threshold = cfg.warp_improvement_threshold;
        out->profile = profile;
        out->smooth_levels = cfg.smooth_levels ? 1 : 0;
    });
}

int ref_laplacian_symbol(int n, dreg_dims3 d, double* out) {
    return guard([&] {
        const auto k = dreg::laplacian_symbol(n, D(d));
        std::memcpy(out, k.values.data(), sizeof(double) * k.values.size());
    });
}

int ref_regulariser_energy(const float* w, dreg_dims3 d, int n, double* out) {
    return guard([&] { *out = dreg::regulariser_energy(vec(w, d), n); });
}

int ref_v_update(const float* target, const float* warped, const float* grad,
                 const float* w_hat, const float* b_hat, dreg_dims3 d,
                 const dreg_solver_cfg* c, float* out) {
    return guard([&] {
        const auto s = solver(c);
        const auto r = s.data_term == 1
                           ? dreg::v_update_l1(scalar(target, d), scalar(warped, d), vec(grad, d),
                                               vec(w_hat, d), vec(b_hat, d), s)
                           : dreg::v_update_l2(scalar(target, d), scalar(warped, d), vec(grad, d),
                                               vec(w_hat, d), vec(b_hat, d), s);
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_w_update(const float* v, const float* b_hat, dreg_dims3 d, const dreg_solver_cfg* c,
                 float* out) {
    return guard([&] {
        const auto s = solver(c);
        const auto k = dreg::laplacian_symbol(s.order, D(d));
        const auto r = dreg::w_update(vec(v, d), vec(b_hat, d), k, s);
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_trilinear_sample(const float* f, int ncomp, dreg_dims3 d, const double* pts, int64_t n, double* out) {
    return guard([&] {
        if (ncomp == 1) {
            const auto vol = scalar(f, d);
            for (int64_t i = 0; i < n; ++i)
                out[i] = dreg::trilinear_sample(vol, dreg::Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
        } else {
            const auto fld = vec(f, d);
            for (int64_t i = 0; i < n; ++i) {
                const dreg::Vec3 r = dreg::trilinear_sample(fld, dreg::Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
                out[3 * i] = r.x;
                out[3 * i + 1] = r.y;
                out[3 * i + 2] = r.z;
            }
        }
    });
}

int ref_data_term_value(const float* target, const float* warped, const float* grad,
                        const float* v, dreg_dims3 d, int s, double* out) {
    return guard([&] {
        *out = dreg::data_term_value(scalar(target, d), scalar(warped, d), vec(grad, d), vec(v, d), s);
    });
}

int ref_solve_velocity(const float* target, const float* warped, dreg_dims3 d,
                       const dreg_solver_cfg* c, float* v_out, dreg_solver_diag* diag) {
    return guard([&] {
        const auto r = dreg::solve_velocity(scalar(target, d), scalar(warped, d), solver(c));
        std::memcpy(v_out, r.velocity.data.data(), sizeof(float) * r.velocity.data.size());
        if (diag) {
            diag->iterations = r.diagnostics.iterations;
            diag->final_change = r.diagnostics.final_change;
            diag->converged = r.diagnostics.converged ? 1 : 0;
            if (diag->objective)
                std::copy(r.diagnostics.objective.begin(), r.diagnostics.objective.end(),
                          diag->objective);
            if (diag->constraint_residual)
                std::copy(r.diagnostics.constraint_residual.begin(),
                          r.diagnostics.constraint_residual.end(), diag->constraint_residual);
        }
    });
}

int ref_warp_image(const float* img, const float* disp, dreg_dims3 d, float* out) {
    return guard([&] {
        const auto r = dreg::warp_image(scalar(img, d), dreg::make_deformation(vec(disp, d)));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_image_gradient(const float* img, dreg_dims3 d, float* out) {
    return guard([&] {
        const auto r = dreg::image_gradient(scalar(img, d));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_compose_deformation(const float* disp, const float* v, dreg_dims3 d, float* out) {
    return guard([&] {
        const auto r = dreg::compose_deformation(dreg::make_deformation(vec(disp, d)), vec(v, d));
        std::memcpy(out, r.disp.data.data(), sizeof(float) * r.disp.data.size());
    });
}

int ref_jacobian(const float* disp, dreg_dims3 d, float* det_out, dreg_jacobian_stats* st) {
    return guard([&] {
        const auto phi = dreg::make_deformation(vec(disp, d));
        if (det_out) {
            const auto r = dreg::jacobian_determinant(phi);
            std::memcpy(det_out, r.data.data(), sizeof(float) * r.data.size());
        }
        if (st) {
            const auto s = dreg::jacobian_stats(phi);
            st->pct_nonpositive = s.pct_nonpositive;
            st->min_det = s.min_det;
            // raw counts of the same interior scan (metrics.cpp:217-227)
            const auto det = dreg::jacobian_determinant(phi);
            int64_t nonpos = 0, interior = 0;
            for (int z = 1; z < d.z - 1; ++z)
                for (int y = 1; y < d.y - 1; ++y)
                    for (int x = 1; x < d.x - 1; ++x) {
                        nonpos += static_cast<double>(det.at(x, y, z)) <= 0.0;
                        ++interior;
                    }
            st->nonpositive = nonpos;
            st->interior = interior;
        }
    });
}

int ref_normalize_intensity_pair(const float* a, const float* b, dreg_dims3 d, float* oa,
                                 float* ob) {
    return guard([&] {
        const auto r = dreg::normalize_intensity_pair(scalar(a, d), scalar(b, d));
        std::memcpy(oa, r.first.data.data(), sizeof(float) * r.first.data.size());
        std::memcpy(ob, r.second.data.data(), sizeof(float) * r.second.data.size());
    });
}

int ref_binomial_smooth(const float* img, dreg_dims3 d, float* out) {
    return guard([&] {
        const auto r = dreg::binomial_smooth(scalar(img, d));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_mean_sad(const float* a, const float* b, dreg_dims3 d, double* out) {
    return guard([&] { *out = dreg::mean_sad(scalar(a, d), scalar(b, d)); });
}

int ref_downsample(const float* img, dreg_dims3 d, float* out) {
    return guard([&] {
        const auto r = dreg::downsample(scalar(img, d));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_upsample_velocity(const float* v, dreg_dims3 src, dreg_dims3 dst, float* out) {
    return guard([&] {
        const auto r = dreg::upsample_velocity(vec(v, src), D(dst));
        std::memcpy(out, r.data.data(), sizeof(float) * r.data.size());
    });
}

int ref_register_pair(const float* target, const float* source, dreg_dims3 d,
                      dreg_spacing3 sp, const dreg_reg_cfg* c, float* phi_out,
                      float* warped_out, dreg_pair_result* res) {
    return guard([&] {
        dreg::RegistrationConfig cfg;
        cfg.solver = solver(&c->solver);
        cfg.levels = c->levels;
        cfg.max_warps_per_level.assign(c->max_warps_per_level,
                                       c->max_warps_per_level + std::max(0, c->levels));
        cfg.max_admm_iters_per_level.assign(c->max_admm_iters_per_level,
                                            c->max_admm_iters_per_level + std::max(0, c->levels));
        cfg.warp_improvement_threshold = c->warp_improvement_threshold;
        cfg.profile = c->profile == DREG_PROFILE_CONVERGED ? dreg::Profile::converged
                                                           : dreg::Profile::capped;
        cfg.smooth_levels = c->smooth_levels != 0;
        dreg::ScalarVolume t = scalar(target, d);
        dreg::ScalarVolume s = scalar(source, d);
        t.spacing = s.spacing = {sp.x, sp.y, sp.z};
        const auto r = dreg::register_pair(t, s, cfg);
        if (phi_out) std::memcpy(phi_out, r.phi.disp.data.data(), sizeof(float) * r.phi.disp.data.size());
        if (warped_out) std::memcpy(warped_out, r.warped.data.data(), sizeof(float) * r.warped.data.size());
        if (res) {
            std::memset(res, 0, sizeof(*res));
            res->status = DREG_OK;
            res->velocity_count = r.velocity_count;
            res->levels = static_cast<int>(r.per_level.size());
            for (size_t l = 0; l < r.per_level.size() && l < DREG_MAX_LEVELS; ++l) {
                const auto& lg = r.per_level[l];
                auto& o = res->per_level[l];
                o.dims = {lg.dims.x, lg.dims.y, lg.dims.z};
                o.warps = lg.warps;
                for (size_t i = 0; i < lg.mean_sad.size() && i <= DREG_MAX_WARPS; ++i)
                    o.mean_sad[i] = lg.mean_sad[i];
                for (size_t i = 0; i < lg.solver_iterations.size() && i < DREG_MAX_WARPS; ++i)
                    o.solver_iterations[i] = lg.solver_iterations[i];
            }
            res->elapsed_seconds = r.elapsed_seconds;
        }
    });
}

// The reference's own synthetic cases (synth.hpp), for restating its registration and
// acceptance tests on identical inputs: kind 0 translate (shift), 1 sphere->ellipsoid,
// 2 random smooth (seed).  Labels are uint16 as in LabelVolume (nullable).
int ref_make_case(int kind, dreg_dims3 d, const double* shift, unsigned seed, float* target, float* source,
                  unsigned short* target_labels, unsigned short* source_labels) {
    return guard([&] {
        dreg::SynthPair p;
        if (kind == 0) p = dreg::make_translate_case(D(d), dreg::Vec3{shift[0], shift[1], shift[2]});
        else if (kind == 1) p = dreg::make_sphere_ellipsoid_case(D(d));
        else p = dreg::make_random_smooth_case(D(d), seed);
        std::memcpy(target, p.target.data.data(), sizeof(float) * p.target.data.size());
        std::memcpy(source, p.source.data.data(), sizeof(float) * p.source.data.size());
        if (target_labels)
            std::memcpy(target_labels, p.target_labels.labels.data(), 2 * p.target_labels.labels.size());
        if (source_labels)
            std::memcpy(source_labels, p.source_labels.labels.data(), 2 * p.source_labels.labels.size());
    });
}

// dice(warp_labels(moving, phi), fixed, label)   (metrics.hpp:31,39)
int ref_warped_label_dice(const unsigned short* moving, const float* disp, const unsigned short* fixed, dreg_dims3 d,
                          int label, double* out) {
    return guard([&] {
        dreg::LabelVolume mv(D(d), {1.0, 1.0, 1.0}), fx(D(d), {1.0, 1.0, 1.0});
        std::memcpy(mv.labels.data(), moving, 2 * mv.labels.size());
        std::memcpy(fx.labels.data(), fixed, 2 * fx.labels.size());
        const auto w = dreg::warp_labels(mv, dreg::make_deformation(vec(disp, d)));
        *out = dreg::dice(w, fx, label);
    });
}

// add_salt_pepper (synth.hpp) on a scalar volume, in place.
int ref_add_salt_pepper(float* vol, dreg_dims3 d, double fraction, unsigned seed) {
    return guard([&] {
        auto v = scalar(vol, d);
        dreg::add_salt_pepper(v, fraction, seed);
        std::memcpy(vol, v.data.data(), sizeof(float) * v.data.size());
    });
}

dreg::LabelVolume labels_of(const unsigned short* p, dreg_dims3 d, dreg_spacing3 s) {
    dreg::LabelVolume v(D(d), {s.x, s.y, s.z});
    std::memcpy(v.labels.data(), p, 2 * v.labels.size());
    return v;
}

// dice / hausdorff_slice_avg / warp_labels (metrics.hpp:31-42)
int ref_dice(const unsigned short* a, const unsigned short* b, dreg_dims3 d, int label, double* out) {
    return guard([&] { *out = dreg::dice(labels_of(a, d, {1, 1, 1}), labels_of(b, d, {1, 1, 1}), label); });
}
int ref_hausdorff_slice_avg(const unsigned short* a, const unsigned short* b, dreg_dims3 d, dreg_spacing3 s,
                            int label, double* out) {
    return guard([&] { *out = dreg::hausdorff_slice_avg(labels_of(a, d, s), labels_of(b, d, s), label); });
}
int ref_warp_labels(const unsigned short* lbl, const float* disp, dreg_dims3 d, unsigned short* out) {
    return guard([&] {
        const auto w = dreg::warp_labels(labels_of(lbl, d, {1, 1, 1}), dreg::make_deformation(vec(disp, d)));
        std::memcpy(out, w.labels.data(), 2 * w.labels.size());
    });
}

// write_volume / read_volume (io.hpp:27-40) on raw payloads
int ref_write_volume(const char* path, int kind, dreg_dims3 d, dreg_spacing3 s, const void* payload) {
    return guard([&] {
        const dreg::Spacing3 sp{s.x, s.y, s.z};
        if (kind == 0) {
            dreg::ScalarVolume v(D(d), sp);
            std::memcpy(v.data.data(), payload, 4 * v.data.size());
            dreg::write_volume(path, v);
        } else if (kind == 1) {
            dreg::VectorField v(D(d), sp);
            std::memcpy(v.data.data(), payload, 4 * v.data.size());
            dreg::write_volume(path, v);
        } else {
            dreg::LabelVolume v(D(d), sp);
            std::memcpy(v.labels.data(), payload, 2 * v.labels.size());
            dreg::write_volume(path, v);
        }
    });
}
// expected_kind: -1 read_volume, 0 read_scalar, 1 read_vector, 2 read_label
int ref_read_volume(const char* path, int expected_kind, dreg_volume_info* info, void* payload, size_t cap) {
    return guard([&] {
        dreg::AnyVolume any;
        if (expected_kind == 0) any = dreg::read_scalar(path);
        else if (expected_kind == 1) any = dreg::read_vector(path);
        else if (expected_kind == 2) any = dreg::read_label(path);
        else any = dreg::read_volume(path);
        std::visit(
            [&](const auto& v) {
                using T = std::decay_t<decltype(v)>;
                info->dims = {v.dims.x, v.dims.y, v.dims.z};
                info->spacing = {v.spacing.x, v.spacing.y, v.spacing.z};
                if constexpr (std::is_same_v<T, dreg::LabelVolume>) {
                    info->kind = 2;
                    if (payload && cap >= 2 * v.labels.size()) std::memcpy(payload, v.labels.data(), 2 * v.labels.size());
                } else {
                    info->kind = std::is_same_v<T, dreg::ScalarVolume> ? 0 : 1;
                    if (payload && cap >= 4 * v.data.size()) std::memcpy(payload, v.data.data(), 4 * v.data.size());
                }
            },
            any);
    });
}
// write_report (io.hpp:64-66)
int ref_write_report(const char* path, const dreg_run_report* r) {
    return guard([&] {
        dreg::RunReport rep;
        for (int i = 0; i < r->n_dice; ++i) rep.dice[r->dice_labels[i]] = r->dice[i];
        for (int i = 0; i < r->n_hausdorff; ++i) rep.hausdorff_mm[r->hausdorff_labels[i]] = r->hausdorff_mm[i];
        rep.jacobian_pct_nonpositive = r->jacobian_pct_nonpositive;
        rep.runtime_seconds = r->runtime_seconds;
        rep.velocity_count = r->velocity_count;
        const dreg_report_config& c = r->config;
        rep.config = {c.data_term, c.order, c.lambda, c.theta, c.levels, c.profile,
                      c.tol, c.warp_improvement_threshold, c.epsilon, c.threads};
        dreg::write_report(path, rep);
    });
}

}  // extern "C"
