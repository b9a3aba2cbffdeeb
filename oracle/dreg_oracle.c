/*
 * TEST INFRASTRUCTURE ONLY -- see dreg_oracle.h.  Plain-C restatement of the
 * reference hot path.  Citations are to /root/reference/proj/core/...
 */
#include "dreg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "fft_core.h"

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* dro_last_error(void) { return g_err; }

static size_t nvox(dreg_dims3 d) { return (size_t)d.x * (size_t)d.y * (size_t)d.z; }
static size_t flat(dreg_dims3 d, int x, int y, int z) {
    return (size_t)x + (size_t)d.x * ((size_t)y + (size_t)d.y * (size_t)z);
}
static int dims_ok(dreg_dims3 d) { return d.x >= 1 && d.y >= 1 && d.z >= 1; }

/* ---- admm.cpp:198-200 ------------------------------------------------------- */
double dro_nesterov_next_alpha(double a) { return 0.5 * (1.0 + sqrt(1.0 + 4.0 * a * a)); }

/* ---- admm.cpp:174-196 ------------------------------------------------------- */
int dro_validate(const dreg_solver_cfg* c) {
    if (c->data_term != 1 && c->data_term != 2)
        return fail(DREG_INVALID_ARGUMENT, "solver: data term exponent must be 1 or 2");
    if (c->order < 1 || c->order > 6)
        return fail(DREG_INVALID_ARGUMENT, "solver: regulariser order must be in [1, 6]");
    if (!(c->lambda >= 0.0)) return fail(DREG_INVALID_ARGUMENT, "solver: lambda must be >= 0");
    if (!(c->theta > 0.0)) return fail(DREG_INVALID_ARGUMENT, "solver: theta must be > 0");
    if (!(c->epsilon > 0.0)) return fail(DREG_INVALID_ARGUMENT, "solver: epsilon must be > 0");
    if (c->max_iters < 1) return fail(DREG_INVALID_ARGUMENT, "solver: max_iters must be >= 1");
    if (!(c->tol >= 0.0)) return fail(DREG_INVALID_ARGUMENT, "solver: tol must be >= 0");
    return DREG_OK;
}

/* ---- registration.cpp:62-83 ------------------------------------------------- */
int dro_make_registration_config(int profile, const dreg_solver_cfg* c, int levels,
                                 dreg_reg_cfg* out) {
    if (levels < 1) return fail(DREG_INVALID_ARGUMENT, "registration: levels must be >= 1");
    if (levels > DREG_MAX_LEVELS) return fail(DREG_INVALID_ARGUMENT, "registration: too many levels");
    memset(out, 0, sizeof *out);
    out->solver = *c;
    out->levels = levels;
    out->profile = profile;
    out->warp_improvement_threshold = 0.02;
    out->smooth_levels = 1;
    if (profile == DREG_PROFILE_CAPPED) {
        for (int l = 0; l < levels; ++l) {
            out->max_admm_iters_per_level[l] = 5;
            out->max_warps_per_level[l] = 10;
        }
        out->max_admm_iters_per_level[0] = 10;
        out->max_warps_per_level[levels - 1] = 5;
    } else {
        for (int l = 0; l < levels; ++l) {
            out->max_admm_iters_per_level[l] = 200;
            out->max_warps_per_level[l] = 50;
        }
        if (out->solver.tol <= 0.0) out->solver.tol = 0.01;
    }
    return DREG_OK;
}

/* ---- regularizer.cpp:24-31 (axis_cosines) and :51-79 (laplacian_symbol) ----- */
static double* axis_cosines(int n) {
    double* c = (double*)malloc(sizeof(double) * (size_t)n);
    for (int k = 0; k < n; ++k) c[k] = cos(2.0 * 3.14159265358979323846 * k / n);
    c[0] = 1.0;
    return c;
}

int dro_laplacian_symbol(int n, dreg_dims3 d, double* out) {
    if (n < 1 || n > 6) return fail(DREG_INVALID_ARGUMENT, "laplacian_symbol: order must be in [1, 6]");
    if (d.x < 2 || d.y < 2 || d.z < 2)
        return fail(DREG_INVALID_ARGUMENT, "laplacian_symbol: every axis must have size >= 2");
    double* cx = axis_cosines(d.x);
    double* cy = axis_cosines(d.y);
    double* cz = axis_cosines(d.z);
    size_t i = 0;
    for (int r = 0; r < d.z; ++r)
        for (int q = 0; q < d.y; ++q) {
            const double yz = 3.0 - cy[q] - cz[r];
            for (int p = 0; p < d.x; ++p, ++i) {
                const double base = 2.0 * (yz - cx[p]);
                double v = base;
                for (int e = 1; e < n; ++e) v *= base;
                out[i] = v;
            }
        }
    free(cx);
    free(cy);
    free(cz);
    return DREG_OK;
}

/* spectral energy of one field under a full-grid kernel: admm.cpp:103-127 and
 * regularizer.cpp:81-108 (identical loops) */
static double spectral_energy(const float* w, dreg_dims3 d, const double* kernel, oc_fft3* fft,
                              double* real, oc_complex* spec) {
    const size_t n = nvox(d);
    const int half = d.x / 2;
    const int hx = half + 1;
    double energy = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (size_t i = 0; i < n; ++i) real[i] = w[3 * i + (size_t)c];
        oc_fft3_r2c(fft, real, spec);
        for (int r = 0; r < d.z; ++r)
            for (int q = 0; q < d.y; ++q)
                for (int p = 0; p <= half; ++p) {
                    const int self_conj = (p == 0) || (2 * p == d.x);
                    const oc_complex s = spec[(size_t)p + (size_t)hx * ((size_t)q + (size_t)d.y * r)];
                    energy += (self_conj ? 1.0 : 2.0) * kernel[flat(d, p, q, r)] *
                              (s.re * s.re + s.im * s.im);
                }
    }
    return 0.5 * energy / (double)n;
}

int dro_regulariser_energy(const float* w, dreg_dims3 d, int n, double* out) {
    const size_t nv = nvox(d);
    double* kernel = (double*)malloc(sizeof(double) * nv);
    int st = dro_laplacian_symbol(n, d, kernel);
    if (st) {
        free(kernel);
        return st;
    }
    oc_fft3* fft = oc_fft3_create(d.x, d.y, d.z);
    double* real = (double*)malloc(sizeof(double) * nv);
    oc_complex* spec = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(d.x / 2 + 1) * d.y * d.z);
    *out = spectral_energy(w, d, kernel, fft, real, spec);
    free(spec);
    free(real);
    oc_fft3_destroy(fft);
    free(kernel);
    return DREG_OK;
}

/* ---- admm.cpp:23-42 (v_update_l1_into) -------------------------------------- */
static void v_update_l1_into(const float* target, const float* warped, const float* grad,
                             const float* w_hat, const float* b_hat, size_t n, double theta,
                             double eps, float* out) {
    for (size_t i = 0; i < n; ++i) {
        const double gx = grad[3 * i], gy = grad[3 * i + 1], gz = grad[3 * i + 2];
        const double ux = (double)w_hat[3 * i] - (double)b_hat[3 * i];
        const double uy = (double)w_hat[3 * i + 1] - (double)b_hat[3 * i + 1];
        const double uz = (double)w_hat[3 * i + 2] - (double)b_hat[3 * i + 2];
        const double residual = (gx * ux + gy * uy + gz * uz) + (double)warped[i] - (double)target[i];
        const double zhat = theta * residual / ((gx * gx + gy * gy + gz * gz) + eps);
        const double clip = zhat / fmax(fabs(zhat), 1.0);
        const double s = clip / theta;
        out[3 * i] = (float)(ux - gx * s);
        out[3 * i + 1] = (float)(uy - gy * s);
        out[3 * i + 2] = (float)(uz - gz * s);
    }
}

/* ---- admm.cpp:45-63 (v_update_l2_into) -------------------------------------- */
static void v_update_l2_into(const float* target, const float* warped, const float* grad,
                             const float* w_hat, const float* b_hat, size_t n, double theta,
                             float* out) {
    for (size_t i = 0; i < n; ++i) {
        const double gx = grad[3 * i], gy = grad[3 * i + 1], gz = grad[3 * i + 2];
        const double ux = (double)w_hat[3 * i] - (double)b_hat[3 * i];
        const double uy = (double)w_hat[3 * i + 1] - (double)b_hat[3 * i + 1];
        const double uz = (double)w_hat[3 * i + 2] - (double)b_hat[3 * i + 2];
        const double diff = (double)warped[i] - (double)target[i];
        const double rx = ux * theta - gx * diff;
        const double ry = uy * theta - gy * diff;
        const double rz = uz * theta - gz * diff;
        const double gg = gx * gx + gy * gy + gz * gz;
        const double it = 1.0 / theta;
        const double s = (gx * rx + gy * ry + gz * rz) / (theta * (theta + gg));
        out[3 * i] = (float)(rx * it - gx * s);
        out[3 * i + 1] = (float)(ry * it - gy * s);
        out[3 * i + 2] = (float)(rz * it - gz * s);
    }
}

int dro_v_update(const float* target, const float* warped, const float* grad,
                 const float* w_hat, const float* b_hat, dreg_dims3 d,
                 const dreg_solver_cfg* c, float* out) {
    if (!dims_ok(d)) return fail(DREG_INVALID_ARGUMENT, "volume dims must be positive");
    if (c->data_term == 1) {
        if (!(c->epsilon > 0.0)) return fail(DREG_INVALID_ARGUMENT, "v_update_l1: epsilon must be > 0");
        v_update_l1_into(target, warped, grad, w_hat, b_hat, nvox(d), c->theta, c->epsilon, out);
    } else {
        v_update_l2_into(target, warped, grad, w_hat, b_hat, nvox(d), c->theta, out);
    }
    return DREG_OK;
}

/* ---- admm.cpp:66-101 (w_update_into) ---------------------------------------- */
static void w_update_into(const float* v, const float* b_hat, dreg_dims3 d, const double* kernel,
                          double lambda, double theta, oc_fft3* fft, double* real,
                          oc_complex* spec, float* out) {
    const size_t n = nvox(d);
    const double inv_count = 1.0 / (double)n;
    const int half = d.x / 2;
    for (int c = 0; c < 3; ++c) {
        for (size_t i = 0; i < n; ++i)
            real[i] = (double)v[3 * i + (size_t)c] + (double)b_hat[3 * i + (size_t)c];
        oc_fft3_r2c(fft, real, spec);
        size_t b = 0;
        for (int r = 0; r < d.z; ++r)
            for (int q = 0; q < d.y; ++q) {
                const double* krow = kernel + (size_t)d.x * ((size_t)q + (size_t)d.y * r);
                for (int p = 0; p <= half; ++p, ++b) {
                    const double m = theta / (lambda * krow[p] + theta) * inv_count;
                    spec[b].re *= m;
                    spec[b].im *= m;
                }
            }
        oc_fft3_c2r(fft, spec, real);
        for (size_t i = 0; i < n; ++i) out[3 * i + (size_t)c] = (float)real[i];
    }
}

int dro_w_update(const float* v, const float* b_hat, dreg_dims3 d, const dreg_solver_cfg* c,
                 float* out) {
    const size_t n = nvox(d);
    double* kernel = (double*)malloc(sizeof(double) * n);
    int st = dro_laplacian_symbol(c->order, d, kernel);
    if (st) {
        free(kernel);
        return st;
    }
    oc_fft3* fft = oc_fft3_create(d.x, d.y, d.z);
    double* real = (double*)malloc(sizeof(double) * n);
    oc_complex* spec = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(d.x / 2 + 1) * d.y * d.z);
    w_update_into(v, b_hat, d, kernel, c->lambda, c->theta, fft, real, spec, out);
    free(spec);
    free(real);
    oc_fft3_destroy(fft);
    free(kernel);
    return DREG_OK;
}

/* ---- admm.cpp:239-250 ------------------------------------------------------- */
static double data_term_value(const float* target, const float* warped, const float* grad,
                              const float* v, size_t n, int s) {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double rho = ((double)grad[3 * i] * v[3 * i] + (double)grad[3 * i + 1] * v[3 * i + 1] +
                            (double)grad[3 * i + 2] * v[3 * i + 2]) +
                           (double)warped[i] - (double)target[i];
        sum += (s == 1) ? fabs(rho) : 0.5 * rho * rho;
    }
    return sum;
}

int dro_data_term_value(const float* target, const float* warped, const float* grad,
                        const float* v, dreg_dims3 d, int s, double* out) {
    *out = data_term_value(target, warped, grad, v, nvox(d), s);
    return DREG_OK;
}

/* ---- admm.cpp:130-139 (extrapolate), :142-153 (dual_update),
 *      :155-170 (mean_abs_difference, l2_difference) --------------------------- */
static void extrapolate(const float* a, const float* b, double scale, float* out, size_t n) {
    for (size_t k = 0; k < n; ++k) {
        const double av = a[k];
        out[k] = (float)(av + scale * (av - (double)b[k]));
    }
}
static void dual_update(const float* b_hat, const float* v, const float* w, float* out, size_t n) {
    for (size_t k = 0; k < n; ++k) out[k] = (float)((double)b_hat[k] + (double)v[k] - (double)w[k]);
}
static double mean_abs_difference(const float* a, const float* b, size_t n) {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) sum += fabs((double)a[i] - (double)b[i]);
    return sum / (double)n;
}
static double l2_difference(const float* a, const float* b, size_t n) {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double dd = (double)a[i] - (double)b[i];
        sum += dd * dd;
    }
    return sqrt(sum);
}

/* ---- volume.cpp:123-159 (image_gradient) ------------------------------------ */
static double diff1(const float* f, size_t i, int pos, int dim, size_t stride) {
    if (pos == 0) return (double)f[i + stride] - (double)f[i];
    if (pos == dim - 1) return (double)f[i] - (double)f[i - stride];
    return 0.5 * ((double)f[i + stride] - (double)f[i - stride]);
}

int dro_image_gradient(const float* img, dreg_dims3 d, float* out) {
    if (d.x < 2 || d.y < 2 || d.z < 2)
        return fail(DREG_INVALID_ARGUMENT, "image_gradient: every axis must have size >= 2");
    const size_t sy = (size_t)d.x, sz = (size_t)d.x * d.y;
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y) {
            size_t i = flat(d, 0, y, z);
            for (int x = 0; x < d.x; ++x, ++i) {
                out[3 * i] = (float)diff1(img, i, x, d.x, 1);
                out[3 * i + 1] = (float)diff1(img, i, y, d.y, sy);
                out[3 * i + 2] = (float)diff1(img, i, z, d.z, sz);
            }
        }
    return DREG_OK;
}

/* ---- admm.cpp:252-314 (solve_velocity) ------------------------------------- */
int dro_solve_velocity(const float* target, const float* warped, dreg_dims3 d,
                       const dreg_solver_cfg* c, float* v_out, dreg_solver_diag* diag) {
    int st = dro_validate(c);
    if (st) return st;
    if (!dims_ok(d)) return fail(DREG_INVALID_ARGUMENT, "volume dims must be positive");
    const size_t n = nvox(d), n3 = 3 * n;
    float* grad = (float*)malloc(sizeof(float) * n3);
    st = dro_image_gradient(warped, d, grad);
    if (st) {
        free(grad);
        return st;
    }
    double* kernel = (double*)malloc(sizeof(double) * n);
    st = dro_laplacian_symbol(c->order, d, kernel);
    if (st) {
        free(grad);
        free(kernel);
        return st;
    }
    oc_fft3* fft = oc_fft3_create(d.x, d.y, d.z);
    double* real = (double*)malloc(sizeof(double) * n);
    oc_complex* spec = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(d.x / 2 + 1) * d.y * d.z);
    float* buf = (float*)calloc(8 * n3, sizeof(float));
    float* v = buf;
    float* v_next = buf + n3;
    float* w = buf + 2 * n3;
    float* w_prev = buf + 3 * n3;
    float* b = buf + 4 * n3;
    float* b_prev = buf + 5 * n3;
    float* w_hat = buf + 6 * n3;
    float* b_hat = buf + 7 * n3;
    double alpha = 1.0;
    int iterations = 0, converged = 0;
    double final_change = 0.0;
    for (int k = 0; k < c->max_iters; ++k) {
        if (c->data_term == 1)
            v_update_l1_into(target, warped, grad, w_hat, b_hat, n, c->theta, c->epsilon, v_next);
        else
            v_update_l2_into(target, warped, grad, w_hat, b_hat, n, c->theta, v_next);
        const double change = mean_abs_difference(v_next, v, n3);
        float* t = v; v = v_next; v_next = t;

        w_update_into(v, b_hat, d, kernel, c->lambda, c->theta, fft, real, spec, w);
        dual_update(b_hat, v, w, b, n3);
        if (diag && diag->constraint_residual) diag->constraint_residual[k] = l2_difference(v, w, n3);
        if (c->log_objective && diag && diag->objective)
            diag->objective[k] = data_term_value(target, warped, grad, v, n, c->data_term) +
                                 c->lambda * spectral_energy(v, d, kernel, fft, real, spec);

        const double alpha_next = dro_nesterov_next_alpha(alpha);
        const double coef = c->accelerate ? (alpha - 1.0) / alpha_next : 0.0;
        extrapolate(w, w_prev, coef, w_hat, n3);
        extrapolate(b, b_prev, coef, b_hat, n3);
        t = w_prev; w_prev = w; w = t;
        t = b_prev; b_prev = b; b = t;
        alpha = alpha_next;

        iterations = k + 1;
        final_change = change;
        if (change <= c->tol) {
            converged = 1;
            break;
        }
    }
    int finite = 1;
    for (size_t i = 0; i < n3; ++i) finite &= isfinite(v[i]) ? 1 : 0;
    memcpy(v_out, v, sizeof(float) * n3);
    if (diag) {
        diag->iterations = iterations;
        diag->final_change = final_change;
        diag->converged = converged;
    }
    free(buf);
    free(spec);
    free(real);
    oc_fft3_destroy(fft);
    free(kernel);
    free(grad);
    if (!finite) return fail(DREG_NUMERIC, "solve_velocity: velocity field contains non-finite values");
    return DREG_OK;
}

/* ---- volume.cpp:36-41 (axis_sample), :55-99 (trilinear_sample) --------------- */
typedef struct {
    int lo, hi;
    double frac;
} axs;

static axs axis_sample(double coord, int dim) {
    const double hi = (double)(dim - 1);
    const double c = coord < 0.0 ? 0.0 : (hi < coord ? hi : coord); /* std::clamp */
    const double f = floor(c);
    axs a;
    a.lo = (int)f;
    a.hi = a.lo + 1 < dim - 1 ? a.lo + 1 : dim - 1;
    a.frac = c - f;
    return a;
}

static double trilinear_scalar(const float* vol, dreg_dims3 d, double px, double py, double pz) {
    const axs ax = axis_sample(px, d.x), ay = axis_sample(py, d.y), az = axis_sample(pz, d.z);
    const double c000 = vol[flat(d, ax.lo, ay.lo, az.lo)];
    const double c100 = vol[flat(d, ax.hi, ay.lo, az.lo)];
    const double c010 = vol[flat(d, ax.lo, ay.hi, az.lo)];
    const double c110 = vol[flat(d, ax.hi, ay.hi, az.lo)];
    const double c001 = vol[flat(d, ax.lo, ay.lo, az.hi)];
    const double c101 = vol[flat(d, ax.hi, ay.lo, az.hi)];
    const double c011 = vol[flat(d, ax.lo, ay.hi, az.hi)];
    const double c111 = vol[flat(d, ax.hi, ay.hi, az.hi)];
    const double c00 = c000 + (c100 - c000) * ax.frac;
    const double c10 = c010 + (c110 - c010) * ax.frac;
    const double c01 = c001 + (c101 - c001) * ax.frac;
    const double c11 = c011 + (c111 - c011) * ax.frac;
    const double c0 = c00 + (c10 - c00) * ay.frac;
    const double c1 = c01 + (c11 - c01) * ay.frac;
    return c0 + (c1 - c0) * az.frac;
}

static void trilinear_vec(const float* f, dreg_dims3 d, double px, double py, double pz,
                          double out[3]) {
    const axs ax = axis_sample(px, d.x), ay = axis_sample(py, d.y), az = axis_sample(pz, d.z);
    const size_t i000 = 3 * flat(d, ax.lo, ay.lo, az.lo), i100 = 3 * flat(d, ax.hi, ay.lo, az.lo);
    const size_t i010 = 3 * flat(d, ax.lo, ay.hi, az.lo), i110 = 3 * flat(d, ax.hi, ay.hi, az.lo);
    const size_t i001 = 3 * flat(d, ax.lo, ay.lo, az.hi), i101 = 3 * flat(d, ax.hi, ay.lo, az.hi);
    const size_t i011 = 3 * flat(d, ax.lo, ay.hi, az.hi), i111 = 3 * flat(d, ax.hi, ay.hi, az.hi);
    for (int c = 0; c < 3; ++c) {
        const double c000 = f[i000 + c], c100 = f[i100 + c], c010 = f[i010 + c], c110 = f[i110 + c];
        const double c001 = f[i001 + c], c101 = f[i101 + c], c011 = f[i011 + c], c111 = f[i111 + c];
        const double c00 = c000 + (c100 - c000) * ax.frac;
        const double c10 = c010 + (c110 - c010) * ax.frac;
        const double c01 = c001 + (c101 - c001) * ax.frac;
        const double c11 = c011 + (c111 - c011) * ax.frac;
        const double c0 = c00 + (c10 - c00) * ay.frac;
        const double c1 = c01 + (c11 - c01) * ay.frac;
        out[c] = c0 + (c1 - c0) * az.frac;
    }
}

/* volume.hpp:107,110: trilinear_sample at n points (x, y, z); ncomp 1 = scalar volume,
 * 3 = AoS vector field */
int dro_trilinear_sample(const float* f, int ncomp, dreg_dims3 d, const double* pts, int64_t n, double* out) {
    if ((ncomp != 1 && ncomp != 3) || n < 0) return fail(DREG_INVALID_ARGUMENT, "trilinear_sample: bad arguments");
    for (int64_t i = 0; i < n; ++i) {
        if (ncomp == 1) out[i] = trilinear_scalar(f, d, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        else trilinear_vec(f, d, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], out + 3 * i);
    }
    return DREG_OK;
}

/* ---- volume.cpp:101-121 (warp_image) ---------------------------------------- */
int dro_warp_image(const float* img, const float* disp, dreg_dims3 d, float* out) {
    if (!dims_ok(d)) return fail(DREG_INVALID_ARGUMENT, "volume dims must be positive");
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y) {
            size_t i = flat(d, 0, y, z);
            for (int x = 0; x < d.x; ++x, ++i)
                out[i] = (float)trilinear_scalar(img, d, x + (double)disp[3 * i], y + (double)disp[3 * i + 1],
                                                 z + (double)disp[3 * i + 2]);
        }
    return DREG_OK;
}

/* ---- volume.cpp:161-181 (compose_deformation) ------------------------------- */
int dro_compose_deformation(const float* disp, const float* v, dreg_dims3 d, float* out) {
    if (!dims_ok(d)) return fail(DREG_INVALID_ARGUMENT, "volume dims must be positive");
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y) {
            size_t i = flat(d, 0, y, z);
            for (int x = 0; x < d.x; ++x, ++i) {
                const double sx = v[3 * i], sy = v[3 * i + 1], sz = v[3 * i + 2];
                double s[3];
                trilinear_vec(disp, d, x + sx, y + sy, z + sz, s);
                out[3 * i] = (float)(sx + s[0]);
                out[3 * i + 1] = (float)(sy + s[1]);
                out[3 * i + 2] = (float)(sz + s[2]);
            }
        }
    return DREG_OK;
}

/* ---- volume.cpp:183-230 (jacobian_determinant), metrics.cpp:211-228 ---------- */
int dro_jacobian(const float* u, dreg_dims3 d, float* det_out, dreg_jacobian_stats* st) {
    if (d.x < 3 || d.y < 3 || d.z < 3)
        return fail(DREG_INVALID_ARGUMENT, "jacobian_determinant: every axis must have size >= 3");
    const size_t n = nvox(d);
    float* det = det_out ? det_out : (float*)malloc(sizeof(float) * n);
    const size_t sx = 3, sy = 3 * (size_t)d.x, sz = 3 * (size_t)d.x * d.y;
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y) {
            size_t vox = flat(d, 0, y, z);
            for (int x = 0; x < d.x; ++x, ++vox) {
                const size_t i = 3 * vox;
                double j[3][3];
                for (int c = 0; c < 3; ++c) {
                    j[c][0] = diff1(u, i + c, x, d.x, sx) + (c == 0 ? 1.0 : 0.0);
                    j[c][1] = diff1(u, i + c, y, d.y, sy) + (c == 1 ? 1.0 : 0.0);
                    j[c][2] = diff1(u, i + c, z, d.z, sz) + (c == 2 ? 1.0 : 0.0);
                }
                const double value = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                                     j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                                     j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
                det[vox] = (float)value;
            }
        }
    if (st) {
        int64_t nonpos = 0, interior = 0;
        double min_det = DBL_MAX;
        for (int z = 1; z < d.z - 1; ++z)
            for (int y = 1; y < d.y - 1; ++y)
                for (int x = 1; x < d.x - 1; ++x) {
                    const double value = det[flat(d, x, y, z)];
                    if (value < min_det) min_det = value;
                    nonpos += value <= 0.0;
                    ++interior;
                }
        st->nonpositive = nonpos;
        st->interior = interior;
        st->pct_nonpositive = 100.0 * (double)nonpos / (double)interior;
        st->min_det = min_det;
    }
    if (!det_out) free(det);
    return DREG_OK;
}

/* ---- registration.cpp:154-178 (normalize_intensity_pair) -------------------- */
int dro_normalize_intensity_pair(const float* a, const float* b, dreg_dims3 d, float* oa,
                                 float* ob) {
    const size_t n = nvox(d);
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (size_t i = 0; i < n; ++i) {
        lo = a[i] < lo ? a[i] : lo; /* std::min(lo, v) keeps lo unless v < lo */
        hi = hi < a[i] ? a[i] : hi;
    }
    for (size_t i = 0; i < n; ++i) {
        lo = b[i] < lo ? b[i] : lo;
        hi = hi < b[i] ? b[i] : hi;
    }
    const double range = (double)hi - (double)lo;
    const double scale = range > 0.0 ? 1.0 / range : 0.0;
    for (size_t i = 0; i < n; ++i) oa[i] = (float)(((double)a[i] - lo) * scale);
    for (size_t i = 0; i < n; ++i) ob[i] = (float)(((double)b[i] - lo) * scale);
    return DREG_OK;
}

/* ---- registration.cpp:32-58 (smooth_axis), :141-143 (binomial_smooth) -------- */
static void smooth_axis(const float* f, dreg_dims3 d, int axis, float* out) {
    const int extent = axis == 0 ? d.x : (axis == 1 ? d.y : d.z);
    const size_t stride = axis == 0 ? 1 : (axis == 1 ? (size_t)d.x : (size_t)d.x * d.y);
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y) {
            size_t i = flat(d, 0, y, z);
            for (int x = 0; x < d.x; ++x, ++i) {
                const int pos = axis == 0 ? x : (axis == 1 ? y : z);
                const double lo = f[pos > 0 ? i - stride : i];
                const double hi = f[pos < extent - 1 ? i + stride : i];
                out[i] = (float)(0.25 * (lo + hi) + 0.5 * f[i]);
            }
        }
}

int dro_binomial_smooth(const float* img, dreg_dims3 d, float* out) {
    const size_t n = nvox(d);
    float* t1 = (float*)malloc(sizeof(float) * n);
    float* t2 = (float*)malloc(sizeof(float) * n);
    smooth_axis(img, d, 0, t1);
    smooth_axis(t1, d, 1, t2);
    smooth_axis(t2, d, 2, out);
    free(t1);
    free(t2);
    return DREG_OK;
}

/* ---- registration.cpp:145-152 (mean_sad) ------------------------------------ */
static double mean_sad(const float* a, const float* b, size_t n) {
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) sum += fabs((double)a[i] - (double)b[i]);
    return sum / (double)n;
}

int dro_mean_sad(const float* a, const float* b, dreg_dims3 d, double* out) {
    *out = mean_sad(a, b, nvox(d));
    return DREG_OK;
}

/* ---- registration.cpp:85-112 (downsample) ----------------------------------- */
int dro_downsample(const float* img, dreg_dims3 d, float* out) {
    const dreg_dims3 o = {(d.x + 1) / 2, (d.y + 1) / 2, (d.z + 1) / 2};
    for (int z = 0; z < o.z; ++z)
        for (int y = 0; y < o.y; ++y)
            for (int x = 0; x < o.x; ++x) {
                double sum = 0.0;
                for (int dz = 0; dz < 2; ++dz)
                    for (int dy = 0; dy < 2; ++dy)
                        for (int dx = 0; dx < 2; ++dx) {
                            const int xx = 2 * x + dx < d.x - 1 ? 2 * x + dx : d.x - 1;
                            const int yy = 2 * y + dy < d.y - 1 ? 2 * y + dy : d.y - 1;
                            const int zz = 2 * z + dz < d.z - 1 ? 2 * z + dz : d.z - 1;
                            sum += img[flat(d, xx, yy, zz)];
                        }
                out[flat(o, x, y, z)] = (float)(sum / 8.0);
            }
    return DREG_OK;
}

/* ---- registration.cpp:24-30 (source_coord), :114-135 (upsample_velocity) ----- */
static double source_coord(int i, int te, int se) {
    if (te <= 1) return 0.0;
    return (double)i * (double)(se - 1) / (double)(te - 1);
}

int dro_upsample_velocity(const float* v, dreg_dims3 src, dreg_dims3 dst, float* out) {
    if (dst.x < src.x || dst.y < src.y || dst.z < src.z)
        return fail(DREG_INVALID_ARGUMENT, "upsample_velocity: target dims smaller than source");
    for (int z = 0; z < dst.z; ++z)
        for (int y = 0; y < dst.y; ++y) {
            size_t i = flat(dst, 0, y, z);
            for (int x = 0; x < dst.x; ++x, ++i) {
                double s[3];
                trilinear_vec(v, src, source_coord(x, dst.x, src.x), source_coord(y, dst.y, src.y),
                              source_coord(z, dst.z, src.z), s);
                out[3 * i] = (float)(2.0 * s[0]);
                out[3 * i + 1] = (float)(2.0 * s[1]);
                out[3 * i + 2] = (float)(2.0 * s[2]);
            }
        }
    return DREG_OK;
}

/* ---- registration.cpp:180-283 (register_pair) ------------------------------- */
int dro_register_pair(const float* target, const float* source, dreg_dims3 d,
                      dreg_spacing3 sp, const dreg_reg_cfg* c, float* phi_out,
                      float* warped_out, dreg_pair_result* res) {
    (void)sp;
    if (!dims_ok(d)) return fail(DREG_INVALID_ARGUMENT, "volume dims must be positive");
    int st = dro_validate(&c->solver);
    if (st) return st;
    if (c->levels < 1) return fail(DREG_INVALID_ARGUMENT, "register_pair: levels must be >= 1");
    if (c->levels > DREG_MAX_LEVELS)
        return fail(DREG_INVALID_ARGUMENT, "register_pair: per-level caps must list one entry per level");
    if (!(c->warp_improvement_threshold > 0.0 && c->warp_improvement_threshold < 1.0))
        return fail(DREG_INVALID_ARGUMENT, "register_pair: warp improvement threshold must be in (0,1)");
    const int min_extent = 4 << (c->levels - 1);
    if (d.x < min_extent || d.y < min_extent || d.z < min_extent)
        return fail(DREG_INVALID_ARGUMENT, "register_pair: dims too small for the level count");
    const size_t n = nvox(d);
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(target[i]) || !isfinite(source[i]))
            return fail(DREG_NUMERIC, "register_pair: input volumes contain non-finite values");

    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const int L = c->levels;
    dreg_dims3 dims[DREG_MAX_LEVELS];
    float* pt[DREG_MAX_LEVELS];
    float* ps[DREG_MAX_LEVELS];
    dims[L - 1] = d;
    pt[L - 1] = (float*)malloc(sizeof(float) * n);
    ps[L - 1] = (float*)malloc(sizeof(float) * n);
    dro_normalize_intensity_pair(target, source, d, pt[L - 1], ps[L - 1]);
    for (int l = L - 1; l > 0; --l) {
        const dreg_dims3 o = {(dims[l].x + 1) / 2, (dims[l].y + 1) / 2, (dims[l].z + 1) / 2};
        dims[l - 1] = o;
        pt[l - 1] = (float*)malloc(sizeof(float) * nvox(o));
        ps[l - 1] = (float*)malloc(sizeof(float) * nvox(o));
        dro_downsample(pt[l], dims[l], pt[l - 1]);
        dro_downsample(ps[l], dims[l], ps[l - 1]);
    }
    if (c->smooth_levels) {
        for (int l = 0; l < L; ++l) {
            float* t = (float*)malloc(sizeof(float) * nvox(dims[l]));
            dro_binomial_smooth(pt[l], dims[l], t);
            free(pt[l]);
            pt[l] = t;
            t = (float*)malloc(sizeof(float) * nvox(dims[l]));
            dro_binomial_smooth(ps[l], dims[l], t);
            free(ps[l]);
            ps[l] = t;
        }
    }
    if (res) {
        memset(res, 0, sizeof *res);
        res->levels = L;
    }
    float* phi = NULL;
    dreg_dims3 phi_dims = dims[0];
    int velocity_count = 0, solves = 0;
    st = DREG_OK;
    for (int l = 0; l < L && st == DREG_OK; ++l) {
        const dreg_dims3 dl = dims[l];
        const size_t nl = nvox(dl);
        if (l == 0) {
            phi = (float*)calloc(3 * nl, sizeof(float));
        } else {
            float* up = (float*)malloc(sizeof(float) * 3 * nl);
            dro_upsample_velocity(phi, phi_dims, dl, up);
            free(phi);
            phi = up;
        }
        phi_dims = dl;
        dreg_solver_cfg solver = c->solver;
        solver.max_iters = c->max_admm_iters_per_level[l];
        dreg_level_log* lg = res ? &res->per_level[l] : NULL;
        if (lg) lg->dims = dl;
        float* warped = (float*)malloc(sizeof(float) * nl);
        float* warped_c = (float*)malloc(sizeof(float) * nl);
        float* phi_c = (float*)malloc(sizeof(float) * 3 * nl);
        float* v = (float*)malloc(sizeof(float) * 3 * nl);
        dro_warp_image(ps[l], phi, dl, warped);
        double sad_prev = mean_sad(warped, pt[l], nl);
        if (lg) lg->mean_sad[0] = sad_prev;
        for (int w = 0; w < c->max_warps_per_level[l]; ++w) {
            dreg_solver_diag diag = {0, 0.0, 0, NULL, NULL};
            st = dro_solve_velocity(pt[l], warped, dl, &solver, v, &diag);
            if (st) break;
            solves += 1;
            dro_compose_deformation(phi, v, dl, phi_c);
            dro_warp_image(ps[l], phi_c, dl, warped_c);
            const double sad_new = mean_sad(warped_c, pt[l], nl);
            if (sad_new > sad_prev) break;
            float* t = phi; phi = phi_c; phi_c = t;
            t = warped; warped = warped_c; warped_c = t;
            if (lg && lg->warps < DREG_MAX_WARPS) {
                lg->mean_sad[lg->warps + 1] = sad_new;
                lg->solver_iterations[lg->warps] = diag.iterations;
            }
            if (lg) lg->warps += 1;
            velocity_count += 1;
            const double improvement = (sad_prev - sad_new) / (sad_prev > DBL_MIN ? sad_prev : DBL_MIN);
            sad_prev = sad_new;
            if (improvement < c->warp_improvement_threshold) break;
        }
        free(warped);
        free(warped_c);
        free(phi_c);
        free(v);
    }
    for (int l = 0; l < L; ++l) {
        free(pt[l]);
        free(ps[l]);
    }
    if (st == DREG_OK) {
        for (size_t i = 0; i < 3 * n; ++i)
            if (!isfinite(phi[i])) {
                st = fail(DREG_NUMERIC, "register_pair: deformation contains non-finite values");
                break;
            }
    }
    if (st == DREG_OK) {
        if (phi_out) memcpy(phi_out, phi, sizeof(float) * 3 * n);
        if (warped_out) dro_warp_image(source, phi, d, warped_out);
    }
    free(phi);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (res) {
        res->status = st;
        res->velocity_count = velocity_count;
        res->solves = solves;
        res->elapsed_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    }
    return st;
}
