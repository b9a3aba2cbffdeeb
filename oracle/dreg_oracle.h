/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the checker.
 *
 * Plain-C restatement of the reference `dreg` hot path (arXiv 2109.12688 reference,
 * /root/reference/proj/core), function by function, each citing the reference
 * file:line it follows.  Same arithmetic as the reference: fp32 storage, fp64
 * per-voxel math, fp64 FFT (oracle/fft_core.c standing in for FFTW3).
 * Parity pin: tests/test_oracle_pin.py checks every entry point against the
 * unmodified reference compiled into oracle/_ref/ (bit-exact where the reference
 * is deterministic) and against the golden fixtures in tests/golden/.
 *
 * Signatures match oracle/ref_capi.cpp with the prefix dro_ instead of ref_.
 * Vector fields are AoS (vx,vy,vz) per voxel like the reference's VectorField.
 */
#ifndef DREG_ORACLE_H
#define DREG_ORACLE_H

#include "dreg_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* dro_last_error(void);
double dro_nesterov_next_alpha(double a);
int dro_validate(const dreg_solver_cfg* c);
int dro_make_registration_config(int profile, const dreg_solver_cfg* c, int levels,
                                 dreg_reg_cfg* out);
int dro_laplacian_symbol(int n, dreg_dims3 d, double* out);
int dro_regulariser_energy(const float* w, dreg_dims3 d, int n, double* out);
int dro_v_update(const float* target, const float* warped, const float* grad,
                 const float* w_hat, const float* b_hat, dreg_dims3 d,
                 const dreg_solver_cfg* c, float* out);
int dro_w_update(const float* v, const float* b_hat, dreg_dims3 d, const dreg_solver_cfg* c,
                 float* out);
int dro_trilinear_sample(const float* f, int ncomp, dreg_dims3 d, const double* pts, int64_t n, double* out);
int dro_data_term_value(const float* target, const float* warped, const float* grad,
                        const float* v, dreg_dims3 d, int s, double* out);
int dro_solve_velocity(const float* target, const float* warped, dreg_dims3 d,
                       const dreg_solver_cfg* c, float* v_out, dreg_solver_diag* diag);
int dro_warp_image(const float* img, const float* disp, dreg_dims3 d, float* out);
int dro_image_gradient(const float* img, dreg_dims3 d, float* out);
int dro_compose_deformation(const float* disp, const float* v, dreg_dims3 d, float* out);
int dro_jacobian(const float* disp, dreg_dims3 d, float* det_out, dreg_jacobian_stats* st);
int dro_normalize_intensity_pair(const float* a, const float* b, dreg_dims3 d, float* oa,
                                 float* ob);
int dro_binomial_smooth(const float* img, dreg_dims3 d, float* out);
int dro_mean_sad(const float* a, const float* b, dreg_dims3 d, double* out);
int dro_downsample(const float* img, dreg_dims3 d, float* out);
int dro_upsample_velocity(const float* v, dreg_dims3 src, dreg_dims3 dst, float* out);
int dro_register_pair(const float* target, const float* source, dreg_dims3 d,
                      dreg_spacing3 sp, const dreg_reg_cfg* c, float* phi_out,
                      float* warped_out, dreg_pair_result* res);

#ifdef __cplusplus
}
#endif

#endif
