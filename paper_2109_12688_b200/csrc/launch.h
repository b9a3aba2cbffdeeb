// Host-side launch interface between the engine (engine.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

// Work-skipping switches exist only in experiment builds (make EXPERIMENTS=1); the
// release library has no way to skip part of an iteration.
#ifdef DREG_EXPERIMENTS
#define DREG_SKIP(a, bit) (((a).dbg_skip & (bit)) != 0)
#else
#define DREG_SKIP(a, bit) false
#endif

namespace dregb {

// X_FIRST/SECOND/GENERAL: ADMM iteration k = 0 / 1 / >= 2; X_TAIL: w and residual of the
// last iteration only (diagnostics); X_FWD: r2c of V (+ BH when add_bh) into S;
// X_INV: c2r of S into WP.
// X_SS / X_SSN: spectral-state iteration (k >= 1; see plane_fast.cuh MODE 2): the staged
// spectrum is w_hat - b_hat itself, the tile does c2r -> v-update -> r2c of v and streams
// only v, grad and diff; X_SSN neither reads v (no change norm: tol = 0) nor writes it
// before the last iteration.
enum XMode { X_FIRST = 0, X_SECOND = 1, X_GENERAL = 2, X_TAIL = 3, X_FWD = 4, X_INV = 5, X_SS = 6, X_SSN = 7 };

struct XArgs {
    Fields F;
    AxisPlan px;        // line plan of length M/2 (M even) or M (M odd)
    const float2* twx;  // W_L^e, e in [0, L)
    const float2* xtw;  // W_M^k, k in [0, hx]
    const int* xpos;    // position of frequency k in the digit-reversed line, k in [0, L)
    SolverParams sp;
    double coef;        // Nesterov coefficient c_{k-1} (admm.cpp:294-295)
    double coef_prev;   // c_{k-2}: b_hat_{k-1} = b_{k-1} + c_{k-2} (b_{k-1} - b_{k-2}) is re-formed, not stored
    int k;              // iteration index
    int TL;             // x-lines per CTA
    int PM;             // shared-memory line pitch (complex, odd)
    int odd;            // M odd
    int add_bh;         // X_FWD: transform V + BH instead of V
    int vec;            // point-wise vector width (1, 2 or 4; 4/2 need M % 4 / M % 2 == 0)
    int prefetch;       // L2 bulk prefetch of the tile's field rows at kernel start
    int f64;            // fp64 point-wise arithmetic in the generic x-pass (DREG_F64)
    int minb;           // x-pass launch-bounds variant: min CTAs per SM (3 or 4)
    int fast_x;         // use the specialised x-pass (xpass_fast.cu) for M in {64, 128, 256}
    int fx_variant;     // point-wise loop variant of the specialised x-pass: 10 * VEC + unroll (22 default)
    int precise;        // fp64 x-FFT arithmetic (long solves; see plane_split.cu)
    const double2* twx64;
    const double2* xtw64;
#ifdef DREG_EXPERIMENTS
    int dbg_skip;       // timing experiments only (DREG_DBG_SKIP): 1 = skip x-FFTs, 2 = skip point-wise, 4 = skip spectrum I/O
#endif
    FastDiv fd_lines;   // divide by 3 * TL
    int pipe;           // warp-specialised persistent x-pass for X_GENERAL, M in {64, 128} (DREG_PIPE: 0 off; default on)
    int pipe256;        // pipelined x-pass at M = 256 (two-buffer ring; DREG_PIPE256)
    int pipe_ss;        // warp split of the spectral-state x-pass (DREG_PIPE_SS)
    int ss_last;        // X_SSN: this is the solve's last iteration (v is written)
    int pipe_all;       // A/B knob (DREG_PIPE_ALL): split all pairs' tiles statically, not just the iterating ones
};

struct PArgs {
    Fields F;
    AxisPlan py, pz;
    const float2* twy;
    const float2* twz;
    const float* sx;    // [hx]  1 - cos(2 pi p / M)
    const float* sy;    // [Ny]  1 - cos(2 pi q / N) at digit-reversed positions
    const float* sz;    // [Nz]
    const float* sy_fast;  // [Ny] position table of the specialised plane kernel (radix split R1 x R2)
    const float* sz_fast;  // [Nz]
    int fast;              // 1: plane_fast_kernel, 2: plane_reg_kernel
    int precise;           // fp64 butterflies/multiplier via the split path
    const double2* twy64;
    const double2* twz64;
    const double* sx64;
    const double* sy64;
    const double* sz64;
    double lambda64, theta64, scale64;
    // precise multiplier with the reference's own arithmetic (regularizer.cpp:24-31,51-79,
    // admm.cpp:92): axis cosines cos(2 pi k / n) (cos 0 := 1) at x-frequency p and at the
    // digit-reversed y / z positions of the generic plans, and 1 / voxels
    const double* cx64;
    const double* cy64;
    const double* cz64;
    const double* cy64_fast;     // the same cosines at the cluster plane kernel's positions (precise, 128 x 128)
    const double* cz64_fast;
    double inv_count;
    float lambda, theta, scale;  // scale = theta / voxels
    float lam_n, n_f;            // lambda N / theta and N: multiplier 1 / (lam_n K + n_f)
    int pf_ahead;                // plane_reg_kernel: L2-prefetch the plane this many blocks ahead (0 = off)
    // spectral-state iteration (plane_reg_kernel MODE 2): the two 3-D Fourier-domain iterates
    const float2* U1;            // U_{j-1}                 [P][3][hx][Ny*Nz]
    float2* U0;                  // U_{j-2} in, U_j out
    float c_cur, c_prev;         // Nesterov coefficients c_{j-1}, c_{j-2}
    float inv_nf;                // 1 / voxels
    int ss_variant;              // DREG_PLANE_SS experiment knob
    int cluster;                 // 2-CTA cluster plane kernel for planes over one CTA's shared memory (DREG_CLUSTER)
    int ss_stream;               // MODE 2: streaming (evict-first) loads / stores of the plane itself (DREG_PLANE_STREAM)
    int ss_prefetch;             // L2-prefetch the plane's state iterates at CTA start (DREG_PLANE_UPF)
    int has1, has0;              // U_{j-1} exists (j >= 2); U_{j-2} enters (c_{j-2} != 0)
    int order;
    int PY;             // plane row pitch (complex, odd)
    int k;
    int need_tail;
    double* energy_out; // [P] (mode 1)
    FastDiv fd_ny, fd_nz;
};

size_t xpass_smem_bytes(int L, int hx, int TL, int PM);
size_t xpass_smem_bytes_c(int L, int hx, int TL, int PM, size_t complex_bytes);
size_t plane_smem_bytes(int Ny, int Nz, int PY);
// radix split used by the specialised plane kernel for an axis of length n (0 = unsupported)
int plane_fast_r1(int n);
bool plane_fast_supported(int Ny, int Nz);
// register-blocked plane kernel (radix-8 first stages on both axes held in registers)
bool plane_reg_supported(int Ny, int Nz);
// three-pass plane for planes above one CTA's shared memory (plane_split.cu)
bool plane_split_needed(const PArgs& a);
bool plane_cluster_eligible(const PArgs& a);
bool plane_cluster_fast_supported(int Ny, int Nz);
bool plane_cluster_fast64_supported(int Ny, int Nz);
cudaError_t launch_plane_cluster(const PArgs& a, int npairs, cudaStream_t s);
cudaError_t launch_plane_split(const PArgs& a, int mode, int npairs, cudaStream_t s);
cudaError_t launch_xpass(const XArgs& a, int mode, int npairs, cudaStream_t s);
bool xpass_fast_eligible(const XArgs& a);
bool xpass_ss_eligible(const XArgs& a);
cudaError_t launch_xpass_fast(const XArgs& a, int mode, int npairs, cudaStream_t s);
cudaError_t launch_plane(const PArgs& a, int mode, int npairs, cudaStream_t s);

// ---- field kernels (field_kernels.cu) ----
struct VolGeom {
    int M, Ny, Nz;
    long long N;
};

cudaError_t launch_state_reset(PairState* st, int npairs, cudaStream_t s);
// diag[k].objective += lambda * energy (admm.cpp:288-292)
cudaError_t launch_objective_accumulate(Fields F, const double* energy, double lambda, int k, int npairs,
                                        cudaStream_t s);
// Per-solve setup: grad(warped[cur]) and D = warped - target (volume.cpp:123-159); with
// keep_warped (l1 data term) D = warped, and the x-pass forms g.u + warped - target in
// fp64 exactly like admm.cpp:35-36.
cudaError_t launch_grad_diff(VolGeom g, const RegBuffers& R, Fields F, bool keep_warped, int npairs, cudaStream_t s);
// compose + warp + SAD + accept/revert/stop (volume.cpp:161-181, registration.cpp:250-271)
cudaError_t launch_compose_decide(VolGeom g, const RegBuffers& R, Fields F, double thr, int max_warps,
                                  int npairs, cudaStream_t s);
// normalise (registration.cpp:154-178) into R.tmpA (target) / R.tmpB (source)
cudaError_t launch_prep_normalize(VolGeom g, const RegBuffers& R, Fields F, int npairs, cudaStream_t s);
// separable [1 2 1]/4 (registration.cpp:32-58): in -> out along axis, [P][N]
cudaError_t launch_smooth_axis(VolGeom g, const float* in, float* out, int axis, int npairs, cudaStream_t s);
// initial level state: phi = 0, warped = I1, sad_prev (registration.cpp:245-247)
cudaError_t launch_level_init(VolGeom g, const RegBuffers& R, Fields F, int level, int npairs, cudaStream_t s);
// final warp of the original source + finiteness of phi (registration.cpp:275-281)
cudaError_t launch_finalize(VolGeom g, const RegBuffers& R, Fields F, int npairs, cudaStream_t s);
// Jacobian determinant + interior stats (volume.cpp:183-230, metrics.cpp:211-228)
cudaError_t launch_jacobian(VolGeom g, const float* phi_soa, float* det, double* part, double* out3,
                            unsigned int* counter, cudaStream_t s);

// building blocks on single volumes (SoA device buffers)
cudaError_t launch_warp_image(VolGeom g, const float* img, const float* disp, float* out, cudaStream_t s);
cudaError_t launch_gradient(VolGeom g, const float* img, float* out, cudaStream_t s);
cudaError_t launch_compose(VolGeom g, const float* disp, const float* v, float* out, cudaStream_t s);
cudaError_t launch_v_update(VolGeom g, int data_term, const float* target, const float* warped,
                            const float* grad, const float* w_hat, const float* b_hat, double theta,
                            double eps, float* out, cudaStream_t s);
cudaError_t launch_sad(VolGeom g, const float* a, const float* b, double* part, double* out,
                       unsigned int* counter, cudaStream_t s);
cudaError_t launch_minmax_normalize(VolGeom g, const float* a, const float* b, float* oa, float* ob,
                                    float* part, unsigned int* counter, cudaStream_t s);
cudaError_t launch_downsample(VolGeom src, VolGeom dst, const float* in, float* out, cudaStream_t s);
// pyramid (registration.cpp:208-247): batched downsample of target+source, level transition
cudaError_t launch_pyr_down(VolGeom src, VolGeom dst, const float* ta, const float* sa, float* tb, float* sb,
                            int npairs, cudaStream_t s);
cudaError_t launch_level_up(VolGeom src, VolGeom dst, const RegBuffers& Rs, const RegBuffers& Rd, Fields F, int level,
                            int npairs, cudaStream_t s);
cudaError_t launch_upsample(VolGeom src, VolGeom dst, const float* in, float* out, int ncomp,
                            cudaStream_t s);
// ---- label metrics (metrics_kernels.cu) ----
cudaError_t launch_warp_labels(VolGeom g, const uint16_t* lbl, const float* disp_aos, uint16_t* out, cudaStream_t s);
cudaError_t launch_label_counts(VolGeom g, const uint16_t* a, const uint16_t* b, const int* labels, int n_labels,
                                unsigned long long* counts, cudaStream_t s);
size_t hausdorff_scratch_doubles(VolGeom g, int ctas);
size_t hausdorff_scratch_ints(VolGeom g, int ctas);
cudaError_t launch_hausdorff_slices(VolGeom g, const uint16_t* a, const uint16_t* b, const int* labels, int n_labels,
                                    double sx, double sy, int ctas, double* scratch, int* iscratch, double* worst,
                                    cudaStream_t s);

// data_term_value (admm.cpp:239-250) into out[0]
cudaError_t launch_data_term(VolGeom g, const float* target, const float* warped, const float* grad_soa,
                             const float* v_soa, int s, double* part, double* out, unsigned int* counter,
                             cudaStream_t st);
// trilinear_sample at n points (x, y, z) (volume.cpp:55-99); ncomp 1 or 3 (SoA field)
cudaError_t launch_trilinear_points(VolGeom g, const float* field, int ncomp, const double* pts, long long n,
                                    double* out, cudaStream_t st);
// per-pair dreg_pair_record of the multi-device all-gather
cudaError_t launch_pack_records(const PairState* st, int npairs, int pair_base, int device, int levels,
                                dreg_pair_record* out, cudaStream_t s);

cudaError_t launch_aos_to_soa(long long N, const float* aos, float* soa, cudaStream_t s);
cudaError_t launch_soa_to_aos(long long N, const float* soa, float* aos, cudaStream_t s);
cudaError_t launch_add(long long n, const float* a, const float* b, float* out, cudaStream_t s);

}  // namespace dregb
