/*
 * dreg_cuda.h -- C ABI of the B200-native accelerated-ADMM registration path.
 *
 * This is the drop-in boundary for the reference `dreg` hot path
 * (arXiv 2109.12688; reference C++ library at proj/core).  The reference exposes a
 * C++ value-semantics API (`dreg::solve_velocity`, `dreg::register_pair`, ...);
 * this header is the thin `extern "C"` layer underneath the C++ mirror in
 * include/dreg_b200.hpp, so any FFI (ctypes, cgo, JNI, N-API) can bind it.
 *
 * Conventions (identical to the reference):
 *   - grids are x-fastest, index = x + M*(y + N*z)   (volume.hpp:10-21)
 *   - vector fields on HOST buffers are interleaved AoS (vx,vy,vz) per voxel
 *     (volume.hpp:70-94); device-resident buffers are SoA planes [3][voxels]
 *   - displacements are in voxel units; phi(x) = x + disp(x)   (volume.hpp:96-101)
 *
 * Status codes (no exceptions cross the ABI; the C++ mirror rethrows):
 *   DREG_OK 0, DREG_INVALID_ARGUMENT 2  -> std::invalid_argument
 *             DREG_IO_ERROR 3           -> dreg::io_error        (errors.hpp; file I/O only)
 *             DREG_NUMERIC 4            -> dreg::numeric_error   (errors.hpp:15-17)
 *             DREG_RUNTIME 5            -> std::runtime_error (CUDA / allocation)
 *
 * A context is bound to one CUDA device, owns all device buffers (reused across
 * calls) and is not thread-safe: use one context per host thread / GPU.  There is
 * no CPU fallback: every compute entry point runs sm_100a kernels and returns
 * DREG_RUNTIME when no usable device exists.
 */
#ifndef DREG_CUDA_H
#define DREG_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DREG_OK 0
#define DREG_INVALID_ARGUMENT 2
#define DREG_IO_ERROR 3
#define DREG_NUMERIC 4
#define DREG_RUNTIME 5

/* Capacities of the fixed-size per-level arrays below.  The reference has no limits,
 * but (a) levels > 10 need every axis >= 4 << 10 = 4096 voxels (registration.cpp:195),
 * far beyond one device's memory, and (b) 256 composed fields per level is 5x the
 * converged profile's cap (registration.cpp:62-83).  Configs past these are rejected
 * with DREG_INVALID_ARGUMENT; see INTEGRATION.md. */
#define DREG_MAX_LEVELS 10
#define DREG_MAX_WARPS 256

#define DREG_PROFILE_CAPPED 0
#define DREG_PROFILE_CONVERGED 1

/* dreg::Dims3 (volume.hpp:11-21) */
typedef struct { int x, y, z; } dreg_dims3;
/* dreg::Spacing3 (volume.hpp:25-30) */
typedef struct { double x, y, z; } dreg_spacing3;

/* dreg::SolverConfig (admm.hpp:13-23), same fields and meaning.
 * Defaults (dreg_solver_cfg_default): data_term 1, order 2, lambda 0, theta 0.1,
 * epsilon 1e-6, max_iters 100, tol 0, accelerate 1, log_objective 1. */
typedef struct {
    int data_term;      /* s: 1 = sum of absolute differences, 2 = sum of squares */
    int order;          /* n: regulariser order, 1..6 */
    double lambda;      /* >= 0 */
    double theta;       /* ADMM penalty (north-star "rho"), > 0 */
    double epsilon;     /* guards |grad|^2 in the s=1 update, > 0 */
    int max_iters;      /* >= 1 */
    double tol;         /* stop when mean |v_k - v_{k-1}| <= tol */
    int accelerate;     /* Nesterov extrapolation of w and b */
    int log_objective;  /* record the objective per iteration */
} dreg_solver_cfg;

/* dreg::RegistrationConfig (registration.hpp:16-24). Per-level arrays are indexed
 * coarsest first; only the first `levels` entries are read. */
typedef struct {
    dreg_solver_cfg solver;
    int levels;
    int max_warps_per_level[DREG_MAX_LEVELS];
    int max_admm_iters_per_level[DREG_MAX_LEVELS];
    double warp_improvement_threshold;
    int profile;        /* DREG_PROFILE_* */
    int smooth_levels;
} dreg_reg_cfg;

/* dreg::SolverDiagnostics (admm.hpp:28-34).  objective / constraint_residual are
 * caller-owned arrays of at least max_iters entries (nullable). */
typedef struct {
    int iterations;
    double final_change;
    int converged;
    double* objective;
    double* constraint_residual;
} dreg_solver_diag;

/* dreg::LevelLog (registration.hpp:32-37) with fixed capacity. */
typedef struct {
    dreg_dims3 dims;
    int warps;
    double mean_sad[DREG_MAX_WARPS + 1];
    int solver_iterations[DREG_MAX_WARPS];
} dreg_level_log;

/* dreg::RegistrationResult (registration.hpp:39-45) minus the fields, which are
 * returned through caller buffers. */
typedef struct {
    int status;          /* per-pair DREG_* status */
    int velocity_count;
    int solves;          /* solve_velocity calls, including a reverted last one */
    int levels;
    dreg_level_log per_level[DREG_MAX_LEVELS];
    double elapsed_seconds;
    /* jacobian_stats(phi) of the returned phi (metrics.cpp:211-228), computed on the
     * device in the final pass: interior voxels with fp32 det J <= 0 and their min. */
    int64_t folding_voxels;
    double min_det;
} dreg_pair_result;

/* dreg::JacobianStats (metrics.hpp:44-48) plus the raw counts. */
typedef struct {
    double pct_nonpositive;
    double min_det;
    int64_t nonpositive;
    int64_t interior;
} dreg_jacobian_stats;

typedef struct dreg_cuda_ctx dreg_cuda_ctx;

/* ---- configuration helpers (host only, pure) ---------------------------------- */
void dreg_solver_cfg_default(dreg_solver_cfg* cfg);
/* dreg::validate (admm.cpp:174-196): DREG_OK or DREG_INVALID_ARGUMENT */
int dreg_validate_solver_cfg(const dreg_solver_cfg* cfg);
/* dreg::make_registration_config (registration.cpp:62-83) */
int dreg_make_registration_config(int profile, const dreg_solver_cfg* solver, int levels,
                                  dreg_reg_cfg* out);
/* dreg::nesterov_next_alpha (admm.cpp:198-200) */
double dreg_nesterov_next_alpha(double alpha);
/* dreg::laplacian_symbol (regularizer.cpp:51-79); out has x*y*z doubles */
int dreg_laplacian_symbol(int order, dreg_dims3 dims, double* out);

/* ---- context ------------------------------------------------------------------ */
int dreg_cuda_ctx_create(int device, dreg_cuda_ctx** out);
void dreg_cuda_ctx_destroy(dreg_cuda_ctx* ctx);
/* Message of the last failing call on this context (never NULL). */
const char* dreg_cuda_last_error(const dreg_cuda_ctx* ctx);
/* Work is issued on `stream` (a cudaStream_t; NULL = the context's own stream). */
int dreg_cuda_set_stream(dreg_cuda_ctx* ctx, void* stream);
/* Number of kernels this context launched since creation (evidence counter). */
int64_t dreg_cuda_kernel_launches(const dreg_cuda_ctx* ctx);
/* Pairs processed concurrently per batch chunk (0 = automatic). */
int dreg_cuda_set_batch_chunk(dreg_cuda_ctx* ctx, int pairs);
/* Spectral-solve arithmetic: 0 = auto (fp64 butterflies/twiddles/multiplier for solves
 * of more than 100 iterations, fp32 otherwise), 1 = always fp32, 2 = always fp64.
 * Field and spectrum storage are fp32 in every mode, like the reference's fields. */
int dreg_cuda_set_precision(dreg_cuda_ctx* ctx, int mode);
/* 1 = capture each registration chunk as a CUDA graph (default), 0 = plain launches */
int dreg_cuda_set_use_graphs(dreg_cuda_ctx* ctx, int enable);

/* ---- hot path: registration (registration.hpp:74-75) ---------------------------
 * Host buffers.  phi_out: AoS 3*voxels floats (nullable); warped_out: voxels
 * floats (nullable).  Returns the first failing pair's status. */
int dreg_cuda_register_pair(dreg_cuda_ctx* ctx, const float* target, const float* source,
                            dreg_dims3 dims, dreg_spacing3 spacing, const dreg_reg_cfg* cfg,
                            float* phi_out, float* warped_out, dreg_pair_result* result);

/* n_pairs independent registrations sharing dims and cfg; per-pair host pointers. */
int dreg_cuda_register_batch(dreg_cuda_ctx* ctx, int n_pairs, const float* const* targets,
                             const float* const* sources, dreg_dims3 dims,
                             dreg_spacing3 spacing, const dreg_reg_cfg* cfg,
                             float* const* phi_out, float* const* warped_out,
                             dreg_pair_result* results);

/* Device-resident variant: targets_dev / sources_dev are device arrays laid out
 * [n_pairs][voxels]; phi_dev_out is [n_pairs][3][voxels] SoA (nullable),
 * warped_dev_out [n_pairs][voxels] (nullable).  No host<->device copies of fields;
 * results (small per-pair records) are returned on the host. */
int dreg_cuda_register_batch_device(dreg_cuda_ctx* ctx, int n_pairs, const float* targets_dev,
                                    const float* sources_dev, dreg_dims3 dims,
                                    dreg_spacing3 spacing, const dreg_reg_cfg* cfg,
                                    float* phi_dev_out, float* warped_dev_out,
                                    dreg_pair_result* results);

/* ---- multi-GPU batch (BASELINE config 3) ------------------------
 * Independent pairs sharded over the devices of one box: shard s takes the
 * contiguous pair range dreg_shard_range(n_pairs, n_devices, s), registered by one
 * host thread driving its own per-device context.  No field data crosses devices.
 * The only collective is ONE ncclAllGather of fixed-size per-pair records
 * (dreg_pair_record, written on each device by the final registration pass) over
 * NVLink / NVSwitch; the gathered records are returned in pair order.  NCCL
 * (libnccl.so.2) is loaded at dreg_cuda_multi_create.  The reference has no
 * multi-device path: every per-pair result equals dreg_cuda_register_batch's. */
typedef struct {
    int32_t pair;             /* global pair index; -1 marks gather padding */
    int32_t device;           /* CUDA device that registered it */
    int32_t status;           /* per-pair DREG_* status */
    int32_t velocity_count;
    int32_t solves;
    int32_t levels;
    int64_t folding_voxels;   /* interior det J <= 0 of the returned phi (metrics.cpp:211-228) */
    int64_t admm_iterations;  /* ADMM iterations of the accepted velocity solves, all levels */
    double final_mean_sad;    /* mean SAD after the last accepted warp at the finest level */
    double min_det;           /* interior min det J */
    int64_t reserved;
} dreg_pair_record;          /* 64 bytes */

typedef struct dreg_cuda_multi dreg_cuda_multi;

/* One context per listed device + an NCCL communicator clique (ncclCommInitAll). */
int dreg_cuda_multi_create(const int* devices, int n_devices, dreg_cuda_multi** out);
void dreg_cuda_multi_destroy(dreg_cuda_multi* m);
const char* dreg_cuda_multi_last_error(const dreg_cuda_multi* m);
int dreg_cuda_multi_device_count(const dreg_cuda_multi* m);
/* dreg_cuda_register_batch over all devices; results (nullable) and records
 * (nullable, n_pairs entries, pair order) are host arrays.  Returns the first
 * non-OK per-pair status (per-pair statuses are in results / records). */
int dreg_cuda_multi_register_batch(dreg_cuda_multi* m, int n_pairs, const float* const* targets,
                                   const float* const* sources, dreg_dims3 dims, dreg_spacing3 spacing,
                                   const dreg_reg_cfg* cfg, float* const* phi_out,
                                   float* const* warped_out, dreg_pair_result* results,
                                   dreg_pair_record* records);
/* Host helpers (pure, no device): the contiguous block [begin, end) of shard `shard`
 * (sizes differ by at most one), and the inverse of the all-gather layout -- n_shards
 * blocks of `cap` records, shard s's pairs first then padding -- into pair order.
 * unpack returns DREG_INVALID_ARGUMENT unless every pair 0..n_pairs-1 appears once. */
int dreg_shard_range(int n_pairs, int n_shards, int shard, int* begin, int* end);
int dreg_records_unpack(const dreg_pair_record* gathered, int n_shards, int cap, int n_pairs,
                        dreg_pair_record* out);

/* ---- hot path: one velocity solve (admm.hpp:76-77) ----------------------------- */
int dreg_cuda_solve_velocity(dreg_cuda_ctx* ctx, const float* target,
                             const float* warped_source, dreg_dims3 dims,
                             const dreg_solver_cfg* cfg, float* velocity_out,
                             dreg_solver_diag* diag);

/* ---- measurement -----------------------------------------------------------------
 * Times the two per-iteration kernels (fused x-pass, yz-plane spectral pass) on the
 * current workspace (after a registration call), `reps` launches each, with CUDA
 * events on the context stream.  out[0] = x-pass ms/launch, out[1] = plane ms/launch,
 * out[2] / out[3] = their algorithmic HBM bytes per launch, out[4] = pairs per launch. */
int dreg_cuda_time_kernels(dreg_cuda_ctx* ctx, int reps, double* out);
/* Same, with `cfg`'s data term / order / lambda / theta and the precision the
 * context's policy picks for cfg->max_iters; out[5] = 1 when the precise (fp64
 * spectral arithmetic) kernels were timed; out[6] = 0 when the real-space-state kernels
 * were timed, 1 / 2 for the spectral-state pair with / without the change norm (the
 * kernels a registration's solves run for this configuration).  out holds 7 doubles. */
int dreg_cuda_time_iteration(dreg_cuda_ctx* ctx, const dreg_solver_cfg* cfg, int reps, double* out);

/* ---- DREG volume container (io.hpp:15-41; README.md:99-114) ---------------------
 * Host-only file I/O, byte-compatible with the reference.  Status DREG_IO_ERROR with
 * the reference's message in `err` (nullable, err_len bytes incl. NUL) on failure. */
#define DREG_KIND_SCALAR 0
#define DREG_KIND_VECTOR 1
#define DREG_KIND_LABEL 2
typedef struct {
    int kind;               /* DREG_KIND_* */
    dreg_dims3 dims;
    dreg_spacing3 spacing;
} dreg_volume_info;
/* Header of `path` (validated like read_volume, io.cpp:88-130). */
int dreg_volume_info_read(const char* path, dreg_volume_info* out, char* err, size_t err_len);
/* read_volume / read_scalar / read_vector / read_label (io.hpp:27-35): the whole file
 * is validated (length, finiteness); expected_kind -1 accepts any kind.  payload gets
 * f32 (scalar voxels / vector 3*voxels interleaved) or u16 (label) words; capacity in
 * bytes.  payload may be NULL to validate only. */
int dreg_volume_read(const char* path, int expected_kind, dreg_volume_info* info, void* payload,
                     size_t capacity, char* err, size_t err_len);
/* write_volume (io.hpp:37-40) */
int dreg_volume_write(const char* path, int kind, dreg_dims3 dims, dreg_spacing3 spacing,
                      const void* payload, char* err, size_t err_len);

/* dreg::ReportConfig / RunReport (io.hpp:43-62); label maps as parallel arrays. */
typedef struct {
    const char* data_term;  /* "l1" | "l2" */
    int order;
    double lambda;
    double theta;
    int levels;
    const char* profile;    /* "capped" | "converged" */
    double tol;
    double warp_improvement_threshold;
    double epsilon;
    int threads;
} dreg_report_config;
typedef struct {
    int n_dice;
    const int* dice_labels;
    const double* dice;
    int n_hausdorff;
    const int* hausdorff_labels;
    const double* hausdorff_mm;
    double jacobian_pct_nonpositive;
    double runtime_seconds;
    int velocity_count;
    dreg_report_config config;
} dreg_run_report;
/* write_report (io.hpp:64-66): same keys, order, 6 significant digits, 2-space JSON. */
int dreg_report_write(const char* path, const dreg_run_report* report, char* err, size_t err_len);

/* ---- label metrics (metrics.hpp:31-42), GPU ---------------------------------------
 * Label volumes are u16, x-fastest.  warp_labels: nearest-neighbour (lround, clamp)
 * lookup at x + disp(x), disp AoS.  dice: 2|A∩B|/(|A|+|B|), 1 when both are empty.
 * hausdorff: per z-slice exact anisotropic EDT (in-plane spacing) symmetric
 * Hausdorff, averaged over slices where both masks are non-empty;
 * DREG_INVALID_ARGUMENT when no slice contributes. */
int dreg_cuda_warp_labels(dreg_cuda_ctx* ctx, const uint16_t* labels, const float* disp,
                          dreg_dims3 dims, uint16_t* out);
int dreg_cuda_dice(dreg_cuda_ctx* ctx, const uint16_t* a, const uint16_t* b, dreg_dims3 dims,
                   int label, double* out);
int dreg_cuda_hausdorff_slice_avg(dreg_cuda_ctx* ctx, const uint16_t* a, const uint16_t* b,
                                  dreg_dims3 dims, dreg_spacing3 spacing, int label, double* out);
/* All labels in one upload: dice_out[i], hausdorff_out[i] for labels[i];
 * hausdorff_valid[i] = 0 where no slice carries labels[i] in both volumes
 * (hausdorff_out[i] is then NaN).  Any output may be NULL. */
int dreg_cuda_label_metrics(dreg_cuda_ctx* ctx, const uint16_t* a, const uint16_t* b,
                            dreg_dims3 dims, dreg_spacing3 spacing, int n_labels,
                            const int* labels, double* dice_out, double* hausdorff_out,
                            int* hausdorff_valid);

/* ---- building blocks (host AoS buffers; each a GPU launch) ---------------------- */
/* v_update_l1 / v_update_l2 (admm.hpp:49-58); data_term selects which */
int dreg_cuda_v_update(dreg_cuda_ctx* ctx, const float* target, const float* warped_source,
                       const float* grad, const float* w_hat, const float* b_hat,
                       dreg_dims3 dims, const dreg_solver_cfg* cfg, float* out);
/* w_update (admm.hpp:64-65): spectral solve with the order-cfg->order kernel */
/* data_term_value (admm.hpp:68, admm.cpp:239-250): sum over voxels of |rho| (s = 1)
 * or rho^2 / 2 (s = 2), rho = grad.v + warped - target; grad and v AoS host fields. */
int dreg_cuda_data_term_value(dreg_cuda_ctx* ctx, const float* target, const float* warped_source,
                              const float* grad, const float* v, dreg_dims3 dims, int s, double* out);
/* trilinear_sample (volume.hpp:107,110; volume.cpp:55-99) at n points given as (x, y, z)
 * voxel coordinates (3n doubles): ncomp 1 samples a scalar volume (out: n doubles),
 * ncomp 3 an AoS vector field (out: 3n doubles). */
int dreg_cuda_trilinear_sample(dreg_cuda_ctx* ctx, const float* field, int ncomp, dreg_dims3 dims,
                               const double* points, int64_t n, double* out);
int dreg_cuda_w_update(dreg_cuda_ctx* ctx, const float* v, const float* b_hat,
                       dreg_dims3 dims, const dreg_solver_cfg* cfg, float* out);
/* regulariser_energy (regularizer.hpp:45) */
int dreg_cuda_regulariser_energy(dreg_cuda_ctx* ctx, const float* w, dreg_dims3 dims,
                                 int order, double* out);
/* warp_image (volume.hpp:113) */
int dreg_cuda_warp_image(dreg_cuda_ctx* ctx, const float* img, const float* disp,
                         dreg_dims3 dims, float* out);
/* image_gradient (volume.hpp:117) */
int dreg_cuda_image_gradient(dreg_cuda_ctx* ctx, const float* img, dreg_dims3 dims,
                             float* out);
/* compose_deformation (volume.hpp:121) */
int dreg_cuda_compose_deformation(dreg_cuda_ctx* ctx, const float* disp, const float* v,
                                  dreg_dims3 dims, float* out);
/* jacobian_determinant (volume.hpp:125); det_out nullable; stats nullable */
int dreg_cuda_jacobian(dreg_cuda_ctx* ctx, const float* disp, dreg_dims3 dims,
                       float* det_out, dreg_jacobian_stats* stats);
/* Same on a device-resident SoA field [3][voxels] (e.g. register_batch_device output). */
int dreg_cuda_jacobian_device(dreg_cuda_ctx* ctx, const float* disp_soa_dev, dreg_dims3 dims,
                              float* det_dev_out, dreg_jacobian_stats* stats);
/* normalize_intensity_pair (registration.hpp:65-66) */
int dreg_cuda_normalize_intensity_pair(dreg_cuda_ctx* ctx, const float* a, const float* b,
                                       dreg_dims3 dims, float* out_a, float* out_b);
/* binomial_smooth (registration.hpp:59) */
int dreg_cuda_binomial_smooth(dreg_cuda_ctx* ctx, const float* img, dreg_dims3 dims,
                              float* out);
/* mean_sad (registration.hpp:62) */
int dreg_cuda_mean_sad(dreg_cuda_ctx* ctx, const float* a, const float* b, dreg_dims3 dims,
                       double* out);
/* downsample (registration.hpp:49): out has ceil-half dims */
int dreg_cuda_downsample(dreg_cuda_ctx* ctx, const float* img, dreg_dims3 dims, float* out);
/* upsample_velocity (registration.hpp:54): AoS in (src dims) -> AoS out (dst dims) */
int dreg_cuda_upsample_velocity(dreg_cuda_ctx* ctx, const float* v, dreg_dims3 src_dims,
                                dreg_dims3 dst_dims, float* out);

#ifdef __cplusplus
}
#endif

#endif /* DREG_CUDA_H */
