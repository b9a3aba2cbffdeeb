// Kernel argument blocks and launch declarations (dreg B200 path).
#pragma once

#include "common.cuh"

namespace dregb {

// Device-resident per-chunk state.  Every buffer is [pair][component][voxels]
// (SoA planes) so each kernel's per-pair tile is a contiguous, coalesced range.
struct Fields {
    int M, Ny, Nz;     // grid (x fastest)
    int hx;            // M/2 + 1 stored x bins
    long long N;       // voxels
    long long lines;   // Ny * Nz x-lines
    float* V;          // v_k                 [P][3][N]
    float* BH;         // dual iterate b_{k-2} in, b_k out (the two b buffers swap roles every
                       // iteration; b_hat is re-formed from them)  [P][3][N]
    float* WP;         // w_{k-1} (w_prev)    [P][3][N]
    float* BP;         // dual iterate b_{k-1}  [P][3][N]
    float* G;          // grad(warped)        [P][3][N]
    float* D;          // warped - target     [P][N]; l1 data term: the warped image itself
    const float* T;    // target (I0)         [P][N]; l1: residual = g.u + warped - target
    float2* S;         // x-spectrum, plane-major [P][3][hx][lines]
    double2* S64;      // the same in fp64 for the precise mode (nullptr unless allocated)
    PairState* st;     // [P]
    double* part;      // partial sums        [P][3][kMaxPartials]
    double* diag;      // per-iteration diagnostics [P][max_iters][3] (nullable)
    int diag_stride;   // max_iters
};

// The x-spectrum of one pair in the storage precision that goes with transform type C:
// fp32 (F.S) for the fast path, fp64 (F.S64) in precise mode, so the 3-D transform's
// intermediate is never rounded to fp32 (the reference keeps it in double, fft.cpp:45-46).
template <class C>
__device__ __forceinline__ C* spectrum_of(const Fields& F, int pair) {
    const size_t off = (size_t)pair * 3 * F.hx * (size_t)F.lines;
    if constexpr (sizeof(C) == 16) return reinterpret_cast<C*>(F.S64) + off;
    else return reinterpret_cast<C*>(F.S) + off;
}

// Registration-level buffers.
struct RegBuffers {
    float* I0;          // smoothed normalised target [P][N]
    float* I1;          // smoothed normalised source [P][N]
    float* PHI[2];      // displacement SoA [P][3][N] x2
    float* WARPED[2];   // warped level source [P][N] x2
    const float* const* tgt_in;  // [P] raw target pointers (device)
    const float* const* src_in;  // [P] raw source pointers (device)
    float* const* phi_out;       // [P] SoA outputs (nullable entries)
    float* const* warped_out;    // [P] (nullable entries)
    float* tmpA;        // scratch [P][N]
    float* tmpB;        // scratch [P][N]
};

struct SolverParams {
    double theta, epsilon, lambda, tol;
    int data_term, order;
    int log_objective;
    int accelerate;
};

}  // namespace dregb
