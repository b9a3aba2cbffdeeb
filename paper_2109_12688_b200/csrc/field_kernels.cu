// Deformation-side kernels: warp + gradient, composition + warp + SAD + the
// accept/revert/stop decision, Jacobian folding check, intensity preparation.
// All gathers use software trilinear interpolation in fp64 with the reference's
// clamp-then-floor rule (volume.cpp:36-99); no texture filtering (its 8-bit
// weights would break parity).
#include <cfloat>

#include <cstdlib>
#include "kernels.cuh"
#include "launch.h"
#include "pointwise.cuh"

namespace dregb {

constexpr int kVT = 256;  // threads per voxel-kernel block

static unsigned voxel_blocks(long long N) {
    long long b = (N + kVT - 1) / kVT;
    if (b > 1184) b = 1184;  // 148 SMs x 8 resident blocks; grid-stride beyond
    if (b < 1) b = 1;
    return (unsigned)b;
}

__device__ __forceinline__ void unflat(long long i, int M, int Ny, int& x, int& y, int& z) {
    const long long row = i / M;
    x = (int)(i - row * M);
    z = (int)(row / Ny);
    y = (int)(row - (long long)z * Ny);
}

// ---- per-solve setup: grad(warped) + (warped - target) -------------------------
__global__ void __launch_bounds__(kVT) grad_diff_kernel(VolGeom g, RegBuffers R, Fields F, int keep_warped) {
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    if (!st->active || st->status) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->solve_done = 0;
        st->iterations = 0;
        st->done_iter = -1;
    }
    const long long N = g.N;
    const float* W = (st->cur ? R.WARPED[1] : R.WARPED[0]) + (size_t)pair * N;  // no param-array indexing
    const float* T = R.I0 + (size_t)pair * N;
    float* G = F.G + (size_t)pair * 3 * N;
    float* D = F.D + (size_t)pair * N;
    const size_t sy = (size_t)g.M, sz = (size_t)g.M * g.Ny;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        G[i] = (float)diff1(W, i, x, g.M, 1);
        G[N + i] = (float)diff1(W, i, y, g.Ny, sy);
        G[2 * N + i] = (float)diff1(W, i, z, g.Nz, sz);
        D[i] = keep_warped ? W[i] : (float)((double)W[i] - (double)T[i]);
    }
}

cudaError_t launch_grad_diff(VolGeom g, const RegBuffers& R, Fields F, bool keep_warped, int npairs, cudaStream_t s) {
    grad_diff_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F, keep_warped ? 1 : 0);
    return cudaGetLastError();
}

// ---- compose + warp + SAD + decide -------------------------------------------
__device__ __forceinline__ void compose_warp_voxel(const VolGeom& g, const float* __restrict__ phi,
                                                   const float* __restrict__ V, const float* __restrict__ I1,
                                                   const float* __restrict__ I0, float* __restrict__ phin,
                                                   float* __restrict__ wn, long long i, double& sad, double& bad) {
    const long long N = g.N;
    int x, y, z;
    unflat(i, g.M, g.Ny, x, y, z);
    const float v0 = V[i], v1 = V[N + i], v2 = V[2 * N + i];
    if (!(isfinite(v0) && isfinite(v1) && isfinite(v2))) bad += 1.0;
    // compose_deformation: disp'(x) = v(x) + disp(x + v(x))   (volume.cpp:161-181)
    double s[3];
    trilinear3(phi, (size_t)N, g.M, g.Ny, g.Nz, x + (double)v0, y + (double)v1, z + (double)v2, s);
    const float p0 = (float)((double)v0 + s[0]);
    const float p1 = (float)((double)v1 + s[1]);
    const float p2 = (float)((double)v2 + s[2]);
    phin[i] = p0;
    phin[N + i] = p1;
    phin[2 * N + i] = p2;
    // warp_image(level_source, phi_candidate)   (registration.cpp:253)
    const float w = (float)trilinear(I1, g.M, g.Ny, g.Nz, x + (double)p0, y + (double)p1, z + (double)p2);
    wn[i] = w;
    sad += fabs((double)w - (double)I0[i]);  // mean_sad (registration.cpp:145-152)
}

// Two voxels per loop trip (restrict pointers let their gather chains interleave:
// the kernel is gather-latency bound).
template <int MINB>
__global__ void __launch_bounds__(kVT, MINB) compose_decide_kernel(VolGeom g, RegBuffers R, Fields F, double thr,
                                                                   int max_warps) {
    __shared__ double red[32];
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    if (!st->active || st->status) return;
    const long long N = g.N;
    const int cur = st->cur;
    // select, not index: a run-time index into the parameter arrays copies them to local memory
    const float* __restrict__ phi = (cur ? R.PHI[1] : R.PHI[0]) + (size_t)pair * 3 * N;
    float* __restrict__ phin = (cur ? R.PHI[0] : R.PHI[1]) + (size_t)pair * 3 * N;
    float* __restrict__ wn = (cur ? R.WARPED[0] : R.WARPED[1]) + (size_t)pair * N;
    const float* __restrict__ I1 = R.I1 + (size_t)pair * N;
    const float* __restrict__ I0 = R.I0 + (size_t)pair * N;
    const float* __restrict__ V = F.V + (size_t)pair * 3 * N;
    double sad = 0.0, bad = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + stride < N; i += 2 * stride) {
        compose_warp_voxel(g, phi, V, I1, I0, phin, wn, i, sad, bad);
        compose_warp_voxel(g, phi, V, I1, I0, phin, wn, i + stride, sad, bad);
    }
    if (i < N) compose_warp_voxel(g, phi, V, I1, I0, phin, wn, i, sad, bad);
    const double vals[2] = {block_sum<kVT>(sad, red), block_sum<kVT>(bad, red)};
    double tot[2];
    if (reduce_partials<kVT, 2>(vals, F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot, red) &&
        threadIdx.x == 0) {
        {
            const double sum = tot[0], nbad = tot[1];
            if (nbad > 0.0) {
                // solve_velocity's all_finite(v) -> numeric_error (admm.cpp:310-312)
                st->status = DREG_NUMERIC;
                st->active = 0;
                return;
            }
            st->solves += 1;
            const double sad_new = sum / (double)N;
            const int lvl = st->level;
            if (sad_new > st->sad_prev) {  // revert (registration.cpp:256-258)
                st->active = 0;
                return;
            }
            st->cur = cur ^ 1;
            const int w = st->warps;
            if (w < DREG_MAX_WARPS) {
                st->mean_sad[lvl][w + 1] = sad_new;
                st->solver_iterations[lvl][w] = st->iterations;
            }
            st->warps = w + 1;
            st->level_warps[lvl] = w + 1;
            st->velocity_count += 1;
            const double prev = st->sad_prev;
            const double improvement = (prev - sad_new) / fmax(prev, DBL_MIN);  // :266-267
            st->sad_prev = sad_new;
            if (improvement < thr || st->warps >= max_warps) st->active = 0;
        }
    }
}

cudaError_t launch_compose_decide(VolGeom g, const RegBuffers& R, Fields F, double thr, int max_warps,
                                  int npairs, cudaStream_t s) {
    // DREG_COMPOSE_MINB: resident blocks per SM the register budget targets (3 or 4)
    static const int minb = [] {
        const char* e = std::getenv("DREG_COMPOSE_MINB");
        return e ? std::atoi(e) : 3;
    }();
    if (minb == 4) compose_decide_kernel<4><<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F, thr, max_warps);
    else compose_decide_kernel<3><<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F, thr, max_warps);
    return cudaGetLastError();
}

// ---- intensity preparation ----------------------------------------------------
// Pass 1: shared min/max of target and source + all_finite (registration.cpp:199-201,
// :157-166); the last block of each pair stores the range.
__global__ void __launch_bounds__(kVT) minmax_kernel(VolGeom g, RegBuffers R, Fields F) {
    __shared__ double red[32];
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    const long long N = g.N;
    const float* A = R.tgt_in[pair];
    const float* B = R.src_in[pair];
    float lo = FLT_MAX, hi = -FLT_MAX;
    double bad = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        const float a = A[i], b = B[i];
        if (!isfinite(a) || !isfinite(b)) bad += 1.0;
        lo = fminf(lo, fminf(a, b));
        hi = fmaxf(hi, fmaxf(a, b));
    }
    const double vals[3] = {block_min<kVT>((double)lo, red), block_min<kVT>(-(double)hi, red),
                            block_min<kVT>(-bad, red)};
    double tot[3];
    if (reduce_partials<kVT, 3>(vals, F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot, red,
                                0x7u) &&
        threadIdx.x == 0) {
        st->lo = (float)tot[0];
        st->hi = (float)(-tot[1]);
        if (tot[2] < 0.0) {
            st->status = DREG_NUMERIC;
            st->active = 0;
        }
    }
}

// Pass 2: affine map onto [0,1] with the scale computed in fp64.
__global__ void __launch_bounds__(kVT) normalize_kernel(VolGeom g, RegBuffers R, Fields F) {
    const int pair = blockIdx.y;
    const PairState* st = F.st + pair;
    if (st->status) return;
    const long long N = g.N;
    const float* A = R.tgt_in[pair];
    const float* B = R.src_in[pair];
    float* oa = R.tmpA + (size_t)pair * N;
    float* ob = R.tmpB + (size_t)pair * N;
    const double lo = st->lo;
    const double range = (double)st->hi - lo;
    const double scale = range > 0.0 ? 1.0 / range : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        oa[i] = (float)(((double)A[i] - lo) * scale);
        ob[i] = (float)(((double)B[i] - lo) * scale);
    }
}

__global__ void state_reset_kernel(PairState* st, int npairs) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npairs) return;
    PairState& s = st[p];
    s.active = 1;
    s.cur = 0;
    s.solve_done = 0;
    s.iterations = 0;
    s.status = DREG_OK;
    s.velocity_count = 0;
    s.warps = 0;
    s.level = 0;
    s.solves = 0;
    s.counter = 0;
    s.done_iter = -1;
    s.sad_prev = 0.0;
    s.final_change = 0.0;
    s.folding = 0.0;
    s.min_det = 0.0;
    for (int l = 0; l < DREG_MAX_LEVELS; ++l) s.level_warps[l] = 0;
}

cudaError_t launch_state_reset(PairState* st, int npairs, cudaStream_t s) {
    state_reset_kernel<<<(npairs + 127) / 128, 128, 0, s>>>(st, npairs);
    return cudaGetLastError();
}

__global__ void objective_acc_kernel(Fields F, const double* energy, double lambda, int k, int npairs) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npairs) return;
    const PairState* st = F.st + p;
    if (!st->active || st->status) return;
    if (st->solve_done && k > st->done_iter) return;
    F.diag[((size_t)p * F.diag_stride + k) * 3 + 2] += lambda * energy[p];
}

cudaError_t launch_objective_accumulate(Fields F, const double* energy, double lambda, int k, int npairs,
                                        cudaStream_t s) {
    objective_acc_kernel<<<(npairs + 127) / 128, 128, 0, s>>>(F, energy, lambda, k, npairs);
    return cudaGetLastError();
}

cudaError_t launch_prep_normalize(VolGeom g, const RegBuffers& R, Fields F, int npairs, cudaStream_t s) {
    state_reset_kernel<<<(npairs + 127) / 128, 128, 0, s>>>(F.st, npairs);
    minmax_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F);
    normalize_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F);
    return cudaGetLastError();
}

// ---- separable [1 2 1]/4 with edge clamping (registration.cpp:32-58) ----------
__global__ void __launch_bounds__(kVT) smooth_axis_kernel(VolGeom g, const float* in, float* out, int axis) {
    const long long N = g.N;
    const float* f = in + (size_t)blockIdx.y * N;
    float* o = out + (size_t)blockIdx.y * N;
    const int extent = axis == 0 ? g.M : (axis == 1 ? g.Ny : g.Nz);
    const size_t stride = axis == 0 ? 1 : (axis == 1 ? (size_t)g.M : (size_t)g.M * g.Ny);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        const int pos = axis == 0 ? x : (axis == 1 ? y : z);
        const double lo = f[pos > 0 ? i - stride : i];
        const double hi = f[pos < extent - 1 ? i + stride : i];
        o[i] = (float)(0.25 * (lo + hi) + 0.5 * (double)f[i]);
    }
}

cudaError_t launch_smooth_axis(VolGeom g, const float* in, float* out, int axis, int npairs, cudaStream_t s) {
    smooth_axis_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, in, out, axis);
    return cudaGetLastError();
}

// ---- level start: phi = identity, warped = source, initial mean SAD ------------
__global__ void __launch_bounds__(kVT) level_init_kernel(VolGeom g, RegBuffers R, Fields F, int level) {
    __shared__ double red[32];
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    if (st->status) return;
    const long long N = g.N;
    float* phi = R.PHI[0] + (size_t)pair * 3 * N;
    float* W = R.WARPED[0] + (size_t)pair * N;
    const float* I1 = R.I1 + (size_t)pair * N;
    const float* I0 = R.I0 + (size_t)pair * N;
    double sad = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        phi[i] = 0.f;
        phi[N + i] = 0.f;
        phi[2 * N + i] = 0.f;
        const float w = I1[i];  // trilinear at integer coordinates is exact
        W[i] = w;
        sad += fabs((double)w - (double)I0[i]);
    }
    const double vals[1] = {block_sum<kVT>(sad, red)};
    double tot[1];
    if (reduce_partials<kVT, 1>(vals, F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot, red) &&
        threadIdx.x == 0) {
        st->sad_prev = tot[0] / (double)N;
        st->mean_sad[level][0] = st->sad_prev;
        st->cur = 0;
        st->warps = 0;
        st->level = level;
        st->active = 1;
    }
}

cudaError_t launch_level_init(VolGeom g, const RegBuffers& R, Fields F, int level, int npairs, cudaStream_t s) {
    level_init_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F, level);
    return cudaGetLastError();
}

// det J of I + grad u at voxel (x, y, z) (volume.cpp:183-230): fp64 differences with
// one-sided faces, cofactor expansion along row 0, rounded to fp32 like the stored
// determinant volume (:224)
__device__ __forceinline__ float jacobian_det(const VolGeom& g, const float* __restrict__ u, long long i, int x, int y,
                                              int z) {
    const long long N = g.N;
    const size_t sy = (size_t)g.M, sz = (size_t)g.M * g.Ny;
    double j[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float* uc = u + (size_t)c * N;
        j[c][0] = diff1(uc, i, x, g.M, 1) + (c == 0 ? 1.0 : 0.0);
        j[c][1] = diff1(uc, i, y, g.Ny, sy) + (c == 1 ? 1.0 : 0.0);
        j[c][2] = diff1(uc, i, z, g.Nz, sz) + (c == 2 ? 1.0 : 0.0);
    }
    const double value = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                         j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                         j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
    return (float)value;
}

__device__ __forceinline__ bool interior(const VolGeom& g, int x, int y, int z) {
    return x >= 1 && x < g.M - 1 && y >= 1 && y < g.Ny - 1 && z >= 1 && z < g.Nz - 1;
}

// ---- end of registration: finiteness of phi, phi out, warp of the ORIGINAL source,
// and the folding record of the final phi (jacobian_stats, metrics.cpp:211-228) -----
__global__ void __launch_bounds__(kVT) finalize_kernel(VolGeom g, RegBuffers R, Fields F) {
    __shared__ double red[32];
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    if (st->status) return;
    const long long N = g.N;
    const float* __restrict__ phi = (st->cur ? R.PHI[1] : R.PHI[0]) + (size_t)pair * 3 * N;
    const float* src = R.src_in[pair];
    float* po = R.phi_out ? R.phi_out[pair] : nullptr;
    float* wo = R.warped_out ? R.warped_out[pair] : nullptr;
    const bool jac = g.M >= 3 && g.Ny >= 3 && g.Nz >= 3;
    double bad = 0.0, nonpos = 0.0, mind = 1e300;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        const float u0 = phi[i], u1 = phi[N + i], u2 = phi[2 * N + i];
        if (!(isfinite(u0) && isfinite(u1) && isfinite(u2))) bad += 1.0;
        if (po) {
            po[i] = u0;
            po[N + i] = u1;
            po[2 * N + i] = u2;
        }
        if (wo) wo[i] = (float)trilinear(src, g.M, g.Ny, g.Nz, x + (double)u0, y + (double)u1, z + (double)u2);
        if (jac && interior(g, x, y, z)) {
            const double d = (double)jacobian_det(g, phi, i, x, y, z);
            mind = fmin(mind, d);
            nonpos += d <= 0.0 ? 1.0 : 0.0;
        }
    }
    const double vals[3] = {block_sum<kVT>(bad, red), block_sum<kVT>(nonpos, red), block_min<kVT>(mind, red)};
    double tot[3];
    if (reduce_partials<kVT, 3>(vals, F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot, red,
                                0x4u) &&
        threadIdx.x == 0) {
        st->folding = tot[1];
        st->min_det = jac ? tot[2] : 0.0;
        if (tot[0] > 0.0) st->status = DREG_NUMERIC;  // registration.cpp:275-277
    }
}

cudaError_t launch_finalize(VolGeom g, const RegBuffers& R, Fields F, int npairs, cudaStream_t s) {
    finalize_kernel<<<dim3(voxel_blocks(g.N), npairs), kVT, 0, s>>>(g, R, F);
    return cudaGetLastError();
}

// ---- Jacobian determinant + interior folding statistics ------------------------
__global__ void __launch_bounds__(kVT) jacobian_kernel(VolGeom g, const float* __restrict__ u, float* det,
                                                       double* part, double* out3, unsigned int* counter) {
    __shared__ double red[32];
    const long long N = g.N;
    double nonpos = 0.0, mind = 1e300;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        const float dv = jacobian_det(g, u, i, x, y, z);
        if (det) det[i] = dv;
        if (interior(g, x, y, z)) {
            const double d = (double)dv;  // metrics.cpp:217-227 compares the fp32 value
            mind = fmin(mind, d);
            nonpos += d <= 0.0 ? 1.0 : 0.0;
        }
    }
    const double vals[2] = {block_sum<kVT>(nonpos, red), block_min<kVT>(mind, red)};
    double tot[2];
    if (reduce_partials<kVT, 2>(vals, part, counter, gridDim.x, tot, red, 0x2u) && threadIdx.x == 0) {
        out3[0] = tot[0];
        out3[1] = (double)(g.M - 2) * (double)(g.Ny - 2) * (double)(g.Nz - 2);
        out3[2] = tot[1];
    }
}

cudaError_t launch_jacobian(VolGeom g, const float* phi_soa, float* det, double* part, double* out3,
                            unsigned int* counter, cudaStream_t s) {
    jacobian_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, phi_soa, det, part, out3, counter);
    return cudaGetLastError();
}

// ---- building blocks -------------------------------------------------------------
__global__ void warp_image_kernel(VolGeom g, const float* img, const float* disp, float* out) {
    const long long N = g.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        out[i] = (float)trilinear(img, g.M, g.Ny, g.Nz, x + (double)disp[i], y + (double)disp[N + i],
                                  z + (double)disp[2 * N + i]);
    }
}

cudaError_t launch_warp_image(VolGeom g, const float* img, const float* disp, float* out, cudaStream_t s) {
    warp_image_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, img, disp, out);
    return cudaGetLastError();
}

__global__ void gradient_kernel(VolGeom g, const float* W, float* G) {
    const long long N = g.N;
    const size_t sy = (size_t)g.M, sz = (size_t)g.M * g.Ny;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        G[i] = (float)diff1(W, i, x, g.M, 1);
        G[N + i] = (float)diff1(W, i, y, g.Ny, sy);
        G[2 * N + i] = (float)diff1(W, i, z, g.Nz, sz);
    }
}

cudaError_t launch_gradient(VolGeom g, const float* img, float* out, cudaStream_t s) {
    gradient_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, img, out);
    return cudaGetLastError();
}

__global__ void compose_kernel(VolGeom g, const float* phi, const float* V, float* out) {
    const long long N = g.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, g.M, g.Ny, x, y, z);
        const float v0 = V[i], v1 = V[N + i], v2 = V[2 * N + i];
        double s[3];
        trilinear3(phi, (size_t)N, g.M, g.Ny, g.Nz, x + (double)v0, y + (double)v1, z + (double)v2, s);
        out[i] = (float)((double)v0 + s[0]);
        out[N + i] = (float)((double)v1 + s[1]);
        out[2 * N + i] = (float)((double)v2 + s[2]);
    }
}

cudaError_t launch_compose(VolGeom g, const float* disp, const float* v, float* out, cudaStream_t s) {
    compose_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, disp, v, out);
    return cudaGetLastError();
}

template <int DT>
__global__ void v_update_kernel(VolGeom g, const float* T, const float* W, const float* G, const float* WH,
                                const float* BH, double theta, double eps, float* out) {
    const long long N = g.N;
    const double inv_theta = 1.0 / theta;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        const float wh[3] = {WH[i], WH[N + i], WH[2 * N + i]};
        const float bh[3] = {BH[i], BH[N + i], BH[2 * N + i]};
        const float gg[3] = {G[i], G[N + i], G[2 * N + i]};
        float v[3];
        v_update_voxel<DT>(wh, bh, gg, (double)W[i] - (double)T[i], theta, inv_theta, eps, v);
        out[i] = v[0];
        out[N + i] = v[1];
        out[2 * N + i] = v[2];
    }
}

cudaError_t launch_v_update(VolGeom g, int data_term, const float* target, const float* warped,
                            const float* grad, const float* w_hat, const float* b_hat, double theta,
                            double eps, float* out, cudaStream_t s) {
    if (data_term == 1)
        v_update_kernel<1><<<voxel_blocks(g.N), kVT, 0, s>>>(g, target, warped, grad, w_hat, b_hat, theta, eps, out);
    else
        v_update_kernel<2><<<voxel_blocks(g.N), kVT, 0, s>>>(g, target, warped, grad, w_hat, b_hat, theta, eps, out);
    return cudaGetLastError();
}

__global__ void sad_kernel(VolGeom g, const float* a, const float* b, double* part, double* out,
                           unsigned int* counter) {
    __shared__ double red[32];
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N;
         i += (long long)gridDim.x * blockDim.x)
        s += fabs((double)a[i] - (double)b[i]);
    const double vals[1] = {block_sum<kVT>(s, red)};
    double tot[1];
    if (reduce_partials<kVT, 1>(vals, part, counter, gridDim.x, tot, red) && threadIdx.x == 0)
        *out = tot[0] / (double)g.N;
}

cudaError_t launch_sad(VolGeom g, const float* a, const float* b, double* part, double* out,
                       unsigned int* counter, cudaStream_t s) {
    sad_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, a, b, part, out, counter);
    return cudaGetLastError();
}

__global__ void minmax1_kernel(VolGeom g, const float* a, const float* b, float* part, unsigned int* counter) {
    __shared__ double red[32];
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N;
         i += (long long)gridDim.x * blockDim.x) {
        lo = fminf(lo, fminf(a[i], b[i]));
        hi = fmaxf(hi, fmaxf(a[i], b[i]));
    }
    const double tl = block_min<kVT>((double)lo, red);
    const double th = -block_min<kVT>(-(double)hi, red);
    if (threadIdx.x == 0) {
        part[2 + 2 * blockIdx.x] = (float)tl;
        part[3 + 2 * blockIdx.x] = (float)th;
        if (last_block_ticket(counter, gridDim.x)) {
            float l = FLT_MAX, h = -FLT_MAX;
            for (unsigned k = 0; k < gridDim.x; ++k) {
                l = fminf(l, part[2 + 2 * k]);
                h = fmaxf(h, part[3 + 2 * k]);
            }
            part[0] = l;
            part[1] = h;
        }
    }
}

__global__ void normalize1_kernel(VolGeom g, const float* a, const float* b, float* oa, float* ob,
                                  const float* part) {
    const double lo = part[0];
    const double range = (double)part[1] - lo;
    const double scale = range > 0.0 ? 1.0 / range : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N;
         i += (long long)gridDim.x * blockDim.x) {
        oa[i] = (float)(((double)a[i] - lo) * scale);
        ob[i] = (float)(((double)b[i] - lo) * scale);
    }
}

cudaError_t launch_minmax_normalize(VolGeom g, const float* a, const float* b, float* oa, float* ob,
                                    float* part, unsigned int* counter, cudaStream_t s) {
    minmax1_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, a, b, part, counter);
    normalize1_kernel<<<voxel_blocks(g.N), kVT, 0, s>>>(g, a, b, oa, ob, part);
    return cudaGetLastError();
}

// registration.cpp:85-112: 2x2x2 mean with clamped (edge-replicated) reads
__global__ void downsample_kernel(VolGeom gs, VolGeom gd, const float* in, float* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, gd.M, gd.Ny, x, y, z);
        double sum = 0.0;
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int xx = min(2 * x + dx, gs.M - 1), yy = min(2 * y + dy, gs.Ny - 1),
                              zz = min(2 * z + dz, gs.Nz - 1);
                    sum += in[xx + (size_t)gs.M * (yy + (size_t)gs.Ny * zz)];
                }
        out[i] = (float)(sum / 8.0);
    }
}

cudaError_t launch_downsample(VolGeom src, VolGeom dst, const float* in, float* out, cudaStream_t s) {
    downsample_kernel<<<voxel_blocks(dst.N), kVT, 0, s>>>(src, dst, in, out);
    return cudaGetLastError();
}

__device__ __forceinline__ double source_coord(int i, int te, int se) {
    if (te <= 1) return 0.0;
    return (double)i * (double)(se - 1) / (double)(te - 1);
}

// Pyramid construction for a chunk of pairs: level l-1 = downsample(level l) for the
// normalised target and source (registration.cpp:208-214), [P][N] buffers.
__global__ void __launch_bounds__(kVT) pyr_down_kernel(VolGeom gs, VolGeom gd, const float* ta, const float* sa,
                                                       float* tb, float* sb) {
    const int pair = blockIdx.y;
    const float* in0 = ta + (size_t)pair * gs.N;
    const float* in1 = sa + (size_t)pair * gs.N;
    float* o0 = tb + (size_t)pair * gd.N;
    float* o1 = sb + (size_t)pair * gd.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, gd.M, gd.Ny, x, y, z);
        double s0 = 0.0, s1 = 0.0;
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const size_t j = min(2 * x + dx, gs.M - 1) +
                                     (size_t)gs.M * (min(2 * y + dy, gs.Ny - 1) + (size_t)gs.Ny * min(2 * z + dz, gs.Nz - 1));
                    s0 += in0[j];
                    s1 += in1[j];
                }
        o0[i] = (float)(s0 / 8.0);
        o1[i] = (float)(s1 / 8.0);
    }
}

cudaError_t launch_pyr_down(VolGeom src, VolGeom dst, const float* ta, const float* sa, float* tb, float* sb,
                            int npairs, cudaStream_t s) {
    pyr_down_kernel<<<dim3(voxel_blocks(dst.N), npairs), kVT, 0, s>>>(src, dst, ta, sa, tb, sb);
    return cudaGetLastError();
}

// Level transition (registration.cpp:232-247): phi = upsample_deformation(phi_coarse)
// (corner-aligned trilinear, x2, stored fp32; :114-139), warped = warp(level source,
// phi), sad_prev = mean_sad(warped, level target); per-level state reset.
__global__ void __launch_bounds__(kVT) level_up_kernel(VolGeom gs, VolGeom gd, RegBuffers Rs, RegBuffers Rd, Fields F,
                                                       int level) {
    __shared__ double red[32];
    const int pair = blockIdx.y;
    PairState* st = F.st + pair;
    if (st->status) return;
    const float* phis = Rs.PHI[st->cur] + (size_t)pair * 3 * gs.N;
    float* phid = Rd.PHI[0] + (size_t)pair * 3 * gd.N;
    float* W = Rd.WARPED[0] + (size_t)pair * gd.N;
    const float* I1 = Rd.I1 + (size_t)pair * gd.N;
    const float* I0 = Rd.I0 + (size_t)pair * gd.N;
    double sad = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, gd.M, gd.Ny, x, y, z);
        const double px = source_coord(x, gd.M, gs.M), py = source_coord(y, gd.Ny, gs.Ny),
                     pz = source_coord(z, gd.Nz, gs.Nz);
        double u[3];
        trilinear3(phis, (size_t)gs.N, gs.M, gs.Ny, gs.Nz, px, py, pz, u);
        const float u0 = (float)(2.0 * u[0]), u1 = (float)(2.0 * u[1]), u2 = (float)(2.0 * u[2]);
        phid[i] = u0;
        phid[gd.N + i] = u1;
        phid[2 * gd.N + i] = u2;
        const float w = (float)trilinear(I1, gd.M, gd.Ny, gd.Nz, x + (double)u0, y + (double)u1, z + (double)u2);
        W[i] = w;
        sad += fabs((double)w - (double)I0[i]);
    }
    const double vals[1] = {block_sum<kVT>(sad, red)};
    double tot[1];
    if (reduce_partials<kVT, 1>(vals, F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot, red) &&
        threadIdx.x == 0) {
        st->sad_prev = tot[0] / (double)gd.N;
        st->mean_sad[level][0] = st->sad_prev;
        st->cur = 0;
        st->warps = 0;
        st->level = level;
        st->active = 1;
    }
}

cudaError_t launch_level_up(VolGeom src, VolGeom dst, const RegBuffers& Rs, const RegBuffers& Rd, Fields F, int level,
                            int npairs, cudaStream_t s) {
    level_up_kernel<<<dim3(voxel_blocks(dst.N), npairs), kVT, 0, s>>>(src, dst, Rs, Rd, F, level);
    return cudaGetLastError();
}

// registration.cpp:114-135: corner-aligned trilinear resample, x2 on every component

__global__ void upsample_kernel(VolGeom gs, VolGeom gd, const float* in, float* out, int ncomp) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat(i, gd.M, gd.Ny, x, y, z);
        const double px = source_coord(x, gd.M, gs.M), py = source_coord(y, gd.Ny, gs.Ny),
                     pz = source_coord(z, gd.Nz, gs.Nz);
        for (int c = 0; c < ncomp; ++c)
            out[(size_t)c * gd.N + i] = (float)(2.0 * trilinear(in + (size_t)c * gs.N, gs.M, gs.Ny, gs.Nz, px, py, pz));
    }
}

cudaError_t launch_upsample(VolGeom src, VolGeom dst, const float* in, float* out, int ncomp, cudaStream_t s) {
    upsample_kernel<<<voxel_blocks(dst.N), kVT, 0, s>>>(src, dst, in, out, ncomp);
    return cudaGetLastError();
}

__global__ void aos_to_soa_kernel(long long N, const float* aos, float* soa) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        soa[i] = aos[3 * i];
        soa[N + i] = aos[3 * i + 1];
        soa[2 * N + i] = aos[3 * i + 2];
    }
}
__global__ void soa_to_aos_kernel(long long N, const float* soa, float* aos) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        aos[3 * i] = soa[i];
        aos[3 * i + 1] = soa[N + i];
        aos[3 * i + 2] = soa[2 * N + i];
    }
}
__global__ void add_kernel(long long n, const float* a, const float* b, float* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = a[i] + b[i];
}

cudaError_t launch_aos_to_soa(long long N, const float* aos, float* soa, cudaStream_t s) {
    aos_to_soa_kernel<<<voxel_blocks(N), kVT, 0, s>>>(N, aos, soa);
    return cudaGetLastError();
}
cudaError_t launch_soa_to_aos(long long N, const float* soa, float* aos, cudaStream_t s) {
    soa_to_aos_kernel<<<voxel_blocks(N), kVT, 0, s>>>(N, soa, aos);
    return cudaGetLastError();
}
cudaError_t launch_add(long long n, const float* a, const float* b, float* out, cudaStream_t s) {
    add_kernel<<<voxel_blocks(n), kVT, 0, s>>>(n, a, b, out);
    return cudaGetLastError();
}

}  // namespace dregb

namespace dregb {

// Per-pair records for the multi-device all-gather (dreg_pair_record), one thread per
// pair, written straight from the device-side pair state after the final pass.
__global__ void pack_records_kernel(const PairState* st, int npairs, int pair_base, int device, int levels,
                                    dreg_pair_record* out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npairs) return;
    const PairState& s = st[p];
    dreg_pair_record r;
    r.pair = pair_base + p;
    r.device = device;
    r.status = s.status;
    r.velocity_count = s.velocity_count;
    r.solves = s.solves;
    r.levels = levels;
    r.folding_voxels = (int64_t)s.folding;
    long long iters = 0;
    for (int l = 0; l < levels && l < DREG_MAX_LEVELS; ++l)
        for (int w = 0; w < s.level_warps[l] && w < DREG_MAX_WARPS; ++w) iters += s.solver_iterations[l][w];
    r.admm_iterations = iters;
    const int lf = levels - 1, wf = s.level_warps[lf] < DREG_MAX_WARPS ? s.level_warps[lf] : DREG_MAX_WARPS;
    r.final_mean_sad = s.mean_sad[lf][wf];
    r.min_det = s.min_det;
    r.reserved = 0;
    out[p] = r;
}

cudaError_t launch_pack_records(const PairState* st, int npairs, int pair_base, int device, int levels,
                                dreg_pair_record* out, cudaStream_t s) {
    pack_records_kernel<<<(npairs + 127) / 128, 128, 0, s>>>(st, npairs, pair_base, device, levels, out);
    return cudaGetLastError();
}

}  // namespace dregb

namespace dregb {

// data_term_value (admm.cpp:239-250): sum of |rho| (s = 1) or rho^2 / 2 (s = 2),
// rho = g.v + warped - target in the reference's operation order; fixed-order
// fp64 reduction (run-to-run identical).
__global__ void __launch_bounds__(kVT) data_term_kernel(VolGeom g, const float* T, const float* W, const float* G,
                                                        const float* V, int s, double* part, double* out,
                                                        unsigned int* counter) {
    __shared__ double red[32];
    const long long N = g.N;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        const float gv[3] = {G[i], G[N + i], G[2 * N + i]};
        const float vv[3] = {V[i], V[N + i], V[2 * N + i]};
        const double rho = data_residual_exact(gv, vv, W[i], T[i]);
        acc += s == 1 ? fabs(rho) : 0.5 * rho * rho;
    }
    const double vals[1] = {block_sum<kVT>(acc, red)};
    double tot[1];
    if (reduce_partials<kVT, 1>(vals, part, counter, gridDim.x, tot, red) && threadIdx.x == 0) out[0] = tot[0];
}

cudaError_t launch_data_term(VolGeom g, const float* target, const float* warped, const float* grad_soa,
                             const float* v_soa, int s, double* part, double* out, unsigned int* counter,
                             cudaStream_t st) {
    data_term_kernel<<<voxel_blocks(g.N), kVT, 0, st>>>(g, target, warped, grad_soa, v_soa, s, part, out, counter);
    return cudaGetLastError();
}

// trilinear_sample at arbitrary points (volume.cpp:55-99): clamp-then-floor per axis,
// fp64 lerps x -> y -> z; ncomp 1 (scalar volume) or 3 (SoA vector field).
__global__ void trilinear_points_kernel(VolGeom g, const float* f, int ncomp, const double* pts, long long n,
                                        double* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
        if (ncomp == 1) {
            out[i] = trilinear(f, g.M, g.Ny, g.Nz, px, py, pz);
        } else {
            double r[3];
            trilinear3(f, (size_t)g.N, g.M, g.Ny, g.Nz, px, py, pz, r);
            out[3 * i] = r[0];
            out[3 * i + 1] = r[1];
            out[3 * i + 2] = r[2];
        }
    }
}

cudaError_t launch_trilinear_points(VolGeom g, const float* field, int ncomp, const double* pts, long long n,
                                    double* out, cudaStream_t st) {
    long long b = (n + kVT - 1) / kVT;
    b = b < 1 ? 1 : (b > 1184 ? 1184 : b);
    trilinear_points_kernel<<<(unsigned)b, kVT, 0, st>>>(g, field, ncomp, pts, n, out);
    return cudaGetLastError();
}

}  // namespace dregb
