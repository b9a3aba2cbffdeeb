// Per-voxel device math shared by the fused kernels and the building blocks.
#pragma once

#include "common.cuh"

namespace dregb {

// v-update of one voxel (admm.cpp:23-63), fp64 arithmetic like the reference.
template <int DT>
__device__ __forceinline__ void v_update_voxel(const float wh[3], const float bh[3], const float g[3],
                                               double d, double theta, double inv_theta, double eps,
                                               float v[3]) {
    const double gx = g[0], gy = g[1], gz = g[2];
    const double ux = (double)wh[0] - (double)bh[0];
    const double uy = (double)wh[1] - (double)bh[1];
    const double uz = (double)wh[2] - (double)bh[2];
    const double gg = gx * gx + gy * gy + gz * gz;
    if (DT == 1) {
        const double residual = (gx * ux + gy * uy + gz * uz) + d;
        const double zhat = theta * residual / (gg + eps);
        const double clip = zhat / fmax(fabs(zhat), 1.0);
        const double s = clip / theta;
        v[0] = (float)(ux - gx * s);
        v[1] = (float)(uy - gy * s);
        v[2] = (float)(uz - gz * s);
    } else {
        const double diff = d;
        const double rx = ux * theta - gx * diff;
        const double ry = uy * theta - gy * diff;
        const double rz = uz * theta - gz * diff;
        const double s = (gx * rx + gy * ry + gz * rz) / (theta * (theta + gg));
        v[0] = (float)(rx * inv_theta - gx * s);
        v[1] = (float)(ry * inv_theta - gy * s);
        v[2] = (float)(rz * inv_theta - gz * s);
    }
}


// The reference's v-update with its exact operation order and no FMA contraction
// (explicit _rn intrinsics), from the UNROUNDED warped / target values (admm.cpp:23-63:
// residual = g.u + double(warped) - double(target); Vec3 dot = (x x' + y y') + z z').
// Used by the fused x-pass for the l1 data term, whose shrinkage branch |zhat| <= 1
// is decided on this value.
template <int DT>
__device__ __forceinline__ void v_update_voxel_exact(const float wh[3], const float bh[3], const float g[3],
                                                     float warped, float target, double theta, double eps,
                                                     float v[3]) {
    const double gx = g[0], gy = g[1], gz = g[2];
    const double ux = __dsub_rn((double)wh[0], (double)bh[0]);
    const double uy = __dsub_rn((double)wh[1], (double)bh[1]);
    const double uz = __dsub_rn((double)wh[2], (double)bh[2]);
    const double gg = __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
    if (DT == 1) {
        const double gu = __dadd_rn(__dadd_rn(__dmul_rn(gx, ux), __dmul_rn(gy, uy)), __dmul_rn(gz, uz));
        const double residual = __dsub_rn(__dadd_rn(gu, (double)warped), (double)target);
        const double zhat = __ddiv_rn(__dmul_rn(theta, residual), __dadd_rn(gg, eps));
        const double clip = __ddiv_rn(zhat, fmax(fabs(zhat), 1.0));
        const double s = __ddiv_rn(clip, theta);
        v[0] = (float)__dsub_rn(ux, __dmul_rn(gx, s));
        v[1] = (float)__dsub_rn(uy, __dmul_rn(gy, s));
        v[2] = (float)__dsub_rn(uz, __dmul_rn(gz, s));
    } else {
        const double diff = __dsub_rn((double)warped, (double)target);
        const double rx = __dsub_rn(__dmul_rn(ux, theta), __dmul_rn(gx, diff));
        const double ry = __dsub_rn(__dmul_rn(uy, theta), __dmul_rn(gy, diff));
        const double rz = __dsub_rn(__dmul_rn(uz, theta), __dmul_rn(gz, diff));
        const double grhs = __dadd_rn(__dadd_rn(__dmul_rn(gx, rx), __dmul_rn(gy, ry)), __dmul_rn(gz, rz));
        const double s = __ddiv_rn(grhs, __dmul_rn(theta, __dadd_rn(theta, gg)));
        const double it = __ddiv_rn(1.0, theta);
        v[0] = (float)__dsub_rn(__dmul_rn(rx, it), __dmul_rn(gx, s));
        v[1] = (float)__dsub_rn(__dmul_rn(ry, it), __dmul_rn(gy, s));
        v[2] = (float)__dsub_rn(__dmul_rn(rz, it), __dmul_rn(gz, s));
    }
}

// rho = g.v + double(warped) - double(target) (data_term_value, admm.cpp:239-250)
__device__ __forceinline__ double data_residual_exact(const float g[3], const float v[3], float warped, float target) {
    const double gv = __dadd_rn(__dadd_rn(__dmul_rn((double)g[0], (double)v[0]), __dmul_rn((double)g[1], (double)v[1])),
                                __dmul_rn((double)g[2], (double)v[2]));
    return __dsub_rn(__dadd_rn(gv, (double)warped), (double)target);
}

// fp32 form of the same update (the point-wise path of the fused x-pass).
// l2: v = u - g (g.u + d) / (theta + |g|^2), algebraically equal to the reference's
//     rhs/theta - g (g.rhs) / (theta (theta + |g|^2)), rhs = theta u - d g;
// l1: identical expression order to admm.cpp:33-39.
// FASTDIV (spectral-state x-pass, theta + |g|^2 >= theta > 0): MUFU.RCP + one Newton step
// instead of the IEEE division's slow path.
template <int DT, bool FASTDIV = false>
__device__ __forceinline__ void v_update_voxel_f32(const float wh[3], const float bh[3], const float g[3], float d,
                                                   float theta, float inv_theta, float eps, float v[3]) {
    const float ux = wh[0] - bh[0], uy = wh[1] - bh[1], uz = wh[2] - bh[2];
    const float gg = fmaf(g[0], g[0], fmaf(g[1], g[1], g[2] * g[2]));
    const float gu = fmaf(g[0], ux, fmaf(g[1], uy, g[2] * uz));
    float s;
    if (DT == 1) {
        const float zhat = theta * (gu + d) / (gg + eps);
        const float clip = zhat / fmaxf(fabsf(zhat), 1.0f);
        s = clip * inv_theta;
    } else {
        s = FASTDIV ? (gu + d) * rcp_nr(theta + gg) : (gu + d) / (theta + gg);
    }
    v[0] = fmaf(-g[0], s, ux);
    v[1] = fmaf(-g[1], s, uy);
    v[2] = fmaf(-g[2], s, uz);
}

// volume.cpp:36-41 (axis_sample): clamp to [0, dim-1] BEFORE floor; hi = min(lo+1, dim-1).
__device__ __forceinline__ void axis_sample(double coord, int dim, int& lo, int& hi, double& frac) {
    const double top = (double)(dim - 1);
    const double c = coord < 0.0 ? 0.0 : (top < coord ? top : coord);
    const double f = floor(c);
    lo = (int)f;
    hi = min(lo + 1, dim - 1);
    frac = c - f;
}

// volume.cpp:55-76: scalar clamp-trilinear in fp64, lerp order x -> y -> z.
__device__ __forceinline__ double trilinear(const float* __restrict__ vol, int M, int Ny, int Nz, double px,
                                            double py, double pz) {
    int x0, x1, y0, y1, z0, z1;
    double fx, fy, fz;
    axis_sample(px, M, x0, x1, fx);
    axis_sample(py, Ny, y0, y1, fy);
    axis_sample(pz, Nz, z0, z1, fz);
    const size_t r00 = (size_t)M * (y0 + (size_t)Ny * z0), r10 = (size_t)M * (y1 + (size_t)Ny * z0);
    const size_t r01 = (size_t)M * (y0 + (size_t)Ny * z1), r11 = (size_t)M * (y1 + (size_t)Ny * z1);
    const double c000 = vol[r00 + x0], c100 = vol[r00 + x1];
    const double c010 = vol[r10 + x0], c110 = vol[r10 + x1];
    const double c001 = vol[r01 + x0], c101 = vol[r01 + x1];
    const double c011 = vol[r11 + x0], c111 = vol[r11 + x1];
    const double c00 = c000 + (c100 - c000) * fx;
    const double c10 = c010 + (c110 - c010) * fx;
    const double c01 = c001 + (c101 - c001) * fx;
    const double c11 = c011 + (c111 - c011) * fx;
    const double c0 = c00 + (c10 - c00) * fy;
    const double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// volume.cpp:78-99: component-wise trilinear of an SoA vector field.
__device__ __forceinline__ void trilinear3(const float* __restrict__ f, size_t N, int M, int Ny, int Nz,
                                           double px, double py, double pz, double out[3]) {
    int x0, x1, y0, y1, z0, z1;
    double fx, fy, fz;
    axis_sample(px, M, x0, x1, fx);
    axis_sample(py, Ny, y0, y1, fy);
    axis_sample(pz, Nz, z0, z1, fz);
    const size_t r00 = (size_t)M * (y0 + (size_t)Ny * z0), r10 = (size_t)M * (y1 + (size_t)Ny * z0);
    const size_t r01 = (size_t)M * (y0 + (size_t)Ny * z1), r11 = (size_t)M * (y1 + (size_t)Ny * z1);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float* v = f + c * N;
        const double c000 = v[r00 + x0], c100 = v[r00 + x1];
        const double c010 = v[r10 + x0], c110 = v[r10 + x1];
        const double c001 = v[r01 + x0], c101 = v[r01 + x1];
        const double c011 = v[r11 + x0], c111 = v[r11 + x1];
        const double c00 = c000 + (c100 - c000) * fx;
        const double c10 = c010 + (c110 - c010) * fx;
        const double c01 = c001 + (c101 - c001) * fx;
        const double c11 = c011 + (c111 - c011) * fx;
        const double c0 = c00 + (c10 - c00) * fy;
        const double c1 = c01 + (c11 - c01) * fy;
        out[c] = c0 + (c1 - c0) * fz;
    }
}

// volume.cpp:137-143: central difference inside, one-sided (no 1/2) on faces.
__device__ __forceinline__ double diff1(const float* __restrict__ f, size_t i, int pos, int dim, size_t stride) {
    if (pos == 0) return (double)f[i + stride] - (double)f[i];
    if (pos == dim - 1) return (double)f[i] - (double)f[i - stride];
    return 0.5 * ((double)f[i + stride] - (double)f[i - stride]);
}

}  // namespace dregb
