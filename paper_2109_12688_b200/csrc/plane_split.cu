// Split yz-plane spectral pass: three passes over the spectrum instead of one (the
// w-update multiply of admm.cpp:83-95 sits in the middle):
//   Y   : per tile of ZT z-rows, y-FFT forward (DIF, digit-reversed out)
//   Z   : per tile of YT y-columns, z-FFT forward, x theta/(lambda K_n + theta)/N,
//         z-FFT adjoint (or the spectral energy sum, mode 1)
//   Y^-1: per tile of z-rows, y-FFT adjoint (natural order out)
// Used (a) for planes larger than one CTA's shared memory (config 5: 256 x 192
// complex = 384 KB) and (b) by the precise mode (C = double2: fp64 butterflies,
// twiddles and multiplier, fp32 spectrum storage) for long solves, whose
// accelerated-ADMM iterations amplify per-iteration rounding.
// Generic mixed-radix line transforms (fft_device.cuh), so any Ny, Nz work; the
// position->frequency tables are the generic plans' (sy, sz).
#include <type_traits>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"

namespace dregb {

namespace {
constexpr int kST = 256;

__device__ __forceinline__ bool plane_runnable(const PArgs& a, const PairState* st) {
    if (!st->active || st->status) return false;
    return !(st->solve_done && (!a.need_tail || a.k > st->done_iter));
}

template <class C>
struct Tabs {
    const C* twy;
    const C* twz;
};
template <class C>
__device__ __forceinline__ Tabs<C> tabs(const PArgs& a) {
    if constexpr (std::is_same<C, double2>::value) return {a.twy64, a.twz64};
    else return {a.twy, a.twz};
}
}  // namespace

// rows: tile of ZT consecutive z-rows of one plane; row length Ny (contiguous in global)
template <bool INV, class C>
__global__ void __launch_bounds__(kST) plane_y_kernel(PArgs a, int ZT, FastDiv fd_zt) {
    const int pair = blockIdx.z;
    const PairState* st = a.F.st + pair;
    if (!plane_runnable(a, st)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int Ny = a.F.Ny, Nz = a.F.Nz, hx = a.F.hx;
    const int PY = (Ny % 2 == 0) ? Ny + 1 : Ny;
    C* rows = reinterpret_cast<C*>(smem);  // [ZT][PY]
    C* tw = rows + (size_t)ZT * PY;
    const int tid = threadIdx.x;
    const int plane = blockIdx.y;  // c * hx + p
    const int z0 = blockIdx.x * ZT;
    const int nz = min(ZT, Nz - z0);
    C* Sp = spectrum_of<C>(a.F, pair) + (size_t)plane * (size_t)a.F.lines + (size_t)z0 * Ny;
    const C* twg = tabs<C>(a).twy;
    for (int i = tid; i < Ny; i += kST) tw[i] = twg[i];
    for (int i = tid; i < ZT * Ny; i += kST) {
        const int r = i / Ny, y = i - r * Ny;
        rows[r * PY + y] = r < nz ? Sp[i] : CT<C>::make(0, 0);
    }
    __syncthreads();
    fft_lines<INV>(rows, ZT, fd_zt, PY, 1, a.py, (const C*)tw, tid, kST);
    for (int i = tid; i < nz * Ny; i += kST) {
        const int r = i / Ny, y = i - r * Ny;
        Sp[i] = rows[r * PY + y];
    }
}

// columns: tile of YT consecutive y positions, all Nz z (stride Ny in global)
template <int MODE, class C>
__global__ void __launch_bounds__(kST) plane_z_kernel(PArgs a, int YT, FastDiv fd_yt) {
    using R = typename CT<C>::R;
    const int pair = blockIdx.z;
    PairState* st = a.F.st + pair;
    if (!plane_runnable(a, st)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int Ny = a.F.Ny, Nz = a.F.Nz, hx = a.F.hx;
    const int PC = YT + 1;  // odd pitch between z rows of the tile
    C* cols = reinterpret_cast<C*>(smem);  // [Nz][PC]
    C* tw = cols + (size_t)Nz * PC;
    double* red = reinterpret_cast<double*>(tw + Nz);
    const int tid = threadIdx.x;
    const int plane = blockIdx.y;
    const int c = plane / hx, p = plane - c * hx;
    const int y0 = blockIdx.x * YT;
    const int ny = min(YT, Ny - y0);
    C* Sp = spectrum_of<C>(a.F, pair) + (size_t)plane * (size_t)a.F.lines;
    const C* twg = tabs<C>(a).twz;
    for (int i = tid; i < Nz; i += kST) tw[i] = twg[i];
    for (int i = tid; i < Nz * YT; i += kST) {
        const int z = i / YT, yy = i - z * YT;
        cols[z * PC + yy] = yy < ny ? Sp[(size_t)z * Ny + y0 + yy] : CT<C>::make(0, 0);
    }
    __syncthreads();
    fft_lines<false>(cols, YT, fd_yt, 1, PC, a.pz, (const C*)tw, tid, kST);
    constexpr bool F64 = std::is_same<C, double2>::value;
    const R sxp = F64 ? (R)a.sx64[p] : (R)a.sx[p];
    if (MODE == 0 && F64) {
        // spec *= theta / (lambda K + theta) * inv_count with K = (2 ((3 - cy) - cz - cx))^n,
        // operation for operation as admm.cpp:92 / regularizer.cpp:69-76 (no contraction)
        const double lam = a.lambda64, th = a.theta64, cxp = a.cx64[p];
        for (int i = tid; i < Nz * YT; i += kST) {
            const int z = i / YT, yy = i - z * YT;
            if (yy >= ny) continue;
            const double yz = __dsub_rn(__dsub_rn(3.0, a.cy64[y0 + yy]), a.cz64[z]);
            const double base = __dmul_rn(2.0, __dsub_rn(yz, cxp));
            double K = base;
            for (int e = 1; e < a.order; ++e) K = __dmul_rn(K, base);
            const double m = __dmul_rn(__ddiv_rn(th, __dadd_rn(__dmul_rn(lam, K), th)), a.inv_count);
            const C v = cols[z * PC + yy];
            cols[z * PC + yy] = CT<C>::make(__dmul_rn((double)v.x, m), __dmul_rn((double)v.y, m));
        }
        __syncthreads();
        fft_lines<true>(cols, YT, fd_yt, 1, PC, a.pz, (const C*)tw, tid, kST);
        for (int i = tid; i < Nz * YT; i += kST) {
            const int z = i / YT, yy = i - z * YT;
            if (yy < ny) Sp[(size_t)z * Ny + y0 + yy] = cols[z * PC + yy];
        }
    } else if (MODE == 0) {
        const R lam = F64 ? (R)a.lambda64 : (R)a.lambda, th = F64 ? (R)a.theta64 : (R)a.theta;
        const R scale = F64 ? (R)a.scale64 : (R)a.scale;
        for (int i = tid; i < Nz * YT; i += kST) {
            const int z = i / YT, yy = i - z * YT;
            if (yy >= ny) continue;
            const R sy = F64 ? (R)a.sy64[y0 + yy] : (R)a.sy[y0 + yy];
            const R sz = F64 ? (R)a.sz64[z] : (R)a.sz[z];
            const R base = (R)2 * (sxp + sy + sz);
            R K = base;
            for (int e = 1; e < a.order; ++e) K *= base;
            const R m = scale / (lam * K + th);
            const C v = cols[z * PC + yy];
            cols[z * PC + yy] = CT<C>::make(v.x * m, v.y * m);
        }
        __syncthreads();
        fft_lines<true>(cols, YT, fd_yt, 1, PC, a.pz, (const C*)tw, tid, kST);
        for (int i = tid; i < Nz * YT; i += kST) {
            const int z = i / YT, yy = i - z * YT;
            if (yy < ny) Sp[(size_t)z * Ny + y0 + yy] = cols[z * PC + yy];
        }
    } else {
        double acc = 0.0;
        for (int i = tid; i < Nz * YT; i += kST) {
            const int z = i / YT, yy = i - z * YT;
            if (yy >= ny) continue;
            const double base = 2.0 * ((double)sxp + (double)(F64 ? a.sy64[y0 + yy] : a.sy[y0 + yy]) +
                                       (double)(F64 ? a.sz64[z] : a.sz[z]));
            double K = base;
            for (int e = 1; e < a.order; ++e) K *= base;
            const C v = cols[z * PC + yy];
            acc += K * ((double)v.x * v.x + (double)v.y * v.y);
        }
        const bool self_conj = (p == 0) || (2 * p == a.F.M);
        const double vals[1] = {block_sum<kST>(acc, red) * (self_conj ? 1.0 : 2.0)};
        double tot[1];
        const unsigned nblocks = gridDim.x * gridDim.y;
        if (reduce_partials<kST, 1>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, nblocks, tot, red,
                                    0u, (int)(blockIdx.y * gridDim.x + blockIdx.x)) &&
            tid == 0)
            a.energy_out[pair] = 0.5 * tot[0] / (double)a.F.N;
    }
}

bool plane_split_needed(const PArgs& a) {
    return a.precise || (!a.fast && plane_smem_bytes(a.F.Ny, a.F.Nz, a.PY) > 227 * 1024);
}

template <class C>
static cudaError_t launch_split_t(const PArgs& a, int mode, int npairs, cudaStream_t s) {
    const int Ny = a.F.Ny, Nz = a.F.Nz;
    const int PY = (Ny % 2 == 0) ? Ny + 1 : Ny;
    int ZT = 16;
    while (ZT > 1 && sizeof(C) * ((size_t)ZT * PY + Ny) > 96 * 1024) ZT /= 2;
    int YT = 16;
    while (YT > 1 && sizeof(C) * ((size_t)Nz * (YT + 1) + Nz) + 256 > 96 * 1024) YT /= 2;
    if ((size_t)3 * a.F.hx * ((Ny + YT - 1) / YT) > (size_t)kMaxPartials && mode == 1)
        return cudaErrorInvalidConfiguration;
    FastDiv fz, fy;
    fz.init((unsigned)ZT);
    fy.init((unsigned)YT);
    const size_t sy_bytes = sizeof(C) * ((size_t)ZT * PY + Ny);
    const size_t sz_bytes = sizeof(C) * ((size_t)Nz * (YT + 1) + Nz) + sizeof(double) * 32;
    const dim3 gy((unsigned)((Nz + ZT - 1) / ZT), (unsigned)(3 * a.F.hx), (unsigned)npairs);
    const dim3 gz((unsigned)((Ny + YT - 1) / YT), (unsigned)(3 * a.F.hx), (unsigned)npairs);
    cudaError_t e;
    e = cudaFuncSetAttribute(plane_y_kernel<false, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sy_bytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(plane_y_kernel<true, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sy_bytes);
    if (e != cudaSuccess) return e;
    void (*kz)(PArgs, int, FastDiv) = mode == 0 ? plane_z_kernel<0, C> : plane_z_kernel<1, C>;
    e = cudaFuncSetAttribute(kz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sz_bytes);
    if (e != cudaSuccess) return e;
    plane_y_kernel<false, C><<<gy, kST, sy_bytes, s>>>(a, ZT, fz);
    kz<<<gz, kST, sz_bytes, s>>>(a, YT, fy);
    if (mode == 0) plane_y_kernel<true, C><<<gy, kST, sy_bytes, s>>>(a, ZT, fz);
    return cudaGetLastError();
}

cudaError_t launch_plane_split(const PArgs& a, int mode, int npairs, cudaStream_t s) {
    return a.precise ? launch_split_t<double2>(a, mode, npairs, s) : launch_split_t<float2>(a, mode, npairs, s);
}

}  // namespace dregb
