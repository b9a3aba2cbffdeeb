// Single-pass yz-plane spectral kernel for planes larger than one CTA's shared memory
// (config 5: 256 x 192 complex = 384 KB): a thread-block cluster of two CTAs holds the
// plane in distributed shared memory, half each, so the spectrum crosses HBM once per
// w-update (admm.cpp:83-95) instead of three times (plane_split.cu).
//
//   CTA r owns the z-rows [r Nz/2, (r+1) Nz/2): load, y-FFT forward on its rows;
//   exchange through DSMEM to the column layout (CTA r: columns [r Ny/2, (r+1) Ny/2), all z);
//   z-FFT forward, x theta / (lambda K_n + theta) / N, z-FFT adjoint;
//   exchange back to rows, y-FFT adjoint, store.
// An exchange reads the peer's (and the own) shared memory into registers, cluster-syncs,
// then writes the other layout in place.  Generic mixed-radix line transforms
// (fft_device.cuh), so any even Ny, Nz whose half-plane fits work; position tables are the
// generic plans' (sy, sz), as in plane_split.cu.
//
// Status (profiles/r2d_config5.md): parity-green on the config-5 grid but opt-in
// (DREG_CLUSTER=1).  With the generic stage-by-stage line transforms (twelve shared-memory
// passes, run-time radices) at one 1024-thread CTA per SM it takes 0.516 ms per w-update
// against 0.434 ms for the three HBM passes of plane_split.cu; it needs the
// register-blocked radix-16 x 16 / 12 x 16 stages of plane_fast.cuh to pay off.
#include <cooperative_groups.h>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace dregb {

namespace {
constexpr int kCT = 1024;   // threads per CTA
constexpr int kCE = 24;     // elements per thread in an exchange (half-plane <= kCT * kCE)
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCT, 1)
    plane_cluster_kernel(PArgs a, FastDiv fd_zh, FastDiv fd_yh) {
    const int pair = blockIdx.z;
    const PairState* st = a.F.st + pair;
    // both CTAs of a cluster see the same pair flags: they leave together, before any cluster barrier
    if (!st->active || st->status) return;
    if (st->solve_done && (!a.need_tail || a.k > st->done_iter)) return;

    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank();
    extern __shared__ __align__(16) unsigned char smem[];
    const int Ny = a.F.Ny, Nz = a.F.Nz, hx = a.F.hx;
    const int ZH = Nz / 2, YH = Ny / 2;
    const int PY = Ny + 1, PC = YH + 1;  // odd pitches (complex)
    const int half = ZH * Ny;            // = Nz * YH elements per CTA in either layout
    float2* buf = reinterpret_cast<float2*>(smem);
    const int bufn = max(ZH * PY, Nz * PC);
    float2* twy = buf + bufn;
    float2* twz = twy + Ny;
    const float2* peer = cluster.map_shared_rank(buf, r ^ 1);
    const int tid = threadIdx.x;
    const int plane = blockIdx.y;  // c * hx + p
    const int p = plane - (plane / hx) * hx;
    const int z0 = r * ZH, y0 = r * YH;
    float2* Sp = a.F.S + ((size_t)pair * 3 * hx + plane) * (size_t)a.F.lines + (size_t)z0 * Ny;

    for (int i = tid; i < Ny; i += kCT) twy[i] = a.twy[i];
    for (int i = tid; i < Nz; i += kCT) twz[i] = a.twz[i];
    // rows: ZH x Ny, contiguous in global
    for (int i = tid; i < half; i += kCT) {
        const int row = i / Ny, y = i - row * Ny;
        buf[row * PY + y] = __ldcs(Sp + i);
    }
    __syncthreads();
    fft_lines<false>(buf, ZH, fd_zh, PY, 1, a.py, (const float2*)twy, tid, kCT);

    // rows -> columns: element (z, y0 + yy) comes from the CTA that owns row z
    float2 e[kCE];
    cluster.sync();  // the peer's rows are transformed
#pragma unroll
    for (int n = 0; n < kCE; ++n) {
        const int i = tid + n * kCT;
        if (i < half) {
            const int z = i / YH, yy = i - z * YH;
            const bool mine = (z >= z0) && (z < z0 + ZH);
            const int zr = mine ? z - z0 : z - (ZH - z0);  // row index inside its owner (the peer starts at ZH - z0)
            e[n] = (mine ? buf : peer)[zr * PY + y0 + yy];
        }
    }
    cluster.sync();  // both CTAs have read both row halves
#pragma unroll
    for (int n = 0; n < kCE; ++n) {
        const int i = tid + n * kCT;
        if (i < half) {
            const int z = i / YH, yy = i - z * YH;
            buf[z * PC + yy] = e[n];
        }
    }
    __syncthreads();
    fft_lines<false>(buf, YH, fd_yh, 1, PC, a.pz, (const float2*)twz, tid, kCT);
    {
        // theta / (lambda K + theta) / N at the digit-reversed positions (regularizer.cpp:69-73)
        const float sxp = a.sx[p], lam = a.lambda, th = a.theta, scale = a.scale;
        for (int i = tid; i < half; i += kCT) {
            const int z = i / YH, yy = i - z * YH;
            const float base = 2.0f * (sxp + a.sy[y0 + yy] + a.sz[z]);
            float K = base;
            for (int q = 1; q < a.order; ++q) K *= base;
            const float m = scale / (lam * K + th);
            const float2 v = buf[z * PC + yy];
            buf[z * PC + yy] = make_float2(v.x * m, v.y * m);
        }
    }
    __syncthreads();
    fft_lines<true>(buf, YH, fd_yh, 1, PC, a.pz, (const float2*)twz, tid, kCT);

    // columns -> rows: element (z0 + row, y) comes from the CTA that owns column y
    cluster.sync();  // the peer's columns are filtered
#pragma unroll
    for (int n = 0; n < kCE; ++n) {
        const int i = tid + n * kCT;
        if (i < half) {
            const int row = i / Ny, y = i - row * Ny;
            const bool mine = (y >= y0) && (y < y0 + YH);
            const int yc = mine ? y - y0 : y - (YH - y0);
            e[n] = (mine ? buf : peer)[(z0 + row) * PC + yc];
        }
    }
    cluster.sync();
#pragma unroll
    for (int n = 0; n < kCE; ++n) {
        const int i = tid + n * kCT;
        if (i < half) {
            const int row = i / Ny, y = i - row * Ny;
            buf[row * PY + y] = e[n];
        }
    }
    __syncthreads();
    fft_lines<true>(buf, ZH, fd_zh, PY, 1, a.py, (const float2*)twy, tid, kCT);
    for (int i = tid; i < half; i += kCT) {
        const int row = i / Ny, y = i - row * Ny;
        __stcs(Sp + i, buf[row * PY + y]);
    }
    // a CTA must not exit while its peer may still read its shared memory: the last remote
    // reads precede the second cluster.sync of the exchange above, so nothing is pending here
}

static size_t cluster_smem(int Ny, int Nz) {
    const int ZH = Nz / 2, YH = Ny / 2;
    const size_t bufn = (size_t)std::max(ZH * (Ny + 1), Nz * (YH + 1));
    return sizeof(float2) * (bufn + Ny + Nz);
}

bool plane_cluster_eligible(const PArgs& a) {
    const int Ny = a.F.Ny, Nz = a.F.Nz;
    if (a.precise || !a.cluster || Ny % 2 || Nz % 2) return false;
    if ((size_t)(Nz / 2) * Ny > (size_t)kCT * kCE) return false;
    return cluster_smem(Ny, Nz) <= 227 * 1024;
}

cudaError_t launch_plane_cluster(const PArgs& a, int npairs, cudaStream_t s) {
    const int Ny = a.F.Ny, Nz = a.F.Nz;
    const size_t smem = cluster_smem(Ny, Nz);
    cudaError_t e = cudaFuncSetAttribute(plane_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    FastDiv fz, fy;
    fz.init((unsigned)(Nz / 2));
    fy.init((unsigned)(Ny / 2));
    plane_cluster_kernel<<<dim3(2, (unsigned)(3 * a.F.hx), (unsigned)npairs), kCT, smem, s>>>(a, fz, fy);
    return cudaGetLastError();
}

}  // namespace dregb
