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
// Status (profiles/r2d_config5.md): the generic version below (DREG_CLUSTER=2) is parity-green
// but slower than the 3-pass split (0.517 vs 0.434 ms per w-update at config 5: twelve
// shared-memory passes with run-time radices); the register-blocked version further down
// (plane_cluster_fast_kernel, DREG_CLUSTER=1, the default where it applies) takes 0.236 ms.
#include <cooperative_groups.h>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"
#include "plane_fast.cuh"

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

// ---- register-blocked version for NY = 16 R2Y, NZ = 16 R1Z (config 5: 256 x 192) ----------
// CTA r keeps the z-rows [r NZ/2, (r+1) NZ/2) for the whole kernel, element (zl, y) at
// zl * PR + y + y / R2Y.  Two-stage DIF transforms as in plane_fast.cuh:
//   Y1 (radix 16 over stride R2Y, straight from global) -> Y2 (radix R2Y on contiguous blocks)
//   Z1 (radix R1Z over stride 16 rows: half of each task's rows live in the peer -> DSMEM, in place)
//   Z2 (radix 16 on 16 contiguous rows, all local since NZ/2 is a multiple of 16) x multiplier x Z2^-1
//   Z1^-1 (DSMEM again), Y2^-1, Y1^-1 straight to global.
// No layout exchange: only Z1 / Z1^-1 touch the peer's shared memory (6 of their 12 elements).
template <bool INV>
__device__ __forceinline__ void dft12(float2* x) {
    // n = n1 + 3 n2, k = 4 k1 + k2: four-point DFTs over n2, twiddles W12^(n1 k2), three-point over n1
    const float c = 0.86602540378443864676f, h = 0.5f;
    float2 y[3][4];
#pragma unroll
    for (int n1 = 0; n1 < 3; ++n1) {
        float2 t[4] = {x[n1], x[n1 + 3], x[n1 + 6], x[n1 + 9]};
        dft4<INV>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) y[n1][k2] = t[k2];
    }
    const float2 w1 = make_float2(c, -h), w2 = make_float2(h, -c), w4 = make_float2(-h, -c);
    y[1][1] = cmul_tw<INV>(y[1][1], w1);
    y[1][2] = cmul_tw<INV>(y[1][2], w2);
    y[1][3] = rot_mi<INV>(y[1][3]);
    y[2][1] = cmul_tw<INV>(y[2][1], w2);
    y[2][2] = cmul_tw<INV>(y[2][2], w4);
    y[2][3] = make_float2(-y[2][3].x, -y[2][3].y);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
        float2 t[3] = {y[0][k2], y[1][k2], y[2][k2]};
        dft3<INV>(t);
#pragma unroll
        for (int k1 = 0; k1 < 3; ++k1) x[4 * k1 + k2] = t[k1];
    }
}

template <bool INV, int R, class C>
__device__ __forceinline__ void rdftz(C* x) {
    if constexpr (R == 12) dft12<INV>(x);
    else rdft<INV, R>(x);
}

constexpr int kFT2 = 512;

// C = double2 is the precise mode (config 4: 128 x 128 planes): fp64 spectrum storage, butterflies
// and twiddles, and the reference's own multiplier expression (admm.cpp:92, regularizer.cpp:69-76,
// no contraction) from its axis cosines at this kernel's digit-reversed positions.
template <int NY, int NZ, class C>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFT2, 1) plane_cluster_fast_kernel(PArgs a) {
    using R = typename CT<C>::R;
    constexpr bool F64 = sizeof(C) == 16;
    constexpr int R1Y = 16, R2Y = NY / 16, R1Z = NZ / 16, R2Z = 16, ZH = NZ / 2, YH = NY / 2;
    constexpr int PR = NY + NY / R2Y + 4;
    static_assert(R2Y == 16 || R2Y == 8, "y second stage radix");
    static_assert(R1Z == 12 || R1Z == 8 || R1Z == 16, "z first stage radix");
    static_assert(ZH % R2Z == 0, "z blocks must not straddle the two CTAs");
    static_assert(!F64 || R1Z != 12, "dft12 is fp32 only");
    const int pair = blockIdx.z;
    const PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;  // both CTAs of the cluster leave together
    if (st->solve_done && (!a.need_tail || a.k > st->done_iter)) return;

    cg::cluster_group cluster = cg::this_cluster();
    const int r = (int)cluster.block_rank();
    extern __shared__ __align__(16) unsigned char smem[];
    C* buf = reinterpret_cast<C*>(smem);  // [ZH][PR]
    C* twy = buf + ZH * PR;
    C* twz = twy + NY;
    R* sys = reinterpret_cast<R*>(twz + NZ);  // fp32: doubled 1 - cos tables; fp64: the reference's axis cosines
    R* szs = sys + NY;
    C* peer = cluster.map_shared_rank(buf, r ^ 1);
    const int tid = threadIdx.x;
    const int hx = a.F.hx;
    const int plane = blockIdx.y;
    const int p = plane - (plane / hx) * hx;
    C* Sp = spectrum_of<C>(a.F, pair) + (size_t)plane * (size_t)a.F.lines + (size_t)(r * ZH) * NY;
    auto at = [](int zl, int y) { return zl * PR + y + y / R2Y; };
    if (a.pf_ahead && tid == 0) {
        // L2-prefetch the half-plane the cluster that takes over these two SMs will load
        // (clusters are dispatched in linear (plane, pair) order, one wave = pf_ahead clusters)
        const unsigned lin = blockIdx.z * gridDim.y + blockIdx.y + (unsigned)a.pf_ahead;
        if (lin < gridDim.y * gridDim.z) {
            const C* nxt = spectrum_of<C>(a.F, 0) + (size_t)lin * (size_t)a.F.lines + (size_t)(r * ZH) * NY;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"((unsigned)(ZH * NY * sizeof(C))) : "memory");
        }
    }

    for (int i = tid; i < NY; i += kFT2) {
        if constexpr (F64) {
            twy[i] = a.twy64[i];
            sys[i] = a.cy64_fast[i];
        } else {
            twy[i] = a.twy[i];
            sys[i] = 2.0f * a.sy_fast[i];
        }
    }
    for (int i = tid; i < NZ; i += kFT2) {
        if constexpr (F64) {
            twz[i] = a.twz64[i];
            szs[i] = a.cz64_fast[i];
        } else {
            twz[i] = a.twz[i];
            szs[i] = 2.0f * a.sz_fast[i];
        }
    }
    __syncthreads();
    // Y1: global -> radix 16 over t (stride R2Y) -> twiddle W_NY^(j1 k) -> shared
    for (int w = tid; w < ZH * R2Y; w += kFT2) {
        const int j1 = w % R2Y, row = w / R2Y;
        C x[R1Y];
#pragma unroll
        for (int t = 0; t < R1Y; ++t) x[t] = __ldcs(Sp + row * NY + j1 + R2Y * t);
        rdft<false, R1Y>(x);
#pragma unroll
        for (int k = 1; k < R1Y; ++k) x[k] = cmul(x[k], twy[j1 * k]);
#pragma unroll
        for (int k = 0; k < R1Y; ++k) buf[at(row, j1 + R2Y * k)] = x[k];
    }
    __syncthreads();
    // Y2: radix R2Y on contiguous blocks
    for (int w = tid; w < ZH * R1Y; w += kFT2) {
        const int blk = w % R1Y, row = w / R1Y;
        C v[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) v[e] = buf[at(row, blk * R2Y + e)];
        rdft<false, R2Y>(v);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[at(row, blk * R2Y + e)] = v[e];
    }
    cluster.sync();  // all rows of both halves are y-transformed
    // Z1: radix R1Z over rows j1 + 16 t; rows of the other half are the peer's (DSMEM), in place
    for (int w = tid; w < YH * R2Z; w += kFT2) {
        const int y = r * YH + w % YH, j1 = w / YH;
        C x[R1Z];
#pragma unroll
        for (int t = 0; t < R1Z; ++t) {
            const int z = j1 + R2Z * t;  // t < R1Z / 2 <=> z < ZH: owner 0
            x[t] = (((t < R1Z / 2) == (r == 0)) ? buf : peer)[at(z % ZH, y)];
        }
        rdftz<false, R1Z>(x);
#pragma unroll
        for (int k = 1; k < R1Z; ++k) x[k] = cmul(x[k], twz[j1 * k]);
#pragma unroll
        for (int k = 0; k < R1Z; ++k) {
            const int z = j1 + R2Z * k;
            (((k < R1Z / 2) == (r == 0)) ? buf : peer)[at(z % ZH, y)] = x[k];
        }
    }
    cluster.sync();
    // Z2 on the local blocks (R1Z / 2 of them): radix 16, multiplier, adjoint radix 16
    {
        const int order = a.order;
        for (int w = tid; w < NY * (R1Z / 2); w += kFT2) {
            const int y = w % NY, bl = w / NY;
            C v[R2Z];
#pragma unroll
            for (int e = 0; e < R2Z; ++e) v[e] = buf[at(bl * R2Z + e, y)];
            rdft<false, R2Z>(v);
            const int zp0 = (r * (R1Z / 2) + bl) * R2Z;
            if constexpr (F64) {
                const double lam = a.lambda64, th = a.theta64, cxp = a.cx64[p], cyp = sys[y];
#pragma unroll
                for (int e = 0; e < R2Z; ++e) {
                    const double yz = __dsub_rn(__dsub_rn(3.0, cyp), szs[zp0 + e]);
                    const double base = __dmul_rn(2.0, __dsub_rn(yz, cxp));
                    double K = base;
                    for (int q = 1; q < order; ++q) K = __dmul_rn(K, base);
                    const double m = __dmul_rn(__ddiv_rn(th, __dadd_rn(__dmul_rn(lam, K), th)), a.inv_count);
                    v[e] = CT<C>::make(__dmul_rn(v[e].x, m), __dmul_rn(v[e].y, m));
                }
            } else {
                const float sxy = 2.0f * __ldg(a.sx + p) + sys[y];
                const float lam_n = a.lam_n, n_f = a.n_f;
#pragma unroll
                for (int e = 0; e < R2Z; ++e) {
                    // theta / (lambda (2 s)^n + theta) / N = 1 / ((lambda N / theta) K_n + N) (regularizer.cpp:69-73)
                    const float K = kn_pow<0>(sxy + szs[zp0 + e], order);
                    const float m = rcp_nr(fmaf(lam_n, K, n_f));
                    v[e] = CT<C>::make(v[e].x * m, v[e].y * m);
                }
            }
            rdft<true, R2Z>(v);
#pragma unroll
            for (int e = 0; e < R2Z; ++e) buf[at(bl * R2Z + e, y)] = v[e];
        }
    }
    cluster.sync();
    // Z1 adjoint
    for (int w = tid; w < YH * R2Z; w += kFT2) {
        const int y = r * YH + w % YH, j1 = w / YH;
        C x[R1Z];
#pragma unroll
        for (int k = 0; k < R1Z; ++k) {
            const int z = j1 + R2Z * k;
            x[k] = (((k < R1Z / 2) == (r == 0)) ? buf : peer)[at(z % ZH, y)];
        }
#pragma unroll
        for (int k = 1; k < R1Z; ++k) x[k] = cmulc(x[k], twz[j1 * k]);
        rdftz<true, R1Z>(x);
#pragma unroll
        for (int t = 0; t < R1Z; ++t) {
            const int z = j1 + R2Z * t;
            (((t < R1Z / 2) == (r == 0)) ? buf : peer)[at(z % ZH, y)] = x[t];
        }
    }
    cluster.sync();  // last remote accesses are behind this barrier
    // Y2 adjoint
    for (int w = tid; w < ZH * R1Y; w += kFT2) {
        const int blk = w % R1Y, row = w / R1Y;
        C v[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) v[e] = buf[at(row, blk * R2Y + e)];
        rdft<true, R2Y>(v);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[at(row, blk * R2Y + e)] = v[e];
    }
    __syncthreads();
    // Y1 adjoint, straight to global
    for (int w = tid; w < ZH * R2Y; w += kFT2) {
        const int j1 = w % R2Y, row = w / R2Y;
        C x[R1Y];
#pragma unroll
        for (int k = 0; k < R1Y; ++k) x[k] = buf[at(row, j1 + R2Y * k)];
#pragma unroll
        for (int k = 1; k < R1Y; ++k) x[k] = cmulc(x[k], twy[j1 * k]);
        rdft<true, R1Y>(x);
#pragma unroll
        for (int t = 0; t < R1Y; ++t) __stcs(Sp + row * NY + j1 + R2Y * t, x[t]);
    }
}

// fp32: config 5's 256 x 192 plane; precise (fp64): config 4's 128 x 128 plane
bool plane_cluster_fast_supported(int Ny, int Nz) { return Ny == 256 && Nz == 192; }
bool plane_cluster_fast64_supported(int Ny, int Nz) { return Ny == 128 && Nz == 128; }

template <int NY, int NZ, class C>
static cudaError_t launch_plane_cluster_fast_t(const PArgs& a, int npairs, cudaStream_t s) {
    using R = typename CT<C>::R;
    constexpr size_t smem = sizeof(C) * ((NZ / 2) * (NY + NY / (NY / 16) + 4) + NY + NZ) + sizeof(R) * (NY + NZ);
    cudaError_t e = cudaFuncSetAttribute(plane_cluster_fast_kernel<NY, NZ, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    PArgs b = a;
    if (b.pf_ahead) {  // one wave of resident clusters ahead
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        b.pf_ahead = b.pf_ahead * (sms / 2);
    }
    plane_cluster_fast_kernel<NY, NZ, C><<<dim3(2, (unsigned)(3 * a.F.hx), (unsigned)npairs), kFT2, smem, s>>>(b);
    return cudaGetLastError();
}

static cudaError_t launch_plane_cluster_fast(const PArgs& a, int npairs, cudaStream_t s) {
    if (a.precise) return launch_plane_cluster_fast_t<128, 128, double2>(a, npairs, s);
    return launch_plane_cluster_fast_t<256, 192, float2>(a, npairs, s);
}

static size_t cluster_smem(int Ny, int Nz) {
    const int ZH = Nz / 2, YH = Ny / 2;
    const size_t bufn = (size_t)std::max(ZH * (Ny + 1), Nz * (YH + 1));
    return sizeof(float2) * (bufn + Ny + Nz);
}

bool plane_cluster_eligible(const PArgs& a) {
    const int Ny = a.F.Ny, Nz = a.F.Nz;
    if (!a.cluster || Ny % 2 || Nz % 2) return false;
    if (a.cluster == 1) {  // register-blocked versions; 2 = the generic one
        if (a.precise) return plane_cluster_fast64_supported(Ny, Nz) && a.cy64_fast && a.cz64_fast && a.F.S64;
        return plane_cluster_fast_supported(Ny, Nz) && a.sy_fast && a.sz_fast;
    }
    if (a.precise) return false;
    if ((size_t)(Nz / 2) * Ny > (size_t)kCT * kCE) return false;
    return cluster_smem(Ny, Nz) <= 227 * 1024;
}

cudaError_t launch_plane_cluster(const PArgs& a, int npairs, cudaStream_t s) {
    const int Ny = a.F.Ny, Nz = a.F.Nz;
    if (a.cluster == 1) return launch_plane_cluster_fast(a, npairs, s);
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
