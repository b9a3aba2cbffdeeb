// Label metrics on the GPU: warp_labels, Dice counts and the per-slice Hausdorff
// distance (reference metrics.hpp:31-42, metrics.cpp:23-204).  Evaluation-side
// kernels; they run once per registration, so they are
// written for exactness first: every floating-point operation of the reference's
// distance transform is issued as an explicitly rounded fp64 op (no FMA
// contraction), so the distances -- and therefore the Hausdorff values -- are
// bit-identical to the CPU reference.
#include <cstdint>

#include "launch.h"

namespace dregb {

namespace {

constexpr int kMT = 256;  // threads per metrics block

__device__ __forceinline__ void unflat3(long long i, int M, int Ny, int& x, int& y, int& z) {
    const long long line = i / M;
    x = (int)(i - line * M);
    y = (int)(line % Ny);
    z = (int)(line / Ny);
}

}  // namespace

// metrics.cpp:182-204: out(x) = lbl(clamp(lround(x + u(x)))) -- nearest neighbour,
// labels never blended.  disp is the reference's AoS field; lround = round half away
// from zero, like CUDA's llround.
__global__ void warp_labels_kernel(VolGeom g, const uint16_t* __restrict__ lbl, const float* __restrict__ disp,
                                   uint16_t* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N;
         i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        unflat3(i, g.M, g.Ny, x, y, z);
        const long long px = llround(__dadd_rn((double)x, (double)disp[3 * i]));
        const long long py = llround(__dadd_rn((double)y, (double)disp[3 * i + 1]));
        const long long pz = llround(__dadd_rn((double)z, (double)disp[3 * i + 2]));
        const int cx = (int)(px < 0 ? 0 : (px > g.M - 1 ? g.M - 1 : px));
        const int cy = (int)(py < 0 ? 0 : (py > g.Ny - 1 ? g.Ny - 1 : py));
        const int cz = (int)(pz < 0 ? 0 : (pz > g.Nz - 1 ? g.Nz - 1 : pz));
        out[i] = lbl[(size_t)cx + (size_t)g.M * ((size_t)cy + (size_t)g.Ny * cz)];
    }
}

// metrics.cpp:131-147: per label j, counts[j] = {|A|, |B|, |A n B|} (integer atomics:
// order-independent, exact).
__global__ void label_count_kernel(VolGeom g, const uint16_t* __restrict__ a, const uint16_t* __restrict__ b,
                                   const int* __restrict__ labels, unsigned long long* __restrict__ counts) {
    const int label = labels[blockIdx.y];
    unsigned long long ca = 0, cb = 0, cab = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.N;
         i += (long long)gridDim.x * blockDim.x) {
        const bool la = a[i] == label, lb = b[i] == label;
        ca += la;
        cb += lb;
        cab += la && lb;
    }
    for (int o = 16; o > 0; o >>= 1) {
        ca += __shfl_xor_sync(0xffffffffu, ca, o);
        cb += __shfl_xor_sync(0xffffffffu, cb, o);
        cab += __shfl_xor_sync(0xffffffffu, cab, o);
    }
    if ((threadIdx.x & 31) == 0 && (ca | cb | cab)) {
        atomicAdd(&counts[3 * blockIdx.y + 0], ca);
        atomicAdd(&counts[3 * blockIdx.y + 1], cb);
        atomicAdd(&counts[3 * blockIdx.y + 2], cab);
    }
}

// metrics.cpp:27-71 (edt_1d): lower envelope of parabolas f(q) + (x - q*step)^2 over
// one line, f in {finite, +inf}; run sequentially by one thread with the reference's
// exact operation order.  f(q) is read through `F`, output written through `Dst`.
template <class F, class Dst>
__device__ void edt_line(F f, Dst d, int n, double step, int* v, double* zb) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    int k = -1;
    for (int q = 0; q < n; ++q) {
        const double fq = f(q);
        if (fq == inf) continue;
        const double xq = __dmul_rn((double)q, step);
        double s = 0.0;
        while (k >= 0) {
            const double xv = __dmul_rn((double)v[k], step);
            s = __ddiv_rn(__dsub_rn(__dadd_rn(fq, __dmul_rn(xq, xq)), __dadd_rn(f(v[k]), __dmul_rn(xv, xv))),
                          __dmul_rn(2.0, __dsub_rn(xq, xv)));
            if (s > zb[k]) break;
            --k;
        }
        if (k < 0) {
            k = 0;
            v[0] = q;
            zb[0] = -inf;
            zb[1] = inf;
        } else {
            ++k;
            v[k] = q;
            zb[k] = s;
            zb[k + 1] = inf;
        }
    }
    if (k < 0) {
        for (int q = 0; q < n; ++q) d(q, inf);
        return;
    }
    int j = 0;
    for (int q = 0; q < n; ++q) {
        const double xq = __dmul_rn((double)q, step);
        while (zb[j + 1] < xq) ++j;
        const double xv = __dmul_rn((double)v[j], step);
        const double t = __dsub_rn(xq, xv);
        d(q, __dadd_rn(__dmul_rn(t, t), f(v[j])));
    }
}

__device__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    return m;
}

// metrics.cpp:74-103 (slice_edt, row pass then column pass) and :105-115
// (directed_max): squared distance from every pixel to `to`, max over `from`.
__device__ double directed_slice(const uint16_t* __restrict__ to_sl, const uint16_t* __restrict__ from_sl, int label,
                                 int nx, int ny, double sx, double sy, double* dist2, double* colf, int* v,
                                 double* zb, double* red) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int y = threadIdx.x; y < ny; y += blockDim.x) {
        const uint16_t* row = to_sl + (size_t)y * nx;
        double* out = dist2 + (size_t)y * nx;
        edt_line([&](int q) { return row[q] == label ? 0.0 : inf; }, [&](int q, double val) { out[q] = val; }, nx, sx,
                 v, zb);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nx; x += blockDim.x) {
        for (int y = 0; y < ny; ++y) colf[y] = dist2[(size_t)y * nx + x];
        edt_line([&](int q) { return colf[q]; }, [&](int q, double val) { dist2[(size_t)q * nx + x] = val; }, ny, sy,
                 v, zb);
    }
    __syncthreads();
    double worst = 0.0;
    for (int i = threadIdx.x; i < nx * ny; i += blockDim.x)
        if (from_sl[i] == label) worst = fmax(worst, dist2[i]);
    return block_max(worst, red);
}

// metrics.cpp:149-180: one CTA per (z-slice, label) work item.  worst[j][z] = the
// squared symmetric Hausdorff distance of the slice, or -1 when a mask is empty (the
// slice does not contribute).  Scratch per resident CTA: dist2 (nx*ny), and per
// thread a column copy, the envelope's vertex and boundary arrays.
__global__ void __launch_bounds__(128) hausdorff_slices_kernel(VolGeom g, const uint16_t* __restrict__ a,
                                                               const uint16_t* __restrict__ b,
                                                               const int* __restrict__ labels, int n_labels,
                                                               double sx, double sy, double* __restrict__ scratch,
                                                               int* __restrict__ iscratch, double* __restrict__ worst) {
    __shared__ double red[32];
    const int nx = g.M, ny = g.Ny, nmax = nx > ny ? nx : ny;
    const size_t slice = (size_t)nx * ny;
    double* dist2 = scratch + (size_t)blockIdx.x * (slice + (size_t)blockDim.x * (2 * nmax + 2));
    double* colf = dist2 + slice + (size_t)threadIdx.x * (2 * nmax + 2);
    double* zb = colf + nmax;
    int* v = iscratch + ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * nmax;
    const int items = g.Nz * n_labels;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int j = it / g.Nz, z = it - j * g.Nz, label = labels[j];
        const uint16_t* as = a + slice * z;
        const uint16_t* bs = b + slice * z;
        int fa = 0, fb = 0;
        for (size_t i = threadIdx.x; i < slice; i += blockDim.x) {
            fa |= as[i] == label;
            fb |= bs[i] == label;
        }
        fa = __syncthreads_or(fa);
        fb = __syncthreads_or(fb);
        if (!fa || !fb) {  // slices with an empty mask are skipped (metrics.cpp:166-168)
            if (threadIdx.x == 0) worst[it] = -1.0;
            continue;
        }
        const double w1 = directed_slice(bs, as, label, nx, ny, sx, sy, dist2, colf, v, zb, red);
        __syncthreads();
        const double w2 = directed_slice(as, bs, label, nx, ny, sx, sy, dist2, colf, v, zb, red);
        if (threadIdx.x == 0) worst[it] = fmax(w1, w2);
        __syncthreads();
    }
}

cudaError_t launch_warp_labels(VolGeom g, const uint16_t* lbl, const float* disp_aos, uint16_t* out, cudaStream_t s) {
    long long blocks = (g.N + kMT - 1) / kMT;
    if (blocks > 148 * 16) blocks = 148 * 16;
    warp_labels_kernel<<<(unsigned)blocks, kMT, 0, s>>>(g, lbl, disp_aos, out);
    return cudaGetLastError();
}

cudaError_t launch_label_counts(VolGeom g, const uint16_t* a, const uint16_t* b, const int* labels, int n_labels,
                                unsigned long long* counts, cudaStream_t s) {
    long long blocks = (g.N + kMT - 1) / kMT;
    if (blocks > 148 * 4) blocks = 148 * 4;
    cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 3 * n_labels, s);
    if (e != cudaSuccess) return e;
    label_count_kernel<<<dim3((unsigned)blocks, n_labels), kMT, 0, s>>>(g, a, b, labels, counts);
    return cudaGetLastError();
}

size_t hausdorff_scratch_doubles(VolGeom g, int ctas) {
    const size_t nmax = (size_t)(g.M > g.Ny ? g.M : g.Ny);
    return (size_t)ctas * ((size_t)g.M * g.Ny + 128 * (2 * nmax + 2));
}
size_t hausdorff_scratch_ints(VolGeom g, int ctas) {
    const size_t nmax = (size_t)(g.M > g.Ny ? g.M : g.Ny);
    return (size_t)ctas * 128 * nmax;
}

cudaError_t launch_hausdorff_slices(VolGeom g, const uint16_t* a, const uint16_t* b, const int* labels, int n_labels,
                                    double sx, double sy, int ctas, double* scratch, int* iscratch, double* worst,
                                    cudaStream_t s) {
    hausdorff_slices_kernel<<<ctas, 128, 0, s>>>(g, a, b, labels, n_labels, sx, sy, scratch, iscratch, worst);
    return cudaGetLastError();
}

}  // namespace dregb
