// In-shared-memory batched line FFTs for the spectral w-update (admm.cpp:66-101).
//
// Forward transforms are decimation-in-frequency (natural order in, digit-reversed
// order out); inverse transforms are the exact adjoint stage sequence (digit-
// reversed in, natural out).  Because the regulariser multiply between them is
// point-wise, the digit-reversed order is never undone: the multiplier is looked up
// through per-axis position->frequency tables instead.  This removes every
// permutation pass from the 3-D FFT (FFTW's plan in the reference does the
// equivalent internally; fft.cpp:52-55).
//
// Everything is templated on the complex type C: float2 (fast path) or double2
// (precise mode: fp64 butterflies for long solves, storage stays fp32).
//
// Layout: element e of line l lives at buf[l*ls + e*es].  Threads are mapped
// line-fastest, which with an odd line pitch makes every stage shared-memory
// bank-conflict free for both contiguous and strided lines.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace dregb {

template <class C>
struct CT;
template <>
struct CT<float2> {
    using R = float;
    __device__ static __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};
template <>
struct CT<double2> {
    using R = double;
    __device__ static __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

template <class C>
__device__ __forceinline__ C cvt_c(float2 v) {
    return CT<C>::make(v.x, v.y);
}
__device__ __forceinline__ float2 to_f2(float2 v) { return v; }
__device__ __forceinline__ float2 to_f2(double2 v) { return make_float2((float)v.x, (float)v.y); }
// spectrum storage element <-> transform element (identity when they match)
template <class D>
__device__ __forceinline__ D cconv(float2 v) {
    return CT<D>::make(v.x, v.y);
}
template <class D>
__device__ __forceinline__ D cconv(double2 v) {
    return CT<D>::make(v.x, v.y);
}

template <bool INV, class C>
__device__ __forceinline__ C rot_mi(C z) {  // multiply by -i (fwd) / +i (inv)
    return INV ? CT<C>::make(-z.y, z.x) : CT<C>::make(z.y, -z.x);
}

template <bool INV, class C>
__device__ __forceinline__ void dft2(C* x) {
    const C a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
}

template <bool INV, class C>
__device__ __forceinline__ void dft4(C* x) {
    if constexpr (std::is_same<C, float2>::value) {
        // packed: the +-i rotation of (x1 - x3) folds into one FFMA2 per output
        const float2 sp = INV ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f);
        const float2 sm = make_float2(-sp.x, -sp.y);
        const C a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
        const C b0 = cadd(x[1], x[3]), d = csub(x[1], x[3]);
        x[0] = cadd(a0, b0);
        x[2] = csub(a0, b0);
        x[1] = cadd_swp(a1, d, sp);
        x[3] = cadd_swp(a1, d, sm);
    } else {
        const C a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
        const C b0 = cadd(x[1], x[3]), b1 = rot_mi<INV>(csub(x[1], x[3]));
        x[0] = cadd(a0, b0);
        x[2] = csub(a0, b0);
        x[1] = cadd(a1, b1);
        x[3] = csub(a1, b1);
    }
}

// dft4 of (x0, x1, rot(x2), x3) with rot = multiply by -i (fwd) / +i (inv): the
// rotation folds into the first butterfly level (packed fp32 only).
template <bool INV>
__device__ __forceinline__ void dft4_rot2(float2* x) {
    const float2 sp = INV ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f);
    const float2 sm = make_float2(-sp.x, -sp.y);
    const float2 a0 = cadd_swp(x[0], x[2], sp), a1 = cadd_swp(x[0], x[2], sm);
    const float2 b0 = cadd(x[1], x[3]), d = csub(x[1], x[3]);
    x[0] = cadd(a0, b0);
    x[2] = csub(a0, b0);
    x[1] = cadd_swp(a1, d, sp);
    x[3] = cadd_swp(a1, d, sm);
}

template <bool INV, class C>
__device__ __forceinline__ void dft8(C* x) {
    using R = typename CT<C>::R;
    const R h = (R)0.70710678118654752440084436210485;
    C a[4], b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        a[j] = cadd(x[j], x[j + 4]);
        b[j] = csub(x[j], x[j + 4]);
    }
    // b_j *= W_8^j (conjugated for the inverse)
    if constexpr (std::is_same<C, float2>::value) {
        const float2 sp = INV ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f);
        const float2 sm = make_float2(-sp.x, -sp.y);
        b[1] = cscale(cadd_swp(b[1], b[1], sp), h);
        b[3] = cscale(cadd_swp(b[3], b[3], sm), -h);
        dft4<INV>(a);
        dft4_rot2<INV>(b);
    } else {
        b[1] = INV ? CT<C>::make(h * (b[1].x - b[1].y), h * (b[1].x + b[1].y))
                   : CT<C>::make(h * (b[1].x + b[1].y), h * (b[1].y - b[1].x));
        b[2] = rot_mi<INV>(b[2]);
        b[3] = INV ? CT<C>::make(-h * (b[3].x + b[3].y), h * (b[3].x - b[3].y))
                   : CT<C>::make(h * (b[3].y - b[3].x), -h * (b[3].x + b[3].y));
        dft4<INV>(a);
        dft4<INV>(b);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        x[2 * m] = a[m];
        x[2 * m + 1] = b[m];
    }
}

template <bool INV, class C>
__device__ __forceinline__ void dft3(C* x) {
    using R = typename CT<C>::R;
    const R c = (R)-0.5, s = (R)0.86602540378443864676372317075294;
    const C t1 = cadd(x[1], x[2]);
    const C t2 = CT<C>::make(x[0].x + c * t1.x, x[0].y + c * t1.y);
    const C d = csub(x[1], x[2]);
    const C t3 = rot_mi<INV>(CT<C>::make(s * d.x, s * d.y));
    x[0] = cadd(x[0], t1);
    x[1] = cadd(t2, t3);
    x[2] = csub(t2, t3);
}

// Generic radix-R DFT with roots W_R^e = tw[e * (n / R)] (conjugated for INV).
template <bool INV, int R, class C>
__device__ __forceinline__ void dft_generic(C* x, const C* __restrict__ tw, int n) {
    C y[R];
    const int st = n / R;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        C acc = x[0];
#pragma unroll
        for (int t = 1; t < R; ++t) {
            const C w = tw[((t * k) % R) * st];
            acc = cadd(acc, INV ? cmulc(x[t], w) : cmul(x[t], w));
        }
        y[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) x[k] = y[k];
}

template <bool INV, int R, class C>
__device__ __forceinline__ void dft_r(C* x, const C* __restrict__ tw, int n) {
    if constexpr (R == 2) dft2<INV>(x);
    else if constexpr (R == 3) dft3<INV>(x);
    else if constexpr (R == 4) dft4<INV>(x);
    else if constexpr (R == 8) dft8<INV>(x);
    else dft_generic<INV, R>(x, tw, n);
}

// One butterfly of stage with radix R.  p points at element j1 of its sub-block,
// step = n1 * es.  DIF: x -> DFT_R -> * W^{j1 k}.  Inverse (adjoint):
// * conj(W^{j1 k}) -> IDFT_R.
template <bool INV, int R, class C>
__device__ __forceinline__ void butterfly(C* p, int step, int j1, int tws, const C* __restrict__ tw, int n) {
    C x[R];
#pragma unroll
    for (int t = 0; t < R; ++t) x[t] = p[t * step];
    if constexpr (INV) {
        if (j1 != 0) {
#pragma unroll
            for (int k = 1; k < R; ++k) x[k] = cmulc(x[k], tw[j1 * k * tws]);
        }
        dft_r<true, R>(x, tw, n);
    } else {
        dft_r<false, R>(x, tw, n);
        if (j1 != 0) {
#pragma unroll
            for (int k = 1; k < R; ++k) x[k] = cmul(x[k], tw[j1 * k * tws]);
        }
    }
#pragma unroll
    for (int t = 0; t < R; ++t) p[t * step] = x[t];
}

// Slow path for prime radices without a template instance (7 < R <= kMaxRadix).
template <bool INV, class C>
__device__ void butterfly_dyn(C* p, int step, int j1, int tws, const C* __restrict__ tw, int n, int R) {
    C x[kMaxRadix];
    for (int t = 0; t < R; ++t) x[t] = p[t * step];
    const int st = n / R;
    if (INV && j1 != 0)
        for (int k = 1; k < R; ++k) x[k] = cmulc(x[k], tw[j1 * k * tws]);
    for (int k = 0; k < R; ++k) {
        C acc = x[0];
        for (int t = 1; t < R; ++t) {
            const C w = tw[((t * k) % R) * st];
            acc = cadd(acc, INV ? cmulc(x[t], w) : cmul(x[t], w));
        }
        if (!INV && j1 != 0 && k != 0) acc = cmul(acc, tw[j1 * k * tws]);
        p[k * step] = acc;  // inputs were copied to x[] first: in place is safe
    }
}

// Batched in-place line transform over `nlines` lines.  All threads of the block
// participate; ends with __syncthreads().
template <bool INV, class C>
__device__ void fft_lines(C* buf, int nlines, const FastDiv& fdl, int ls, int es, const AxisPlan& P,
                          const C* __restrict__ tw, int tid, int nthr) {
    for (int si = 0; si < P.nst; ++si) {
        const int s = INV ? P.nst - 1 - si : si;
        const int r = P.radix[s], n1 = P.n1[s], tws = P.tws[s];
        const int ns = n1 * r;
        const int nb = P.n / r;
        const int total = nlines * nb;
        const int step = n1 * es;
        const FastDiv fd1 = P.fn1[s];
        for (int w = tid; w < total; w += nthr) {
            const int b = (int)fdl.div((unsigned)w);
            const int line = w - b * nlines;
            const int blk = (int)fd1.div((unsigned)b);
            const int j1 = b - blk * n1;
            C* p = buf + line * ls + (blk * ns + j1) * es;
            switch (r) {
                case 2: butterfly<INV, 2>(p, step, j1, tws, tw, P.n); break;
                case 3: butterfly<INV, 3>(p, step, j1, tws, tw, P.n); break;
                case 4: butterfly<INV, 4>(p, step, j1, tws, tw, P.n); break;
                case 5: butterfly<INV, 5>(p, step, j1, tws, tw, P.n); break;
                case 7: butterfly<INV, 7>(p, step, j1, tws, tw, P.n); break;
                case 8: butterfly<INV, 8>(p, step, j1, tws, tw, P.n); break;
                default: butterfly_dyn<INV>(p, step, j1, tws, tw, P.n, r); break;
            }
        }
        __syncthreads();
    }
}

}  // namespace dregb
