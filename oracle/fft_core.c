/*
 * TEST INFRASTRUCTURE ONLY -- see fft_core.h.
 *
 * Stockham autosort mixed-radix complex FFT (radix 4/2/3/5 butterflies plus a
 * direct DFT for any other prime factor), with twiddles computed in double by
 * sin/cos of exact integer ratios.  The 3-D real transforms reproduce FFTW's
 * r2c/c2r conventions as the reference uses them (`proj/core/src/fft.cpp:52-55`):
 * r2c halves the x axis (x-fastest storage = FFTW's last dimension), both
 * directions unnormalised.
 */
#include "fft_core.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OC_MAX_STAGES 64

struct oc_fft1 {
    int n;
    int nstages;
    int radix[OC_MAX_STAGES];
    int span[OC_MAX_STAGES];       /* p before the stage (product of earlier radices) */
    oc_complex* tw[OC_MAX_STAGES]; /* tw[s][k*r + t] = exp(-2 pi i t k / (p r)) */
    oc_complex* root[OC_MAX_STAGES]; /* root[s][t] = exp(-2 pi i t / r) */
};

static oc_complex cexp_neg(long num, long den) {
    /* exp(-2 pi i num/den) with the ratio reduced first for accuracy */
    long q = num % den;
    if (q < 0) q += den;
    const double a = -2.0 * 3.14159265358979323846264338327950288 * (double)q / (double)den;
    oc_complex c = {cos(a), sin(a)};
    return c;
}

oc_fft1* oc_fft1_create(int n) {
    if (n < 1) return NULL;
    oc_fft1* p = (oc_fft1*)calloc(1, sizeof(oc_fft1));
    p->n = n;
    int rem = n;
    int s = 0;
    while (rem > 1) {
        int r;
        if (rem % 4 == 0) r = 4;
        else if (rem % 2 == 0) r = 2;
        else if (rem % 3 == 0) r = 3;
        else if (rem % 5 == 0) r = 5;
        else {
            r = 7;
            while (rem % r) r += 2;
        }
        p->radix[s++] = r;
        rem /= r;
    }
    p->nstages = s;
    int span = 1;
    for (int i = 0; i < s; ++i) {
        const int r = p->radix[i];
        p->span[i] = span;
        p->tw[i] = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)span * (size_t)r);
        for (int k = 0; k < span; ++k)
            for (int t = 0; t < r; ++t) p->tw[i][k * r + t] = cexp_neg((long)t * k, (long)span * r);
        p->root[i] = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)r);
        for (int t = 0; t < r; ++t) p->root[i][t] = cexp_neg(t, r);
        span *= r;
    }
    return p;
}

void oc_fft1_destroy(oc_fft1* p) {
    if (!p) return;
    for (int i = 0; i < p->nstages; ++i) {
        free(p->tw[i]);
        free(p->root[i]);
    }
    free(p);
}

static inline oc_complex cmul(oc_complex a, oc_complex b) {
    oc_complex c = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return c;
}
static inline oc_complex cconj(oc_complex a) {
    oc_complex c = {a.re, -a.im};
    return c;
}

void oc_fft1_exec(const oc_fft1* p, oc_complex* data, oc_complex* scratch, int sign) {
    const int n = p->n;
    if (n == 1) return;
    oc_complex* src = data;
    oc_complex* dst = scratch;
    oc_complex u[64];
    oc_complex v[64];
    oc_complex* big_u = NULL;
    oc_complex* big_v = NULL;
    for (int s = 0; s < p->nstages; ++s) {
        const int r = p->radix[s];
        const int span = p->span[s];
        const int m = n / r;
        oc_complex* uu = u;
        oc_complex* vv = v;
        if (r > 64) {
            big_u = (oc_complex*)realloc(big_u, sizeof(oc_complex) * (size_t)r);
            big_v = (oc_complex*)realloc(big_v, sizeof(oc_complex) * (size_t)r);
            uu = big_u;
            vv = big_v;
        }
        for (int i = 0; i < m; ++i) {
            const int k = i % span;
            const oc_complex* twk = p->tw[s] + (size_t)k * r;
            for (int t = 0; t < r; ++t) {
                const oc_complex w = sign < 0 ? twk[t] : cconj(twk[t]);
                uu[t] = cmul(src[i + t * m], w);
            }
            if (r == 2) {
                vv[0].re = uu[0].re + uu[1].re; vv[0].im = uu[0].im + uu[1].im;
                vv[1].re = uu[0].re - uu[1].re; vv[1].im = uu[0].im - uu[1].im;
            } else if (r == 4) {
                const double a0r = uu[0].re + uu[2].re, a0i = uu[0].im + uu[2].im;
                const double a1r = uu[0].re - uu[2].re, a1i = uu[0].im - uu[2].im;
                const double b0r = uu[1].re + uu[3].re, b0i = uu[1].im + uu[3].im;
                const double b1r = uu[1].re - uu[3].re, b1i = uu[1].im - uu[3].im;
                /* -i*sign rotation of b1 for the odd outputs */
                const double rr = sign < 0 ? b1i : -b1i;
                const double ri = sign < 0 ? -b1r : b1r;
                vv[0].re = a0r + b0r; vv[0].im = a0i + b0i;
                vv[2].re = a0r - b0r; vv[2].im = a0i - b0i;
                vv[1].re = a1r + rr;  vv[1].im = a1i + ri;
                vv[3].re = a1r - rr;  vv[3].im = a1i - ri;
            } else {
                const oc_complex* root = p->root[s];
                for (int q = 0; q < r; ++q) {
                    double sr = 0.0, si = 0.0;
                    for (int t = 0; t < r; ++t) {
                        const int e = (int)(((long)t * q) % r);
                        const oc_complex w = sign < 0 ? root[e] : cconj(root[e]);
                        sr += uu[t].re * w.re - uu[t].im * w.im;
                        si += uu[t].re * w.im + uu[t].im * w.re;
                    }
                    vv[q].re = sr;
                    vv[q].im = si;
                }
            }
            const int j = (i - k) * r + k;
            for (int q = 0; q < r; ++q) dst[j + q * span] = vv[q];
        }
        oc_complex* tmp = src;
        src = dst;
        dst = tmp;
    }
    free(big_u);
    free(big_v);
    if (src != data) memcpy(data, src, sizeof(oc_complex) * (size_t)n);
}

/* ------------------------------------------------------------------------------- */

struct oc_fft3 {
    int nx, ny, nz, hx;
    oc_fft1* fx;  /* length nx/2 when nx even (half-length trick), nx otherwise */
    oc_fft1* fy;
    oc_fft1* fz;
    oc_complex* xtw; /* exp(-2 pi i k / nx), k in [0, nx/2] */
    oc_complex* line;
    oc_complex* line2;
    oc_complex* scratch;
    oc_complex* work; /* half spectrum copy for c2r */
};

oc_fft3* oc_fft3_create(int nx, int ny, int nz) {
    if (nx < 1 || ny < 1 || nz < 1) return NULL;
    oc_fft3* p = (oc_fft3*)calloc(1, sizeof(oc_fft3));
    p->nx = nx;
    p->ny = ny;
    p->nz = nz;
    p->hx = nx / 2 + 1;
    const int even = (nx % 2 == 0) && nx >= 2;
    p->fx = oc_fft1_create(even ? nx / 2 : nx);
    p->fy = oc_fft1_create(ny);
    p->fz = oc_fft1_create(nz);
    p->xtw = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)p->hx);
    for (int k = 0; k < p->hx; ++k) p->xtw[k] = cexp_neg(k, nx);
    int maxn = nx;
    if (ny > maxn) maxn = ny;
    if (nz > maxn) maxn = nz;
    p->line = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(maxn + 1));
    p->line2 = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(maxn + 1));
    p->scratch = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)(maxn + 1));
    p->work = (oc_complex*)malloc(sizeof(oc_complex) * (size_t)p->hx * ny * nz);
    return p;
}

void oc_fft3_destroy(oc_fft3* p) {
    if (!p) return;
    oc_fft1_destroy(p->fx);
    oc_fft1_destroy(p->fy);
    oc_fft1_destroy(p->fz);
    free(p->xtw);
    free(p->line);
    free(p->line2);
    free(p->scratch);
    free(p->work);
    free(p);
}

/* complex transforms along y and z of a half spectrum, in place */
static void yz_pass(oc_fft3* p, oc_complex* spec, int sign) {
    const int hx = p->hx, ny = p->ny, nz = p->nz;
    if (ny > 1) {
        for (int r = 0; r < nz; ++r)
            for (int k = 0; k < hx; ++k) {
                oc_complex* base = spec + k + (size_t)hx * ny * r;
                for (int q = 0; q < ny; ++q) p->line[q] = base[(size_t)hx * q];
                oc_fft1_exec(p->fy, p->line, p->scratch, sign);
                for (int q = 0; q < ny; ++q) base[(size_t)hx * q] = p->line[q];
            }
    }
    if (nz > 1) {
        const size_t plane = (size_t)hx * ny;
        for (int q = 0; q < ny; ++q)
            for (int k = 0; k < hx; ++k) {
                oc_complex* base = spec + k + (size_t)hx * q;
                for (int r = 0; r < nz; ++r) p->line[r] = base[plane * r];
                oc_fft1_exec(p->fz, p->line, p->scratch, sign);
                for (int r = 0; r < nz; ++r) base[plane * r] = p->line[r];
            }
    }
}

void oc_fft3_r2c(oc_fft3* p, const double* in, oc_complex* out) {
    const int nx = p->nx, ny = p->ny, nz = p->nz, hx = p->hx;
    const int even = (nx % 2 == 0) && nx >= 2;
    for (size_t l = 0; l < (size_t)ny * nz; ++l) {
        const double* x = in + l * nx;
        oc_complex* X = out + l * hx;
        if (even) {
            const int h = nx / 2;
            for (int j = 0; j < h; ++j) {
                p->line[j].re = x[2 * j];
                p->line[j].im = x[2 * j + 1];
            }
            oc_fft1_exec(p->fx, p->line, p->scratch, -1);
            for (int k = 0; k <= h; ++k) {
                const oc_complex zk = p->line[k % h];
                const oc_complex zc = cconj(p->line[(h - k) % h]);
                const oc_complex e = {0.5 * (zk.re + zc.re), 0.5 * (zk.im + zc.im)};
                /* o = (zk - zc) / (2i) */
                const oc_complex o = {0.5 * (zk.im - zc.im), -0.5 * (zk.re - zc.re)};
                const oc_complex wo = cmul(p->xtw[k], o);
                X[k].re = e.re + wo.re;
                X[k].im = e.im + wo.im;
            }
        } else {
            for (int j = 0; j < nx; ++j) {
                p->line[j].re = x[j];
                p->line[j].im = 0.0;
            }
            oc_fft1_exec(p->fx, p->line, p->scratch, -1);
            for (int k = 0; k < hx; ++k) X[k] = p->line[k];
        }
    }
    yz_pass(p, out, -1);
}

void oc_fft3_c2r(oc_fft3* p, const oc_complex* in, double* out) {
    const int nx = p->nx, ny = p->ny, nz = p->nz, hx = p->hx;
    const int even = (nx % 2 == 0) && nx >= 2;
    memcpy(p->work, in, sizeof(oc_complex) * (size_t)hx * ny * nz);
    yz_pass(p, p->work, +1);
    for (size_t l = 0; l < (size_t)ny * nz; ++l) {
        oc_complex* X = p->work + l * hx;
        double* x = out + l * nx;
        X[0].im = 0.0;
        if (even) {
            const int h = nx / 2;
            X[h].im = 0.0;
            for (int k = 0; k < h; ++k) {
                const oc_complex a = X[k];
                const oc_complex b = cconj(X[h - k]);
                const oc_complex e = {a.re + b.re, a.im + b.im};
                const oc_complex d = {a.re - b.re, a.im - b.im};
                const oc_complex o = cmul(d, cconj(p->xtw[k]));
                /* Z = E + i O */
                p->line[k].re = e.re - o.im;
                p->line[k].im = e.im + o.re;
            }
            oc_fft1_exec(p->fx, p->line, p->scratch, +1);
            for (int j = 0; j < h; ++j) {
                x[2 * j] = p->line[j].re;
                x[2 * j + 1] = p->line[j].im;
            }
        } else {
            p->line[0] = X[0];
            for (int k = 1; k < hx; ++k) {
                p->line[k] = X[k];
                p->line[nx - k] = cconj(X[k]);
            }
            oc_fft1_exec(p->fx, p->line, p->scratch, +1);
            for (int j = 0; j < nx; ++j) x[j] = p->line[j].re;
        }
    }
}
