/*
 * TEST INFRASTRUCTURE ONLY -- FFTW3 API shim over oracle/fft_core.c (see fftw3.h).
 * Row-major (n0, n1, n2) with n2 fastest, as FFTW defines it; the reference passes
 * (z, y, x) so x is the halved axis (`proj/core/src/fft.cpp:52-55`).
 */
#include "fftw3.h"

#include <stdlib.h>

#include "../fft_core.h"

struct fftw_plan_s {
    int forward;
    oc_fft3* fft;
    double* real;
    oc_complex* cplx;
};

static fftw_plan make(int n0, int n1, int n2, double* real, fftw_complex* cplx, int fwd) {
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->forward = fwd;
    p->fft = oc_fft3_create(n2, n1, n0);
    p->real = real;
    p->cplx = (oc_complex*)cplx;
    if (!p->fft) {
        free(p);
        return NULL;
    }
    return p;
}

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out,
                               unsigned flags) {
    (void)flags;
    return make(n0, n1, n2, in, out, 1);
}

fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out,
                               unsigned flags) {
    (void)flags;
    return make(n0, n1, n2, out, in, 0);
}

void fftw_execute(const fftw_plan p) {
    if (p->forward) oc_fft3_r2c(p->fft, p->real, p->cplx);
    else oc_fft3_c2r(p->fft, p->cplx, p->real);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    oc_fft3_destroy(p->fft);
    free(p);
}
