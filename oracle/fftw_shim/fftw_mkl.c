/*
 * TEST / BASELINE INFRASTRUCTURE ONLY -- the FFTW3 API subset the reference uses
 * (fft.cpp:23-69), backed by Intel MKL's DFTI (the copy exported by PyTorch's
 * libtorch_cpu.so, dlopen'ed at first use).  Used only for TIMING the reference CPU
 * path (oracle/_ref/libdreg_ref_mkl.so: bench.py's cpu_baseline and --impl reference),
 * so the baseline runs on a production FFT like the FFTW the reference links, not on
 * the portable parity shim (fftw_shim.c, ~pocketfft speed).  Parity tests keep the
 * portable shim (bit-exact vs the C restatement).
 *
 * mkl_dfti.h is not in the image; the enum values below are Intel's published DFTI
 * constants.  Transforms are unnormalised like FFTW (default scales 1.0),
 * out-of-place, conjugate-even storage as complex (CCE) -- FFTW's r2c layout: row-major
 * (n0, n1, n2/2+1).  Each plan is single-threaded (DFTI_THREAD_LIMIT 1): the
 * throughput baseline runs one reference registration per host core.
 */
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>

#include "fftw3.h"

typedef void* DFTI_HANDLE;
enum { DFTI_PLACEMENT = 11, DFTI_INPUT_STRIDES = 12, DFTI_OUTPUT_STRIDES = 13, DFTI_CONJUGATE_EVEN_STORAGE = 10,
       DFTI_THREAD_LIMIT = 27 };
enum { DFTI_REAL = 33, DFTI_COMPLEX_COMPLEX = 39, DFTI_NOT_INPLACE = 44 };

typedef long (*create_md_t)(DFTI_HANDLE*, int, long, long*);
typedef long (*set_t)(DFTI_HANDLE, int, ...);
typedef long (*commit_t)(DFTI_HANDLE);
typedef long (*compute_t)(DFTI_HANDLE, void*, void*);
typedef long (*free_t)(DFTI_HANDLE*);

static create_md_t p_create;
static set_t p_set;
static commit_t p_commit;
static compute_t p_fwd, p_bwd;
static free_t p_free;

#ifndef DREG_TORCH_LIB
#define DREG_TORCH_LIB "libtorch_cpu.so"
#endif

static void load(void) {
    if (p_create) return;
    const char* path = getenv("DREG_MKL_LIB");
    void* h = dlopen(path ? path : DREG_TORCH_LIB, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        fprintf(stderr, "fftw_mkl: cannot load %s: %s\n", path ? path : DREG_TORCH_LIB, dlerror());
        abort();
    }
    p_set = (set_t)dlsym(h, "DftiSetValue");
    p_commit = (commit_t)dlsym(h, "DftiCommitDescriptor");
    p_fwd = (compute_t)dlsym(h, "DftiComputeForward");
    p_bwd = (compute_t)dlsym(h, "DftiComputeBackward");
    p_free = (free_t)dlsym(h, "DftiFreeDescriptor");
    p_create = (create_md_t)dlsym(h, "DftiCreateDescriptor_d_md");
    if (!p_create || !p_set || !p_commit || !p_fwd || !p_bwd || !p_free) {
        fprintf(stderr, "fftw_mkl: DFTI symbols missing\n");
        abort();
    }
}

struct fftw_plan_s {
    DFTI_HANDLE d;
    int forward;
    double* real;
    fftw_complex* cplx;
};

static void check(long st, const char* what) {
    if (st != 0) {
        fprintf(stderr, "fftw_mkl: %s failed (%ld)\n", what, st);
        abort();
    }
}

static fftw_plan make(int n0, int n1, int n2, double* real, fftw_complex* cplx, int fwd) {
    load();
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    long n[3] = {n0, n1, n2};
    long rs[4] = {0, (long)n1 * n2, n2, 1};
    long cs[4] = {0, (long)n1 * (n2 / 2 + 1), n2 / 2 + 1, 1};
    check(p_create(&p->d, DFTI_REAL, 3, n), "DftiCreateDescriptor");
    check(p_set(p->d, DFTI_PLACEMENT, DFTI_NOT_INPLACE), "placement");
    check(p_set(p->d, DFTI_CONJUGATE_EVEN_STORAGE, DFTI_COMPLEX_COMPLEX), "storage");
    check(p_set(p->d, DFTI_INPUT_STRIDES, fwd ? rs : cs), "input strides");
    check(p_set(p->d, DFTI_OUTPUT_STRIDES, fwd ? cs : rs), "output strides");
    check(p_set(p->d, DFTI_THREAD_LIMIT, 1L), "thread limit");
    check(p_commit(p->d), "commit");
    p->forward = fwd;
    p->real = real;
    p->cplx = cplx;
    return p;
}

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned flags) {
    (void)flags;
    return make(n0, n1, n2, in, out, 1);
}

fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned flags) {
    (void)flags;
    return make(n0, n1, n2, out, in, 0);
}

void fftw_execute(const fftw_plan p) {
    if (p->forward) check(p_fwd(p->d, p->real, p->cplx), "forward");
    else check(p_bwd(p->d, p->cplx, p->real), "backward");
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    p_free(&p->d);
    free(p);
}
