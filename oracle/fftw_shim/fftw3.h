/*
 * TEST INFRASTRUCTURE ONLY.  Minimal FFTW3 (double) API shim so the unmodified
 * reference `proj/core/src/fft.cpp` compiles into oracle/_ref/ in an image without
 * libfftw3.  Declares exactly the symbols that file uses (`fft.cpp:23-24,29-32,
 * 52-55,67,69`); the transforms are computed by oracle/fft_core.c.
 * FFTW3 itself is unpinned in the reference (`core/cmake/dreg-fftw.cmake:3-4`).
 */
#ifndef DREG_ORACLE_FFTW3_SHIM_H
#define DREG_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out,
                               unsigned flags);
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out,
                               unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
