/*
 * TEST INFRASTRUCTURE ONLY -- never linked into the product library.
 *
 * Double-precision mixed-radix FFT used by the CPU oracle.  It plays the role of
 * FFTW3 (double) in the reference (`proj/core/src/fft.cpp:52-55`, r2c/c2r 3-D,
 * unnormalised, x fastest = last FFTW dimension), which is absent from this image.
 * Two consumers:
 *   - oracle/dreg_oracle.c  : the plain-C restatement of the reference path;
 *   - oracle/fftw_shim/     : an FFTW-API shim so the UNMODIFIED reference sources
 *                             (proj/core/src, all .cpp files) compile into oracle/_ref/.
 * Validated against numpy.fft (pocketfft) in tests/test_oracle_fft.py.
 */
#ifndef DREG_ORACLE_FFT_CORE_H
#define DREG_ORACLE_FFT_CORE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } oc_complex;

typedef struct oc_fft1 oc_fft1;  /* 1-D complex plan of length n */

oc_fft1* oc_fft1_create(int n);
void oc_fft1_destroy(oc_fft1* p);
/* In-place unnormalised DFT; sign = -1 forward (e^{-2 pi i jk/n}), +1 inverse.
 * scratch must hold n entries. */
void oc_fft1_exec(const oc_fft1* p, oc_complex* data, oc_complex* scratch, int sign);

/* 3-D real transforms on an (nx, ny, nz) x-fastest grid.  Half spectrum layout is
 * bin = p + (nx/2+1) * (q + ny * r), exactly the reference's `Fft3::bin`
 * (`proj/core/include/dreg/fft.hpp:37-41`). */
typedef struct oc_fft3 oc_fft3;

oc_fft3* oc_fft3_create(int nx, int ny, int nz);
void oc_fft3_destroy(oc_fft3* p);
void oc_fft3_r2c(oc_fft3* p, const double* in, oc_complex* out);
/* c2r destroys nothing in `in` (works on a private copy); imaginary parts of the
 * self-conjugate x bins are ignored as a 1-D c2r does. */
void oc_fft3_c2r(oc_fft3* p, const oc_complex* in, double* out);

#ifdef __cplusplus
}
#endif

#endif
