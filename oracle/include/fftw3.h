/*
 * TEST INFRASTRUCTURE — oracle only, never linked into the product.
 *
 * Declarations of the nine FFTW3 (double precision) entry points that the
 * reference's FFT layer calls (reference: proj/src/fft_plan.cpp:19,35,59-66,
 * 72-75,87,94).  FFTW itself is not installed in this image and its version is
 * unpinned by the reference (proj/CMakeLists.txt:14-16 uses find_library), so
 * oracle/fftw_shim.c implements these symbols with a double-precision
 * mixed-radix CPU FFT.  Semantics follow FFTW's published contract:
 * row-major multi-dimensional r2c with the last axis halved to n/2+1,
 * unnormalised c2r that reads only the Hermitian half.
 */
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

int fftw_init_threads(void);
void fftw_plan_with_nthreads(int nthreads);
double* fftw_alloc_real(size_t n);
fftw_complex* fftw_alloc_complex(size_t n);
fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in,
                            fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in,
                            double* out, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);
void fftw_free(void* p);

#ifdef __cplusplus
}
#endif
