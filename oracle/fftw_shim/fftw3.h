/*
 * ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * Minimal FFTW3-API shim so the UNMODIFIED reference sources
 * (/root/reference/proj/src/*.cpp) compile and link in a container that has
 * no FFTW3.  Only the surface the reference uses is provided
 * (reference proj/src/fft.cpp:3,25-28,42): fftw_plan_dft_2d with
 * FFTW_ESTIMATE|FFTW_UNALIGNED, fftw_execute_dft (re-entrant across threads),
 * FFTW_FORWARD (-1) / FFTW_BACKWARD (+1), unnormalised like FFTW.
 *
 * The transform is our own iterative radix-2 code for power-of-two axes and a
 * direct DFT for any other length (the reference FFT tests use 16x12 and 4x5,
 * proj/tests/test_field_fft.cpp:75-112).  It is NOT FFTW: CPU timings made with
 * this shim say so.
 */
#ifndef PDD_FFTW_SHIM_H
#define PDD_FFTW_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct pdd_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
