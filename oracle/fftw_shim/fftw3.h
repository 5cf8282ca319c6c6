/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Minimal FFTW3-API provider so the reference's unmodified
 * /root/reference/proj/src/fourier.cpp (which includes <fftw3.h> at :3 and
 * calls fftw_plan_dft_1d / fftw_execute / fftw_destroy_plan at :22-35) can be
 * compiled here, where libfftw3 is not installed.  Only the
 * three entry points and the constants the reference uses are declared.
 * Semantics follow the FFTW 3 manual for a 1D complex DFT: unnormalised,
 * FFTW_FORWARD = -1, FFTW_BACKWARD = +1; in == out allowed.  The arithmetic
 * is oracle/skfft.cpp (Stockham radix 4/2/3/5/7/odd-prime + Bluestein). */
#ifndef SK_FFTW3_SHIM_H
#define SK_FFTW3_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
#endif
