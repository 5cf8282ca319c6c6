// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// skfft: a small, self-contained double-precision complex FFT used by
//   (1) the FFTW-API shim (oracle/fftw_shim) that lets the reference's own
//       sources (/root/reference/proj/src/fourier.cpp:22-35 call
//       fftw_plan_dft_1d / fftw_execute / fftw_destroy_plan) compile and run
//       here, where libfftw3 is not installed;
//   (2) the C++ restatement of the hot path (oracle/sk_oracle.cpp).
//
// Semantics follow FFTW's documented 1D complex DFT (the third-party
// algorithm the reference calls; version unpinned by the reference's
// CMakeLists, proj/CMakeLists.txt:13):
//     out[k] = sum_j in[j] * exp(sign * 2*pi*i * j*k / n),  unnormalised,
// sign = -1 (FFTW_FORWARD) or +1 (FFTW_BACKWARD); in-place allowed.
// Algorithm: Stockham autosort, radices 4/2/3/5/7 plus a direct odd-prime
// pass for primes <= 61 and Bluestein (chirp-z) otherwise.
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct skfft_plan skfft_plan;

skfft_plan* skfft_plan_create(int n, int sign);
// in and out are interleaved (re, im) arrays of n complex values; may alias.
void skfft_execute(const skfft_plan* p, const double* in, double* out);
void skfft_destroy(skfft_plan* p);

#ifdef __cplusplus
}
#endif
