// Device-side FFT engine: in-place mixed-radix Cooley-Tukey in shared memory.
//
// Replaces the FFTW calls of fourier.cpp:22-35 (run_fft, one plan per 1D
// transform under a global mutex).  Here a whole CTA transforms one sequence
// resident in shared memory: forward stages are decimation-in-frequency
// (natural order in, digit-reversed out), inverse stages decimation-in-time
// (digit-reversed in, natural out), so a forward + pointwise/solve + inverse
// sequence never needs a reordering pass.  Each butterfly reads and writes the
// same R slots, so stages need no ping-pong buffer and only R complex values
// per thread live in registers.
#pragma once

#include <cuda_runtime.h>

#include "sk_internal.h"

namespace sk {

struct cd {
    double x, y;
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }
// multiply by (sign * i)
template <int SIGN>
__device__ __forceinline__ double2 mul_si(double2 a) {
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

// Twiddle table access (exp(-2 pi i m / 2L)), tables staged in shared memory.
struct Tw {
    const double2* hi;
    const double2* lo;
    int shift;
    int mask;
    __device__ __forceinline__ double2 operator()(int m) const { return cmul(hi[m >> shift], lo[m & mask]); }
};

// ---------------------------------------------------------------- radix DFTs
// y_s = sum_q x_q exp(SIGN 2 pi i q s / R), in place.
template <int SIGN>
__device__ __forceinline__ void dft2(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2* x) {
    const double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    const double2 t2 = cadd(x[1], x[3]), t3 = mul_si<SIGN>(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* x) {
    constexpr double r = 0.70710678118654752440084436210484903928;
    double2 e[4] = {x[0], x[2], x[4], x[6]};
    double2 o[4] = {x[1], x[3], x[5], x[7]};
    dft4<SIGN>(e);
    dft4<SIGN>(o);
    // W^1 = r (1 + SIGN i), W^2 = SIGN i, W^3 = r (-1 + SIGN i)
    const double2 w1o = make_double2(r * (o[1].x - SIGN * o[1].y), r * (o[1].y + SIGN * o[1].x));
    const double2 w2o = mul_si<SIGN>(o[2]);
    const double2 w3o = make_double2(r * (-o[3].x - SIGN * o[3].y), r * (-o[3].y + SIGN * o[3].x));
    x[0] = cadd(e[0], o[0]);
    x[4] = csub(e[0], o[0]);
    x[1] = cadd(e[1], w1o);
    x[5] = csub(e[1], w1o);
    x[2] = cadd(e[2], w2o);
    x[6] = csub(e[2], w2o);
    x[3] = cadd(e[3], w3o);
    x[7] = csub(e[3], w3o);
}

template <int SIGN>
__device__ __forceinline__ void dft3(double2* x) {
    constexpr double s3 = 0.86602540378443864676372317075293618347;  // sin(2pi/3)
    const double2 t1 = cadd(x[1], x[2]);
    const double2 t2 = make_double2(x[0].x - 0.5 * t1.x, x[0].y - 0.5 * t1.y);
    const double2 t3 = mul_si<SIGN>(cscale(csub(x[1], x[2]), s3));
    x[0] = cadd(x[0], t1);
    x[1] = cadd(t2, t3);
    x[2] = csub(t2, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft5(double2* x) {
    constexpr double c1 = 0.30901699437494742410229341718281905886;   // cos(2pi/5)
    constexpr double c2 = -0.80901699437494742410229341718281905886;  // cos(4pi/5)
    constexpr double s1 = 0.95105651629515357211643933337938214340;   // sin(2pi/5)
    constexpr double s2 = 0.58778525229247312916870595463907276860;   // sin(4pi/5)
    const double2 t1 = cadd(x[1], x[4]), t2 = cadd(x[2], x[3]);
    const double2 t3 = csub(x[1], x[4]), t4 = csub(x[2], x[3]);
    const double2 a1 = make_double2(x[0].x + c1 * t1.x + c2 * t2.x, x[0].y + c1 * t1.y + c2 * t2.y);
    const double2 a2 = make_double2(x[0].x + c2 * t1.x + c1 * t2.x, x[0].y + c2 * t1.y + c1 * t2.y);
    const double2 b1 = mul_si<SIGN>(make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y));
    const double2 b2 = mul_si<SIGN>(make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y));
    x[0] = make_double2(x[0].x + t1.x + t2.x, x[0].y + t1.y + t2.y);
    x[1] = cadd(a1, b1);
    x[4] = csub(a1, b1);
    x[2] = cadd(a2, b2);
    x[3] = csub(a2, b2);
}

template <int SIGN>
__device__ __forceinline__ void dft7(double2* x) {
    // c[q][s] = cos(2 pi q s / 7), sn[q][s] = sin(2 pi q s / 7), q,s = 1..3
    constexpr double C1 = 0.62348980185873353052500488400423981063;
    constexpr double C2 = -0.22252093395631440428890256449679475947;
    constexpr double C3 = -0.90096886790241912623610231950744505116;
    constexpr double S1 = 0.78183148246802980870844452667405775023;
    constexpr double S2 = 0.97492791218182360701813168299393121723;
    constexpr double S3 = 0.43388373911755812047576833284835875461;
    const double2 p1 = cadd(x[1], x[6]), p2 = cadd(x[2], x[5]), p3 = cadd(x[3], x[4]);
    const double2 m1 = csub(x[1], x[6]), m2 = csub(x[2], x[5]), m3 = csub(x[3], x[4]);
    const double2 x0 = x[0];
    auto A = [&](double a, double b, double c) {
        return make_double2(x0.x + a * p1.x + b * p2.x + c * p3.x, x0.y + a * p1.y + b * p2.y + c * p3.y);
    };
    auto B = [&](double a, double b, double c) {
        return mul_si<SIGN>(make_double2(a * m1.x + b * m2.x + c * m3.x, a * m1.y + b * m2.y + c * m3.y));
    };
    const double2 a1 = A(C1, C2, C3), b1 = B(S1, S2, S3);
    const double2 a2 = A(C2, C3, C1), b2 = B(S2, -S3, -S1);
    const double2 a3 = A(C3, C1, C2), b3 = B(S3, -S1, S2);
    x[0] = make_double2(x0.x + p1.x + p2.x + p3.x, x0.y + p1.y + p2.y + p3.y);
    x[1] = cadd(a1, b1);
    x[6] = csub(a1, b1);
    x[2] = cadd(a2, b2);
    x[5] = csub(a2, b2);
    x[3] = cadd(a3, b3);
    x[4] = csub(a3, b3);
}

// exp(-2 pi i m / R) for the composite radices (correctly rounded constants)
static __constant__ double2 kW10[10] = {{1, 0}, {0.80901699437494745, -0.58778525229247314}, {0.30901699437494745, -0.95105651629515353}, {-0.30901699437494745, -0.95105651629515353}, {-0.80901699437494745, -0.58778525229247314}, {-1, 0}, {-0.80901699437494745, 0.58778525229247314}, {-0.30901699437494745, 0.95105651629515353}, {0.30901699437494745, 0.95105651629515353}, {0.80901699437494745, 0.58778525229247314}};
static __constant__ double2 kW16[16] = {{1, 0}, {0.92387953251128674, -0.38268343236508978}, {0.70710678118654757, -0.70710678118654757}, {0.38268343236508978, -0.92387953251128674}, {0, -1}, {-0.38268343236508978, -0.92387953251128674}, {-0.70710678118654757, -0.70710678118654757}, {-0.92387953251128674, -0.38268343236508978}, {-1, 0}, {-0.92387953251128674, 0.38268343236508978}, {-0.70710678118654757, 0.70710678118654757}, {-0.38268343236508978, 0.92387953251128674}, {0, 1}, {0.38268343236508978, 0.92387953251128674}, {0.70710678118654757, 0.70710678118654757}, {0.92387953251128674, 0.38268343236508978}};
static __constant__ double2 kW20[20] = {{1, 0}, {0.95105651629515353, -0.30901699437494745}, {0.80901699437494745, -0.58778525229247314}, {0.58778525229247314, -0.80901699437494745}, {0.30901699437494745, -0.95105651629515353}, {0, -1}, {-0.30901699437494745, -0.95105651629515353}, {-0.58778525229247314, -0.80901699437494745}, {-0.80901699437494745, -0.58778525229247314}, {-0.95105651629515353, -0.30901699437494745}, {-1, 0}, {-0.95105651629515353, 0.30901699437494745}, {-0.80901699437494745, 0.58778525229247314}, {-0.58778525229247314, 0.80901699437494745}, {-0.30901699437494745, 0.95105651629515353}, {0, 1}, {0.30901699437494745, 0.95105651629515353}, {0.58778525229247314, 0.80901699437494745}, {0.80901699437494745, 0.58778525229247314}, {0.95105651629515353, 0.30901699437494745}};
static __constant__ double2 kW25[25] = {{1, 0}, {0.96858316112863108, -0.24868988716485479}, {0.87630668004386358, -0.48175367410171527}, {0.72896862742141155, -0.68454710592868873}, {0.53582679497899666, -0.84432792550201508}, {0.30901699437494745, -0.95105651629515353}, {0.062790519529313374, -0.99802672842827156}, {-0.18738131458572463, -0.98228725072868872}, {-0.42577929156507266, -0.90482705246601958}, {-0.63742398974868975, -0.77051324277578925}, {-0.80901699437494745, -0.58778525229247314}, {-0.92977648588825146, -0.36812455268467797}, {-0.99211470131447788, -0.12533323356430426}, {-0.99211470131447788, 0.12533323356430426}, {-0.92977648588825146, 0.36812455268467797}, {-0.80901699437494745, 0.58778525229247314}, {-0.63742398974868975, 0.77051324277578925}, {-0.42577929156507266, 0.90482705246601958}, {-0.18738131458572463, 0.98228725072868872}, {0.062790519529313374, 0.99802672842827156}, {0.30901699437494745, 0.95105651629515353}, {0.53582679497899666, 0.84432792550201508}, {0.72896862742141155, 0.68454710592868873}, {0.87630668004386358, 0.48175367410171527}, {0.96858316112863108, 0.24868988716485479}};
static __constant__ double2 kW32[32] = {{1, 0}, {0.98078528040323043, -0.19509032201612828}, {0.92387953251128674, -0.38268343236508978}, {0.83146961230254524, -0.55557023301960218}, {0.70710678118654757, -0.70710678118654757}, {0.55557023301960218, -0.83146961230254524}, {0.38268343236508978, -0.92387953251128674}, {0.19509032201612828, -0.98078528040323043}, {0, -1}, {-0.19509032201612828, -0.98078528040323043}, {-0.38268343236508978, -0.92387953251128674}, {-0.55557023301960218, -0.83146961230254524}, {-0.70710678118654757, -0.70710678118654757}, {-0.83146961230254524, -0.55557023301960218}, {-0.92387953251128674, -0.38268343236508978}, {-0.98078528040323043, -0.19509032201612828}, {-1, 0}, {-0.98078528040323043, 0.19509032201612828}, {-0.92387953251128674, 0.38268343236508978}, {-0.83146961230254524, 0.55557023301960218}, {-0.70710678118654757, 0.70710678118654757}, {-0.55557023301960218, 0.83146961230254524}, {-0.38268343236508978, 0.92387953251128674}, {-0.19509032201612828, 0.98078528040323043}, {0, 1}, {0.19509032201612828, 0.98078528040323043}, {0.38268343236508978, 0.92387953251128674}, {0.55557023301960218, 0.83146961230254524}, {0.70710678118654757, 0.70710678118654757}, {0.83146961230254524, 0.55557023301960218}, {0.92387953251128674, 0.38268343236508978}, {0.98078528040323043, 0.19509032201612828}};

template <int R>
__device__ __forceinline__ double2 wconst(int m) {
    if constexpr (R == 10) return kW10[m];
    else if constexpr (R == 16) return kW16[m];
    else if constexpr (R == 20) return kW20[m];
    else if constexpr (R == 25) return kW25[m];
    else return kW32[m];
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(double2* x);

// DFT of length R = R1 R2 in registers (Cooley-Tukey, n = R2 n1 + n2,
// k = k1 + R1 k2): R2 inner DFTs of length R1, constant twiddles
// exp(SIGN 2 pi i n2 k1 / R), R1 outer DFTs of length R2; natural order out.
template <int R1, int R2, int SIGN>
__device__ __forceinline__ void dftc(double2* x) {
    constexpr int R = R1 * R2;
    double2 z[R];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
        double2 y[R1];
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) y[n1] = x[R2 * n1 + n2];
        dft<R1, SIGN>(y);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            const int m = (n2 * k1) % R;
            if (m == 0) {
                z[k1 * R2 + n2] = y[k1];
            } else {
                double2 w = wconst<R>(m);
                if (SIGN > 0) w.y = -w.y;
                z[k1 * R2 + n2] = cmul(y[k1], w);
            }
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
        double2 y[R2];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) y[n2] = z[k1 * R2 + n2];
        dft<R2, SIGN>(y);
#pragma unroll
        for (int k2 = 0; k2 < R2; ++k2) x[k1 + R1 * k2] = y[k2];
    }
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(double2* x) {
    if constexpr (R == 2) dft2<SIGN>(x);
    else if constexpr (R == 3) dft3<SIGN>(x);
    else if constexpr (R == 4) dft4<SIGN>(x);
    else if constexpr (R == 5) dft5<SIGN>(x);
    else if constexpr (R == 7) dft7<SIGN>(x);
    else if constexpr (R == 8) dft8<SIGN>(x);
    else if constexpr (R == 10) dftc<2, 5, SIGN>(x);
    else if constexpr (R == 16) dftc<4, 4, SIGN>(x);
    else if constexpr (R == 20) dftc<4, 5, SIGN>(x);
    else if constexpr (R == 25) dftc<5, 5, SIGN>(x);
    else dftc<4, 8, SIGN>(x);
}

// ------------------------------------------------------------------- stages
__device__ __forceinline__ int fdiv(int n, unsigned mag, int sh1, int sh2) {
    const unsigned t = __umulhi(static_cast<unsigned>(n), mag);
    return static_cast<int>((t + ((static_cast<unsigned>(n) - t) >> sh1)) >> sh2);
}

// Shared-memory slot swizzle: XOR the low three bits of a complex slot index
// with a hash of its higher bits (a bijection on every aligned 8-slot block),
// so indices that differ by multiples of 8 slots hit different banks.
template <bool SWZ>
__device__ __forceinline__ int swz(int p) {
    if constexpr (SWZ) return p ^ (((p >> 3) ^ (p >> 6) ^ (p >> 9) ^ (p >> 12)) & 7);
    else return p;
}

// One butterfly's registers.
template <int R>
struct Bfly {
    double2 x[R];
    int base, j;
};

template <int R, bool SWZ>
__device__ __forceinline__ void bf_load(Bfly<R>& B, const double2* a, int b, int span, unsigned mag, int sh1, int sh2) {
    const int g = fdiv(b, mag, sh1, sh2);
    B.j = b - g * span;
    B.base = g * span * R + B.j;
#pragma unroll
    for (int q = 0; q < R; ++q) B.x[q] = a[swz<SWZ>(B.base + q * span)];
}

// Twiddle powers w^q, q = 1..R-1, w = T(j tw) for SIGN = -1 (exp(-2 pi i ...))
// and its conjugate for SIGN = +1, built by repeated multiplication.
template <int R, int SIGN>
__device__ __forceinline__ void bf_twiddle(double2* x, int j, int tw, const Tw& T) {
    if (j == 0) return;
    double2 w1 = T(j * tw);
    if (SIGN > 0) w1.y = -w1.y;
    double2 w = w1;
#pragma unroll
    for (int q = 1; q < R; ++q) {
        x[q] = cmul(x[q], w);
        if (q + 1 < R) w = cmul(w, w1);
    }
}

// DIF butterfly: y = DFT_R(x); y_q *= w^(q j); store in place.
template <int R, int SIGN, bool SWZ>
__device__ __forceinline__ void bf_dif(Bfly<R>& B, double2* a, int span, int tw, const Tw& T) {
    dft<R, SIGN>(B.x);
    bf_twiddle<R, SIGN>(B.x, B.j, tw, T);
#pragma unroll
    for (int q = 0; q < R; ++q) a[swz<SWZ>(B.base + q * span)] = B.x[q];
}

// DIT butterfly: x_q *= w^(q j); y = DFT_R(x); store in place.
template <int R, int SIGN, bool SWZ>
__device__ __forceinline__ void bf_dit(Bfly<R>& B, double2* a, int span, int tw, const Tw& T) {
    bf_twiddle<R, SIGN>(B.x, B.j, tw, T);
    dft<R, SIGN>(B.x);
#pragma unroll
    for (int q = 0; q < R; ++q) a[swz<SWZ>(B.base + q * span)] = B.x[q];
}

// One stage over all butterflies; small radices keep two butterflies'
// shared-memory loads in flight.
// nb_lim >= 0: only the first nb_lim butterflies (the leading sub-transforms
// of a pruned forward transform, theta_sym.cu).
template <int R, bool DIF, int SIGN, bool SWZ>
__device__ __forceinline__ void fft_stage(double2* a, const FftDesc& d, int s, const Tw& T, int tid, int nthr,
                                          int nb_lim = -1) {
    const int span = d.span[s], tw = d.tw[s];
    const unsigned mag = d.mag[s];
    const int sh1 = d.sh1[s], sh2 = d.sh2[s];
    const int nb = nb_lim >= 0 ? nb_lim : d.L / R;
    int b = tid;
    if constexpr (R <= 8) {
        for (; b + nthr < nb; b += 2 * nthr) {
            Bfly<R> p, q;
            bf_load<R, SWZ>(p, a, b, span, mag, sh1, sh2);
            bf_load<R, SWZ>(q, a, b + nthr, span, mag, sh1, sh2);
            if constexpr (DIF) {
                bf_dif<R, SIGN, SWZ>(p, a, span, tw, T);
                bf_dif<R, SIGN, SWZ>(q, a, span, tw, T);
            } else {
                bf_dit<R, SIGN, SWZ>(p, a, span, tw, T);
                bf_dit<R, SIGN, SWZ>(q, a, span, tw, T);
            }
        }
    }
    for (; b < nb; b += nthr) {
        Bfly<R> p;
        bf_load<R, SWZ>(p, a, b, span, mag, sh1, sh2);
        if constexpr (DIF) bf_dif<R, SIGN, SWZ>(p, a, span, tw, T);
        else bf_dit<R, SIGN, SWZ>(p, a, span, tw, T);
    }
}

// MAXR: largest radix the caller's plans use (kernels compiled for a small
// register budget only instantiate the small radices).
template <bool DIF, int SIGN, bool SWZ, int MAXR = 25>
__device__ __forceinline__ void fft_stage_dispatch(double2* a, const FftDesc& d, int s, const Tw& T, int tid,
                                                   int nthr, int nb_lim = -1) {
    if constexpr (MAXR > 8) {
        switch (d.R[s]) {
            case 2: fft_stage<2, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 3: fft_stage<3, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 4: fft_stage<4, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 5: fft_stage<5, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 7: fft_stage<7, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 8: fft_stage<8, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 10: fft_stage<10, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 16: fft_stage<16, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 20: fft_stage<20, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            default: fft_stage<25, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
        }
    } else {  // plans built with radices <= 8 (the plan checks this)
        switch (d.R[s]) {
            case 2: fft_stage<2, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 3: fft_stage<3, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 4: fft_stage<4, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 5: fft_stage<5, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            case 7: fft_stage<7, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
            default: fft_stage<8, DIF, SIGN, SWZ>(a, d, s, T, tid, nthr, nb_lim); break;
        }
    }
}

template <bool DIF, int SIGN, bool SWZ, int MAXR = 25>
__device__ __forceinline__ void fft_run(double2* a, const FftDesc& d, const Tw& T, int tid, int nthr) {
    if constexpr (DIF) {
        for (int s = 0; s < d.nst; ++s) {
            fft_stage_dispatch<true, SIGN, SWZ, MAXR>(a, d, s, T, tid, nthr);
            __syncthreads();
        }
    } else {
        for (int s = d.nst - 1; s >= 0; --s) {
            fft_stage_dispatch<false, SIGN, SWZ, MAXR>(a, d, s, T, tid, nthr);
            __syncthreads();
        }
    }
}
template <bool SWZ = false, int MAXR = 25>
__device__ __forceinline__ void fft_forward(double2* a, const FftDesc& d, const Tw& T, int tid, int nthr) {
    fft_run<true, -1, SWZ, MAXR>(a, d, T, tid, nthr);
}
template <bool SWZ = false, int MAXR = 25>
__device__ __forceinline__ void fft_inverse(double2* a, const FftDesc& d, const Tw& T, int tid, int nthr) {
    fft_run<false, +1, SWZ, MAXR>(a, d, T, tid, nthr);
}

// Stage the 2L-th-root twiddle tables of `d` into shared memory.
__device__ __forceinline__ Tw load_tw(const FftDesc& d, double2* s_hi, double2* s_lo, int tid, int nthr) {
    for (int i = tid; i < d.nhi; i += nthr) s_hi[i] = d.hi[i];
    for (int i = tid; i < d.nlo; i += nthr) s_lo[i] = d.lo[i];
    return Tw{s_hi, s_lo, d.shift, (1 << d.shift) - 1};
}

}  // namespace sk
