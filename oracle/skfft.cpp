// ORACLE / TEST INFRASTRUCTURE ONLY — see skfft.h.
#include "skfft.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.141592653589793238462643383279502884;

// exp(sign * 2 pi i m / n). The angle is reduced by quadrant (n % 4 == 0)
// or by the half-turn symmetry, so libm only sees angles <= pi/4 (resp. pi).
cd unit_root(long long m, long long n, int sign) {
    m %= n;
    if (m < 0) m += n;
    auto ang = [n](long long num) { return 2.0 * kPi * static_cast<double>(num) / static_cast<double>(n); };
    if (n % 4 == 0) {
        const long long quarter = n / 4;
        const long long q = m / quarter;  // quadrant 0..3
        const long long r = m - q * quarter;  // angle = q*pi/2 + ang(r)
        double c, s;
        if (2 * r > quarter) {  // use the complementary angle for accuracy
            const double a = ang(quarter - r);
            // cos(pi/2 - a) = sin a, sin(pi/2 - a) = cos a
            c = std::sin(a);
            s = std::cos(a);
        } else {
            const double a = ang(r);
            c = std::cos(a);
            s = std::sin(a);
        }
        double cc, ss;  // rotate (c, s) by q quarter turns
        switch (q & 3) {
            case 0: cc = c; ss = s; break;
            case 1: cc = -s; ss = c; break;
            case 2: cc = -c; ss = -s; break;
            default: cc = s; ss = -c; break;
        }
        return cd(cc, sign * ss);
    }
    if (2 * m > n) {
        const double a = ang(n - m);
        return cd(std::cos(a), -sign * std::sin(a));
    }
    const double a = ang(m);
    return cd(std::cos(a), sign * std::sin(a));
}

struct Stage {
    int p;
    long long ls;
    std::vector<cd> tw;  // tw[(q-1)*ls + k] = w^(q k n/(ls p)), q = 1..p-1, k = 0..ls-1
};

}  // namespace

struct skfft_plan {
    int n = 0;
    int sign = -1;
    std::vector<Stage> stages;
    std::vector<cd> w;  // w[m] = exp(sign 2 pi i m / n)
    // Bluestein
    bool bluestein = false;
    int L = 0;
    std::vector<cd> chirp;   // w_j = exp(sign pi i j^2 / n)
    std::vector<cd> bhat;    // FFT_L of conj chirp kernel
    skfft_plan* fwdL = nullptr;
    skfft_plan* invL = nullptr;
};

namespace {

// Complex arithmetic on (re, im) pairs written out (no std::complex calls in
// the inner loops).
struct C {
    double r, i;
};
inline C add(C a, C b) { return {a.r + b.r, a.i + b.i}; }
inline C sub(C a, C b) { return {a.r - b.r, a.i - b.i}; }
inline C mul(C a, C b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
inline C scl(C a, double s) { return {a.r * s, a.i * s}; }
// multiply by sign * i
inline C rot(C a, int sign) { return sign < 0 ? C{a.i, -a.r} : C{-a.i, a.r}; }

// One Stockham autosort stage of radix R: out[(j R + s) ls + k] =
// sum_q (in[j ls + k + q m ls] w^(q k n/(ls R))) omega_R^(q s), m = n/(ls R).
template <int R>
inline void butterfly(C* x, int sign);

template <>
inline void butterfly<2>(C* x, int) {
    const C a = x[0], b = x[1];
    x[0] = add(a, b);
    x[1] = sub(a, b);
}
template <>
inline void butterfly<4>(C* x, int sign) {
    const C t0 = add(x[0], x[2]), t1 = sub(x[0], x[2]);
    const C t2 = add(x[1], x[3]), t3 = rot(sub(x[1], x[3]), sign);
    x[0] = add(t0, t2);
    x[2] = sub(t0, t2);
    x[1] = add(t1, t3);
    x[3] = sub(t1, t3);
}
template <>
inline void butterfly<3>(C* x, int sign) {
    constexpr double s3 = 0.86602540378443864676372317075293618347;
    const C t1 = add(x[1], x[2]);
    const C t2 = {x[0].r - 0.5 * t1.r, x[0].i - 0.5 * t1.i};
    const C t3 = rot(scl(sub(x[1], x[2]), s3), sign);
    x[0] = add(x[0], t1);
    x[1] = add(t2, t3);
    x[2] = sub(t2, t3);
}
template <>
inline void butterfly<5>(C* x, int sign) {
    constexpr double c1 = 0.30901699437494742410229341718281905886;
    constexpr double c2 = -0.80901699437494742410229341718281905886;
    constexpr double s1 = 0.95105651629515357211643933337938214340;
    constexpr double s2 = 0.58778525229247312916870595463907276860;
    const C t1 = add(x[1], x[4]), t2 = add(x[2], x[3]);
    const C t3 = sub(x[1], x[4]), t4 = sub(x[2], x[3]);
    const C a1 = {x[0].r + c1 * t1.r + c2 * t2.r, x[0].i + c1 * t1.i + c2 * t2.i};
    const C a2 = {x[0].r + c2 * t1.r + c1 * t2.r, x[0].i + c2 * t1.i + c1 * t2.i};
    const C b1 = rot({s1 * t3.r + s2 * t4.r, s1 * t3.i + s2 * t4.i}, sign);
    const C b2 = rot({s2 * t3.r - s1 * t4.r, s2 * t3.i - s1 * t4.i}, sign);
    x[0] = {x[0].r + t1.r + t2.r, x[0].i + t1.i + t2.i};
    x[1] = add(a1, b1);
    x[4] = sub(a1, b1);
    x[2] = add(a2, b2);
    x[3] = sub(a2, b2);
}

template <int R>
void stage_fixed(const Stage& st, int n, int sign, const C* in, C* out) {
    const long long ls = st.ls;
    const long long m = n / (ls * R);
    const C* tw = reinterpret_cast<const C*>(st.tw.data());
    for (long long j = 0; j < m; ++j) {
        const C* ib = in + j * ls;
        C* ob = out + j * ls * R;
        {  // k = 0: no twiddles
            C x[R];
            for (int q = 0; q < R; ++q) x[q] = ib[q * m * ls];
            butterfly<R>(x, sign);
            for (int s = 0; s < R; ++s) ob[s * ls] = x[s];
        }
        for (long long k = 1; k < ls; ++k) {
            C x[R];
            x[0] = ib[k];
            for (int q = 1; q < R; ++q) x[q] = mul(ib[k + q * m * ls], tw[(q - 1) * ls + k]);
            butterfly<R>(x, sign);
            for (int s = 0; s < R; ++s) ob[k + s * ls] = x[s];
        }
    }
}

// Odd radices without a fixed butterfly (7 .. 61): direct O(R^2) DFT with the
// R-th roots from the plan's table.
void stage_generic(const skfft_plan* p, const Stage& st, const C* in, C* out) {
    const int n = p->n, r = st.p;
    const long long ls = st.ls;
    const long long m = n / (ls * r);
    const long long step = n / r;
    const C* w = reinterpret_cast<const C*>(p->w.data());
    const C* tw = reinterpret_cast<const C*>(st.tw.data());
    C x[64];
    for (long long j = 0; j < m; ++j) {
        for (long long k = 0; k < ls; ++k) {
            const C* ib = in + j * ls + k;
            x[0] = ib[0];
            for (int q = 1; q < r; ++q) x[q] = k ? mul(ib[q * m * ls], tw[(q - 1) * ls + k]) : ib[q * m * ls];
            C* ob = out + j * ls * r + k;
            for (int s = 0; s < r; ++s) {
                C acc = x[0];
                int e = 0;
                for (int q = 1; q < r; ++q) {
                    e += s;
                    if (e >= r) e -= r;
                    acc = add(acc, mul(x[q], w[e * step]));
                }
                ob[s * ls] = acc;
            }
        }
    }
}

void stockham(const skfft_plan* p, cd* a, cd* b) {
    const int n = p->n;
    C* in = reinterpret_cast<C*>(a);
    C* out = reinterpret_cast<C*>(b);
    for (const Stage& st : p->stages) {
        switch (st.p) {
            case 2: stage_fixed<2>(st, n, p->sign, in, out); break;
            case 3: stage_fixed<3>(st, n, p->sign, in, out); break;
            case 4: stage_fixed<4>(st, n, p->sign, in, out); break;
            case 5: stage_fixed<5>(st, n, p->sign, in, out); break;
            default: stage_generic(p, st, in, out); break;
        }
        std::swap(in, out);
    }
    if (in != reinterpret_cast<C*>(a)) std::memcpy(a, in, sizeof(cd) * n);
}

bool factor(int n, std::vector<int>& radices) {
    int m = n;
    while (m % 4 == 0) { radices.push_back(4); m /= 4; }
    while (m % 2 == 0) { radices.push_back(2); m /= 2; }
    for (int q = 3; q <= 61 && m > 1; q += 2) {
        while (m % q == 0) { radices.push_back(q); m /= q; }
    }
    return m == 1;
}

}  // namespace

extern "C" skfft_plan* skfft_plan_create(int n, int sign) {
    if (n <= 0) return nullptr;
    auto* p = new skfft_plan;
    p->n = n;
    p->sign = sign < 0 ? -1 : 1;
    std::vector<int> radices;
    if (factor(n, radices)) {
        p->w.resize(n);
        for (int m = 0; m < n; ++m) p->w[m] = unit_root(m, n, p->sign);
        long long ls = 1;
        for (int r : radices) {
            Stage st{r, ls, {}};
            const long long stride = n / (ls * r);
            st.tw.resize(static_cast<size_t>((r - 1) * ls));
            for (int q = 1; q < r; ++q)
                for (long long k = 0; k < ls; ++k) st.tw[(q - 1) * ls + k] = p->w[(q * k * stride) % n];
            p->stages.push_back(std::move(st));
            ls *= r;
        }
        return p;
    }
    // Bluestein with a power-of-two convolution length.
    p->bluestein = true;
    int L = 1;
    while (L < 2 * n - 1) L <<= 1;
    p->L = L;
    p->chirp.resize(n);
    const long long two_n = 2LL * n;
    for (int j = 0; j < n; ++j) {
        const long long e = (static_cast<long long>(j) * j) % two_n;  // pi j^2 / n = 2 pi e / (2n)
        p->chirp[j] = unit_root(e, two_n, p->sign);
    }
    p->fwdL = skfft_plan_create(L, -1);
    p->invL = skfft_plan_create(L, +1);
    std::vector<cd> bk(L, cd{});
    bk[0] = std::conj(p->chirp[0]);
    for (int j = 1; j < n; ++j) {
        bk[j] = std::conj(p->chirp[j]);
        bk[L - j] = std::conj(p->chirp[j]);
    }
    skfft_execute(p->fwdL, reinterpret_cast<double*>(bk.data()), reinterpret_cast<double*>(bk.data()));
    p->bhat = std::move(bk);
    return p;
}

extern "C" void skfft_execute(const skfft_plan* p, const double* in, double* out) {
    const int n = p->n;
    const cd* src = reinterpret_cast<const cd*>(in);
    cd* dst = reinterpret_cast<cd*>(out);
    if (!p->bluestein) {
        thread_local std::vector<cd> a, b;  // work buffers reused across calls
        if (static_cast<int>(a.size()) < n) {
            a.resize(n);
            b.resize(n);
        }
        std::memcpy(a.data(), src, sizeof(cd) * n);
        stockham(p, a.data(), b.data());
        std::memcpy(dst, a.data(), sizeof(cd) * n);
        return;
    }
    const int L = p->L;
    std::vector<cd> a(L, cd{});
    for (int j = 0; j < n; ++j) a[j] = src[j] * p->chirp[j];
    skfft_execute(p->fwdL, reinterpret_cast<double*>(a.data()), reinterpret_cast<double*>(a.data()));
    for (int j = 0; j < L; ++j) a[j] *= p->bhat[j];
    skfft_execute(p->invL, reinterpret_cast<double*>(a.data()), reinterpret_cast<double*>(a.data()));
    const double inv = 1.0 / L;
    for (int k = 0; k < n; ++k) dst[k] = p->chirp[k] * a[k] * inv;
}

extern "C" void skfft_destroy(skfft_plan* p) {
    if (!p) return;
    skfft_destroy(p->fwdL);
    skfft_destroy(p->invL);
    delete p;
}
