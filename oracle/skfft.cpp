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

void stockham(const skfft_plan* p, cd* a, cd* b) {
    const int n = p->n;
    cd* in = a;
    cd* out = b;
    for (const Stage& st : p->stages) {
        const int r = st.p;
        const long long ls = st.ls;
        const long long nb = n / r;
        const long long tw_stride = n / (ls * r);
        cd x[64];
        cd y[64];
        for (long long bi = 0; bi < nb; ++bi) {
            const long long k = bi % ls;
            const long long j = bi / ls;
            for (int q = 0; q < r; ++q) {
                cd v = in[bi + q * nb];
                if (k != 0 && q != 0) v *= p->w[(static_cast<long long>(q) * k * tw_stride) % n];
                x[q] = v;
            }
            switch (r) {
                case 2:
                    y[0] = x[0] + x[1];
                    y[1] = x[0] - x[1];
                    break;
                case 4: {
                    const cd t0 = x[0] + x[2], t1 = x[0] - x[2];
                    const cd t2 = x[1] + x[3], t3 = x[1] - x[3];
                    // multiply t3 by (sign * i)
                    const cd t3r = p->sign < 0 ? cd(t3.imag(), -t3.real()) : cd(-t3.imag(), t3.real());
                    y[0] = t0 + t2;
                    y[2] = t0 - t2;
                    y[1] = t1 + t3r;
                    y[3] = t1 - t3r;
                    break;
                }
                default: {
                    const long long step = n / r;  // omega_r = w[step]
                    for (int s = 0; s < r; ++s) {
                        cd acc = x[0];
                        for (int q = 1; q < r; ++q)
                            acc += x[q] * p->w[(static_cast<long long>(q) * s % r) * step];
                        y[s] = acc;
                    }
                }
            }
            for (int s = 0; s < r; ++s) out[j * ls * r + k + s * ls] = y[s];
        }
        std::swap(in, out);
    }
    if (in != a) std::memcpy(a, in, sizeof(cd) * n);
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
            p->stages.push_back({r, ls});
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
        std::vector<cd> a(src, src + n), b(n);
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
