// ORACLE / TEST INFRASTRUCTURE ONLY — see sk_oracle.h.
//
// A from-the-algorithm restatement of the reference hot path; each function
// cites the reference lines it follows.  Plain IEEE double (the Makefile does
// not enable FMA contraction), std::complex arithmetic as in the reference so
// that the coefficient-space solve is bit-comparable with it.
#include "sk_oracle.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "skfft.h"

namespace {

using cplx = std::complex<double>;
constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kTwoPi = 2.0 * kPi;

enum { OK = 0, E_SIZE = 1, E_PRECOND = 2, E_STRUCT = 3, E_OTHER = 9 };
struct size_err : std::runtime_error { using std::runtime_error::runtime_error; };
struct precond_err : std::runtime_error { using std::runtime_error::runtime_error; };
struct struct_err : std::runtime_error { using std::runtime_error::runtime_error; };

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const size_err& e) {
        g_err = e.what();
        return E_SIZE;
    } catch (const precond_err& e) {
        g_err = e.what();
        return E_PRECOND;
    } catch (const struct_err& e) {
        g_err = e.what();
        return E_STRUCT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

const cplx* as_c(const double* p) { return reinterpret_cast<const cplx*>(p); }
cplx* as_c(double* p) { return reinterpret_cast<cplx*>(p); }

// ---------------------------------------------------------------- band matrix
// Square complex band matrix, storage a[i*(kl+ku+1) + (j-i+kl)]
// (banded.hpp:11-41).
struct Band {
    int n = 0, kl = 0, ku = 0;
    std::vector<cplx> a;
    Band() = default;
    Band(int n_, int kl_, int ku_) : n(n_), kl(kl_), ku(ku_), a(static_cast<size_t>(n_) * (kl_ + ku_ + 1)) {}
    bool in(int i, int j) const { return j - i >= -kl && j - i <= ku && j >= 0 && j < n; }
    cplx get(int i, int j) const { return in(i, j) ? a[static_cast<size_t>(i) * (kl + ku + 1) + (j - i + kl)] : cplx{}; }
    cplx& at(int i, int j) { return a[static_cast<size_t>(i) * (kl + ku + 1) + (j - i + kl)]; }
    // banded.cpp:8-19: ascending-j accumulation, exact zeros included.
    std::vector<cplx> apply(const cplx* x) const {
        std::vector<cplx> y(n);
        for (int i = 0; i < n; ++i) {
            cplx acc{};
            for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) acc += get(i, j) * x[j];
            y[i] = acc;
        }
        return y;
    }
};

// The theta operators of poisson.cpp:15-40, restated from their closed form.
// msin: (i,i+1) = +i/2, (i,i-1) = -i/2; mcos: 1/2 on both; Dm = diag(i j).
// lap = Msin (Msin Dm) Dm + Mcos (Msin Dm); with the square truncation its
// entries are the real dyadic numbers below (every product in band_mul is
// exact, so this equals the reference bit for bit; tests pin it).
Band lap_band(int m) {
    Band L(m, 2, 2);
    const int h = m / 2;
    for (int i = 0; i < m; ++i) {
        const double j = i - h;
        if (i - 2 >= 0) L.at(i, i - 2) = cplx((j - 2) * (j - 1) / 4.0, 0.0);
        if (i + 2 < m) L.at(i, i + 2) = cplx((j + 2) * (j + 1) / 4.0, 0.0);
        if (i - 1 >= 0) L.at(i, i - 1) = cplx(0.0, 0.0);
        if (i + 1 < m) L.at(i, i + 1) = cplx(0.0, 0.0);
        double d = -j * j / 2.0;
        if (i == 0) d = -j * (j - 1) / 4.0;          // j = -M/2: only the (j+1) term survives
        if (i == m - 1) d = -j * (j + 1) / 4.0;      // j = M/2-1
        L.at(i, i) = cplx(d, 0.0);
    }
    return L;
}

// Msin^2 = band_mul(msin, msin): (-1/4, 1/2, -1/4) at offsets (-2,0,+2), 1/4 on
// the first and last diagonal entries, exact zeros at +-1 (poisson.cpp:61).
Band msin2_band(int m) {
    Band S(m, 2, 2);
    for (int i = 0; i < m; ++i) {
        if (i - 2 >= 0) S.at(i, i - 2) = cplx(-0.25, 0.0);
        if (i + 2 < m) S.at(i, i + 2) = cplx(-0.25, 0.0);
        if (i - 1 >= 0) S.at(i, i - 1) = cplx(0.0, 0.0);
        if (i + 1 < m) S.at(i, i + 1) = cplx(0.0, 0.0);
        S.at(i, i) = cplx((i == 0 || i == m - 1) ? 0.25 : 0.5, 0.0);
    }
    return S;
}

std::vector<cplx> weights(int m) {  // poisson.cpp:42-50
    std::vector<cplx> w(m);
    for (int i = 0; i < m; ++i) {
        const int k = i - m / 2;
        if (k % 2 != 0) continue;
        w[i] = 2.0 / (1.0 - static_cast<double>(k) * k);
    }
    return w;
}

// ------------------------------------------------------------- band solvers
// Gaussian elimination with partial pivoting inside the band, restated from
// banded.cpp:101-158.  Each row keeps a window of `width` = 2 kl + ku + 1
// entries starting at global column base[r]; a row is shifted left (aligned)
// before it is used at column c, exactly as banded.cpp:89-97 does.
struct Win {
    int base = 0, len = 0;
    cplx* e = nullptr;
    cplx val(int col) const {
        const int t = col - base;
        return (t >= 0 && t < len) ? e[t] : cplx{};
    }
    void align(int col, int width) {
        if (base >= col) return;
        const int sh = col - base;
        const int keep = std::max(0, len - sh);
        for (int t = 0; t < keep; ++t) e[t] = e[t + sh];
        for (int t = keep; t < width; ++t) e[t] = cplx{};
        base = col;
        len = width;
    }
};

std::vector<cplx> band_solve(const Band& A, const cplx* b) {
    const int n = A.n, kl = A.kl, ku = A.ku;
    const int width = 2 * kl + ku + 1;
    std::vector<cplx> store(static_cast<size_t>(n) * width);
    std::vector<Win> row(n);
    std::vector<cplx> rhs(b, b + n);
    std::vector<int> perm(n);
    for (int i = 0; i < n; ++i) {
        perm[i] = i;
        row[i].base = std::max(0, i - kl);
        row[i].len = width;
        row[i].e = store.data() + static_cast<size_t>(i) * width;
        for (int j = row[i].base; j <= std::min(n - 1, i + ku); ++j) row[i].e[j - row[i].base] = A.get(i, j);
    }
    for (int c = 0; c < n; ++c) {
        const int last = std::min(n - 1, c + kl);
        int piv = c;
        double best = std::abs(row[perm[c]].val(c));
        for (int r = c + 1; r <= last; ++r) {
            const double v = std::abs(row[perm[r]].val(c));
            if (v > best) {  // strict: ties keep the earlier row
                best = v;
                piv = r;
            }
        }
        if (best < 1e-300) throw struct_err("band_solve: matrix is numerically singular");
        std::swap(perm[c], perm[piv]);
        Win& P = row[perm[c]];
        P.align(c, width);
        const cplx pv = P.e[0];
        for (int r = c + 1; r <= last; ++r) {
            Win& R = row[perm[r]];
            const cplx v = R.val(c);
            if (v == cplx{}) continue;
            R.align(c, width);
            const cplx f = v / pv;
            R.e[0] = cplx{};
            for (int t = 1; t < width; ++t) R.e[t] -= f * P.e[t];
            rhs[perm[r]] -= f * rhs[perm[c]];
        }
    }
    std::vector<cplx> x(n);
    for (int c = n - 1; c >= 0; --c) {
        const Win& P = row[perm[c]];
        cplx acc = rhs[perm[c]];
        for (int j = c + 1; j <= std::min(n - 1, c + width - 1); ++j) acc -= P.val(j) * x[j];
        x[c] = acc / P.e[c - P.base];
    }
    return x;
}

// Bordered solve restated from banded.cpp:160-328: the band rows (minus
// skip_row) plus one dense row.  Band rows are admitted to the active set in
// order of their first column; at each column the largest band candidate is
// preferred unless it is below 1e-10 times the largest dense candidate, in
// which case a dense row pivots and any band rows it touches are promoted to
// dense rows.  Back substitution runs over the recorded pivot rows.
std::vector<cplx> band_solve_dense(const Band& A, int skip, const cplx* w, cplx wrhs, const cplx* b) {
    const int n = A.n, kl = A.kl, ku = A.ku;
    const int width = 2 * kl + ku + 1;
    struct BR {
        Win win;
        cplx rhs;
        bool used = false;
    };
    struct DR {
        std::vector<cplx> e;
        cplx rhs;
        bool used = false;
    };
    std::vector<cplx> store(static_cast<size_t>(n) * width);
    std::vector<BR> band;
    band.reserve(n);
    for (int i = 0; i < n; ++i) {
        if (i == skip) continue;
        BR r;
        r.win.base = std::max(0, i - kl);
        r.win.len = width;
        r.win.e = store.data() + band.size() * width;
        for (int j = r.win.base; j <= std::min(n - 1, i + ku); ++j) r.win.e[j - r.win.base] = A.get(i, j);
        r.rhs = b[i];
        band.push_back(r);
    }
    std::vector<int> order(band.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::stable_sort(order.begin(), order.end(), [&](int p, int q) { return band[p].win.base < band[q].win.base; });
    std::vector<DR> dense;
    dense.push_back({std::vector<cplx>(w, w + n), wrhs, false});
    struct Up {
        bool dense = false;
        int idx = -1;
    };
    std::vector<Up> up(n);
    std::vector<int> active;
    size_t next = 0;
    for (int c = 0; c < n; ++c) {
        while (next < order.size() && band[order[next]].win.base <= c) active.push_back(order[next++]);
        int bb = -1;
        double bb_abs = 0;
        for (int idx : active) {
            if (band[idx].used) continue;
            const double v = std::abs(band[idx].win.val(c));
            if (v > bb_abs) {
                bb_abs = v;
                bb = idx;
            }
        }
        int bd = -1;
        double bd_abs = 0;
        for (size_t d = 0; d < dense.size(); ++d) {
            if (dense[d].used) continue;
            const double v = std::abs(dense[d].e[c]);
            if (v > bd_abs) {
                bd_abs = v;
                bd = static_cast<int>(d);
            }
        }
        if (bb >= 0 && bb_abs >= 1e-10 * bd_abs && bb_abs >= 1e-300) {
            BR& P = band[bb];
            P.used = true;
            P.win.align(c, width);
            up[c] = {false, bb};
            const cplx pv = P.win.e[0];
            for (int idx : active) {
                BR& R = band[idx];
                if (R.used) continue;
                const cplx v = R.win.val(c);
                if (v == cplx{}) continue;
                R.win.align(c, width);
                const cplx f = v / pv;
                R.win.e[0] = cplx{};
                for (int t = 1; t < width; ++t) R.win.e[t] -= f * P.win.e[t];
                R.rhs -= f * P.rhs;
            }
            for (DR& D : dense) {
                if (D.used) continue;
                const cplx v = D.e[c];
                if (v == cplx{}) continue;
                const cplx f = v / pv;
                D.e[c] = cplx{};
                for (int t = 1; t < width && c + t < n; ++t) D.e[c + t] -= f * P.win.e[t];
                D.rhs -= f * P.rhs;
            }
        } else if (bd >= 0 && bd_abs >= 1e-300) {
            dense[bd].used = true;
            up[c] = {true, bd};
            const std::vector<cplx> pe = dense[bd].e;  // copy: `dense` may grow
            const cplx prhs = dense[bd].rhs;
            const cplx pv = pe[c];
            for (int idx : active) {
                BR& R = band[idx];
                if (R.used) continue;
                const cplx v = R.win.val(c);
                if (v == cplx{}) continue;
                DR pr;
                pr.e.assign(n, cplx{});
                for (int t = 0; t < R.win.len; ++t) {
                    const int col = R.win.base + t;
                    if (col >= 0 && col < n) pr.e[col] = R.win.e[t];
                }
                pr.rhs = R.rhs;
                const cplx f = v / pv;
                for (int j = c; j < n; ++j) pr.e[j] -= f * pe[j];
                pr.e[c] = cplx{};
                pr.rhs -= f * prhs;
                R.used = true;
                dense.push_back(std::move(pr));
            }
            for (size_t d = 0; d < dense.size(); ++d) {
                DR& D = dense[d];
                if (D.used || static_cast<int>(d) == bd) continue;
                const cplx v = D.e[c];
                if (v == cplx{}) continue;
                const cplx f = v / pv;
                for (int j = c; j < n; ++j) D.e[j] -= f * pe[j];
                D.e[c] = cplx{};
                D.rhs -= f * prhs;
            }
        } else {
            throw struct_err("band_solve_with_dense_row: singular bordered system");
        }
    }
    std::vector<cplx> x(n);
    for (int c = n - 1; c >= 0; --c) {
        cplx acc, pv;
        if (up[c].dense) {
            const DR& r = dense[up[c].idx];
            acc = r.rhs;
            for (int j = c + 1; j < n; ++j) acc -= r.e[j] * x[j];
            pv = r.e[c];
        } else {
            const BR& r = band[up[c].idx];
            acc = r.rhs;
            for (int j = c + 1; j <= std::min(n - 1, r.win.base + r.win.len - 1); ++j) acc -= r.win.val(j) * x[j];
            pv = r.win.val(c);
        }
        x[c] = acc / pv;
    }
    return x;
}

std::vector<cplx> div_sin(const std::vector<cplx>& c) {  // fourier.cpp:92-103
    const int n = static_cast<int>(c.size());
    if (n == 0) throw size_err("div_sin: empty input");
    Band ms(n, 1, 1);
    for (int i = 0; i < n; ++i) {
        if (i + 1 < n) ms.at(i, i + 1) = cplx(0, 0.5);
        if (i - 1 >= 0) ms.at(i, i - 1) = cplx(0, -0.5);
    }
    return band_solve(ms, c.data());
}

double max_abs(const cplx* a, size_t len) {
    double m = 0;
    for (size_t i = 0; i < len; ++i) m = std::max(m, std::abs(a[i]));
    return m;
}

// poisson.cpp:101-117
void check_mean_zero(int m, int n, const cplx* F) {
    std::vector<cplx> f0(m);
    for (int i = 0; i < m; ++i) f0[i] = F[static_cast<size_t>(i) * n + n / 2];
    const double fscale = max_abs(F, static_cast<size_t>(m) * n);
    if (fscale == 0.0) return;
    if (m % 2 != 0) throw size_err("CoeffVec: length must be even");
    const std::vector<cplx> a = div_sin(div_sin(f0));
    const std::vector<cplx> w = weights(m);
    cplx mean{};
    for (int i = 0; i < m; ++i) mean += w[i] * a[i];
    mean *= kTwoPi;
    if (std::abs(mean) > 1e-6 * 4.0 * kPi * fscale)
        throw precond_err("poisson solve: right-hand side has a nonzero surface mean");
}

void solve_impl(int m, int n, const cplx* F, cplx* X, int threads) {
    if (m <= 0 || n <= 0 || m % 2 != 0 || n % 2 != 0) throw size_err("poisson solve: sizes must be positive and even");
    check_mean_zero(m, n, F);
    const Band lap = lap_band(m);
    const std::vector<cplx> w = weights(m);
    auto column = [&](int kc) {
        const int k = kc - n / 2;
        std::vector<cplx> rhs(m);
        for (int i = 0; i < m; ++i) rhs[i] = F[static_cast<size_t>(i) * n + kc];
        std::vector<cplx> x;
        if (k != 0) {
            Band a = lap;
            for (int i = 0; i < m; ++i) a.at(i, i) += cplx(-static_cast<double>(k) * k, 0.0);
            x = band_solve(a, rhs.data());
        } else {
            x = band_solve_dense(lap, m / 2, w.data(), cplx{}, rhs.data());
        }
        for (int i = 0; i < m; ++i) X[static_cast<size_t>(i) * n + kc] = x[i];
    };
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0) hw = 1;
    if (threads >= 1) hw = std::min<unsigned>(hw, static_cast<unsigned>(threads));
    const int T = n < 64 ? 1 : static_cast<int>(std::min<unsigned>(hw, 16));
    if (T <= 1) {
        for (int kc = 0; kc < n; ++kc) column(kc);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (int kc = t; kc < n; kc += T) column(kc);
            });
        for (auto& th : pool) th.join();
    }
}

// ----------------------------------------------------------------- transforms
void fft_inplace(std::vector<cplx>& v, int sign) {
    skfft_plan* p = skfft_plan_create(static_cast<int>(v.size()), sign);
    skfft_execute(p, reinterpret_cast<double*>(v.data()), reinterpret_cast<double*>(v.data()));
    skfft_destroy(p);
}

// fourier.cpp:39-53: c_k = (1/n) (-1)^k F_{(k+n) mod n}, ascending k.
std::vector<cplx> analyze_1d(const cplx* s, int n) {
    if (n <= 0 || n % 2 != 0) throw size_err("analyze_1d: sample count must be even");
    std::vector<cplx> w(s, s + n);
    fft_inplace(w, -1);
    std::vector<cplx> out(n);
    for (int k = -n / 2; k < n / 2; ++k) {
        const double sg = (k % 2 == 0) ? 1.0 : -1.0;
        out[k + n / 2] = sg / n * w[(k + n) % n];
    }
    return out;
}

// fourier.cpp:55-66: zero-pad / truncate, (-1)^k, backward FFT (unnormalised).
std::vector<cplx> synthesize_1d(const cplx* c, int nc, int n_out) {
    if (n_out <= 0 || n_out % 2 != 0) throw size_err("synthesize_1d: output size must be even");
    std::vector<cplx> g(n_out, cplx{});
    const int kmin = -nc / 2;
    const int lo = std::max(kmin, -n_out / 2), hi = std::min(-kmin, n_out / 2);
    for (int k = lo; k < hi; ++k) {
        const double sg = (k % 2 == 0) ? 1.0 : -1.0;
        g[(k + n_out) % n_out] += sg * c[k - kmin];
    }
    fft_inplace(g, +1);
    return g;
}

void analyze_2d(int m, int n, const cplx* grid, cplx* X) {  // fourier.cpp:170-188
    if (m <= 0 || n <= 0 || m % 2 || n % 2) throw size_err("BMCGrid: sample counts must be positive and even");
    std::vector<cplx> half(static_cast<size_t>(m) * n), col(m), row(n);
    for (int k = 0; k < n; ++k) {
        for (int j = 0; j < m; ++j) col[j] = grid[static_cast<size_t>(j) * n + k];
        const std::vector<cplx> c = analyze_1d(col.data(), m);
        for (int j = 0; j < m; ++j) half[static_cast<size_t>(j) * n + k] = c[j];
    }
    for (int j = 0; j < m; ++j) {
        const std::vector<cplx> c = analyze_1d(half.data() + static_cast<size_t>(j) * n, n);
        std::copy(c.begin(), c.end(), X + static_cast<size_t>(j) * n);
    }
}

void sample_grid(int rows, int cols, const cplx* X, int m, int n, cplx* g) {  // fourier.cpp:190-209
    if (m % 2 != 0 || n % 2 != 0) throw size_err("sample_grid: output sizes must be even");
    std::vector<cplx> half(static_cast<size_t>(m) * cols), c(rows);
    for (int k = 0; k < cols; ++k) {
        for (int j = 0; j < rows; ++j) c[j] = X[static_cast<size_t>(j) * cols + k];
        const std::vector<cplx> v = synthesize_1d(c.data(), rows, m);
        for (int j = 0; j < m; ++j) half[static_cast<size_t>(j) * cols + k] = v[j];
    }
    for (int j = 0; j < m; ++j) {
        const std::vector<cplx> v = synthesize_1d(half.data() + static_cast<size_t>(j) * cols, cols, n);
        std::copy(v.begin(), v.end(), g + static_cast<size_t>(j) * n);
    }
}

// DFS doubling of physical samples: the index map of sphere_domain.cpp:19-26
// evaluated on the grid of :46-52 — theta_i >= 0 (i >= M/2) reads physical
// row i - M/2; theta_i < 0 reads row M/2 - i at longitude shifted by pi,
// i.e. column (q + N/2) mod N.
// theta_i is evaluated as sphere_domain.hpp:54 does (-kPi + kTwoPi i / m):
// for some m (22, 30, 44, 60, ...) theta_{m/2} rounds below zero and the
// reference glides the pole row p = 0 as well.
void dfs_double(int m, int n, const double* phys, cplx* g) {
    const double kPi_ = 3.141592653589793238462643383279502884, kTwoPi_ = 2.0 * kPi_;
    for (int i = 0; i < m; ++i)
        for (int q = 0; q < n; ++q) {
            double v;
            const double th = -kPi_ + kTwoPi_ * i / m;
            if (th >= 0.0) v = phys[static_cast<size_t>(i - m / 2) * n + q];
            else v = phys[static_cast<size_t>(m / 2 - i) * n + (q + n / 2) % n];
            g[static_cast<size_t>(i) * n + q] = cplx(v, 0.0);
        }
}

// ------------------------------------------------------ spherical harmonics
// Orthonormal associated Legendre P~_l^m(cos th) (no Condon-Shortley phase,
// matching std::assoc_legendre in tests/support/helpers.hpp:18-27) by the
// standard stable recurrences, with an extended exponent so that
// sin(th)^m does not underflow for large m.
void legendre_row(int L, int mm, double x, double s, std::vector<double>& out) {
    // out[l - mm] = P~_l^mm(x) for l = mm..L
    const double big = std::ldexp(1.0, 400), small = std::ldexp(1.0, -400);
    double pmm = 1.0 / std::sqrt(4.0 * kPi);
    int e = 0;
    for (int i = 1; i <= mm; ++i) {
        pmm *= std::sqrt((2.0 * i + 1.0) / (2.0 * i)) * s;
        if (pmm != 0.0 && std::fabs(pmm) < small) {
            pmm *= big;
            e -= 400;
        }
    }
    out.assign(L - mm + 1, 0.0);
    if (pmm == 0.0) return;
    auto emit = [&](int l, double v) { out[l - mm] = std::ldexp(v, e); };
    double p2 = pmm;  // P_{l-2}
    emit(mm, p2);
    if (mm == L) return;
    double p1 = std::sqrt(2.0 * mm + 3.0) * x * pmm;  // P_{mm+1}
    emit(mm + 1, p1);
    for (int l = mm + 2; l <= L; ++l) {
        const double ll = l, m2 = static_cast<double>(mm) * mm;
        const double a = std::sqrt((4.0 * ll * ll - 1.0) / (ll * ll - m2));
        const double b = std::sqrt(((ll - 1.0) * (ll - 1.0) - m2) / (4.0 * (ll - 1.0) * (ll - 1.0) - 1.0));
        const double p = a * (x * p1 - b * p2);
        p2 = p1;
        p1 = p;
        if (std::fabs(p1) > big) {
            p1 *= small;
            p2 *= small;
            e += 400;
        }
        emit(l, p1);
    }
}

}  // namespace

extern "C" {

const char* sko_last_error(void) { return g_err.c_str(); }

int sko_build_lap(int m, double* lap) {
    return guarded([&] {
        if (m <= 0 || m % 2 != 0) throw size_err("build_operators: m must be positive and even");
        const Band L = lap_band(m);
        for (int i = 0; i < m; ++i)
            for (int d = -2; d <= 2; ++d) lap[i * 5 + d + 2] = L.get(i, i + d).real();
    });
}

int sko_integration_weights(int m, double* w) {
    return guarded([&] {
        const std::vector<cplx> v = weights(m);
        for (int i = 0; i < m; ++i) w[i] = v[i].real();
    });
}

int sko_band_solve(int n, int kl, int ku, const double* band, const double* b, double* x) {
    return guarded([&] {
        Band A(n, kl, ku);
        std::memcpy(static_cast<void*>(A.a.data()), band, sizeof(cplx) * A.a.size());
        const std::vector<cplx> r = band_solve(A, as_c(b));
        std::memcpy(x, static_cast<const void*>(r.data()), sizeof(cplx) * n);
    });
}

int sko_band_solve_dense_row(int n, int kl, int ku, const double* band, int skip_row, const double* w,
                             double wrhs_re, double wrhs_im, const double* b, double* x) {
    return guarded([&] {
        Band A(n, kl, ku);
        std::memcpy(static_cast<void*>(A.a.data()), band, sizeof(cplx) * A.a.size());
        const std::vector<cplx> r = band_solve_dense(A, skip_row, as_c(w), cplx(wrhs_re, wrhs_im), as_c(b));
        std::memcpy(x, static_cast<const void*>(r.data()), sizeof(cplx) * n);
    });
}

int sko_div_sin(int n, const double* c, double* out) {
    return guarded([&] {
        if (n % 2 != 0) throw size_err("CoeffVec: length must be even");
        const std::vector<cplx> u = div_sin(std::vector<cplx>(as_c(c), as_c(c) + n));
        std::memcpy(out, static_cast<const void*>(u.data()), sizeof(cplx) * n);
    });
}

int sko_solve(int m, int n, const double* F, double* X, int threads) {
    return guarded([&] { solve_impl(m, n, as_c(F), as_c(X), threads); });
}

int sko_residual(int m, int n, const double* Fd, const double* Xd, double* out) {  // poisson.cpp:163-186
    return guarded([&] {
        const cplx* F = as_c(Fd);
        const cplx* X = as_c(Xd);
        const Band lap = lap_band(m);
        double interior = 0, replaced = 0;
        std::vector<cplx> xk(m);
        for (int kc = 0; kc < n; ++kc) {
            const int k = kc - n / 2;
            for (int i = 0; i < m; ++i) xk[i] = X[static_cast<size_t>(i) * n + kc];
            std::vector<cplx> r = lap.apply(xk.data());
            for (int i = 0; i < m; ++i) {
                r[i] -= static_cast<double>(k) * k * xk[i] + F[static_cast<size_t>(i) * n + kc];
                if (k == 0 && i == m / 2) replaced = std::abs(r[i]);
                else interior = std::max(interior, std::abs(r[i]));
            }
        }
        const std::vector<cplx> w = weights(m);
        cplx c{};
        for (int i = 0; i < m; ++i) c += w[i] * X[static_cast<size_t>(i) * n + n / 2];
        out[0] = interior;
        out[1] = replaced;
        out[2] = std::abs(kTwoPi * c);
    });
}

int sko_msin2_columns(int m, int n, const double* Xd, double* Fd) {
    return guarded([&] {
        const Band S = msin2_band(m);
        std::vector<cplx> col(m);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < m; ++i) col[i] = as_c(Xd)[static_cast<size_t>(i) * n + k];
            const std::vector<cplx> y = S.apply(col.data());
            for (int i = 0; i < m; ++i) as_c(Fd)[static_cast<size_t>(i) * n + k] = y[i];
        }
    });
}

int sko_analyze_1d(int n, const double* s, double* c) {
    return guarded([&] {
        const std::vector<cplx> v = analyze_1d(as_c(s), n);
        std::memcpy(c, static_cast<const void*>(v.data()), sizeof(cplx) * n);
    });
}

int sko_synthesize_1d(int n, const double* c, int n_out, double* g) {
    return guarded([&] {
        if (n % 2 != 0) throw size_err("CoeffVec: length must be even");
        const std::vector<cplx> v = synthesize_1d(as_c(c), n, n_out);
        std::memcpy(g, static_cast<const void*>(v.data()), sizeof(cplx) * n_out);
    });
}

// ---- structure-preserving GE on a doubled BMC grid (lowrank.hpp:73-93; the
// phase-1 loop of construct, lowrank.cpp:318-415, runs the same update on the
// upper half grid)

// lowrank.cpp:60-72  pinv_2x2: spectral form of the eps-pseudoinverse of [a b; b a]
static void pinv_2x2(cplx a, cplx b, double alpha, cplx& me, cplx& mo) {
    const cplx s = a + b, d = a - b;
    const double sp = std::abs(s), dp = std::abs(d);
    if (sp == 0.0 && dp == 0.0) throw std::runtime_error("pinv_2x2: zero pivot matrix");
    me = mo = cplx{};
    if (dp == 0.0) { me = 1.0 / s; return; }
    if (sp == 0.0) { mo = 1.0 / d; return; }
    if (dp < alpha * sp) { me = 1.0 / s; return; }
    if (sp < alpha * dp) { mo = 1.0 / d; return; }
    me = 1.0 / s;
    mo = 1.0 / d;
}

// lowrank.cpp:84-112  pivot_search: theta* = 2 pi t / m, t = 0..m/2 ascending
// (grid rows m/2 .. m-1, then row 0 for theta* = pi), lambda index k = n/2 ..
// n-1 ascending; sigma_1 = max(|a + b|, |a - b|) of the pair (k - n/2, k);
// strict '>' keeps the first maximal block.
static bool ge_pivot_search(int m, int n, const cplx* g, double alpha, int& bt, int& bk, cplx* v4) {
    double best = 0;
    bt = bk = -1;
    for (int t = 0; t <= m / 2; ++t) {
        const int j = (m / 2 + t) % m;
        for (int k = n / 2; k < n; ++k) {
            const cplx a = g[static_cast<size_t>(j) * n + k - n / 2], b = g[static_cast<size_t>(j) * n + k];
            const double s1 = std::max(std::abs(a + b), std::abs(a - b));
            if (s1 > best) {
                best = s1;
                bt = t;
                bk = k;
            }
        }
    }
    if (best == 0.0) return false;
    const int j = (m / 2 + bt) % m;
    v4[0] = g[static_cast<size_t>(j) * n + bk - n / 2];
    v4[1] = g[static_cast<size_t>(j) * n + bk];
    pinv_2x2(v4[0], v4[1], alpha, v4[2], v4[3]);
    return true;
}

// lowrank.cpp:127-162  ge_step at the grid node (js, ks): js = row of theta*,
// ks = column of lambda*; jm = row of -theta*, km = column of lambda* - pi.
static void ge_step(int m, int n, const cplx* g, int js, int ks, cplx me, cplx mo, cplx* out) {
    const int jm = (m - js) % m, km = (ks + n / 2) % n;
    std::vector<cplx> ce(m), co(m), re(n), ro(n);
    for (int j = 0; j < m; ++j) {
        const cplx cm = g[static_cast<size_t>(j) * n + km], cp = g[static_cast<size_t>(j) * n + ks];
        ce[j] = cm + cp;
        co[j] = cm - cp;
    }
    for (int k = 0; k < n; ++k) {
        const cplx rp = g[static_cast<size_t>(js) * n + k], rm = g[static_cast<size_t>(jm) * n + k];
        re[k] = rp + rm;
        ro[k] = rp - rm;
    }
    const cplx de = 0.5 * me, dodd = 0.5 * mo;
    const bool has_e = me != cplx{}, has_o = mo != cplx{};
    for (int j = 0; j < m; ++j)
        for (int k = 0; k < n; ++k) {
            cplx upd{};
            if (has_e) upd += de * ce[j] * re[k];
            if (has_o) upd += dodd * co[j] * ro[k];
            out[static_cast<size_t>(j) * n + k] = g[static_cast<size_t>(j) * n + k] - upd;
        }
}

int sko_analyze_2d(int m, int n, const double* grid, double* X) {
    return guarded([&] { analyze_2d(m, n, as_c(grid), as_c(X)); });
}
// construct's phase-1 loop body on the upper half grid e[h x g], h = g/2 + 1,
// row i <-> theta_i = 2 pi i / g (lowrank.cpp:345-392): complete pivoting
// over i ascending, k = g/2 .. g-1 ascending (:345-360), the pivot cross with
// the row of -theta* taken as the pivot row shifted by pi in lambda
// (:362-380), and the update (:381-392).
static bool ge_pivot_search_half(int g, const cplx* e, double alpha, int& bi, int& bk, cplx* v4) {
    const int h = g / 2 + 1;
    double best = 0;
    bi = bk = -1;
    for (int i = 0; i < h; ++i) {
        const size_t row = static_cast<size_t>(i) * g;
        for (int k = g / 2; k < g; ++k) {
            const cplx a = e[row + k - g / 2], b = e[row + k];
            const double s1 = std::max(std::abs(a + b), std::abs(a - b));
            if (s1 > best) {
                best = s1;
                bi = i;
                bk = k;
            }
        }
    }
    if (best == 0.0) return false;
    v4[0] = e[static_cast<size_t>(bi) * g + bk - g / 2];
    v4[1] = e[static_cast<size_t>(bi) * g + bk];
    pinv_2x2(v4[0], v4[1], alpha, v4[2], v4[3]);
    return true;
}
static void ge_step_half(int g, const cplx* e, int bi, int bk, cplx me, cplx mo, cplx* out) {
    const int h = g / 2 + 1;
    std::vector<cplx> ce(h), co(h), re(g), ro(g);
    for (int i = 0; i < h; ++i) {
        const cplx cm = e[static_cast<size_t>(i) * g + bk - g / 2], cp = e[static_cast<size_t>(i) * g + bk];
        ce[i] = cm + cp;
        co[i] = cm - cp;
    }
    const size_t row = static_cast<size_t>(bi) * g;
    for (int k = 0; k < g; ++k) {
        const cplx rp = e[row + k], rm = e[row + (k + g / 2) % g];
        re[k] = rp + rm;
        ro[k] = rp - rm;
    }
    const cplx de = 0.5 * me, dodd = 0.5 * mo;
    const bool has_e = me != cplx{}, has_o = mo != cplx{};
    for (int i = 0; i < h; ++i)
        for (int k = 0; k < g; ++k) {
            cplx upd{};
            if (has_e) upd += de * ce[i] * re[k];
            if (has_o) upd += dodd * co[i] * ro[k];
            out[static_cast<size_t>(i) * g + k] = e[static_cast<size_t>(i) * g + k] - upd;
        }
}
// one phase-1 step on the half grid e ((g/2+1) x g): out_i = found, bi, bk; out_d = a, b, m_even, m_odd
int sko_ge_half_step(int g, const double* e, double alpha, int* out_i, double* out_d, double* out) {
    return guarded([&] {
        int bi, bk;
        cplx v4[4] = {};
        const bool found = ge_pivot_search_half(g, as_c(e), alpha, bi, bk, v4);
        out_i[0] = found ? 1 : 0;
        out_i[1] = found ? bi : -1;
        out_i[2] = found ? bk : -1;
        for (int i = 0; i < 8; ++i) out_d[i] = 0.0;
        if (!found) return;
        for (int i = 0; i < 4; ++i) {
            out_d[2 * i] = v4[i].real();
            out_d[2 * i + 1] = v4[i].imag();
        }
        ge_step_half(g, as_c(e), bi, bk, v4[2], v4[3], reinterpret_cast<cplx*>(out));
    });
}
int sko_pivot_search(int m, int n, const double* grid, double alpha, int* out_i, double* out_d) {
    return guarded([&] {
        int bt, bk;
        cplx v4[4] = {};
        const bool found = ge_pivot_search(m, n, as_c(grid), alpha, bt, bk, v4);
        out_i[0] = found ? 1 : 0;
        out_i[1] = found ? bt : -1;
        out_i[2] = found ? bk : -1;
        for (int i = 0; i < 10; ++i) out_d[i] = 0.0;
        if (!found) return;
        for (int i = 0; i < 4; ++i) {
            out_d[2 * i] = v4[i].real();
            out_d[2 * i + 1] = v4[i].imag();
        }
        const double twopi = 6.283185307179586476925286766559;
        out_d[8] = twopi * bt / m;                                // lowrank.cpp:106
        out_d[9] = -3.14159265358979323846 + twopi * bk / n;      // BMCGrid::lambda, sphere_domain.hpp:55
    });
}
int sko_ge_step(int m, int n, const double* grid, const double* piv, double* out) {
    return guarded([&] {
        const double twopi = 6.283185307179586476925286766559, pi = 3.14159265358979323846;
        // locate_on_grid (lowrank.cpp:116-123)
        const long js = std::lround((piv[8] + pi) / (twopi / m)), ks = std::lround((piv[9] + pi) / (twopi / n));
        ge_step(m, n, as_c(grid), static_cast<int>(((js % m) + m) % m), static_cast<int>(((ks % n) + n) % n),
                cplx(piv[4], piv[5]), cplx(piv[6], piv[7]), reinterpret_cast<cplx*>(out));
    });
}

int sko_sample_grid(int rows, int cols, const double* X, int m_out, int n_out, double* grid) {
    return guarded([&] { sample_grid(rows, cols, as_c(X), m_out, n_out, as_c(grid)); });
}

int sko_dfs_double(int m, int n, const double* phys, double* grid) {
    return guarded([&] {
        if (m <= 0 || n <= 0 || m % 2 || n % 2) throw size_err("BMCGrid: sample counts must be positive and even");
        dfs_double(m, n, phys, as_c(grid));
    });
}

// assemble_poisson (poisson.cpp:52-86) of a low-rank function given by its
// factors f = sum_j d_j a_j(theta) b_j(lambda): F = sum_j (d_j Msin^2 pad(a_j, m))
// pad(b_j, n)^T accumulated term by term (ascending j, zero da skipped as
// :66 does), then the mean test with sum2 (calculus.cpp:89-103) and the
// removal of mu * coeffs(sin^2 theta) (:76-82).  rep[3] = {removed?, re, im}.
int sko_assemble(int K, int mf, int nf, const double* dd, const double* col, const double* row, double vscale, int m,
                 int n, double* Fd, double* rep) {
    return guarded([&] {
        if (m % 2 != 0 || n % 2 != 0 || m <= 0 || n <= 0)
            throw size_err("assemble_poisson: sizes must be positive and even");
        if (mf % 2 != 0 || nf % 2 != 0 || mf < 0 || nf < 0) throw size_err("CoeffVec: length must be even");
        const cplx* d = as_c(dd);
        cplx* F = as_c(Fd);
        std::fill(F, F + static_cast<size_t>(m) * n, cplx{});
        // pad_to (fourier.cpp:105-112): mode k of a length-L vector sits at k + L/2
        auto pad = [](const cplx* c, int len, int L) {
            std::vector<cplx> out(L);
            const int lo = std::max(-len / 2, -L / 2), hi = std::min(len / 2, L / 2);
            for (int k = lo; k < hi; ++k) out[k + L / 2] = c[k + len / 2];
            return out;
        };
        const Band S = msin2_band(m);
        for (int j = 0; j < K; ++j) {
            const std::vector<cplx> a = pad(as_c(col) + static_cast<size_t>(j) * mf, mf, m);
            const std::vector<cplx> b = pad(as_c(row) + static_cast<size_t>(j) * nf, nf, n);
            const std::vector<cplx> sa = S.apply(a.data());
            for (int i = 0; i < m; ++i) {
                const cplx da = d[j] * sa[i];
                if (da == cplx{}) continue;
                for (int k = 0; k < n; ++k) F[static_cast<size_t>(i) * n + k] += da * b[k];
            }
        }
        // sum2: per term (sum_k w_k a_k)(2 pi b_0), even k only, ascending k
        cplx total{};
        for (int j = 0; j < K; ++j) {
            const cplx* a = as_c(col) + static_cast<size_t>(j) * mf;
            cplx ci{};
            for (int k = -mf / 2; k < mf / 2; ++k) {
                if (k % 2 != 0) continue;
                ci += 2.0 / (1.0 - static_cast<double>(k) * k) * a[k + mf / 2];
            }
            const cplx b0 = nf > 0 ? as_c(row)[static_cast<size_t>(j) * nf + nf / 2] : cplx{};
            total += d[j] * ci * (kTwoPi * b0);
        }
        const cplx mu = total / (4.0 * kPi);
        rep[0] = 0.0;
        rep[1] = rep[2] = 0.0;
        if (std::abs(mu) > 1e-11 * std::max(vscale, 1e-300)) {
            rep[0] = 1.0;
            rep[1] = mu.real();
            rep[2] = mu.imag();
            F[static_cast<size_t>(m / 2) * n + n / 2] -= mu * 0.5;
            if (m / 2 + 2 < m) F[static_cast<size_t>(m / 2 + 2) * n + n / 2] -= mu * -0.25;
            F[static_cast<size_t>(m / 2 - 2) * n + n / 2] -= mu * -0.25;
        }
    });
}

int sko_grid_pipeline(int m, int n, const double* phys, double* Xout, double* u_doubled, double* u_phys,
                      int threads, double* mean_out) {
    return guarded([&] {
        if (m <= 0 || n <= 0 || m % 2 || n % 2) throw size_err("sizes must be positive and even");
        const size_t mn = static_cast<size_t>(m) * n;
        std::vector<cplx> g(mn), A(mn), F(mn), X(mn), U(mn);
        dfs_double(m, n, phys, g.data());
        analyze_2d(m, n, g.data(), A.data());
        if (mean_out) {  // the surface mean 2 pi w^T a_0 of f~ (poisson.cpp:101-117)
            const std::vector<cplx> w = weights(m);
            cplx mu{};
            for (int i = 0; i < m; ++i) mu += w[i] * A[static_cast<size_t>(i) * n + n / 2];
            mean_out[0] = (kTwoPi * mu).real();
            mean_out[1] = (kTwoPi * mu).imag();
        }
        const Band S = msin2_band(m);
        std::vector<cplx> col(m);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < m; ++i) col[i] = A[static_cast<size_t>(i) * n + k];
            const std::vector<cplx> y = S.apply(col.data());
            for (int i = 0; i < m; ++i) F[static_cast<size_t>(i) * n + k] = y[i];
        }
        solve_impl(m, n, F.data(), X.data(), threads);
        sample_grid(m, n, X.data(), m, n, U.data());
        if (Xout) std::memcpy(Xout, static_cast<const void*>(X.data()), sizeof(cplx) * mn);
        if (u_doubled) std::memcpy(u_doubled, static_cast<const void*>(U.data()), sizeof(cplx) * mn);
        if (u_phys) {
            for (int p = 0; p <= m / 2; ++p) {
                const int i = p < m / 2 ? m / 2 + p : 0;
                for (int q = 0; q < n; ++q) u_phys[static_cast<size_t>(p) * n + q] = U[static_cast<size_t>(i) * n + q].real();
            }
        }
    });
}

int sko_bench_problem(int nsizes, const int* sizes, double* F_last) {  // poisson.cpp:190-216
    return guarded([&] {
        std::mt19937_64 rng(0x5eedu);
        std::uniform_real_distribution<double> unit(-1.0, 1.0);
        for (int si = 0; si < nsizes; ++si) {
            const int s = sizes[si];
            if (s < 16 || s % 2 != 0) throw size_err("bench_poisson: sizes must be even and >= 16");
            const Band S = msin2_band(s);
            const std::vector<cplx> w = weights(s);
            const int band = std::max(2, s / 8);
            std::vector<cplx> col(s);
            for (int kc = 0; kc < s; ++kc) {
                const int k = kc - s / 2;
                std::fill(col.begin(), col.end(), cplx{});
                if (std::abs(k) <= band)
                    for (int i = 0; i < s; ++i)
                        if (std::abs(i - s / 2) <= band) col[i] = cplx(unit(rng), unit(rng));
                if (k == 0) {
                    cplx mean{};
                    for (int i = 0; i < s; ++i) mean += w[i] * col[i];
                    col[s / 2] -= mean / w[s / 2];
                }
                const std::vector<cplx> y = S.apply(col.data());
                if (si == nsizes - 1)
                    for (int i = 0; i < s; ++i) as_c(F_last)[static_cast<size_t>(i) * s + kc] = y[i];
            }
        }
    });
}

int sko_random_mean_zero_problem(int m, int n, unsigned seed, double* Fd) {  // poisson_oracle.hpp:119-154
    return guarded([&] {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unit(-1.0, 1.0);
        const Band S = msin2_band(m);
        const std::vector<cplx> w = weights(m);
        const int bt = m / 4, bl = n / 4;
        std::vector<cplx> col(m);
        for (int kc = 0; kc < n; ++kc) {
            const int k = kc - n / 2;
            std::fill(col.begin(), col.end(), cplx{});
            if (std::abs(k) <= bl) {
                const double sg = k % 2 == 0 ? 1.0 : -1.0;
                for (int j = 1; j <= bt; ++j) {
                    const cplx v(unit(rng), unit(rng));
                    col[m / 2 + j] = v;
                    col[m / 2 - j] = sg * v;
                }
                if (k % 2 == 0) col[m / 2] = cplx(unit(rng), unit(rng));
            }
            if (k == 0) {
                cplx mean{};
                for (int i = 0; i < m; ++i) mean += w[i] * col[i];
                col[m / 2] -= mean / w[m / 2];
            }
            const std::vector<cplx> y = S.apply(col.data());
            for (int i = 0; i < m; ++i) as_c(Fd)[static_cast<size_t>(i) * n + kc] = y[i];
        }
    });
}

int sko_shgen(int m, int n, int L, const double* coeffs, double* phys, int threads) {
    return guarded([&] {
        const int rows = m / 2 + 1;
        const int T = std::max(1, threads);
        auto work = [&](int t) {
            std::vector<double> P, A(2 * L + 1);
            for (int p = t; p < rows; p += T) {
                const double th = kTwoPi * p / m;
                const double x = std::cos(th), s = std::sin(th);
                std::fill(A.begin(), A.end(), 0.0);
                for (int mm = 0; mm <= L; ++mm) {
                    legendre_row(L, mm, x, s, P);
                    for (int l = std::max(mm, 1); l <= L; ++l) {
                        const double pl = P[l - mm];
                        A[L + mm] += coeffs[static_cast<size_t>(l) * l + l + mm] * pl;
                        if (mm > 0) A[L - mm] += coeffs[static_cast<size_t>(l) * l + l - mm] * pl;
                    }
                }
                for (int q = 0; q < n; ++q) {
                    double acc = A[L];
                    for (int mm = 1; mm <= L; ++mm) {
                        // m * lambda_q = m(-pi + 2 pi q/N): exact index reduction
                        const long r = (static_cast<long>(mm) * q) % n;
                        const double a = kTwoPi * static_cast<double>(r) / n;
                        const double sg = (mm % 2 == 0) ? 1.0 : -1.0;
                        acc += std::sqrt(2.0) * sg * (A[L + mm] * std::cos(a) + A[L - mm] * std::sin(a));
                    }
                    phys[static_cast<size_t>(p) * n + q] = acc;
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    });
}

}  // extern "C"
