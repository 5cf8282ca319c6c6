// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" entry points over the UNMODIFIED reference library, compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libspherekit_ref.so (FFT arithmetic: oracle/fftw_shim).
// Used by tests/ to (a) pin the C++ restatement (oracle/sk_oracle.cpp) against
// the reference itself and (b) generate the golden fixtures under
// tests/golden/, and by bench.py's cpu_baseline / --impl reference arm.
//
// Every wrapper calls the reference function named in its comment; the only
// new code here is argument marshalling and the two test-input generators
// that the reference keeps inside bench_poisson (poisson.cpp:190-216) and
// tests/support/poisson_oracle.hpp:119-154 (restated, same RNG draws).
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "spherekit/banded.hpp"
#include "spherekit/calculus.hpp"
#include "spherekit/fourier.hpp"
#include "spherekit/lowrank.hpp"
#include "spherekit/poisson.hpp"
#include "spherekit/sphere_domain.hpp"

using namespace spherekit;

namespace {

enum { OK = 0, E_SIZE = 1, E_PRECOND = 2, E_STRUCT = 3, E_OTHER = 9 };

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const size_error& e) {
        g_err = e.what();
        return E_SIZE;
    } catch (const precondition_error& e) {
        g_err = e.what();
        return E_PRECOND;
    } catch (const structure_error& e) {
        g_err = e.what();
        return E_STRUCT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

Matrix to_matrix(int m, int n, const double* a) {
    Matrix x(m, n);
    std::memcpy(x.data().data(), a, sizeof(complex) * static_cast<size_t>(m) * n);
    return x;
}

void from_matrix(const Matrix& x, double* out) {
    std::memcpy(out, x.data().data(), sizeof(complex) * x.data().size());
}

void set_threads(int threads) {
    if (threads > 0) {
        setenv("SPHEREKIT_THREADS", std::to_string(threads).c_str(), 1);
    } else {
        unsetenv("SPHEREKIT_THREADS");
    }
}

// Real orthonormal spherical harmonic in the reference tests' convention
// (tests/support/helpers.hpp:18-27: no Condon-Shortley phase, sqrt(2) for
// m != 0, cos(m lam) for m > 0 and sin(|m| lam) for m < 0). Written here
// from the definition; valid for small l (std::assoc_legendre).
double ysh(int l, int m, double lam, double th) {
    const int am = std::abs(m);
    double ratio = 1.0;
    for (int k = l - am + 1; k <= l + am; ++k) ratio /= k;
    const double norm = std::sqrt((2 * l + 1) / (4.0 * kPi) * ratio);
    const double p = std::assoc_legendre(l, am, std::cos(th));
    if (m == 0) return norm * p;
    return std::sqrt(2.0) * norm * p * (m > 0 ? std::cos(am * lam) : std::sin(am * lam));
}

// Test functions for known-answer fixtures (ids are ours).
sphere_fn test_fn(int id, const double* par, int npar) {
    switch (id) {
        case 0:  // cos(theta)  (test_poisson.cpp:16-18, :53-67)
            return [](double, double th) { return complex(std::cos(th), 0.0); };
        case 1:  // 1 + cos(theta)  (test_poisson.cpp:186-206)
            return [](double, double th) { return complex(1.0 + std::cos(th), 0.0); };
        case 2:  // sum_i c_i Y_{l_i}^{m_i}; par = [l0, m0, c0, l1, m1, c1, ...]
            return [v = std::vector<double>(par, par + npar)](double lam, double th) {
                double acc = 0;
                for (size_t i = 0; i + 2 < v.size(); i += 3)
                    acc += v[i + 2] * ysh(static_cast<int>(v[i]), static_cast<int>(v[i + 1]), lam, th);
                return complex(acc, 0.0);
            };
        case 3:  // sin(50 x y z)  (acceptance_main.cpp:220-236)
            return [](double lam, double th) {
                const double x = std::cos(lam) * std::sin(th);
                const double y = std::sin(lam) * std::sin(th);
                const double z = std::cos(th);
                return complex(std::sin(50 * x * y * z), 0.0);
            };
        default:  // sin(th) sin(lam) + cos(2 th)  (test_fourier.cpp:198-211)
            return [](double lam, double th) {
                return complex(std::sin(th) * std::sin(lam) + std::cos(2 * th), 0.0);
            };
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// poisson.cpp:121-161  spherekit::solve
int ref_solve(int m, int n, const double* F, double* X, int threads) {
    return guarded([&] {
        PoissonProblem pb;
        pb.m = m;
        pb.n = n;
        pb.f = to_matrix(m, n, F);
        set_threads(threads);
        const PoissonSolution sol = solve(pb);
        set_threads(0);
        from_matrix(sol.x, X);
    });
}

// poisson.cpp:163-186  spherekit::residual -> out[3]
int ref_residual(int m, int n, const double* F, const double* X, double* out) {
    return guarded([&] {
        PoissonProblem pb;
        pb.m = m;
        pb.n = n;
        pb.f = to_matrix(m, n, F);
        PoissonSolution sol;
        sol.x = to_matrix(m, n, X);
        const ResidualReport r = residual(pb, sol);
        out[0] = r.interior_max;
        out[1] = r.replaced_row_abs;
        out[2] = r.constraint_abs;
    });
}

// poisson.cpp:15-40  build_operators(m).lap as a dense band: lap[i*5 + (j-i+2)]
int ref_build_lap(int m, double* lap) {
    return guarded([&] {
        const ThetaOperators ops = build_operators(m);
        for (int i = 0; i < m; ++i)
            for (int d = -2; d <= 2; ++d) {
                const complex v = ops.lap.get(i, i + d);
                lap[2 * (i * 5 + d + 2)] = v.real();
                lap[2 * (i * 5 + d + 2) + 1] = v.imag();
            }
    });
}

// poisson.cpp:42-50
int ref_integration_weights(int m, double* w) {
    return guarded([&] {
        const std::vector<complex> v = integration_weights(m);
        std::memcpy(w, v.data(), sizeof(complex) * m);
    });
}

// msin2.apply per column, as at poisson.cpp:61,65 and :214
int ref_msin2_columns(int m, int n, const double* X, double* F) {
    return guarded([&] {
        const ThetaOperators ops = build_operators(m);
        const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
        const Matrix x = to_matrix(m, n, X);
        Matrix f(m, n);
        std::vector<complex> col(m);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < m; ++i) col[i] = x.at(i, k);
            const std::vector<complex> y = msin2.apply(col);
            for (int i = 0; i < m; ++i) f.at(i, k) = y[i];
        }
        from_matrix(f, F);
    });
}

// banded.cpp:101-158  band_solve; band[i*(kl+ku+1) + (j-i+kl)]
int ref_band_solve(int n, int kl, int ku, const double* band, const double* b, double* x) {
    return guarded([&] {
        BandMatrix a(n, kl, ku);
        for (int i = 0; i < n; ++i)
            for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) {
                const double* v = band + 2 * (static_cast<size_t>(i) * (kl + ku + 1) + (j - i + kl));
                a.at(i, j) = complex(v[0], v[1]);
            }
        const auto* bb = reinterpret_cast<const complex*>(b);
        const std::vector<complex> r = band_solve(a, std::span<const complex>(bb, n));
        std::memcpy(x, r.data(), sizeof(complex) * n);
    });
}

// banded.cpp:160-328  band_solve_with_dense_row
int ref_band_solve_dense_row(int n, int kl, int ku, const double* band, int skip_row, const double* w,
                             double wrhs_re, double wrhs_im, const double* b, double* x) {
    return guarded([&] {
        BandMatrix a(n, kl, ku);
        for (int i = 0; i < n; ++i)
            for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) {
                const double* v = band + 2 * (static_cast<size_t>(i) * (kl + ku + 1) + (j - i + kl));
                a.at(i, j) = complex(v[0], v[1]);
            }
        const auto* ww = reinterpret_cast<const complex*>(w);
        const auto* bb = reinterpret_cast<const complex*>(b);
        const std::vector<complex> r = band_solve_with_dense_row(
            a, skip_row, std::span<const complex>(ww, n), complex(wrhs_re, wrhs_im), std::span<const complex>(bb, n));
        std::memcpy(x, r.data(), sizeof(complex) * n);
    });
}

// fourier.cpp:92-103
int ref_div_sin(int n, const double* c, double* out) {
    return guarded([&] {
        CoeffVec v(std::vector<complex>(reinterpret_cast<const complex*>(c), reinterpret_cast<const complex*>(c) + n));
        const CoeffVec u = div_sin(v);
        std::memcpy(out, u.raw().data(), sizeof(complex) * n);
    });
}

// fourier.cpp:39-53
int ref_analyze_1d(int n, const double* s, double* c) {
    return guarded([&] {
        const CoeffVec v = analyze_1d(std::span<const complex>(reinterpret_cast<const complex*>(s), n));
        std::memcpy(c, v.raw().data(), sizeof(complex) * n);
    });
}

// fourier.cpp:55-66
int ref_synthesize_1d(int n, const double* c, int n_out, double* g) {
    return guarded([&] {
        CoeffVec v(std::vector<complex>(reinterpret_cast<const complex*>(c), reinterpret_cast<const complex*>(c) + n));
        const std::vector<complex> r = synthesize_1d(v, n_out);
        std::memcpy(g, r.data(), sizeof(complex) * n_out);
    });
}

// fourier.cpp:170-188; grid is an m x n BMCGrid, row-major complex
int ref_analyze_2d(int m, int n, const double* grid, double* X) {
    return guarded([&] {
        BMCGrid g(m, n);
        std::memcpy(g.v.data(), grid, sizeof(complex) * static_cast<size_t>(m) * n);
        from_matrix(analyze_2d(g), X);
    });
}

// fourier.cpp:190-209
int ref_sample_grid(int rows, int cols, const double* X, int m_out, int n_out, double* grid) {
    return guarded([&] {
        const BMCGrid g = sample_grid(CoeffMatrix::from_dense(to_matrix(rows, cols, X)), m_out, n_out);
        std::memcpy(grid, g.v.data(), sizeof(complex) * static_cast<size_t>(m_out) * n_out);
    });
}

// sphere_domain.cpp:46-52 sample_dfs applied to a lookup into a physical
// real grid phys[(m/2+1) x n] (theta_p = 2 pi p/m, lambda_q = -pi + 2 pi q/n):
// realises the DFS doubling of already-sampled data through the reference's
// own dfs_extend (sphere_domain.cpp:19-26).
int ref_sample_dfs_phys(int m, int n, const double* phys, double* grid) {
    return guarded([&] {
        const int rows = m / 2 + 1;
        const sphere_fn f = [=](double lam, double th) {
            const long p = std::lround(th * m / kTwoPi);
            long q = std::lround((lam + kPi) * n / kTwoPi);
            q = ((q % n) + n) % n;
            if (p < 0 || p >= rows) throw index_error("sample_dfs_phys: theta out of range");
            return complex(phys[static_cast<size_t>(p) * n + q], 0.0);
        };
        const BMCGrid g = sample_dfs(f, m, n);
        std::memcpy(grid, g.v.data(), sizeof(complex) * static_cast<size_t>(m) * n);
    });
}

// The grid-level composition: sample_dfs -> analyze_2d ->
// Msin^2 per column -> solve -> sample_grid.  Outputs the coefficient matrix
// X (m x n complex) and the doubled solution grid u (m x n complex).
int ref_grid_pipeline_timed(int m, int n, const double* phys, double* X, double* u, int threads, double* t) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        const auto t0 = clk::now();
        std::vector<double> grid(2 * static_cast<size_t>(m) * n);
        if (ref_sample_dfs_phys(m, n, phys, grid.data()) != OK) throw std::runtime_error(g_err);
        BMCGrid g(m, n);
        std::memcpy(g.v.data(), grid.data(), sizeof(complex) * static_cast<size_t>(m) * n);
        const auto t1 = clk::now();
        const Matrix a = analyze_2d(g);
        const auto t2 = clk::now();
        const ThetaOperators ops = build_operators(m);
        const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
        PoissonProblem pb;
        pb.m = m;
        pb.n = n;
        pb.f = Matrix(m, n);
        std::vector<complex> col(m);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < m; ++i) col[i] = a.at(i, k);
            const std::vector<complex> y = msin2.apply(col);
            for (int i = 0; i < m; ++i) pb.f.at(i, k) = y[i];
        }
        const auto t3 = clk::now();
        set_threads(threads);
        const PoissonSolution sol = solve(pb);
        set_threads(0);
        const auto t4 = clk::now();
        if (X) from_matrix(sol.x, X);
        const BMCGrid ug = sample_grid(CoeffMatrix::from_dense(sol.x), m, n);
        const auto t5 = clk::now();
        if (u) std::memcpy(u, ug.v.data(), sizeof(complex) * static_cast<size_t>(m) * n);
        if (t) {
            t[0] = sec(t0, t1);  // sample_dfs (+ copy into the BMCGrid)
            t[1] = sec(t1, t2);  // analyze_2d
            t[2] = sec(t2, t3);  // Msin^2 per column
            t[3] = sec(t3, t4);  // solve
            t[4] = sec(t4, t5);  // sample_grid (with its CoeffMatrix copies)
        }
    });
}

int ref_grid_pipeline(int m, int n, const double* phys, double* X, double* u, int threads) {
    return ref_grid_pipeline_timed(m, n, phys, X, u, threads, nullptr);
}

// bench_poisson's coefficient-space workload generator (poisson.cpp:190-216),
// restated with the same mt19937_64(0x5eed) draw order. The RNG is shared
// across sizes in the reference; `sizes` lists every size generated before and
// including the wanted one, so the stream position matches.
int ref_bench_problem(int nsizes, const int* sizes, double* F_last) {
    return guarded([&] {
        std::mt19937_64 rng(0x5eedu);
        std::uniform_real_distribution<double> unit(-1.0, 1.0);
        for (int si = 0; si < nsizes; ++si) {
            const int s = sizes[si];
            Matrix f(s, s);
            const ThetaOperators ops = build_operators(s);
            const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
            const std::vector<complex> w = integration_weights(s);
            const int band = std::max(2, s / 8);
            std::vector<complex> col(s);
            for (int kc = 0; kc < s; ++kc) {
                const int k = kc - s / 2;
                std::fill(col.begin(), col.end(), complex{});
                if (std::abs(k) <= band)
                    for (int i = 0; i < s; ++i)
                        if (std::abs(i - s / 2) <= band) col[i] = complex(unit(rng), unit(rng));
                if (k == 0) {
                    complex mean{};
                    for (int i = 0; i < s; ++i) mean += w[i] * col[i];
                    col[s / 2] -= mean / w[s / 2];
                }
                const std::vector<complex> y = msin2.apply(col);
                for (int i = 0; i < s; ++i) f.at(i, kc) = y[i];
            }
            if (si == nsizes - 1) from_matrix(f, F_last);
        }
    });
}

// tests/support/poisson_oracle.hpp:119-154 random_mean_zero_problem, restated
// (same mt19937_64 seed and draw order).
int ref_random_mean_zero_problem(int m, int n, unsigned seed, double* F) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unit(-1.0, 1.0);
        const ThetaOperators ops = build_operators(m);
        const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
        const std::vector<complex> w = integration_weights(m);
        Matrix f(m, n);
        const int bt = m / 4, bl = n / 4;
        std::vector<complex> col(m);
        for (int kc = 0; kc < n; ++kc) {
            const int k = kc - n / 2;
            std::fill(col.begin(), col.end(), complex{});
            if (std::abs(k) <= bl) {
                const double sign = k % 2 == 0 ? 1.0 : -1.0;
                for (int j = 1; j <= bt; ++j) {
                    const complex v(unit(rng), unit(rng));
                    col[m / 2 + j] = v;
                    col[m / 2 - j] = sign * v;
                }
                if (k % 2 == 0) col[m / 2] = complex(unit(rng), unit(rng));
            }
            if (k == 0) {
                complex mean{};
                for (int i = 0; i < m; ++i) mean += w[i] * col[i];
                col[m / 2] -= mean / w[m / 2];
            }
            const std::vector<complex> y = msin2.apply(col);
            for (int i = 0; i < m; ++i) f.at(i, kc) = y[i];
        }
        from_matrix(f, F);
    });
}

// assemble_poisson(construct(f), m, n) for the known-answer fixtures
// (poisson.cpp:52-86; lowrank.cpp:608-721). out_mean[3] = {removed?, re, im}.
int ref_assemble_fn(int fn_id, const double* par, int npar, int m, int n, double* F, double* out_mean) {
    return guarded([&] {
        const LowRankSphereFun f = construct(test_fn(fn_id, par, npar));
        AssembleReport rep;
        const PoissonProblem pb = assemble_poisson(f, m, n, &rep);
        from_matrix(pb.f, F);
        if (out_mean) {
            out_mean[0] = rep.mean_removed ? 1.0 : 0.0;
            out_mean[1] = rep.removed_mean.real();
            out_mean[2] = rep.removed_mean.imag();
        }
    });
}

// construct(f) of a test function (lowrank.cpp:608-721), exported as raw
// factors: d[K] complex, col[K][mf] complex, row[K][nf] complex, vscale.
// Call with d == nullptr to query K, mf, nf.
int ref_construct_fn(int fn_id, const double* par, int npar, int* K, int* mf, int* nf, double* d, double* col,
                     double* row, double* vscale) {
    return guarded([&] {
        const LowRankSphereFun f = construct(test_fn(fn_id, par, npar));
        *K = f.rank();
        *mf = f.theta_modes();
        *nf = f.lambda_modes();
        if (!d) return;
        for (int j = 0; j < f.rank(); ++j) {
            std::memcpy(d + 2 * j, &f.d[j], sizeof(complex));
            std::memcpy(col + 2 * static_cast<size_t>(j) * (*mf), f.col_coeffs[j].raw().data(), sizeof(complex) * (*mf));
            std::memcpy(row + 2 * static_cast<size_t>(j) * (*nf), f.row_coeffs[j].raw().data(), sizeof(complex) * (*nf));
        }
        *vscale = f.vscale;
    });
}

// assemble_poisson (poisson.cpp:52-86) of a low-rank function given by raw
// factors (layout as ref_construct_fn).  out_mean[3] = {removed?, re, im}.
int ref_assemble_lowrank(int K, int mf, int nf, const double* d, const double* col, const double* row, double vscale,
                         int m, int n, double* F, double* out_mean) {
    return guarded([&] {
        LowRankSphereFun f;
        for (int j = 0; j < K; ++j) {
            complex dj;
            std::memcpy(&dj, d + 2 * j, sizeof(complex));
            f.d.push_back(dj);
            std::vector<complex> c(mf), r(nf);
            std::memcpy(c.data(), col + 2 * static_cast<size_t>(j) * mf, sizeof(complex) * mf);
            std::memcpy(r.data(), row + 2 * static_cast<size_t>(j) * nf, sizeof(complex) * nf);
            f.col_coeffs.emplace_back(std::move(c));
            f.row_coeffs.emplace_back(std::move(r));
            f.parity.push_back(Parity::even);
        }
        f.vscale = vscale;
        AssembleReport rep;
        const PoissonProblem pb = assemble_poisson(f, m, n, &rep);
        from_matrix(pb.f, F);
        if (out_mean) {
            out_mean[0] = rep.mean_removed ? 1.0 : 0.0;
            out_mean[1] = rep.removed_mean.real();
            out_mean[2] = rep.removed_mean.imag();
        }
    });
}

// sample_dfs(f, m, n) of a test function (sphere_domain.cpp:46-52)
int ref_sample_dfs_fn(int fn_id, const double* par, int npar, int m, int n, double* grid) {
    return guarded([&] {
        const BMCGrid g = sample_dfs(test_fn(fn_id, par, npar), m, n);
        std::memcpy(grid, g.v.data(), sizeof(complex) * static_cast<size_t>(m) * n);
    });
}

// poisson.cpp:188-230 bench_poisson; writes seconds[i] (best of reps).
int ref_bench_poisson(int nsizes, const int* sizes, int threads, double* seconds, int* reps) {
    return guarded([&] {
        set_threads(threads);
        const std::vector<BenchRow> rows = bench_poisson(std::vector<int>(sizes, sizes + nsizes));
        set_threads(0);
        for (int i = 0; i < nsizes; ++i) {
            seconds[i] = rows[i].seconds;
            reps[i] = rows[i].reps;
        }
    });
}

// Timing helper for the CPU baseline on a BOUNDED sample of a large grid
// workload (bench.py cpu_baseline / --impl reference): runs the reference's
// per-column and per-row building blocks exactly as analyze_2d / solve /
// sample_grid call them (fourier.cpp:176-186, poisson.cpp:132-145,
// fourier.cpp:195-207), on `ncols` of the n lambda-mode columns and `nrows`
// of the m theta rows, with `threads` std::threads dealing columns like
// solve() does (poisson.cpp:147-159). Returns seconds per stage:
// t[0] theta analysis per column, t[1] lambda analysis per row,
// t[2] Msin^2+solve per column, t[3] theta synthesis per column,
// t[4] lambda synthesis per row (all per-unit, averaged over the sample).
int ref_time_sample(int m, int n, int ncols, int nrows, int threads, double* t) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        std::mt19937_64 rng(1234);
        std::uniform_real_distribution<double> unit(-1.0, 1.0);
        auto randv = [&](int len) {
            std::vector<complex> v(len);
            for (auto& x : v) x = complex(unit(rng), unit(rng));
            return v;
        };
        const ThetaOperators ops = build_operators(m);
        const std::vector<complex> w = integration_weights(m);
        const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
        const int T = std::max(1, threads);
        auto par = [&](int count, auto&& body) {
            std::vector<std::thread> pool;
            for (int th = 0; th < T; ++th)
                pool.emplace_back([&, th] {
                    for (int c = th; c < count; c += T) body(c);
                });
            for (auto& p : pool) p.join();
        };
        std::vector<std::vector<complex>> cols(ncols), rows(nrows);
        for (int c = 0; c < ncols; ++c) cols[c] = randv(m);
        for (int r = 0; r < nrows; ++r) rows[r] = randv(n);
        volatile double sink = 0;
        // theta analysis (single-threaded as shipped: analyze_2d has no threads)
        auto t0 = clk::now();
        for (int c = 0; c < ncols; ++c) sink = sink + std::abs(analyze_1d(cols[c])[1]);
        auto t1 = clk::now();
        for (int r = 0; r < nrows; ++r) sink = sink + std::abs(analyze_1d(rows[r])[1]);
        auto t2 = clk::now();
        // Msin^2 (assembly side) + per-column solve with the thread pool.
        std::vector<double> acc(ncols);
        par(ncols, [&](int c) {
            const int k = 1 + c % std::max(1, n / 2 - 1);  // a k != 0 column
            std::vector<complex> f = msin2.apply(cols[c]);
            BandMatrix a = ops.lap;
            band_shift_diag(a, -static_cast<double>(k) * k);
            const std::vector<complex> x = band_solve(a, f);
            acc[c] = std::abs(x[m / 2]);
        });
        auto t3 = clk::now();
        for (int c = 0; c < ncols; ++c) {
            CoeffVec cv(cols[c]);
            sink = sink + std::abs(synthesize_1d(cv, m)[0]);
        }
        auto t4 = clk::now();
        for (int r = 0; r < nrows; ++r) {
            CoeffVec rv(rows[r]);
            sink = sink + std::abs(synthesize_1d(rv, n)[0]);
        }
        auto t5 = clk::now();
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        t[0] = sec(t0, t1) / std::max(1, ncols);
        t[1] = sec(t1, t2) / std::max(1, nrows);
        t[2] = sec(t2, t3) / std::max(1, ncols);
        t[3] = sec(t3, t4) / std::max(1, ncols);
        t[4] = sec(t4, t5) / std::max(1, nrows);
        (void)w;
    });
}


// Stock-composition sample for the CPU baseline (bench.py cpu_baseline /
// --impl reference): the reference's grid composition (ref_grid_pipeline:
// analyze_2d fourier.cpp:170-188 -> Msin^2 per column -> solve
// poisson.cpp:121-161 -> sample_grid fourier.cpp:190-209) run with its OWN
// loops and access patterns on full-size m x n matrices, restricted to a
// block of `ncols` consecutive lambda-mode columns (kc0 .. kc0+ncols-1: the
// strided column gathers / scatters of analyze_2d, solve and sample_grid
// share cache lines between neighbouring columns exactly as in the full
// loops) and `nrows` consecutive theta rows.  The column solves run on
// solve()'s thread pool (min(hw, threads, 16) threads, round-robin,
// poisson.cpp:147-159); the transforms are single-threaded as shipped.  The
// matrices persist across calls (allocated and filled once per size).
// Returns seconds: t[0] theta analysis per column, t[1] lambda analysis per
// row, t[2] Msin^2 + solve per column, t[3] theta synthesis per column,
// t[4] lambda synthesis per row, t[5] wall time of this sample, t[6]
// sample_dfs per row (dfs_extend of every point of the row block from the
// physical samples, as sample_dfs / ref_sample_dfs_phys evaluate them).
int ref_time_stock_sample(int m, int n, int kc0, int ncols, int j0, int nrows, int threads, double* t) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        struct Mats {
            int m = 0, n = 0;
            Matrix a, half, f, x;
            std::vector<double> phys;
        };
        static Mats S;
        if (S.m != m || S.n != n) {
            S = Mats{};
            S.m = m;
            S.n = n;
            S.a = Matrix(m, n);
            std::mt19937_64 rng(1234);
            std::uniform_real_distribution<double> unit(-1.0, 1.0);
            for (int i = 0; i < m; ++i)
                for (int k = 0; k < n; ++k) S.a.at(i, k) = complex(unit(rng), unit(rng));
            S.half = Matrix(m, n);
            S.f = Matrix(m, n);
            S.x = Matrix(m, n);
            S.phys.assign(static_cast<size_t>(m / 2 + 1) * n, 0.0);
            for (auto& v : S.phys) v = unit(rng);
        }
        kc0 = std::max(0, std::min(kc0, n - ncols));
        j0 = std::max(0, std::min(j0, m - nrows));
        const auto w0 = clk::now();
        // sample_dfs on the row block (sphere_domain.cpp:46-52 over rows j0..)
        {
            const int prow = m / 2 + 1;
            const double* ph = S.phys.data();
            const sphere_fn fn = [=](double lam, double th) {
                const long p = std::lround(th * m / kTwoPi);
                long q = std::lround((lam + kPi) * n / kTwoPi);
                q = ((q % n) + n) % n;
                if (p < 0 || p >= prow) throw index_error("sample_dfs: theta out of range");
                return complex(ph[static_cast<size_t>(p) * n + q], 0.0);
            };
            // grid coordinates as BMCGrid::theta / lambda define them (sphere_domain.hpp:54-55)
            for (int j = j0; j < j0 + nrows; ++j) {
                const double th = -kPi + kTwoPi * j / m;
                for (int k = 0; k < n; ++k) {
                    const double lam = -kPi + kTwoPi * k / n;
                    S.a.at(j, k) = dfs_extend(fn, {lam, th});
                }
            }
        }
        const auto wd = clk::now();
        const ThetaOperators ops = build_operators(m);
        const std::vector<complex> w = integration_weights(m);
        const BandMatrix msin2 = band_mul(ops.msin, ops.msin);
        volatile double sink = 0;
        // analyze_2d, column stage (fourier.cpp:176-180)
        const auto t0 = clk::now();
        {
            std::vector<complex> col(m);
            for (int k = kc0; k < kc0 + ncols; ++k) {
                for (int j = 0; j < m; ++j) col[j] = S.a.at(j, k);
                CoeffVec c = analyze_1d(col);
                for (int j = 0; j < m; ++j) S.half.at(j, k) = c[j];
            }
        }
        // analyze_2d, row stage (fourier.cpp:182-186)
        const auto t1 = clk::now();
        {
            std::vector<complex> row(n);
            for (int j = j0; j < j0 + nrows; ++j) {
                for (int k = 0; k < n; ++k) row[k] = S.half.at(j, k);
                CoeffVec c = analyze_1d(row);
                for (int k = 0; k < n; ++k) S.f.at(j, k) = c[k];
            }
        }
        // Msin^2 per column (the composition's assembly of F) + solve's
        // solve_column on its thread pool (poisson.cpp:132-159)
        const auto t2 = clk::now();
        {
            std::vector<complex> col(m);
            for (int k = kc0; k < kc0 + ncols; ++k) {
                for (int i = 0; i < m; ++i) col[i] = S.f.at(i, k);
                const std::vector<complex> y = msin2.apply(col);
                for (int i = 0; i < m; ++i) S.f.at(i, k) = y[i];
            }
            auto solve_column = [&](int kc) {
                const int k = kc - n / 2;
                std::vector<complex> rhs(m);
                for (int i = 0; i < m; ++i) rhs[i] = S.f.at(i, kc);
                std::vector<complex> x;
                if (k != 0) {
                    BandMatrix a = ops.lap;
                    band_shift_diag(a, -static_cast<double>(k) * k);
                    x = band_solve(a, rhs);
                } else {
                    x = band_solve_with_dense_row(ops.lap, m / 2, w, complex{}, rhs);
                }
                for (int i = 0; i < m; ++i) S.x.at(i, kc) = x[i];
            };
            unsigned hw = std::thread::hardware_concurrency();
            const int T = static_cast<int>(std::max(1u, std::min({hw ? hw : 1u, static_cast<unsigned>(std::max(1, threads)), 16u})));
            if (n < 64 || T <= 1) {
                for (int kc = kc0; kc < kc0 + ncols; ++kc) solve_column(kc);
            } else {
                std::vector<std::thread> pool;
                for (int th = 0; th < T; ++th)
                    pool.emplace_back([&, th] {
                        for (int kc = kc0 + th; kc < kc0 + ncols; kc += T) solve_column(kc);
                    });
                for (auto& p : pool) p.join();
            }
        }
        // sample_grid, column stage (fourier.cpp:195-200)
        const auto t3 = clk::now();
        {
            for (int k = kc0; k < kc0 + ncols; ++k) {
                CoeffVec c(m);
                for (int j = 0; j < m; ++j) c[j] = S.x.at(j, k);
                std::vector<complex> vals = synthesize_1d(c, m);
                for (int j = 0; j < m; ++j) S.half.at(j, k) = vals[j];
            }
        }
        // sample_grid, row stage (fourier.cpp:201-207)
        const auto t4 = clk::now();
        {
            for (int j = j0; j < j0 + nrows; ++j) {
                CoeffVec c(n);
                for (int k = 0; k < n; ++k) c[k] = S.half.at(j, k);
                std::vector<complex> vals = synthesize_1d(c, n);
                for (int k = 0; k < n; ++k) S.a.at(j, k) = vals[k];  // into the input grid: keeps it O(1)
                sink = sink + std::abs(vals[0]);
            }
        }
        const auto t5 = clk::now();
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        t[0] = sec(t0, t1) / std::max(1, ncols);
        t[1] = sec(t1, t2) / std::max(1, nrows);
        t[2] = sec(t2, t3) / std::max(1, ncols);
        t[3] = sec(t3, t4) / std::max(1, ncols);
        t[4] = sec(t4, t5) / std::max(1, nrows);
        t[5] = sec(w0, t5);
        t[6] = sec(w0, wd) / std::max(1, nrows);
    });
}

// lowrank.cpp:84-112  pivot_search (complete pivoting over theta* in [0, pi],
// lambda* in [0, pi)).  out_i: found, t (theta* = 2 pi t / m), k (lambda index);
// out_d: a, b, m_even, m_odd (re, im each), theta_star, lambda_star.
int ref_pivot_search(int m, int n, const double* grid, double alpha, int* out_i, double* out_d) {
    return guarded([&] {
        BMCGrid g(m, n);
        std::memcpy(g.v.data(), grid, sizeof(complex) * static_cast<size_t>(m) * n);
        const auto p = pivot_search(g, alpha);
        out_i[0] = p.has_value() ? 1 : 0;
        out_i[1] = out_i[2] = -1;
        for (int i = 0; i < 10; ++i) out_d[i] = 0.0;
        if (!p) return;
        out_i[1] = static_cast<int>(std::lround(p->theta_star / (kTwoPi / m)));
        out_i[2] = static_cast<int>(std::lround((p->lambda_star + kPi) / (kTwoPi / n))) % n;
        const complex v[4] = {p->a, p->b, p->m_even, p->m_odd};
        for (int i = 0; i < 4; ++i) {
            out_d[2 * i] = v[i].real();
            out_d[2 * i + 1] = v[i].imag();
        }
        out_d[8] = p->theta_star;
        out_d[9] = p->lambda_star;
    });
}

// lowrank.cpp:127-162  ge_step; piv = a, b, m_even, m_odd, theta_star, lambda_star (as above)
int ref_ge_step(int m, int n, const double* grid, const double* piv, double* out) {
    return guarded([&] {
        BMCGrid g(m, n);
        std::memcpy(g.v.data(), grid, sizeof(complex) * static_cast<size_t>(m) * n);
        PivotBlock p;
        p.a = complex(piv[0], piv[1]);
        p.b = complex(piv[2], piv[3]);
        p.m_even = complex(piv[4], piv[5]);
        p.m_odd = complex(piv[6], piv[7]);
        p.theta_star = piv[8];
        p.lambda_star = piv[9];
        const BMCGrid r = ge_step(g, p);
        std::memcpy(out, r.v.data(), sizeof(complex) * static_cast<size_t>(m) * n);
    });
}

}  // extern "C"
