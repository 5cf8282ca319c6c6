// poisson_b200.hpp — header-only C++ shim over the C ABI (sk_poisson.h) with
// the reference's own types and signatures, so existing spherekit callers can
// switch to the B200 path without code changes beyond the namespace:
//
//   reference (proj/include/spherekit/poisson.hpp)     this shim
//   PoissonSolution solve(const PoissonProblem&)  :47  spherekit::b200::solve
//   ResidualReport residual(const PoissonProblem&,     spherekit::b200::residual
//                           const PoissonSolution&) :54
//   (grid composition)                   spherekit::b200::solve_grid
//   PoissonProblem assemble_poisson(const              spherekit::b200::assemble_poisson
//       LowRankSphereFun&, int, int, AssembleReport*) :40-41
//   fourier.hpp: Matrix analyze_2d(const BMCGrid&) :107 spherekit::b200::analyze_2d
//   BMCGrid sample_grid(const CoeffMatrix&, int, int)  spherekit::b200::sample_grid
//       :108
//   sphere_domain.hpp: sample_dfs (of samples) :61     spherekit::b200::sample_dfs
//
// Exceptions are the reference's (types.hpp:43-65): size_error,
// precondition_error, structure_error; device failures throw
// std::runtime_error (there is no CPU fallback).  Include AFTER the
// reference's "spherekit/poisson.hpp" (it provides Matrix, PoissonProblem,
// PoissonSolution, ResidualReport and the error types).
#pragma once

#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <optional>
#include <vector>

#include "sk_poisson.h"
#include "spherekit/fourier.hpp"
#include "spherekit/lowrank.hpp"
#include "spherekit/poisson.hpp"
#include "spherekit/sphere_domain.hpp"

namespace spherekit {
namespace b200 {

inline void check(sk_status s) {
    if (s == SK_OK) return;
    const std::string msg = sk_last_error();
    switch (s) {
        case SK_ERR_SIZE: throw size_error(msg);
        case SK_ERR_PRECONDITION: throw precondition_error(msg);
        case SK_ERR_SINGULAR: throw structure_error(msg);
        default: throw std::runtime_error("sk_poisson: " + msg);
    }
}

// One cached plan per (m, n, nrhs, device); plans are not re-entrant, so the
// cache hands each thread its own.
class PlanCache {
public:
    sk_plan_t get(int m, int n, int nrhs = 1, int device = 0) {
        std::lock_guard<std::mutex> lock(mu_);
        auto key = std::make_tuple(m, n, nrhs, device, std::hash<std::thread::id>{}(std::this_thread::get_id()));
        auto it = plans_.find(key);
        if (it != plans_.end()) return it->second;
        sk_plan_t p = nullptr;
        check(sk_plan_create(m, n, nrhs, device, &p));
        plans_.emplace(key, p);
        return p;
    }
    ~PlanCache() {
        for (auto& kv : plans_) sk_plan_destroy(kv.second);
    }
    static PlanCache& instance() {
        static PlanCache c;
        return c;
    }

private:
    std::mutex mu_;
    std::map<std::tuple<int, int, int, int, size_t>, sk_plan_t> plans_;
};

// spherekit::solve (poisson.cpp:121-161): X for every k != 0 column is
// bit-identical to the reference; k = 0 agrees to rounding.
inline PoissonSolution solve(const PoissonProblem& pb) {
    if (pb.m <= 0 || pb.n <= 0 || pb.m % 2 != 0 || pb.n % 2 != 0)
        throw size_error("poisson solve: sizes must be positive and even");
    sk_plan_t p = PlanCache::instance().get(pb.m, pb.n);
    PoissonSolution sol;
    sol.x = Matrix(pb.m, pb.n);
    // std::complex<double> arrays are layout-compatible with double[2]
    check(sk_solve_coeffs(p, reinterpret_cast<const double*>(pb.f.data().data()),
                          reinterpret_cast<double*>(sol.x.data().data()), SK_HOST));
    return sol;
}

// spherekit::residual (poisson.cpp:163-186)
inline ResidualReport residual(const PoissonProblem& pb, const PoissonSolution& sol) {
    sk_plan_t p = PlanCache::instance().get(pb.m, pb.n);
    double out[3];
    check(sk_residual(p, reinterpret_cast<const double*>(pb.f.data().data()),
                      reinterpret_cast<const double*>(sol.x.data().data()), out, SK_HOST));
    ResidualReport r;
    r.interior_max = out[0];
    r.replaced_row_abs = out[1];
    r.constraint_abs = out[2];
    return r;
}

// Grid-level solve of Lap u = f, integral(u) = 0: physical samples
// f[(m/2+1) x n] (theta_p = 2 pi p/m, lambda_q = -pi + 2 pi q/n) -> u, same
// layout.  Equivalent to sample_dfs -> analyze_2d -> Msin^2 -> solve ->
// sample_grid for real data.
inline std::vector<double> solve_grid(const std::vector<double>& f, int m, int n) {
    if (static_cast<long long>(f.size()) != static_cast<long long>(m / 2 + 1) * n)
        throw size_error("solve_grid: f must hold (m/2+1) x n samples");
    sk_plan_t p = PlanCache::instance().get(m, n);
    std::vector<double> u(f.size());
    check(sk_solve_grid(p, f.data(), u.data(), nullptr, SK_HOST));
    return u;
}

// The reference's own grid composition on the device (sk_solve_grid_exact):
// sample_dfs -> analyze_2d -> Msin^2 -> solve (all n lambda modes) ->
// sample_grid.  f: physical samples as in solve_grid; returns the complex
// doubled m x n grid the reference returns (for ANY input, under-resolved
// data included); *X, if given, receives the solution coefficients.
inline BMCGrid solve_grid_exact(const std::vector<double>& f, int m, int n, Matrix* X = nullptr) {
    if (m % 2 != 0 || n % 2 != 0 || m <= 0 || n <= 0) throw size_error("solve_grid_exact: sizes must be positive and even");
    if (static_cast<long long>(f.size()) != static_cast<long long>(m / 2 + 1) * n)
        throw size_error("solve_grid_exact: f must hold (m/2+1) x n samples");
    sk_plan_t p = PlanCache::instance().get(m, n);
    BMCGrid g;
    g.rows = m;
    g.cols = n;
    g.v.assign(static_cast<size_t>(m) * n, complex{});
    if (X) *X = Matrix(m, n);
    check(sk_solve_grid_exact(p, f.data(), reinterpret_cast<double*>(g.v.data()),
                              X ? reinterpret_cast<double*>(X->data().data()) : nullptr, SK_HOST));
    return g;
}

// spherekit::assemble_poisson (poisson.cpp:52-86), bit-identical F.
inline PoissonProblem assemble_poisson(const LowRankSphereFun& f, int m, int n, AssembleReport* report = nullptr) {
    if (m % 2 != 0 || n % 2 != 0 || m <= 0 || n <= 0)
        throw size_error("assemble_poisson: sizes must be positive and even");
    const int K = f.rank(), mf = f.theta_modes(), nf = f.lambda_modes();
    std::vector<complex> col(static_cast<size_t>(K) * mf), row(static_cast<size_t>(K) * nf);
    for (int j = 0; j < K; ++j) {
        if (f.col_coeffs[j].size() != mf || f.row_coeffs[j].size() != nf)
            throw size_error("assemble_poisson: factor lengths differ");
        std::copy(f.col_coeffs[j].raw().begin(), f.col_coeffs[j].raw().end(), col.begin() + static_cast<size_t>(j) * mf);
        std::copy(f.row_coeffs[j].raw().begin(), f.row_coeffs[j].raw().end(), row.begin() + static_cast<size_t>(j) * nf);
    }
    sk_plan_t p = PlanCache::instance().get(m, n);
    PoissonProblem pb;
    pb.m = m;
    pb.n = n;
    pb.f = Matrix(m, n);
    double rep[3];
    check(sk_assemble(p, K, mf, nf, reinterpret_cast<const double*>(f.d.data()),
                      reinterpret_cast<const double*>(col.data()), reinterpret_cast<const double*>(row.data()),
                      f.vscale, reinterpret_cast<double*>(pb.f.data().data()), rep, SK_HOST));
    if (report) {
        report->mean_removed = rep[0] != 0.0;
        report->removed_mean = complex(rep[1], rep[2]);
    }
    return pb;
}

// Plan for the standalone transforms (they take their own sizes).
inline sk_plan_t transform_plan() { return PlanCache::instance().get(8, 4); }

inline BMCGrid make_grid(int m, int n) {  // BMCGrid(m, n) without the out-of-line constructor
    if (m % 2 != 0 || n % 2 != 0 || m <= 0 || n <= 0) throw size_error("BMCGrid: sample counts must be positive and even");
    BMCGrid g;
    g.rows = m;
    g.cols = n;
    g.v.assign(static_cast<size_t>(m) * n, complex{});
    return g;
}

// spherekit::analyze_2d (fourier.cpp:170-188)
inline Matrix analyze_2d(const BMCGrid& g) {
    Matrix x(g.rows, g.cols);
    check(sk_analyze_2d(transform_plan(), g.rows, g.cols, reinterpret_cast<const double*>(g.v.data()),
                        reinterpret_cast<double*>(x.data().data()), SK_HOST));
    return x;
}

// spherekit::sample_grid (fourier.cpp:190-209), zero-padding / truncating
inline BMCGrid sample_grid(const Matrix& x, int m, int n) {
    if (m % 2 != 0 || n % 2 != 0) throw size_error("sample_grid: output sizes must be even");
    BMCGrid g = make_grid(m, n);
    check(sk_sample_grid(transform_plan(), x.rows(), x.cols(), reinterpret_cast<const double*>(x.data().data()), m, n,
                         reinterpret_cast<double*>(g.v.data()), SK_HOST));
    return g;
}
// (CoeffMatrix::densified is the reference's, fourier.cpp; link its library)
inline BMCGrid sample_grid(const CoeffMatrix& xm, int m, int n) { return sample_grid(xm.densified(), m, n); }

// spherekit::sample_dfs (sphere_domain.cpp:46-52) of physical samples
// phys[(m/2+1) x n] (theta_p = 2 pi p/m): the doubled m x n grid.
inline BMCGrid sample_dfs(const std::vector<double>& phys, int m, int n) {
    if (static_cast<long long>(phys.size()) != static_cast<long long>(m / 2 + 1) * n)
        throw size_error("sample_dfs: phys must hold (m/2+1) x n samples");
    BMCGrid g = make_grid(m, n);
    check(sk_sample_dfs(transform_plan(), m, n, phys.data(), reinterpret_cast<double*>(g.v.data()), SK_HOST));
    return g;
}

// spherekit::pivot_search (lowrank.hpp:89, lowrank.cpp:84-112)
inline std::optional<PivotBlock> pivot_search(const BMCGrid& residual, double alpha = 0.01) {
    int oi[3];
    double od[10];
    check(sk_ge_pivot_search(transform_plan(), residual.rows, residual.cols,
                             reinterpret_cast<const double*>(residual.v.data()), alpha, oi, od, SK_HOST));
    if (!oi[0]) return std::nullopt;
    PivotBlock p;
    p.a = complex(od[0], od[1]);
    p.b = complex(od[2], od[3]);
    p.m_even = complex(od[4], od[5]);
    p.m_odd = complex(od[6], od[7]);
    p.theta_star = od[8];
    p.lambda_star = od[9];
    return p;
}

// spherekit::ge_step (lowrank.hpp:93, lowrank.cpp:127-162), bit-identical
inline BMCGrid ge_step(const BMCGrid& residual, const PivotBlock& p) {
    const double piv[10] = {p.a.real(),     p.a.imag(),     p.b.real(),   p.b.imag(),   p.m_even.real(),
                            p.m_even.imag(), p.m_odd.real(), p.m_odd.imag(), p.theta_star, p.lambda_star};
    BMCGrid out = make_grid(residual.rows, residual.cols);
    const sk_status s = sk_ge_step(transform_plan(), residual.rows, residual.cols,
                                   reinterpret_cast<const double*>(residual.v.data()), piv,
                                   reinterpret_cast<double*>(out.v.data()), SK_HOST);
    if (s == SK_ERR_ARGUMENT) throw index_error(sk_last_error());  // a pivot that is not a grid node
    check(s);
    return out;
}

}  // namespace b200
}  // namespace spherekit
