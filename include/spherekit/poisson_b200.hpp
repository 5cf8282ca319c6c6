// poisson_b200.hpp — header-only C++ shim over the C ABI (sk_poisson.h) with
// the reference's own types and signatures, so existing spherekit callers can
// switch to the B200 path without code changes beyond the namespace:
//
//   reference (proj/include/spherekit/poisson.hpp)     this shim
//   PoissonSolution solve(const PoissonProblem&)  :47  spherekit::b200::solve
//   ResidualReport residual(const PoissonProblem&,     spherekit::b200::residual
//                           const PoissonSolution&) :54
//   (grid composition)                   spherekit::b200::solve_grid
//
// Exceptions are the reference's (types.hpp:43-65): size_error,
// precondition_error, structure_error; device failures throw
// std::runtime_error (there is no CPU fallback).  Include AFTER the
// reference's "spherekit/poisson.hpp" (it provides Matrix, PoissonProblem,
// PoissonSolution, ResidualReport and the error types).
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "sk_poisson.h"
#include "spherekit/poisson.hpp"

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

}  // namespace b200
}  // namespace spherekit
