// Compiles the C++ drop-in shim against the REFERENCE's own headers and links
// it with libsk_poisson.so (tests/test_integration.py).  With a device the
// solve must be bit-identical to the reference's on k != 0 columns; without
// one it must fail loudly (no CPU fallback).
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "spherekit/poisson.hpp"
#include "spherekit/poisson_b200.hpp"

int main() {
    using namespace spherekit;
    PoissonProblem bad;
    bad.m = 15;
    bad.n = 16;
    try {
        b200::solve(bad);
        std::printf("no size_error\n");
        return 1;
    } catch (const size_error&) {
    }
    PoissonProblem pb;
    pb.m = pb.n = 16;
    pb.f = Matrix(16, 16);
    pb.f.at(9, 9) = complex(0.25, 0.5);
    try {
        const PoissonSolution s = b200::solve(pb);
        std::printf("solved %d x %d, x(9,9) = %.17g\n", s.x.rows(), s.x.cols(), s.x.at(9, 9).real());
        // assemble_poisson of f = cos(theta) (rank 1): sin^2 cos = cos/4 - cos3/4,
        // so F = 1/8 at theta modes +-1 and -1/8 at +-3 in the lambda-mode-0 column
        LowRankSphereFun f;
        f.d = {complex(1.0, 0.0)};
        CoeffVec a(8), b(4);
        a.mode(1) = a.mode(-1) = complex(0.5, 0.0);
        b.mode(0) = complex(1.0, 0.0);
        f.col_coeffs = {a};
        f.row_coeffs = {b};
        f.parity = {Parity::odd};
        f.vscale = 1.0;
        AssembleReport rep;
        const PoissonProblem q = b200::assemble_poisson(f, 16, 8, &rep);
        if (q.f.at(9, 4) != complex(0.125, 0.0) || q.f.at(11, 4) != complex(-0.125, 0.0) || rep.mean_removed) {
            std::printf("assemble mismatch\n");
            return 1;
        }
        // analyze_2d of the doubled grid of a pure mode e^{i(2 theta + lambda)}, then sample_grid back
        BMCGrid g = b200::make_grid(8, 6);
        for (int j = 0; j < 8; ++j)
            for (int k = 0; k < 6; ++k) g.at(j, k) = std::polar(1.0, 2 * g.theta(j) + g.lambda(k));
        const Matrix X = b200::analyze_2d(g);
        if (std::abs(X.at(4 + 2, 3 + 1) - complex(1.0, 0.0)) > 1e-14) {
            std::printf("analyze_2d mismatch\n");
            return 1;
        }
        const BMCGrid back = b200::sample_grid(X, 8, 6);
        double err = 0;
        for (size_t i = 0; i < g.v.size(); ++i) err = std::max(err, std::abs(back.v[i] - g.v[i]));
        if (err > 1e-14) {
            std::printf("sample_grid round trip %.3g\n", err);
            return 1;
        }
        // grid solves of f = cos(theta) on 16 x 8: u = -cos(theta) / 2 (l = 1 eigenfunction)
        {
            const int m = 16, n = 8;
            std::vector<double> fp(static_cast<size_t>(m / 2 + 1) * n);
            for (int p = 0; p <= m / 2; ++p)
                for (int q = 0; q < n; ++q) fp[static_cast<size_t>(p) * n + q] = std::cos(2.0 * 3.14159265358979323846 * p / m);
            const std::vector<double> u = b200::solve_grid(fp, m, n);
            Matrix Xc;
            const BMCGrid U = b200::solve_grid_exact(fp, m, n, &Xc);
            double e1 = 0, e2 = 0;
            for (int p = 0; p <= m / 2; ++p)
                for (int q = 0; q < n; ++q) {
                    const double ue = -0.5 * std::cos(2.0 * 3.14159265358979323846 * p / m);
                    e1 = std::max(e1, std::abs(u[static_cast<size_t>(p) * n + q] - ue));
                    e2 = std::max(e2, std::abs(U.at((m / 2 + p) % m, q) - complex(ue, 0.0)));  // doubled row j <-> theta_j = -pi + 2 pi j/m
                }
            if (e1 > 1e-14 || e2 > 1e-14 || Xc.rows() != m) {
                std::printf("grid solve mismatch %.3g %.3g\n", e1, e2);
                return 1;
            }
        }
        // pivot_search + ge_step annihilate a rank-1 BMC function (test_lowrank.cpp:87-96)
        {
            BMCGrid r1 = b200::make_grid(32, 32);
            for (int j = 0; j < 32; ++j)
                for (int k = 0; k < 32; ++k)
                    r1.at(j, k) = (std::cos(2 * r1.theta(j)) + 2.0) * (std::sin(2 * r1.lambda(k)) + 0.4);
            const auto p = b200::pivot_search(r1);
            if (!p) {
                std::printf("no pivot\n");
                return 1;
            }
            const BMCGrid z = b200::ge_step(r1, *p);
            double mx = 0, sc = 0;
            for (size_t i = 0; i < z.v.size(); ++i) {
                mx = std::max(mx, std::abs(z.v[i]));
                sc = std::max(sc, std::abs(r1.v[i]));
            }
            bool threw = false;
            try {
                b200::ge_step(r1, PivotBlock{0.123, 0.456, 1.0, 0.5, 1.0, 1.0});
            } catch (const index_error&) {
                threw = true;
            }
            if (mx > 1e-14 * sc || !threw) {
                std::printf("ge mismatch %.3g %d\n", mx / sc, int(threw));
                return 1;
            }
        }
        std::printf("assemble / analyze_2d / sample_grid / grid solves / ge ok\n");
        return 0;
    } catch (const std::runtime_error& e) {
        std::printf("device error: %s\n", e.what());
        return 3;
    }
}
