// Compiles the C++ drop-in shim against the REFERENCE's own headers and links
// it with libsk_poisson.so (tests/test_integration.py).  With a device the
// solve must be bit-identical to the reference's on k != 0 columns; without
// one it must fail loudly (no CPU fallback).
#include <cstdio>
#include <cstring>

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
        return 0;
    } catch (const std::runtime_error& e) {
        std::printf("device error: %s\n", e.what());
        return 3;
    }
}
