// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// CPU restatement (C++20, scalar, plain IEEE double, no FMA contraction) of
// the reference's DFS spectral Poisson hot path.  Only tests/, the smoke()
// check in __graft_entry__.py and bench.py's cpu_baseline leg may load it, and
// only as the checker / CPU baseline — never as the product path.
//
// Layouts follow the reference exactly:
//   * coefficient matrices: row-major M x N complex (interleaved re,im),
//     row i <-> theta mode j = i - M/2, column kc <-> lambda mode k = kc - N/2
//     (proj/include/spherekit/types.hpp:17-41, poisson.hpp:23-30);
//   * doubled grids: row-major M x N complex, theta_i = -pi + 2 pi i/M,
//     lambda_q = -pi + 2 pi q/N (sphere_domain.hpp:43-58);
//   * physical grids: row-major (M/2+1) x N real, theta_p = 2 pi p/M (both
//     poles), lambda_q = -pi + 2 pi q/N.
// Status codes: 0 ok, 1 size_error, 2 precondition_error, 3 structure_error.
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

const char* sko_last_error(void);

// poisson.cpp:15-40 build_operators(m).lap as real band lap[i*5 + (j-i+2)]
int sko_build_lap(int m, double* lap);
// poisson.cpp:42-50 (real parts; imaginary parts are zero)
int sko_integration_weights(int m, double* w);

// banded.cpp:101-158 (complex band, band[i*(kl+ku+1) + (j-i+kl)])
int sko_band_solve(int n, int kl, int ku, const double* band, const double* b, double* x);
// banded.cpp:160-328
int sko_band_solve_dense_row(int n, int kl, int ku, const double* band, int skip_row, const double* w,
                             double wrhs_re, double wrhs_im, const double* b, double* x);
// fourier.cpp:92-103
int sko_div_sin(int n, const double* c, double* out);

// poisson.cpp:121-161 (solve) incl. check_mean_zero (:101-117); threads like
// thread_budget (:90-99) with an explicit cap (<=0: hardware concurrency).
int sko_solve(int m, int n, const double* F, double* X, int threads);
// poisson.cpp:163-186 -> out[3] = {interior_max, replaced_row_abs, constraint_abs}
int sko_residual(int m, int n, const double* F, const double* X, double* out);
// Msin^2 applied per column (poisson.cpp:61-71, :214)
int sko_msin2_columns(int m, int n, const double* X, double* F);

// fourier.cpp:39-66
int sko_analyze_1d(int n, const double* s, double* c);
int sko_synthesize_1d(int n, const double* c, int n_out, double* g);
// fourier.cpp:170-209
int sko_analyze_2d(int m, int n, const double* grid, double* X);
// lowrank.cpp:84-112 / :127-162 (out_i: found, t, k; out_d / piv: a, b, m_even, m_odd, theta_star, lambda_star)
int sko_pivot_search(int m, int n, const double* grid, double alpha, int* out_i, double* out_d);
int sko_ge_step(int m, int n, const double* grid, const double* piv, double* out);
// lowrank.cpp:345-392: one phase-1 step (search + update) on the (g/2+1) x g upper half grid
int sko_ge_half_step(int g, const double* e, double alpha, int* out_i, double* out_d, double* out);
int sko_sample_grid(int rows, int cols, const double* X, int m_out, int n_out, double* grid);

// sphere_domain.cpp:19-26, :46-52 applied to physical samples (index map a3)
int sko_dfs_double(int m, int n, const double* phys, double* grid);

// poisson.cpp:52-86 on raw low-rank factors: d[K], col[K][mf], row[K][nf]
// (complex); F (m x n complex); rep[3] = {mean removed?, mu re, mu im}
int sko_assemble(int K, int mf, int nf, const double* d, const double* col, const double* row, double vscale, int m,
                 int n, double* F, double* rep);

// doubling -> analyze_2d -> Msin^2 -> solve -> sample_grid.
// X (M x N complex) and u_doubled (M x N complex) may be NULL.
// u_phys ((M/2+1) x N real) = Re(u_doubled) on physical rows (p < M/2 from
// doubled row M/2+p, p = M/2 from doubled row 0), may be NULL.
int sko_grid_pipeline(int m, int n, const double* phys, double* X, double* u_doubled, double* u_phys,
                      int threads, double* mean_out);

// Test-input generators (same RNG streams as the reference):
// bench_poisson's coefficient workload (poisson.cpp:190-216); `sizes` lists
// every size generated before the wanted (last) one in the same call.
int sko_bench_problem(int nsizes, const int* sizes, double* F_last);
// tests/support/poisson_oracle.hpp:119-154
int sko_random_mean_zero_problem(int m, int n, unsigned seed, double* F);

// Real spherical-harmonic sum on the physical grid (BASELINE configs):
// f = sum_{l=1..L} sum_{|m|<=l} c[l*l+l+m] Y_l^m, Y in the reference tests'
// convention (tests/support/helpers.hpp:18-27).  Direct evaluation, small
// sizes only (checks the device generator).
int sko_shgen(int m, int n, int L, const double* coeffs, double* phys, int threads);

#ifdef __cplusplus
}
#endif
