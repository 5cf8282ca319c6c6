// Coefficient-space kernels (sm_100a), compiled with --fmad=false:
//
//   K5 coeff_solve — drop-in for spherekit::solve (poisson.cpp:121-161).
//   K6 residual    — spherekit::residual (poisson.cpp:163-186).
//   check_mean     — check_mean_zero (poisson.cpp:101-117).
//
// Layout: F, X row-major M x N complex (types.hpp:17-41); a lambda-mode column
// is strided by N, so a warp owns 32 consecutive columns and every row access
// of the warp is one contiguous 512-byte segment.
//
// Why four independent real recurrences reproduce the reference bit for bit:
// lap (poisson.cpp:35-38) has exact-zero +-1 offsets and real entries, its
// entries lap[+-2][0] and lap[+-1][-+1] are exact zeros, so for k != 0 the
// system splits into the chains {even, odd} x {j < 0, j > 0} plus the row
// j = 0, which couples x_0 to x_-2 and x_2 only.  The matrix is strictly
// column diagonally dominant for k != 0, so band_solve's partial pivoting
// (banded.cpp:121-133) never swaps and its elimination is the ascending Thomas
// recurrence.  Each complex operation of the reference has a zero imaginary
// part in the operator, so it decomposes into the real IEEE mul/sub/div used
// here, in the same order and without FMA contraction.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "params.h"

namespace sk {


// lap entries (exact dyadic values; see oracle/sk_oracle.cpp lap_band)
__device__ __forceinline__ double lapc_lower(int i, int M) {  // lap[i][i-2]
    const double j = i - M / 2;
    return __dmul_rn(__dmul_rn(j - 2.0, j - 1.0), 0.25);
}
__device__ __forceinline__ double lapc_upper(int i, int M) {  // lap[i][i+2]
    const double j = i - M / 2;
    return __dmul_rn(__dmul_rn(j + 2.0, j + 1.0), 0.25);
}
__device__ __forceinline__ double lapc_diag(int i, int M) {
    const double j = i - M / 2;
    if (i == 0) return -__dmul_rn(__dmul_rn(j, j - 1.0), 0.25);
    if (i == M - 1) return -__dmul_rn(__dmul_rn(j, j + 1.0), 0.25);
    return -__dmul_rn(__dmul_rn(j, j), 0.5);
}

// 0 / d for finite nonzero d: a zero with sign(num) xor sign(d) (IEEE 754)
__device__ __forceinline__ double signed_zero(double num, double d) {
    return __longlong_as_double((__double_as_longlong(num) ^ __double_as_longlong(d)) & static_cast<long long>(0x8000000000000000ULL));
}

// Chain rows of warp w (storage index i ascending): 0 even j<0, 1 odd j<0,
// 2 even j>0, 3 odd j>0.
__device__ __forceinline__ void chain_rows(int w, int M, int& i0, int& i1) {
    const int h = M / 2;
    const int even_lo = (h & 1) ? 1 : 0;  // i with j = i - h even
    if (w == 0) { i0 = even_lo; i1 = h - 2; }
    else if (w == 1) { i0 = 1 - even_lo; i1 = h - 1; }
    else if (w == 2) { i0 = h + 2; i1 = ((M - 1 - (h + 2)) / 2) * 2 + h + 2; }
    else { i0 = h + 1; i1 = ((M - 1 - (h + 1)) / 2) * 2 + h + 1; }
    if (i1 > M - 1) i1 -= 2;
}

// The elimination's data-independent half, once per plan: for every column
// and chain the pivots d'_i = b_i - l_i c_{i-2} and multipliers l_i = a_i /
// d'_{i-2} of band_solve's forward sweep (banded.cpp:121-147), by the same
// sequential IEEE recurrence, so that the per-solve sweeps below carry no
// division on the forward path and read d' instead of recomputing it.
// bad[0] counts the rows where band_solve would have swapped (|a| > |d'|) and
// 2^20 per singular pivot.  One lane per (column, chain).
__global__ void __launch_bounds__(128) coeff_tables_kernel(int M, int N, double* __restrict__ D, double* __restrict__ Lm,
                                                           double* bad_out) {
    const int h = M / 2;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int kc = blockIdx.x * 32 + lane;
    if (kc >= N) return;
    const int k = kc - N / 2;
    const double negk2 = __dmul_rn(-static_cast<double>(k), static_cast<double>(k));
    int i0, i1;
    chain_rows(w, M, i0, i1);
    (void)h;
    int bad = 0;
    double dprev = 0.0;
    for (int i = i0, q = 0; i <= i1; i += 2, ++q) {
        const double b = __dadd_rn(lapc_diag(i, M), negk2);
        double d = b, l = 0.0;
        if (q > 0) {
            const double a = lapc_lower(i, M);
            if (a != 0.0) {
                if (fabs(a) > fabs(dprev)) ++bad;  // band_solve would have swapped rows
                l = __ddiv_rn(a, dprev);
                d = __dsub_rn(b, __dmul_rn(l, lapc_upper(i - 2, M)));
            } else {
                bad += 1 << 20;  // a vanishing sub-diagonal inside a chain: not this operator
            }
        }
        if (fabs(d) < 1e-300) bad += 1 << 20;
        D[static_cast<size_t>(i) * N + kc] = d;
        Lm[static_cast<size_t>(i) * N + kc] = l;
        dprev = d;
    }
    if (bad) atomicAdd(bad_out, static_cast<double>(bad));
}

// K5.  A lane owns ONE REAL COMPONENT of one column: lanes (2c, 2c+1) hold the
// real and imaginary parts of column c (the operator is real, so the two
// components of the complex right-hand side are independent real recurrences
// sharing the tables).  A warp's row access is one contiguous 256-byte segment
// of the interleaved complex row, there are twice as many independent
// recurrences in flight, and each back-substitution step carries one division.
// Each thread's sweeps are a long dependent recurrence over M/4 rows; the
// loads of the rows ahead (F and l forward, r and d' backward) do not depend
// on it, so they are issued a block of kPf rows ahead, which keeps kPf * 16 B
// per thread in flight instead of one row's latency per step.  (A rolling
// one-row ring shares the few hardware scoreboards between old and young
// loads: waiting for the oldest row also waits for rows requested a few steps
// ago.)
constexpr int kPf = 16;

__global__ void __launch_bounds__(128) coeff_solve_kernel(CoeffParams P) {
    __shared__ double s_rm2[32];  // r'_{-2}
    __shared__ double s_x2[32];   // x_2
    const int M = P.M, N = P.N, h = M / 2, N2 = 2 * N;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int kc2 = blockIdx.x * 32 + lane;  // component column: 2 kc + (0 re, 1 im)
    const int kc = kc2 >> 1;
    const int rhs = blockIdx.y;
    const bool live = kc2 < N2;
    const unsigned lmask = __ballot_sync(0xffffffffu, live);  // live lanes come in (re, im) pairs
    const size_t off = static_cast<size_t>(rhs) * M * N;
    const double* __restrict__ F = reinterpret_cast<const double*>(P.F + off);
    double* __restrict__ X = reinterpret_cast<double*>(P.X + off);
    const double* __restrict__ D = P.D;
    const double* __restrict__ Lm = P.Lm;
    const int k = kc - N / 2;
    const double negk2 = __dmul_rn(-static_cast<double>(k), static_cast<double>(k));  // -static_cast<double>(k) * k
    const int even_lo = (h & 1) ? 1 : 0;  // i with j = i - h even
    int i0, i1;
    chain_rows(w, M, i0, i1);
    const int nrow = (live && i0 <= i1) ? (i1 - i0) / 2 + 1 : 0;  // rows i0, i0+2, ..., i1
    double fmx = 0.0;  // max of the pair's re^2 + im^2
    // ---- forward elimination: r_i = F_i - l_i r_{i-2}
    double rprev = 0.0;
    if (nrow > 0) {
        double cur[kPf], nxt[kPf], lc[kPf], ln[kPf];
#pragma unroll
        for (int u = 0; u < kPf; ++u) {
            cur[u] = u < nrow ? F[static_cast<size_t>(i0 + 2 * u) * N2 + kc2] : 0.0;
            lc[u] = u < nrow ? Lm[static_cast<size_t>(i0 + 2 * u) * N + kc] : 0.0;
        }
        for (int q0 = 0; q0 < nrow; q0 += kPf) {
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                const bool in = q0 + kPf + u < nrow;
                const int i = i0 + 2 * (q0 + kPf + u);
                nxt[u] = in ? F[static_cast<size_t>(i) * N2 + kc2] : 0.0;
                ln[u] = in ? Lm[static_cast<size_t>(i) * N + kc] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                const int q = q0 + u;
                if (q < nrow) {
                    const int i = i0 + 2 * q;
                    const double f = cur[u];
                    // |F|^2 = re^2 + im^2 from the lane pair (max|F| only scales the precondition test)
                    const double f2 = f * f;
                    fmx = fmax(fmx, f2 + __shfl_xor_sync(lmask, f2, 1));
                    const double r = (q > 0) ? __dsub_rn(f, __dmul_rn(lc[u], rprev)) : f;
                    X[static_cast<size_t>(i) * N2 + kc2] = r;
                    rprev = r;
                }
            }
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                cur[u] = nxt[u];
                lc[u] = ln[u];
            }
        }
    }
    if (w == 0 && live) s_rm2[lane] = rprev;  // chain ends at j = -2
    // ---- back substitution: x_i = (r_i - c_i x_{i+2}) / d'_i  (rows i1, i1-2, ..., i0)
    double xnext = 0.0;
    if (nrow > 0) {
        double rr[kPf], dr[kPf], rn[kPf], dn[kPf];
#pragma unroll
        for (int u = 0; u < kPf; ++u) {
            rr[u] = u < nrow ? X[static_cast<size_t>(i1 - 2 * u) * N2 + kc2] : 0.0;
            dr[u] = u < nrow ? D[static_cast<size_t>(i1 - 2 * u) * N + kc] : 1.0;
        }
        for (int q0 = 0; q0 < nrow; q0 += kPf) {
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                const bool in = q0 + kPf + u < nrow;
                const int i = i1 - 2 * (q0 + kPf + u);
                rn[u] = in ? X[static_cast<size_t>(i) * N2 + kc2] : 0.0;
                dn[u] = in ? D[static_cast<size_t>(i) * N + kc] : 1.0;
            }
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                const int q = q0 + u;
                if (q < nrow) {
                    const int i = i1 - 2 * q;
                    double acc = rr[u];
                    if (i + 2 <= M - 1) {
                        const double c = lapc_upper(i, M);
                        if (c != 0.0) acc = __dsub_rn(acc, __dmul_rn(c, xnext));
                    }
                    // a zero numerator leaves the division's fast path (its range
                    // check reads the quotient's magnitude) for a long subroutine;
                    // band-limited right-hand sides are mostly zeros: +-0 directly,
                    // with the IEEE sign of 0 / d
                    const double x = (acc == 0.0) ? signed_zero(acc, dr[u]) : __ddiv_rn(acc, dr[u]);
                    X[static_cast<size_t>(i) * N2 + kc2] = x;
                    xnext = x;
                }
            }
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                rr[u] = rn[u];
                dr[u] = dn[u];
            }
        }
    }
    if (w == 2 && live) s_x2[lane] = xnext;  // chain starts at j = 2
    __syncthreads();
    // ---- row j = 0
    if (w == 0 && live) {
        const double f0 = F[static_cast<size_t>(h) * N2 + kc2];
        const double f02 = f0 * f0;
        fmx = fmax(fmx, f02 + __shfl_xor_sync(lmask, f02, 1));
        const bool has_m2 = (h - 2) >= 0;
        const bool has_p2 = (h + 2) <= M - 1;
        if (k != 0) {
            double r0 = f0;
            if (has_m2) {  // eliminate with pivot row j = -2: f = lap[0][-2] / d'_{-2}
                const double l = __ddiv_rn(lapc_lower(h, M), D[static_cast<size_t>(h - 2) * N + kc]);
                r0 = __dsub_rn(r0, __dmul_rn(l, s_rm2[lane]));
            }
            if (has_p2) {
                const double c = lapc_upper(h, M);
                r0 = __dsub_rn(r0, __dmul_rn(c, s_x2[lane]));
            }
            const double d0 = __dadd_rn(lapc_diag(h, M), negk2);
            X[static_cast<size_t>(h) * N2 + kc2] = __ddiv_rn(r0, d0);
        }
    }
    __syncthreads();
    if (k == 0 && live && w == 0) {
        // constraint row 2 pi w^T X_0 = 0 replaces row j = 0:
        // x_0 = -(sum_{j != 0, j even} w_j x_j) / w_0, w_j = 2 / (1 - j^2)
        double s = 0.0;
        for (int i = even_lo; i < M; i += 2) {
            if (i == h) continue;
            const double j = i - h;
            const double wj = 2.0 / (1.0 - j * j);
            s = __dadd_rn(s, __dmul_rn(wj, X[static_cast<size_t>(i) * N2 + kc2]));
        }
        X[static_cast<size_t>(h) * N2 + kc2] = -__ddiv_rn(s, 2.0);
    }
    // stats
    const double fm = sqrt(warp_max(live ? fmx : 0.0));
    if (lane == 0) atomic_max_nonneg(P.stats + 4 * rhs + 2, fm);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double tb = *P.tab_bad;
        if (tb != 0.0) atomicAdd(P.stats + 4 * rhs + 3, tb);
    }
}

// check_mean_zero (poisson.cpp:101-117): the reference computes
// 2 pi w^T div_sin(div_sin(F_0)); with Msin^T = -Msin this equals
// 2 pi z^T F_0 for z = Msin^-1 Msin^-1 w, precomputed per plan.
__global__ void __launch_bounds__(256) mean_kernel(CoeffParams P) {
    __shared__ double red[64];
    const int rhs = blockIdx.x;
    const double2* F = P.F + static_cast<size_t>(rhs) * P.M * P.N;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < P.M; i += blockDim.x) {
        const double2 f = F[static_cast<size_t>(i) * P.N + P.N / 2];
        const double2 z = P.z[i];
        acc.x += z.x * f.x - z.y * f.y;
        acc.y += z.x * f.y + z.y * f.x;
    }
    acc = block_sum2(acc, red);
    if (threadIdx.x == 0) {
        const double twopi = 6.283185307179586476925286766559;
        P.stats[4 * rhs + 0] = twopi * acc.x;
        P.stats[4 * rhs + 1] = twopi * acc.y;
    }
}


// residual (poisson.cpp:163-186): r = lap x_k - (k^2 x_k + F_k) per column.
__global__ void __launch_bounds__(128) residual_kernel(ResidualParams P) {
    const int M = P.M, N = P.N, h = M / 2;
    const int kc = blockIdx.x * blockDim.x + threadIdx.x;
    double imax = 0.0;
    if (kc < N) {
        const double k = kc - N / 2;
        const double k2 = k * k;
        double2 xw[5];  // x_{i-2} .. x_{i+2}
        for (int q = 0; q < 5; ++q) {
            const int i = q - 2;
            xw[q] = (i >= 0 && i < M) ? P.X[static_cast<size_t>(i) * N + kc] : make_double2(0.0, 0.0);
        }
        double2 wsum = make_double2(0.0, 0.0);
        for (int i = 0; i < M; ++i) {
            double2 r = make_double2(0.0, 0.0);
            if (i - 2 >= 0) {
                const double a = lapc_lower(i, M);
                r.x += a * xw[0].x;
                r.y += a * xw[0].y;
            }
            {
                const double b = lapc_diag(i, M);
                r.x += b * xw[2].x;
                r.y += b * xw[2].y;
            }
            if (i + 2 < M) {
                const double c = lapc_upper(i, M);
                r.x += c * xw[4].x;
                r.y += c * xw[4].y;
            }
            const double2 f = P.F[static_cast<size_t>(i) * N + kc];
            r.x -= k2 * xw[2].x + f.x;
            r.y -= k2 * xw[2].y + f.y;
            const double ab = hypot(r.x, r.y);
            if (kc == N / 2 && i == h) {
                P.out[1] = ab;
            } else {
                imax = fmax(imax, ab);
            }
            if (kc == N / 2) {
                const int j = i - h;
                if ((j & 1) == 0) {
                    const double wj = 2.0 / (1.0 - static_cast<double>(j) * j);
                    wsum.x += wj * xw[2].x;
                    wsum.y += wj * xw[2].y;
                }
            }
            for (int q = 0; q < 4; ++q) xw[q] = xw[q + 1];
            xw[4] = (i + 3 < M) ? P.X[static_cast<size_t>(i + 3) * N + kc] : make_double2(0.0, 0.0);
        }
        if (kc == N / 2) {
            P.out[2] = wsum.x;
            P.out[3] = wsum.y;
        }
    }
    const double m = warp_max(imax);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(P.out, m);
}

// F = Msin^2 A column by column (the reference's composition applies
// band_mul(msin, msin).apply to every column, poisson.cpp:61 / ref harness):
// row i of Msin^2 is (-1/4, 0, 1/2, 0, -1/4) at offsets -2..2 with 1/4 on the
// first and last diagonal entries, all imaginary parts +0; the products and
// the ascending accumulation (including the exact-zero +-1 terms) are those of
// BandMatrix::apply (banded.cpp:8-19), so F is bit-identical.  One thread per
// entry, consecutive threads on consecutive columns (coalesced rows).
__global__ void __launch_bounds__(256) msin2_kernel(int M, int N, const double2* __restrict__ A, double2* __restrict__ F) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(M) * N) return;
    const int i = static_cast<int>(idx / N);
    const int kc = static_cast<int>(idx - static_cast<long long>(i) * N);
    double2 acc = make_double2(0.0, 0.0);
    const int jlo = i - 2 < 0 ? 0 : i - 2, jhi = i + 2 > M - 1 ? M - 1 : i + 2;
    for (int c = jlo; c <= jhi; ++c) {
        const int off = c - i;
        double s;
        if (off == 0) s = (i == 0 || i == M - 1) ? 0.25 : 0.5;
        else if (off == 2 || off == -2) s = -0.25;
        else s = 0.0;
        const double2 x = A[static_cast<long long>(c) * N + kc];
        // (s + 0i) * x, as std::complex multiplication
        const double2 pr = make_double2(s * x.x - 0.0 * x.y, s * x.y + 0.0 * x.x);
        acc = make_double2(acc.x + pr.x, acc.y + pr.y);
    }
    F[idx] = acc;
}

cudaError_t launch_msin2(int M, int N, const double2* A, double2* F, cudaStream_t st) {
    const long long n = static_cast<long long>(M) * N;
    msin2_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(M, N, A, F);
    return cudaGetLastError();
}

cudaError_t launch_coeff_tables(int M, int N, double* D, double* Lm, double* bad, cudaStream_t st) {
    coeff_tables_kernel<<<(N + 31) / 32, 128, 0, st>>>(M, N, D, Lm, bad);
    return cudaGetLastError();
}

cudaError_t launch_coeff_solve(const CoeffParams& P, cudaStream_t st) {
    if (P.z) {
        mean_kernel<<<P.nrhs, 256, 0, st>>>(P);
    }
    dim3 grid((2 * P.N + 31) / 32, P.nrhs);  // one lane per real component of a column
    coeff_solve_kernel<<<grid, 128, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_residual(const ResidualParams& P, cudaStream_t st) {
    residual_kernel<<<(P.N + 127) / 128, 128, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace sk
