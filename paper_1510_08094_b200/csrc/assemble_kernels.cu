// assemble_poisson on the GPU (poisson.cpp:52-86): the coefficients F of
// sin^2(theta) f~ for a low-rank function f~ = sum_j d_j a_j(theta) b_j(lambda)
// given by its factors (LowRankSphereFun, lowrank.hpp:47-59).
//
//   K8 assemble_factors_kernel — per term j: SA_j = d_j * Msin^2 pad(a_j, M)
//        (band_mul(msin, msin).apply, banded.cpp:8-19, ascending band index,
//        exact-zero +-1 entries included) and B_j = pad(b_j, N) (pad_to,
//        fourier.cpp:105-112); one thread per (j, i) entry.
//   K9 assemble_outer_kernel — F[i][k] = sum_j SA_j[i] B_j[k], accumulated
//        term by term in ascending j with the j-terms whose SA_j[i] is an
//        exact zero skipped (poisson.cpp:62-71); a thread owns one column of
//        a 16-row tile, rows of F written coalesced.  K complex multiply-adds
//        (8 FP64 instructions each, no FMA) per 16-byte store: HBM-bound
//        (16 M N bytes) for small K, FP64-bound beyond K ~ 6.
//   K10 assemble_terms_kernel + assemble_mean_kernel — sum2 (calculus.cpp:
//        89-103): per term (one warp each) the weighted even-mode sum of a_j
//        (ascending k) times 2 pi b_j(0); the terms summed in order;
//        mu = sum2 / (4 pi); if |mu| > 1e-11 max(vscale, 1e-300) the
//        coefficients of mu sin^2(theta) are subtracted (:76-82).
//
// This translation unit is compiled with --fmad=false: every complex product
// is (ac - bd, ad + bc) with separately rounded multiplies, as std::complex
// evaluates it in the reference build (no FMA contraction on x86-64), so F is
// bit-identical to the reference.
#include <cuda_runtime.h>

#include "params.h"

namespace sk {

namespace {

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// pad_to: mode t of a length-len vector sits at t + len/2; reads outside are 0
__device__ __forceinline__ double2 pad_at(const double2* v, int len, int t) {
    const int i = t + len / 2;
    return (i >= 0 && i < len) ? v[i] : make_double2(0.0, 0.0);
}

}  // namespace

__global__ void assemble_factors_kernel(AssembleParams P) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long nsa = static_cast<long long>(P.K) * P.M;
    if (idx < nsa) {
        const int j = static_cast<int>(idx / P.M), i = static_cast<int>(idx - static_cast<long long>(j) * P.M);
        const double2* a = P.col + static_cast<long long>(j) * P.mf;
        // Msin^2 row i: (-1/4, 0, 1/2, 0, -1/4) at offsets -2..2, 1/4 on the
        // first and last diagonal entries; all imaginary parts +0
        double2 acc = make_double2(0.0, 0.0);
        const int jlo = i - 2 < 0 ? 0 : i - 2, jhi = i + 2 > P.M - 1 ? P.M - 1 : i + 2;
        for (int c = jlo; c <= jhi; ++c) {
            const int off = c - i;
            double s;
            if (off == 0) s = (i == 0 || i == P.M - 1) ? 0.25 : 0.5;
            else if (off == 2 || off == -2) s = -0.25;
            else s = 0.0;
            const double2 pr = zmul(make_double2(s, 0.0), pad_at(a, P.mf, c - P.M / 2));
            acc = make_double2(acc.x + pr.x, acc.y + pr.y);
        }
        P.sa[idx] = zmul(P.d[j], acc);
        return;
    }
    const long long ib = idx - nsa;
    if (ib < static_cast<long long>(P.K) * P.N) {
        const int j = static_cast<int>(ib / P.N), k = static_cast<int>(ib - static_cast<long long>(j) * P.N);
        P.bp[ib] = pad_at(P.row + static_cast<long long>(j) * P.nf, P.nf, k - P.N / 2);
    }
}

// Register tile: each thread owns column k and kTileRows consecutive rows; the
// SA_j values of the tile rows are staged in shared memory (warp-uniform
// broadcast reads) a chunk of terms at a time, B_j[k] is one coalesced load
// reused across the tile rows.
constexpr int kTileRows = 16;
constexpr int kTermChunk = 32;

__global__ void __launch_bounds__(256) assemble_outer_kernel(AssembleParams P) {
    __shared__ double2 s_sa[kTermChunk][kTileRows];
    __shared__ unsigned s_nz[kTermChunk];  // bit r: SA_j[i0 + r] != 0 (the skip test, off the FP64 pipe)
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i0 = blockIdx.y * kTileRows;
    const int nrow = min(kTileRows, P.M - i0);
    double2 f[kTileRows];
#pragma unroll
    for (int r = 0; r < kTileRows; ++r) f[r] = make_double2(0.0, 0.0);
    for (int j0 = 0; j0 < P.K; j0 += kTermChunk) {
        const int nj = min(kTermChunk, P.K - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < kTermChunk * kTileRows; e += blockDim.x) {
            const int jj = e / kTileRows, r = e - jj * kTileRows;
            const double2 v = (jj < nj && r < nrow) ? P.sa[static_cast<long long>(j0 + jj) * P.M + i0 + r]
                                                    : make_double2(0.0, 0.0);
            s_sa[jj][r] = v;
            // kTileRows = 16 consecutive e share jj: a half-warp ballot builds the mask
            const unsigned bal = __ballot_sync(0xffffffffu, v.x != 0.0 || v.y != 0.0);
            if ((threadIdx.x & 15) == 0) s_nz[jj] = (bal >> (threadIdx.x & 16)) & 0xffffu;
        }
        __syncthreads();
        if (k < P.N) {
            for (int jj = 0; jj < nj; ++jj) {
                const double2 b = P.bp[static_cast<long long>(j0 + jj) * P.N + k];
                const unsigned nz = s_nz[jj];
#pragma unroll
                for (int r = 0; r < kTileRows; ++r) {
                    if (!((nz >> r) & 1u)) continue;  // poisson.cpp:66 (block-uniform)
                    const double2 pr = zmul(s_sa[jj][r], b);
                    f[r] = make_double2(f[r].x + pr.x, f[r].y + pr.y);
                }
            }
        }
    }
    if (k < P.N) {
#pragma unroll
        for (int r = 0; r < kTileRows; ++r)
            if (r < nrow) P.F[static_cast<long long>(i0 + r) * P.N + k] = f[r];
    }
}

// sum2 terms: one warp per term j.  The lanes form the products w_t a_t of 32
// consecutive modes (the divisions run in parallel), lane 0 adds them in
// ascending mode order (calculus.cpp:94-98); times d_j and 2 pi b_j(0).
__global__ void assemble_terms_kernel(AssembleParams P) {
    __shared__ double2 s_p[4][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int j = blockIdx.x * 4 + wib;
    if (j >= P.K) return;
    constexpr double kTwoPi = 2.0 * 3.141592653589793238462643383279502884;
    const double2* a = P.col + static_cast<long long>(j) * P.mf;
    double2 ci = make_double2(0.0, 0.0);
    for (int t0 = -P.mf / 2; t0 < P.mf / 2; t0 += 32) {
        const int t = t0 + lane;
        double2 pr = make_double2(0.0, 0.0);
        if (t < P.mf / 2 && t % 2 == 0) {
            const double w = 2.0 / (1.0 - static_cast<double>(t) * t);
            const double2 v = a[t + P.mf / 2];
            pr = make_double2(w * v.x, w * v.y);
        }
        s_p[wib][lane] = pr;
        __syncwarp();
        if (lane == 0) {
            for (int u = 0; u < 32 && t0 + u < P.mf / 2; ++u) {
                if ((t0 + u) % 2 != 0) continue;
                ci = make_double2(ci.x + s_p[wib][u].x, ci.y + s_p[wib][u].y);
            }
        }
        __syncwarp();
    }
    if (lane != 0) return;
    const double2 b0 = pad_at(P.row + static_cast<long long>(j) * P.nf, P.nf, 0);
    P.sa[static_cast<long long>(P.K) * P.M + j] = zmul(zmul(P.d[j], ci), make_double2(kTwoPi * b0.x, kTwoPi * b0.y));
}

__global__ void assemble_mean_kernel(AssembleParams P) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    constexpr double kPi = 3.141592653589793238462643383279502884;
    double2 total = make_double2(0.0, 0.0);
    for (int j = 0; j < P.K; ++j) {  // term order, as sum2 accumulates
        const double2 term = P.sa[static_cast<long long>(P.K) * P.M + j];
        total = make_double2(total.x + term.x, total.y + term.y);
    }
    const double2 mu = make_double2(total.x / (4.0 * kPi), total.y / (4.0 * kPi));
    const double vs = P.vscale > 1e-300 ? P.vscale : 1e-300;
    const bool removed = hypot(mu.x, mu.y) > 1e-11 * vs;
    P.report[0] = removed ? 1.0 : 0.0;
    P.report[1] = removed ? mu.x : 0.0;
    P.report[2] = removed ? mu.y : 0.0;
    if (!removed) return;
    auto sub = [&](int i, double s) {
        double2& f = P.F[static_cast<long long>(i) * P.N + P.N / 2];
        f = make_double2(f.x - mu.x * s, f.y - mu.y * s);
    };
    sub(P.M / 2, 0.5);
    if (P.M / 2 + 2 < P.M) sub(P.M / 2 + 2, -0.25);
    sub(P.M / 2 - 2, -0.25);
}

cudaError_t launch_assemble(const AssembleParams& P, cudaStream_t st) {
    const long long n1 = static_cast<long long>(P.K) * (P.M + P.N);
    if (n1 > 0) assemble_factors_kernel<<<static_cast<unsigned>((n1 + 255) / 256), 256, 0, st>>>(P);
    dim3 g((P.N + 255) / 256, (P.M + kTileRows - 1) / kTileRows);
    assemble_outer_kernel<<<g, 256, 0, st>>>(P);
    if (P.K > 0) assemble_terms_kernel<<<(P.K + 3) / 4, 128, 0, st>>>(P);
    assemble_mean_kernel<<<1, 32, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace sk
