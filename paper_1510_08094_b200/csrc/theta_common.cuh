// Shared device helpers of the theta-stage kernels (grid_kernels.cu,
// grid_large.cu): spectrum addressing, the per-mode chain structure of
// (lap - k^2) and the pivot windows.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "sk_internal.h"

namespace sk {

// Last cluster barrier of a kernel whose CTAs read peer shared memory just
// before it: it only has to keep each CTA's shared memory alive until the
// peer has finished reading. Every such read feeds a global store issued
// before the reader arrives, so a relaxed arrive suffices; cluster.sync()'s
// release would also wait for all of the CTA's global stores to complete
// (ncu: 10 % membar stalls in lambda_fwd_pair_kernel). relaxed = 0 for A/B
// (host side: exit_relaxed(), SK_PAIR_SYNC_EXIT=1).
// CONTRACT at every call site: between the previous cluster barrier and this
// one a CTA may only LOAD peer shared memory, and every loaded value must be
// consumed (feed a store or a register the CTA later uses) before the
// arrive.  A kernel that STORES to peer shared memory (st.shared::cluster,
// DSMEM atomics), or issues a DSMEM load whose value is unused, must pass
// relaxed = 0 (release-ordered cluster.sync()).  Kernels with no DSMEM
// access after their last barrier need no exit barrier at all
// (lambda_fwd_split_kernel).  tests/test_gpu_layer.py
// test_exit_barrier_variants_bitwise runs every call site under both forms.
__device__ __forceinline__ void cluster_exit_barrier(int relaxed) {
    if (relaxed) {
        asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
        asm volatile("barrier.cluster.wait;" ::: "memory");
    } else {
        cooperative_groups::this_cluster().sync();
    }
}


// ------------------------------------------------------------------ layout
// Element (kl, p) of a lambda-mode column on the theta rank: pieces from each
// source rank s are [kl][p - row_b[s]] blocks of ncols x rows_s, concatenated.
__device__ __forceinline__ size_t theta_addr(const Slabs& sl, int ncols, int kl, int p) {
    int s = 0;
    while (s + 1 < sl.P && p >= sl.row_b[s + 1]) ++s;
    const int r0 = sl.row_b[s];
    const int rows_s = sl.row_b[s + 1] - r0;
    return static_cast<size_t>(ncols) * r0 + static_cast<size_t>(kl) * rows_s + (p - r0);
}


__device__ __forceinline__ double2* peer_ptr(const PeerMap& pm, int idx, long long a, long long b) {
    int d = 0;
    while (d + 1 < pm.n && idx >= pm.bound[d + 1]) ++d;
    return pm.base[d] + (pm.off[d] + a * pm.mul[d] + b);
}

// theta-mode index of natural FFT index tau in parity class par (t = 2 tau + par
// folded into [-M/2, M/2)).
__device__ __forceinline__ int t_of(int tau, int par, int L) {
    const int t = 2 * tau + par;
    return t < L ? t : t - 2 * L;
}

// The four chains of one lambda mode.  Parity class par (t = 2 tau + par),
// side +: t = t0, t0+2, ... (tau ascending from tau0), side -: t = -2+par,
// -4+par, ... (tau descending from L-1).  Element i of a chain is coupled to
// i-1 (towards j = 0) and i+1 (towards the truncation boundary).
constexpr int kSegMax = 12;  // register-resident chain segment length per thread
constexpr int kFoldMax = 12;  // column pairs per thread in the fold
constexpr int kFoldMaxHi = 6;  // same, high-occupancy theta variant

struct Chain {
    int n;       // length
    int tau0;    // natural FFT index of element 0
    int dtau;    // +1 (t > 0 chain) or -1 (t < 0 chain)
    int t0;      // theta mode of element 0
    int dt;      // +2 or -2
};

__device__ __forceinline__ void make_chains(int par, int L, Chain& cp, Chain& cm) {
    if (par == 0) {
        cp = Chain{(L - 1 >= 2) ? (L - 1 - 2) / 2 + 1 : 0, 1, +1, 2, +2};
        cm = Chain{(L >= 2) ? (L - 2) / 2 + 1 : 0, L - 1, -1, -2, -2};
    } else {
        cp = Chain{(L - 1 >= 1) ? (L - 1 - 1) / 2 + 1 : 0, 0, +1, 1, +2};
        cm = Chain{(L >= 1) ? (L - 1) / 2 + 1 : 0, L - 1, -1, -1, -2};
    }
}

// Coefficients of row t of (lap - k^2) (poisson.cpp:15-40 closed form; the
// +-1 offsets are exact zeros): lower = lap[t][t-2], upper = lap[t][t+2].
__device__ __forceinline__ double lap_lower(int t, int L) {
    return (t - 2 >= -L) ? (double)(t - 2) * (double)(t - 1) * 0.25 : 0.0;
}
__device__ __forceinline__ double lap_upper(int t, int L) {
    return (t + 2 <= L - 1) ? (double)(t + 2) * (double)(t + 1) * 0.25 : 0.0;
}
__device__ __forceinline__ double lap_diag(int t, int L) {
    const double tt = t;
    if (t == -L) return -tt * (tt - 1.0) * 0.25;
    if (t == L - 1) return -tt * (tt + 1.0) * 0.25;
    return -tt * tt * 0.5;
}
// Msin^2 diagonal (poisson.cpp:61; 1/4 on the first and last rows)
__device__ __forceinline__ double msin2_diag(int t, int L) { return (t == -L || t == L - 1) ? 0.25 : 0.5; }

// chain-local coefficients: A couples to element i-1, C to element i+1.
// With sigma = sign(dt): A = (t - 2 sigma)(t - sigma)/4 (it vanishes at the
// first element, t0 in {+-1, +-2}), C = (t + 2 sigma)(t + sigma)/4 except at
// the last element, where the neighbour falls off the truncated operator.
__device__ __forceinline__ double chainA(const Chain& ch, int i, int L) {
    const double t = ch.t0 + ch.dt * i, sg = ch.dt > 0 ? 1.0 : -1.0;
    (void)L;
    return 0.25 * (t - 2.0 * sg) * (t - sg);
}
__device__ __forceinline__ double chainC(const Chain& ch, int i, int L) {
    const double t = ch.t0 + ch.dt * i, sg = ch.dt > 0 ? 1.0 : -1.0;
    (void)L;
    return (i + 1 < ch.n) ? 0.25 * (t + 2.0 * sg) * (t + sg) : 0.0;
}
// Msin^2 diagonal along a chain: 1/4 only at the truncation rows t = -L and
// t = L-1, which can only be a chain's last element.
__device__ __forceinline__ double chainD2(const Chain& ch, int i, int L) {
    const int t = ch.t0 + ch.dt * i;
    return (i + 1 == ch.n && (t == -L || t == L - 1)) ? 0.25 : 0.5;
}

// Issue the bulk copy of a chain's pivot window (16-byte aligned superset of
// table entries [row + tau_lo, row + tau_hi)) into `dst`; returns the pointer
// p with p[tau] = pivot of the element at natural index tau, and the bytes.
__device__ __forceinline__ const double* pivot_window(double* dst, const double* row, size_t row_abs, int tau_lo,
                                                      int tau_hi, uint32_t& bytes) {
    const size_t a0 = (row_abs + tau_lo) & ~static_cast<size_t>(1);
    const size_t a1 = (row_abs + tau_hi + 1) & ~static_cast<size_t>(1);
    bytes = static_cast<uint32_t>((a1 - a0) * 8);
    return dst + (static_cast<long long>(row_abs) - static_cast<long long>(a0));
}

// Same for a chain's entries of the digit-reversal table (ints, windows
// aligned to 16 bytes; the table is padded to a multiple of 4 entries).
__device__ __forceinline__ const int* rev_window(int* dst, int tau_lo, int tau_hi, int& a0, uint32_t& bytes) {
    a0 = tau_lo & ~3;
    const int a1 = (tau_hi + 3) & ~3;
    bytes = static_cast<uint32_t>(a1 - a0) * 4;
    return dst - a0;
}

}  // namespace sk
