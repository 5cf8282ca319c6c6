// Structure-preserving Gaussian elimination on a doubled BMC grid (sm_100a),
// compiled with --fmad=false: the device side of the reference's
//   pivot_search  lowrank.cpp:84-112  (complete pivoting over 2x2 blocks)
//   ge_step       lowrank.cpp:127-162 (the rank-<=2 update of the whole grid)
// and so of the phase-1 loop of construct (lowrank.cpp:318-415, the update
// of :384-392), which runs the same arithmetic on the upper half grid.
//
// Layout: the reference's BMCGrid (sphere_domain.hpp:43-58): m x n complex,
// row-major, row j <-> theta_j = -pi + 2 pi j/m, column k <-> lambda_k.
//
// Bit-exactness of the update: the reference accumulates
//   upd = 0; upd += de * ce[j] * re[k]; upd += dodd * co[j] * ro[k]; out -= upd
// with std::complex products evaluated left to right, each (x + iy)(u + iv) =
// (xu - yv) + i(xv + yu) in separate IEEE operations (libgcc __muldc3's
// non-NaN path; no FMA on x86-64 baseline): reproduced here operation by
// operation, including the additions to the zero-initialised accumulator.
// The pivot search compares sigma_1 = max(|a + b|, |a - b|) by hypot(); a
// candidate is taken only if strictly larger, so the first maximal block in
// (theta* ascending, lambda* ascending) order wins: the reduction below keeps
// the smallest candidate index among equal maxima.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "params.h"

namespace sk {

namespace {

__device__ __forceinline__ double2 cmul_ref(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

struct Cand {
    double s;        // sigma_1 of the block (0: none)
    long long c;     // candidate index t * (n/2) + (k - n/2), -1: none
};
__device__ __forceinline__ Cand better(Cand x, Cand y) {  // larger sigma_1, then smaller index
    if (y.c < 0) return x;
    if (x.c < 0) return y;
    if (y.s > x.s || (y.s == x.s && y.c < x.c)) return y;
    return x;
}
__device__ __forceinline__ Cand warp_best(Cand v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Cand o;
        o.s = __shfl_xor_sync(0xffffffffu, v.s, off);
        o.c = __shfl_xor_sync(0xffffffffu, v.c, off);
        v = better(v, o);
    }
    return v;
}
__device__ __forceinline__ Cand block_best(Cand v, Cand* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_best(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    Cand t = red[0];
    for (int w = 1; w < nw; ++w) t = better(t, red[w]);
    return t;
}

}  // namespace

// part[blockIdx.x] = best candidate of this block's share
// half: g holds only the upper half grid, row i <-> theta_i = 2 pi i / m (i = 0..m/2), as construct's phase 1
// keeps it (lowrank.cpp:246-252); else the doubled grid (row of theta* = 2 pi t / m is (m/2 + t) mod m)
__global__ void __launch_bounds__(256) ge_search_kernel(int m, int n, int half, const double2* __restrict__ g, Cand* part) {
    __shared__ Cand red[8];
    const int hn = n / 2;
    const long long total = static_cast<long long>(m / 2 + 1) * hn;
    Cand best{0.0, -1};
    for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < total;
         c += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(c / hn), kk = static_cast<int>(c - static_cast<long long>(t) * hn);
        const int j = half ? t : (m / 2 + t) % m;
        const double2 a = g[static_cast<size_t>(j) * n + kk], b = g[static_cast<size_t>(j) * n + kk + hn];
        const double sp = hypot(a.x + b.x, a.y + b.y), sm = hypot(a.x - b.x, a.y - b.y);
        const double s1 = (sp < sm) ? sm : sp;  // std::max
        if (s1 > best.s) best = Cand{s1, c};    // a thread's candidates ascend: the first maximal stays
    }
    best = block_best(best, red);
    if (threadIdx.x == 0) part[blockIdx.x] = best;
}

// out[0] = sigma_1, out[1] = candidate index (as double, -1: none), out[2..5] = a, b
__global__ void __launch_bounds__(256) ge_search_final_kernel(int m, int n, int half, const double2* __restrict__ g,
                                                              const Cand* part, int nparts, double* out) {
    __shared__ Cand red[8];
    Cand best{0.0, -1};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) best = better(best, part[i]);
    best = block_best(best, red);
    if (threadIdx.x == 0) {
        out[0] = best.s;
        out[1] = static_cast<double>(best.c);
        double2 a = make_double2(0.0, 0.0), b = a;
        if (best.c >= 0) {
            const int hn = n / 2;
            const int t = static_cast<int>(best.c / hn), kk = static_cast<int>(best.c - static_cast<long long>(t) * hn);
            const int j = half ? t : (m / 2 + t) % m;
            a = g[static_cast<size_t>(j) * n + kk];
            b = g[static_cast<size_t>(j) * n + kk + hn];
        }
        out[2] = a.x;
        out[3] = a.y;
        out[4] = b.x;
        out[5] = b.y;
    }
}

// The pivot cross of the PRE-update residual: dce[j] = de (g[j][km] + g[j][ks]),
// dco[j] = dodd (g[j][km] - g[j][ks]), re[k] = g[js][k] + g[jm][k], ro[k] = g[js][k] - g[jm][k]
// over the `rows` stored rows.  Half grid (lowrank.cpp:362-380): the row of
// -theta* is the pivot row itself shifted by pi in lambda (glide symmetry),
// re[k] = e[bi][k] + e[bi][(k + n/2) mod n].
__global__ void __launch_bounds__(256) ge_cross_kernel(int rows, int n, int half, const double2* __restrict__ g, int js, int jm,
                                                       int ks, double2 de, double2 dodd, double2* dce, double2* dco,
                                                       double2* re, double2* ro) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int km = (ks + n / 2) % n;
    if (i < rows) {
        const double2 cm = g[static_cast<size_t>(i) * n + km], cp = g[static_cast<size_t>(i) * n + ks];
        dce[i] = cmul_ref(de, make_double2(cm.x + cp.x, cm.y + cp.y));
        dco[i] = cmul_ref(dodd, make_double2(cm.x - cp.x, cm.y - cp.y));
    }
    if (i < n) {
        const double2 rp = g[static_cast<size_t>(js) * n + i];
        const double2 rm = half ? g[static_cast<size_t>(js) * n + (i + n / 2) % n] : g[static_cast<size_t>(jm) * n + i];
        re[i] = make_double2(rp.x + rm.x, rp.y + rm.y);
        ro[i] = make_double2(rp.x - rm.x, rp.y - rm.y);
    }
}

// out = g - upd over the whole grid; mx (may be null) receives max |out|.
// One grid row per blockIdx.y trip (its column factors loaded once), four
// independent entries per thread and trip.
__global__ void __launch_bounds__(256) ge_update_kernel(int m, int n, const double2* g,  // g may be out (in place)
                                                        const double2* __restrict__ dce, const double2* __restrict__ dco,
                                                        const double2* __restrict__ re, const double2* __restrict__ ro,
                                                        int has_e, int has_o, double2* out, double* mx) {
    __shared__ double red[64];
    double lm = 0.0;
    constexpr int kU = 4;
    for (int j = blockIdx.y; j < m; j += gridDim.y) {
        const double2 ce = dce[j], co = dco[j];
        const double2* gr = g + static_cast<size_t>(j) * n;
        double2* orow = out + static_cast<size_t>(j) * n;
        for (int k0 = blockIdx.x * blockDim.x * kU + threadIdx.x; k0 < n; k0 += gridDim.x * blockDim.x * kU) {
            double2 v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int k = k0 + u * blockDim.x;
                v[u] = k < n ? gr[k] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int k = k0 + u * blockDim.x;
                if (k < n) {
                    double2 upd = make_double2(0.0, 0.0);
                    if (has_e) {
                        const double2 t = cmul_ref(ce, re[k]);
                        upd = make_double2(upd.x + t.x, upd.y + t.y);
                    }
                    if (has_o) {
                        const double2 t = cmul_ref(co, ro[k]);
                        upd = make_double2(upd.x + t.x, upd.y + t.y);
                    }
                    const double2 r = make_double2(v[u].x - upd.x, v[u].y - upd.y);
                    orow[k] = r;
                    if (mx) lm = fmax(lm, hypot(r.x, r.y));
                }
            }
        }
    }
    if (mx) {
        lm = block_max(lm, red);
        if (threadIdx.x == 0) atomic_max_nonneg(mx, lm);
    }
}

__global__ void __launch_bounds__(256) ge_maxabs_kernel(long long total, const double2* __restrict__ g, double* mx) {
    __shared__ double red[64];
    double lm = 0.0;
    for (long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double2 v = g[idx];
        lm = fmax(lm, hypot(v.x, v.y));
    }
    lm = block_max(lm, red);
    if (threadIdx.x == 0) atomic_max_nonneg(mx, lm);
}

// scratch layout (bytes): [0, 64): search result (6 doubles) + max slot; parts: kGeParts Cand; cross: 2 m + 2 n complex
size_t ge_scratch_bytes(int m, int n) {
    return 128 + sizeof(Cand) * kGeParts + sizeof(double2) * (2 * static_cast<size_t>(m) + 2 * static_cast<size_t>(n));
}

static int ge_blocks(long long work) {
    long long b = (work + 255) / 256;
    if (b > kGeParts) b = kGeParts;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

cudaError_t launch_ge_search(int m, int n, bool half, const double2* g, void* scratch, cudaStream_t st) {
    double* res = static_cast<double*>(scratch);
    Cand* part = reinterpret_cast<Cand*>(static_cast<char*>(scratch) + 128);
    const int nb = ge_blocks(static_cast<long long>(m / 2 + 1) * (n / 2));
    ge_search_kernel<<<nb, 256, 0, st>>>(m, n, half ? 1 : 0, g, part);
    ge_search_final_kernel<<<1, 256, 0, st>>>(m, n, half ? 1 : 0, g, part, nb, res);
    return cudaGetLastError();
}

// (js, ks): the pivot node; full grid: js the doubled row of theta*; half grid: js = t
cudaError_t launch_ge_step(int m, int n, bool half, const double2* g, int js, int ks, double2 de, double2 dodd, int has_e,
                           int has_o, double2* out, void* scratch, bool want_max, cudaStream_t st) {
    double* mx = static_cast<double*>(scratch) + 8;
    double2* cross = reinterpret_cast<double2*>(static_cast<char*>(scratch) + 128 + sizeof(Cand) * kGeParts);
    double2 *dce = cross, *dco = cross + m, *re = cross + 2 * m, *ro = cross + 2 * m + n;
    const int rows = half ? m / 2 + 1 : m;
    const int jm = half ? js : (m - js) % m;
    const int mn = rows > n ? rows : n;
    ge_cross_kernel<<<(mn + 255) / 256, 256, 0, st>>>(rows, n, half ? 1 : 0, g, js, jm, ks, de, dodd, dce, dco, re, ro);
    if (want_max) cudaMemsetAsync(mx, 0, sizeof(double), st);
    const int bx = (n + 1023) / 1024;
    const int by = rows < 2048 ? rows : 2048;
    ge_update_kernel<<<dim3(bx, by), 256, 0, st>>>(rows, n, g, dce, dco, re, ro, has_e, has_o, out, want_max ? mx : nullptr);
    return cudaGetLastError();
}

cudaError_t launch_ge_maxabs(long long total, const double2* g, void* scratch, cudaStream_t st) {
    double* mx = static_cast<double*>(scratch) + 8;
    cudaMemsetAsync(mx, 0, sizeof(double), st);
    ge_maxabs_kernel<<<ge_blocks(total), 256, 0, st>>>(total, g, mx);
    return cudaGetLastError();
}

}  // namespace sk
