// Standalone coefficient <-> grid transforms of the reference's Fourier layer
// (fourier.hpp:107-108, sphere_domain.hpp:61), on complex data of any even
// size whose transform lengths factor into 2, 3, 5, 7 and fit one CTA:
//
//   analyze_2d(BMCGrid)      fourier.cpp:170-188  -> two xform_kernel<ANALYZE> passes
//   sample_grid(X, m, n)     fourier.cpp:190-209  -> two xform_kernel<SYNTH> passes
//                            (zero-pads or truncates as synthesize_1d, :55-66)
//   sample_dfs of samples    sphere_domain.cpp:19-26, :46-52 -> dfs_double_kernel
//
// One CTA per sequence: the row (contiguous in HBM) is loaded coalesced,
// transformed in shared memory by the same mixed-radix engine as the solve
// (fft_dev.cuh), and written TRANSPOSED, so the second pass again reads
// contiguous rows and both 1D directions run on coalesced loads; the 2D
// transform is separable, so doing the lambda direction first (the reference
// does theta first) changes only rounding.  Per pass each element is read once
// and written once: 32 bytes per complex entry, HBM-bound.
#include <cuda_runtime.h>

#include "fft_dev.cuh"
#include "params.h"
#include "sk_internal.h"
#include "tma.cuh"

namespace sk {

// ANALYZE (analyze_1d, fourier.cpp:39-53): c_k = (-1)^k / n * FFT(x)_{(k+n) mod n},
//   stored at k + n/2 (k = -n/2 .. n/2-1).
// SYNTH (synthesize_1d, fourier.cpp:55-66): g[(k+n_out) mod n_out] = (-1)^k c_k for
//   the modes both lengths hold, then the unnormalised backward transform.
// SWZ: XOR-swizzled slots (plans whose first span is even, e.g. power-of-two
// lengths, where the butterflies of a stage otherwise share one bank).
// HI: high-occupancy variant for short transforms (<= 256 threads, radices <= 8).
template <bool ANALYZE, bool SWZ, bool HI>
__global__ void __launch_bounds__(HI ? 256 : 512, HI ? 4 : 1)
    xform_kernel(XformParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int n = P.fd.L;  // transform length (n for ANALYZE, n_out for SYNTH)
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + P.aslots;  // whole 8-slot swizzle blocks (gather: whole boxes)
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int r = blockIdx.x;
    if (P.gather) {
        // Sequence r is COLUMN r of the row-major input (element j at
        // src[j ld_in + r]): the copy engine gathers it as boxes of 256
        // elements through the tensor map, and the result leaves as one
        // contiguous row dst[r ld_out ..].  The transposition sits on the load
        // side: gathered 16-byte loads run several times faster here than
        // per-thread 16-byte stores one row apart.
        uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((n + 3) & ~3));
        const int n_src = ANALYZE ? n : P.n_in;
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const int nbox = (n_src + kXformBox - 1) / kXformBox;
            mbar_expect_tx(bar, static_cast<uint32_t>(nbox) * kXformBox * 16);
            for (int b = 0; b < nbox; ++b) tma_load_3d(a + b * kXformBox, &tmap, 2 * r, b * kXformBox, 0, bar);
        }
        const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
        for (int i = tid; i < n; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
        __syncthreads();
        mbar_wait(bar, 0);
        double2* out = P.dst + static_cast<long long>(r) * P.ld_out;
        constexpr int kStage = HI ? kXformStageHi : kXformStage;
        double2 v[kStage];
        if constexpr (ANALYZE) {
            if constexpr (SWZ) {  // natural slots -> swizzled slots through registers
#pragma unroll
                for (int u = 0; u < kStage; ++u) {
                    const int j = tid + u * nthr;
                    if (j < n) v[u] = a[j];
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < kStage; ++u) {
                    const int j = tid + u * nthr;
                    if (j < n) a[swz<SWZ>(j)] = v[u];
                }
                __syncthreads();
            }
            fft_forward<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);  // X_t at a[swz(rev[t])]
            const double inv = 1.0 / n;
            for (int kp = tid; kp < n; kp += nthr) {
                const int k = kp - n / 2;
                const int t = k < 0 ? k + n : k;
                const double s = (k % 2 == 0) ? inv : -inv;
                const double2 x = a[swz<SWZ>(s_rev[t])];
                out[kp] = make_double2(s * x.x, s * x.y);
            }
        } else {
            const int lo = max(-P.n_in / 2, -n / 2), hi = min(P.n_in / 2, n / 2);
#pragma unroll
            for (int u = 0; u < kStage; ++u) {
                const int k = lo + tid + u * nthr;
                if (k < hi) v[u] = a[k + P.n_in / 2];
            }
            __syncthreads();
            for (int j = tid; j < n; j += nthr) a[swz<SWZ>(j)] = make_double2(0.0, 0.0);
            __syncthreads();
#pragma unroll
            for (int u = 0; u < kStage; ++u) {
                const int k = lo + tid + u * nthr;
                if (k < hi) {
                    const int t = k < 0 ? k + n : k;
                    a[swz<SWZ>(s_rev[t])] = (k % 2 == 0) ? v[u] : make_double2(-v[u].x, -v[u].y);  // DIT input: digit-reversed
                }
            }
            __syncthreads();
            fft_inverse<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);  // natural order
            for (int j = tid; j < n; j += nthr) out[j] = a[swz<SWZ>(j)];
        }
        return;
    }
    const double2* src = P.src + static_cast<long long>(r) * P.ld_in;
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    for (int i = tid; i < n; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
    if constexpr (ANALYZE) {
        for (int j = tid; j < n; j += nthr) a[swz<SWZ>(j)] = src[j];
        __syncthreads();
        fft_forward<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);  // X_t at a[swz(rev[t])]
        const double inv = 1.0 / n;
        for (int kp = tid; kp < n; kp += nthr) {
            const int k = kp - n / 2;
            const int t = k < 0 ? k + n : k;
            const double s = (k % 2 == 0) ? inv : -inv;
            const double2 v = a[swz<SWZ>(s_rev[t])];
            P.dst[static_cast<long long>(kp) * P.ld_out + r] = make_double2(s * v.x, s * v.y);
        }
    } else {
        for (int j = tid; j < n; j += nthr) a[swz<SWZ>(j)] = make_double2(0.0, 0.0);
        __syncthreads();
        const int lo = max(-P.n_in / 2, -n / 2), hi = min(P.n_in / 2, n / 2);
        for (int k = lo + tid; k < hi; k += nthr) {
            const double2 c = src[k + P.n_in / 2];
            const int t = k < 0 ? k + n : k;
            a[swz<SWZ>(s_rev[t])] = (k % 2 == 0) ? c : make_double2(-c.x, -c.y);  // DIT input: digit-reversed
        }
        __syncthreads();
        fft_inverse<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);  // natural order
        for (int j = tid; j < n; j += nthr) P.dst[static_cast<long long>(j) * P.ld_out + r] = a[swz<SWZ>(j)];
    }
}

// Bluestein (chirp-z) transforms for lengths n with a prime factor > 7 (the
// reference accepts any even length through FFTW, fourier.cpp:22-35;
// acceptance c11 round-trips n = 602 = 2 * 7 * 43):
//   X_k = sum_j x_j e^{-2 pi i jk/n} = w_k (a * b)_k,  a_j = x_j w_j,
//   b_m = conj(w_m),  w_m = exp(-i pi m^2 / n)
// (the backward transform of SYNTH uses the conjugate chirps), with the
// cyclic convolution of length Lb >= 2n - 1 done by the same in-shared-memory
// engine: forward DIF, slot-wise product with bhat = FFT(b)/Lb (precomputed
// in the engine's output slot order by xform_blue_prep_kernel), inverse DIT.
// One CTA per sequence; loads and transposed stores as xform_kernel.
template <bool ANALYZE, bool SWZ>
__global__ void __launch_bounds__(512, 1) xform_blue_kernel(XformParams P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int Lb = P.fd.L, n = P.nb;
    const int Lp = (Lb + 7) & ~7;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lp;
    double2* s_lo = s_hi + P.fd.nhi;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int r = blockIdx.x;
    const double2* src = P.src + static_cast<long long>(r) * P.ld_in;
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    if constexpr (ANALYZE) {
        for (int j = tid; j < Lp; j += nthr) {
            double2 v = make_double2(0.0, 0.0);
            if (j < n) v = cmul(src[j], __ldg(P.chirp + j));
            if (j < Lb) a[swz<SWZ>(j)] = v;
        }
    } else {
        // synthesize_1d placement g[(k + n) mod n] = (-1)^k c_k, then * conj(w)
        const int lo = max(-P.n_in / 2, -n / 2), hi = min(P.n_in / 2, n / 2);
        for (int j = tid; j < Lb; j += nthr) a[swz<SWZ>(j)] = make_double2(0.0, 0.0);
        __syncthreads();
        for (int k = lo + tid; k < hi; k += nthr) {
            const double2 c = src[k + P.n_in / 2];
            const int t = k < 0 ? k + n : k;
            const double2 g = (k % 2 == 0) ? c : make_double2(-c.x, -c.y);
            a[swz<SWZ>(t)] = cmulc(g, __ldg(P.chirp + t));
        }
    }
    __syncthreads();
    fft_forward<SWZ, 25>(a, P.fd, T, tid, nthr);
    for (int i = tid; i < Lp; i += nthr) a[i] = cmul(a[i], __ldg(P.bhat + i));
    __syncthreads();
    fft_inverse<SWZ, 25>(a, P.fd, T, tid, nthr);
    if constexpr (ANALYZE) {
        const double inv = 1.0 / n;
        for (int kp = tid; kp < n; kp += nthr) {
            const int k = kp - n / 2;
            const int t = k < 0 ? k + n : k;
            const double s = (k % 2 == 0) ? inv : -inv;
            const double2 v = cmul(a[swz<SWZ>(t)], __ldg(P.chirp + t));
            P.dst[static_cast<long long>(kp) * P.ld_out + r] = make_double2(s * v.x, s * v.y);
        }
    } else {
        for (int j = tid; j < n; j += nthr)
            P.dst[static_cast<long long>(j) * P.ld_out + r] = cmulc(a[swz<SWZ>(j)], __ldg(P.chirp + j));
    }
}

// bhat = FFT_Lb(b) / Lb in physical slot order: b_m = conj(w_m) (ANALYZE) or
// w_m (SYNTH) for m in (-n, n), wrapped cyclically.
template <bool SWZ>
__global__ void __launch_bounds__(512, 1) xform_blue_prep_kernel(FftDesc fd, int n, const double2* chirp, int analyze,
                                                                 double2* bhat) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int Lb = fd.L;
    const int Lp = (Lb + 7) & ~7;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lp;
    double2* s_lo = s_hi + fd.nhi;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const Tw T = load_tw(fd, s_hi, s_lo, tid, nthr);
    for (int j = tid; j < Lb; j += nthr) {
        const int m = j < n ? j : (j > Lb - n ? Lb - j : -1);
        double2 v = make_double2(0.0, 0.0);
        if (m >= 0) {
            const double2 w = chirp[m];
            v = analyze ? make_double2(w.x, -w.y) : w;
        }
        a[swz<SWZ>(j)] = v;
    }
    __syncthreads();
    fft_forward<SWZ, 25>(a, fd, T, tid, nthr);
    const double inv = 1.0 / Lb;
    for (int i = tid; i < Lp; i += nthr) bhat[i] = (i < Lb || SWZ) ? cscale(a[i], inv) : make_double2(0.0, 0.0);
}

cudaError_t launch_blue_prep(const FftDesc& fd, int nb, const double2* chirp, bool analyze, int nthr, size_t smem,
                             int swizzle, double2* bhat, cudaStream_t st) {
    if (swizzle) {
        cudaFuncSetAttribute(xform_blue_prep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        xform_blue_prep_kernel<true><<<1, nthr, smem, st>>>(fd, nb, chirp, analyze ? 1 : 0, bhat);
    } else {
        cudaFuncSetAttribute(xform_blue_prep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        xform_blue_prep_kernel<false><<<1, nthr, smem, st>>>(fd, nb, chirp, analyze ? 1 : 0, bhat);
    }
    return cudaGetLastError();
}

template <bool ANALYZE, bool SWZ>
static cudaError_t launch_blue_t(const XformParams& P, int nrows, int nthr, size_t smem, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(xform_blue_kernel<ANALYZE, SWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    xform_blue_kernel<ANALYZE, SWZ><<<nrows, nthr, smem, st>>>(P);
    return cudaGetLastError();
}

// doubled[j][k] = phys[j - m/2][k] (j >= m/2), phys[m/2 - j][(k + n/2) mod n]
// (j < m/2): the glide reflection f(lambda -+ pi, -theta) of dfs_extend as an
// index map on the physical rows theta_p = 2 pi p / m, p = 0..m/2.
// pole_glide: row j = m/2 glides too (theta_{m/2} rounds below zero in the
// reference for some m; sk_internal.h GridGeom::pole_glide).
__global__ void dfs_double_kernel(int m, int n, const double* phys, double2* grid, int pole_glide) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(m) * n) return;
    const int j = static_cast<int>(idx / n), k = static_cast<int>(idx - static_cast<long long>(j) * n);
    const bool glide = j < m / 2 || (pole_glide && j == m / 2);
    const double v = glide ? phys[static_cast<long long>(m / 2 - j) * n + (k + n / 2) % n]
                           : phys[static_cast<long long>(j - m / 2) * n + k];
    grid[idx] = make_double2(v, 0.0);
}

// n_src > 0: gather mode, the data slots hold whole boxes of the n_src-element input column
int xform_slots(int n, int n_src) {
    const int s = (n + 7) & ~7;
    return n_src > 0 ? max(s, (n_src + kXformBox - 1) / kXformBox * kXformBox) : s;
}
size_t xform_smem_bytes(int n, int nhi, int nlo, int n_src) {
    return static_cast<size_t>(xform_slots(n, n_src)) * 16 + static_cast<size_t>(nhi + nlo) * 16 +
           static_cast<size_t>((n + 3) & ~3) * 4 + 16;
}

template <bool ANALYZE, bool SWZ, bool HI>
static cudaError_t launch_xform_t(const XformParams& P, const CUtensorMap& map, int nrows, int nthr, size_t smem,
                                  cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(xform_kernel<ANALYZE, SWZ, HI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    xform_kernel<ANALYZE, SWZ, HI><<<nrows, nthr, smem, st>>>(P, map);
    return cudaGetLastError();
}

// map: the input as a column-gather tensor map (make_spec_map), read when P.gather
cudaError_t launch_xform(const XformParams& P, const CUtensorMap& map, bool analyze, int nrows, int nthr, size_t smem,
                         cudaStream_t st) {
    if (nrows <= 0) return cudaSuccess;
    if (P.nb) {
        if (analyze) return P.swizzle ? launch_blue_t<true, true>(P, nrows, nthr, smem, st)
                                      : launch_blue_t<true, false>(P, nrows, nthr, smem, st);
        return P.swizzle ? launch_blue_t<false, true>(P, nrows, nthr, smem, st)
                         : launch_blue_t<false, false>(P, nrows, nthr, smem, st);
    }
    const bool hi = P.hiocc && nthr <= 256;
    if (analyze) {
        if (hi) return P.swizzle ? launch_xform_t<true, true, true>(P, map, nrows, nthr, smem, st)
                                 : launch_xform_t<true, false, true>(P, map, nrows, nthr, smem, st);
        return P.swizzle ? launch_xform_t<true, true, false>(P, map, nrows, nthr, smem, st)
                         : launch_xform_t<true, false, false>(P, map, nrows, nthr, smem, st);
    }
    if (hi) return P.swizzle ? launch_xform_t<false, true, true>(P, map, nrows, nthr, smem, st)
                             : launch_xform_t<false, false, true>(P, map, nrows, nthr, smem, st);
    return P.swizzle ? launch_xform_t<false, true, false>(P, map, nrows, nthr, smem, st)
                     : launch_xform_t<false, false, false>(P, map, nrows, nthr, smem, st);
}

cudaError_t launch_dfs_double(int m, int n, const double* phys, double2* grid, cudaStream_t st) {
    const long long tot = static_cast<long long>(m) * n;
    if (tot > 0)
        dfs_double_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(m, n, phys, grid, pole_glide(m));
    return cudaGetLastError();
}

}  // namespace sk
