// Grid-path kernels of the DFS spectral Poisson solve (sm_100a).
//
//   K1 lambda_fwd  — DFS doubling + forward lambda transform of each physical
//                    row (replaces sample_dfs sphere_domain.cpp:46-52 and the
//                    row stage of analyze_2d fourier.cpp:181-186);
//   K3 theta_stage — per lambda mode: theta transform (column stage of
//                    analyze_2d :174-180), Msin^2 (poisson.cpp:61-71), the
//                    banded solve with the k=0 constraint (solve :121-161,
//                    band_solve banded.cpp:101-158, band_solve_with_dense_row
//                    :160-328), inverse theta transform (sample_grid :194-200);
//   K4 lambda_inv  — inverse lambda transform per physical row (sample_grid
//                    :202-207);
//   K7 shgen       — seeded spherical-harmonic input generator (untimed).
//
// Data in HBM between the kernels is the half spectrum S[k][p], k = 0..N/2
// (real data: the k < 0 half is its Hermitian mirror), p = 0..M/2 (physical
// rows only: the doubled rows j < M/2 are (-1)^k times row M/2-j in lambda-
// spectral space, so the doubled grid is never stored).
#include <cstdlib>
#include <cooperative_groups.h>
#include <type_traits>
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "fft_dev.cuh"
#include "theta_common.cuh"
#include "tma.cuh"
#include "params.h"
#include "sk_internal.h"

namespace cg = cooperative_groups;

namespace sk {

#ifdef SK_PHASES
__device__ unsigned long long g_phase[4096][24];
#define SK_PROBE(i)                                                         \
    do {                                                                    \
        __syncthreads();                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_phase[blockIdx.x][i] = clock64(); \
    } while (0)
// phase probes of the lambda kernels (their own table: they run before / after the theta stage)
__device__ unsigned long long g_phase_l[2][4096][8];
#define SK_PROBE_LAM(w, i)                                                         \
    do {                                                                           \
        __syncthreads();                                                           \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_phase_l[w][blockIdx.x][i] = clock64(); \
    } while (0)
#else
#define SK_PROBE(i) \
    do {            \
    } while (0)
#define SK_PROBE_LAM(w, i) \
    do {                   \
    } while (0)
#endif

// Box of the spectrum tensor map: 256 lambda modes x one physical row
// (2 doubles), i.e. the strided [k][p] column slice of one row.
constexpr int kBoxModes = 256;
constexpr int kLamPairs = 12;   // mode pairs per thread held in registers
constexpr int kLamPairsHi = 6;  // same, high-occupancy lambda variant

// One CTA per physical row: TMA bulk load of the real row (N/2 complex
// pairs), forward DIF FFT, split into the N/2+1 modes of the real transform
// with analyze_1d's (-1)^k / N (fourier.cpp:44-51), stored mode-major.
// SWZ (power-of-two rows, C2/C4): XOR-swizzled slots, filled by per-thread
// loads instead of the bulk copy (the bulk copy lands elements in order).
// HI: high-occupancy variant for short rows (<= 128 threads per CTA, radices
// <= 8): 64 registers per thread, twice the CTAs per SM.
template <bool SWZ, bool HI>
__global__ void __launch_bounds__(256, HI ? 4 : 2) lambda_fwd_kernel(LambdaParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = P.fd.L;
    const int Lpad = (L / kBoxModes + 1) * kBoxModes;  // >= L+1, whole boxes
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int row = blockIdx.x % P.rows_local;
    const int rhs = blockIdx.x / P.rows_local;
    const double2* src =
        reinterpret_cast<const double2*>(P.f + rhs * P.in_rhs_stride + static_cast<long long>(row) * P.g.N);
    if constexpr (!SWZ) {
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(bar, static_cast<uint32_t>(L) * 16);
            bulk_g2s_chunked(a, src, static_cast<uint32_t>(L) * 16, bar);  // the real row as N/2 complex pairs
        }
    } else {
#pragma unroll 4
        for (int i = tid; i < L; i += nthr) a[swz<true>(i)] = __ldg(src + i);
    }
    // twiddles and the digit-reversal table by the threads while the row is in
    // flight (measured faster here than adding them to the bulk copies)
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    for (int i = tid; i < L; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
    __syncthreads();
    if constexpr (!SWZ) mbar_wait(bar, 0);
    fft_forward<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);
    const double invN = 1.0 / P.g.N;
    double2* out = P.spec + rhs * P.out_rhs_stride;
    (void)tmap;  // scattered fire-and-forget stores measured faster than staged TMA tensor stores here
    for (int k = tid; k <= L / 2; k += nthr) {
        const int km = L - k;  // partner mode
        const double2 z = a[swz<SWZ>(s_rev[k])];
        const double2 zp = a[swz<SWZ>(s_rev[km == L ? 0 : km])];
        // A = (Z_k + conj Z_{L-k}) / 2,  B = -i (Z_k - conj Z_{L-k}) / 2
        const double2 A = make_double2(0.5 * (z.x + zp.x), 0.5 * (z.y - zp.y));
        const double2 B = make_double2(0.5 * (z.y + zp.y), -0.5 * (z.x - zp.x));
        // T(L - k) = -conj T(k) (2L-th roots): X_{L-k} = conj(A) + T(L-k) conj(B) = conj(A - T(k) B)
        const double2 Pk = cmul(T(k), B);
        const double2 Xk = cadd(A, Pk);
        const double2 Xm = conjd(csub(A, Pk));
        const double2 vk = cscale(Xk, (k & 1) ? -invN : invN);
        const double2 vm = cscale(Xm, (km & 1) ? -invN : invN);
        if (P.peers.n) {  // fused transpose: store into the theta rank's receive buffer over NVLink
            *peer_ptr(P.peers, k, k, row) = vk;
            if (km != k) *peer_ptr(P.peers, km, km, row) = vm;
        } else if (P.pair & 8) {
            // row-major spectrum R[rhs][p][k]: the row's modes are contiguous, adjacent lanes write
            // adjacent modes (k ascending, L - k descending); the theta stage gathers its columns
            double2* rr = P.spec + (static_cast<size_t>(rhs) * P.rows_local + row) * (L + 1);
            rr[k] = vk;
            if (km != k) rr[km] = vm;
        } else {
            out[static_cast<size_t>(k) * P.rows_local + row] = vk;
            if (km != k) out[static_cast<size_t>(km) * P.rows_local + row] = vm;
        }
    }
}

// Row pairs (p, p+1) on a 2-CTA cluster (single RHS, unswizzled rows, no
// peer stores; C3): each CTA transforms its row as above and leaves the N/2+1
// modes in natural order in its shared memory; CTA c then stores the modes of
// its half of k for both rows, adjacent lanes writing the (p, p+1) neighbours
// of one mode, so a warp's store covers 16 modes x 32 contiguous bytes where
// the per-row stores covered 32 modes x 16 bytes.  The peer row is read
// through DSMEM in natural order (contiguous).  Grid = rows rounded up to even;
// the padding CTA only takes part in the cluster barriers.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) lambda_fwd_pair_kernel(LambdaParams P, int relaxed_exit) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L = P.fd.L;
    const int Lpad = (L / kBoxModes + 1) * kBoxModes;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = static_cast<int>(cluster.block_rank());
    const int row = blockIdx.x;
    const bool live = row < P.rows_local;  // CTA-uniform
    SK_PROBE_LAM(0, 0);
    if (live && tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bar, static_cast<uint32_t>(L) * 16);
        bulk_g2s_chunked(a, reinterpret_cast<const double2*>(P.f + static_cast<long long>(row) * P.g.N),
                         static_cast<uint32_t>(L) * 16, bar);
    }
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    for (int i = tid; i < L; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
    __syncthreads();
    if (live) {
        mbar_wait(bar, 0);
        SK_PROBE_LAM(0, 1);
        fft_forward<false, 25>(a, P.fd, T, tid, nthr);
        SK_PROBE_LAM(0, 2);
        const double invN = 1.0 / P.g.N;
        double2 vk[kLamPairs], vm[kLamPairs];
#pragma unroll
        for (int u = 0; u < kLamPairs; ++u) {
            const int k = tid + u * nthr;
            if (k <= L / 2) {
                const int km = L - k;
                const double2 z = a[s_rev[k]];
                const double2 zp = a[s_rev[km == L ? 0 : km]];
                const double2 A = make_double2(0.5 * (z.x + zp.x), 0.5 * (z.y - zp.y));
                const double2 B = make_double2(0.5 * (z.y + zp.y), -0.5 * (z.x - zp.x));
                const double2 Pk = cmul(T(k), B);  // T(L - k) = -conj T(k): X_{L-k} = conj(A - T(k) B)
                vk[u] = cscale(cadd(A, Pk), (k & 1) ? -invN : invN);
                vm[u] = cscale(conjd(csub(A, Pk)), (km & 1) ? -invN : invN);
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kLamPairs; ++u) {
            const int k = tid + u * nthr;
            if (k <= L / 2) {
                a[k] = vk[u];
                if (L - k != k) a[L - k] = vm[u];
            }
        }
    }
    SK_PROBE_LAM(0, 3);
    cluster.sync();
    SK_PROBE_LAM(0, 4);
    const double2* other = cluster.map_shared_rank(a, c ^ 1);
    const int r0 = row & ~1;
    const int nk = L + 1;
    const int k_lo = c == 0 ? 0 : nk / 2;
    const int k_hi = c == 0 ? nk / 2 : nk;
    const int sub_hi = min(2, P.rows_local - r0);  // 1 when the padding CTA is the partner
    // four (mode, row) entries per thread and trip, their (half remote) loads
    // issued together through one generic pointer: the DSMEM latency is paid
    // once per four stores
    constexpr int kU = 4;
    const int tot = 2 * (k_hi - k_lo);
    for (int i0 = tid; i0 < tot; i0 += kU * nthr) {
        double2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = min(i0 + u * nthr, tot - 1);
            const double2* src = ((i & 1) == c) ? a : other;
            v[u] = src[k_lo + (i >> 1)];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = i0 + u * nthr;
            const int k = k_lo + (i >> 1), sub = i & 1;
            if (i < tot && sub < sub_hi) P.spec[static_cast<size_t>(k) * P.rows_local + r0 + sub] = v[u];
        }
    }
    SK_PROBE_LAM(0, 5);
    cluster_exit_barrier(relaxed_exit);
    SK_PROBE_LAM(0, 6);
}

// Row groups of G = 4 (p .. p+3) on a 4-CTA cluster (single RHS, unswizzled
// rows; C3), the generalisation of lambda_fwd_pair_kernel: each CTA
// transforms its row and leaves the N/2+1 modes in natural order in shared
// memory; CTA c then stores the modes of its quarter of k for all four rows,
// four adjacent lanes writing (p .. p+3) of one mode: a warp's store covers 8
// modes x 64 contiguous bytes (two full 32-byte sectors each) where the pair
// kernel covered 16 x 32 and the one-row kernel 32 x 16.  The peers' rows are
// read through DSMEM in natural order (eight consecutive modes per CTA per
// warp access).  With peer stores (fused multi-GPU transpose) the same 64-byte
// runs go to the owner of mode k over NVLink.  Grid = rows rounded up to a
// multiple of 4; padding CTAs only take part in the cluster barriers.
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 2) lambda_fwd_quad_kernel(LambdaParams P, int relaxed_exit) {
    constexpr int G = 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L = P.fd.L;
    const int Lpad = (L / kBoxModes + 1) * kBoxModes;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = static_cast<int>(cluster.block_rank());
    const int row = blockIdx.x;
    const bool live = row < P.rows_local;  // CTA-uniform
    if (live && tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bar, static_cast<uint32_t>(L) * 16);
        bulk_g2s_chunked(a, reinterpret_cast<const double2*>(P.f + static_cast<long long>(row) * P.g.N),
                         static_cast<uint32_t>(L) * 16, bar);
    }
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    for (int i = tid; i < L; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
    __syncthreads();
    if (live) {
        mbar_wait(bar, 0);
        fft_forward<false, 25>(a, P.fd, T, tid, nthr);
        const double invN = 1.0 / P.g.N;
        double2 vk[kLamPairs], vm[kLamPairs];
#pragma unroll
        for (int u = 0; u < kLamPairs; ++u) {
            const int k = tid + u * nthr;
            if (k <= L / 2) {
                const int km = L - k;
                const double2 z = a[s_rev[k]];
                const double2 zp = a[s_rev[km == L ? 0 : km]];
                const double2 A = make_double2(0.5 * (z.x + zp.x), 0.5 * (z.y - zp.y));
                const double2 B = make_double2(0.5 * (z.y + zp.y), -0.5 * (z.x - zp.x));
                const double2 Pk = cmul(T(k), B);  // T(L - k) = -conj T(k): X_{L-k} = conj(A - T(k) B)
                vk[u] = cscale(cadd(A, Pk), (k & 1) ? -invN : invN);
                vm[u] = cscale(conjd(csub(A, Pk)), (km & 1) ? -invN : invN);
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kLamPairs; ++u) {
            const int k = tid + u * nthr;
            if (k <= L / 2) {
                a[k] = vk[u];
                if (L - k != k) a[L - k] = vm[u];
            }
        }
    }
    cluster.sync();
    const double2* src[G];
#pragma unroll
    for (int g = 0; g < G; ++g) src[g] = cluster.map_shared_rank(a, g);
    const int r0 = row - c;  // first row of the group
    const int nk = L + 1;
    const int k_lo = (c * nk) / G, k_hi = ((c + 1) * nk) / G;
    const int sub_hi = min(G, P.rows_local - r0);  // rows of the group that exist
    for (int i = tid; i < G * (k_hi - k_lo); i += nthr) {
        const int k = k_lo + (i >> 2), sub = i & 3;
        if (sub < sub_hi) {
            const double2 v = src[sub][k];
            if (P.peers.n) *peer_ptr(P.peers, k, k, r0 + sub) = v;  // fused transpose over NVLink
            else P.spec[static_cast<size_t>(k) * P.rows_local + r0 + sub] = v;
        }
    }
    cluster_exit_barrier(relaxed_exit);  // only consumed DSMEM loads since the last cluster barrier
}

// Inverse: TMA tensor loads gather the row's N/2+1 modes from the mode-major
// spectrum; sample_grid's (-1)^k (fourier.cpp:61-62) and the packing into
// N/2 complex go through registers into digit-reversed order; inverse DIT
// FFT; the real row is stored (unnormalised, as FFTW_BACKWARD).
template <bool SWZ, bool HI>
__global__ void __launch_bounds__(256, HI ? 4 : 2) lambda_inv_kernel(LambdaParams P, const __grid_constant__ CUtensorMap tmap) {
    constexpr int kPairs = HI ? kLamPairsHi : kLamPairs;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = P.fd.L;
    const int Lpad = (L / kBoxModes + 1) * kBoxModes;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int row = blockIdx.x % P.rows_local;
    const int rhs = blockIdx.x / P.rows_local;
    SK_PROBE_LAM(1, 0);
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int nbox = L / kBoxModes + 1;
        const uint32_t rb = static_cast<uint32_t>((L + 3) & ~3) * 4;  // rev table, padded to 16 bytes
        mbar_expect_tx(bar, static_cast<uint32_t>(nbox) * kBoxModes * 16 + (P.fd.nhi + P.fd.nlo) * 16 + rb);
        for (int k0 = 0; k0 <= L; k0 += kBoxModes) tma_load_3d(a + k0, &tmap, 2 * row, k0, rhs, bar);
        bulk_g2s_chunked(s_hi, P.fd.hi, P.fd.nhi * 16, bar);
        bulk_g2s_chunked(s_lo, P.fd.lo, P.fd.nlo * 16, bar);
        bulk_g2s_chunked(s_rev, P.fd.rev, rb, bar);
    }
    const Tw T{s_hi, s_lo, P.fd.shift, (1 << P.fd.shift) - 1};
    __syncthreads();
    mbar_wait(bar, 0);
    SK_PROBE_LAM(1, 1);
    double2 zk[kPairs], zm[kPairs];
#pragma unroll
    for (int u = 0; u < kPairs; ++u) {
        const int k = tid + u * nthr;
        if (k <= L / 2) {
            const int km = L - k;
            double2 v = a[k];
            double2 w = a[km];
            if (k & 1) v = make_double2(-v.x, -v.y);
            if (km & 1) w = make_double2(-w.x, -w.y);
            if (k == 0) {  // DC and Nyquist of a real signal are real
                v.y = 0.0;
                w.y = 0.0;
            }
            // Z_k = E_k + i O_k, E_k = V_k + conj V_{L-k}, O_k = (V_k - conj V_{L-k}) conj(T(k))
            {
                // conj T(L - k) = -T(k): E_{L-k} = conj E_k, O_{L-k} = conj O_k, one twiddle product for both
                const double2 E = make_double2(v.x + w.x, v.y - w.y);
                const double2 O = cmulc(make_double2(v.x - w.x, v.y + w.y), T(k));
                zk[u] = make_double2(E.x - O.y, E.y + O.x);
                zm[u] = make_double2(E.x + O.y, O.x - E.y);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPairs; ++u) {
        const int k = tid + u * nthr;
        if (k <= L / 2) {
            const int km = L - k;
            a[swz<SWZ>(s_rev[k])] = zk[u];
            if (k != 0 && km != k) a[swz<SWZ>(s_rev[km])] = zm[u];
        }
    }
    __syncthreads();
    SK_PROBE_LAM(1, 2);
    fft_inverse<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);
    SK_PROBE_LAM(1, 3);
    double2* dst = reinterpret_cast<double2*>(P.u + rhs * P.out_rhs_stride + static_cast<long long>(row) * P.g.N);
    for (int j = tid; j < L; j += nthr) dst[j] = a[swz<SWZ>(j)];
    SK_PROBE_LAM(1, 4);
}

// Inverse on row pairs (p, p+1), the mirror image of lambda_fwd_pair_kernel
// (single RHS, unswizzled rows; C3): a 2-row x 256-mode box of the spectrum
// map gathers 32-byte (p, p+1) segments, CTA c loading the boxes of its half
// of the modes for both rows into its own row buffer ([mode][row] order; the
// box count nb is even, so half the boxes fill exactly the buffer). After a
// cluster barrier each CTA reads its row's modes from both buffers (the peer
// through DSMEM) into registers; a second barrier frees the buffers for the
// digit-reversed C2R pack, then the inverse FFT runs as in lambda_inv_kernel.
// The padding CTA of an odd row count loads its boxes (row p+1 is zero-filled
// out of bounds) but transforms and stores nothing.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2)
    lambda_inv_pair_kernel(LambdaParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L = P.fd.L;
    const int nb = L / kBoxModes + 1;  // even (lambda_inv_pair_ok)
    const int Lpad = nb * kBoxModes;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = static_cast<int>(cluster.block_rank());
    const int row = blockIdx.x;
    const bool live = row < P.rows_local;  // CTA-uniform
    const int r0 = row & ~1;
    const int kspl = (nb / 2) * kBoxModes;  // modes [0, kspl) in CTA 0, the rest in CTA 1
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t rb = static_cast<uint32_t>((L + 3) & ~3) * 4;
        mbar_expect_tx(bar, static_cast<uint32_t>(nb / 2) * kBoxModes * 32 + (P.fd.nhi + P.fd.nlo) * 16 + rb);
        for (int b = 0; b < nb / 2; ++b)
            tma_load_3d(a + b * 2 * kBoxModes, &tmap, 2 * r0, c * kspl + b * kBoxModes, 0, bar);
        bulk_g2s_chunked(s_hi, P.fd.hi, P.fd.nhi * 16, bar);
        bulk_g2s_chunked(s_lo, P.fd.lo, P.fd.nlo * 16, bar);
        bulk_g2s_chunked(s_rev, P.fd.rev, rb, bar);
    }
    const Tw T{s_hi, s_lo, P.fd.shift, (1 << P.fd.shift) - 1};
    __syncthreads();
    mbar_wait(bar, 0);
    cluster.sync();
    const double2* other = cluster.map_shared_rank(a, c ^ 1);
    const int sub = row & 1;
    auto mode = [&](int k) -> double2 {
        const int o = k >= kspl ? 1 : 0;
        return (o == c ? a : other)[(k - o * kspl) * 2 + sub];
    };
    double2 zk[kLamPairs], zm[kLamPairs];
    if (live) {
#pragma unroll
        for (int u = 0; u < kLamPairs; ++u) {
            const int k = tid + u * nthr;
            if (k <= L / 2) {
                const int km = L - k;
                double2 v = mode(k);
                double2 w = mode(km);
                if (k & 1) v = make_double2(-v.x, -v.y);
                if (km & 1) w = make_double2(-w.x, -w.y);
                if (k == 0) {
                    v.y = 0.0;
                    w.y = 0.0;
                }
                {
                    // conj T(L - k) = -T(k): E_{L-k} = conj E_k, O_{L-k} = conj O_k, one twiddle product for both
                    const double2 E = make_double2(v.x + w.x, v.y - w.y);
                    const double2 O = cmulc(make_double2(v.x - w.x, v.y + w.y), T(k));
                    zk[u] = make_double2(E.x - O.y, E.y + O.x);
                    zm[u] = make_double2(E.x + O.y, O.x - E.y);
                }
            }
        }
    }
    cluster.sync();  // the peer has finished reading this CTA's buffer
    if (!live) return;
#pragma unroll
    for (int u = 0; u < kLamPairs; ++u) {
        const int k = tid + u * nthr;
        if (k <= L / 2) {
            const int km = L - k;
            a[s_rev[k]] = zk[u];
            if (k != 0 && km != k) a[s_rev[km]] = zm[u];
        }
    }
    __syncthreads();
    fft_inverse<false, 25>(a, P.fd, T, tid, nthr);
    double2* dst = reinterpret_cast<double2*>(P.u + static_cast<long long>(row) * P.g.N);
    for (int j = tid; j < L; j += nthr) dst[j] = a[j];
}

// -------------------------------------------------------------- theta stage
// Pivot table: for every lambda mode k >= 0 and parity class, the reciprocal
// Thomas pivots 1/d'_i of both chains, indexed by the natural FFT index tau
// of the element: ipt[(k * 2 + par) * L + tau].  The pivots depend only on
// (M, k), so they are computed once per plan by the sequential recurrence
// d'_0 = b_0, d'_i = b_i - a_i c_{i-1} / d'_{i-1} — the same recurrence the
// reference's band_solve runs (banded.cpp:121-147, no row ever swaps for
// these systems) — which keeps the parallel sweeps below as accurate as the
// sequential algorithm.
// Row (kl, par) of the table (stride doubles) holds 1/d' of both chains of
// that parity at the natural index tau of each element.
__global__ void __launch_bounds__(128) pivot_table_kernel(int L, int k0, int ncols, double* ipt, int stride) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= ncols * 4) return;
    const int kl = id >> 2, par = (id >> 1) & 1, side = id & 1;
    const int kg = k0 + kl;
    const double k2 = static_cast<double>(kg) * static_cast<double>(kg);
    Chain cp, cm;
    make_chains(par, L, cp, cm);
    const Chain& ch = side == 0 ? cp : cm;
    double* out = ipt + (static_cast<size_t>(kl) * 2 + par) * stride;
    double ip = 0.0, cprev = 0.0;
    for (int i = 0; i < ch.n; ++i) {
        const int t = ch.t0 + ch.dt * i;
        const double A = chainA(ch, i, L);
        const double d = lap_diag(t, L) - k2 - A * cprev * ip;
        ip = 1.0 / d;
        out[ch.tau0 + ch.dtau * i] = ip;
        cprev = chainC(ch, i, L);
    }
}

// Solves one chain in place: rows a_i x_{i-1} + b_i x_i + c_i x_{i+1} = F_i
// with F = Msin^2 X computed on the fly from the transform output.  With the
// pivots given, the Thomas sweeps are two affine recurrences
//   r'_i = F_i + alpha_i r'_{i-1},   alpha_i = -a_i / d'_{i-1}
//   x_i  = r'_i / d'_i + beta_i x_{i+1},  beta_i = -c_i / d'_i
// Each thread owns a contiguous segment: a local pass composes its segment's
// affine map, a block scan gives every segment its incoming value, and a
// second pass applies it.  ip[tau] is the pivot of the element at natural
// FFT index tau (shared-memory window of the plan table).
__device__ void solve_chain(double2* a, const int* rev, const double* ip, V4* wsc, const Chain& ch, int L,
                            double2 inner, double& fmax_acc, double2& wsum, bool want_wsum, double2* x_first) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int n = ch.n;
    const int s = static_cast<int>((static_cast<long long>(tid) * n) / nthr);
    const int e = static_cast<int>((static_cast<long long>(tid + 1) * n) / nthr);
    auto pos = [&](int i) { return rev[ch.tau0 + ch.dtau * i]; };
    auto Fof = [&](double2 xm, double2 x0, double2 xp, int i) {
        const double d2 = chainD2(ch, i, L);
        return make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
    };
    // boundary neighbours (original transform values) before anyone writes
    double2 xlo = make_double2(0.0, 0.0), xhi = make_double2(0.0, 0.0);
    if (s < e) {
        xlo = (s == 0) ? inner : a[pos(s - 1)];
        xhi = (e < n) ? a[pos(e)] : make_double2(0.0, 0.0);
    }
    __syncthreads();

    // ---- local forward summary: r'_{e-1} = P r'_{s-1} + rt
    V4 aff = AffOp::identity();
    {
        double2 xm = xlo;
        double2 x0 = (s < e) ? a[pos(s)] : make_double2(0.0, 0.0);
        double ipp = (s > 0) ? ip[ch.tau0 + ch.dtau * (s - 1)] : 0.0;
        for (int i = s; i < e; ++i) {
            const double2 xp = (i + 1 < e) ? a[pos(i + 1)] : xhi;
            const double2 F = Fof(xm, x0, xp, i);
            fmax_acc = fmax(fmax_acc, F.x * F.x + F.y * F.y);  // squared; sqrt at the end
            const double al = -chainA(ch, i, L) * ipp;
            aff = V4{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y), 0.0};
            ipp = ip[ch.tau0 + ch.dtau * i];
            xm = x0;
            x0 = xp;
        }
    }
    const V4 rin = block_exclusive_scan<AffOp, false>(aff, wsc);  // r'_{s-1} = rin.(b, c)

    // ---- forward sweep with the true incoming value, r' in place
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = (s > 0) ? ip[ch.tau0 + ch.dtau * (s - 1)] : 0.0;
        double2 xm = xlo;
        double2 x0 = (s < e) ? a[pos(s)] : make_double2(0.0, 0.0);
        for (int i = s; i < e; ++i) {
            const int pi = pos(i);
            const double2 xp = (i + 1 < e) ? a[pos(i + 1)] : xhi;
            const double2 F = Fof(xm, x0, xp, i);
            const double al = -chainA(ch, i, L) * ipp;
            rp = make_double2(fma(al, rp.x, F.x), fma(al, rp.y, F.y));
            a[pi] = rp;
            ipp = ip[ch.tau0 + ch.dtau * i];
            xm = x0;
            x0 = xp;
        }
    }
    __syncthreads();

    // ---- local backward summary x_s = P x_e + xt
    V4 baff = AffOp::identity();
    for (int i = e - 1; i >= s; --i) {
        const double iv = ip[ch.tau0 + ch.dtau * i];
        const double2 r = a[pos(i)];
        const double be = -chainC(ch, i, L) * iv;
        baff = V4{be * baff.a, fma(be, baff.b, r.x * iv), fma(be, baff.c, r.y * iv), 0.0};
    }
    const V4 xin = block_exclusive_scan<AffOp, true>(baff, wsc);  // x_e

    // ---- back substitution, x in place
    double2 ws = make_double2(0.0, 0.0);
    {
        double2 x = make_double2(xin.b, xin.c);
        for (int i = e - 1; i >= s; --i) {
            const int pi = pos(i);
            const double iv = ip[ch.tau0 + ch.dtau * i];
            const double2 r = a[pi];
            const double c = -chainC(ch, i, L) * iv;
            x = make_double2(fma(c, x.x, r.x * iv), fma(c, x.y, r.y * iv));
            a[pi] = x;
            if (want_wsum) {
                const double t = ch.t0 + ch.dt * i;
                const double w = 2.0 / (1.0 - t * t);
                ws.x = fma(w, x.x, ws.x);
                ws.y = fma(w, x.y, ws.y);
            }
            if (i == 0) *x_first = x;
        }
    }
    wsum.x += ws.x;
    wsum.y += ws.y;
    __syncthreads();
}

// Chain solve with a fixed segment of S elements per thread (threads past the
// chain end, and elements past it, carry zero pivots and data, which makes
// their maps send everything to 0 — exactly the x_n = 0 truncation).
//   pass 1: X -> F = Msin^2 X (registers) and the segment's forward map;
//   pass 2: forward sweep r' -> g = r'/d' (to shared memory) while
//           accumulating the segment's backward map x_s = G + P x_e
//           (P = prod c_u, G = sum g_u prod_{j<u} c_j, c = -C/d');
//   pass 3: back substitution x_u = c_u x_(u+1) + g_u.
// Positions (digit-reversed slots, < 2^16) are kept packed two per register;
// pivots stay in registers.  Chain coefficients come from t by FMAs
// (4A = t (t - 3s) + 2, 4C = t (t + 3s) + 2, s = sign dt); max |F|^2 is kept
// on the high word of its IEEE pattern (relative resolution 2^-20 of the
// squared value; it only scales the precondition threshold).
// Affine-map scan of the V4-based walks through the one-barrier Aff3 scan
// (slot set `set` of the 32-entry scratch).
template <bool REV>
__device__ __forceinline__ V4 scan_v4(V4 v, V4* wsc, int set = 0) {
    const Aff3 r = block_scan_aff1<REV>(Aff3{v.a, v.b, v.c}, reinterpret_cast<Aff3*>(wsc) + set);
    return V4{r.a, r.b, r.c, 0.0};
}

// Register-resident variant of solve_chain for segments of at most SMAX
// elements per thread: every chain element is read from shared memory once
// (its position through the digit-reversal table once), F, r' and the pivots
// stay in registers across the four sweeps, and x is written once.
template <int SMAX>
__device__ void solve_chain_reg(double2* a, const int* rev, const double* ip, V4* wsc, const Chain& ch, int L,
                                double2 inner, double& fmax_acc, double2& wsum, bool want_wsum, double2* x_first) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int n = ch.n;
    const int s = static_cast<int>((static_cast<long long>(tid) * n) / nthr);
    const int e = static_cast<int>((static_cast<long long>(tid + 1) * n) / nthr);
    const int m = e - s;
    int pos[SMAX];
    double2 v[SMAX];   // X, then F, then r'
    double ipv[SMAX];
#pragma unroll
    for (int u = 0; u < SMAX; ++u)
        if (u < m) pos[u] = rev[ch.tau0 + ch.dtau * (s + u)];
    const double ip_before = (s > 0 && m > 0) ? ip[ch.tau0 + ch.dtau * (s - 1)] : 0.0;
    double2 xlo = make_double2(0.0, 0.0), xhi = make_double2(0.0, 0.0);
    if (m > 0) {
        xlo = (s == 0) ? inner : a[rev[ch.tau0 + ch.dtau * (s - 1)]];
        xhi = (e < n) ? a[rev[ch.tau0 + ch.dtau * e]] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < SMAX; ++u) {
        if (u < m) {
            v[u] = a[pos[u]];
            ipv[u] = ip[ch.tau0 + ch.dtau * (s + u)];
        }
    }
    if (ch.dt > 0) SK_PROBE(12);
    // F = Msin^2 X in registers (ascending, keeping the previous original X)
    {
        double2 xm = xlo;
#pragma unroll
        for (int u = 0; u < SMAX; ++u) {
            if (u < m) {
                const double2 x0 = v[u];
                const double2 xp = (u + 1 < m) ? v[u + 1] : xhi;
                const double d2 = chainD2(ch, s + u, L);
                v[u] = make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
                fmax_acc = fmax(fmax_acc, v[u].x * v[u].x + v[u].y * v[u].y);  // squared
                xm = x0;
            }
        }
    }
    if (ch.dt > 0) SK_PROBE(13);
    // local forward summary
    V4 aff = AffOp::identity();
    {
        double ipp = ip_before;
#pragma unroll
        for (int u = 0; u < SMAX; ++u) {
            if (u < m) {
                const double al = -chainA(ch, s + u, L) * ipp;
                aff = V4{al * aff.a, fma(al, aff.b, v[u].x), fma(al, aff.c, v[u].y), 0.0};
                ipp = ipv[u];
            }
        }
    }
    if (ch.dt > 0) SK_PROBE(14);
    const V4 rin = scan_v4<false>(aff, wsc);
    if (ch.dt > 0) SK_PROBE(15);
    // forward sweep: r' in registers
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
#pragma unroll
        for (int u = 0; u < SMAX; ++u) {
            if (u < m) {
                const double al = -chainA(ch, s + u, L) * ipp;
                rp = make_double2(fma(al, rp.x, v[u].x), fma(al, rp.y, v[u].y));
                v[u] = rp;
                ipp = ipv[u];
            }
        }
    }
    if (ch.dt > 0) SK_PROBE(16);
    // local backward summary
    V4 baff = AffOp::identity();
#pragma unroll
    for (int u = SMAX - 1; u >= 0; --u) {
        if (u < m) {
            const double iv = ipv[u];
            const double be = -chainC(ch, s + u, L) * iv;
            baff = V4{be * baff.a, fma(be, baff.b, v[u].x * iv), fma(be, baff.c, v[u].y * iv), 0.0};
        }
    }
    if (ch.dt > 0) SK_PROBE(17);
    const V4 xin = scan_v4<true>(baff, wsc, 16);  // also orders every read above before the writes below
    if (ch.dt > 0) SK_PROBE(18);
    double2 ws = make_double2(0.0, 0.0);
    {
        double2 x = make_double2(xin.b, xin.c);
#pragma unroll
        for (int u = SMAX - 1; u >= 0; --u) {
            if (u < m) {
                const double iv = ipv[u];
                const double c = -chainC(ch, s + u, L) * iv;
                x = make_double2(fma(c, x.x, v[u].x * iv), fma(c, x.y, v[u].y * iv));
                a[pos[u]] = x;
                if (want_wsum) {
                    const double t = ch.t0 + ch.dt * (s + u);
                    const double w = 2.0 / (1.0 - t * t);
                    ws.x = fma(w, x.x, ws.x);
                    ws.y = fma(w, x.y, ws.y);
                }
                if (s + u == 0) *x_first = x;
            }
        }
    }
    wsum.x += ws.x;
    wsum.y += ws.y;
    __syncthreads();
    if (ch.dt > 0) SK_PROBE(19);
}

// Opaque copies: stop the compiler from keeping per-element values derived in
// one pass (t_u, unpacked slots) alive across the block scans into the next.
__device__ __forceinline__ double launder(double x) {
    double y;
    asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ unsigned launder(unsigned x) {
    unsigned y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

#ifndef SK_CHAIN_ATTR
#define SK_CHAIN_ATTR __noinline__
#endif
template <int S, bool HI>
__device__ SK_CHAIN_ATTR void solve_chain_fast(double2* a, const int* __restrict__ rev, const double* ip, Aff3* wsc,
                                                 const Chain& ch, int L, double2 inner, unsigned* fmax_hi,
                                                 double2* wsum, bool want_wsum, double2* x_first) {
    constexpr int SP = (S + 1) / 2;
    const int tid = threadIdx.x;
    const int n = ch.n;
    if (n <= 0) return;
    const int s = tid * S;
    const double s3 = ch.dt > 0 ? 3.0 : -3.0;
    const double dtd = ch.dt;
    const double t_s = static_cast<double>(ch.t0) + dtd * static_cast<double>(s);
    const double tlo = -static_cast<double>(L), thi = static_cast<double>(L - 1);
    unsigned pk[SP];
    double2 v[S];
    double ipv[S];
    // Loads with compile-time offsets from a per-thread base: element u sits at
    // natural index tau0 + dtau (s + u).  Elements past the chain end read
    // slot 0 and no table entry: with the digit-reversal window (rev_win) the
    // entries beyond the chain lie outside the window, and a stray slot index
    // would address beyond the CTA's shared memory.
    auto load_seg = [&](auto dir) {
        constexpr int D = decltype(dir)::value;
        const int tb = ch.tau0 + (D > 0 ? s : -s);
        const int* rb = rev + tb;
        const double* ib = ip + tb;
#pragma unroll
        for (int u = 0; u < S; u += 2) {
            const unsigned p0 = (s + u < n) ? static_cast<unsigned>(rb[D * u]) : 0u;
            const unsigned p1 = (u + 1 < S && s + u + 1 < n) ? static_cast<unsigned>(rb[D * (u + 1)]) : 0u;
            pk[u / 2] = p0 | (p1 << 16);
        }
#pragma unroll
        for (int u = 0; u < S; ++u) ipv[u] = (s + u < n) ? ib[D * u] : 0.0;
    };
    if (ch.dtau > 0) load_seg(std::integral_constant<int, 1>{});
    else load_seg(std::integral_constant<int, -1>{});
    auto posu = [&](int u) { return static_cast<int>((u & 1) ? (pk[u / 2] >> 16) : (pk[u / 2] & 0xffffu)); };
    double2 xlo = inner, xhi = make_double2(0.0, 0.0);
    double ip_before = 0.0;
    if (s > 0 && s <= n) {
        const int tb = ch.tau0 + ch.dtau * (s - 1);
        xlo = a[rev[tb]];
        ip_before = ip[tb];
    }
    if (s + S < n) xhi = a[rev[ch.tau0 + ch.dtau * (s + S)]];
#pragma unroll
    for (int u = 0; u < S; ++u) {
        const bool ok = s + u < n;
        const double2 x = a[posu(u)];
        v[u] = ok ? x : make_double2(0.0, 0.0);
        if (!ok) ipv[u] = 0.0;
    }
    // ---- pass 1
    Aff3 aff = aff_identity();
    {
        unsigned fh = 0u;
        double2 xm = xlo;
        double ipp = ip_before;
        double t = t_s;
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const double2 x0 = v[u];
            const double2 xp = (u + 1 < S) ? v[u + 1] : xhi;
            const double d2 = (t == tlo || t == thi) ? 0.25 : 0.5;
            double2 F = make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
            if (s + u >= n) F = make_double2(0.0, 0.0);
            fh = max(fh, static_cast<unsigned>(__double2hiint(fma(F.x, F.x, F.y * F.y))));
            const double al = (-0.25 * ipp) * fma(t, t - s3, 2.0);
            aff = Aff3{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y)};
            v[u] = F;
            ipp = ipv[u];
            xm = x0;
            t += dtd;
        }
        *fmax_hi = max(*fmax_hi, fh);
    }
    const Aff3 rin = block_scan_aff1<false>(aff, wsc);  // also orders every X read above before the writes below
#pragma unroll
    for (int u = 0; u < SP; ++u) pk[u] = launder(pk[u]);
    // ---- pass 2
    Aff3 baff;
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
        double t = launder(t_s);
        double Pm = 1.0;
        double2 G = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const double al = (-0.25 * ipp) * fma(t, t - s3, 2.0);
            rp = make_double2(fma(al, rp.x, v[u].x), fma(al, rp.y, v[u].y));
            const double iv = ipv[u];
            const double2 g = make_double2(rp.x * iv, rp.y * iv);
            const double c = (-0.25 * iv) * fma(t, t + s3, 2.0);
            G = make_double2(fma(Pm, g.x, G.x), fma(Pm, g.y, G.y));
            Pm *= c;
            if (s + u < n) a[posu(u)] = g;
            ipv[u] = c;
            ipp = iv;
            t += dtd;
        }
        baff = Aff3{Pm, G.x, G.y};
    }
    const Aff3 xin = block_scan_aff1<true>(baff, wsc + 16);
    // ---- pass 3
#pragma unroll
    for (int u = 0; u < SP; ++u) pk[u] = launder(pk[u]);
    const double t_s3 = launder(t_s);
    double2 x = make_double2(xin.b, xin.c);
    double2 ws = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = S - 1; u >= 0; --u) {
        if (s + u < n) {
            const int p = posu(u);
            const double2 g = a[p];
            x = make_double2(fma(ipv[u], x.x, g.x), fma(ipv[u], x.y, g.y));
            a[p] = x;
            if (want_wsum) {
                const double t = t_s3 + dtd * u;
                const double w = 2.0 / (1.0 - t * t);
                ws.x = fma(w, x.x, ws.x);
                ws.y = fma(w, x.y, ws.y);
            }
        } else {
            x = make_double2(0.0, 0.0);
        }
    }
    wsum->x += ws.x;
    wsum->y += ws.y;
    if (tid == 0) *x_first = x;
    __syncthreads();
}

// Both chains of a parity class from ONE segmented solve (the pairing of
// theta_sym.cu, here on the unpruned transform of short columns, L even):
// chain- (t < 0) sees s = (-1)^k times chain+'s right-hand side except on its
// last rows (X_{-t} = s X_t + (1 - s) X_0 makes F- = s F+ in the interior and
// at the inner end) and the same pivots up to there, so x- = s x+ + Phi Delta
// with Phi_i = prod_{j=i}^{n-2} c_j the backward sweep's own product and Delta
// the difference of the chains' last unknowns, computed by the thread that
// owns chain+'s last element from the boundary rows (chain- values are read
// directly: the whole transform is present).  ip: chain+'s pivot window
// (ip[tau]); ip_extra: table entry tau = L/2 (par 0: chain-'s extra element
// t = -L; par 1: chain-'s last element, an interior row where chain+ ends on
// the truncation row).  g = r'/d' stays in F's registers between the sweeps.
template <int S, bool HI>
__device__ SK_CHAIN_ATTR void solve_chains_pair_fast(double2* a, const int* __restrict__ rev, const double* ip, Aff3* wsc,
                                                     double2* misc, int par, int L, double sgn, double2 inner,
                                                     double ip_extra, unsigned* fmax_hi, double2* wsum,
                                                     bool want_wsum) {
    constexpr int SP = (S + 1) / 2;
    const int tid = threadIdx.x;
    const int n = par == 0 ? L / 2 - 1 : L / 2;  // chain+ length
    const int tau0 = par == 0 ? 1 : 0;
    const int s = tid * S;
    const double t_s = (par == 0 ? 2.0 : 1.0) + 2.0 * static_cast<double>(s);
    const double tl = static_cast<double>(L - 1);
    unsigned pk[SP];
    double2 v[S];
    double ipv[S];
    {
        const int* rb = rev + tau0 + s;
        const double* ib = ip + tau0 + s;
#pragma unroll
        for (int u = 0; u < S; u += 2) {
            const unsigned p0 = (s + u < n) ? static_cast<unsigned>(rb[u]) : 0u;
            const unsigned p1 = (u + 1 < S && s + u + 1 < n) ? static_cast<unsigned>(rb[u + 1]) : 0u;
            pk[u / 2] = p0 | (p1 << 16);
        }
#pragma unroll
        for (int u = 0; u < S; ++u) ipv[u] = (s + u < n) ? ib[u] : 0.0;
    }
    auto posu = [&](int u) { return static_cast<int>((u & 1) ? (pk[u / 2] >> 16) : (pk[u / 2] & 0xffffu)); };
    double2 xlo = inner, xhi = make_double2(0.0, 0.0);
    double ip_before = 0.0;
    if (s > 0 && s <= n) {
        xlo = a[rev[tau0 + s - 1]];
        ip_before = ip[tau0 + s - 1];
    }
    if (s + S < n) xhi = a[rev[tau0 + s + S]];
#pragma unroll
    for (int u = 0; u < S; ++u) {
        const bool ok = s + u < n;
        const double2 x = a[posu(u)];
        v[u] = ok ? x : make_double2(0.0, 0.0);
        if (!ok) ipv[u] = 0.0;
    }
    const int ulast = n - 1 - s;  // chain+'s last element in this segment if 0 <= ulast < S
    // ---- pass 1: F = Msin^2 X, forward affine summary
    Aff3 aff = aff_identity();
    double2 xlast = make_double2(0.0, 0.0), xlast_m = make_double2(0.0, 0.0);
    unsigned fh = 0u;
    {
        double2 xm = xlo;
        double ipp = ip_before;
        double t = t_s;
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const double2 x0 = v[u];
            const double2 xp = (u + 1 < S) ? v[u + 1] : xhi;
            if (u == ulast) {
                xlast = x0;
                xlast_m = xm;
            }
            const double d2 = (t == tl) ? 0.25 : 0.5;
            double2 F = make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
            if (s + u >= n) F = make_double2(0.0, 0.0);
            fh = max(fh, static_cast<unsigned>(__double2hiint(fma(F.x, F.x, F.y * F.y))));
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);
            aff = Aff3{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y)};
            v[u] = F;
            ipp = ipv[u];
            xm = x0;
            t += 2.0;
        }
    }
    const Aff3 rin = block_scan_aff1<false>(aff, wsc);
#pragma unroll
    for (int u = 0; u < SP; ++u) pk[u] = launder(pk[u]);
    // ---- pass 2: r', g = r'/d' (registers), backward summary with the last multiplier 1
    Aff3 baff;
    double2 rlast = make_double2(0.0, 0.0);
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
        double t = launder(t_s);
        double Pm = 1.0;
        double2 G = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);
            rp = make_double2(fma(al, rp.x, v[u].x), fma(al, rp.y, v[u].y));
            if (u == ulast) rlast = rp;
            const double iv = ipv[u];
            const double2 g = make_double2(rp.x * iv, rp.y * iv);
            double c = (-0.25 * iv) * fma(t, t + 3.0, 2.0);
            if (u == ulast || s + u >= n) c = 1.0;
            G = make_double2(fma(Pm, g.x, G.x), fma(Pm, g.y, G.y));
            Pm *= c;
            v[u] = g;
            ipv[u] = c;
            ipp = iv;
            t += 2.0;
        }
        baff = Aff3{Pm, G.x, G.y};
    }
    // ---- the boundary rows (theta_mp.cu TC): Delta = x-_{n-1} - s x+_{n-1}
    if (ulast >= 0 && ulast < S) {
        const double ipl = ip[tau0 + n - 1];
        const double2 xp_last = make_double2(rlast.x * ipl, rlast.y * ipl);
        const double2 Xm_last = a[rev[L - 1 - (n - 1)]];   // chain- element n-1
        const double2 Xm_last2 = a[rev[L - 1 - (n - 2)]];  // chain- element n-2
        double2 xm_last, xm_extra = make_double2(0.0, 0.0);
        unsigned fb;
        const double2 Fp = make_double2((par ? 0.25 : 0.5) * xlast.x - 0.25 * xlast_m.x,
                                        (par ? 0.25 : 0.5) * xlast.y - 0.25 * xlast_m.y);  // F+_{n-1}
        if (par == 0) {
            const double Ld = L;
            const double2 XmL = a[rev[L / 2]];  // X at t = -L
            const double2 Fm1 = make_double2(0.5 * Xm_last.x - 0.25 * (Xm_last2.x + XmL.x),
                                             0.5 * Xm_last.y - 0.25 * (Xm_last2.y + XmL.y));
            const double2 rm1 = make_double2(sgn * rlast.x + (Fm1.x - sgn * Fp.x), sgn * rlast.y + (Fm1.y - sgn * Fp.y));
            const double2 Fn = make_double2(0.25 * (XmL.x - Xm_last.x), 0.25 * (XmL.y - Xm_last.y));
            const double An = 0.25 * (Ld - 2.0) * (Ld - 1.0);  // coupling of t = -L to t = -(L-2)
            const double Cm = 0.25 * Ld * (Ld - 1.0);          // coupling of t = -(L-2) to t = -L
            const double al = -An * ipl;
            const double2 rn = make_double2(fma(al, rm1.x, Fn.x), fma(al, rm1.y, Fn.y));
            xm_extra = make_double2(rn.x * ip_extra, rn.y * ip_extra);
            const double be = -Cm * ipl;
            xm_last = make_double2(fma(be, xm_extra.x, rm1.x * ipl), fma(be, xm_extra.y, rm1.y * ipl));
            fb = max(static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y))),
                     static_cast<unsigned>(__double2hiint(fma(Fn.x, Fn.x, Fn.y * Fn.y))));
        } else {
            const double2 Fm1 = make_double2(0.5 * Xm_last.x - 0.25 * Xm_last2.x, 0.5 * Xm_last.y - 0.25 * Xm_last2.y);
            const double2 rm1 = make_double2(sgn * rlast.x + (Fm1.x - sgn * Fp.x), sgn * rlast.y + (Fm1.y - sgn * Fp.y));
            xm_last = make_double2(rm1.x * ip_extra, rm1.y * ip_extra);
            fb = static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y)));
        }
        fh = max(fh, fb);
        misc[5] = make_double2(xm_last.x - sgn * xp_last.x, xm_last.y - sgn * xp_last.y);  // Delta
        misc[6] = xm_extra;
    }
    *fmax_hi = max(*fmax_hi, fh);
    const Aff3 xin = block_scan_aff1<true>(baff, wsc + 16);  // its barrier publishes Delta and orders the X reads above
    const double2 Dl = misc[5];
    // ---- pass 3: x+ = g + c x+, x- = s x+ + Phi Delta into both chains' slots
#pragma unroll
    for (int u = 0; u < SP; ++u) pk[u] = launder(pk[u]);
    const double t_s3 = launder(t_s);
    double2 x = make_double2(xin.b, xin.c);
    double phi = xin.a;
    double2 ws = make_double2(0.0, 0.0);
    double2 xf_p = make_double2(0.0, 0.0), xf_m = make_double2(0.0, 0.0);
    const int* rm = rev + (L - 1 - s);  // chain- element i at natural index L - 1 - i
#pragma unroll
    for (int u = S - 1; u >= 0; --u) {
        if (s + u < n) {
            const double c = ipv[u];
            const double2 g = v[u];
            x = (u != ulast) ? make_double2(fma(c, x.x, g.x), fma(c, x.y, g.y)) : g;
            phi *= c;
            const double2 xm = make_double2(fma(phi, Dl.x, sgn * x.x), fma(phi, Dl.y, sgn * x.y));
            a[posu(u)] = x;
            a[rm[-u]] = xm;
            if (want_wsum) {
                const double t = t_s3 + 2.0 * u;
                const double w = 2.0 / (1.0 - t * t);  // w(t) = w(-t)
                ws.x = fma(w, x.x + xm.x, ws.x);
                ws.y = fma(w, x.y + xm.y, ws.y);
            }
            xf_p = x;
            xf_m = xm;
        }
    }
    if (par == 0 && ulast >= 0 && ulast < S) {
        const double2 xe = misc[6];
        a[rev[L / 2]] = xe;  // x at t = -L
        if (want_wsum) {
            const double Ld = L;
            const double w = 2.0 / (1.0 - Ld * Ld);
            ws.x = fma(w, xe.x, ws.x);
            ws.y = fma(w, xe.y, ws.y);
        }
    }
    wsum->x += ws.x;
    wsum->y += ws.y;
    if (tid == 0) {
        misc[3] = xf_p;  // x+_0
        misc[4] = xf_m;  // x-_0
    }
    __syncthreads();
}

// Smallest register segment S with ceil(n / S) <= nthr; 0 if none fits.
__device__ __forceinline__ int chain_segment(int n, int nthr) {
    const int need = (n + nthr - 1) / nthr;
    if (need <= 2) return 2;
    if (need <= 4) return 4;
    if (need <= 6) return 6;
    if (need <= 8) return 8;
    if (need <= 10) return 10;
    if (need <= 12) return 12;
    return 0;
}

template <bool HI>
__device__ __forceinline__ bool solve_chain_fast_dispatch(double2* a, const int* rev, const double* ip, Aff3* wsc,
                                                          const Chain& ch, int L, double2 inner, unsigned* fmax_hi,
                                                          double2* wsum, bool want_wsum, double2* x_first) {
#define SK_CH(S) solve_chain_fast<S, HI>(a, rev, ip, wsc, ch, L, inner, fmax_hi, wsum, want_wsum, x_first)
    switch (chain_segment(ch.n, blockDim.x)) {
        case 2: SK_CH(2); return true;
        case 4: SK_CH(4); return true;
        case 6: SK_CH(6); return true;
        case 8: SK_CH(8); return true;
        case 10: SK_CH(10); return true;
        case 12: SK_CH(12); return true;
        default: return false;
    }
#undef SK_CH
}

template <bool HI>
__device__ __forceinline__ bool solve_chains_pair_dispatch(double2* a, const int* rev, const double* ip, Aff3* wsc,
                                                           double2* misc, int par, int L, double sgn, double2 inner,
                                                           double ip_extra, unsigned* fmax_hi, double2* wsum,
                                                           bool want_wsum) {
    const int n = par == 0 ? L / 2 - 1 : L / 2;
#define SK_CH(S) solve_chains_pair_fast<S, HI>(a, rev, ip, wsc, misc, par, L, sgn, inner, ip_extra, fmax_hi, wsum, want_wsum)
    switch (chain_segment(n, blockDim.x)) {
        case 2: SK_CH(2); return true;
        case 4: SK_CH(4); return true;
        case 6: SK_CH(6); return true;
        default: return false;
    }
#undef SK_CH
}

// The lowest lambda modes are only weakly diagonally dominant (k = 0 not at
// all); for them the segmented sweeps lose digits, so one thread runs the
// plain sequential recurrences (pivots from the table).  The chain is walked
// in chunks of U elements whose shared-memory operands are fetched one chunk
// ahead (the chunks touch disjoint slots), so only the FMA recurrence itself
// is on the critical path.
__device__ void solve_chain_seq(double2* a, const int* rev, const double* ip, const Chain& ch, int L, double2 inner,
                                double& fmax_acc, double2& wsum, bool want_wsum, double2* x_first) {
    constexpr int U = 8;
    if (threadIdx.x == 0 && ch.n > 0) {
        const int n = ch.n;
        auto pos = [&](int i) { return rev[ch.tau0 + ch.dtau * i]; };
        // ---- forward: r'_i = F_i + alpha_i r'_{i-1}
        int pc[U];
        double2 xc[U];
        double2 xnext0;  // X of the first element of the following chunk
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pc[u] = u < n ? pos(u) : 0;
            xc[u] = u < n ? a[pc[u]] : make_double2(0.0, 0.0);
        }
        xnext0 = U < n ? a[pos(U)] : make_double2(0.0, 0.0);
        double2 xm = inner, rp = make_double2(0.0, 0.0);
        double ipp = 0.0;
        for (int c0 = 0; c0 < n; c0 += U) {
            // prefetch the next chunk (slots disjoint from this chunk's)
            int pn[U];
            double2 xn[U];
            double2 xnn;
            double ipc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ipc[u] = (c0 + u < n) ? ip[ch.tau0 + ch.dtau * (c0 + u)] : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = c0 + U + u;
                pn[u] = i < n ? pos(i) : 0;
                xn[u] = i < n ? a[pn[u]] : make_double2(0.0, 0.0);
            }
            xnn = (c0 + 2 * U < n) ? a[pos(c0 + 2 * U)] : make_double2(0.0, 0.0);
            double2 rc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = c0 + u;
                if (i < n) {
                    const double2 x0 = xc[u];
                    const double2 xp = (u + 1 < U) ? ((i + 1 < n) ? xc[u + 1] : make_double2(0.0, 0.0)) : xnext0;
                    const double d2 = chainD2(ch, i, L);
                    const double2 F =
                        make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
                    fmax_acc = fmax(fmax_acc, F.x * F.x + F.y * F.y);  // squared; sqrt at the end
                    const double al = -chainA(ch, i, L) * ipp;
                    rp = make_double2(fma(al, rp.x, F.x), fma(al, rp.y, F.y));
                    rc[u] = rp;
                    ipp = ipc[u];
                    xm = x0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c0 + u < n) a[pc[u]] = rc[u];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                pc[u] = pn[u];
                xc[u] = xn[u];
            }
            xnext0 = xnn;
        }
        // ---- backward: x_i = r'_i / d'_i - c_i / d'_i x_{i+1}
        double2 x = make_double2(0.0, 0.0);
        double2 ws = make_double2(0.0, 0.0);
        const int last = n - 1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = last - u;
            pc[u] = i >= 0 ? pos(i) : 0;
            xc[u] = i >= 0 ? a[pc[u]] : make_double2(0.0, 0.0);
        }
        for (int c0 = last; c0 >= 0; c0 -= U) {
            int pn[U];
            double2 xn[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = c0 - U - u;
                pn[u] = i >= 0 ? pos(i) : 0;
                xn[u] = i >= 0 ? a[pn[u]] : make_double2(0.0, 0.0);
            }
            double ipc[U];
            double2 xo[U];
#pragma unroll
            for (int u = 0; u < U; ++u) ipc[u] = (c0 - u >= 0) ? ip[ch.tau0 + ch.dtau * (c0 - u)] : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = c0 - u;
                if (i >= 0) {
                    const double iv = ipc[u];
                    const double c = -chainC(ch, i, L) * iv;
                    x = make_double2(fma(c, x.x, xc[u].x * iv), fma(c, x.y, xc[u].y * iv));
                    xo[u] = x;
                    if (want_wsum) {
                        const double t = ch.t0 + ch.dt * i;
                        const double w = 2.0 / (1.0 - t * t);
                        ws.x = fma(w, x.x, ws.x);
                        ws.y = fma(w, x.y, ws.y);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c0 - u >= 0) a[pc[u]] = xo[u];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                pc[u] = pn[u];
                xc[u] = xn[u];
            }
        }
        *x_first = x;
        wsum.x += ws.x;
        wsum.y += ws.y;
    }
    __syncthreads();
}

// One 2-CTA cluster per lambda mode k: CTA `par` (0/1) owns the theta modes
// of parity par.  Folding the DFS-symmetric column onto the two parity
// classes is the first radix-2 step of the length-M theta transform; each CTA
// then runs a length-M/2 transform, the chains of its parity (the +-1 band
// offsets of lap are exact zeros, so even and odd modes never couple), and the
// inverse transform.  The two halves are recombined through distributed
// shared memory.
// CH selects the chain solver at compile time (one per kernel so that the
// register allocation of each is independent): 0 shared-memory walk,
// 1 fixed short segments (solve_chain_fast), 2 SMAX = 12 register walk.
// HI: high-occupancy variant for short columns (<= 256 threads per CTA, radices
// <= 8): 64 registers per thread, so twice the CTAs per SM hide the latency of
// a transform that gives each thread only one or two butterflies per stage.
template <bool SWZ, int CH, bool HI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(HI ? 256 : 512, HI ? 4 : 1)
    theta_kernel(ThetaParams P, int relaxed_exit, const __grid_constant__ CUtensorMap cmap,
                 const __grid_constant__ CUtensorMap cmap_tail) {
    constexpr int kFold = HI ? kFoldMaxHi : kFoldMax;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L = P.fd.L;  // M/2
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + theta_data_slots(L);  // raw column (L+1 values), then the swizzled transform
    double2* s_lo = s_hi + P.fd.nhi;
    double* ip = reinterpret_cast<double*>(s_lo + P.fd.nlo);
    V4* wsc = reinterpret_cast<V4*>(ip + theta_chain_slots(L));
    double2* misc = reinterpret_cast<double2*>(wsc + 32);
    double* red = reinterpret_cast<double*>(misc + 16);
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 64);
    int* rw = reinterpret_cast<int*>(bars + 2);  // digit-reversal window (P.rev_win)

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int par = static_cast<int>(cluster.block_rank());
    const int col = blockIdx.x >> 1;
    const int rhs = col / P.ncols;
    const int kl = col - rhs * P.ncols;
    const int kg = P.k0 + kl;  // global lambda mode, 0..N/2
    const double k2 = static_cast<double>(kg) * static_cast<double>(kg);
    const double sgn = (kg & 1) ? -1.0 : 1.0;
    const int* rev = P.fd.rev;
    double2* colbase = P.buf + rhs * P.rhs_stride;

    Chain cp, cm;
    make_chains(par, L, cp, cm);
    const size_t prow = (static_cast<size_t>(kl) * 2 + par) * P.piv_stride;  // pivot row (table index)


    // ---- bulk copies: the raw column (L+1 values) and the t > 0 chain's pivots
    SK_PROBE(0);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t bytes = 0, pb = 0;
        const double* pv = pivot_window(ip, P.pivots, prow, cp.tau0, cp.tau0 + cp.n, pb);
        (void)pv;
        for (int s = 0; s < P.sl.P; ++s) {
            const int r0 = P.sl.row_b[s], r1 = P.sl.row_b[s + 1];
            if (r1 > r0) bytes += (r1 - r0) * 16;
        }
        int ra0 = 0;
        uint32_t rbytes = 0;
        if (P.rev_win) rev_window(rw, cp.tau0, cp.tau0 + cp.n, ra0, rbytes);
        if (P.gather) bytes = static_cast<uint32_t>(P.gather_nbox * 256 + P.gather_tail) * 16;
        mbar_expect_tx(&bars[0], bytes + pb + rbytes);
        if (rbytes) bulk_g2s_chunked(rw, P.fd.rev + ra0, rbytes, &bars[0]);
        if (P.gather) {
            // column kl of the row-major spectrum R[rhs][p][k] (lambda_fwd_kernel's contiguous rows):
            // gather_nbox boxes of 256 rows and a tail box (a multiple of 8 rows: 128-byte destinations),
            // 16 bytes per row, through the two tensor maps; rows past M/2 are zero-filled
            for (int b = 0; b < P.gather_nbox; ++b) tma_load_3d(a + b * 256, &cmap, 2 * kl, b * 256, rhs, &bars[0]);
            if (P.gather_tail)
                tma_load_3d(a + P.gather_nbox * 256, &cmap_tail, 2 * kl, P.gather_nbox * 256, rhs, &bars[0]);
        } else {
            for (int s = 0; s < P.sl.P; ++s) {
                const int r0 = P.sl.row_b[s], r1 = P.sl.row_b[s + 1];
                if (r1 > r0)
                    bulk_g2s_chunked(a + r0, colbase + theta_addr(P.sl, P.ncols, kl, r0), (r1 - r0) * 16, &bars[0]);
            }
        }
        const size_t a0 = (prow + cp.tau0) & ~static_cast<size_t>(1);
        if (pb) bulk_g2s_chunked(ip, P.pivots + a0, pb, &bars[0]);
    }
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    uint32_t pb_unused = 0;
    const double* ipp = pivot_window(ip, P.pivots, prow, cp.tau0, cp.tau0 + cp.n, pb_unused);
    const int* rev_p = rev;
    if (P.rev_win) {
        int ra0;
        uint32_t rb;
        rev_p = rev_window(rw, cp.tau0, cp.tau0 + cp.n, ra0, rb);
    }
    mbar_wait(&bars[0], 0);
    __syncthreads();
    if (P.g.pole_glide && (kg & 1)) {  // the reference's doubled row j = M/2 (sk_internal.h GridGeom)
        if (tid == 0) a[0] = make_double2(-a[0].x, -a[0].y);
        __syncthreads();
    }

    SK_PROBE(1);
    // ---- DFS fold (first radix-2 step), scaled by 1/M.  With the swizzled
    // slot layout the fold goes through registers (kFoldMax pairs per thread,
    // so no slot is overwritten before it is read); otherwise in place.
    const double invM = 1.0 / P.g.M;
    if constexpr (SWZ) {
        double2 v0[kFold], v1[kFold];
#pragma unroll
        for (int u = 0; u < kFold; ++u) {
            const int r = tid + u * nthr;
            if (r <= L / 2) {
                const int rm = L - r;
                const double2 ar = a[r];
                const double2 am = a[rm];
                if (par == 0) {
                    v0[u] = make_double2((ar.x + sgn * am.x) * invM, (ar.y + sgn * am.y) * invM);
                    v1[u] = make_double2((am.x + sgn * ar.x) * invM, (am.y + sgn * ar.y) * invM);
                } else {
                    v0[u] = cscale(cmul(make_double2(ar.x - sgn * am.x, ar.y - sgn * am.y), T(r)), invM);
                    v1[u] = cscale(cmul(make_double2(am.x - sgn * ar.x, am.y - sgn * ar.y), T(rm)), invM);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kFold; ++u) {
            const int r = tid + u * nthr;
            if (r <= L / 2) {
                const int rm = L - r;
                a[swz<true>(r)] = v0[u];
                if (rm < L && rm != r) a[swz<true>(rm)] = v1[u];
            }
        }
    } else {
        for (int r = tid; r <= L / 2; r += nthr) {
            const int rm = L - r;
            const double2 ar = a[r];
            const double2 am = a[rm];
            if (par == 0) {
                // e_r = a_r + s a_{L-r}
                a[r] = make_double2((ar.x + sgn * am.x) * invM, (ar.y + sgn * am.y) * invM);
                if (rm < L && rm != r) a[rm] = make_double2((am.x + sgn * ar.x) * invM, (am.y + sgn * ar.y) * invM);
            } else {
                // o_r = (a_r - s a_{L-r}) w_M^{-r}
                a[r] = cscale(cmul(make_double2(ar.x - sgn * am.x, ar.y - sgn * am.y), T(r)), invM);
                if (rm < L && rm != r)
                    a[rm] = cscale(cmul(make_double2(am.x - sgn * ar.x, am.y - sgn * ar.y), T(rm)), invM);
            }
        }
    }
    __syncthreads();
    SK_PROBE(2);
    fft_forward<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);
    SK_PROBE(3);

    // ---- k = 0, even class: surface mean 2 pi w^T X_0 (poisson.cpp:101-117)
    double* st = P.stats + 4 * rhs;
    if (kg == 0 && par == 0) {
        double2 acc = make_double2(0.0, 0.0);
        for (int tau = tid; tau < L; tau += nthr) {
            const double t = t_of(tau, 0, L);
            const double w = 2.0 / (1.0 - t * t);
            const double2 x = a[__ldg(rev + tau)];
            acc.x = fma(w, x.x, acc.x);
            acc.y = fma(w, x.y, acc.y);
        }
        acc = block_sum2(acc, red);
        if (tid == 0) {
            const double twopi = 6.283185307179586476925286766559;
            st[0] = twopi * acc.x;
            st[1] = twopi * acc.y;
        }
    }

    // ---- chains
    // inner neighbours and the j = 0 row data, read before any chain writes
    if (tid == 0) {
        if (par == 0) {
            const double2 x0 = a[__ldg(rev + 0)];
            const double2 xp2 = cp.n > 0 ? a[__ldg(rev + 1)] : make_double2(0.0, 0.0);
            const double2 xm2 = cm.n > 0 ? a[__ldg(rev + L - 1)] : make_double2(0.0, 0.0);
            misc[0] = x0;
            misc[1] = x0;
            // F_0 = -1/4 X_{-2} + d2(0) X_0 - 1/4 X_2
            const double d2 = msin2_diag(0, L);
            misc[2] = make_double2(d2 * x0.x - 0.25 * (xm2.x + xp2.x), d2 * x0.y - 0.25 * (xm2.y + xp2.y));
        } else {
            misc[0] = cm.n > 0 ? a[__ldg(rev + L - 1)] : make_double2(0.0, 0.0);  // X_{-1}: inner of t>0 chain
            misc[1] = cp.n > 0 ? a[__ldg(rev + 0)] : make_double2(0.0, 0.0);      // X_{+1}: inner of t<0 chain
            misc[2] = make_double2(0.0, 0.0);
        }
        misc[3] = make_double2(0.0, 0.0);
        misc[4] = make_double2(0.0, 0.0);
        misc[5] = misc[6] = make_double2(0.0, 0.0);
        // pivot table entry tau = L/2 (solve_chains_pair_fast's ip_extra)
        misc[8] = make_double2(__ldg(P.pivots + prow + L / 2), 0.0);
    }
    __syncthreads();
    const double2 inner_p = misc[0], inner_m = misc[1], F0 = misc[2];
    double fmax_acc = (par == 0) ? F0.x * F0.x + F0.y * F0.y : 0.0;  // max |F|^2
    double2 wsum = make_double2(0.0, 0.0);
    const bool want_wsum = (kg == 0 && par == 0);
    const bool seq = kg < P.kseq;
    unsigned fmax_hi = 0u;
    Aff3* wsc3 = reinterpret_cast<Aff3*>(wsc);
    auto solve_side = [&](const Chain& ch, const double* ipc, const int* rev, double2 inner, double2* xf) {
        const bool reg12 = ch.n <= kSegMax * nthr;
        if (seq) {
            solve_chain_seq(a, rev, ipc, ch, L, inner, fmax_acc, wsum, want_wsum, xf);
        } else if constexpr (CH == 2) {
            if (reg12) solve_chain_reg<kSegMax>(a, rev, ipc, wsc, ch, L, inner, fmax_acc, wsum, want_wsum, xf);
            else solve_chain(a, rev, ipc, wsc, ch, L, inner, fmax_acc, wsum, want_wsum, xf);
        } else if constexpr (CH == 1) {
            if (!solve_chain_fast_dispatch<HI>(a, rev, ipc, wsc3, ch, L, inner, &fmax_hi, &wsum, want_wsum, xf))
                solve_chain(a, rev, ipc, wsc, ch, L, inner, fmax_acc, wsum, want_wsum, xf);
        } else {
            solve_chain(a, rev, ipc, wsc, ch, L, inner, fmax_acc, wsum, want_wsum, xf);
        }
    };
    // short even columns on the segment solver: both chains from one solve
    // (no second pivot window, no second solve)
    bool paired = false;
    if constexpr (CH == 1) {
        if (P.pair_chains && !seq && !P.rev_win && (L & 1) == 0 && L >= 16)
            paired = solve_chains_pair_dispatch<HI>(a, rev, ipp, wsc3, misc, par, L, sgn, inner_p, misc[8].x, &fmax_hi,
                                                    &wsum, want_wsum);
    }
    if (!paired) solve_side(cp, ipp, rev_p, inner_p, &misc[3]);
    SK_PROBE(4);
    // the t < 0 chain's pivots replace the t > 0 chain's in the window
    const double* ipm = ip;
    const int* rev_m = rev;
    if (cm.n > 0 && !paired) {
        uint32_t pb = 0, rbytes = 0;
        int ra0 = 0;
        ipm = pivot_window(ip, P.pivots, prow, L - cm.n, L, pb);
        if (P.rev_win) rev_m = rev_window(rw, L - cm.n, L, ra0, rbytes);
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(&bars[1], pb + rbytes);
            bulk_g2s_chunked(ip, P.pivots + ((prow + L - cm.n) & ~static_cast<size_t>(1)), pb, &bars[1]);
            if (rbytes) bulk_g2s_chunked(rw, P.fd.rev + ra0, rbytes, &bars[1]);
        }
        mbar_wait(&bars[1], 0);
    }
    SK_PROBE(5);
    if (!paired) solve_side(cm, ipm, rev_m, inner_m, &misc[4]);
    fmax_acc = fmax(fmax_acc, __hiloint2double(static_cast<int>(fmax_hi), 0));
    SK_PROBE(6);
    if (want_wsum) wsum = block_sum2(wsum, red);
    if (par == 0 && tid == 0) {
        double2 x0;
        if (kg != 0) {
            // row j = 0: 1/2 x_{-2} - k^2 x_0 + 1/2 x_2 = F_0
            const double2 xp2 = misc[3], xm2 = misc[4];
            x0 = make_double2((F0.x - 0.5 * xm2.x - 0.5 * xp2.x) / (-k2), (F0.y - 0.5 * xm2.y - 0.5 * xp2.y) / (-k2));
        } else {
            // constraint row 2 pi w^T X_0 = 0 replaces row j = 0 (w_0 = 2)
            x0 = make_double2(-0.5 * wsum.x, -0.5 * wsum.y);
        }
        a[__ldg(rev + 0)] = x0;
    }
    const double fm = sqrt(block_max(fmax_acc, red));
    if (tid == 0) atomic_max_nonneg(st + 2, fm);
    __syncthreads();

    // optional: export the solution coefficients of this parity class
    if (P.xhalf) {
        double2* xo = P.xhalf + static_cast<long long>(rhs) * (P.g.N / 2 + 1) * P.g.M +
                      static_cast<long long>(kg) * P.g.M;
        for (int tau = tid; tau < L; tau += nthr) {
            const int t = t_of(tau, par, L);
            xo[t + L] = a[__ldg(rev + tau)];
        }
    }
    __syncthreads();

    SK_PROBE(7);
    fft_inverse<SWZ, HI ? 8 : 25>(a, P.fd, T, tid, nthr);
    SK_PROBE(8);

    // ---- recombine the parity classes: v_p = Ve_p + w_M^p Vo_p, p = 0..M/2
    cluster.sync();
    const double2* ve = par == 0 ? a : cluster.map_shared_rank(a, 0);
    const double2* vo = par == 1 ? a : cluster.map_shared_rank(a, 1);
    const int half = L / 2;
    const int p_lo = par == 0 ? 0 : half;
    const int p_hi = par == 0 ? half : L + 1;
    for (int p = p_lo + tid; p < p_hi; p += nthr) {
        const int pm = swz<SWZ>(p == L ? 0 : p);
        const double2 v = cadd(ve[pm], cmulc(vo[pm], T(p)));
        if (P.peers.n) *peer_ptr(P.peers, p, kg, p) = v;  // fused return transpose
        else colbase[theta_addr(P.sl, P.ncols, kl, p)] = v;
    }
    SK_PROBE(9);
    cluster_exit_barrier(relaxed_exit);
    SK_PROBE(10);
}

// ------------------------------------------------------------------ shgen

// One CTA per physical latitude: per order m the orthonormal associated
// Legendre recurrence (no Condon-Shortley phase, as std::assoc_legendre in
// tests/support/helpers.hpp:18-27) accumulates A_m = sum_l c_lm P_l^m and
// A_-m; the lambda synthesis is the inverse lambda transform (K4) applied to
// v_m = (A_m - i A_-m)/sqrt(2), v_0 = A_0.  An extended exponent keeps
// sin^m(theta) from underflowing at large m.
__global__ void __launch_bounds__(256) shgen_kernel(ShgenParams P) {
    const int p = blockIdx.x;
    const double th = 6.283185307179586476925286766559 * p / P.g.M;
    double sn, cs;
    sincos(th, &sn, &cs);
    const int L = P.L;
    const double big = 0x1p400, small = 0x1p-400;
    const double inv_sqrt2 = 0.70710678118654752440084436210484903928;
    for (int m = threadIdx.x; m <= P.g.N / 2; m += blockDim.x) {
        double Ap = 0.0, Am = 0.0;
        if (m <= L) {
            double pmm = 0.28209479177387814347403972578038629292;  // 1/sqrt(4 pi)
            int e = 0;
            for (int i = 1; i <= m; ++i) {
                pmm *= sqrt((2.0 * i + 1.0) / (2.0 * i)) * sn;
                if (pmm != 0.0 && fabs(pmm) < small) {
                    pmm *= big;
                    e -= 400;
                }
            }
            if (pmm != 0.0) {
                auto emit = [&](int l, double v) {
                    if (l >= 1) {
                        const double val = ldexp(v, e);
                        Ap = fma(P.coeffs[(long long)l * l + l + m], val, Ap);
                        if (m > 0) Am = fma(P.coeffs[(long long)l * l + l - m], val, Am);
                    }
                };
                double p2 = pmm;
                emit(m, p2);
                if (m < L) {
                    double p1 = sqrt(2.0 * m + 3.0) * cs * pmm;
                    emit(m + 1, p1);
                    const double m2 = static_cast<double>(m) * m;
                    for (int l = m + 2; l <= L; ++l) {
                        const double ll = l;
                        const double aa = sqrt((4.0 * ll * ll - 1.0) / (ll * ll - m2));
                        const double bb = sqrt(((ll - 1.0) * (ll - 1.0) - m2) / (4.0 * (ll - 1.0) * (ll - 1.0) - 1.0));
                        const double pl = aa * (cs * p1 - bb * p2);
                        p2 = p1;
                        p1 = pl;
                        if (fabs(p1) > big) {
                            p1 *= small;
                            p2 *= small;
                            e += 400;
                        }
                        emit(l, p1);
                    }
                }
            }
        }
        double2 v;
        if (m == 0) v = make_double2(Ap, 0.0);
        else v = make_double2(Ap * inv_sqrt2, -Am * inv_sqrt2);
        P.spec[static_cast<size_t>(m) * P.rows + p] = v;
    }
}

// --------------------------------------------------------- host launchers
// SK_PAIR_SYNC_EXIT=1: full cluster.sync() as the exit barrier (A/B)
int exit_relaxed() {
    static const int r = std::getenv("SK_PAIR_SYNC_EXIT") ? 0 : 1;
    return r;
}
template <bool SWZ, bool HI>
static cudaError_t launch_lambda_fwd_t(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem,
                                       cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(lambda_fwd_kernel<SWZ, HI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    lambda_fwd_kernel<SWZ, HI><<<P.rows_local * P.nrhs, nthr, smem, st>>>(P, map);
    return cudaGetLastError();
}
bool lambda_pair_ok(const LambdaParams& P, int nthr) {
    return !P.swizzle && !P.hiocc && P.nrhs == 1 && P.peers.n == 0 && nthr <= 256 &&
           P.fd.L / 2 + 1 <= kLamPairs * nthr;
}
bool lambda_quad_ok(const LambdaParams& P, int nthr) {
    return !P.swizzle && !P.hiocc && P.nrhs == 1 && nthr <= 256 && P.fd.L / 2 + 1 <= kLamPairs * nthr;
}
cudaError_t launch_lambda_fwd(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem, cudaStream_t st) {
    if (P.pair & 8) {  // row-major spectrum: the per-row kernel, contiguous stores
        if (P.hiocc)
            return P.swizzle ? launch_lambda_fwd_t<true, true>(P, map, nthr, smem, st)
                             : launch_lambda_fwd_t<false, true>(P, map, nthr, smem, st);
        return P.swizzle ? launch_lambda_fwd_t<true, false>(P, map, nthr, smem, st)
                         : launch_lambda_fwd_t<false, false>(P, map, nthr, smem, st);
    }
    if ((P.pair & 4) && lambda_quad_ok(P, nthr)) {
        static std::atomic<unsigned long long> attr{0};
        configure_on_device(attr, [] {
            cudaFuncSetAttribute(lambda_fwd_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        });
        lambda_fwd_quad_kernel<<<(P.rows_local + 3) & ~3, nthr, smem, st>>>(P, exit_relaxed());
        return cudaGetLastError();
    }
    if ((P.pair & 1) && lambda_pair_ok(P, nthr)) {
        static std::atomic<unsigned long long> attr{0};
        configure_on_device(attr, [] {
            cudaFuncSetAttribute(lambda_fwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        });
        lambda_fwd_pair_kernel<<<(P.rows_local + 1) & ~1, nthr, smem, st>>>(P, exit_relaxed());
        return cudaGetLastError();
    }
    if (P.hiocc)
        return P.swizzle ? launch_lambda_fwd_t<true, true>(P, map, nthr, smem, st)
                         : launch_lambda_fwd_t<false, true>(P, map, nthr, smem, st);
    return P.swizzle ? launch_lambda_fwd_t<true, false>(P, map, nthr, smem, st)
                     : launch_lambda_fwd_t<false, false>(P, map, nthr, smem, st);
}

template <bool SWZ, bool HI>
static cudaError_t launch_lambda_inv_t(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem,
                                       cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(lambda_inv_kernel<SWZ, HI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    lambda_inv_kernel<SWZ, HI><<<P.rows_local * P.nrhs, nthr, smem, st>>>(P, map);
    return cudaGetLastError();
}
bool lambda_inv_pair_ok(const LambdaParams& P, int nthr) {
    return lambda_pair_ok(P, nthr) && (P.fd.L / kBoxModes + 1) % 2 == 0;
}
cudaError_t launch_lambda_inv(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem, cudaStream_t st) {
    if ((P.pair & 2) && lambda_inv_pair_ok(P, nthr)) {  // map has 2-row boxes (make_spec_map box_rows = 2)
        static std::atomic<unsigned long long> attr{0};
        configure_on_device(attr, [] {
            cudaFuncSetAttribute(lambda_inv_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        });
        lambda_inv_pair_kernel<<<(P.rows_local + 1) & ~1, nthr, smem, st>>>(P, map);
        return cudaGetLastError();
    }
    if (P.hiocc)
        return P.swizzle ? launch_lambda_inv_t<true, true>(P, map, nthr, smem, st)
                         : launch_lambda_inv_t<false, true>(P, map, nthr, smem, st);
    return P.swizzle ? launch_lambda_inv_t<true, false>(P, map, nthr, smem, st)
                     : launch_lambda_inv_t<false, false>(P, map, nthr, smem, st);
}

template <bool SWZ, int CH, bool HI = false>
static cudaError_t launch_theta_t(const ThetaParams& P, const CUtensorMap& cmap, const CUtensorMap& ctail, int nthr,
                                  size_t smem, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(theta_kernel<SWZ, CH, HI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_kernel<SWZ, CH, HI>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    theta_kernel<SWZ, CH, HI><<<2 * P.ncols * P.nrhs, nthr, smem, st>>>(P, exit_relaxed(), cmap, ctail);
    return cudaGetLastError();
}

// cmap / ctail: the row-major spectrum as column-gather tensor maps (boxes of 256 rows / the tail box; read when P.gather)
cudaError_t launch_theta(const ThetaParams& P, const CUtensorMap& cmap, const CUtensorMap& ctail, int nthr, size_t smem,
                         cudaStream_t st) {
    const int ch = P.regsolve;  // chain solver chosen by the plan
    if (P.hiocc && ch == 1 && nthr <= 256)  // short columns (plan: radices <= 8, fixed-segment chains)
        return P.swizzle ? launch_theta_t<true, 1, true>(P, cmap, ctail, nthr, smem, st) : launch_theta_t<false, 1, true>(P, cmap, ctail, nthr, smem, st);
    if (P.swizzle) {
        if (ch == 2) return launch_theta_t<true, 2>(P, cmap, ctail, nthr, smem, st);
        if (ch == 1) return launch_theta_t<true, 1>(P, cmap, ctail, nthr, smem, st);
        return launch_theta_t<true, 0>(P, cmap, ctail, nthr, smem, st);
    }
    if (ch == 2) return launch_theta_t<false, 2>(P, cmap, ctail, nthr, smem, st);
    if (ch == 1) return launch_theta_t<false, 1>(P, cmap, ctail, nthr, smem, st);
    return launch_theta_t<false, 0>(P, cmap, ctail, nthr, smem, st);
}

cudaError_t launch_pivot_table(int L, int k0, int ncols, double* ipt, int stride, cudaStream_t st) {
    const int n = ncols * 4;
    pivot_table_kernel<<<(n + 127) / 128, 128, 0, st>>>(L, k0, ncols, ipt, stride);
    return cudaGetLastError();
}

cudaError_t launch_shgen(const ShgenParams& P, cudaStream_t st) {
    shgen_kernel<<<P.rows, 256, 0, st>>>(P);
    return cudaGetLastError();
}

}  // namespace sk
