// K1D / K4D lambda stages on row pairs inside ONE CTA (single RHS, rows that
// fit shared memory twice: C3's N/2 = 5000), sm_100a.
//
// Same job as lambda_fwd_kernel / lambda_inv_kernel (grid_kernels.cu: the row
// stage of analyze_2d fourier.cpp:181-187 with analyze_1d's (-1)^k / N
// :44-51, and the row stage of sample_grid fourier.cpp:201-207 with
// synthesize_1d's (-1)^k :61-62).  The spectrum is mode-major ([k][p]), so a
// row's modes are 16-byte entries a column apart; rows p and p+1 of one mode
// are adjacent.  Here the two halves of a 512-thread CTA transform rows p and
// p+1 side by side (the same plan in lockstep, one barrier sequence), so that
//   * the forward stores write (p, p+1) of a mode as one 32-byte segment from
//     adjacent lanes, both rows read from the CTA's own shared memory
//     (lambda_fwd_pair_kernel reads the peer row through DSMEM behind a
//     cluster barrier), and
//   * the inverse gathers 2-row x 256-mode boxes (32-byte segments: half the
//     TMA elements and whole sectors) into one [mode][row] buffer that both
//     halves read locally.
#include <cuda_runtime.h>

#include <atomic>

#include "fft_dev.cuh"
#include "params.h"
#include "sk_internal.h"
#include "tma.cuh"

namespace sk {

namespace {
constexpr int kBox = 256;    // modes per spectrum box (make_spec_map)
constexpr int kPairsD = 12;  // mode pairs (k, L-k) per thread held in registers
}  // namespace

__global__ void __launch_bounds__(512, 1) lambda_fwd_duo_kernel(LambdaParams P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = P.fd.L;
    const int Lpad = (L / kBox + 1) * kBox;
    double2* a0 = reinterpret_cast<double2*>(smem_raw);
    double2* a1 = a0 + Lpad;
    double2* s_hi = a1 + Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x, nh = nthr >> 1;
    const int h = tid >= nh ? 1 : 0, t = tid - h * nh;
    const int r0 = 2 * blockIdx.x;
    const int nlive = min(2, P.rows_local - r0);  // 1: the last CTA of an odd row count
    const bool live = h < nlive;
    double2* a = h ? a1 : a0;
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bar, static_cast<uint32_t>(nlive) * static_cast<uint32_t>(L) * 16);
        for (int r = 0; r < nlive; ++r)  // the real rows as N/2 complex pairs
            bulk_g2s_chunked(r ? a1 : a0, reinterpret_cast<const double2*>(P.f + static_cast<long long>(r0 + r) * P.g.N),
                             static_cast<uint32_t>(L) * 16, bar);
    }
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    for (int i = tid; i < L; i += nthr) s_rev[i] = __ldg(P.fd.rev + i);
    if (!live)
        for (int i = t; i < L; i += nh) a[i] = make_double2(0.0, 0.0);  // the half without a row transforms zeros
    __syncthreads();
    mbar_wait(bar, 0);
    fft_forward<false, 25>(a, P.fd, T, t, nh);  // block-wide barriers: both halves run the same stages
    const double invN = 1.0 / P.g.N;
    double2 vk[kPairsD], vm[kPairsD];
#pragma unroll
    for (int u = 0; u < kPairsD; ++u) {
        const int k = t + u * nh;
        if (k <= L / 2) {
            const int km = L - k;  // partner mode
            const double2 z = a[s_rev[k]];
            const double2 zp = a[s_rev[km == L ? 0 : km]];
            // A = (Z_k + conj Z_{L-k}) / 2,  B = -i (Z_k - conj Z_{L-k}) / 2
            const double2 A = make_double2(0.5 * (z.x + zp.x), 0.5 * (z.y - zp.y));
            const double2 B = make_double2(0.5 * (z.y + zp.y), -0.5 * (z.x - zp.x));
            const double2 Pk = cmul(T(k), B);  // T(L - k) = -conj T(k): X_{L-k} = conj(A - T(k) B)
            vk[u] = cscale(cadd(A, Pk), (k & 1) ? -invN : invN);
            vm[u] = cscale(conjd(csub(A, Pk)), (km & 1) ? -invN : invN);
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPairsD; ++u) {  // natural order, slots 0..L
        const int k = t + u * nh;
        if (k <= L / 2) {
            a[k] = vk[u];
            if (L - k != k) a[L - k] = vm[u];
        }
    }
    __syncthreads();
    // adjacent lanes write rows r0, r0+1 of one mode: 32-byte segments
    const int tot = 2 * (L + 1);
#pragma unroll 4
    for (int i = tid; i < tot; i += nthr) {
        const int k = i >> 1, sub = i & 1;
        const double2 v = (sub ? a1 : a0)[k];
        if (sub < nlive) P.spec[static_cast<size_t>(k) * P.rows_local + r0 + sub] = v;
    }
}

__global__ void __launch_bounds__(512, 1) lambda_inv_duo_kernel(LambdaParams P, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = P.fd.L;
    const int nb = L / kBox + 1;
    const int Lpad = nb * kBox;
    double2* a = reinterpret_cast<double2*>(smem_raw);  // [mode][row] boxes, then the two packed rows (a, a + Lpad)
    double2* s_hi = a + 2 * Lpad;
    double2* s_lo = s_hi + P.fd.nhi;
    int* s_rev = reinterpret_cast<int*>(s_lo + P.fd.nlo);
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_rev + ((L + 3) & ~3));
    const int tid = threadIdx.x, nthr = blockDim.x, nh = nthr >> 1;
    const int h = tid >= nh ? 1 : 0, t = tid - h * nh;
    const int r0 = 2 * blockIdx.x;
    const bool live = r0 + h < P.rows_local;
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t rb = static_cast<uint32_t>((L + 3) & ~3) * 4;  // rev table, padded to 16 bytes
        mbar_expect_tx(bar, static_cast<uint32_t>(nb) * kBox * 32 + (P.fd.nhi + P.fd.nlo) * 16 + rb);
        // boxes of 2 rows x 256 modes (row r0+1 past the last row and modes
        // past N/2 are zero-filled by the tensor map)
        for (int b = 0; b < nb; ++b) tma_load_3d(a + b * 2 * kBox, &tmap, 2 * r0, b * kBox, 0, bar);
        bulk_g2s_chunked(s_hi, P.fd.hi, P.fd.nhi * 16, bar);
        bulk_g2s_chunked(s_lo, P.fd.lo, P.fd.nlo * 16, bar);
        bulk_g2s_chunked(s_rev, P.fd.rev, rb, bar);
    }
    const Tw T{s_hi, s_lo, P.fd.shift, (1 << P.fd.shift) - 1};
    __syncthreads();
    mbar_wait(bar, 0);
    double2 zk[kPairsD], zm[kPairsD];
#pragma unroll
    for (int u = 0; u < kPairsD; ++u) {
        const int k = t + u * nh;
        if (k <= L / 2) {
            const int km = L - k;
            double2 v = a[2 * k + h];
            double2 w = a[2 * km + h];
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
    __syncthreads();  // every mode has been read: the buffer becomes the two packed rows
    double2* ah = a + h * Lpad;
#pragma unroll
    for (int u = 0; u < kPairsD; ++u) {
        const int k = t + u * nh;
        if (k <= L / 2) {
            const int km = L - k;
            ah[s_rev[k]] = zk[u];
            if (k != 0 && km != k) ah[s_rev[km]] = zm[u];
        }
    }
    __syncthreads();
    fft_inverse<false, 25>(ah, P.fd, T, t, nh);
    if (live) {
        double2* dst = reinterpret_cast<double2*>(P.u + static_cast<long long>(r0 + h) * P.g.N);
        for (int j = t; j < L; j += nh) dst[j] = ah[j];
    }
}

size_t lambda_duo_smem_bytes(int L, int nhi, int nlo) {
    const size_t lpad = static_cast<size_t>((L / kBox + 1) * kBox);
    return 2 * lpad * 16 + static_cast<size_t>(nhi + nlo) * 16 + static_cast<size_t>((L + 3) & ~3) * 4 + 32;
}

// nthr: threads per row (the plan's lambda thread count)
bool lambda_duo_ok(const LambdaParams& P, int nthr) {
    return !P.swizzle && !P.hiocc && P.nrhs == 1 && nthr <= 256 && nthr % 32 == 0 &&
           P.fd.L / 2 + 1 <= kPairsD * nthr && lambda_duo_smem_bytes(P.fd.L, P.fd.nhi, P.fd.nlo) <= 227 * 1024;
}

cudaError_t launch_lambda_fwd_duo(const LambdaParams& P, int nthr, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(lambda_fwd_duo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    lambda_fwd_duo_kernel<<<(P.rows_local + 1) / 2, 2 * nthr, lambda_duo_smem_bytes(P.fd.L, P.fd.nhi, P.fd.nlo), st>>>(P);
    return cudaGetLastError();
}

// map: spectrum map with 2-row boxes (make_spec_map box_rows = 2)
cudaError_t launch_lambda_inv_duo(const LambdaParams& P, const CUtensorMap& map, int nthr, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(lambda_inv_duo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    lambda_inv_duo_kernel<<<(P.rows_local + 1) / 2, 2 * nthr, lambda_duo_smem_bytes(P.fd.L, P.fd.nhi, P.fd.nlo), st>>>(P, map);
    return cudaGetLastError();
}

}  // namespace sk
