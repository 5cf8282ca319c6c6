// Multi-pass theta stage for columns too long for one CTA (C5: M/2 = 32768),
// sm_100a.  Same job as theta_kernel / theta_large_kernel (the column stage of
// analyze_2d fourier.cpp:174-180, Msin^2 poisson.cpp:61, solve
// poisson.cpp:121-161 with band_solve banded.cpp:101-158 /
// band_solve_with_dense_row :160-328, the column stage of sample_grid
// fourier.cpp:194-200), but streamed through HBM/L2 in five coalesced passes
// instead of one cluster holding a whole column in distributed shared memory:
//
//   TA  fold (e_r, o_r of both parities, fourier pole row as the reference
//       samples it) + four-step pass 1 of the forward length-L transforms:
//       L = L1 L2, r = r1 + L1 r2; L2-point DFTs over r2, twiddle w_L^(r1 t2)
//   TB  pass 2: L1-point DFTs over r1 -> X_tau, tau = t2 + L2 t1, natural order
//   TC  the chains of (lap - k^2) X = Msin^2 F along tau, on a 2-CTA cluster per
//       (mode, parity): chain+ by affine scans (segment totals exchanged
//       through DSMEM), chain- from it as x- = s x+ + Phi Delta (theta_sym.cu),
//       one pivot row per (mode, parity) (pivot_table_sym_kernel)
//   TD  inverse pass 1: L1-point inverse DFTs over t1, twiddle w_L^-(p1 t2)
//   TE  inverse pass 2: L2-point inverse DFTs over t2, the parity recombination
//       v_p = Ve_p + w_M^-p Vo_p, and the (peer) stores of the column.
//
// Each pass keeps 16 threads per sequence and 16 sequences per CTA of the
// in-shared-memory engine (fft_dev.cuh, all groups run the same plan in
// lockstep), and every HBM access is a 256- or 512-byte contiguous run.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "fft_dev.cuh"
#include "params.h"
#include "sk_internal.h"
#include "theta_common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace sk {

namespace {

// The FFT passes run 256-thread CTAs of 16 sequences x 16 threads at 64
// registers (register radices <= 8) so that several CTAs share an SM; the
// chain pass runs 8-CTA clusters of 256 threads (several per SM).
constexpr int kThr = 256;  // threads per CTA of the FFT passes
constexpr int kSeqs = 16;  // sequences per CTA
constexpr int kGrp = 16;   // threads per sequence
constexpr int kBlkR = 8;   // r1 / p1 per CTA in TA / TE (two parities -> 16 sequences)
constexpr int kLgR = 3;    // log2 kBlkR
constexpr int kBlkT = 16;  // t2 per CTA in TB / TD
constexpr int kLgT = 4;    // log2 kBlkT
// chain elements per thread in TC: ODD, so that a warp's per-element accesses
// to the CTA's staged X (16 B) and pivots (8 B), a segment apart from lane to
// lane, rotate through the bank groups (with 8 every lane hit the same one:
// 32-way conflicts, the shared-memory pipe was TC's bound)
#ifndef SK_TC_SEG
#define SK_TC_SEG 9
#define SK_TC_THR 256
#endif
constexpr int kSeg = SK_TC_SEG;
#ifndef SK_TC_MINB
#define SK_TC_MINB 2  // CTAs per SM the chain pass is compiled for (A/B: 3 spills at 80 registers)
#endif
constexpr int kCq = 8;     // CTAs per TC cluster (portable maximum)
constexpr int kCthr = SK_TC_THR; // threads per TC CTA
// A CTA's sequences sit L + kPad slots apart in shared memory: the tile loads
// and stores of every pass walk the SEQUENCE index fastest (8 or 16
// neighbouring lanes, the contiguous direction in HBM), and with a stride of
// L slots (a multiple of 128 bytes) those lanes all hit one bank group (ncu:
// shared-memory pipe 80-92 % busy, short-scoreboard stalls on top); one slot
// of padding rotates consecutive sequences through the eight bank groups.
constexpr int kPad = 1;

// raw column element p of column c (rhs-major) in the (slab) spectrum layout
__device__ __forceinline__ double2* raw_ptr(const ThetaParams& P, int c, int p) {
    const int rhs = c / P.ncols, kl = c - rhs * P.ncols;
    return P.buf + rhs * P.rhs_stride + theta_addr(P.sl, P.ncols, kl, p);
}
// Column accessor: one rank's column is contiguous (rows of mode kl), several
// ranks' pieces go through theta_addr
struct ColRef {
    double2* base;  // P.sl.P == 1: element p at base[p]
    const ThetaParams* P;
    int c;
    __device__ __forceinline__ double2& operator[](int p) const { return P->sl.P == 1 ? base[p] : *raw_ptr(*P, c, p); }
};
__device__ __forceinline__ ColRef col_ref(const ThetaParams& P, int c) {
    const int rhs = c / P.ncols, kl = c - rhs * P.ncols;
    return ColRef{P.buf + rhs * P.rhs_stride + static_cast<size_t>(kl) * P.g.rows, &P, c};
}
__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }  // v a power of two

}  // namespace

// ----------------------------------------------------------------- TA
__global__ void __launch_bounds__(kThr, 3) theta_mp_a_kernel(ThetaMpParams Q) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const ThetaParams& P = Q.t;
    const int L = P.fd.L, L1 = Q.f1.L, L2 = Q.f2.L;
    const int nb = L1 / kBlkR;
    const int S2 = L2 + kPad;
    double2* a = reinterpret_cast<double2*>(smem_raw);  // 16 sequences of L2 (par * 8 + q), S2 slots apart
    double2* t2hi = a + kSeqs * S2;
    double2* t2lo = t2hi + Q.f2.nhi;
    double2* tmhi = t2lo + Q.f2.nlo;  // 2L-th roots (the theta plan's table)
    double2* tmlo = tmhi + P.fd.nhi;
    int* rev2 = reinterpret_cast<int*>(tmlo + P.fd.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = blockIdx.x / nb, b = blockIdx.x - c * nb;
    const int kg = P.k0 + (c % P.ncols);
    const double sgn = (kg & 1) ? -1.0 : 1.0;
    const Tw T2 = load_tw(Q.f2, t2hi, t2lo, tid, nthr);
    const Tw TM = load_tw(P.fd, tmhi, tmlo, tid, nthr);
    for (int i = tid; i < L2; i += nthr) rev2[i] = __ldg(Q.f2.rev + i);
    __syncthreads();
    const double invM = 1.0 / P.g.M;
    const ColRef cr = col_ref(P, c);
    // fold: element (q, r2) of this block, r = r1 + L1 r2, r1 = kBlkR b + q.
    // A thread keeps its q and walks r2 in steps of kThr / kBlkR, so the
    // fold's twiddle T(r) advances by a constant factor per trip (one table
    // lookup per thread instead of one per element: the passes are bound by
    // the shared-memory pipe, profiles/r2_c5_mp_launches.md).
    constexpr int kR2Step = kThr / kBlkR;
    {
        const int q = tid & (kBlkR - 1);
        const int r1 = kBlkR * b + q;
        double2 wf = TM(r1 + L1 * (tid >> kLgR));
        const double2 Wf = TM(kR2Step * L1);  // < 2L: L2 >= 32
#pragma unroll 8
        for (int r2 = tid >> kLgR; r2 < L2; r2 += kR2Step) {
            const int r = r1 + L1 * r2;
            double2 ar = cr[r];
            const double2 am = cr[L - r];  // a_L for r = 0
            if (r == 0 && P.g.pole_glide) ar = cscale(ar, sgn);  // sk_internal.h GridGeom::pole_glide
            const double2 ev = make_double2((ar.x + sgn * am.x) * invM, (ar.y + sgn * am.y) * invM);
            const double2 od = cscale(cmul(make_double2(ar.x - sgn * am.x, ar.y - sgn * am.y), wf), invM);
            a[q * S2 + swz<true>(r2)] = ev;
            a[(kBlkR + q) * S2 + swz<true>(r2)] = od;
            wf = cmul(wf, Wf);
        }
    }
    __syncthreads();
    const int seq = tid / kGrp, g = tid - seq * kGrp;
    fft_forward<true, 8>(a + seq * S2, Q.f2, T2, g, kGrp);  // t2 at slot swz(rev2[t2])
    // twiddle w_L^(r1 t2) = T(2 r1 t2) and the store of (par, t2, r1): both
    // parities of a (t2, r1) share the twiddle, which advances by T(2 r1
    // kR2Step) per trip
    {
        const int q = tid & (kBlkR - 1);
        const int r1 = kBlkR * b + q;
        double2 wt = TM(2 * r1 * (tid >> kLgR));  // 2 r1 t2 < 2 L1 L2 = 2L: no reduction
        const double2 Wt = TM(2 * kR2Step * r1);  // < 2L: r1 < L1, L2 >= 32
        for (int t2 = tid >> kLgR; t2 < L2; t2 += kR2Step) {
            const int sl = swz<true>(rev2[t2]);
#pragma unroll
            for (int par = 0; par < 2; ++par) {
                const double2 v = a[(par * kBlkR + q) * S2 + sl];
                Q.w1[((static_cast<size_t>(c) * 2 + par) * L2 + t2) * L1 + r1] = cmul(v, wt);
            }
            wt = cmul(wt, Wt);
        }
    }
}

// ----------------------------------------------------------------- TB
__global__ void __launch_bounds__(kThr, 3) theta_mp_b_kernel(ThetaMpParams Q) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const ThetaParams& P = Q.t;
    const int L = P.fd.L, L1 = Q.f1.L, L2 = Q.f2.L;
    const int nb = L2 / kBlkT;
    const int S1 = L1 + kPad;
    double2* a = reinterpret_cast<double2*>(smem_raw);  // 16 sequences of L1, S1 slots apart
    double2* t1hi = a + kSeqs * S1;
    double2* t1lo = t1hi + Q.f1.nhi;
    int* rev1 = reinterpret_cast<int*>(t1lo + Q.f1.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int cp = blockIdx.x / nb, b = blockIdx.x - cp * nb;  // cp = 2 c + par
    const Tw T1 = load_tw(Q.f1, t1hi, t1lo, tid, nthr);
    for (int i = tid; i < L1; i += nthr) rev1[i] = __ldg(Q.f1.rev + i);
    const double2* src = Q.w1 + static_cast<size_t>(cp) * L2 * L1;
    const int lg1 = ilog2(L1);
#pragma unroll 8
    for (int e = tid; e < kBlkT * L1; e += nthr) {
        const int r1 = e & (L1 - 1), q = e >> lg1;
        a[q * S1 + swz<true>(r1)] = src[static_cast<size_t>(kBlkT * b + q) * L1 + r1];
    }
    __syncthreads();
    const int seq = tid / kGrp, g = tid - seq * kGrp;
    fft_forward<true, 8>(a + seq * S1, Q.f1, T1, g, kGrp);
    double2* dst = Q.w2 + static_cast<size_t>(cp) * L;
    for (int e = tid; e < kBlkT * L1; e += nthr) {
        const int q = e & (kBlkT - 1), t1 = e >> kLgT;
        dst[static_cast<size_t>(t1) * L2 + kBlkT * b + q] = a[q * S1 + swz<true>(rev1[t1])];
    }
}

// ----------------------------------------------------------------- TC
// Cluster of kCq CTAs per (column, parity); CTA h owns chain+ elements
// [h H, h H + H) (H = kCthr kSeg) in shared memory with one neighbour either side.
__global__ void __cluster_dims__(kCq, 1, 1) __launch_bounds__(kCthr, SK_TC_MINB) theta_mp_c_kernel(ThetaMpParams Q, int relaxed_exit) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const ThetaParams& P = Q.t;
    const int L = P.fd.L;
    constexpr int H = kCthr * kSeg;
    double2* x = reinterpret_cast<double2*>(smem_raw);  // x[1 + j] = X+ of element h H + j, x[0], x[H + 1] the neighbours
    double* ip = reinterpret_cast<double*>(x + H + 2);  // ip[j] = pivot of element h H + j
    Aff3* wsc = reinterpret_cast<Aff3*>(ip + H + 2);    // 2 x 16 scan slots
    double2* misc = reinterpret_cast<double2*>(wsc + 32);
    double* red = reinterpret_cast<double*>(misc + 16);
    uint64_t* bar = reinterpret_cast<uint64_t*>(red + 64);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int h = static_cast<int>(cluster.block_rank());
    const int cp = blockIdx.x / kCq;
    const int c = cp >> 1, par = cp & 1;
    const int rhs = c / P.ncols, kl = c - rhs * P.ncols;
    const int kg = P.k0 + kl;
    const double k2 = static_cast<double>(kg) * static_cast<double>(kg);
    const double sgn = (kg & 1) ? -1.0 : 1.0;
    const int n = par == 0 ? L / 2 - 1 : L / 2;  // chain+ length
    const int tau0 = par == 0 ? 1 : 0;
    const double t0 = par == 0 ? 2.0 : 1.0;
    double2* col = Q.w2 + static_cast<size_t>(cp) * L;
    const double* prow = P.pivots + (static_cast<size_t>(kl) * 2 + par) * P.piv_stride;
    const int i0 = h * H, i1 = min(n, i0 + H);  // this CTA's elements
    const bool active = i0 < n;                 // (a short chain leaves CTA 1 without elements)
    // ---- loads: X at tau0 + [i0 - 1, i1 + 1), pivots [i0, i1 + 1)
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int xlo_i = max(i0 - 1, 0);  // first element loaded
    const int x_hi = min(i1 + 1, n);   // one past the last element loaded
    const int xcnt = x_hi - xlo_i;
    const int pcnt = min(i1 + 1, n + 1) - i0;  // par 1 reads entry n (chain-'s last pivot) too
    if (active && tid == 0) {
        const uint32_t xb = static_cast<uint32_t>(xcnt) * 16;
        const size_t pa0 = (reinterpret_cast<uintptr_t>(prow + i0) & 15) ? 1 : 0;  // 16-byte aligned bulk source
        const uint32_t pb = static_cast<uint32_t>(((pcnt + pa0 + 1) & ~1)) * 8;
        mbar_expect_tx(bar, xb + pb);
        bulk_g2s_chunked(x + 1 + (xlo_i - i0), col + tau0 + xlo_i, xb, bar);
        bulk_g2s_chunked(ip - pa0, prow + i0 - pa0, pb, bar);
    }
    // scalars of the rows outside the chain+ range (global reads)
    double2 inner = make_double2(0.0, 0.0), XmL = make_double2(0.0, 0.0), Xm_last = make_double2(0.0, 0.0),
            Xm_last2 = make_double2(0.0, 0.0), Xm2 = make_double2(0.0, 0.0);
    const double2 X0 = col[0];
    if (par == 0) {
        inner = X0;                        // X_0: inner neighbour of chain+
        Xm2 = col[L - 1];                  // X_{-2}
        XmL = col[L / 2];                  // X_{-L}
        Xm_last = col[L - 1 - (n - 1)];    // chain- element n-1 (t = -(L-2))
        Xm_last2 = col[L - 1 - (n - 2)];   // chain- element n-2
    } else {
        inner = col[L - 1];                // X_{-1}: inner neighbour of chain+
        Xm_last = col[L - 1 - (n - 1)];    // chain- element n-1 (t = -(L-1))
        Xm_last2 = col[L - 1 - (n - 2)];
    }
    if (active) mbar_wait(bar, 0);
    if (tid == 0) misc[8] = misc[9] = make_double2(0.0, 0.0);
    if (active && tid == 0) {
        if (i0 == 0) x[0] = inner;  // neighbour of element 0
        if (i1 >= n) x[1 + (i1 - i0)] = make_double2(0.0, 0.0);  // past the chain end
        if (par == 0 && h == 0) {
            // row j = 0 data before the chain overwrites X_2: F_0 = 1/2 X_0 - (X_{-2} + X_2)/4
            const double2 X2 = x[1];
            misc[7] = make_double2(0.5 * X0.x - 0.25 * (Xm2.x + X2.x), 0.5 * X0.y - 0.25 * (Xm2.y + X2.y));
        }
    }
    __syncthreads();
    // k = 0, even class: surface mean 2 pi w^T X_0 (poisson.cpp:101-117)
    double* st = P.stats + 4 * rhs;
    const bool want_wsum = (kg == 0 && par == 0);
    if (want_wsum) {
        double2 acc = make_double2(0.0, 0.0);
        for (int j = tid; j < i1 - i0; j += nthr) {
            const double t = t0 + 2.0 * (i0 + j);
            const double w = 2.0 / (1.0 - t * t);
            acc.x = fma(2.0 * w, x[1 + j].x, acc.x);
            acc.y = fma(2.0 * w, x[1 + j].y, acc.y);
        }
        if (h == 0 && tid == 0) {
            const double Ld = L;
            const double wl = 2.0 / (1.0 - Ld * Ld);
            acc.x += 2.0 * X0.x + wl * XmL.x;
            acc.y += 2.0 * X0.y + wl * XmL.y;
        }
        acc = block_sum2(acc, red);
        if (tid == 0) misc[8] = acc;
    }
    // ---- the chain+ solve (theta_sym.cu solve_chains_sym, segment-local positions)
    const int s = i0 + tid * kSeg;  // first element of this thread
    const double t_s = t0 + 2.0 * s;
    double2 v[kSeg];
    double ipv[kSeg];
#pragma unroll
    for (int u = 0; u < kSeg; ++u) {
        const bool ok = s + u < i1;
        v[u] = ok ? x[1 + s + u - i0] : make_double2(0.0, 0.0);
        ipv[u] = ok ? ip[s + u - i0] : 0.0;
    }
    const bool any = s < i1;
    const double2 xlo = any ? x[s - i0] : make_double2(0.0, 0.0);
    const double2 xhi = (s + kSeg < n) ? x[1 + s + kSeg - i0] : make_double2(0.0, 0.0);
    const double ip_before = (any && s > 0) ? ((s - 1 >= i0) ? ip[s - 1 - i0] : __ldg(prow + s - 1)) : 0.0;
    const int ulast = n - 1 - s;
    const double tl = static_cast<double>(L - 1);
    unsigned fh = 0u;
    Aff3 aff = aff_identity();
    double2 xlast = make_double2(0.0, 0.0), xlast_m = make_double2(0.0, 0.0);
    {
        double2 xm = xlo;
        double ipp = ip_before;
        double t = t_s;
#pragma unroll
        for (int u = 0; u < kSeg; ++u) {
            const double2 x0 = v[u];
            const double2 xp = (u + 1 < kSeg) ? v[u + 1] : xhi;
            if (u == ulast) {
                xlast = x0;
                xlast_m = xm;
            }
            const double d2 = (t == tl) ? 0.25 : 0.5;
            double2 F = make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
            if (s + u >= i1) F = make_double2(0.0, 0.0);
            fh = max(fh, static_cast<unsigned>(__double2hiint(fma(F.x, F.x, F.y * F.y))));
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);
            aff = Aff3{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y)};
            v[u] = F;
            ipp = ipv[u];
            xm = x0;
            t += 2.0;
        }
    }
    // forward scan within the CTA, then across the pair (CTA 0's elements first)
    Aff3 rin = block_scan_aff1<false>(aff, wsc);
    {
        // CTA total = last thread's exclusive prefix composed with its own map
        if (tid == nthr - 1) {
            const Aff3 tot = aff_combine(rin, aff);
            reinterpret_cast<Aff3*>(misc + 10)[0] = tot;
        }
        cluster.sync();
        if (h > 0) {
            // the totals of the CTAs before this one: all remote loads issue
            // together (one DSMEM latency), then the ordered composition
            Aff3 tot[kCq - 1];
#pragma unroll
            for (int o = 0; o < kCq - 1; ++o)
                tot[o] = reinterpret_cast<const Aff3*>(cluster.map_shared_rank(misc + 10, o < h ? o : 0))[0];
            Aff3 pre = tot[0];
#pragma unroll
            for (int o = 1; o < kCq - 1; ++o)
                if (o < h) pre = aff_combine(pre, tot[o]);
            rin = aff_combine(pre, rin);
        }
    }
    Aff3 baff;
    double2 rlast = make_double2(0.0, 0.0);
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
        double t = t_s;
        double Pm = 1.0;
        double2 G = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < kSeg; ++u) {
            const bool ok = s + u < i1;
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);
            rp = make_double2(fma(al, rp.x, v[u].x), fma(al, rp.y, v[u].y));
            if (u == ulast) rlast = rp;
            const double iv = ipv[u];
            const double2 gg = make_double2(rp.x * iv, rp.y * iv);
            double cc = (-0.25 * iv) * fma(t, t + 3.0, 2.0);
            if (u == ulast || !ok) cc = 1.0;
            G = make_double2(fma(Pm, gg.x, G.x), fma(Pm, gg.y, G.y));
            Pm *= cc;
            v[u] = gg;
            ipv[u] = cc;
            ipp = iv;
            t += 2.0;
        }
        baff = Aff3{Pm, G.x, G.y};
    }
    // the boundary rows (theta_sym.cu; chain- values read directly here)
    if (ulast >= 0 && ulast < kSeg) {
        const double ipl = ip[n - 1 - i0];
        const double2 xp_last = make_double2(rlast.x * ipl, rlast.y * ipl);
        double2 xm_last, xm_extra = make_double2(0.0, 0.0);
        unsigned fb = 0u;
        const double2 Fp = make_double2((par ? 0.25 : 0.5) * xlast.x - 0.25 * xlast_m.x,
                                        (par ? 0.25 : 0.5) * xlast.y - 0.25 * xlast_m.y);  // F+_{n-1}
        if (par == 0) {
            const double Ld = L;
            const double2 Fm1 = make_double2(0.5 * Xm_last.x - 0.25 * (Xm_last2.x + XmL.x),
                                             0.5 * Xm_last.y - 0.25 * (Xm_last2.y + XmL.y));
            const double2 rm1 = make_double2(sgn * rlast.x + (Fm1.x - sgn * Fp.x), sgn * rlast.y + (Fm1.y - sgn * Fp.y));
            const double2 Fn = make_double2(0.25 * (XmL.x - Xm_last.x), 0.25 * (XmL.y - Xm_last.y));
            const double An = 0.25 * (Ld - 2.0) * (Ld - 1.0);
            const double Cm = 0.25 * Ld * (Ld - 1.0);
            const double al = -An * ipl;
            const double2 rn = make_double2(fma(al, rm1.x, Fn.x), fma(al, rm1.y, Fn.y));
            const double ipn = ip[n - i0];
            xm_extra = make_double2(rn.x * ipn, rn.y * ipn);
            const double be = -Cm * ipl;
            xm_last = make_double2(fma(be, xm_extra.x, rm1.x * ipl), fma(be, xm_extra.y, rm1.y * ipl));
            fb = max(static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y))),
                     static_cast<unsigned>(__double2hiint(fma(Fn.x, Fn.x, Fn.y * Fn.y))));
        } else {
            const double2 Fm1 = make_double2(0.5 * Xm_last.x - 0.25 * Xm_last2.x, 0.5 * Xm_last.y - 0.25 * Xm_last2.y);
            const double2 rm1 = make_double2(sgn * rlast.x + (Fm1.x - sgn * Fp.x), sgn * rlast.y + (Fm1.y - sgn * Fp.y));
            const double ipm = ip[n - i0];
            xm_last = make_double2(rm1.x * ipm, rm1.y * ipm);
            fb = static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y)));
        }
        fh = max(fh, fb);
        misc[5] = make_double2(xm_last.x - sgn * xp_last.x, xm_last.y - sgn * xp_last.y);  // Delta
        misc[6] = xm_extra;
    }
    // backward scan within the CTA, then across the pair (CTA 1's elements first)
    Aff3 xin = block_scan_aff1<true>(baff, wsc + 16);
    if (tid == 0) {
        const Aff3 tot = aff_combine(xin, baff);
        reinterpret_cast<Aff3*>(misc + 12)[0] = tot;
    }
    cluster.sync();
    const int owner = (n - 1) / H;  // CTA holding the last element (Delta)
    const double2 Dl = cluster.map_shared_rank(misc, owner)[5];
    if (h < kCq - 1) {
        Aff3 tot[kCq - 1];  // tot[j]: total of CTA kCq - 1 - j (loads issued together, as above)
#pragma unroll
        for (int j = 0; j < kCq - 1; ++j) {
            const int o = kCq - 1 - j;
            tot[j] = reinterpret_cast<const Aff3*>(cluster.map_shared_rank(misc + 12, o > h ? o : kCq - 1))[0];
        }
        Aff3 pre = tot[0];
#pragma unroll
        for (int j = 1; j < kCq - 1; ++j)
            if (kCq - 1 - j > h) pre = aff_combine(pre, tot[j]);
        xin = aff_combine(pre, xin);
    }
    double2 xr = make_double2(xin.b, xin.c);
    double phi = xin.a;
    double2 ws = make_double2(0.0, 0.0);
    double2 xf_p = make_double2(0.0, 0.0), xf_m = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = kSeg - 1; u >= 0; --u) {
        if (s + u < i1) {
            const double cc = ipv[u];
            const double2 gg = v[u];
            if (u != ulast) xr = make_double2(fma(cc, xr.x, gg.x), fma(cc, xr.y, gg.y));
            else xr = gg;
            phi *= cc;
            const double2 xm = make_double2(fma(phi, Dl.x, sgn * xr.x), fma(phi, Dl.y, sgn * xr.y));
            x[1 + s + u - i0] = xr;  // own element (no other thread reads it any more)
            v[u] = xm;                // chain- element, stored below
            if (want_wsum) {
                const double t = t_s + 2.0 * u;
                const double w = 2.0 / (1.0 - t * t);
                ws.x = fma(w, xr.x + xm.x, ws.x);
                ws.y = fma(w, xr.y + xm.y, ws.y);
            }
            xf_p = xr;
            xf_m = xm;
        }
    }
    if (par == 0 && ulast >= 0 && ulast < kSeg) {
        const double2 xe = misc[6];
        col[L / 2] = xe;  // x at t = -L
        if (want_wsum) {
            const double Ld = L;
            const double w = 2.0 / (1.0 - Ld * Ld);
            ws.x = fma(w, xe.x, ws.x);
            ws.y = fma(w, xe.y, ws.y);
        }
    }
    if (h == 0 && tid == 0) {
        misc[3] = xf_p;
        misc[4] = xf_m;
    }
    __syncthreads();
    // chain+ then chain- back to HBM as contiguous runs through shared memory
    for (int j = tid; j < i1 - i0; j += nthr) col[tau0 + i0 + j] = x[1 + j];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kSeg; ++u)
        if (s + u < i1) x[1 + s + u - i0] = v[u];
    __syncthreads();
    for (int j = tid; j < i1 - i0; j += nthr) col[L - 1 - (i0 + j)] = x[1 + j];
    // statistics, row j = 0 / constraint
    const double fm = sqrt(block_max(__hiloint2double(static_cast<int>(fh), 0), red));
    if (want_wsum) {
        ws = block_sum2(ws, red);
        if (tid == 0) misc[9] = ws;
    }
    // only the k = 0 constraint needs the other CTAs' sums; otherwise x_0 comes
    // from CTA 0's own values and the cluster meets again only to keep every
    // CTA's shared memory alive until the peers' DSMEM reads above are done
    if (kg == 0) cluster.sync();
    if (h == 0 && tid == 0) {
        double fmx = fm;
        if (par == 0) {
            const double2 xp2 = misc[3], xm2 = misc[4];
            const double2 F0 = misc[7];
            double2 x0;
            if (kg != 0) {
                x0 = make_double2((F0.x - 0.5 * xm2.x - 0.5 * xp2.x) / (-k2), (F0.y - 0.5 * xm2.y - 0.5 * xp2.y) / (-k2));
            } else {
                double2 w2 = make_double2(0.0, 0.0), m2 = make_double2(0.0, 0.0);
                for (int o = 0; o < kCq; ++o) {
                    const double2 w1 = cluster.map_shared_rank(misc, o)[9];
                    const double2 m1 = cluster.map_shared_rank(misc, o)[8];
                    w2.x += w1.x;
                    w2.y += w1.y;
                    m2.x += m1.x;
                    m2.y += m1.y;
                }
                x0 = make_double2(-0.5 * w2.x, -0.5 * w2.y);
                const double twopi = 6.283185307179586476925286766559;
                st[0] = twopi * m2.x;
                st[1] = twopi * m2.y;
            }
            col[0] = x0;
            fmx = fmax(fmx, hypot(F0.x, F0.y));
        }
        atomic_max_nonneg(st + 2, fmx);
    } else if (tid == 0) {
        atomic_max_nonneg(st + 2, fm);
    }
    // exit: only consumed DSMEM loads since the last cluster barrier
    // (theta_common.cuh cluster_exit_barrier's contract)
    cluster_exit_barrier(relaxed_exit);
}

// X_half export of the multi-pass path: X(t) of column c at t = t_of(tau, par) + L
__global__ void theta_mp_export_kernel(ThetaMpParams Q) {
    const ThetaParams& P = Q.t;
    const int L = P.fd.L;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long per = 2LL * L;
    if (idx >= per * P.ncols * P.nrhs) return;
    const int c = static_cast<int>(idx / per);
    const int par = static_cast<int>((idx / L) & 1), tau = static_cast<int>(idx % L);
    const int rhs = c / P.ncols, kg = P.k0 + (c - rhs * P.ncols);
    double2* xo = P.xhalf + static_cast<long long>(rhs) * (P.g.N / 2 + 1) * P.g.M + static_cast<long long>(kg) * P.g.M;
    xo[t_of(tau, par, L) + L] = Q.w2[idx];
}

// ----------------------------------------------------------------- TD
__global__ void __launch_bounds__(kThr, 3) theta_mp_d_kernel(ThetaMpParams Q) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const ThetaParams& P = Q.t;
    const int L = P.fd.L, L1 = Q.f1.L, L2 = Q.f2.L;
    const int nb = L2 / kBlkT;
    const int S1 = L1 + kPad;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* t1hi = a + kSeqs * S1;
    double2* t1lo = t1hi + Q.f1.nhi;
    double2* tmhi = t1lo + Q.f1.nlo;
    double2* tmlo = tmhi + P.fd.nhi;
    int* rev1 = reinterpret_cast<int*>(tmlo + P.fd.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int cp = blockIdx.x / nb, b = blockIdx.x - cp * nb;
    const Tw T1 = load_tw(Q.f1, t1hi, t1lo, tid, nthr);
    const Tw TM = load_tw(P.fd, tmhi, tmlo, tid, nthr);
    for (int i = tid; i < L1; i += nthr) rev1[i] = __ldg(Q.f1.rev + i);
    __syncthreads();
    const double2* src = Q.w2 + static_cast<size_t>(cp) * L;
#pragma unroll 8
    for (int e = tid; e < kBlkT * L1; e += nthr) {
        const int q = e & (kBlkT - 1), t1 = e >> kLgT;
        a[q * S1 + swz<true>(rev1[t1])] = src[static_cast<size_t>(t1) * L2 + kBlkT * b + q];  // DIT input order
    }
    __syncthreads();
    const int seq = tid / kGrp, g = tid - seq * kGrp;
    fft_inverse<true, 8>(a + seq * S1, Q.f1, T1, g, kGrp);  // natural p1
    double2* dst = Q.w1 + static_cast<size_t>(cp) * L1 * L2;
    {
        // w_L^-(p1 t2) = conj T(2 p1 t2): a thread keeps its t2 and walks p1 in
        // steps of kThr / kBlkT, the twiddle advancing by T(2 t2 step) per trip
        constexpr int kP1Step = kThr / kBlkT;
        const int q = tid & (kBlkT - 1);
        const int t2 = kBlkT * b + q;
        double2 wt = TM(2 * (tid >> kLgT) * t2);  // < 2L
        const double2 Wt = TM(2 * kP1Step * t2);  // < 2L: t2 < L2, L1 >= 16
        for (int p1 = tid >> kLgT; p1 < L1; p1 += kP1Step) {
            dst[static_cast<size_t>(p1) * L2 + t2] = cmulc(a[q * S1 + swz<true>(p1)], wt);
            wt = cmul(wt, Wt);
        }
    }
}

// ----------------------------------------------------------------- TE
__global__ void __launch_bounds__(kThr, 3) theta_mp_e_kernel(ThetaMpParams Q) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const ThetaParams& P = Q.t;
    const int L = P.fd.L, L1 = Q.f1.L, L2 = Q.f2.L;
    const int nb = L1 / kBlkR;
    const int S2 = L2 + kPad;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* t2hi = a + kSeqs * S2;
    double2* t2lo = t2hi + Q.f2.nhi;
    double2* tmhi = t2lo + Q.f2.nlo;
    double2* tmlo = tmhi + P.fd.nhi;
    int* rev2 = reinterpret_cast<int*>(tmlo + P.fd.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = blockIdx.x / nb, b = blockIdx.x - c * nb;
    const int kg = P.k0 + (c % P.ncols);
    const Tw T2 = load_tw(Q.f2, t2hi, t2lo, tid, nthr);
    const Tw TM = load_tw(P.fd, tmhi, tmlo, tid, nthr);
    for (int i = tid; i < L2; i += nthr) rev2[i] = __ldg(Q.f2.rev + i);
    __syncthreads();
    const int lg2 = ilog2(L2);
#pragma unroll 8
    for (int e = tid; e < 2 * kBlkR * L2; e += nthr) {
        const int t2 = e & (L2 - 1), q = (e >> lg2) & (kBlkR - 1), par = e >> (lg2 + kLgR);
        const int p1 = kBlkR * b + q;
        a[(par * kBlkR + q) * S2 + swz<true>(rev2[t2])] =
            Q.w1[((static_cast<size_t>(c) * 2 + par) * L1 + p1) * L2 + t2];
    }
    __syncthreads();
    const int seq = tid / kGrp, g = tid - seq * kGrp;
    fft_inverse<true, 8>(a + seq * S2, Q.f2, T2, g, kGrp);  // natural p2
    // v_p = Ve_p + w_M^-p Vo_p, p = p1 + L1 p2 (and p = L = Ve_0 - Vo_0 from p1 = 0)
    const ColRef cr = col_ref(P, c);
    {
        // a thread keeps its p1 and walks p2; T(p) advances by T(L1 step) per trip
        constexpr int kP2Step = kThr / kBlkR;
        const int q = tid & (kBlkR - 1);
        const int p1 = kBlkR * b + q;
        double2 wp = TM(p1 + L1 * (tid >> kLgR));
        const double2 Wp = TM(kP2Step * L1);  // < 2L: L2 >= 32
        for (int p2 = tid >> kLgR; p2 < L2; p2 += kP2Step) {
            const int p = p1 + L1 * p2;
            const double2 ve = a[q * S2 + swz<true>(p2)];
            const double2 vo = a[(kBlkR + q) * S2 + swz<true>(p2)];
            const double2 v = cadd(ve, cmulc(vo, wp));
            if (P.peers.n) *peer_ptr(P.peers, p, kg, p) = v;  // fused return transpose
            else cr[p] = v;
            wp = cmul(wp, Wp);
        }
        if (tid == 0 && b == 0) {  // p = L (theta = pi): Ve_0 - Vo_0, T(L) = -1
            const double2 ve = a[swz<true>(0)];
            const double2 vo = a[kBlkR * S2 + swz<true>(0)];
            const double2 v = cadd(ve, cmulc(vo, TM(L)));
            if (P.peers.n) *peer_ptr(P.peers, L, kg, L) = v;
            else cr[L] = v;
        }
    }
}

size_t theta_mp_smem_bytes(int which, int L1, int L2, int nhi1, int nlo1, int nhi2, int nlo2, int nhiM, int nloM) {
    switch (which) {
        case 0:  // TA / TE
            return static_cast<size_t>(kSeqs) * (L2 + kPad) * 16 + static_cast<size_t>(nhi2 + nlo2 + nhiM + nloM) * 16 +
                   static_cast<size_t>(L2) * 4;
        case 1:  // TB
            return static_cast<size_t>(kSeqs) * (L1 + kPad) * 16 + static_cast<size_t>(nhi1 + nlo1) * 16 +
                   static_cast<size_t>(L1) * 4;
        case 2:  // TD
            return static_cast<size_t>(kSeqs) * (L1 + kPad) * 16 + static_cast<size_t>(nhi1 + nlo1 + nhiM + nloM) * 16 +
                   static_cast<size_t>(L1) * 4;
        default:  // TC
            return static_cast<size_t>(kCthr * kSeg + 2) * 16 + static_cast<size_t>(kCthr * kSeg + 2 + 2) * 8 + 32 * 24 +
                   16 * 16 + 64 * 8 + 16;
    }
}

// chain+ elements a TC cluster holds: kCq CTAs x kCthr threads x kSeg
int theta_mp_chain_cap() { return kCq * kCthr * kSeg; }

cudaError_t launch_theta_mp(const ThetaMpParams& Q, cudaStream_t st) {
    const int L1 = Q.f1.L, L2 = Q.f2.L;
    const int NC = Q.t.ncols * Q.t.nrhs;
    const size_t sa = theta_mp_smem_bytes(0, L1, L2, Q.f1.nhi, Q.f1.nlo, Q.f2.nhi, Q.f2.nlo, Q.t.fd.nhi, Q.t.fd.nlo);
    const size_t sb = theta_mp_smem_bytes(1, L1, L2, Q.f1.nhi, Q.f1.nlo, Q.f2.nhi, Q.f2.nlo, Q.t.fd.nhi, Q.t.fd.nlo);
    const size_t sd = theta_mp_smem_bytes(2, L1, L2, Q.f1.nhi, Q.f1.nlo, Q.f2.nhi, Q.f2.nlo, Q.t.fd.nhi, Q.t.fd.nlo);
    const size_t sc = theta_mp_smem_bytes(3, L1, L2, 0, 0, 0, 0, 0, 0);
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(theta_mp_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_mp_b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_mp_c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_mp_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_mp_e_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    theta_mp_a_kernel<<<NC * (L1 / kBlkR), kThr, sa, st>>>(Q);
    theta_mp_b_kernel<<<NC * 2 * (L2 / kBlkT), kThr, sb, st>>>(Q);
    theta_mp_c_kernel<<<NC * 2 * kCq, kCthr, sc, st>>>(Q, exit_relaxed());
    if (Q.t.xhalf) {
        const long long tot = 2LL * Q.t.fd.L * NC;
        theta_mp_export_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(Q);
    }
    theta_mp_d_kernel<<<NC * 2 * (L2 / kBlkT), kThr, sd, st>>>(Q);
    theta_mp_e_kernel<<<NC * (L1 / kBlkR), kThr, sa, st>>>(Q);
    return cudaGetLastError();
}

}  // namespace sk
