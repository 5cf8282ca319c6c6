// Grid-path kernels for transform lengths that do not fit one CTA's shared
// memory (config C5: M/2 = 32768 theta modes per parity, N/2 = 16384 lambda
// pairs).  Same algorithm as grid_kernels.cu, distributed over a thread-block
// cluster with distributed shared memory (DSMEM):
//
//   theta_large_kernel<Q>  — one cluster of 2Q CTAs per lambda mode: CTA
//     (par, q) holds the q-th contiguous quarter (Q = 4) of parity class par.
//     Forward transform = Q decimated length-L/Q FFTs (CTA q transforms the
//     inputs j = Q r + q) + a radix-Q combine across the cluster that leaves
//     every CTA with a contiguous range of theta modes in natural order, so
//     each chain (t > 0 or t < 0) lives in Q/2 consecutive CTAs and the chain
//     scans only exchange segment totals between CTAs.  Inverse = radix-Q
//     split across the cluster + local length-L/Q FFTs; the two parity classes
//     are recombined CTA to CTA.
//   lambda_fwd_split_kernel / lambda_inv_split_kernel — one 2-CTA cluster per
//     physical row: the first radix-2 step splits the length-N/2 transform by
//     parity of the mode index; the real-to-complex split needs only modes
//     of one parity (N/2 even), the inverse recombines through DSMEM.
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

constexpr int kStage = 16;  // values per thread staged in registers across cluster exchanges
constexpr int kFoldStages = 3;  // TMA stages of fold inputs in flight (in the pivot window)

#ifdef SK_PHASES
extern __device__ unsigned long long g_phase[4096][24];
#define SK_PROBE_L(i)                                                        \
    do {                                                                    \
        __syncthreads();                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_phase[blockIdx.x][i] = clock64(); \
    } while (0)
#else
#define SK_PROBE_L(i) \
    do {              \
    } while (0)
#endif

// exp(-2 pi i m / n) for the 2L-th-root table (M-th roots): w_L^(-m) = T(2m)
// (0 <= m < 4L: the callers' exponents s tau, s < Q, tau < L; 32-bit
// reduction by subtraction — a 64-bit modulo here cost a third of the kernel)
__device__ __forceinline__ double2 wL(const Tw& T, int m, int L) {
    const int n2 = 2 * L;
    int mm = 2 * m;
    while (mm >= n2) mm -= n2;
    return T(mm);
}

// ---------------------------------------------------------------- theta
// Solves this CTA's part [i_lo, i_hi) of a chain whose parts lie in
// consecutive CTAs (chain position cpos of ncta).  Shared memory holds the
// CTA's theta modes in natural order; slot(i) maps a chain element to its
// (swizzled) local slot.  Segment totals of the two affine scans are
// exchanged through DSMEM (`tot` slots of every CTA of this chain).
template <class SlotFn, class RemoteTot>
__device__ void solve_chain_part(double2* a, const double* ipw, V4* wsc, V4* tot, const Chain& ch, int L, int i_lo,
                                 int i_hi, double2 xlo_cta, double2 xhi_cta, SlotFn slot, RemoteTot remote_tot,
                                 int cpos, int ncta, cg::cluster_group& cluster, double& fmax_acc, double2& wsum,
                                 bool want_wsum) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int n = i_hi - i_lo;
    const int s = i_lo + static_cast<int>((static_cast<long long>(tid) * n) / nthr);
    const int e = i_lo + static_cast<int>((static_cast<long long>(tid + 1) * n) / nthr);
    auto ip = [&](int i) { return ipw[ch.tau0 + ch.dtau * i]; };
    auto Fof = [&](double2 xm, double2 x0, double2 xp, int i) {
        const double d2 = chainD2(ch, i, L);
        return make_double2(d2 * x0.x - 0.25 * (xm.x + xp.x), d2 * x0.y - 0.25 * (xm.y + xp.y));
    };
    double2 xlo = make_double2(0.0, 0.0), xhi = make_double2(0.0, 0.0);
    if (s < e) {
        xlo = (s == i_lo) ? xlo_cta : a[slot(s - 1)];
        xhi = (e < i_hi) ? a[slot(e)] : xhi_cta;
    }
    const double ip_before = (s > 0 && s < e) ? ip(s - 1) : 0.0;
    __syncthreads();

    // local forward summary
    V4 aff = AffOp::identity();
    {
        double2 xm = xlo;
        double2 x0 = (s < e) ? a[slot(s)] : make_double2(0.0, 0.0);
        double ipp = ip_before;
        for (int i = s; i < e; ++i) {
            const double2 xp = (i + 1 < e) ? a[slot(i + 1)] : xhi;
            const double2 F = Fof(xm, x0, xp, i);
            fmax_acc = fmax(fmax_acc, F.x * F.x + F.y * F.y);
            const double al = -chainA(ch, i, L) * ipp;
            aff = V4{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y), 0.0};
            ipp = ip(i);
            xm = x0;
            x0 = xp;
        }
    }
    V4 rin = block_exclusive_scan<AffOp, false>(aff, wsc);
    if (tid == nthr - 1) tot[0] = AffOp::combine(rin, aff);
    cluster.sync();
    {
        V4 acc = AffOp::identity();
        for (int c = 0; c < cpos; ++c) acc = AffOp::combine(acc, remote_tot(c, 0));
        rin = AffOp::combine(acc, rin);
    }
    // forward sweep, r' in place
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
        double2 xm = xlo;
        double2 x0 = (s < e) ? a[slot(s)] : make_double2(0.0, 0.0);
        for (int i = s; i < e; ++i) {
            const int pi = slot(i);
            const double2 xp = (i + 1 < e) ? a[slot(i + 1)] : xhi;
            const double2 F = Fof(xm, x0, xp, i);
            const double al = -chainA(ch, i, L) * ipp;
            rp = make_double2(fma(al, rp.x, F.x), fma(al, rp.y, F.y));
            a[pi] = rp;
            ipp = ip(i);
            xm = x0;
            x0 = xp;
        }
    }
    __syncthreads();
    // local backward summary
    V4 baff = AffOp::identity();
    for (int i = e - 1; i >= s; --i) {
        const double iv = ip(i);
        const double2 r = a[slot(i)];
        const double be = -chainC(ch, i, L) * iv;
        baff = V4{be * baff.a, fma(be, baff.b, r.x * iv), fma(be, baff.c, r.y * iv), 0.0};
    }
    V4 xin = block_exclusive_scan<AffOp, true>(baff, wsc);
    if (tid == 0) tot[1] = AffOp::combine(xin, baff);
    cluster.sync();
    {
        V4 acc = AffOp::identity();
        for (int c = ncta - 1; c > cpos; --c) acc = AffOp::combine(acc, remote_tot(c, 1));
        xin = AffOp::combine(acc, xin);
    }
    // back substitution, x in place
    double2 ws = make_double2(0.0, 0.0);
    {
        double2 x = make_double2(xin.b, xin.c);
        for (int i = e - 1; i >= s; --i) {
            const int pi = slot(i);
            const double iv = ip(i);
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
        }
    }
    wsum.x += ws.x;
    wsum.y += ws.y;
    __syncthreads();
}

template <int Q>
__global__ void __launch_bounds__(512, 1) theta_large_kernel(ThetaLargeParams PL, const __grid_constant__ CUtensorMap cmap, int relaxed_exit) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const ThetaParams& P = PL.t;
    const FftDesc& fq = PL.fq;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int par = rank / Q, q = rank % Q;
    const int L = P.fd.L;  // M/2
    const int Lq = L / Q;
    double2* a = reinterpret_cast<double2*>(smem_raw);              // Lq slots, swizzled
    double2* tM_hi = a + ((Lq + 7) & ~7);
    double2* tM_lo = tM_hi + P.fd.nhi;
    double2* tq_hi = tM_lo + P.fd.nlo;
    double2* tq_lo = tq_hi + fq.nhi;
    double* ipw = reinterpret_cast<double*>(tq_lo + fq.nlo);          // Lq + 4 pivots
    V4* wsc = reinterpret_cast<V4*>(ipw + ((Lq + 4 + 1) & ~1));
    V4* tot = wsc + 32;                                                 // 2 slots
    double2* misc = reinterpret_cast<double2*>(tot + 2);               // 16
    double* red = reinterpret_cast<double*>(misc + 16);                 // 64
    uint64_t* bar = reinterpret_cast<uint64_t*>(red + 64);

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int col = blockIdx.x / (2 * Q);
    const int rhs = col / P.ncols;
    const int kl = col - rhs * P.ncols;
    const int kg = P.k0 + kl;
    const double k2 = static_cast<double>(kg) * static_cast<double>(kg);
    const double sgn = (kg & 1) ? -1.0 : 1.0;
    double2* colbase = P.buf + rhs * P.rhs_stride;
    auto gcol = [&](int p) { return colbase + theta_addr(P.sl, P.ncols, kl, p); };
    auto rmt = [&](int r) { return cluster.map_shared_rank(a, r); };  // CTA r's data slots
    // output row p: in place, or straight into its lambda rank's return buffer
    auto gout = [&](int p) { return P.peers.n ? peer_ptr(P.peers, p, kg, p) : gcol(p); };
    const int* revq = fq.rev;
    SK_PROBE_L(0);

    // chain of this CTA and its element range
    Chain cp, cm;
    make_chains(par, L, cp, cm);
    const bool plus = q < Q / 2;
    const Chain& ch = plus ? cp : cm;
    const int cpos = plus ? q : (Q - 1 - q);
    int i_lo, i_hi;
    if (plus) {
        i_lo = max(0, q * Lq - ch.tau0);
        i_hi = min(ch.n, (q + 1) * Lq - ch.tau0);
    } else {
        i_lo = max(0, L - (q + 1) * Lq);
        i_hi = min(ch.n, L - q * Lq);
    }
    if (i_hi < i_lo) i_hi = i_lo;
    auto slot = [&](int i) { return swz<true>(ch.tau0 + ch.dtau * i - q * Lq); };

    // pivot window of this CTA's chain part (TMA, overlaps the transforms)
    const size_t prow = (static_cast<size_t>(kl) * 2 + par) * P.piv_stride;
    // (includes the pivot of element i_lo - 1, owned by the previous CTA)
    const int tau_a = plus ? ch.tau0 + max(i_lo - 1, 0) : ch.tau0 - (i_hi - 1);
    const int tau_b = plus ? ch.tau0 + i_hi : ch.tau0 - max(i_lo - 1, 0) + 1;
    uint32_t pbytes = 0;
    const double* ipv = pivot_window(ipw, P.pivots, prow, tau_a, tau_b, pbytes);
    if (tid == 0) {
        for (int b = 0; b < 4; ++b) mbar_init(&bar[b], 1);  // [0] pivots, [1..3] fold staging
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue_pivots = [&]() {
        if (tid == 0 && i_hi > i_lo) {
            mbar_expect_tx(bar, pbytes);
            bulk_g2s_chunked(ipw, P.pivots + ((prow + tau_a) & ~static_cast<size_t>(1)), pbytes, bar);
        }
    };
    if (!PL.use_cmap) issue_pivots();  // else after the fold, which stages its inputs in the pivot window
    const Tw TM = load_tw(P.fd, tM_hi, tM_lo, tid, nthr);
    const Tw TQ = load_tw(fq, tq_hi, tq_lo, tid, nthr);
    __syncthreads();
    SK_PROBE_L(1);

    // ---- 1. fold + decimation: inputs x_j, j = Q r + q (first radix-Q split)
    const double invM = 1.0 / P.g.M;
    if (PL.use_cmap) {
        // Inputs a_j (j = Q r + q) and a_(L-j) by TMA boxes of the column
        // tensor map {re/im, j mod Q, j / Q, column} into the pivot window:
        // kFoldStages chunks of kFoldChunk r in flight; a_(L-j) runs backwards
        // through its box (r' = L/Q - 1 - r for q > 0, L/Q - r for q = 0; the
        // one out-of-range element, a_L, comes from global memory).
        const int CB = PL.fold_chunk;  // 512 or 256 (what the pivot window holds)
        constexpr int NS = kFoldStages;
        double2* stg = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(ipw) + 127) & ~static_cast<uintptr_t>(127));
        const int mcol = blockIdx.x / (2 * Q);  // column of the map: rhs * ncols + kl
        const int nch = (Lq + CB - 1) / CB;
        const int qm = (Q - q) % Q;
        auto issue = [&](int c) {
            const int sI = c % NS, r0 = c * CB;
            double2* aj = stg + sI * 2 * CB;
            double2* am = aj + CB;
            mbar_expect_tx(&bar[1 + sI], 2 * CB * 16);
            const int st = q > 0 ? (Lq - r0 - CB) : (Lq - r0 - CB + 1);
            for (int b = 0; b < CB; b += 256) {
                tma_load_4d(aj + b, &cmap, 0, q, r0 + b, mcol, &bar[1 + sI]);
                tma_load_4d(am + b, &cmap, 0, qm, st + b, mcol, &bar[1 + sI]);
            }
        };
        if (tid == 0)
            for (int c = 0; c < NS && c < nch; ++c) issue(c);
        const double2 aL = *gcol(L);
        for (int c = 0; c < nch; ++c) {
            const int sI = c % NS;
            const double2* aj = stg + sI * 2 * CB;
            const double2* am = aj + CB;
            mbar_wait(&bar[1 + sI], (c / NS) & 1);
            for (int i = tid; i < CB; i += nthr) {
                const int r = c * CB + i;
                if (r < Lq) {
                    const int j = Q * r + q;
                    double2 vj = aj[i];
                    if (j == 0 && P.g.pole_glide) vj = cscale(vj, sgn);  // sk_internal.h GridGeom::pole_glide
                    const double2 vm = (q == 0 && r == 0) ? aL : am[CB - 1 - i];
                    double2 x;
                    if (par == 0) x = make_double2((vj.x + sgn * vm.x) * invM, (vj.y + sgn * vm.y) * invM);
                    else x = cscale(cmul(make_double2(vj.x - sgn * vm.x, vj.y - sgn * vm.y), TM(j)), invM);
                    a[swz<true>(__ldg(revq + r))] = x;
                }
            }
            __syncthreads();
            if (tid == 0 && c + NS < nch) {
                fence_proxy_async();  // this stage's generic reads before the next bulk writes
                issue(c + NS);
            }
        }
        if (tid == 0) fence_proxy_async();
        issue_pivots();
    } else {
        // batches of kFoldU inputs per thread: all global loads of a batch are
        // in flight before any shared-memory store
        constexpr int kFoldU = 8;
        for (int r0 = tid; r0 < Lq; r0 += kFoldU * nthr) {
            double2 aj[kFoldU], am[kFoldU];
#pragma unroll
            for (int u = 0; u < kFoldU; ++u) {
                const int r = r0 + u * nthr;
                if (r < Lq) {
                    const int j = Q * r + q;
                    aj[u] = *gcol(j);
                    am[u] = *gcol(L - j);
                    if (j == 0 && P.g.pole_glide) aj[u] = cscale(aj[u], sgn);  // sk_internal.h GridGeom::pole_glide
                }
            }
#pragma unroll
            for (int u = 0; u < kFoldU; ++u) {
                const int r = r0 + u * nthr;
                if (r < Lq) {
                    const int j = Q * r + q;
                    double2 x;
                    if (par == 0) x = make_double2((aj[u].x + sgn * am[u].x) * invM, (aj[u].y + sgn * am[u].y) * invM);
                    else x = cscale(cmul(make_double2(aj[u].x - sgn * am[u].x, aj[u].y - sgn * am[u].y), TM(j)), invM);
                    a[swz<true>(__ldg(revq + r))] = x;
                }
            }
        }
    }
    __syncthreads();
    SK_PROBE_L(2);
    fft_run<false, -1, true>(a, fq, TQ, tid, nthr);  // DIT: Y^q at swz(m), natural order
    SK_PROBE_L(3);
    cluster.sync();

    // ---- 2. radix-Q combine: X_(c Lq + tl) = sum_s w_Q^(-s c) w_L^(-s tl) Y^s_tl,
    // one distributed radix-Q butterfly per tl: CTA q owns the tl in
    // [q Lq/Q, (q+1) Lq/Q), reads Y^s_tl from every CTA s and writes output c
    // into CTA c's slot tl.  Y^s is in natural order (DIT forward), so the
    // DSMEM reads and writes of a warp are contiguous slots (random-order
    // DSMEM ran at a quarter of the contiguous rate), and the butterfly costs
    // Q-1 twiddles per Q outputs.
    {
        constexpr int TP = kStage / Q;  // tl per thread (Lq <= kStage * nthr)
        const int lo = (q * Lq) / Q, hi = ((q + 1) * Lq) / Q;
        double2 st[TP][Q];
#pragma unroll
        for (int u = 0; u < TP; ++u) {
            const int tl = lo + tid + u * nthr;
            if (tl < hi) {
                const int ps = swz<true>(tl);
                double2 z[Q];
                z[0] = rmt(par * Q + 0)[ps];
#pragma unroll
                for (int s2 = 1; s2 < Q; ++s2) z[s2] = cmul(rmt(par * Q + s2)[ps], wL(TM, s2 * tl, L));
                dft<Q, -1>(z);
#pragma unroll
                for (int c = 0; c < Q; ++c) st[u][c] = z[c];
            }
        }
        cluster.sync();
#pragma unroll
        for (int u = 0; u < TP; ++u) {
            const int tl = lo + tid + u * nthr;
            if (tl < hi) {
                const int ps = swz<true>(tl);
#pragma unroll
                for (int c = 0; c < Q; ++c) rmt(par * Q + c)[ps] = st[u][c];
            }
        }
    }
    cluster.sync();
    SK_PROBE_L(4);

    // ---- 3. k = 0 mean, boundary values, F_0
    double* stt = P.stats + 4 * rhs;
    if (kg == 0 && par == 0) {
        double2 acc = make_double2(0.0, 0.0);
        for (int tl = tid; tl < Lq; tl += nthr) {
            const double t = t_of(q * Lq + tl, 0, L);
            const double w = 2.0 / (1.0 - t * t);
            const double2 x = a[swz<true>(tl)];
            acc.x = fma(w, x.x, acc.x);
            acc.y = fma(w, x.y, acc.y);
        }
        acc = block_sum2(acc, red);
        if (tid == 0) misc[8] = acc;
    }
    // X at natural index tau (any CTA of this parity)
    auto Xat = [&](int tau) { return rmt(par * Q + tau / Lq)[swz<true>(tau % Lq)]; };
    double2 xlo_cta = make_double2(0.0, 0.0), xhi_cta = make_double2(0.0, 0.0), F0 = make_double2(0.0, 0.0);
    if (i_hi > i_lo) {
        // element i_lo - 1 (or the chain's inner neighbour) and element i_hi
        if (i_lo > 0) xlo_cta = Xat(ch.tau0 + ch.dtau * (i_lo - 1));
        else if (par == 0) xlo_cta = Xat(0);                       // X_0 is the inner value of both even chains
        else xlo_cta = plus ? Xat(L - 1) : Xat(0);                 // X_{-1} / X_{+1}
        if (i_hi < ch.n) xhi_cta = Xat(ch.tau0 + ch.dtau * i_hi);
    }
    if (par == 0 && q == 0) {
        const double2 x0 = Xat(0), xp2 = Xat(1), xm2 = Xat(L - 1);
        const double d2 = msin2_diag(0, L);
        F0 = make_double2(d2 * x0.x - 0.25 * (xm2.x + xp2.x), d2 * x0.y - 0.25 * (xm2.y + xp2.y));
    }
    cluster.sync();  // every remote read of X happens before the chains overwrite it
    if (kg == 0 && par == 0 && q == 0 && tid == 0) {
        double2 s2 = make_double2(0.0, 0.0);
        for (int c = 0; c < Q; ++c) {
            const double2 v = cluster.map_shared_rank(misc, c)[8];
            s2.x += v.x;
            s2.y += v.y;
        }
        const double twopi = 6.283185307179586476925286766559;
        stt[0] = twopi * s2.x;
        stt[1] = twopi * s2.y;
    }

    // ---- 4. the chain part
    SK_PROBE_L(5);
    if (i_hi > i_lo) mbar_wait(bar, 0);
    SK_PROBE_L(6);
    double fmax_acc = (par == 0 && q == 0) ? F0.x * F0.x + F0.y * F0.y : 0.0;
    double2 wsum = make_double2(0.0, 0.0);
    const bool want_wsum = (kg == 0 && par == 0);
    auto remote_tot = [&](int c, int which) {
        const int r = par * Q + (plus ? c : (Q - 1 - c));
        return cluster.map_shared_rank(tot, r)[which];
    };
    solve_chain_part(a, ipv, wsc, tot, ch, L, i_lo, i_hi, xlo_cta, xhi_cta, slot, remote_tot, cpos, Q / 2, cluster,
                     fmax_acc, wsum, want_wsum);

    SK_PROBE_L(7);
    // ---- 5. row j = 0 / constraint (parity 0, CTA 0)
    if (want_wsum) {
        wsum = block_sum2(wsum, red);
        if (tid == 0) misc[9] = wsum;
    }
    cluster.sync();
    if (par == 0 && q == 0 && tid == 0) {
        double2 x0;
        if (kg != 0) {
            const double2 xp2 = a[swz<true>(1)], xm2 = rmt(Q - 1)[swz<true>(Lq - 1)];
            x0 = make_double2((F0.x - 0.5 * xm2.x - 0.5 * xp2.x) / (-k2), (F0.y - 0.5 * xm2.y - 0.5 * xp2.y) / (-k2));
        } else {
            double2 ws = make_double2(0.0, 0.0);
            for (int c = 0; c < Q; ++c) {
                const double2 v = cluster.map_shared_rank(misc, c)[9];
                ws.x += v.x;
                ws.y += v.y;
            }
            x0 = make_double2(-0.5 * ws.x, -0.5 * ws.y);
        }
        a[swz<true>(0)] = x0;
    }
    {
        const double fm = sqrt(block_max(fmax_acc, red));
        if (tid == 0) atomic_max_nonneg(stt + 2, fm);
    }
    if (P.xhalf) {
        double2* xo = P.xhalf + static_cast<long long>(rhs) * (P.g.N / 2 + 1) * P.g.M +
                      static_cast<long long>(kg) * P.g.M;
        __syncthreads();
        for (int tl = tid; tl < Lq; tl += nthr) xo[t_of(q * Lq + tl, par, L) + L] = a[swz<true>(tl)];
    }
    cluster.sync();
    SK_PROBE_L(8);

    // ---- 6. inverse radix-Q split: u^c_tl = w_L^(+c tl) sum_s x_(tl + s Lq) w_Q^(+c s),
    // again one distributed butterfly per tl (contiguous DSMEM reads and
    // writes); each CTA then permutes its slots locally into digit-reversed
    // order for the DIT inverse (natural order out).
    {
        constexpr int TP = kStage / Q;
        const int lo = (q * Lq) / Q, hi = ((q + 1) * Lq) / Q;
        double2 st[TP][Q];
#pragma unroll
        for (int u = 0; u < TP; ++u) {
            const int tl = lo + tid + u * nthr;
            if (tl < hi) {
                const int ps = swz<true>(tl);
                double2 z[Q];
#pragma unroll
                for (int s2 = 0; s2 < Q; ++s2) z[s2] = rmt(par * Q + s2)[ps];
                dft<Q, +1>(z);
                st[u][0] = z[0];
#pragma unroll
                for (int c = 1; c < Q; ++c) st[u][c] = cmulc(z[c], wL(TM, c * tl, L));
            }
        }
        cluster.sync();
#pragma unroll
        for (int u = 0; u < TP; ++u) {
            const int tl = lo + tid + u * nthr;
            if (tl < hi) {
                const int ps = swz<true>(tl);
#pragma unroll
                for (int c = 0; c < Q; ++c) rmt(par * Q + c)[ps] = st[u][c];
            }
        }
        cluster.sync();
        double2 pv[kStage];
#pragma unroll
        for (int u = 0; u < kStage; ++u) {
            const int tl = tid + u * nthr;
            if (tl < Lq) pv[u] = a[swz<true>(tl)];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kStage; ++u) {
            const int tl = tid + u * nthr;
            if (tl < Lq) a[swz<true>(__ldg(revq + tl))] = pv[u];
        }
    }
    __syncthreads();
    SK_PROBE_L(9);
    fft_run<false, +1, true>(a, fq, TQ, tid, nthr);  // DIT: V_(Q m + q) at swz(m)
    SK_PROBE_L(10);
    cluster.sync();
    SK_PROBE_L(11);

    // ---- 7. parity recombination v_j = Ve_j + w_M^j Vo_j, j = Q m + q
    {
        const double2* ve = rmt(0 * Q + q);
        const double2* vo = rmt(1 * Q + q);
        const int m_lo = par == 0 ? 0 : Lq / 2;
        const int m_hi = par == 0 ? Lq / 2 : Lq;
        for (int m = m_lo + tid; m < m_hi; m += nthr) {
            const int j = Q * m + q;
            const int ps = swz<true>(m);
            *gout(j) = cadd(ve[ps], cmulc(vo[ps], TM(j)));
        }
        if (par == 0 && q == 0 && tid == 0) {
            const int ps = swz<true>(0);
            *gout(L) = csub(ve[ps], vo[ps]);  // j = L: w_M^L = -1
        }
    }
    SK_PROBE_L(12);
    cluster_exit_barrier(relaxed_exit);
    SK_PROBE_L(13);
}

// ---------------------------------------------------------------- lambda
// Forward: CTA c of the pair computes y_r = (z_r + (-1)^c z_(r+L/2)) w_L^(-r c),
// r < L/2, from the row (L complex pairs), transforms it (length L/2) to
// Z_(2 m + c), and emits the real-split modes X_k, k = c (mod 2), plus the
// Nyquist mode (c = 0).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) lambda_fwd_split_kernel(LambdaSplitParams PS, int relaxed_exit) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const LambdaParams& P = PS.l;
    const FftDesc& fh = PS.fh;  // length L/2
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int L = P.fd.L, Lh = L / 2;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* tN_hi = a + PS.aslots;
    double2* tN_lo = tN_hi + P.fd.nhi;
    double2* th_hi = tN_lo + P.fd.nlo;
    double2* th_lo = th_hi + fh.nhi;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int rowi = blockIdx.x / 2;
    const int row = rowi % P.rows_local;
    const int rhs = rowi / P.rows_local;
    const Tw TN = load_tw(P.fd, tN_hi, tN_lo, tid, nthr);  // N-th roots: w_L^(-r) = TN(2r)
    SK_PROBE_L(14);
    const Tw TH = load_tw(fh, th_hi, th_lo, tid, nthr);
    __syncthreads();
    SK_PROBE_L(15);
    const double2* src =
        reinterpret_cast<const double2*>(P.f + rhs * P.in_rhs_stride + static_cast<long long>(row) * P.g.N);
    // (XOR-swizzled slots: the power-of-two transforms of C5 otherwise hit
    // one bank per butterfly; loads in batches of kLoadU per thread)
    constexpr int kLoadU = 8;
    for (int r0 = tid; r0 < Lh; r0 += kLoadU * nthr) {
        double2 z0[kLoadU], z1[kLoadU];
#pragma unroll
        for (int u = 0; u < kLoadU; ++u) {
            const int r = r0 + u * nthr;
            if (r < Lh) {
                z0[u] = __ldg(src + r);
                z1[u] = __ldg(src + r + Lh);
            }
        }
#pragma unroll
        for (int u = 0; u < kLoadU; ++u) {
            const int r = r0 + u * nthr;
            if (r < Lh) a[swz<true>(r)] = c == 0 ? cadd(z0[u], z1[u]) : cmul(csub(z0[u], z1[u]), TN(2 * r));
        }
    }
    __syncthreads();
    SK_PROBE_L(16);
    fft_forward<true>(a, fh, TH, tid, nthr);  // Z_(2m+c) at swz(rev_h(m))
    SK_PROBE_L(17);
    const double invN = 1.0 / P.g.N;
    double2* out = P.spec + rhs * P.out_rhs_stride;
    const int* revh = fh.rev;
    // pairs (k, L - k), k = 2m + c, m = 0..(L/2 - c)/2
    for (int m = tid; 2 * m + c <= L / 2; m += nthr) {
        const int k = 2 * m + c;
        const int km = L - k;
        const int mk = m, mkm = (km == L) ? 0 : (km - c) / 2;
        const double2 z = a[swz<true>(__ldg(revh + mk))];
        const double2 zp = a[swz<true>(__ldg(revh + mkm))];
        const double2 A = make_double2(0.5 * (z.x + zp.x), 0.5 * (z.y - zp.y));
        const double2 B = make_double2(0.5 * (z.y + zp.y), -0.5 * (z.x - zp.x));
        const double2 Xk = cadd(A, cmul(TN(k), B));
        const double2 Xm = cadd(conjd(A), cmul(TN(km), conjd(B)));
        const double2 vk = cscale(Xk, (k & 1) ? -invN : invN);
        const double2 vm = cscale(Xm, (km & 1) ? -invN : invN);
        if (P.peers.n) {
            *peer_ptr(P.peers, k, k, row) = vk;
            if (km != k) *peer_ptr(P.peers, km, km, row) = vm;
        } else {
            out[static_cast<size_t>(k) * P.rows_local + row] = vk;
            if (km != k) out[static_cast<size_t>(km) * P.rows_local + row] = vm;
        }
    }
    SK_PROBE_L(18);
    (void)relaxed_exit;  // no CTA reads its peer's shared memory: no exit barrier needed
}

// Inverse: CTA c gathers the modes k = c (mod 2) (and their partners L - k),
// forms Z_k, runs the length-L/2 inverse transform of its class and the pair
// recombines z_j = W0_j + w_L^j W1_j through DSMEM (CTA c writes half the row).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    lambda_inv_split_kernel(LambdaSplitParams PS, int relaxed_exit, const __grid_constant__ CUtensorMap map0,
                            const __grid_constant__ CUtensorMap map1) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const LambdaParams& P = PS.l;
    const FftDesc& fh = PS.fh;
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int L = P.fd.L, Lh = L / 2;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* tN_hi = a + PS.aslots;
    double2* tN_lo = tN_hi + P.fd.nhi;
    double2* th_hi = tN_lo + P.fd.nlo;
    double2* th_lo = th_hi + fh.nhi;
    uint64_t* bar = reinterpret_cast<uint64_t*>(th_lo + fh.nlo);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int rowi = blockIdx.x / 2;
    const int row = rowi % P.rows_local;
    const int rhs = rowi / P.rows_local;
    const int* revh = fh.rev;
    const int mcount = (L / 2 - c) / 2 + 1;  // pairs (k, L - k), k = 2m + c <= L/2
    if (PS.tma) {
        // this CTA's modes k = 2m + c, m = 0 .. (L - c)/2, gathered by the copy
        // engine through the per-parity tensor map (mode stride 2) into slots
        // m in natural order; out-of-range modes of the last box are zero-filled
        if (tid == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const int nbox = PS.aslots / kSplitBox;
            mbar_expect_tx(bar, static_cast<uint32_t>(nbox) * kSplitBox * 16);
            const CUtensorMap* mp = c == 0 ? &map0 : &map1;
            for (int b = 0; b < nbox; ++b) tma_load_3d(a + b * kSplitBox, mp, 2 * row, b * kSplitBox, rhs, bar);
        }
    }
    const Tw TN = load_tw(P.fd, tN_hi, tN_lo, tid, nthr);
    SK_PROBE_L(19);
    const Tw TH = load_tw(fh, th_hi, th_lo, tid, nthr);
    __syncthreads();
    SK_PROBE_L(20);
    if (PS.tma) {
        // every pair through registers (the packed values land in swizzled
        // digit-reversed slots of the same buffer); the table indices are
        // fetched while the gather is in flight
        double2 zk[kSplitPairs], zm[kSplitPairs];
        int rk[kSplitPairs], rm[kSplitPairs];
#pragma unroll
        for (int u = 0; u < kSplitPairs; ++u) {
            const int m = min(tid + u * nthr, mcount - 1);
            rk[u] = __ldg(revh + m);
            rm[u] = __ldg(revh + min((L - 2 * m - 2 * c) / 2, Lh - 1));  // partner L - k = 2 m' + c
        }
        mbar_wait(bar, 0);
#pragma unroll
        for (int u = 0; u < kSplitPairs; ++u) {
            const int m = tid + u * nthr;
            if (m < mcount) {
                const int k = 2 * m + c;
                const int km = L - k;
                double2 v = a[m];
                double2 w = a[(km - c) / 2];
                if (k & 1) v = make_double2(-v.x, -v.y);
                if (km & 1) w = make_double2(-w.x, -w.y);
                if (k == 0) {  // DC and Nyquist of a real signal are real
                    v.y = 0.0;
                    w.y = 0.0;
                }
                // conj TN(L - k) = -TN(k): E_{L-k} = conj E_k, O_{L-k} = conj O_k, one twiddle product for both
                const double2 E = make_double2(v.x + w.x, v.y - w.y);
                const double2 O = cmulc(make_double2(v.x - w.x, v.y + w.y), TN(k));
                zk[u] = make_double2(E.x - O.y, E.y + O.x);
                zm[u] = make_double2(E.x + O.y, O.x - E.y);
            }
        }
        __syncthreads();  // every gathered mode has been read
#pragma unroll
        for (int u = 0; u < kSplitPairs; ++u) {
            const int m = tid + u * nthr;
            if (m < mcount) {
                const int k = 2 * m + c;
                a[swz<true>(rk[u])] = zk[u];
                if (k != 0 && L - k != k) a[swz<true>(rm[u])] = zm[u];
            }
        }
    }
    const double2* in = P.spec + rhs * P.in_rhs_stride;
    for (int m = PS.tma ? mcount : tid; 2 * m + c <= L / 2; m += nthr) {
        const int k = 2 * m + c;
        const int km = L - k;
        double2 v = __ldg(in + static_cast<size_t>(k) * P.rows_local + row);
        double2 w = __ldg(in + static_cast<size_t>(km) * P.rows_local + row);
        if (k & 1) v = make_double2(-v.x, -v.y);
        if (km & 1) w = make_double2(-w.x, -w.y);
        if (k == 0) {
            v.y = 0.0;
            w.y = 0.0;
        }
        {
            const double2 E = make_double2(v.x + w.x, v.y - w.y);
            const double2 O = cmulc(make_double2(v.x - w.x, v.y + w.y), TN(k));
            a[swz<true>(__ldg(revh + m))] = make_double2(E.x - O.y, E.y + O.x);
        }
        if (k != 0 && km != k) {
            const double2 E = make_double2(w.x + v.x, w.y - v.y);
            const double2 O = cmulc(make_double2(w.x - v.x, w.y + v.y), TN(km));
            a[swz<true>(__ldg(revh + (km - c) / 2))] = make_double2(E.x - O.y, E.y + O.x);
        }
    }
    __syncthreads();
    SK_PROBE_L(21);
    fft_inverse<true>(a, fh, TH, tid, nthr);  // W^c_j natural at swz(j), j < L/2
    SK_PROBE_L(22);
    cluster.sync();
    const double2* w0 = cluster.map_shared_rank(a, 0);
    const double2* w1 = cluster.map_shared_rank(a, 1);
    double2* dst = reinterpret_cast<double2*>(P.u + rhs * P.out_rhs_stride + static_cast<long long>(row) * P.g.N);
    for (int jj = tid; jj < Lh; jj += nthr) {
        const int j = c * Lh + jj;  // z_j = W0_(j mod L/2) + w_L^(+j) W1_(j mod L/2)
        dst[j] = cadd(w0[swz<true>(jj)], cmulc(w1[swz<true>(jj)], TN(2 * j)));
    }
    SK_PROBE_L(23);
    cluster_exit_barrier(relaxed_exit);
}

// --------------------------------------------------------- host launchers
cudaError_t launch_theta_large(const ThetaLargeParams& P, const CUtensorMap& cmap, int Q, int nthr, size_t smem,
                               cudaStream_t st) {
    const int nblk = 2 * Q * P.t.ncols * P.t.nrhs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(nthr);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (Q == 4) {
        cudaFuncSetAttribute(theta_large_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(theta_large_kernel<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return cudaLaunchKernelEx(&cfg, theta_large_kernel<4>, P, cmap, exit_relaxed());
    }
    cudaFuncSetAttribute(theta_large_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return cudaLaunchKernelEx(&cfg, theta_large_kernel<2>, P, cmap, exit_relaxed());
}

cudaError_t launch_lambda_fwd_split(const LambdaSplitParams& P, int nthr, size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(lambda_fwd_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    lambda_fwd_split_kernel<<<2 * P.l.rows_local * P.l.nrhs, nthr, smem, st>>>(P, exit_relaxed());
    return cudaGetLastError();
}

// map0 / map1: the spectrum's even / odd modes (make_spec_map with mode step 2), read when P.tma
cudaError_t launch_lambda_inv_split(const LambdaSplitParams& P, const CUtensorMap& map0, const CUtensorMap& map1, int nthr,
                                    size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(lambda_inv_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    lambda_inv_split_kernel<<<2 * P.l.rows_local * P.l.nrhs, nthr, smem, st>>>(P, exit_relaxed(), map0, map1);
    return cudaGetLastError();
}

}  // namespace sk
