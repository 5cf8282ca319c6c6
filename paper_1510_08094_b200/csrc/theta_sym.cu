// K3S theta_sym_kernel — the theta stage for long columns (C3: M/2 = 10000)
// built on the (-1)^k symmetry of the DFS column, sm_100a.
//
// Same job as theta_kernel (grid_kernels.cu; replaces the column stage of
// analyze_2d fourier.cpp:174-180, Msin^2 poisson.cpp:61, solve
// poisson.cpp:121-161 with band_solve banded.cpp:101-158 /
// band_solve_with_dense_row :160-328, and the column stage of sample_grid
// fourier.cpp:194-200), one 2-CTA cluster per lambda mode k, CTA `par` owning
// the theta modes t = 2 tau + par.  What changes is the arithmetic, not the
// result:
//
//  * Forward transform at half cost.  The parity sequences of the folded
//    column are symmetric: e_{L-r} = s e_r and o_{L-r} = s w_M^{-2r} o_r
//    (s = (-1)^k, L = M/2).  In the first DIF stage (radix R0 = 2^a, odd span
//    S0 = L/R0) butterfly S0-j therefore carries the same inputs as
//    butterfly j, reversed and twisted:
//        z_k(S0-j) = s conj(T(j e)) y_{(R0-k-par) mod R0}(j),
//        z_k(j)    =      T(j e)  y_k(j),        e = 2k + par,
//    (y = DFT_R0 of the folded inputs, T(m) = exp(-2 pi i m / M)), so one
//    R0-point DFT per butterfly PAIR produces both; the fold is fused into it.
//    The stage's sub-transforms k and (R0-k-par) mod R0 are then mirror
//    images (E_{L-tau} = s E_tau, O_{L-1-tau} = s O_tau), so only the
//    R0/2 + 1 - par sub-transforms k in [0, R0/2 + 1 - par) are computed by
//    the later stages; the other outputs are read through the mirror.
//  * Both chains of a parity for the price of one.  Chain- (t < 0) sees s
//    times chain+'s right-hand side and the same pivots except at the
//    truncation end, so x- = s x+ + Phi Delta, where Phi_i = prod_{j=i}^{n-2}
//    beta_j is the backward sweep's own product (the scan's multiplicative
//    part) and Delta is the difference of the two chains' last unknowns,
//    computed from the boundary rows by the thread that owns them.
//  * One pivot window per CTA: the per-plan table stores each (k, parity)'s
//    pivots once by chain element (pivot_table_sym_kernel), half the bytes of
//    the natural-index table.
//
// The inverse transform, the parity recombination through DSMEM and the
// (peer) stores are those of theta_kernel.
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

#ifdef SK_PHASES
extern __device__ unsigned long long g_phase[4096][24];  // grid_kernels.cu (-rdc debug build, tools/build_phases.sh)
#define SK_PROBE_S(i)                                                       \
    do {                                                                    \
        __syncthreads();                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_phase[blockIdx.x][i] = clock64(); \
    } while (0)
#else
#define SK_PROBE_S(i) \
    do {              \
    } while (0)
#endif

namespace {

// Sizes of the chains of parity class par (theta_common make_chains, L even):
// par 0: chain+ t = 2 .. L-2 (n+ = L/2 - 1), chain- t = -2 .. -L (L/2);
// par 1: chain+ t = 1 .. L-1 (L/2),          chain- t = -1 .. -(L-1) (L/2).
__device__ __forceinline__ int nplus(int par, int L) { return par == 0 ? L / 2 - 1 : L / 2; }

// Forward DFT of R registers (radix R0 of the fused first stage).
template <int R0>
__device__ __forceinline__ void dft_r0(double2* x) {
    dft<R0, -1>(x);
}

// exp(-i pi q / R0) (the fold's twiddle T(q S0) for par 1), q < R0 <= 16
template <int R0>
__device__ __forceinline__ double2 half_root(int q) {
    return wconst<32>(q * (16 / R0));
}

// Fused fold + first DIF stage over butterfly pairs (j, S0 - j).
// (par is a template parameter: the mirror index km below must be a compile-time
// register index, a runtime one puts x[] in local memory)
template <int R0, int par>
__device__ __forceinline__ void fold_stage0(double2* a, int L, double sgn, double invM, const Tw& T, int tid,
                                            int nthr, double2* c0_out) {
    const int S0 = L / R0;
    constexpr int kcnt = R0 / 2 + 1 - par;
    for (int j = tid; 2 * j <= S0; j += nthr) {  // j = 0 .. (S0-1)/2 (S0 odd)
        double2 x[R0];
#pragma unroll
        for (int q = 0; q < R0; ++q) {
            const int r = j + q * S0;
            const double2 ar = a[r];
            const double2 am = a[L - r];  // a_L (slot L) for r = 0
            if (par == 0) {
                x[q] = make_double2((ar.x + sgn * am.x) * invM, (ar.y + sgn * am.y) * invM);
            } else {
                const double2 d = make_double2((ar.x - sgn * am.x) * invM, (ar.y - sgn * am.y) * invM);
                x[q] = (q == 0) ? d : cmul(d, half_root<R0>(q));
            }
        }
        if (j == 0) *c0_out = x[0];  // folded value at r = 0 (the pole rows' term, see SymRead)
        dft_r0<R0>(x);
        // twiddles T(j e), e = 2k + par: u = T(j), u2 = T(2j)
        const double2 u = T(j);
        const double2 u2 = T(2 * j);
        double2 w = par ? u : make_double2(1.0, 0.0);
#pragma unroll
        for (int k = 0; k < R0 / 2 + 1; ++k) {
            if (k < kcnt) {
                a[k * S0 + j] = (j == 0 && par == 0) ? x[k] : cmul(x[k], w);
                if (j != 0) {
                    const int km = (R0 - k - par) & (R0 - 1);
                    const double2 v = cmulc(x[km], w);  // y_km conj(T(j e))
                    a[k * S0 + S0 - j] = make_double2(sgn * v.x, sgn * v.y);
                }
            }
            w = cmul(w, u2);
        }
    }
}

// Restricted DIF stages 1..: only the sub-transforms of blocks k < kcnt.
// (the sub-transforms of blocks k < kcnt own the first kcnt * S0 slots, i.e.
// the first kcnt * S0 / R butterflies of every later stage)
template <int MAXR>
__device__ __forceinline__ void fft_forward_sub(double2* a, const FftDesc& d, const Tw& T, int tid, int nthr,
                                                int kcnt) {
    const int S0 = d.L / d.R[0];
    for (int s = 1; s < d.nst; ++s) {
        fft_stage_dispatch<true, -1, false, MAXR>(a, d, s, T, tid, nthr, kcnt * (S0 / d.R[s]));
        __syncthreads();
    }
}

// Value X_tau of chain+ element i (natural index tau = tau0 + i): read
// directly when its first-stage digit lies in a computed block, else through
// the mirror.  The folded sequence is symmetric except at r = 0, whose value
// c0 (the pole rows' combination a_0 +- s a_L) breaks it when s = -1: with
// the rest exactly (anti)symmetric, X_tau = s X_mirror + (1 - s) c0
// (mirror L - tau for par 0, L - 1 - tau for par 1).
struct SymRead {
    const double2* a;
    const uint32_t* pw;
    int tau0, par, R0;
    double sgn;
    double2 cofs;  // (1 - s) c0
    __device__ __forceinline__ double2 operator()(int i) const {
        const uint32_t pk = pw[i];
        const int d0 = (tau0 + i) & (R0 - 1);
        const bool direct = par == 0 ? d0 <= R0 / 2 : d0 < R0 / 2;
        const double2 v = a[direct ? (pk & 0xffffu) : (pk >> 16)];  // one load either way
        return direct ? v : make_double2(fma(sgn, v.x, cofs.x), fma(sgn, v.y, cofs.y));
    }
};

// Both chains of parity `par`, S chain+ elements per thread (S * nthr >= n+).
// Pass 1: X -> F = Msin^2 X, forward affine summary; scan; pass 2: r' and
// g = r'/d' (kept in F's registers), backward summary (the last multiplier set
// to 1 so that the scan's product is Phi); the owner of the last element
// computes Delta from the boundary rows; scan; pass 3: x+ = g + c x+ and
// x- = s x+ + Phi Delta into both chains' slots.
// (inlined: as a called function it saved and restored ~100 callee-saved
// registers per thread around the body, 200 KB of local-memory traffic per CTA)
template <int S>
__device__ __forceinline__ void solve_chains_sym(double2* a, const uint32_t* __restrict__ pw, const double* ip, Aff3* wsc,
                                              double2* misc, int par, int L, int R0, double sgn, double k2,
                                              double2 inner, double2 cofs, unsigned* fmax_hi, double2* wsum,
                                              bool want_wsum) {
    const int tid = threadIdx.x;
    const int n = nplus(par, L);
    const int tau0 = par == 0 ? 1 : 0;
    const double t0 = par == 0 ? 2.0 : 1.0;
    const SymRead rd{a, pw, tau0, par, R0, sgn, cofs};
    const int s = tid * S;
    const double t_s = t0 + 2.0 * s;
    double2 v[S];
    double ipv[S];
#pragma unroll
    for (int u = 0; u < S; ++u) {
        const bool ok = s + u < n;
        v[u] = ok ? rd(s + u) : make_double2(0.0, 0.0);
        ipv[u] = ok ? ip[s + u] : 0.0;
    }
    double2 xlo = inner, xhi = make_double2(0.0, 0.0);
    double ip_before = 0.0;
    if (s > 0 && s <= n) {
        xlo = rd(s - 1);
        ip_before = ip[s - 1];
    }
    if (s + S < n) xhi = rd(s + S);
    SK_PROBE_S(12);
    const int ulast = n - 1 - s;  // index of chain+'s last element in this segment (if 0 <= ulast < S)
    const double tl = static_cast<double>(L - 1);
    // ---- pass 1: F = Msin^2 X (d2 = 1/4 only on the truncation row t = L-1)
    Aff3 aff = aff_identity();
    double2 xlast = make_double2(0.0, 0.0), xlast_m = make_double2(0.0, 0.0);  // X of the last two elements
    {
        unsigned fh = 0u;
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
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);  // -A / d'_{i-1}, 4A = t(t-3)+2
            aff = Aff3{al * aff.a, fma(al, aff.b, F.x), fma(al, aff.c, F.y)};
            v[u] = F;
            ipp = ipv[u];
            xm = x0;
            t += 2.0;
        }
        *fmax_hi = max(*fmax_hi, fh);
    }
    SK_PROBE_S(13);
    const Aff3 rin = block_scan_aff1<false>(aff, wsc);  // also orders every X read above before the writes below
    SK_PROBE_S(14);
    // ---- pass 2
    Aff3 baff;
    double2 rlast = make_double2(0.0, 0.0);
    {
        double2 rp = make_double2(rin.b, rin.c);
        double ipp = ip_before;
        double t = t_s;
        double Pm = 1.0;
        double2 G = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const bool ok = s + u < n;
            const double al = (-0.25 * ipp) * fma(t, t - 3.0, 2.0);
            rp = make_double2(fma(al, rp.x, v[u].x), fma(al, rp.y, v[u].y));
            if (u == ulast) rlast = rp;
            const double iv = ipv[u];
            const double2 g = make_double2(rp.x * iv, rp.y * iv);
            // c = -C / d', 4C = t(t+3)+2; the last element's multiplier is 1 so
            // that the scanned product is Phi (its neighbour x_n = 0 anyway)
            double c = (-0.25 * iv) * fma(t, t + 3.0, 2.0);
            if (u == ulast) c = 1.0;
            if (!ok) c = 1.0;
            G = make_double2(fma(Pm, g.x, G.x), fma(Pm, g.y, G.y));
            Pm *= c;
            v[u] = g;  // F is dead: g stays in its registers for pass 3
            ipv[u] = c;
            ipp = iv;
            t += 2.0;
        }
        baff = Aff3{Pm, G.x, G.y};
    }
    // ---- the boundary rows: Delta = x-_{n-1} - s x+_{n-1} (and par 0's extra unknown x-_n at t = -L)
    if (ulast >= 0 && ulast < S) {
        const double ipl = ip[n - 1];
        const double2 xp_last = make_double2(rlast.x * ipl, rlast.y * ipl);  // x+_{n-1} = g+_{n-1}
        double2 xm_last, xm_extra = make_double2(0.0, 0.0);
        unsigned fh = 0u;
        if (par == 0) {
            const double Ld = static_cast<double>(L);
            const double2 XmL = a[pw[n] >> 16];  // X at t = -L (tau = L/2): direct, its own mirror
            // chain- values are X-_i = s X+_i + cofs: F-_i = s F+_i but for the
            // last row, which gains the neighbour t = -L:
            // r'-_{n-1} = s r'+_{n-1} + (cofs - X_{-L})/4
            const double2 dd = make_double2(0.25 * (cofs.x - XmL.x), 0.25 * (cofs.y - XmL.y));
            const double2 rm1 = make_double2(fma(sgn, rlast.x, dd.x), fma(sgn, rlast.y, dd.y));
            const double2 Fm1 = make_double2(sgn * (0.5 * xlast.x - 0.25 * xlast_m.x) + dd.x,
                                             sgn * (0.5 * xlast.y - 0.25 * xlast_m.y) + dd.y);
            // row t = -L: F = X_{-L}/4 - X_{-(L-2)}/4, X_{-(L-2)} = s X+_{n-1} + cofs
            const double2 Fn = make_double2(0.25 * (XmL.x - fma(sgn, xlast.x, cofs.x)),
                                            0.25 * (XmL.y - fma(sgn, xlast.y, cofs.y)));
            const double An = 0.25 * (Ld - 2.0) * (Ld - 1.0);  // coupling of t = -L to t = -(L-2)
            const double Cm = 0.25 * Ld * (Ld - 1.0);          // coupling of t = -(L-2) to t = -L
            const double al = -An * ipl;
            const double2 rn = make_double2(fma(al, rm1.x, Fn.x), fma(al, rm1.y, Fn.y));
            const double ipn = ip[n];  // chain-'s pivot at t = -L
            xm_extra = make_double2(rn.x * ipn, rn.y * ipn);
            const double be = -Cm * ipl;
            xm_last = make_double2(fma(be, xm_extra.x, rm1.x * ipl), fma(be, xm_extra.y, rm1.y * ipl));
            fh = max(static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y))),
                     static_cast<unsigned>(__double2hiint(fma(Fn.x, Fn.x, Fn.y * Fn.y))));
            (void)k2;
        } else {
            // chain- last row t = -(L-1) is interior (d2 = 1/2, own pivot ip[n]):
            // F-_{n-1} = s F+_{n-1} + (s X+_{n-1} + cofs)/4
            const double2 dd = make_double2(0.25 * fma(sgn, xlast.x, cofs.x), 0.25 * fma(sgn, xlast.y, cofs.y));
            const double2 rm1 = make_double2(fma(sgn, rlast.x, dd.x), fma(sgn, rlast.y, dd.y));
            const double ipm = ip[n];
            xm_last = make_double2(rm1.x * ipm, rm1.y * ipm);
            const double2 Fm1 = make_double2(0.5 * fma(sgn, xlast.x, cofs.x) - 0.25 * fma(sgn, xlast_m.x, cofs.x),
                                             0.5 * fma(sgn, xlast.y, cofs.y) - 0.25 * fma(sgn, xlast_m.y, cofs.y));
            fh = static_cast<unsigned>(__double2hiint(fma(Fm1.x, Fm1.x, Fm1.y * Fm1.y)));
        }
        *fmax_hi = max(*fmax_hi, fh);
        misc[5] = make_double2(xm_last.x - sgn * xp_last.x, xm_last.y - sgn * xp_last.y);  // Delta
        misc[6] = xm_extra;
    }
    SK_PROBE_S(15);
    const Aff3 xin = block_scan_aff1<true>(baff, wsc + 16);  // publishes Delta (misc) as well
    SK_PROBE_S(16);
    const double2 Dl = misc[5];
    // ---- pass 3
    double2 x = make_double2(xin.b, xin.c);
    double phi = xin.a;
    double2 ws = make_double2(0.0, 0.0);
    double2 xf_p = make_double2(0.0, 0.0), xf_m = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = S - 1; u >= 0; --u) {
        if (s + u < n) {
            const uint32_t pk = pw[s + u];
            const double2 g = v[u];
            const double c = ipv[u];
            if (u != ulast) {
                x = make_double2(fma(c, x.x, g.x), fma(c, x.y, g.y));
            } else {
                x = g;  // last element: no neighbour
            }
            phi *= c;  // Phi_i = c_i Phi_{i+1} (c_{n-1} = 1)
            const double2 xm = make_double2(fma(phi, Dl.x, sgn * x.x), fma(phi, Dl.y, sgn * x.y));
            a[pk & 0xffffu] = x;
            a[pk >> 16] = xm;
            if (want_wsum) {
                const double t = t_s + 2.0 * u;
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
        a[pw[n] >> 16] = xe;  // x at t = -L
        if (want_wsum) {
            const double Ld = static_cast<double>(L);
            const double w = 2.0 / (1.0 - Ld * Ld);
            ws.x = fma(w, xe.x, ws.x);
            ws.y = fma(w, xe.y, ws.y);
        }
    }
    wsum->x += ws.x;
    wsum->y += ws.y;
    if (tid == 0) {
        misc[3] = xf_p;  // x+_0 (t = 2 or 1)
        misc[4] = xf_m;  // x-_0 (t = -2 or -1)
    }
    // no trailing barrier: the caller publishes its per-warp max|F|^2 first and
    // then synchronises once for both
}

// Odd segment lengths: a warp's per-element loads of the pivot (8 B) and
// slot (4 B) windows then stride an odd number of words, conflict-free.
__device__ __forceinline__ int sym_segment(int n, int nthr) {
    const int need = (n + nthr - 1) / nthr;
    return need <= 5 ? 5 : need <= 7 ? 7 : need <= 9 ? 9 : need <= 11 ? 11 : need <= 13 ? 13 : 0;
}

}  // namespace

// Pivot table of the sym kernel: row (kl, par), stride `stride` doubles;
// entry i = 1/d'_i of chain element i computed by the sequential recurrence
// (banded.cpp:121-147; no row ever swaps for these systems).  par 0 stores
// chain- (L/2 entries; chain+ = its first L/2 - 1), par 1 stores chain+
// (L/2 entries) and, at entry L/2, chain-'s last pivot (interior row t =
// -(L-1) where chain+ ends on the truncation row t = L-1).
__global__ void __launch_bounds__(128) pivot_table_sym_kernel(int L, int k0, int ncols, double* ipt, int stride) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= ncols * 2) return;
    const int kl = id >> 1, par = id & 1;
    const double k2 = static_cast<double>(k0 + kl) * static_cast<double>(k0 + kl);
    Chain cp, cm;
    make_chains(par, L, cp, cm);
    double* out = ipt + (static_cast<size_t>(kl) * 2 + par) * stride;
    const Chain& ch = par == 0 ? cm : cp;
    double ip = 0.0, cprev = 0.0;
    for (int i = 0; i < ch.n; ++i) {
        const int t = ch.t0 + ch.dt * i;
        const double A = chainA(ch, i, L);
        const double d = lap_diag(t, L) - k2 - A * cprev * ip;
        ip = 1.0 / d;
        out[i] = ip;
        cprev = chainC(ch, i, L);
    }
    if (par == 1) {  // chain-'s last element (same recurrence up to it)
        double ipm = 0.0, cpm = 0.0;
        for (int i = 0; i < cm.n; ++i) {
            const int t = cm.t0 + cm.dt * i;
            const double A = chainA(cm, i, L);
            const double d = lap_diag(t, L) - k2 - A * cpm * ipm;
            ipm = 1.0 / d;
            cpm = chainC(cm, i, L);
        }
        out[L / 2] = ipm;
    }
}

template <int R0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) theta_sym_kernel(ThetaParams P, int relaxed_exit) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int L = P.fd.L;  // M/2
    const int half = L / 2;
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* s_hi = a + theta_data_slots(L);
    double2* s_lo = s_hi + P.fd.nhi;
    double* ip = reinterpret_cast<double*>(s_lo + P.fd.nlo);
    uint32_t* pw = reinterpret_cast<uint32_t*>(ip + theta_sym_piv_slots(L));
    V4* wsc = reinterpret_cast<V4*>(pw + theta_sym_pos_slots(L));
    double2* misc = reinterpret_cast<double2*>(wsc + 32);
    double* red = reinterpret_cast<double*>(misc + 16);
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 64);

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int par = static_cast<int>(cluster.block_rank());
    const int col = blockIdx.x >> 1;
    const int rhs = col / P.ncols;
    const int kl = col - rhs * P.ncols;
    const int kg = P.k0 + kl;
    const double k2 = static_cast<double>(kg) * static_cast<double>(kg);
    const double sgn = (kg & 1) ? -1.0 : 1.0;
    double2* colbase = P.buf + rhs * P.rhs_stride;
    const size_t prow = (static_cast<size_t>(kl) * 2 + par) * P.piv_stride;

    // ---- bulk copies: raw column (L+1), this (mode, parity)'s pivots, the chain slot window
    SK_PROBE_S(0);
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t bytes = 0;
        for (int s = 0; s < P.sl.P; ++s) {
            const int r0 = P.sl.row_b[s], r1 = P.sl.row_b[s + 1];
            if (r1 > r0) bytes += (r1 - r0) * 16;
        }
        const uint32_t pb = static_cast<uint32_t>(theta_sym_piv_slots(L)) * 8;
        const uint32_t qb = static_cast<uint32_t>(theta_sym_pos_slots(L)) * 4;
        // the column (needed first) and the chain windows (needed after the
        // forward transform) complete on separate barriers
        mbar_expect_tx(&bars[0], bytes);
        mbar_expect_tx(&bars[1], pb + qb);
        for (int s = 0; s < P.sl.P; ++s) {
            const int r0 = P.sl.row_b[s], r1 = P.sl.row_b[s + 1];
            if (r1 > r0)
                bulk_g2s_chunked(a + r0, colbase + theta_addr(P.sl, P.ncols, kl, r0), (r1 - r0) * 16, &bars[0]);
        }
        bulk_g2s_chunked(ip, P.pivots + prow, pb, &bars[1]);
        bulk_g2s_chunked(pw, P.sym_pos + static_cast<size_t>(par) * theta_sym_pos_slots(L), qb, &bars[1]);
    }
    const Tw T = load_tw(P.fd, s_hi, s_lo, tid, nthr);
    mbar_wait(&bars[0], 0);
    __syncthreads();
    if (P.g.pole_glide && (kg & 1)) {  // the reference's doubled row j = M/2 (sk_internal.h GridGeom)
        if (tid == 0) a[0] = make_double2(-a[0].x, -a[0].y);
        __syncthreads();
    }
    SK_PROBE_S(1);

    // ---- fused fold + first DIF stage (butterfly pairs), then the computed sub-transforms
    const double invM = 1.0 / P.g.M;
    if (tid == 0) misc[7] = make_double2(0.0, 0.0);
    if (par == 0) fold_stage0<R0, 0>(a, L, sgn, invM, T, tid, nthr, &misc[7]);
    else fold_stage0<R0, 1>(a, L, sgn, invM, T, tid, nthr, &misc[7]);
    __syncthreads();
    const double2 c0 = misc[7];
    const double2 cofs = make_double2((1.0 - sgn) * c0.x, (1.0 - sgn) * c0.y);
    SK_PROBE_S(2);
    const int kcnt = R0 / 2 + 1 - par;
    fft_forward_sub<25>(a, P.fd, T, tid, nthr, kcnt);
    SK_PROBE_S(3);
    mbar_wait(&bars[1], 0);  // pivot and chain slot windows

    const SymRead rd{a, pw, par == 0 ? 1 : 0, par, R0, sgn, cofs};
    // ---- k = 0, even class: surface mean 2 pi w^T X_0 (poisson.cpp:101-117)
    double* st = P.stats + 4 * rhs;
    if (kg == 0 && par == 0) {
        double2 acc = make_double2(0.0, 0.0);
        const int n = nplus(0, L);
        for (int i = tid; i < n; i += nthr) {
            const double t = 2.0 + 2.0 * i;
            const double w = 2.0 / (1.0 - t * t);
            const double2 x = rd(i);
            acc.x = fma(2.0 * w, x.x, acc.x);  // X-_i = X+_i for k = 0 (s = 1)
            acc.y = fma(2.0 * w, x.y, acc.y);
        }
        if (tid == 0) {
            const double2 x0 = a[0];
            const double2 xl = a[pw[n] >> 16];  // t = -L
            const double Ld = static_cast<double>(L);
            const double wl = 2.0 / (1.0 - Ld * Ld);
            acc.x += 2.0 * x0.x + wl * xl.x;
            acc.y += 2.0 * x0.y + wl * xl.y;
        }
        acc = block_sum2(acc, red);
        if (tid == 0) {
            const double twopi = 6.283185307179586476925286766559;
            st[0] = twopi * acc.x;
            st[1] = twopi * acc.y;
        }
    }

    // ---- inner neighbours and the j = 0 row data
    if (tid == 0) {
        if (par == 0) {
            const double2 x0 = a[0];          // t = 0 (slot of tau = 0)
            const double2 xp2 = rd(0);        // t = 2
            const double2 xm2 = make_double2(fma(sgn, xp2.x, cofs.x), fma(sgn, xp2.y, cofs.y));  // t = -2: mirror of t = 2
            misc[0] = x0;
            const double d2 = msin2_diag(0, L);
            misc[2] = make_double2(d2 * x0.x - 0.25 * (xm2.x + xp2.x), d2 * x0.y - 0.25 * (xm2.y + xp2.y));
        } else {
            const double2 x1 = rd(0);  // t = 1; the t > 0 chain's inner neighbour is t = -1 = s X_1 + cofs
            misc[0] = make_double2(fma(sgn, x1.x, cofs.x), fma(sgn, x1.y, cofs.y));
            misc[2] = make_double2(0.0, 0.0);
        }
        misc[3] = misc[4] = misc[5] = misc[6] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double2 inner = misc[0], F0 = misc[2];
    unsigned fmax_hi = (par == 0) ? static_cast<unsigned>(__double2hiint(fma(F0.x, F0.x, F0.y * F0.y))) : 0u;
    double2 wsum = make_double2(0.0, 0.0);
    const bool want_wsum = (kg == 0 && par == 0);
    Aff3* wsc3 = reinterpret_cast<Aff3*>(wsc);
    SK_PROBE_S(4);
#define SK_SYM(S) \
    solve_chains_sym<S>(a, pw, ip, wsc3, misc, par, L, R0, sgn, k2, inner, cofs, &fmax_hi, &wsum, want_wsum)
    switch (sym_segment(nplus(par, L), nthr)) {
        case 5: SK_SYM(5); break;
        case 7: SK_SYM(7); break;
        case 9: SK_SYM(9); break;
        case 11: SK_SYM(11); break;
        default: SK_SYM(13); break;  // the plan guarantees n+ <= 12 nthr
    }
#undef SK_SYM
    // per-warp max|F|^2 (high words), one barrier for them and the chain's
    // results, then thread 0 alone finishes: CTA maximum -> stats, x_0 -> slot 0
    unsigned* redu = reinterpret_cast<unsigned*>(red + 48);
    {
        const unsigned wm = __reduce_max_sync(0xffffffffu, fmax_hi);
        if ((tid & 31) == 0) redu[tid >> 5] = wm;
    }
    __syncthreads();
    SK_PROBE_S(17);
    SK_PROBE_S(5);
    if (want_wsum) wsum = block_sum2(wsum, red);
    if (tid == 0) {
        unsigned m = 0u;
        for (int w = 0; w < (nthr >> 5); ++w) m = max(m, redu[w]);
        atomic_max_nonneg(st + 2, sqrt(__hiloint2double(static_cast<int>(m), 0)));
        if (par == 0) {
            double2 x0;
            if (kg != 0) {
                // row j = 0: 1/2 x_{-2} - k^2 x_0 + 1/2 x_2 = F_0
                const double2 xp2 = misc[3], xm2 = misc[4];
                x0 = make_double2((F0.x - 0.5 * xm2.x - 0.5 * xp2.x) / (-k2), (F0.y - 0.5 * xm2.y - 0.5 * xp2.y) / (-k2));
            } else {
                // constraint row 2 pi w^T X_0 = 0 replaces row j = 0 (w_0 = 2)
                x0 = make_double2(-0.5 * wsum.x, -0.5 * wsum.y);
            }
            a[0] = x0;
        }
    }
    __syncthreads();

    // optional: export the solution coefficients of this parity class
    if (P.xhalf) {
        double2* xo = P.xhalf + static_cast<long long>(rhs) * (P.g.N / 2 + 1) * P.g.M +
                      static_cast<long long>(kg) * P.g.M;
        for (int tau = tid; tau < L; tau += nthr) {
            const int t = t_of(tau, par, L);
            xo[t + L] = a[__ldg(P.fd.rev + tau)];
        }
        __syncthreads();
    }

    SK_PROBE_S(6);
    fft_inverse<false, 25>(a, P.fd, T, tid, nthr);
    SK_PROBE_S(7);

    // ---- recombine the parity classes: v_p = Ve_p + w_M^p Vo_p, p = 0..M/2
    cluster.sync();
    const double2* ve = par == 0 ? a : cluster.map_shared_rank(a, 0);
    const double2* vo = par == 1 ? a : cluster.map_shared_rank(a, 1);
    const int p_lo = par == 0 ? 0 : half;
    const int p_hi = par == 0 ? half : L + 1;
    // four rows per thread and trip: the (remote) loads of all four issue
    // before the first is used
    constexpr int kU = 4;
    for (int p0 = p_lo + tid; p0 < p_hi; p0 += kU * nthr) {
        double2 e[kU], o[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int p = min(p0 + u * nthr, p_hi - 1);
            const int pm = (p == L) ? 0 : p;
            e[u] = ve[pm];
            o[u] = vo[pm];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int p = p0 + u * nthr;
            if (p < p_hi) {
                const double2 v = cadd(e[u], cmulc(o[u], T(p)));
                if (P.peers.n) *peer_ptr(P.peers, p, kg, p) = v;  // fused return transpose
                else colbase[theta_addr(P.sl, P.ncols, kl, p)] = v;
            }
        }
    }
    SK_PROBE_S(8);
    cluster_exit_barrier(relaxed_exit);  // only consumed DSMEM loads since the last cluster barrier
    SK_PROBE_S(9);
}

cudaError_t launch_pivot_table_sym(int L, int k0, int ncols, double* ipt, int stride, cudaStream_t st) {
    const int n = ncols * 2;
    pivot_table_sym_kernel<<<(n + 127) / 128, 128, 0, st>>>(L, k0, ncols, ipt, stride);
    return cudaGetLastError();
}

template <int R0>
static cudaError_t launch_sym_t(const ThetaParams& P, int nthr, size_t smem, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    configure_on_device(attr, [] {
        cudaFuncSetAttribute(theta_sym_kernel<R0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    theta_sym_kernel<R0><<<2 * P.ncols * P.nrhs, nthr, smem, st>>>(P, exit_relaxed());
    return cudaGetLastError();
}

cudaError_t launch_theta_sym(const ThetaParams& P, int nthr, size_t smem, cudaStream_t st) {
    switch (P.fd.R[0]) {
        case 2: return launch_sym_t<2>(P, nthr, smem, st);
        case 4: return launch_sym_t<4>(P, nthr, smem, st);
        case 8: return launch_sym_t<8>(P, nthr, smem, st);
        default: return launch_sym_t<16>(P, nthr, smem, st);
    }
}

}  // namespace sk
