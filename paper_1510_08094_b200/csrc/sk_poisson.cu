// Host side of the C ABI (include/sk_poisson.h): plans, device buffers, FFT
// tables, launches and the error contract.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/sk_poisson.h"
#include "params.h"
#include "sk_internal.h"

namespace {

thread_local std::string g_err;

sk_status fail(sk_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define CU(call)                                                                                       \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) return fail(SK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Radix plan for an in-place transform of length L run by `nthr` threads:
// the factorisation into register radices {2,3,4,5,7,8,10,16,20,25} that
// minimises a simple time model, sum over stages of
// ceil(L/R / nthr) * (R + 6) + 30 (rounds of butterflies per thread times a
// butterfly's cost, plus a per-stage barrier), so stages stay balanced.
void search_radices(int m, int nthr, int L, int maxr, std::vector<int>& cur, double cost, double& best,
                    std::vector<int>& out) {
    if (cost >= best) return;
    if (m == 1) {
        best = cost;
        out = cur;
        return;
    }
    if (static_cast<int>(cur.size()) >= sk::kMaxStages) return;
    static const int kRad[] = {25, 20, 16, 10, 8, 7, 5, 4, 3, 2};
    for (int r : kRad) {
        if (r > maxr || m % r != 0) continue;
        const long long nb = L / r;
        const double c = static_cast<double>((nb + nthr - 1) / nthr) * (r + 6) + 30;
        cur.push_back(r);
        search_radices(m / r, nthr, L, r, cur, cost + c, best, out);
        cur.pop_back();
    }
}

bool factor_radices(int L, int nthr, std::vector<int>& R, bool odd_first_span = false, int maxr_plan = 25) {
    R.clear();
    if (L < 1) return false;
    if (L == 1) return true;
    std::vector<int> cur;
    double best = 1e300;
    int maxr = maxr_plan;  // largest register radix (SK_MAXRADIX: A/B switch)
    if (const char* e = std::getenv("SK_MAXRADIX")) maxr = std::atoi(e);
    if (odd_first_span) {
        // First radix takes every factor of two, so consecutive natural indices
        // sit an odd number of slots apart in the digit-reversed layout and a
        // warp walking consecutive chain elements spreads over all banks.
        int p2 = 1;
        while (L % (2 * p2) == 0) p2 *= 2;
        if (p2 > 1 && p2 <= 16 && p2 <= maxr && L / p2 > 1) {
            const long long nb = L / p2;
            cur.push_back(p2);
            search_radices(L / p2, nthr, L, maxr, cur, static_cast<double>((nb + nthr - 1) / nthr) * (p2 + 6) + 30,
                           best, R);
            if (!R.empty()) return true;
            cur.clear();
            best = 1e300;
        }
    }
    search_radices(L, nthr, L, maxr, cur, 0.0, best, R);
    return !R.empty();
}

struct DevFft {
    sk::FftDesc d;
    double2* hi = nullptr;
    double2* lo = nullptr;
    int* rev = nullptr;
};

// exp(-2 pi i m / n) with exact index reduction and long double arithmetic.
void root(long long m, long long n, double& c, double& s) {
    m %= n;
    if (m < 0) m += n;
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double a = 2.0L * pi * static_cast<long double>(m) / static_cast<long double>(n);
    c = static_cast<double>(cosl(a));
    s = static_cast<double>(-sinl(a));
}

sk_status build_fft(int L, int nthr, DevFft& out, bool odd_first_span = false, bool swizzle = false, int maxr = 25) {
    std::vector<int> R;
    if (!factor_radices(L, nthr, R, odd_first_span, maxr)) return fail(SK_ERR_UNSUPPORTED, "FFT length " + std::to_string(L) + " has prime factors > 7");
    sk::FftDesc& d = out.d;
    d.L = L;
    d.nst = static_cast<int>(R.size());
    int sz = L;
    for (int s = 0; s < d.nst; ++s) {
        d.R[s] = R[s];
        d.span[s] = sz / R[s];
        d.tw[s] = 2 * L / sz;
        // Granlund-Montgomery constants for unsigned division by span[s]
        const unsigned dv = static_cast<unsigned>(d.span[s]);
        int l = 0;
        while ((1ull << l) < dv) ++l;
        d.mag[s] = static_cast<unsigned>(((1ull << 32) * ((1ull << l) - dv)) / dv + 1);
        d.sh1[s] = l < 1 ? l : 1;
        d.sh2[s] = l > 1 ? l - 1 : 0;
        sz /= R[s];
    }
    const long long n2 = 2LL * L;
    int shift = 0;
    while ((1LL << (2 * shift)) < n2) ++shift;  // B = 2^shift >= sqrt(2L)
    const int B = 1 << shift;
    d.shift = shift;
    d.nlo = B;
    d.nhi = static_cast<int>((n2 + B - 1) / B);
    std::vector<double2> hi(d.nhi), lo(d.nlo);
    for (int h = 0; h < d.nhi; ++h) root(static_cast<long long>(h) * B, n2, hi[h].x, hi[h].y);
    for (int l = 0; l < d.nlo; ++l) root(l, n2, lo[l].x, lo[l].y);
    std::vector<int> rev((L + 3) & ~3, 0);  // padded to 16 bytes for bulk copies
    for (int k = 0; k < L; ++k) {
        int kk = k, pos = 0;
        for (int s = 0; s < d.nst; ++s) {
            pos += (kk % d.R[s]) * d.span[s];
            kk /= d.R[s];
        }
        // theta plans store the swizzled shared-memory slot (fft_dev.cuh swz)
        rev[k] = (swizzle && d.nst > 0 && d.span[0] % 2 == 0) ? (pos ^ (((pos >> 3) ^ (pos >> 6) ^ (pos >> 9) ^ (pos >> 12)) & 7)) : pos;
    }
    CU(cudaMalloc(&out.hi, sizeof(double2) * d.nhi));
    CU(cudaMalloc(&out.lo, sizeof(double2) * d.nlo));
    CU(cudaMalloc(&out.rev, sizeof(int) * rev.size()));
    CU(cudaMemcpy(out.hi, hi.data(), sizeof(double2) * d.nhi, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(out.lo, lo.data(), sizeof(double2) * d.nlo, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(out.rev, rev.data(), sizeof(int) * rev.size(), cudaMemcpyHostToDevice));
    d.hi = out.hi;
    d.lo = out.lo;
    d.rev = out.rev;
    return SK_OK;
}

void free_fft(DevFft& f) {
    cudaFree(f.hi);
    cudaFree(f.lo);
    cudaFree(f.rev);
    f = DevFft{};
}

// Tensor map over a mode-major spectrum [rhs][k][p] (complex, rows p
// contiguous) as a 3-D float64 tensor {2*rows, cols, nrhs}; one box is one
// row's slice of 256 consecutive modes (box_rows = 2: rows p, p+1 together).
// step > 1: the modes first, first + step, ... (count of them) of a spectrum
// whose right-hand sides are rows * cols entries apart
sk_status make_spec_map(CUtensorMap* map, void* base, int rows, int cols, int nrhs, int box_rows = 1, int step = 1,
                        int first = 0, int count = 0, int box_modes = 256) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled is not available");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * rows), static_cast<cuuint64_t>(step > 1 ? count : cols),
                                static_cast<cuuint64_t>(nrhs)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(rows) * 16 * step, static_cast<cuuint64_t>(rows) * cols * 16};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(2 * box_rows), static_cast<cuuint32_t>(box_modes), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    base = static_cast<char*>(base) + static_cast<size_t>(first) * rows * 16;
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return SK_OK;
}

// Tensor map over the theta-stage columns (complex, contiguous, leading
// dimension `rows`) as {re/im, j mod Q, j / Q, column} for j < Q*Lq: one box
// is 256 consecutive j / Q of one residue class j mod Q.
sk_status make_col_map(CUtensorMap* map, void* base, int rows, int Q, int Lq, int ncols) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled is not available");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[4] = {2, static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(Lq),
                                static_cast<cuuint64_t>(ncols)};
    const cuuint64_t strides[3] = {16, static_cast<cuuint64_t>(Q) * 16, static_cast<cuuint64_t>(rows) * 16};
    const cuuint32_t box[4] = {2, 1, 256, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled (columns) failed (" + std::to_string(r) + ")");
    return SK_OK;
}

int round_threads(long long want, int lo, int hi) {
    long long t = ((want + 31) / 32) * 32;
    if (t < lo) t = lo;
    if (t > hi) t = hi;
    return static_cast<int>(t);
}

}  // namespace

namespace {

// z = Msin^-1 Msin^-1 w for the mean check (see coeff_kernels.cu mean_kernel),
// via the pivoted tridiagonal solve of div_sin (fourier.cpp:92-103).
std::vector<std::complex<double>> div_sin_host(const std::vector<std::complex<double>>& c) {
    // Msin (i,i+1) = +i/2, (i,i-1) = -i/2: general partial-pivoting tridiagonal
    // solve (row-permuted, width-3 windows).
    using C = std::complex<double>;
    const int n = static_cast<int>(c.size());
    std::vector<std::vector<C>> row(n, std::vector<C>(4, C{}));  // cols base..base+3
    std::vector<int> base(n);
    std::vector<C> rhs(c);
    for (int i = 0; i < n; ++i) {
        base[i] = std::max(0, i - 1);
        for (int j = base[i]; j <= std::min(n - 1, i + 1); ++j) {
            C v{};
            if (j == i + 1) v = C(0, 0.5);
            if (j == i - 1) v = C(0, -0.5);
            row[i][j - base[i]] = v;
        }
    }
    std::vector<int> perm(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    auto val = [&](int r, int col) {
        const int t = col - base[r];
        return (t >= 0 && t < 4) ? row[r][t] : C{};
    };
    auto align = [&](int r, int col) {
        const int sh = col - base[r];
        if (sh <= 0) return;
        for (int t = 0; t < 4; ++t) row[r][t] = (t + sh < 4) ? row[r][t + sh] : C{};
        base[r] = col;
    };
    for (int cc = 0; cc < n; ++cc) {
        const int last = std::min(n - 1, cc + 1);
        int piv = cc;
        double best = std::abs(val(perm[cc], cc));
        for (int r = cc + 1; r <= last; ++r)
            if (std::abs(val(perm[r], cc)) > best) {
                best = std::abs(val(perm[r], cc));
                piv = r;
            }
        std::swap(perm[cc], perm[piv]);
        align(perm[cc], cc);
        const C pv = row[perm[cc]][0];
        for (int r = cc + 1; r <= last; ++r) {
            const C v = val(perm[r], cc);
            if (v == C{}) continue;
            align(perm[r], cc);
            const C f = v / pv;
            row[perm[r]][0] = C{};
            for (int t = 1; t < 4; ++t) row[perm[r]][t] -= f * row[perm[cc]][t];
            rhs[perm[r]] -= f * rhs[perm[cc]];
        }
    }
    std::vector<C> x(n);
    for (int cc = n - 1; cc >= 0; --cc) {
        C acc = rhs[perm[cc]];
        for (int j = cc + 1; j <= std::min(n - 1, cc + 3); ++j) acc -= val(perm[cc], j) * x[j];
        x[cc] = acc / val(perm[cc], cc);
    }
    return x;
}

std::vector<std::complex<double>> mean_weights(int m) {
    std::vector<std::complex<double>> w(m);
    for (int i = 0; i < m; ++i) {
        const int k = i - m / 2;
        if (k % 2 != 0) continue;
        w[i] = 2.0 / (1.0 - static_cast<double>(k) * k);
    }
    return div_sin_host(div_sin_host(w));
}

}  // namespace

struct sk_plan_s {
    int M = 0, N = 0, nrhs = 1, device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool grid_ok = false;
    std::string grid_why;
    sk::GridGeom g;
    DevFft ft, fl;
    DevFft ftq, flh;           // local transforms of the cluster-split kernels
    int theta_q = 0;           // 0: CTA-pair theta kernel; Q: 2Q-CTA cluster kernel
    int lambda_split = 0;      // lambda rows split over a CTA pair
    int lambda_split_tma = 0;  // ... whose inverse gathers its modes through per-parity tensor maps
    int thr_theta = 0, thr_lambda = 0;
    size_t smem_theta = 0, smem_lambda = 0;
    double2* spec = nullptr;   // nrhs * cols * rows complex
    double2* spec_rows = nullptr;  // nrhs * rows * cols complex: the row-major spectrum R[rhs][p][k] (fwd_rows)
    int fwd_rows = 0;          // single-GPU solves on theta_kernel: lambda_fwd writes contiguous rows of R, theta gathers
    double* stats = nullptr;   // 4 * nrhs
    double2* z = nullptr;      // mean weights, M complex
    double* D = nullptr;       // coefficient solve: per-plan pivots d' (M x N), multipliers l behind them (M x N),
                               // then one double of table-build flags (ensure_coeff_tables)
    bool coeff_tables = false;
    double2* hF = nullptr;     // staging for host-pointer coefficient calls
    double2* hX = nullptr;
    double* hf = nullptr;      // staging for host-pointer grid calls
    double* hu = nullptr;
    double* rbuf = nullptr;    // residual output (4)
    double2* coef_stage = nullptr;  // shgen coefficients
    double* pivots = nullptr;  // theta-stage pivot table, rows (k - piv_k0, parity) for modes [piv_k0, piv_k0 + piv_n)
    int piv_k0 = 0, piv_n = 0;
    // theta-stage statistics of the stage entry points, copied to pinned host
    // memory behind the stage (sk_stage_stats waits for this event only)
    double* stage_stats_h = nullptr;
    cudaEvent_t ev_stats = nullptr;
    int kseq = 0;              // lambda modes solved by the sequential recurrence (SK_KSEQ)
    int pair_chains = 1;       // theta_kernel's segment solver pairs the chains of a parity (SK_PAIR_CHAINS=0: A/B)
    int piv_stride = 0;        // doubles per pivot-table row
    bool theta_hiocc = false;  // high-occupancy theta kernel variant (short columns)
    bool lambda_hiocc = false; // high-occupancy lambda kernel variant (short rows)
    bool lambda_pair = true;   // forward lambda rows on CTA pairs (32-byte stores); SK_LAMBDA_PAIR=0 for A/B
    // forward lambda rows on 4-CTA clusters (64-byte stores): the default for peer stores (fused multi-GPU
    // transpose; the pair kernel has no peer path); for local stores measured slower than the pair kernel at
    // C3 (0.72 vs 0.665 ms: 3/4 of the modes come through DSMEM, half of them from the other SM), so opt-in
    // there: SK_LAMBDA_QUAD=1 (=0 disables it for peer stores too)
    int lambda_quad = -1;
    // inverse lambda rows on CTA pairs (32-byte gathers): opt-in, SK_LAMBDA_PAIR_INV=1. Measured slower at C3
    // (0.80 vs 0.57 ms: the peer's modes are 16-byte DSMEM reads at a 32-byte stride)
    bool lambda_pair_inv = false;
    bool lambda_duo = false;   // opt-in A/B (SK_LAMBDA_DUO=1): both lambda stages on row pairs inside one CTA
                               // (lambda_duo.cu); measured slower at C3 than two independent CTAs per SM
    int regsolve = 1;          // chain solver request (SK_REGSOLVE): 1 auto, 0 shared-memory walk, 2 SMAX=12 registers, 3 fixed short segments
    int chain_mode = 1;        // the theta kernel's chain solver (ThetaParams::regsolve)
    int rev_win = 0;           // theta kernel stages the chains' digit-reversal windows (ThetaParams::rev_win)
    bool theta_sym = false;    // theta_sym_kernel (theta_sym.cu): pruned forward transform, both chains at once
    bool theta_mp = false;     // multi-pass theta stage (theta_mp.cu) for columns longer than one CTA
    DevFft fm1, fm2;           // its length-L1 / length-L2 transforms (16 threads per sequence)
    double2* mp_w1 = nullptr;  // its intermediates, 2 L complex per column each
    double2* mp_w2 = nullptr;
    size_t mp_cols = 0;        // columns the intermediates hold
    uint32_t* sym_pos = nullptr;  // its per-parity chain slot table (2 x theta_sym_pos_slots(M/2))
    // pipelined host-memory solves (SK_HOST | SK_ASYNC)
    static constexpr int kPipe = 3;  // device slots: H2D(i+1), solve(i), D2H(i-1) all in flight
    bool pipe_ready = false;
    double* pipe_buf[kPipe] = {};
    double* pipe_stats[kPipe] = {};  // pinned
    bool pipe_pending[kPipe] = {};
    cudaEvent_t pipe_in[kPipe] = {}, pipe_done[kPipe] = {}, pipe_out[kPipe] = {};
    cudaStream_t pipe_h2d = nullptr, pipe_d2h = nullptr;
    int pipe_slot = 0;
    long long last_launches = 0;
    bool timing = false;
    cudaEvent_t ev[8] = {};
    double times[4] = {0, 0, 0, 0};
    int ev_pending = 0;        // stages whose timing events were recorded but not yet read
    std::vector<double> host_stats;
    // standalone transforms / assemble: FFT plans per length, growable scratch
    std::map<int, DevFft> xf;
    struct BlueFft {
        DevFft f;                   // the convolution FFT, length Lb >= 2n - 1
        double2* chirp = nullptr;   // exp(-i pi j^2 / n), j < n
        double2* bhat_a = nullptr;  // FFT(conj chirp kernel) / Lb, forward transforms (analyze)
        double2* bhat_s = nullptr;  // FFT(chirp kernel) / Lb, backward transforms (synthesize)
    };
    std::map<int, BlueFft> xb;  // Bluestein plans of lengths with a prime factor > 7
    static constexpr int kScratch = 8;  // 0-3 assemble / transforms, 4-7 reference-semantics grid solve
    void* scratch[kScratch] = {};
    size_t scratch_bytes[kScratch] = {};
};

namespace {

sk_status ensure(void** p, size_t bytes) {
    if (*p) return SK_OK;
    CU(cudaMalloc(p, bytes));
    return SK_OK;
}

// The coefficient solve's data-independent elimination tables (coeff_tables_kernel).
sk_status ensure_coeff_tables(sk_plan_t p) {
    if (p->coeff_tables) return SK_OK;
    const size_t mn = static_cast<size_t>(p->M) * p->N;
    sk_status s = ensure(reinterpret_cast<void**>(&p->D), sizeof(double) * (2 * mn + 2));
    if (s != SK_OK) return s;
    CU(cudaMemsetAsync(p->D + 2 * mn, 0, sizeof(double) * 2, p->stream));
    CU(sk::launch_coeff_tables(p->M, p->N, p->D, p->D + mn, p->D + 2 * mn, p->stream));
    p->coeff_tables = true;
    return SK_OK;
}

// Half spectrum of single-GPU grid solves (nrhs x (N/2+1) x (M/2+1) complex).
sk_status ensure_spec(sk_plan_t p) {
    return ensure(reinterpret_cast<void**>(&p->spec), sizeof(double2) * p->nrhs * p->g.rows * p->g.cols);
}

// Pivot rows of the modes [k0, k0 + n): built by the plan's pivot kernel on
// first use (a slab rank asks for its own modes only), rebuilt if a later
// call needs modes outside the cached range.
sk_status ensure_pivots(sk_plan_t p, int k0, int n) {
    if (p->pivots && k0 >= p->piv_k0 && k0 + n <= p->piv_k0 + p->piv_n) return SK_OK;
    if (p->pivots) {
        CU(cudaStreamSynchronize(p->stream));
        CU(cudaFree(p->pivots));
        p->pivots = nullptr;
    }
    const size_t np = static_cast<size_t>(n) * 2 * p->piv_stride;
    sk_status s = ensure(reinterpret_cast<void**>(&p->pivots), sizeof(double) * (np ? np : 2));
    if (s != SK_OK) return s;
    p->piv_k0 = k0;
    p->piv_n = n;
    if (n > 0) {
        CU((p->theta_sym || p->theta_mp) ? sk::launch_pivot_table_sym(p->g.Lt, k0, n, p->pivots, p->piv_stride, p->stream)
                                         : sk::launch_pivot_table(p->g.Lt, k0, n, p->pivots, p->piv_stride, p->stream));
    }
    return SK_OK;
}

sk_status check_plan(sk_plan_t p) {
    if (!p) return fail(SK_ERR_ARGUMENT, "null plan");
    CU(cudaSetDevice(p->device));
    return SK_OK;
}

sk_status precondition_from(const double* st, int nrhs) {
    // poisson.cpp:111-116: |2 pi w^T f0| > 1e-6 * 4 pi * max|F|
    const double fourpi = 12.566370614359172953850573533118;
    for (int r = 0; r < nrhs; ++r) {
        const double* s = &st[4 * r];
        if (s[3] >= double(1 << 20))
            return fail(SK_ERR_SINGULAR, "band_solve: matrix is numerically singular");
        const double fscale = s[2];
        if (fscale == 0.0) continue;
        const double mean = std::hypot(s[0], s[1]);
        if (mean > 1e-6 * fourpi * fscale)
            return fail(SK_ERR_PRECONDITION, "poisson solve: right-hand side has a nonzero surface mean");
    }
    return SK_OK;
}

sk_status check_precondition(sk_plan_t p, int nrhs) {
    p->host_stats.resize(4 * nrhs);
    CU(cudaMemcpyAsync(p->host_stats.data(), p->stats, sizeof(double) * 4 * nrhs, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    return precondition_from(p->host_stats.data(), nrhs);
}

// Host-memory solves with SK_ASYNC: three device slots, the H2D copy of a
// solve on its own stream, the transforms on the plan stream, the D2H copy on
// a third stream, so consecutive solves overlap their copies (both directions
// of the link) with each other's compute; with three slots the H2D of solve
// i+1 never waits for the D2H of solve i-1, and the period is the slowest of
// the two copies and the solve.  The precondition of a solve is
// evaluated when its slot comes round again or at sk_sync.
sk_status pipe_check_slot(sk_plan_t p, int slot) {
    if (!p->pipe_pending[slot]) return SK_OK;
    p->pipe_pending[slot] = false;
    CU(cudaEventSynchronize(p->pipe_done[slot]));
    return precondition_from(p->pipe_stats[slot], p->nrhs);
}

sk_status pipe_init(sk_plan_t p, size_t ng) {
    if (p->pipe_ready) return SK_OK;
    for (int i = 0; i < sk_plan_s::kPipe; ++i) {
        CU(cudaMalloc(&p->pipe_buf[i], sizeof(double) * ng));
        CU(cudaMallocHost(&p->pipe_stats[i], sizeof(double) * 4 * p->nrhs));
        CU(cudaEventCreateWithFlags(&p->pipe_in[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->pipe_done[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->pipe_out[i], cudaEventDisableTiming));
    }
    CU(cudaStreamCreateWithFlags(&p->pipe_h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&p->pipe_d2h, cudaStreamNonBlocking));
    p->pipe_ready = true;
    return SK_OK;
}

}  // namespace

#ifdef SK_PHASES
namespace sk { extern __device__ unsigned long long g_phase[4096][24]; }
extern "C" int sk_debug_phases(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, sk::g_phase, sizeof(unsigned long long) * 4096 * 24) == cudaSuccess ? 0 : 1;
}
namespace sk { extern __device__ unsigned long long g_phase_l[2][4096][8]; }
extern "C" int sk_debug_phases_lambda(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, sk::g_phase_l, sizeof(unsigned long long) * 2 * 4096 * 8) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" {

static void collect_times(sk_plan_t p, int stages);

const char* sk_last_error(void) { return g_err.c_str(); }
const char* sk_version(void) { return "sk_poisson 0.1 (sm_100a)"; }

sk_status sk_plan_create(int M, int N, int nrhs, int device, sk_plan_t* out) {
    if (!out) return fail(SK_ERR_ARGUMENT, "null output plan pointer");
    *out = nullptr;
    if (M <= 0 || N <= 0 || M % 2 != 0 || N % 2 != 0)
        return fail(SK_ERR_SIZE, "poisson solve: sizes must be positive and even");
    if (nrhs < 1) return fail(SK_ERR_ARGUMENT, "nrhs must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(SK_ERR_CUDA, "no CUDA device available (the solver has no CPU fallback)");
    if (device < 0 || device >= ndev) return fail(SK_ERR_ARGUMENT, "bad device ordinal");
    CU(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(SK_ERR_CUDA, "this build targets sm_100a (Blackwell); device is sm_" +
                                                      std::to_string(prop.major) + std::to_string(prop.minor));
    auto* p = new sk_plan_s;
    p->M = M;
    p->N = N;
    p->nrhs = nrhs;
    p->device = device;
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete p;
        return fail(SK_ERR_CUDA, "stream creation failed");
    }
    p->own_stream = true;
    if (const char* e = std::getenv("SK_KSEQ")) p->kseq = std::atoi(e);
    if (const char* e = std::getenv("SK_PAIR_CHAINS")) p->pair_chains = std::atoi(e) != 0;
    if (const char* e = std::getenv("SK_REGSOLVE")) p->regsolve = std::atoi(e);
    p->g.M = M;
    p->g.N = N;
    p->g.Lt = M / 2;
    p->g.Ll = N / 2;
    p->g.rows = M / 2 + 1;
    p->g.cols = N / 2 + 1;
    p->g.pole_glide = sk::pole_glide(M);
    sk_status s;
    if ((s = ensure(reinterpret_cast<void**>(&p->stats), sizeof(double) * 4 * nrhs)) != SK_OK) {
        sk_plan_destroy(p);
        return s;
    }
    // mean weights
    {
        const auto z = mean_weights(M);
        if ((s = ensure(reinterpret_cast<void**>(&p->z), sizeof(double2) * M)) != SK_OK) {
            sk_plan_destroy(p);
            return s;
        }
        if (cudaMemcpy(p->z, z.data(), sizeof(double2) * M, cudaMemcpyHostToDevice) != cudaSuccess) {
            sk_plan_destroy(p);
            return fail(SK_ERR_CUDA, "copy of mean weights failed");
        }
    }
    // grid path: FFT plans + on-chip limits
    p->grid_ok = true;
    if (M < 8 || N < 4) {
        p->grid_ok = false;
        p->grid_why = "grid path needs M >= 8 and N >= 4";
    }
    const size_t cap = 227 * 1024;
    const int Lt = M / 2, Ll = N / 2;
    // theta stage: one CTA pair per mode when a parity half fits shared
    // memory, else a cluster of 2Q CTAs (Q = 4) holding quarters
    p->thr_theta = round_threads(Lt / 8, 64, 512);
    if (const char* e = std::getenv("SK_THETA_THREADS")) p->thr_theta = round_threads(std::atoi(e), 64, 512);  // A/B
    const bool odd_t = !std::getenv("SK_ODDSPAN_THETA") || std::atoi(std::getenv("SK_ODDSPAN_THETA")) != 0;
    const bool odd_l = !std::getenv("SK_ODDSPAN_LAMBDA") || std::atoi(std::getenv("SK_ODDSPAN_LAMBDA")) != 0;
    // short columns (<= 256 threads per CTA) run the high-occupancy theta
    // variant: 64 registers per thread, register radices <= 8, fold and
    // chains within its per-thread limits (SK_NO_HIOCC: A/B switch)
    p->theta_hiocc = p->thr_theta <= 256 && (Lt / 2 + 1) <= 6 * p->thr_theta /* kFoldMaxHi */ &&
                     (Lt / 2 + 1) <= 6 * p->thr_theta && !std::getenv("SK_NO_HIOCC");
    if (p->grid_ok && (s = build_fft(Lt, p->thr_theta, p->ft, odd_t, true, p->theta_hiocc ? 8 : 25)) != SK_OK) {
        p->grid_ok = false;
        p->grid_why = g_err;
    }
    for (int st = 0; p->theta_hiocc && st < p->ft.d.nst; ++st)
        if (p->ft.d.R[st] > 8) p->theta_hiocc = false;  // the variant only instantiates radices <= 8
    if (p->grid_ok) {
        p->smem_theta = sk::theta_smem_bytes(Lt, p->ft.d.nhi, p->ft.d.nlo);
        // stage the chains' digit-reversal entries in shared memory when they fit
        const size_t with_rev = sk::theta_smem_bytes(Lt, p->ft.d.nhi, p->ft.d.nlo, true);
        if (Lt >= 4096 && with_rev <= cap && !std::getenv("SK_NO_REVWIN")) {  // small tables stay L1-resident
            p->smem_theta = with_rev;
            p->rev_win = 1;
        }
        const bool fits = p->smem_theta <= cap && (Lt / 2 + 1) <= 12 * p->thr_theta;
        const bool want_mp = !std::getenv("SK_THETA_MP") || std::atoi(std::getenv("SK_THETA_MP")) != 0;
        if (!fits && want_mp && p->kseq == 0 && Lt % 2 == 0 && Lt / 2 <= sk::theta_mp_chain_cap()) {
            // multi-pass theta stage: L = L1 L2 with L1 % 16 == 0, L2 % 32 == 0,
            // both <= 384 (a CTA's 16 sequences in shared memory), L1 <= L2 closest
            int best1 = 0;
            const bool wide = std::getenv("SK_MP_WIDE") && std::atoi(std::getenv("SK_MP_WIDE")) != 0;  // A/B: L1 >= L2
            for (int l1 = 16; l1 <= 256; l1 *= 2) {  // powers of two (the passes index by shifts)
                if (Lt % l1) continue;
                const int l2 = Lt / l1;
                if (l2 % 32 || l2 > 384 || (l2 & (l2 - 1))) continue;
                if (!wide && l1 > l2) continue;
                if (wide && l1 < l2) continue;
                if (!wide || !best1) best1 = l1;  // narrow: the most balanced (last); wide: the first with L1 >= L2
            }
            if (best1) {
                const int l1 = best1, l2 = Lt / best1;
                if (build_fft(l1, 16, p->fm1, false, false, 8) == SK_OK &&
                    build_fft(l2, 16, p->fm2, false, false, 8) == SK_OK) {
                    p->theta_mp = true;
                    p->thr_theta = 512;
                    p->smem_theta = std::max({sk::theta_mp_smem_bytes(0, l1, l2, p->fm1.d.nhi, p->fm1.d.nlo, p->fm2.d.nhi,
                                                                      p->fm2.d.nlo, p->ft.d.nhi, p->ft.d.nlo),
                                              sk::theta_mp_smem_bytes(2, l1, l2, p->fm1.d.nhi, p->fm1.d.nlo, p->fm2.d.nhi,
                                                                      p->fm2.d.nlo, p->ft.d.nhi, p->ft.d.nlo),
                                              sk::theta_mp_smem_bytes(3, l1, l2, 0, 0, 0, 0, 0, 0)});
                    if (p->smem_theta > cap) p->theta_mp = false;
                }
                if (!p->theta_mp) {
                    free_fft(p->fm1);
                    free_fft(p->fm2);
                    p->fm1 = DevFft{};
                    p->fm2 = DevFft{};
                }
            }
        }
        if (!fits && !p->theta_mp) {
            const int Q = 4;
            const int Lq = Lt / Q;
            p->theta_q = Q;
            p->thr_theta = 512;
            if (Lt % (2 * Q) != 0 || (s = build_fft(Lq, 512, p->ftq)) != SK_OK) {
                p->grid_ok = false;
                p->grid_why = "theta length " + std::to_string(Lt) + " cannot be split over a " +
                              std::to_string(2 * Q) + "-CTA cluster";
            } else {
                p->smem_theta = sk::theta_large_smem_bytes(Lq, p->ft.d.nhi, p->ft.d.nlo, p->ftq.d.nhi, p->ftq.d.nlo);
                if (p->smem_theta > cap || Lq > 16 * 512) {
                    p->grid_ok = false;
                    p->grid_why = "theta length " + std::to_string(Lt) + " exceeds the cluster shared-memory limit";
                }
            }
        }
    }
    // lambda stages: one CTA per row, or a CTA pair splitting the row by parity
    // (odd first span: the digit-reversed split/pack walks spread over all banks)
    p->thr_lambda = round_threads(Ll / 8, 64, 256);
    if (const char* e = std::getenv("SK_LAMBDA_THREADS")) p->thr_lambda = round_threads(std::atoi(e), 64, 256);  // A/B
    // short rows (<= 128 threads per CTA) run the high-occupancy lambda variant
    // (64 registers, radices <= 8, <= 6 mode pairs per thread; SK_NO_HIOCC)
    p->lambda_hiocc = p->thr_lambda <= 128 && (Ll / 2 + 1) <= 6 * p->thr_lambda && !std::getenv("SK_NO_HIOCC");
    if (const char* e = std::getenv("SK_LAMBDA_PAIR")) p->lambda_pair = std::atoi(e) != 0;  // A/B
    if (const char* e = std::getenv("SK_LAMBDA_QUAD")) p->lambda_quad = std::atoi(e) != 0 ? 1 : 0;  // A/B
    if (const char* e = std::getenv("SK_LAMBDA_PAIR_INV")) p->lambda_pair_inv = std::atoi(e) != 0;  // opt-in A/B
    if (const char* e = std::getenv("SK_LAMBDA_DUO")) p->lambda_duo = std::atoi(e) != 0;  // A/B
    // row-major forward spectrum + gathered theta columns (run_grid): on for theta_kernel solves of at
    // least 2^23 spectral entries, where several theta CTAs per SM hide the gather (C4 2.48 -> 2.43 ms,
    // 8 x 4096 x 2048 -3.1 %, 8192^2 -1.4 %; C2 -0.8 %, C1 +1.4 %, C3's one-CTA-per-SM theta_sym +3 %:
    // profiles/r2_phases_c3.md); SK_FWD_ROWS=0/1 forces it
    p->fwd_rows = static_cast<size_t>(p->nrhs) * p->g.rows * p->g.cols >= (static_cast<size_t>(1) << 23);
    if (const char* e = std::getenv("SK_FWD_ROWS")) p->fwd_rows = std::atoi(e) != 0;      // A/B
    if (p->grid_ok && (s = build_fft(Ll, p->thr_lambda, p->fl, odd_l, false, p->lambda_hiocc ? 8 : 25)) != SK_OK) {
        p->grid_ok = false;
        p->grid_why = g_err;
    }
    for (int st = 0; p->lambda_hiocc && st < p->fl.d.nst; ++st)
        if (p->fl.d.R[st] > 8) p->lambda_hiocc = false;
    if (p->grid_ok) {
        p->smem_lambda = sk::lambda_smem_bytes(Ll, p->fl.d.nhi, p->fl.d.nlo);
        const bool fits = p->smem_lambda <= cap && (Ll / 2 + 1) <= 12 * p->thr_lambda;
        if (!fits) {
            p->lambda_split = 1;
            p->thr_lambda = 512;
            if (Ll % 4 != 0 || (s = build_fft(Ll / 2, 512, p->flh)) != SK_OK) {
                p->grid_ok = false;
                p->grid_why = "lambda length " + std::to_string(Ll) + " cannot be split over a CTA pair";
            } else {
                // the inverse gathers through tensor maps when every thread can hold its
                // mode pairs in registers and whole gather boxes fit (SK_SPLIT_TMA=0: A/B)
                const bool want_tma = !std::getenv("SK_SPLIT_TMA") || std::atoi(std::getenv("SK_SPLIT_TMA")) != 0;
                p->lambda_split_tma = want_tma && Ll / 4 + 1 <= sk::kSplitPairs * 512 &&
                                      sk::lambda_split_smem_bytes(Ll / 2, p->fl.d.nhi, p->fl.d.nlo, p->flh.d.nhi,
                                                                  p->flh.d.nlo, true) <= cap;
                p->smem_lambda = sk::lambda_split_smem_bytes(Ll / 2, p->fl.d.nhi, p->fl.d.nlo, p->flh.d.nhi,
                                                             p->flh.d.nlo, p->lambda_split_tma != 0);
                if (p->smem_lambda > cap) {
                    p->grid_ok = false;
                    p->grid_why = "lambda length " + std::to_string(Ll) + " exceeds the CTA-pair shared-memory limit";
                }
            }
        }
    }
    if (p->grid_ok) {
        // the half spectrum (single-GPU solves) and the pivot table are
        // allocated on first use (ensure_spec / ensure_pivots): a slab rank
        // never holds the whole spectrum, only its own modes' pivots
        // data-independent Thomas pivots of every (lambda mode, parity) chain
        p->piv_stride = p->g.Lt + (p->g.Lt & 1);
        // chain solver: fixed short segments up to 6 elements per thread, the
        // 12-element register walk above (it keeps F in registers without
        // spilling there), the shared-memory walk beyond
        {
            const int nmax = p->g.Lt / 2 + 1;
            const int need = (nmax + p->thr_theta - 1) / p->thr_theta;
            p->chain_mode = p->regsolve == 0 ? 0 : p->regsolve == 2 ? 2 : p->regsolve == 3 ? 1 : (need <= 6 ? 1 : 2);
        }
        // theta_sym_kernel: long even columns on the one-CTA-per-parity path
        // whose plan starts with a power-of-two radix over an odd span
        {
            const int Lt2 = p->g.Lt, R0 = p->ft.d.nst > 0 ? p->ft.d.R[0] : 0;
            const bool pow2 = R0 >= 2 && R0 <= 16 && (R0 & (R0 - 1)) == 0;
            const bool want = !std::getenv("SK_THETA_SYM") || std::atoi(std::getenv("SK_THETA_SYM")) != 0;
            p->theta_sym = want && !p->theta_q && !p->theta_hiocc && p->kseq == 0 && Lt2 % 2 == 0 && Lt2 < 65536 &&
                           pow2 && p->ft.d.span[0] % 2 == 1 && p->ft.d.nst >= 2 && Lt2 / 2 <= 12 * p->thr_theta &&
                           sk::theta_sym_smem_bytes(Lt2, p->ft.d.nhi, p->ft.d.nlo) <= cap;
        }
        if (p->theta_mp) p->piv_stride = sk::theta_sym_piv_slots(p->g.Lt);  // pivot_table_sym_kernel rows
        if (p->theta_sym) {
            const int Lt2 = p->g.Lt;
            p->piv_stride = sk::theta_sym_piv_slots(Lt2);
            p->smem_theta = sk::theta_sym_smem_bytes(Lt2, p->ft.d.nhi, p->ft.d.nlo);
            p->rev_win = 0;
            // chain element i of parity par -> (slot of tau+ = tau0 + i) | (slot of tau- = L - 1 - i) << 16
            const int ps = sk::theta_sym_pos_slots(Lt2);
            std::vector<uint32_t> tab(2 * static_cast<size_t>(ps), 0u);
            auto slot = [&](int tau) {
                int kk = tau, pos = 0;
                for (int st = 0; st < p->ft.d.nst; ++st) {
                    pos += (kk % p->ft.d.R[st]) * p->ft.d.span[st];
                    kk /= p->ft.d.R[st];
                }
                return static_cast<uint32_t>(pos);
            };
            for (int par = 0; par < 2; ++par)
                for (int i = 0; i < Lt2 / 2; ++i) {
                    const int tp = (par == 0 ? 1 : 0) + i, tm = Lt2 - 1 - i;
                    tab[static_cast<size_t>(par) * ps + i] = (tp < Lt2 ? slot(tp) : 0u) | (slot(tm) << 16);
                }
            if ((s = ensure(reinterpret_cast<void**>(&p->sym_pos), sizeof(uint32_t) * tab.size())) != SK_OK) {
                sk_plan_destroy(p);
                return s;
            }
            if (cudaMemcpy(p->sym_pos, tab.data(), sizeof(uint32_t) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
                sk_plan_destroy(p);
                return fail(SK_ERR_CUDA, "copy of the chain slot table failed");
            }
        }
    }
    *out = p;
    return SK_OK;
}

sk_status sk_plan_destroy(sk_plan_t p) {
    if (!p) return SK_OK;
    cudaSetDevice(p->device);
    free_fft(p->ft);
    free_fft(p->fl);
    free_fft(p->ftq);
    free_fft(p->flh);
    free_fft(p->fm1);
    free_fft(p->fm2);
    if (p->mp_w1) cudaFree(p->mp_w1);
    if (p->mp_w2) cudaFree(p->mp_w2);
    if (p->spec_rows) cudaFree(p->spec_rows);
    for (void* q : {static_cast<void*>(p->spec), static_cast<void*>(p->stats), static_cast<void*>(p->z),
                    static_cast<void*>(p->D), static_cast<void*>(p->hF), static_cast<void*>(p->hX),
                    static_cast<void*>(p->hf), static_cast<void*>(p->hu), static_cast<void*>(p->rbuf),
                    static_cast<void*>(p->coef_stage), static_cast<void*>(p->pivots), static_cast<void*>(p->sym_pos)})
        if (q) cudaFree(q);
    for (auto& e : p->ev)
        if (e) cudaEventDestroy(e);
    for (auto& kv : p->xf) free_fft(kv.second);
    for (auto& kv : p->xb) {
        free_fft(kv.second.f);
        cudaFree(kv.second.chirp);
        cudaFree(kv.second.bhat_a);
        cudaFree(kv.second.bhat_s);
    }
    for (void* q : p->scratch)
        if (q) cudaFree(q);
    if (p->pipe_ready) {
        cudaStreamSynchronize(p->pipe_h2d);
        cudaStreamSynchronize(p->pipe_d2h);
        cudaStreamSynchronize(p->stream);
        for (int i = 0; i < sk_plan_s::kPipe; ++i) {
            cudaFree(p->pipe_buf[i]);
            cudaFreeHost(p->pipe_stats[i]);
            cudaEventDestroy(p->pipe_in[i]);
            cudaEventDestroy(p->pipe_done[i]);
            cudaEventDestroy(p->pipe_out[i]);
        }
        cudaStreamDestroy(p->pipe_h2d);
        cudaStreamDestroy(p->pipe_d2h);
    }
    if (p->stage_stats_h) cudaFreeHost(p->stage_stats_h);
    if (p->ev_stats) cudaEventDestroy(p->ev_stats);
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
    delete p;
    return SK_OK;
}

sk_status sk_plan_set_stream(sk_plan_t p, void* stream) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
    p->stream = static_cast<cudaStream_t>(stream);
    p->own_stream = false;
    return SK_OK;
}

sk_status sk_sync(sk_plan_t p) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    CU(cudaStreamSynchronize(p->stream));
    if (p->pipe_ready) {
        CU(cudaStreamSynchronize(p->pipe_h2d));
        CU(cudaStreamSynchronize(p->pipe_d2h));
        sk_status first = SK_OK;
        for (int i = 0; i < sk_plan_s::kPipe; ++i) {
            const sk_status a = pipe_check_slot(p, (p->pipe_slot + i) % sk_plan_s::kPipe);  // oldest first
            if (first == SK_OK) first = a;
        }
        if (first != SK_OK) return first;
    }
    return SK_OK;
}

sk_status sk_enable_stage_timing(sk_plan_t p, int on) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (on && !p->ev[0])
        for (auto& e : p->ev) CU(cudaEventCreate(&e));
    p->timing = on != 0;
    return SK_OK;
}

sk_status sk_stage_times(sk_plan_t p, double t[4]) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!t) return fail(SK_ERR_ARGUMENT, "null output");
    collect_times(p, 7);  // stage entry points (slab path) leave their events to be read here
    for (int i = 0; i < 4; ++i) t[i] = p->times[i];
    return SK_OK;
}

sk_status sk_plan_info(sk_plan_t p, long long info[16]) {
    if (!p || !info) return fail(SK_ERR_ARGUMENT, "null argument");
    for (int i = 0; i < 16; ++i) info[i] = 0;
    info[0] = p->M;
    info[1] = p->N;
    info[2] = p->nrhs;
    info[3] = p->device;
    info[4] = p->grid_ok ? 1 : 0;
    info[5] = p->g.rows;
    info[6] = p->theta_q ? 2 * p->theta_q : 2;
    info[7] = p->thr_theta;
    info[8] = p->thr_lambda;
    info[9] = p->last_launches;
    info[10] = static_cast<long long>(p->smem_theta);
    info[11] = static_cast<long long>(p->smem_lambda);
    info[12] = p->chain_mode;
    const bool swz_t = p->ft.d.nst > 0 && p->ft.d.span[0] % 2 == 0;
    const bool swz_l = p->fl.d.nst > 0 && p->fl.d.span[0] % 2 == 0;
    info[13] = (p->theta_hiocc && !p->theta_q && p->chain_mode == 1 && p->thr_theta <= 256 ? 1 : 0) |
               (p->lambda_hiocc && !p->lambda_split ? 2 : 0) | (swz_t ? 4 : 0) | (swz_l ? 8 : 0);
    const bool hi_l = p->lambda_hiocc && !p->lambda_split;
    if (p->grid_ok && p->lambda_pair && !p->lambda_split && !swz_l && !hi_l && p->nrhs == 1 && p->thr_lambda <= 256 &&
        p->N / 4 + 1 <= 12 * p->thr_lambda)
        info[13] |= 16;  // forward lambda rows on CTA pairs (lambda_pair_ok, local stores)
    if (p->grid_ok && p->lambda_pair_inv && !p->lambda_split && !swz_l && !hi_l && p->nrhs == 1 &&
        p->thr_lambda <= 256 && p->N / 4 + 1 <= 12 * p->thr_lambda && (p->N / 2 / 256 + 1) % 2 == 0)
        info[13] |= 32;  // inverse lambda rows on CTA pairs (lambda_inv_pair_ok)
    if (p->grid_ok && p->lambda_duo && !p->lambda_split && !swz_l && !hi_l && p->nrhs == 1 && p->thr_lambda <= 256 &&
        p->N / 4 + 1 <= 12 * p->thr_lambda &&
        sk::lambda_duo_smem_bytes(p->g.Ll, p->fl.d.nhi, p->fl.d.nlo) <= 227 * 1024)
        info[13] |= 512;  // lambda stages on row pairs inside one CTA (lambda_duo_ok; the forward one for local stores)
    if (p->theta_sym) info[13] |= 64;  // theta_sym_kernel
    if (p->fwd_rows && !p->theta_sym && !p->theta_q && !p->theta_mp && !p->lambda_split && !p->lambda_duo)
        info[13] |= 1024;  // row-major forward spectrum, theta_kernel gathers its columns (single-GPU solves)
    if (p->theta_mp) info[13] |= 256;  // multi-pass theta stage (theta_mp.cu)
    if (p->grid_ok && p->lambda_quad != 0 && !p->lambda_split && !swz_l && !hi_l && p->nrhs == 1 &&
        p->thr_lambda <= 256 && p->N / 4 + 1 <= 12 * p->thr_lambda)
        info[13] |= 128;  // forward lambda rows on 4-CTA clusters: peer stores (default) or any (SK_LAMBDA_QUAD=1)
    return SK_OK;
}

sk_status sk_solve_coeffs(sk_plan_t p, const double* F, double* X, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!F || !X) return fail(SK_ERR_ARGUMENT, "null F or X");
    const size_t n = static_cast<size_t>(p->nrhs) * p->M * p->N;
    const double2* dF;
    double2* dX;
    if (flags & SK_DEVICE) {
        dF = reinterpret_cast<const double2*>(F);
        dX = reinterpret_cast<double2*>(X);
    } else {
        if ((s = ensure(reinterpret_cast<void**>(&p->hF), sizeof(double2) * n)) != SK_OK) return s;
        if ((s = ensure(reinterpret_cast<void**>(&p->hX), sizeof(double2) * n)) != SK_OK) return s;
        CU(cudaMemcpyAsync(p->hF, F, sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
        dF = p->hF;
        dX = p->hX;
    }
    if ((s = ensure_coeff_tables(p)) != SK_OK) return s;
    CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4 * p->nrhs, p->stream));
    const size_t mn1 = static_cast<size_t>(p->M) * p->N;
    sk::CoeffParams cp{p->M, p->N, p->nrhs, dF, dX, p->D, p->D + mn1, p->D + 2 * mn1, p->stats, p->z};
    if (p->timing) CU(cudaEventRecord(p->ev[6], p->stream));
    CU(sk::launch_coeff_solve(cp, p->stream));
    if (p->timing) CU(cudaEventRecord(p->ev[7], p->stream));
    p->last_launches = 2;
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(X, dX, sizeof(double2) * n, cudaMemcpyDeviceToHost, p->stream));
    if ((flags & SK_ASYNC) && (flags & SK_DEVICE)) return SK_OK;
    s = check_precondition(p, p->nrhs);
    if (p->timing) {
        float ms = 0;
        cudaEventElapsedTime(&ms, p->ev[6], p->ev[7]);
        p->times[3] = ms;
    }
    return s;
}

sk_status sk_residual(sk_plan_t p, const double* F, const double* X, double out[3], unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!F || !X || !out) return fail(SK_ERR_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(p->M) * p->N;
    const double2 *dF, *dX;
    if (flags & SK_DEVICE) {
        dF = reinterpret_cast<const double2*>(F);
        dX = reinterpret_cast<const double2*>(X);
    } else {
        if ((s = ensure(reinterpret_cast<void**>(&p->hF), sizeof(double2) * n * p->nrhs)) != SK_OK) return s;
        if ((s = ensure(reinterpret_cast<void**>(&p->hX), sizeof(double2) * n * p->nrhs)) != SK_OK) return s;
        CU(cudaMemcpyAsync(p->hF, F, sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
        CU(cudaMemcpyAsync(p->hX, X, sizeof(double2) * n, cudaMemcpyHostToDevice, p->stream));
        dF = p->hF;
        dX = p->hX;
    }
    if ((s = ensure(reinterpret_cast<void**>(&p->rbuf), sizeof(double) * 4)) != SK_OK) return s;
    CU(cudaMemsetAsync(p->rbuf, 0, sizeof(double) * 4, p->stream));
    sk::ResidualParams rp{p->M, p->N, dF, dX, p->rbuf};
    CU(sk::launch_residual(rp, p->stream));
    p->last_launches = 1;
    double h[4];
    CU(cudaMemcpyAsync(h, p->rbuf, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    out[0] = h[0];
    out[1] = h[1];
    out[2] = 6.283185307179586476925286766559 * std::hypot(h[2], h[3]);
    return SK_OK;
}

static sk_status run_grid(sk_plan_t p, const sk::Slabs& sl, int rows_local, int ncols_local, int k0,
                          const double* f_dev, double2* spec, double* u_dev, double2* xhalf, int stages,
                          const sk::PeerMap* peers = nullptr) {
    // stages bit 0: lambda fwd, bit 1: theta, bit 2: lambda inv
    sk::LambdaParams lp{};
    lp.g = p->g;
    lp.fd = p->fl.d;
    lp.swizzle = (p->fl.d.nst > 0 && p->fl.d.span[0] % 2 == 0) ? 1 : 0;  // power-of-two rows
    lp.hiocc = p->lambda_hiocc && !p->lambda_split ? 1 : 0;
    lp.pair = (p->lambda_pair ? 1 : 0) | ((p->lambda_quad == 1 || (p->lambda_quad < 0 && peers)) ? 4 : 0);
    lp.rows_local = rows_local;
    lp.nrhs = (sl.P == 1) ? p->nrhs : 1;
    // row-major forward spectrum + gathered theta columns: whole single-GPU solves on theta_kernel
    bool fwd_rows = false;
    if (p->fwd_rows && sl.P == 1 && !peers && (stages & 3) == 3 && !p->theta_sym && !p->theta_q &&
        !p->theta_mp && !p->lambda_split && !p->lambda_duo) {
        const sk_status es =
            ensure(reinterpret_cast<void**>(&p->spec_rows), sizeof(double2) * p->nrhs * p->g.rows * p->g.cols);
        if (es != SK_OK) return es;
        fwd_rows = true;
    }
    if (stages & 1) {
        lp.in_rhs_stride = static_cast<long long>(rows_local) * p->N;
        lp.out_rhs_stride = static_cast<long long>(rows_local) * p->g.cols;
        lp.f = f_dev;
        lp.spec = spec;
        if (peers) lp.peers = *peers;
        if (p->timing) CU(cudaEventRecord(p->ev[0], p->stream));
        if (p->lambda_split) {
            // (measured and not kept at C5: boxed TMA stores of the modes, 12.4 vs 11.8 ms; row pairs on
            // 4-CTA clusters for 32-byte stores, 12.4 vs 11.3 ms)
            sk::LambdaSplitParams sp{lp, p->flh.d, sk::lambda_split_slots(p->fl.d.L / 2, p->lambda_split_tma != 0), 0};
            CU(sk::launch_lambda_fwd_split(sp, p->thr_lambda, p->smem_lambda, p->stream));
        } else if (p->lambda_duo && !peers && sk::lambda_duo_ok(lp, p->thr_lambda)) {
            CU(sk::launch_lambda_fwd_duo(lp, p->thr_lambda, p->stream));
        } else {
            CUtensorMap map;
            sk_status ms = make_spec_map(&map, spec, rows_local, p->g.cols, lp.nrhs);
            if (ms != SK_OK) return ms;
            if (fwd_rows) {
                lp.pair |= 8;
                lp.spec = p->spec_rows;
            }
            CU(sk::launch_lambda_fwd(lp, map, p->thr_lambda, p->smem_lambda, p->stream));
            lp.pair &= ~8;
            lp.spec = spec;
        }
        if (p->timing) {
            CU(cudaEventRecord(p->ev[1], p->stream));
            p->ev_pending |= 1;
        }
        p->last_launches += 1;
    }
    if (stages & 2) {
        sk::ThetaParams tp{};
        tp.g = p->g;
        tp.fd = p->ft.d;
        tp.sl = sl;
        tp.buf = spec;
        tp.ncols = ncols_local;
        tp.k0 = k0;
        tp.nrhs = (sl.P == 1) ? p->nrhs : 1;
        tp.rhs_stride = static_cast<long long>(p->g.rows) * ncols_local;
        tp.stats = p->stats;
        tp.xhalf = xhalf;
        tp.kseq = p->kseq;
        tp.pair_chains = p->pair_chains;
        tp.regsolve = p->chain_mode;
        tp.hiocc = p->theta_hiocc ? 1 : 0;
        tp.rev_win = p->theta_q ? 0 : p->rev_win;
        tp.swizzle = p->ft.d.nst > 0 && (p->ft.d.span[0] % 2 == 0) ? 1 : 0;
        {
            const sk_status ps = ensure_pivots(p, k0, ncols_local);
            if (ps != SK_OK) return ps;
        }
        tp.pivots = p->pivots + static_cast<size_t>(k0 - p->piv_k0) * 2 * p->piv_stride;  // rows for this rank's modes
        tp.sym_pos = p->sym_pos;
        tp.piv_stride = p->piv_stride;
        if (peers) tp.peers = *peers;
        if (p->timing) CU(cudaEventRecord(p->ev[2], p->stream));
        if (p->theta_mp) {
            const size_t cols = static_cast<size_t>(ncols_local) * tp.nrhs;
            if (cols > p->mp_cols) {
                if (p->mp_w1) {
                    CU(cudaStreamSynchronize(p->stream));
                    CU(cudaFree(p->mp_w1));
                    CU(cudaFree(p->mp_w2));
                    p->mp_w1 = p->mp_w2 = nullptr;
                }
                CU(cudaMalloc(&p->mp_w1, sizeof(double2) * 2 * p->g.Lt * cols));
                CU(cudaMalloc(&p->mp_w2, sizeof(double2) * 2 * p->g.Lt * cols));
                p->mp_cols = cols;
            }
            sk::ThetaMpParams mq{tp, p->fm1.d, p->fm2.d, p->mp_w1, p->mp_w2};
            CU(sk::launch_theta_mp(mq, p->stream));
        } else if (p->theta_q) {
            sk::ThetaLargeParams tl{tp, p->ftq.d, 0, 0};
            CUtensorMap cmap{};
            {
                // fold inputs by TMA when the columns are contiguous (one rank)
                // and the pivot window holds 3 stages of 2 x chunk values
                const int Q = p->theta_q, Lq = p->g.Lt / Q;
                const long long cap = static_cast<long long>((Lq + 4 + 1) & ~1) * 8 - 128;
                const int cb = cap >= 3LL * 2 * 512 * 16 ? 512 : (cap >= 3LL * 2 * 256 * 16 ? 256 : 0);
                if (sl.P == 1 && !peers && cb && !std::getenv("SK_NO_FOLD_TMA")) {
                    sk_status ms = make_col_map(&cmap, tp.buf, p->g.rows, Q, Lq, ncols_local * tp.nrhs);
                    if (ms != SK_OK) return ms;
                    tl.use_cmap = 1;
                    tl.fold_chunk = cb;
                }
            }
            CU(sk::launch_theta_large(tl, cmap, p->theta_q, p->thr_theta, p->smem_theta, p->stream));
        } else if (p->theta_sym) {
            CU(sk::launch_theta_sym(tp, p->thr_theta, p->smem_theta, p->stream));
        } else {
            CUtensorMap cmap{}, ctail{};
            if (fwd_rows) {
                // column k of R[rhs][p][k]: the fast dimension holds the N/2+1 modes, one box = 256 rows p
                // (the tail box rounds M/2 + 1 up to theta_data_slots: every box lands 128-byte aligned)
                tp.gather = 1;
                tp.gather_nbox = p->g.rows / 256;
                tp.gather_tail = sk::theta_data_slots(p->g.Lt) - tp.gather_nbox * 256;
                sk_status ms = SK_OK;
                if (tp.gather_nbox) ms = make_spec_map(&cmap, p->spec_rows, p->g.cols, p->g.rows, tp.nrhs);
                if (ms == SK_OK && tp.gather_tail)
                    ms = make_spec_map(&ctail, p->spec_rows, p->g.cols, p->g.rows, tp.nrhs, 1, 1, 0, 0, tp.gather_tail);
                if (ms != SK_OK) return ms;
            }
            CU(sk::launch_theta(tp, cmap, ctail, p->thr_theta, p->smem_theta, p->stream));
        }
        if (p->timing) {
            CU(cudaEventRecord(p->ev[3], p->stream));
            p->ev_pending |= 2;
        }
        p->last_launches += 1;
    }
    if (stages & 4) {
        lp.in_rhs_stride = static_cast<long long>(rows_local) * p->g.cols;
        lp.out_rhs_stride = static_cast<long long>(rows_local) * p->N;
        lp.f = nullptr;
        lp.spec = spec;
        lp.u = u_dev;
        lp.peers = sk::PeerMap{};
        if (p->timing) CU(cudaEventRecord(p->ev[4], p->stream));
        if (p->lambda_split) {
            sk::LambdaSplitParams sp{lp, p->flh.d, sk::lambda_split_slots(p->fl.d.L / 2, p->lambda_split_tma != 0),
                                     p->lambda_split_tma};
            CUtensorMap m0{}, m1{};
            if (p->lambda_split_tma) {
                const int Lh = p->fl.d.L / 2;
                sk_status ms = make_spec_map(&m0, spec, rows_local, p->g.cols, lp.nrhs, 1, 2, 0, Lh + 1);
                if (ms == SK_OK) ms = make_spec_map(&m1, spec, rows_local, p->g.cols, lp.nrhs, 1, 2, 1, Lh);
                if (ms != SK_OK) return ms;
            }
            CU(sk::launch_lambda_inv_split(sp, m0, m1, p->thr_lambda, p->smem_lambda, p->stream));
        } else if (p->lambda_duo && sk::lambda_duo_ok(lp, p->thr_lambda)) {
            CUtensorMap map;
            sk_status ms = make_spec_map(&map, spec, rows_local, p->g.cols, lp.nrhs, 2);
            if (ms != SK_OK) return ms;
            CU(sk::launch_lambda_inv_duo(lp, map, p->thr_lambda, p->stream));
        } else {
            CUtensorMap map;
            if (p->lambda_pair_inv) lp.pair |= 2;
            const int box_rows = (lp.pair & 2) && sk::lambda_inv_pair_ok(lp, p->thr_lambda) ? 2 : 1;
            sk_status ms = make_spec_map(&map, spec, rows_local, p->g.cols, lp.nrhs, box_rows);
            if (ms != SK_OK) return ms;
            CU(sk::launch_lambda_inv(lp, map, p->thr_lambda, p->smem_lambda, p->stream));
        }
        if (p->timing) {
            CU(cudaEventRecord(p->ev[5], p->stream));
            p->ev_pending |= 4;
        }
        p->last_launches += 1;
    }
    return SK_OK;
}

static void collect_times(sk_plan_t p, int stages) {
    if (!p->timing) return;
    stages &= p->ev_pending;
    p->ev_pending &= ~stages;
    if (!stages) return;
    cudaStreamSynchronize(p->stream);
    float ms = 0;
    if (stages & 1) {
        cudaEventElapsedTime(&ms, p->ev[0], p->ev[1]);
        p->times[0] = ms;
    }
    if (stages & 2) {
        cudaEventElapsedTime(&ms, p->ev[2], p->ev[3]);
        p->times[1] = ms;
    }
    if (stages & 4) {
        cudaEventElapsedTime(&ms, p->ev[4], p->ev[5]);
        p->times[2] = ms;
    }
}

sk_status sk_solve_grid(sk_plan_t p, const double* f, double* u, double* X_half, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    if (!f || !u) return fail(SK_ERR_ARGUMENT, "null f or u");
    const size_t ng = static_cast<size_t>(p->nrhs) * p->g.rows * p->N;
    if ((s = ensure_spec(p)) != SK_OK) return s;
    if (!(flags & SK_DEVICE) && (flags & SK_ASYNC)) {
        if (X_half) return fail(SK_ERR_ARGUMENT, "X_half is not available with asynchronous host-memory solves");
        if ((s = pipe_init(p, ng)) != SK_OK) return s;
        const int slot = p->pipe_slot;
        p->pipe_slot = (slot + 1) % sk_plan_s::kPipe;
        const sk_status prev = pipe_check_slot(p, slot);  // the solve that used this slot kPipe calls ago
        double* buf = p->pipe_buf[slot];
        CU(cudaStreamWaitEvent(p->pipe_h2d, p->pipe_out[slot], 0));  // its result has left the slot
        CU(cudaMemcpyAsync(buf, f, sizeof(double) * ng, cudaMemcpyHostToDevice, p->pipe_h2d));
        CU(cudaEventRecord(p->pipe_in[slot], p->pipe_h2d));
        CU(cudaStreamWaitEvent(p->stream, p->pipe_in[slot], 0));
        CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4 * p->nrhs, p->stream));
        sk::Slabs sl{};
        sl.P = 1;
        sl.row_b[1] = p->g.rows;
        sl.col_b[1] = p->g.cols;
        p->last_launches = 0;
        if ((s = run_grid(p, sl, p->g.rows, p->g.cols, 0, buf, p->spec, buf, nullptr, 7)) != SK_OK) return s;
        CU(cudaMemcpyAsync(p->pipe_stats[slot], p->stats, sizeof(double) * 4 * p->nrhs, cudaMemcpyDeviceToHost,
                           p->stream));
        CU(cudaEventRecord(p->pipe_done[slot], p->stream));
        p->pipe_pending[slot] = true;
        CU(cudaStreamWaitEvent(p->pipe_d2h, p->pipe_done[slot], 0));
        CU(cudaMemcpyAsync(u, buf, sizeof(double) * ng, cudaMemcpyDeviceToHost, p->pipe_d2h));
        CU(cudaEventRecord(p->pipe_out[slot], p->pipe_d2h));
        return prev;
    }
    const double* df;
    double* du;
    if (flags & SK_DEVICE) {
        df = f;
        du = u;
    } else {
        if ((s = ensure(reinterpret_cast<void**>(&p->hf), sizeof(double) * ng)) != SK_OK) return s;
        CU(cudaMemcpyAsync(p->hf, f, sizeof(double) * ng, cudaMemcpyHostToDevice, p->stream));
        df = p->hf;
        du = p->hf;  // in place
    }
    double2* xh = nullptr;
    if (X_half) {
        if (flags & SK_DEVICE) {
            xh = reinterpret_cast<double2*>(X_half);
        } else {
            const size_t nx = static_cast<size_t>(p->nrhs) * p->g.cols * p->M;
            if ((s = ensure(reinterpret_cast<void**>(&p->hX), sizeof(double2) * std::max(nx, static_cast<size_t>(p->nrhs) * p->M * p->N))) != SK_OK)
                return s;
            xh = p->hX;
        }
    }
    CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4 * p->nrhs, p->stream));
    sk::Slabs sl{};
    sl.P = 1;
    sl.rank = 0;
    sl.row_b[0] = 0;
    sl.row_b[1] = p->g.rows;
    sl.col_b[0] = 0;
    sl.col_b[1] = p->g.cols;
    p->last_launches = 0;
    if ((s = run_grid(p, sl, p->g.rows, p->g.cols, 0, df, p->spec, du, xh, 7)) != SK_OK) return s;
    if (!(flags & SK_DEVICE)) {
        CU(cudaMemcpyAsync(u, du, sizeof(double) * ng, cudaMemcpyDeviceToHost, p->stream));
        if (X_half) {
            const size_t nx = static_cast<size_t>(p->nrhs) * p->g.cols * p->M;
            CU(cudaMemcpyAsync(X_half, xh, sizeof(double2) * nx, cudaMemcpyDeviceToHost, p->stream));
        }
    }
    if ((flags & SK_ASYNC) && (flags & SK_DEVICE)) return SK_OK;
    s = check_precondition(p, p->nrhs);
    collect_times(p, 7);
    return s;
}

sk_status sk_last_mean(sk_plan_t p, double out[3]) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    double h[4];
    CU(cudaMemcpyAsync(h, p->stats, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    out[0] = h[0];
    out[1] = h[1];
    out[2] = h[2];
    return SK_OK;
}

sk_status sk_shgen(sk_plan_t p, int L, const double* coeffs_dev, double* phys_dev) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    if (!coeffs_dev || !phys_dev || L < 0) return fail(SK_ERR_ARGUMENT, "bad shgen arguments");
    if (L >= p->N / 2) return fail(SK_ERR_ARGUMENT, "degree L must be below N/2");
    if ((s = ensure_spec(p)) != SK_OK) return s;
    sk::ShgenParams sp{p->g, L, coeffs_dev, p->spec, p->g.rows};
    CU(sk::launch_shgen(sp, p->stream));
    sk::LambdaParams lp{};
    lp.g = p->g;
    lp.fd = p->fl.d;
    lp.swizzle = (p->fl.d.nst > 0 && p->fl.d.span[0] % 2 == 0) ? 1 : 0;  // power-of-two rows
    lp.hiocc = p->lambda_hiocc && !p->lambda_split ? 1 : 0;
    lp.rows_local = p->g.rows;
    lp.nrhs = 1;
    lp.in_rhs_stride = 0;
    lp.out_rhs_stride = 0;
    lp.spec = p->spec;
    lp.u = phys_dev;
    if (p->lambda_split) {
        sk::LambdaSplitParams sp{lp, p->flh.d, sk::lambda_split_slots(p->fl.d.L / 2, p->lambda_split_tma != 0),
                                 p->lambda_split_tma};
        CUtensorMap m0{}, m1{};
        if (p->lambda_split_tma) {
            const int Lh = p->fl.d.L / 2;
            if ((s = make_spec_map(&m0, p->spec, p->g.rows, p->g.cols, 1, 1, 2, 0, Lh + 1)) != SK_OK) return s;
            if ((s = make_spec_map(&m1, p->spec, p->g.rows, p->g.cols, 1, 1, 2, 1, Lh)) != SK_OK) return s;
        }
        CU(sk::launch_lambda_inv_split(sp, m0, m1, p->thr_lambda, p->smem_lambda, p->stream));
    } else {
        CUtensorMap map;
        if ((s = make_spec_map(&map, p->spec, p->g.rows, p->g.cols, 1)) != SK_OK) return s;
        CU(sk::launch_lambda_inv(lp, map, p->thr_lambda, p->smem_lambda, p->stream));
    }
    CU(cudaStreamSynchronize(p->stream));
    return SK_OK;
}

// ------------------------------------------------ assemble / transforms
namespace {

sk_status scratch(sk_plan_t p, int slot, size_t bytes, void** out) {
    if (p->scratch_bytes[slot] < bytes) {
        if (p->scratch[slot]) {
            CU(cudaStreamSynchronize(p->stream));
            CU(cudaFree(p->scratch[slot]));
            p->scratch[slot] = nullptr;
            p->scratch_bytes[slot] = 0;
        }
        CU(cudaMalloc(&p->scratch[slot], bytes < 256 ? 256 : bytes));
        p->scratch_bytes[slot] = bytes < 256 ? 256 : bytes;
    }
    *out = p->scratch[slot];
    return SK_OK;
}

// Input staging: device pointers pass through; host data is copied into
// scratch slot `slot`.
sk_status stage_in(sk_plan_t p, const void* src, size_t bytes, unsigned flags, int slot, const void** out) {
    if (flags & SK_DEVICE) {
        *out = src;
        return SK_OK;
    }
    void* d = nullptr;
    sk_status s = scratch(p, slot, bytes, &d);
    if (s != SK_OK) return s;
    if (bytes) CU(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, p->stream));
    *out = d;
    return SK_OK;
}

int xform_threads(int n) { return round_threads(n / 8, 64, 512); }

// FFT plan of length n for the standalone transforms (cached per plan).
sk_status xform_fft(sk_plan_t p, int n, const DevFft** out) {
    auto it = p->xf.find(n);
    if (it == p->xf.end()) {
        DevFft f;
        // <= 256 threads: high-occupancy kernel variant, register radices <= 8
        const bool hi = xform_threads(n) <= 256 && !std::getenv("SK_NO_HIOCC");
        sk_status s = build_fft(n, xform_threads(n), f, false, false, hi ? 8 : 25);
        if (s != SK_OK) return s;
        if (sk::xform_smem_bytes(n, f.d.nhi, f.d.nlo) > 227 * 1024) {
            free_fft(f);
            return fail(SK_ERR_UNSUPPORTED, "transform length " + std::to_string(n) + " exceeds one CTA's shared memory");
        }
        it = p->xf.emplace(n, f).first;
    }
    *out = &it->second;
    return SK_OK;
}

bool smooth7(long long n) {
    for (int q : {2, 3, 5, 7})
        while (n > 1 && n % q == 0) n /= q;
    return n == 1;
}

// Bluestein plan for a length n with a prime factor > 7: the smallest
// 2,3,5,7-smooth Lb >= 2n - 1 whose in-shared-memory FFT fits one CTA, the
// chirp (long double angles from the exact j^2 mod 2n) and both directions'
// kernel transforms (xform_blue_prep_kernel).
sk_status xform_blue(sk_plan_t p, int n, const sk_plan_s::BlueFft** out) {
    auto it = p->xb.find(n);
    if (it == p->xb.end()) {
        sk_plan_s::BlueFft b;
        int Lb = 2 * n - 1;
        bool ok = false;
        for (; Lb <= 4 * n + 64; ++Lb) {
            if (!smooth7(Lb)) continue;
            if (build_fft(Lb, xform_threads(Lb), b.f, false, false, 25) != SK_OK) continue;
            if (sk::xform_smem_bytes(Lb, b.f.d.nhi, b.f.d.nlo) <= 227 * 1024) {
                ok = true;
                break;
            }
            free_fft(b.f);
            b.f = DevFft{};
        }
        if (!ok)
            return fail(SK_ERR_UNSUPPORTED, "transform length " + std::to_string(n) +
                                                ": its Bluestein convolution exceeds one CTA's shared memory");
        std::vector<double2> ch(n);
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int j = 0; j < n; ++j) {
            const long long e = (static_cast<long long>(j) * j) % (2LL * n);
            const long double ang = pi * static_cast<long double>(e) / static_cast<long double>(n);
            ch[j].x = static_cast<double>(cosl(ang));
            ch[j].y = static_cast<double>(-sinl(ang));
        }
        const size_t lp = static_cast<size_t>((Lb + 7) & ~7);
        CU(cudaMalloc(&b.chirp, sizeof(double2) * n));
        CU(cudaMalloc(&b.bhat_a, sizeof(double2) * lp));
        CU(cudaMalloc(&b.bhat_s, sizeof(double2) * lp));
        CU(cudaMemcpy(b.chirp, ch.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
        const int swz = (b.f.d.nst > 0 && b.f.d.span[0] % 2 == 0) ? 1 : 0;
        const size_t smem = sk::xform_smem_bytes(Lb, b.f.d.nhi, b.f.d.nlo);
        CU(sk::launch_blue_prep(b.f.d, n, b.chirp, true, xform_threads(Lb), smem, swz, b.bhat_a, p->stream));
        CU(sk::launch_blue_prep(b.f.d, n, b.chirp, false, xform_threads(Lb), smem, swz, b.bhat_s, p->stream));
        CU(cudaStreamSynchronize(p->stream));
        it = p->xb.emplace(n, b).first;
    }
    *out = &it->second;
    return SK_OK;
}

// One pass: nrows sequences of the input (row stride ld_in) -> transform of
// length n -> transposed store (output stride ld_out).  Lengths with a prime
// factor > 7 go through Bluestein (xform_blue_kernel).
// gather: the sequences are the nrows COLUMNS of the row-major input (n_in
// rows of ld_in entries), gathered by the copy engine, and each result is
// stored as the contiguous row dst[r * ld_out ..] (xform_gather_ok).
sk_status xform_pass(sk_plan_t p, bool analyze, int nrows, int n, int n_in, long long ld_in, const double2* src,
                     long long ld_out, double2* dst, bool gather = false) {
    CUtensorMap map{};
    if (!smooth7(n)) {
        if (gather) return fail(SK_ERR_UNSUPPORTED, "internal: gathered Bluestein pass");
        const sk_plan_s::BlueFft* b = nullptr;
        sk_status s = xform_blue(p, n, &b);
        if (s != SK_OK) return s;
        const int Lb = b->f.d.L;
        sk::XformParams xp{b->f.d, n_in, ld_in, ld_out, src, dst, (b->f.d.nst > 0 && b->f.d.span[0] % 2 == 0) ? 1 : 0,
                           0, 0, (Lb + 7) & ~7, n, b->chirp, analyze ? b->bhat_a : b->bhat_s};
        CU(sk::launch_xform(xp, map, analyze, nrows, xform_threads(Lb), sk::xform_smem_bytes(Lb, b->f.d.nhi, b->f.d.nlo),
                            p->stream));
        return SK_OK;
    }
    const DevFft* f = nullptr;
    sk_status s = xform_fft(p, n, &f);
    if (s != SK_OK) return s;
    const int n_src = gather ? (analyze ? n : n_in) : 0;
    sk::XformParams xp{f->d, n_in, ld_in, ld_out, src, dst, (f->d.nst > 0 && f->d.span[0] % 2 == 0) ? 1 : 0, 0,
                       gather ? 1 : 0, sk::xform_slots(n, n_src), 0, nullptr, nullptr};
    xp.hiocc = xform_threads(n) <= 256 ? 1 : 0;
    for (int st = 0; st < f->d.nst; ++st)
        if (f->d.R[st] > 8) xp.hiocc = 0;  // the variant only instantiates radices <= 8
    if (gather) {
        s = make_spec_map(&map, const_cast<double2*>(src), static_cast<int>(ld_in), n_src, 1);
        if (s != SK_OK) return s;
    }
    CU(sk::launch_xform(xp, map, analyze, nrows, xform_threads(n), sk::xform_smem_bytes(n, f->d.nhi, f->d.nlo, n_src),
                        p->stream));
    return SK_OK;
}

// Can a pass of output length n over n_in inputs run in gather mode: a plain
// (2, 3, 5, 7)-smooth transform whose thread count re-slots the gathered
// column through kXformStage registers and whose boxes fit shared memory.
bool xform_gather_ok(sk_plan_t p, bool analyze, int n, int n_in) {
    static const bool off = std::getenv("SK_XFORM_GATHER") && std::atoi(std::getenv("SK_XFORM_GATHER")) == 0;
    if (off || !smooth7(n) || n_in <= 0) return false;
    const DevFft* f = nullptr;
    if (xform_fft(p, n, &f) != SK_OK) return false;
    const int n_src = analyze ? n : n_in;
    bool hi = xform_threads(n) <= 256;
    for (int st = 0; st < f->d.nst; ++st)
        if (f->d.R[st] > 8) hi = false;
    const bool swz = f->d.nst > 0 && f->d.span[0] % 2 == 0;
    const bool staged = !analyze || swz;  // (unswizzled analysis transforms the gathered column where it lands)
    const int stage = hi ? sk::kXformStageHi : sk::kXformStage;
    return (!staged || std::max(n, n_src) <= stage * xform_threads(n)) &&
           sk::xform_smem_bytes(n, f->d.nhi, f->d.nlo, n_src) <= 227 * 1024;
}

// The separable 2-D transform of a rows x cols row-major input into an
// m_out x n_out row-major output through the cols x m_out intermediate T
// (gather passes: theta direction first, every store contiguous), or through
// the n_out x rows intermediate of the transposed-store passes.
sk_status xform_2d(sk_plan_t p, bool analyze, int rows, int cols, int m_out, int n_out, const double2* src, double2* T,
                   double2* dst) {
    sk_status s;
    if (xform_gather_ok(p, analyze, m_out, rows) && xform_gather_ok(p, analyze, n_out, cols)) {
        if ((s = xform_pass(p, analyze, cols, m_out, rows, cols, src, m_out, T, true)) != SK_OK) return s;   // theta
        return xform_pass(p, analyze, m_out, n_out, cols, m_out, T, n_out, dst, true);                     // lambda
    }
    if ((s = xform_pass(p, analyze, rows, n_out, cols, cols, src, rows, T)) != SK_OK) return s;  // lambda, transposed
    return xform_pass(p, analyze, n_out, m_out, rows, rows, T, n_out, dst);                     // theta, transposed
}

}  // namespace

sk_status sk_assemble(sk_plan_t p, int K, int mf, int nf, const double* d, const double* col, const double* row,
                      double vscale, double* F, double report[3], unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (K < 0 || mf < 0 || nf < 0 || mf % 2 || nf % 2) return fail(SK_ERR_SIZE, "CoeffVec: length must be even");
    if (!F || (K > 0 && (!d || (mf > 0 && !col) || (nf > 0 && !row)))) return fail(SK_ERR_ARGUMENT, "null argument");
    if (p->M < 4) return fail(SK_ERR_UNSUPPORTED, "assemble_poisson needs m >= 4");
    const int M = p->M, N = p->N;
    const double2 *dd = nullptr, *dc = nullptr, *dr = nullptr;
    if ((s = stage_in(p, d, sizeof(double2) * K, flags, 0, reinterpret_cast<const void**>(&dd))) != SK_OK) return s;
    if ((s = stage_in(p, col, sizeof(double2) * K * static_cast<size_t>(mf), flags, 1,
                      reinterpret_cast<const void**>(&dc))) != SK_OK)
        return s;
    if ((s = stage_in(p, row, sizeof(double2) * K * static_cast<size_t>(nf), flags, 2,
                      reinterpret_cast<const void**>(&dr))) != SK_OK)
        return s;
    // scratch slot 3: [report(4 doubles)] [SA: K x M] [sum2 terms: K] [B: K x N] [F staging: M x N if host]
    const size_t nsa = static_cast<size_t>(K) * M, nb = static_cast<size_t>(K) * N, nfm = static_cast<size_t>(M) * N;
    void* w = nullptr;
    if ((s = scratch(p, 3, 32 + sizeof(double2) * (nsa + K + nb + ((flags & SK_DEVICE) ? 0 : nfm)), &w)) != SK_OK)
        return s;
    double* rep = static_cast<double*>(w);
    double2* sa = reinterpret_cast<double2*>(static_cast<char*>(w) + 32);
    double2* bp = sa + nsa + K;
    double2* dF = (flags & SK_DEVICE) ? reinterpret_cast<double2*>(F) : bp + nb;
    sk::AssembleParams ap{M, N, K, mf, nf, dd, dc, dr, vscale, sa, bp, dF, rep};
    CU(sk::launch_assemble(ap, p->stream));
    p->last_launches = K > 0 ? 4 : 2;
    double h[3];
    CU(cudaMemcpyAsync(h, rep, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(F, dF, sizeof(double2) * nfm, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    if (report) {
        report[0] = h[0];
        report[1] = h[1];
        report[2] = h[2];
    }
    return SK_OK;
}

// ---- structure-preserving GE on a doubled grid (ge_kernels.cu)
namespace {

using cplx = std::complex<double>;

// lowrank.cpp:60-72 (host: std::complex division as the reference's compiler emits it)
bool pinv_2x2_host(cplx a, cplx b, double alpha, cplx& me, cplx& mo) {
    const cplx s = a + b, d = a - b;
    const double sp = std::abs(s), dp = std::abs(d);
    me = mo = cplx{};
    if (sp == 0.0 && dp == 0.0) return false;
    if (dp == 0.0) { me = 1.0 / s; return true; }
    if (sp == 0.0) { mo = 1.0 / d; return true; }
    if (dp < alpha * sp) { me = 1.0 / s; return true; }
    if (sp < alpha * dp) { mo = 1.0 / d; return true; }
    me = 1.0 / s;
    mo = 1.0 / d;
    return true;
}

constexpr double kPiRef = 3.141592653589793238462643383279502884;  // types.hpp:12-13
constexpr double kTwoPiRef = 2.0 * kPiRef;

sk_status ge_check_sizes(int m, int n) {
    if (m <= 0 || n <= 0 || (m & 1) || (n & 1)) return fail(SK_ERR_SIZE, "BMCGrid: sample counts must be positive and even");
    return SK_OK;
}

// search on the device grid g; fills out_i / out_d (host); returns found
sk_status ge_search_dev(sk_plan_t p, int m, int n, bool half, const double2* g, void* scr, double alpha, int out_i[3],
                        double out_d[10]) {
    CU(sk::launch_ge_search(m, n, half, g, scr, p->stream));
    double h[6];
    CU(cudaMemcpyAsync(h, scr, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    for (int i = 0; i < 10; ++i) out_d[i] = 0.0;
    out_i[0] = 0;
    out_i[1] = out_i[2] = -1;
    if (h[1] < 0.0 || !(h[0] > 0.0)) return SK_OK;  // best == 0: no pivot (lowrank.cpp:103)
    const long long c = static_cast<long long>(h[1]);
    const int t = static_cast<int>(c / (n / 2)), k = static_cast<int>(c % (n / 2)) + n / 2;
    const cplx a(h[2], h[3]), b(h[4], h[5]);
    cplx me, mo;
    if (!pinv_2x2_host(a, b, alpha, me, mo)) return fail(SK_ERR_SINGULAR, "pinv_2x2: zero pivot matrix");
    out_i[0] = 1;
    out_i[1] = t;
    out_i[2] = k;
    const cplx v[4] = {a, b, me, mo};
    for (int i = 0; i < 4; ++i) {
        out_d[2 * i] = v[i].real();
        out_d[2 * i + 1] = v[i].imag();
    }
    out_d[8] = kTwoPiRef * t / m;             // lowrank.cpp:106
    out_d[9] = -kPiRef + kTwoPiRef * k / n;   // BMCGrid::lambda, sphere_domain.hpp:55
    return SK_OK;
}

// locate_on_grid (lowrank.cpp:116-123)
sk_status ge_locate(double x, double step, int count, int* idx) {
    const double t = (x + kPiRef) / step;
    const long i = std::lround(t);
    if (std::abs(t - static_cast<double>(i)) > 1e-9) return fail(SK_ERR_ARGUMENT, "ge_step: pivot coordinate is not a grid node");
    *idx = static_cast<int>(((i % count) + count) % count);
    return SK_OK;
}

sk_status ge_step_dev(sk_plan_t p, int m, int n, bool half, const double2* g, const double piv[10], double2* out,
                      void* scr, bool want_max) {
    int js = 0, ks = 0;
    sk_status s = ge_locate(piv[8], kTwoPiRef / m, m, &js);
    if (s != SK_OK) return s;
    if ((s = ge_locate(piv[9], kTwoPiRef / n, n, &ks)) != SK_OK) return s;
    if (half) {  // stored row i <-> theta_i = 2 pi i / m: the doubled row m/2 + i (theta* = pi is doubled row 0)
        js = (js + m - m / 2) % m;
        if (js > m / 2) return fail(SK_ERR_ARGUMENT, "ge_step: theta* lies outside [0, pi]");
    }
    const cplx me(piv[4], piv[5]), mo(piv[6], piv[7]);
    const cplx de = 0.5 * me, dodd = 0.5 * mo;  // lowrank.cpp:147-148
    CU(sk::launch_ge_step(m, n, half, g, js, ks, make_double2(de.real(), de.imag()), make_double2(dodd.real(), dodd.imag()),
                          me != cplx{} ? 1 : 0, mo != cplx{} ? 1 : 0, out, scr, want_max, p->stream));
    return SK_OK;
}

}  // namespace

sk_status sk_ge_pivot_search(sk_plan_t p, int m, int n, const double* grid, double alpha, int out_i[3], double out_d[10],
                             unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!grid || !out_i || !out_d) return fail(SK_ERR_ARGUMENT, "null argument");
    if ((s = ge_check_sizes(m, n)) != SK_OK) return s;
    const bool half = (flags & SK_GE_HALF) != 0;
    const void* g = nullptr;
    void* scr = nullptr;
    if ((s = stage_in(p, grid, sizeof(double2) * (half ? m / 2 + 1 : m) * static_cast<size_t>(n), flags, 0, &g)) != SK_OK)
        return s;
    if ((s = scratch(p, 2, sk::ge_scratch_bytes(m, n), &scr)) != SK_OK) return s;
    p->last_launches = 2;
    return ge_search_dev(p, m, n, half, static_cast<const double2*>(g), scr, alpha, out_i, out_d);
}

sk_status sk_ge_step(sk_plan_t p, int m, int n, const double* grid, const double piv[10], double* out, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!grid || !piv || !out) return fail(SK_ERR_ARGUMENT, "null argument");
    if ((s = ge_check_sizes(m, n)) != SK_OK) return s;
    const bool half = (flags & SK_GE_HALF) != 0;
    const size_t bytes = sizeof(double2) * (half ? m / 2 + 1 : m) * static_cast<size_t>(n);
    const void* g = nullptr;
    void *scr = nullptr, *o = out;
    if ((s = stage_in(p, grid, bytes, flags, 0, &g)) != SK_OK) return s;
    if ((s = scratch(p, 2, sk::ge_scratch_bytes(m, n), &scr)) != SK_OK) return s;
    if (!(flags & SK_DEVICE) && (s = scratch(p, 1, bytes, &o)) != SK_OK) return s;
    if ((s = ge_step_dev(p, m, n, half, static_cast<const double2*>(g), piv, static_cast<double2*>(o), scr, false)) != SK_OK)
        return s;
    p->last_launches = 2;
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(out, o, bytes, cudaMemcpyDeviceToHost, p->stream));
    if (!((flags & SK_ASYNC) && (flags & SK_DEVICE))) CU(cudaStreamSynchronize(p->stream));
    return SK_OK;
}

sk_status sk_ge_run(sk_plan_t p, int m, int n, double* grid, double alpha, double tau, int max_steps, int* nsteps,
                    int* piv_i, double* piv_d, double* resid, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!grid || !nsteps || !piv_i || !piv_d || !resid || max_steps < 0) return fail(SK_ERR_ARGUMENT, "bad argument");
    if ((s = ge_check_sizes(m, n)) != SK_OK) return s;
    const bool half = (flags & SK_GE_HALF) != 0;
    const long long rows = half ? m / 2 + 1 : m;
    const size_t bytes = sizeof(double2) * rows * static_cast<size_t>(n);
    void *g = grid, *scr = nullptr;
    if (!(flags & SK_DEVICE)) {
        if ((s = scratch(p, 0, bytes, &g)) != SK_OK) return s;
        CU(cudaMemcpyAsync(g, grid, bytes, cudaMemcpyHostToDevice, p->stream));
    }
    if ((s = scratch(p, 2, sk::ge_scratch_bytes(m, n), &scr)) != SK_OK) return s;
    double2* gd = static_cast<double2*>(g);
    double* mx = static_cast<double*>(scr) + 8;
    auto read_max = [&](double* v) -> sk_status {
        CU(cudaMemcpyAsync(v, mx, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
        CU(cudaStreamSynchronize(p->stream));
        return SK_OK;
    };
    CU(sk::launch_ge_maxabs(rows * n, gd, scr, p->stream));
    if ((s = read_max(&resid[0])) != SK_OK) return s;
    int step = 0;
    p->last_launches = 1;
    while (step < max_steps && resid[step] > tau) {
        int oi[3];
        if ((s = ge_search_dev(p, m, n, half, gd, scr, alpha, oi, piv_d + 10 * step)) != SK_OK) return s;
        if (!oi[0]) break;  // the residual is exactly zero on the pivot set
        piv_i[2 * step] = oi[1];
        piv_i[2 * step + 1] = oi[2];
        if ((s = ge_step_dev(p, m, n, half, gd, piv_d + 10 * step, gd, scr, true)) != SK_OK) return s;
        if ((s = read_max(&resid[step + 1])) != SK_OK) return s;
        p->last_launches += 4;
        ++step;
    }
    *nsteps = step;
    if (!(flags & SK_DEVICE)) {
        CU(cudaMemcpyAsync(grid, g, bytes, cudaMemcpyDeviceToHost, p->stream));
        CU(cudaStreamSynchronize(p->stream));
    }
    return SK_OK;
}

sk_status sk_analyze_2d(sk_plan_t p, int m, int n, const double* grid, double* X, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (m <= 0 || n <= 0 || m % 2 || n % 2) return fail(SK_ERR_SIZE, "analyze_1d: sample count must be even");
    if (!grid || !X) return fail(SK_ERR_ARGUMENT, "null argument");
    const size_t mn = static_cast<size_t>(m) * n;
    const double2* g = nullptr;
    if ((s = stage_in(p, grid, sizeof(double2) * mn, flags, 0, reinterpret_cast<const void**>(&g))) != SK_OK) return s;
    void* t = nullptr;
    if ((s = scratch(p, 1, sizeof(double2) * mn * ((flags & SK_DEVICE) ? 1 : 2), &t)) != SK_OK) return s;
    double2* T = static_cast<double2*>(t);  // lambda-analysed rows, transposed: n x m
    double2* out = (flags & SK_DEVICE) ? reinterpret_cast<double2*>(X) : T + mn;
    if ((s = xform_2d(p, true, m, n, m, n, g, T, out)) != SK_OK) return s;
    p->last_launches = 2;
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(X, out, sizeof(double2) * mn, cudaMemcpyDeviceToHost, p->stream));
    if (!(flags & SK_ASYNC) || !(flags & SK_DEVICE)) CU(cudaStreamSynchronize(p->stream));
    return SK_OK;
}

sk_status sk_sample_grid(sk_plan_t p, int rows, int cols, const double* X, int m_out, int n_out, double* grid,
                         unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (m_out <= 0 || n_out <= 0 || m_out % 2 || n_out % 2)
        return fail(SK_ERR_SIZE, "sample_grid: output sizes must be even");
    if (rows < 0 || cols < 0 || rows % 2 || cols % 2) return fail(SK_ERR_SIZE, "CoeffVec: length must be even");
    if (!grid || (rows * cols > 0 && !X)) return fail(SK_ERR_ARGUMENT, "null argument");
    const size_t nx = static_cast<size_t>(rows) * cols, ng = static_cast<size_t>(m_out) * n_out;
    const double2* x = nullptr;
    if ((s = stage_in(p, X, sizeof(double2) * nx, flags, 0, reinterpret_cast<const void**>(&x))) != SK_OK) return s;
    const size_t nt = std::max(static_cast<size_t>(rows) * n_out, static_cast<size_t>(cols) * m_out);
    void* t = nullptr;
    if ((s = scratch(p, 1, sizeof(double2) * (nt + ((flags & SK_DEVICE) ? 0 : ng)), &t)) != SK_OK) return s;
    double2* T = static_cast<double2*>(t);  // lambda-synthesised rows, transposed: n_out x rows
    double2* out = (flags & SK_DEVICE) ? reinterpret_cast<double2*>(grid) : T + nt;
    if (rows == 0) {
        CU(cudaMemsetAsync(out, 0, sizeof(double2) * ng, p->stream));
    } else {
        if ((s = xform_2d(p, false, rows, cols, m_out, n_out, x, T, out)) != SK_OK) return s;
    }
    p->last_launches = 2;
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(grid, out, sizeof(double2) * ng, cudaMemcpyDeviceToHost, p->stream));
    if (!(flags & SK_ASYNC) || !(flags & SK_DEVICE)) CU(cudaStreamSynchronize(p->stream));
    return SK_OK;
}

sk_status sk_sample_dfs(sk_plan_t p, int m, int n, const double* phys, double* grid, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (m <= 0 || n <= 0 || m % 2 || n % 2) return fail(SK_ERR_SIZE, "BMCGrid: sample counts must be positive and even");
    if (!phys || !grid) return fail(SK_ERR_ARGUMENT, "null argument");
    const size_t np = static_cast<size_t>(m / 2 + 1) * n, ng = static_cast<size_t>(m) * n;
    const double* ph = nullptr;
    if ((s = stage_in(p, phys, sizeof(double) * np, flags, 0, reinterpret_cast<const void**>(&ph))) != SK_OK) return s;
    double2* out = reinterpret_cast<double2*>(grid);
    if (!(flags & SK_DEVICE)) {
        void* t = nullptr;
        if ((s = scratch(p, 1, sizeof(double2) * ng, &t)) != SK_OK) return s;
        out = static_cast<double2*>(t);
    }
    CU(sk::launch_dfs_double(m, n, ph, out, p->stream));
    p->last_launches = 1;
    if (!(flags & SK_DEVICE)) CU(cudaMemcpyAsync(grid, out, sizeof(double2) * ng, cudaMemcpyDeviceToHost, p->stream));
    if (!(flags & SK_ASYNC) || !(flags & SK_DEVICE)) CU(cudaStreamSynchronize(p->stream));
    return SK_OK;
}


// Reference-semantics grid solve: the composition the reference runs (and
// its tests use) — sample_dfs (sphere_domain.cpp:46-52) ->
// analyze_2d (fourier.cpp:170-188) -> Msin^2 per column (poisson.cpp:61) ->
// solve (poisson.cpp:121-161) -> sample_grid (fourier.cpp:190-209) — with
// every stage on the device: K12 dfs_double, two K11 analyze passes, msin2,
// K5 coeff_solve (bit-exact Thomas, mean precondition), two K11 synthesis
// passes.  All N lambda modes are solved, k < 0 included, so the result is
// the reference's complex doubled grid even where the reference's truncated
// operators make it differ from the Hermitian (real-output) grid path.
sk_status sk_solve_grid_exact(sk_plan_t p, const double* f, double* U, double* X, unsigned flags) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!f || !U) return fail(SK_ERR_ARGUMENT, "null f or U");
    const int M = p->M, N = p->N;
    const size_t np = static_cast<size_t>(M / 2 + 1) * N, mn = static_cast<size_t>(M) * N;
    const bool dev = (flags & SK_DEVICE) != 0;
    void *g = nullptr, *t = nullptr, *h = nullptr, *in = nullptr;
    if ((s = scratch(p, 4, sizeof(double2) * mn, &g)) != SK_OK) return s;
    if ((s = scratch(p, 5, sizeof(double2) * mn, &t)) != SK_OK) return s;
    if ((s = scratch(p, 6, sizeof(double2) * mn, &h)) != SK_OK) return s;
    if (!dev && (s = scratch(p, 7, sizeof(double) * np, &in)) != SK_OK) return s;
    if ((s = ensure_coeff_tables(p)) != SK_OK) return s;
    double2* G = static_cast<double2*>(g);  // doubled grid, then 2D coefficients, then X
    double2* T = static_cast<double2*>(t);  // transposed intermediates, then F
    double2* H = static_cast<double2*>(h);  // u (host calls), X staging
    CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4 * p->nrhs, p->stream));
    p->last_launches = 0;
    for (int r = 0; r < p->nrhs; ++r) {
        const double* fr = f + r * np;
        const double* df = fr;
        if (!dev) {
            CU(cudaMemcpyAsync(in, fr, sizeof(double) * np, cudaMemcpyHostToDevice, p->stream));
            df = static_cast<const double*>(in);
        }
        CU(sk::launch_dfs_double(M, N, df, G, p->stream));                            // sample_dfs
        if ((s = xform_2d(p, true, M, N, M, N, G, T, G)) != SK_OK) return s;            // analyze_2d
        CU(sk::launch_msin2(M, N, G, T, p->stream));                                    // F = Msin^2 A
        double2* dX = (dev && X) ? reinterpret_cast<double2*>(X) + r * mn : G;
        sk::CoeffParams cp{M, N, 1, T, dX, p->D, p->D + mn, p->D + 2 * mn, p->stats + 4 * r, p->z};
        CU(sk::launch_coeff_solve(cp, p->stream));                                      // solve
        if (!dev && X) CU(cudaMemcpyAsync(X + 2 * r * mn, dX, sizeof(double2) * mn, cudaMemcpyDeviceToHost, p->stream));
        double2* dU = dev ? reinterpret_cast<double2*>(U) + r * mn : H;
        if ((s = xform_2d(p, false, M, N, M, N, dX, T, dU)) != SK_OK) return s;         // sample_grid
        if (!dev) CU(cudaMemcpyAsync(U + 2 * r * mn, dU, sizeof(double2) * mn, cudaMemcpyDeviceToHost, p->stream));
        p->last_launches += 9;
    }
    if ((flags & SK_ASYNC) && dev) return SK_OK;
    return check_precondition(p, p->nrhs);
}

// Queue the copy of the theta stage's statistics to pinned host memory and
// mark it with an event, so that a rank can check the precondition without
// draining its stream (sk_stage_stats).
static sk_status stage_stats_async(sk_plan_t p) {
    if (!p->stage_stats_h) {
        CU(cudaMallocHost(&p->stage_stats_h, sizeof(double) * 4));
        CU(cudaEventCreateWithFlags(&p->ev_stats, cudaEventDisableTiming));
    }
    CU(cudaMemcpyAsync(p->stage_stats_h, p->stats, sizeof(double) * 4, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaEventRecord(p->ev_stats, p->stream));
    return SK_OK;
}

static sk_status make_slabs(sk_plan_t p, int P, const int* rb, const int* cb, int rank, sk::Slabs& sl) {
    if (P < 1 || P > sk::kMaxRanks || rank < 0 || rank >= P || !rb || !cb)
        return fail(SK_ERR_ARGUMENT, "bad slab description");
    if (rb[0] != 0 || rb[P] != p->g.rows || cb[0] != 0 || cb[P] != p->g.cols)
        return fail(SK_ERR_ARGUMENT, "slabs must cover rows [0, M/2] and modes [0, N/2]");
    sl.P = P;
    sl.rank = rank;
    for (int i = 0; i <= P; ++i) {
        sl.row_b[i] = rb[i];
        sl.col_b[i] = cb[i];
        if (i > 0 && (rb[i] < rb[i - 1] || cb[i] < cb[i - 1])) return fail(SK_ERR_ARGUMENT, "slabs must be ordered");
    }
    return SK_OK;
}

sk_status sk_stage_lambda_fwd(sk_plan_t p, int P, const int* rb, const int* cb, int rank, const double* f_rows_dev,
                              double* send_dev) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    sk::Slabs sl{};
    if ((s = make_slabs(p, P, rb, cb, rank, sl)) != SK_OK) return s;
    const int rows = rb[rank + 1] - rb[rank];
    if (rows == 0) return SK_OK;
    p->last_launches = 0;
    return run_grid(p, sl, rows, cb[rank + 1] - cb[rank], cb[rank], f_rows_dev,
                    reinterpret_cast<double2*>(send_dev), nullptr, nullptr, 1);
}

sk_status sk_stage_theta(sk_plan_t p, int P, const int* rb, const int* cb, int rank, double* recv_dev) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    sk::Slabs sl{};
    if ((s = make_slabs(p, P, rb, cb, rank, sl)) != SK_OK) return s;
    const int ncols = cb[rank + 1] - cb[rank];
    CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4, p->stream));
    if (ncols == 0) return SK_OK;
    p->last_launches = 0;
    if ((s = run_grid(p, sl, 0, ncols, cb[rank], nullptr, reinterpret_cast<double2*>(recv_dev), nullptr, nullptr, 2)) !=
        SK_OK)
        return s;
    return stage_stats_async(p);
}

sk_status sk_stage_lambda_inv(sk_plan_t p, int P, const int* rb, const int* cb, int rank, const double* back_dev,
                              double* u_rows_dev) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    sk::Slabs sl{};
    if ((s = make_slabs(p, P, rb, cb, rank, sl)) != SK_OK) return s;
    const int rows = rb[rank + 1] - rb[rank];
    if (rows == 0) return SK_OK;
    p->last_launches = 0;
    return run_grid(p, sl, rows, cb[rank + 1] - cb[rank], cb[rank], nullptr,
                    const_cast<double2*>(reinterpret_cast<const double2*>(back_dev)), u_rows_dev, nullptr, 4);
}

sk_status sk_stage_lambda_fwd_peer(sk_plan_t p, int P, const int* rb, const int* cb, int rank,
                                   const double* f_rows_dev, void* const* peer_recv) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    sk::Slabs sl{};
    if ((s = make_slabs(p, P, rb, cb, rank, sl)) != SK_OK) return s;
    if (!peer_recv) return fail(SK_ERR_ARGUMENT, "null peer buffer table");
    const int rows = rb[rank + 1] - rb[rank];
    if (rows == 0) return SK_OK;
    sk::PeerMap pm{};
    pm.n = P;
    for (int d = 0; d < P; ++d) {
        if (!peer_recv[d] && cb[d + 1] > cb[d]) return fail(SK_ERR_ARGUMENT, "null peer receive buffer");
        pm.base[d] = static_cast<double2*>(peer_recv[d]);
        pm.mul[d] = rows;
        pm.off[d] = static_cast<long long>(cb[d + 1] - cb[d]) * rb[rank] - static_cast<long long>(cb[d]) * rows;
        pm.bound[d] = cb[d];
    }
    pm.bound[P] = cb[P];
    p->last_launches = 0;
    return run_grid(p, sl, rows, cb[rank + 1] - cb[rank], cb[rank], f_rows_dev, nullptr, nullptr, nullptr, 1, &pm);
}

sk_status sk_stage_theta_peer(sk_plan_t p, int P, const int* rb, const int* cb, int rank, double* recv_dev,
                              void* const* peer_back) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!p->grid_ok) return fail(SK_ERR_UNSUPPORTED, p->grid_why);
    sk::Slabs sl{};
    if ((s = make_slabs(p, P, rb, cb, rank, sl)) != SK_OK) return s;
    if (!peer_back) return fail(SK_ERR_ARGUMENT, "null peer buffer table");
    const int ncols = cb[rank + 1] - cb[rank];
    CU(cudaMemsetAsync(p->stats, 0, sizeof(double) * 4, p->stream));
    if (ncols == 0) return stage_stats_async(p);
    sk::PeerMap pm{};
    pm.n = P;
    for (int r = 0; r < P; ++r) {
        if (!peer_back[r] && rb[r + 1] > rb[r]) return fail(SK_ERR_ARGUMENT, "null peer return buffer");
        pm.base[r] = static_cast<double2*>(peer_back[r]);
        pm.mul[r] = rb[r + 1] - rb[r];
        pm.off[r] = -static_cast<long long>(rb[r]);
        pm.bound[r] = rb[r];
    }
    pm.bound[P] = rb[P];
    p->last_launches = 0;
    if ((s = run_grid(p, sl, 0, ncols, cb[rank], nullptr, reinterpret_cast<double2*>(recv_dev), nullptr, nullptr, 2,
                      &pm)) != SK_OK)
        return s;
    return stage_stats_async(p);
}

sk_status sk_device_alloc(int device, size_t bytes, void** ptr) {
    if (!ptr) return fail(SK_ERR_ARGUMENT, "null output pointer");
    *ptr = nullptr;
    CU(cudaSetDevice(device));
    CU(cudaMalloc(ptr, bytes ? bytes : 16));
    return SK_OK;
}

sk_status sk_device_free(void* ptr) {
    if (ptr) CU(cudaFree(ptr));
    return SK_OK;
}

sk_status sk_ipc_handle(const void* ptr, unsigned char handle[64]) {
    if (!ptr || !handle) return fail(SK_ERR_ARGUMENT, "null pointer");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handle size");
    std::memcpy(handle, &h, 64);
    return SK_OK;
}

sk_status sk_ipc_open(int device, const unsigned char handle[64], void** ptr) {
    if (!ptr || !handle) return fail(SK_ERR_ARGUMENT, "null pointer");
    *ptr = nullptr;
    CU(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    CU(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return SK_OK;
}

sk_status sk_ipc_close(void* ptr) {
    if (ptr) CU(cudaIpcCloseMemHandle(ptr));
    return SK_OK;
}

sk_status sk_stage_stats(sk_plan_t p, double out[3]) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    if (!out) return fail(SK_ERR_ARGUMENT, "null output");
    if (!p->stage_stats_h) return fail(SK_ERR_ARGUMENT, "no theta stage has run on this plan");
    CU(cudaEventSynchronize(p->ev_stats));
    for (int i = 0; i < 3; ++i) out[i] = p->stage_stats_h[i];
    return SK_OK;
}

sk_status sk_ipc_event_create(int device, unsigned char handle[64], void** event) {
    if (!handle || !event) return fail(SK_ERR_ARGUMENT, "null argument");
    CU(cudaSetDevice(device));
    cudaEvent_t e = nullptr;
    CU(cudaEventCreateWithFlags(&e, cudaEventInterprocess | cudaEventDisableTiming));
    cudaIpcEventHandle_t h;
    CU(cudaIpcGetEventHandle(&h, e));
    std::memcpy(handle, &h, sizeof(h) < 64 ? sizeof(h) : 64);
    *event = e;
    return SK_OK;
}

sk_status sk_ipc_event_open(int device, const unsigned char handle[64], void** event) {
    if (!handle || !event) return fail(SK_ERR_ARGUMENT, "null argument");
    CU(cudaSetDevice(device));
    cudaIpcEventHandle_t h;
    std::memcpy(&h, handle, sizeof(h) < 64 ? sizeof(h) : 64);
    cudaEvent_t e = nullptr;
    CU(cudaIpcOpenEventHandle(&e, h));
    *event = e;
    return SK_OK;
}

sk_status sk_event_destroy(void* event) {
    if (event) CU(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return SK_OK;
}

sk_status sk_event_record(sk_plan_t p, void* event) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    CU(cudaEventRecord(static_cast<cudaEvent_t>(event), p->stream));
    return SK_OK;
}

sk_status sk_stream_wait_event(sk_plan_t p, void* event) {
    sk_status s = check_plan(p);
    if (s != SK_OK) return s;
    CU(cudaStreamWaitEvent(p->stream, static_cast<cudaEvent_t>(event), 0));
    return SK_OK;
}

}  // extern "C"
