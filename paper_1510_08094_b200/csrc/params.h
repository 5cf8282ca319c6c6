// Kernel parameter blocks and launchers shared by the host plan code
// (sk_poisson.cu) and the kernels (grid_kernels.cu, coeff_kernels.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>

#include "sk_internal.h"

namespace sk {

struct LambdaParams {
    GridGeom g;
    FftDesc fd;
    int rows_local;     // physical rows on this rank
    int nrhs;
    long long in_rhs_stride;   // doubles (fwd) or complex (inv) per rhs in the input
    long long out_rhs_stride;  // complex (fwd) or doubles (inv) per rhs in the output
    const double* f;    // fwd: real rows; inv: unused
    double2* spec;      // fwd: output [k][p_local]; inv: input
    double* u;          // inv: real rows
    PeerMap peers;      // fwd: mode k of this rank's rows goes straight to its theta rank's receive buffer
    int swizzle;        // XOR-swizzled shared-memory slots (plans whose first FFT span is even)
    int hiocc;          // high-occupancy kernel variant (short rows: 64 registers, radices <= 8)
    int pair;           // bit 0 fwd, bit 1 inv: row pairs on CTA pairs, 32-byte (p, p+1) segments (lambda_pair_ok decides);
                        // bit 2 fwd: row quads on 4-CTA clusters, 64-byte (p .. p+3) segments (lambda_quad_ok)
                        // bit 3 fwd: spec is the row-major spectrum R[rhs][p][k], contiguous row stores (K1)
};

struct ThetaParams {
    GridGeom g;
    FftDesc fd;       // length M/2, twiddles of the M-th roots
    Slabs sl;
    double2* buf;     // receive buffer, solved in place
    int ncols;        // lambda modes on this rank
    int k0;           // first lambda mode of this rank
    int nrhs;
    long long rhs_stride;  // complex per rhs in buf
    double* stats;    // per rhs: [0..1] mean (re, im), [2] max|F|, [3] unused
    double2* xhalf;   // optional: solution coefficients X[k][i], (N/2+1) x M per rhs
    int kseq;         // lambda modes k < kseq use the sequential Thomas recurrence
    const double* pivots;  // pivot table for modes k0..k0+ncols-1 (pivot_table_kernel)
    int regsolve;          // chain solver: 0 shared-memory walk, 1 fixed short segments, 2 SMAX=12 register walk
    int swizzle;           // XOR-swizzled data slots (plans whose first FFT span is even)
    int piv_stride;        // doubles per (mode, parity) pivot row
    int pair_chains;       // theta_kernel segment solver: both chains of a parity from one solve (solve_chains_pair_fast)
    int gather;            // theta_kernel: the raw column is gathered from the row-major spectrum R[rhs][p][k]
    int gather_nbox;       // ... as gather_nbox tensor-map boxes of 256 rows
    int gather_tail;       // ... and one tail box of gather_tail rows (a multiple of 8; together theta_data_slots)
    PeerMap peers;         // row p of the solved columns goes straight to its lambda rank's return buffer
    int rev_win;           // stage each chain's digit-reversal entries in shared memory (bulk copy)
    int hiocc;             // high-occupancy kernel variant (short columns: 64 registers, radices <= 8)
    const uint32_t* sym_pos;  // theta_sym_kernel: per parity, chain element i -> slots of tau+ (lo 16) and tau- (hi 16)
};

struct AssembleParams {
    int M, N;              // output F: M x N complex
    int K, mf, nf;         // rank, theta / lambda coefficient counts of the factors
    const double2* d;      // K
    const double2* col;    // K x mf
    const double2* row;    // K x nf
    double vscale;
    double2* sa;           // scratch K x M: d_j Msin^2 pad(a_j), then K sum2 terms
    double2* bp;           // scratch K x N: pad(b_j)
    double2* F;            // M x N
    double* report;        // device [3]: removed?, mu re, mu im
};

struct XformParams {
    FftDesc fd;            // transform length n (analyze) or n_out (synthesize)
    int n_in;              // synthesize: coefficients per input row
    long long ld_in;       // complex per input row
    long long ld_out;      // complex between consecutive outputs of one row (transposed store)
    const double2* src;
    double2* dst;
    int swizzle;           // XOR-swizzled shared-memory slots (first FFT span even)
    int hiocc;             // high-occupancy variant (<= 256 threads: 64 registers, radices <= 8)
    int gather;            // sequences are the COLUMNS of src (TMA gather), outputs contiguous rows of ld_out
    int aslots;            // data slots ahead of the tables (xform_slots)
    // Bluestein (chirp-z) for lengths with a prime factor > 7 (xform_blue_kernel):
    // nb = the DFT length (0: plain transform of length fd.L); fd is then the
    // convolution FFT of length Lb >= 2 nb - 1, chirp[j] = exp(-i pi j^2 / nb),
    // bhat = FFT_Lb of the direction's chirp kernel / Lb in the engine's
    // digit-reversed physical slot order
    int nb;
    const double2* chirp;
    const double2* bhat;
};
cudaError_t launch_blue_prep(const FftDesc& fd, int nb, const double2* chirp, bool analyze, int nthr, size_t smem,
                             int swizzle, double2* bhat, cudaStream_t st);

struct ShgenParams {
    GridGeom g;
    int L;                 // max degree
    const double* coeffs;  // (L+1)^2, index l*l + l + m
    double2* spec;         // [m][p] (rows = M/2+1), modes m = 0..N/2
    int rows;
};

struct CoeffParams {
    int M, N, nrhs;
    const double2* F;
    double2* X;
    const double* D;    // per-plan pivots d'_i, M x N (coeff_tables_kernel)
    const double* Lm;   // per-plan multipliers l_i = a_i / d'_{i-2}, M x N (0 at a chain's first row)
    const double* tab_bad;  // [0] pivot-order violations / singular pivots found while building the tables
    double* stats;      // per rhs: [0..1] mean, [2] max|F|, [3] pivot-order violations
    const double2* z;   // Msin^-1 Msin^-1 w (check_mean_zero), length M
};

struct ResidualParams {
    int M, N;
    const double2* F;
    const double2* X;
    double* out;  // [0] interior max, [1] replaced-row abs, [2..3] constraint sum (re, im)
};

// Large transforms (grid_large.cu): the theta stage split over a cluster of
// 2Q CTAs (fq: the local length-L/Q transform), the lambda stages over a CTA
// pair (fh: the length-N/4 transform of one parity class).
struct ThetaLargeParams {
    ThetaParams t;
    FftDesc fq;
    int use_cmap;    // fold inputs through the column tensor map (single rank: contiguous columns)
    int fold_chunk;  // r per TMA stage of the fold (256 or 512, sized to the pivot window)
};
// Multi-pass theta stage (theta_mp.cu): the theta length L = L1 L2 through five
// coalesced passes; w1 / w2 hold 2 L complex per column (both parities).
struct ThetaMpParams {
    ThetaParams t;
    FftDesc f1;   // length L1, 16 threads per sequence
    FftDesc f2;   // length L2, 16 threads per sequence
    double2* w1;
    double2* w2;
};
size_t theta_mp_smem_bytes(int which, int L1, int L2, int nhi1, int nlo1, int nhi2, int nlo2, int nhiM, int nloM);
int theta_mp_chain_cap();
cudaError_t launch_theta_mp(const ThetaMpParams& Q, cudaStream_t st);
constexpr int kSplitBox = 256;   // modes per gather box of the split inverse lambda kernel
constexpr int kSplitPairs = 9;   // mode pairs (k, L - k) per thread it holds in registers (512 threads)
struct LambdaSplitParams {
    LambdaParams l;
    FftDesc fh;
    int aslots;  // data slots ahead of the tables: L/2 rounded up to swizzle blocks, or whole gather boxes
    int tma;     // inverse: gather the modes through the per-parity tensor maps
};
inline size_t theta_large_smem_bytes(int Lq, int nhiM, int nloM, int nhiq, int nloq) {
    return static_cast<size_t>((Lq + 7) & ~7) * 16 + static_cast<size_t>(nhiM + nloM + nhiq + nloq) * 16 +
           static_cast<size_t>((Lq + 4 + 1) & ~1) * 8 + 32 * 32 + 2 * 32 + 16 * 16 + 64 * 8 + 4 * 8;
}
inline int lambda_split_slots(int Lh, bool tma) {
    return tma ? (Lh / kSplitBox + 1) * kSplitBox : ((Lh + 7) & ~7);  // (Lh + 1 modes of the even class)
}
inline size_t lambda_split_smem_bytes(int Lh, int nhiN, int nloN, int nhih, int nloh, bool tma = false) {
    return static_cast<size_t>(lambda_split_slots(Lh, tma)) * 16 + static_cast<size_t>(nhiN + nloN + nhih + nloh) * 16 + 16;
}
cudaError_t launch_theta_large(const ThetaLargeParams& P, const CUtensorMap& cmap, int Q, int nthr, size_t smem,
                               cudaStream_t st);
cudaError_t launch_lambda_fwd_split(const LambdaSplitParams& P, int nthr, size_t smem, cudaStream_t st);
cudaError_t launch_lambda_inv_split(const LambdaSplitParams& P, const CUtensorMap& map0, const CUtensorMap& map1, int nthr,
                                    size_t smem, cudaStream_t st);

// Complex slots of the theta kernel's data buffer: the raw column (L+1)
// and whole 8-slot blocks for the swizzled layout.
__host__ __device__ inline int theta_data_slots(int L) { return ((L + 1) + 7) & ~7; }

// Pivot-reciprocal slots of the theta kernel (even, so later regions stay
// 16-byte aligned).
__host__ __device__ inline int theta_chain_slots(int L) { return ((L / 2 + 4) + 1) & ~1; }

// theta_sym_kernel (theta_sym.cu): pivot window (doubles, even) and chain
// slot window (uint32, multiple of 4) per CTA; the per-plan tables use the
// same row strides.
__host__ __device__ inline int theta_sym_piv_slots(int L) { return ((L / 2 + 2) + 1) & ~1; }
__host__ __device__ inline int theta_sym_pos_slots(int L) { return ((L / 2 + 1) + 3) & ~3; }
__host__ __device__ inline size_t theta_sym_smem_bytes(int L, int nhi, int nlo) {
    return static_cast<size_t>(theta_data_slots(L)) * 16 + static_cast<size_t>(nhi + nlo) * 16 +
           static_cast<size_t>(theta_sym_piv_slots(L)) * 8 + static_cast<size_t>(theta_sym_pos_slots(L)) * 4 +
           32 * 32 + 16 * 16 + 64 * 8 + 2 * 8;
}
cudaError_t launch_theta_sym(const ThetaParams& P, int nthr, size_t smem, cudaStream_t st);
cudaError_t launch_pivot_table_sym(int L, int k0, int ncols, double* ipt, int stride, cudaStream_t st);

// Dynamic shared memory of theta_kernel (bytes).
// ints of the theta kernel's digit-reversal window (one chain's slots)
__host__ __device__ inline int theta_rev_slots(int L) { return ((L / 2 + 9) + 3) & ~3; }
__host__ __device__ inline size_t theta_smem_bytes(int L, int nhi, int nlo, bool rev_win = false) {
    const size_t chain_max = static_cast<size_t>(theta_chain_slots(L));
    return static_cast<size_t>(theta_data_slots(L)) * 16 + static_cast<size_t>(nhi + nlo) * 16 + chain_max * 8 + 32 * 32 +
           16 * 16 + 64 * 8 + 2 * 8 + (rev_win ? static_cast<size_t>(theta_rev_slots(L)) * 4 : 0);
}

cudaError_t launch_lambda_fwd(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem, cudaStream_t st);
int exit_relaxed();  // 1 unless SK_PAIR_SYNC_EXIT is set: relaxed cluster exit barriers
bool lambda_inv_pair_ok(const LambdaParams& P, int nthr);
bool lambda_quad_ok(const LambdaParams& P, int nthr);  // inverse on CTA pairs (needs 2-row boxes)
cudaError_t launch_lambda_inv(const LambdaParams& P, const CUtensorMap& map, int nthr, size_t smem, cudaStream_t st);
// Lambda-stage shared memory (bytes) for transform length L and twiddle table sizes.
inline size_t lambda_smem_bytes(int L, int nhi, int nlo) {
    const size_t lpad = static_cast<size_t>((L / 256 + 1) * 256);
    return lpad * 16 + static_cast<size_t>(nhi + nlo) * 16 + static_cast<size_t>((L + 3) & ~3) * 4 + 32;
}
cudaError_t launch_theta(const ThetaParams& P, const CUtensorMap& cmap, const CUtensorMap& ctail, int nthr, size_t smem,
                         cudaStream_t st);
// lambda stages on row pairs inside one CTA (lambda_duo.cu); nthr = threads per row
size_t lambda_duo_smem_bytes(int L, int nhi, int nlo);
bool lambda_duo_ok(const LambdaParams& P, int nthr);
cudaError_t launch_lambda_fwd_duo(const LambdaParams& P, int nthr, cudaStream_t st);
cudaError_t launch_lambda_inv_duo(const LambdaParams& P, const CUtensorMap& map, int nthr, cudaStream_t st);
cudaError_t launch_shgen(const ShgenParams& P, cudaStream_t st);
cudaError_t launch_assemble(const AssembleParams& P, cudaStream_t st);
constexpr int kXformBox = 256;    // elements per gather box
constexpr int kXformStage = 20;   // gathered elements a thread re-slots through registers (512-thread variant)
constexpr int kXformStageHi = 8;  // ... of the 64-register variant (<= 256 threads, n <= 2048)
int xform_slots(int n, int n_src);
size_t xform_smem_bytes(int n, int nhi, int nlo, int n_src = 0);
cudaError_t launch_xform(const XformParams& P, const CUtensorMap& map, bool analyze, int nrows, int nthr, size_t smem,
                         cudaStream_t st);
cudaError_t launch_dfs_double(int m, int n, const double* phys, double2* grid, cudaStream_t st);
// theta_{m/2} = -pi + 2 pi (m/2) / m evaluated exactly as the reference does
// (sphere_domain.hpp:54, types.hpp:12-13) is negative: the reference's
// sample_dfs glides the pole row p = 0 (sk_internal.h GridGeom::pole_glide)
inline int pole_glide(int m) {
    const double kPi = 3.141592653589793238462643383279502884;
    const double kTwoPi = 2.0 * kPi;
    const int j = m / 2;
    return (-kPi + kTwoPi * j / m) < 0.0 ? 1 : 0;
}
cudaError_t launch_pivot_table(int L, int k0, int ncols, double* ipt, int stride, cudaStream_t st);
cudaError_t launch_coeff_solve(const CoeffParams& P, cudaStream_t st);
cudaError_t launch_coeff_tables(int M, int N, double* D, double* Lm, double* bad, cudaStream_t st);
// structure-preserving GE on a doubled grid (ge_kernels.cu).  scratch: ge_scratch_bytes(m, n) device bytes;
// doubles [0..5] of it receive the search result (sigma_1, candidate index t (n/2) + k - n/2 or -1, a, b),
// double [8] the max |residual| of a step / of launch_ge_maxabs.
constexpr int kGeParts = 2048;
size_t ge_scratch_bytes(int m, int n);
// half: g holds the (m/2+1) x n upper half grid (row i <-> theta_i = 2 pi i/m), as construct's phase 1 keeps it
cudaError_t launch_ge_search(int m, int n, bool half, const double2* g, void* scratch, cudaStream_t st);
cudaError_t launch_ge_step(int m, int n, bool half, const double2* g, int js, int ks, double2 de, double2 dodd, int has_e,
                           int has_o, double2* out, void* scratch, bool want_max, cudaStream_t st);
cudaError_t launch_ge_maxabs(long long total, const double2* g, void* scratch, cudaStream_t st);
cudaError_t launch_msin2(int M, int N, const double2* A, double2* F, cudaStream_t st);
cudaError_t launch_residual(const ResidualParams& P, cudaStream_t st);

}  // namespace sk
