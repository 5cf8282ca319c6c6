/* sk_poisson.h — C ABI of the B200-native DFS spectral Poisson solver.
 *
 * This is the drop-in boundary for the reference's Poisson entry points
 * (namespace spherekit, /root/reference/proj/include/spherekit/poisson.hpp):
 *
 *   reference (C++)                                      here (C ABI)
 *   -------------------------------------------------    ----------------------------
 *   PoissonSolution solve(const PoissonProblem&)         sk_solve_coeffs
 *       poisson.hpp:47, poisson.cpp:121-161
 *   ResidualReport residual(const PoissonProblem&,       sk_residual
 *       const PoissonSolution&)  poisson.hpp:54, .cpp:163-186
 *   PoissonProblem assemble_poisson(const              sk_assemble
 *       LowRankSphereFun&, int m, int n, AssembleReport*)
 *       poisson.hpp:40-41, poisson.cpp:52-86
 *   Matrix analyze_2d(const BMCGrid&)                    sk_analyze_2d
 *       fourier.hpp:107, fourier.cpp:170-188
 *   BMCGrid sample_grid(const CoeffMatrix&, int, int)     sk_sample_grid
 *       fourier.hpp:108, fourier.cpp:190-209
 *   BMCGrid sample_dfs(const sphere_fn&, int, int)        sk_sample_dfs (of samples)
 *       sphere_domain.hpp:61, sphere_domain.cpp:46-52
 *   sample_dfs -> analyze_2d -> Msin^2 -> solve ->       sk_solve_grid
 *       sample_grid (the grid-level composition:
 *       sphere_domain.cpp:46-52, fourier.cpp:170-209,
 *       poisson.cpp:61-71, :121-161)
 *   test helper real_sph_harmonic sums                   sk_shgen (input generator)
 *       (tests/support/helpers.hpp:18-27)
 *
 * Layouts (bit-exact contract):
 *   coefficient matrices F, X: row-major M x N complex double, interleaved
 *     (re, im) — std::complex<double> layout (types.hpp:17-41); row i is theta
 *     mode j = i - M/2, column kc is lambda mode k = kc - N/2;
 *   physical grids f, u: row-major (M/2+1) x N real double; row p is
 *     theta_p = 2 pi p / M (p = 0 and p = M/2 are the poles), column q is
 *     lambda_q = -pi + 2 pi q / N.  The doubled grid of sample_dfs is never
 *     materialised (its rows j < M/2 are the glide reflection of row M/2 - j).
 *
 * Errors: every call returns an sk_status; sk_last_error() describes the last
 * failure on the calling thread.  The C++ shim (spherekit/poisson_b200.hpp)
 * rethrows SK_ERR_SIZE as spherekit::size_error, SK_ERR_PRECONDITION as
 * precondition_error and SK_ERR_SINGULAR as structure_error, as the reference
 * throws them (poisson.cpp:123-124, :115-116; banded.cpp:132, :306).
 *
 * Threading: a plan owns device buffers and a stream; one plan must not be
 * used from two threads at once; distinct plans are independent.  There is no
 * CPU fallback: without a usable sm_100 device every compute call fails with
 * SK_ERR_CUDA.
 */
#ifndef SK_POISSON_H
#define SK_POISSON_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sk_status {
    SK_OK = 0,
    SK_ERR_SIZE = 1,          /* non-positive or odd sizes (reference size_error)     */
    SK_ERR_PRECONDITION = 2,  /* right-hand side with nonzero surface mean            */
    SK_ERR_SINGULAR = 3,      /* numerically singular band system (structure_error)  */
    SK_ERR_CUDA = 4,          /* CUDA runtime / launch failure, or no device          */
    SK_ERR_UNSUPPORTED = 5,   /* size outside this build's FFT / on-chip limits       */
    SK_ERR_ARGUMENT = 6,      /* null pointer, bad flag, wrong plan kind              */
    SK_ERR_NCCL = 7           /* reserved for the collective layer                    */
} sk_status;

typedef struct sk_plan_s* sk_plan_t;

/* flags for data arguments */
#define SK_HOST 0u     /* pointers are host memory (copies inside the call)   */
#define SK_DEVICE 1u   /* pointers are device memory on the plan's device    */
#define SK_GE_HALF 8u  /* sk_ge_*: the grid is the (m/2+1) x n upper half (below)    */
#define SK_ASYNC 2u    /* do not synchronise before returning.  Device
                          pointers: work is queued on the plan stream.  Host
                          pointers (sk_solve_grid): the solve is pipelined —
                          H2D copy, transforms and D2H copy on three streams
                          with three device slots, so consecutive calls overlap
                          their copies with each other's compute; f and u must
                          stay valid (and should be pinned) until sk_sync.
                          Errors that need a host-side check, e.g. the mean
                          precondition, are reported by a later call or by
                          sk_sync */

/* Create a plan for an M x N problem (M = doubled theta count, N = lambda
 * count, both even) with `nrhs` independent right-hand sides on CUDA device
 * `device`.  Grid-path sizes must factor into 2,3,5,7 with M/2 and N/2 within
 * the on-chip limits reported by sk_plan_info (else SK_ERR_UNSUPPORTED; the
 * coefficient-space solve accepts any even sizes).  Replaces the per-call
 * operator construction of poisson.cpp:127-128 / fourier.cpp:22-35. */
sk_status sk_plan_create(int M, int N, int nrhs, int device, sk_plan_t* plan);
sk_status sk_plan_destroy(sk_plan_t plan);
/* Use an external CUDA stream (cudaStream_t) for all work of this plan. */
sk_status sk_plan_set_stream(sk_plan_t plan, void* stream);
sk_status sk_sync(sk_plan_t plan);

/* Coefficient-space solve, the drop-in for spherekit::solve(PoissonProblem):
 * X = solution of the N decoupled banded systems with the (j=0,k=0) row
 * replaced by 2 pi w^T X_0 = 0.  Bit-identical to the reference for every
 * k != 0 column (ascending Thomas on the four exact-zero-decoupled chains,
 * IEEE mul/sub/div in the reference's order, no FMA); k = 0 agrees to
 * rounding.  Checks the nonzero-mean precondition like check_mean_zero
 * (poisson.cpp:101-117).  F and X: nrhs consecutive M x N complex matrices. */
sk_status sk_solve_coeffs(sk_plan_t plan, const double* F, double* X, unsigned flags);

/* Residual report (poisson.cpp:163-186) for one right-hand side:
 * out[0] = interior max |(lap - k^2) X_k - F_k| over all equations but
 * (j=0,k=0); out[1] = that replaced equation's |defect|; out[2] = |2 pi w^T X_0|. */
sk_status sk_residual(sk_plan_t plan, const double* F, const double* X, double out[3], unsigned flags);

/* Grid-level solve: physical samples f -> physical solution u of
 * Lap u = f with integral(u) = 0, through DFS doubling, the 2D trigonometric
 * transforms, Msin^2, the per-mode banded solves and the inverse transforms.
 * f and u: nrhs consecutive (M/2+1) x N real grids (may alias).
 * If X_half != NULL it receives the solution coefficients for lambda modes
 * k = 0..N/2 as an (N/2+1) x M complex array, X_half[k][i] = X[i][k + N/2]
 * (the k < 0 half is its complex conjugate, reflected: real data). */
sk_status sk_solve_grid(sk_plan_t plan, const double* f, double* u, double* X_half, unsigned flags);

/* Reference-semantics grid solve: exactly the composition the reference runs
 * — sample_dfs (sphere_domain.cpp:46-52) -> analyze_2d (fourier.cpp:170-188)
 * -> Msin^2 per column (poisson.cpp:61) -> solve (poisson.cpp:121-161) ->
 * sample_grid (fourier.cpp:190-209) — on the device.  All N lambda modes are
 * solved (k < 0 too), so U is the reference's complex M x N doubled grid
 * (BMCGrid layout, row j <-> theta_j = -pi + 2 pi j/M) for ANY input, also
 * where under-resolved data make it differ from the real, Hermitian grid
 * solve above (the reference's truncated theta operators are not mirror-
 * symmetric at j = -M/2).  f: nrhs x (M/2+1) x N real; U: nrhs x M x N
 * complex; X (may be NULL): nrhs x M x N complex solution coefficients.
 * M and N: any even sizes the standalone transforms take (below).  Same
 * precondition / error behaviour as sk_solve_coeffs. */
sk_status sk_solve_grid_exact(sk_plan_t plan, const double* f, double* U, double* X, unsigned flags);

/* Surface mean 2 pi w^T f~_0 of the last grid solve's right-hand side and
 * max|F| of its coefficients (for callers that want the precondition data). */
sk_status sk_last_mean(sk_plan_t plan, double out[3]);

/* assemble_poisson (poisson.hpp:40-41, poisson.cpp:52-86): the plan's M x N
 * coefficient matrix F of sin^2(theta) f~ for a low-rank function
 * f~ = sum_j d_j a_j(theta) b_j(lambda) given by its factors (the fields of
 * LowRankSphereFun, lowrank.hpp:47-59): d[K] complex, col[K][mf] complex
 * (theta coefficients, mode t at index t + mf/2), row[K][nf] complex, vscale.
 * Factors are zero-padded / truncated to M and N as pad_to does
 * (fourier.cpp:105-112).  If the surface mean mu = sum2(f)/(4 pi) exceeds
 * 1e-11 max(vscale, 1e-300) its sin^2 coefficients are subtracted, as the
 * reference does; report[3] (host, may be NULL) = {removed (0/1), mu re,
 * mu im} (AssembleReport).  F is bit-identical to the reference.  Flags:
 * SK_HOST / SK_DEVICE for d, col, row and F together.  Needs M >= 4. */
sk_status sk_assemble(sk_plan_t plan, int K, int mf, int nf, const double* d, const double* col, const double* row,
                      double vscale, double* F, double report[3], unsigned flags);

/* Standalone transforms of the reference's Fourier layer on complex data of
 * any even size (the plan supplies device, stream and scratch; its own M, N
 * are not used).  Lengths that factor into 2, 3, 5, 7 run the mixed-radix
 * engine (<= ~12000 per CTA); lengths with a larger prime factor (e.g. 602 =
 * 2 * 7 * 43, acceptance c11) a Bluestein chirp-z convolution of a smooth
 * length >= 2n - 1 (n <= ~6000); beyond, SK_ERR_UNSUPPORTED.  Layouts:
 * row-major complex.
 *   sk_analyze_2d   analyze_2d(BMCGrid) (fourier.hpp:107, fourier.cpp:170-188):
 *                   m x n doubled sample grid -> m x n coefficients X.
 *   sk_sample_grid  sample_grid(X, m_out, n_out) (fourier.hpp:108,
 *                   fourier.cpp:190-209): rows x cols coefficients ->
 *                   m_out x n_out grid, zero-padding or truncating the modes
 *                   as synthesize_1d does (:55-66).
 *   sk_sample_dfs   sample_dfs (sphere_domain.hpp:61, sphere_domain.cpp:19-26,
 *                   :46-52) of physical samples ((m/2+1) x n real, rows
 *                   theta_p = 2 pi p/m) -> the m x n doubled grid (complex,
 *                   imaginary parts 0): the glide-reflection index map. */
sk_status sk_analyze_2d(sk_plan_t plan, int m, int n, const double* grid, double* X, unsigned flags);
sk_status sk_sample_grid(sk_plan_t plan, int rows, int cols, const double* X, int m_out, int n_out, double* grid,
                         unsigned flags);
sk_status sk_sample_dfs(sk_plan_t plan, int m, int n, const double* phys, double* grid, unsigned flags);

/* Structure-preserving Gaussian elimination on a doubled BMC grid: the
 * building blocks of the low-rank constructor (lowrank.hpp:
 * 73-93).  The phase-1 loop of construct (lowrank.cpp:318-415, update :384-392)
 * runs the same arithmetic on the upper half grid.
 *   sk_ge_pivot_search  pivot_search (lowrank.cpp:84-112): complete pivoting
 *                       over the 2x2 blocks {(lambda* - pi, theta*), (lambda*,
 *                       theta*)}, theta* = 2 pi t/m (t = 0..m/2 ascending),
 *                       lambda* = lambda_k (k = n/2..n-1 ascending), first
 *                       maximal sigma_1 = max(|a+b|, |a-b|) wins; the weights
 *                       (m_even, m_odd) = pinv_2x2(a, b, alpha) (:60-72).
 *                       out_i = {found, t, k}; out_d = {a, b, m_even, m_odd
 *                       (re, im each), theta_star, lambda_star}.
 *   sk_ge_step          ge_step (lowrank.cpp:127-162): out = grid - (1/2
 *                       m_even ce re^T + 1/2 m_odd co ro^T) for the pivot
 *                       piv (the 10 doubles above; the node is located as
 *                       locate_on_grid does), bit-identical to the reference.
 *   sk_ge_run           the elimination loop with the grid resident on the
 *                       device: max|grid| -> while it exceeds tau and steps <
 *                       max_steps: pivot search, update (in place), max|grid|.
 *                       resid[0] = max before the first step, resid[s + 1]
 *                       after step s; piv_i (2 ints) / piv_d (10 doubles) per
 *                       step as above.  The caller keeps construct's policy
 *                       (plateau bookkeeping, rank limits) on the host.
 * grid / out: m x n complex, row-major (BMCGrid, sphere_domain.hpp:43-58);
 * host or device pointers by flags.  With SK_GE_HALF the arrays hold only the
 * upper half grid, (m/2+1) x n with row i <-> theta_i = 2 pi i/m, exactly as
 * construct's phase 1 keeps it (lowrank.cpp:246-252: the lower half is implied
 * by the glide symmetry; the row of -theta* is the pivot row shifted by pi in
 * lambda, :370-378) - half the bytes per step, the same pivots and the same
 * bits on the stored rows for BMC-symmetric data.  Errors: SK_ERR_SIZE (odd or non-positive
 * sizes), SK_ERR_ARGUMENT (a pivot that is not a grid node: index_error). */
sk_status sk_ge_pivot_search(sk_plan_t plan, int m, int n, const double* grid, double alpha, int out_i[3],
                             double out_d[10], unsigned flags);
sk_status sk_ge_step(sk_plan_t plan, int m, int n, const double* grid, const double piv[10], double* out,
                     unsigned flags);
sk_status sk_ge_run(sk_plan_t plan, int m, int n, double* grid, double alpha, double tau, int max_steps, int* nsteps,
                    int* piv_i, double* piv_d, double* resid, unsigned flags);

/* Seeded spherical-harmonic input generator (untimed helper):
 * phys = sum_{l=1..L} sum_{|m|<=l} coeffs[l*l+l+m] Y_l^m on the plan's
 * physical grid, Y as in the reference tests (helpers.hpp:18-27).
 * coeffs: (L+1)^2 doubles; phys: (M/2+1) x N real; both device pointers. */
sk_status sk_shgen(sk_plan_t plan, int L, const double* coeffs_dev, double* phys_dev);

/* Stage entry points for the slab-decomposed multi-GPU solve (one plan per
 * rank; the transposes between them are collectives run by the caller).
 * Spectrum blocks use the all-to-all layout described in DESIGN.md §5:
 *   sk_stage_lambda_fwd: rows [r0, r1) of f -> send buffer, blocks per
 *     destination d ordered [d][k - k0_d][p - r0] (complex);
 *   sk_stage_theta:      columns [k0, k1) read from the receive buffer,
 *     blocks per source s ordered [s][k - k0][p - r0_s], solved in place;
 *   sk_stage_lambda_inv: rows [r0, r1) of u from the returned blocks.
 * row_bounds[P+1] and col_bounds[P+1] give every rank's slab. */
sk_status sk_stage_lambda_fwd(sk_plan_t plan, int P, const int* row_bounds, const int* col_bounds, int rank,
                              const double* f_rows_dev, double* send_dev);
sk_status sk_stage_theta(sk_plan_t plan, int P, const int* row_bounds, const int* col_bounds, int rank,
                         double* recv_dev);
sk_status sk_stage_lambda_inv(sk_plan_t plan, int P, const int* row_bounds, const int* col_bounds, int rank,
                              const double* back_dev, double* u_rows_dev);

/* Fused-transpose variants (one process per GPU over NVLink / NVSwitch): the
 * forward lambda stage stores mode k of its rows straight into the receive
 * buffer of the rank owning k, and the theta stage stores row p of its solved
 * columns straight into the return buffer of the rank owning p, so neither
 * exchange needs a collective.  peer_recv[d] / peer_back[d] are every rank's
 * buffers as mapped in this process (sk_ipc_open; this rank's own buffer for
 * d = rank); layouts as for sk_stage_theta / sk_stage_lambda_inv.  All ranks
 * must finish a stage before any rank starts the next one (the caller's
 * barrier), and sk_stage_lambda_inv then reads the local return buffer. */
sk_status sk_stage_lambda_fwd_peer(sk_plan_t plan, int P, const int* row_bounds, const int* col_bounds, int rank,
                                   const double* f_rows_dev, void* const* peer_recv);
sk_status sk_stage_theta_peer(sk_plan_t plan, int P, const int* row_bounds, const int* col_bounds, int rank,
                              double* recv_dev, void* const* peer_back);

/* Device buffers that can be shared with other processes, and their CUDA IPC
 * handles (64 bytes) / mappings. */
sk_status sk_device_alloc(int device, size_t bytes, void** ptr);
sk_status sk_device_free(void* ptr);
sk_status sk_ipc_handle(const void* ptr, unsigned char handle[64]);
sk_status sk_ipc_open(int device, const unsigned char handle[64], void** ptr);
sk_status sk_ipc_close(void* ptr);

/* Stream-ordered hand-over between ranks of the fused slab solve without
 * draining a stream: interprocess events (cudaEventInterprocess) recorded
 * on a plan's stream behind a stage, opened by the peers from their 64-byte
 * handles, and waited on by the peers' streams before the stage that reads
 * what it wrote (the host only orders the record before the wait).  No
 * kernel ever spins on another rank. */
sk_status sk_ipc_event_create(int device, unsigned char handle[64], void** event);
sk_status sk_ipc_event_open(int device, const unsigned char handle[64], void** event);
sk_status sk_event_destroy(void* event);
sk_status sk_event_record(sk_plan_t plan, void* event);
sk_status sk_stream_wait_event(sk_plan_t plan, void* event);
/* Mean / max|F| statistics of the plan's last theta stage entry point
 * (out[0..1] the surface mean of the k = 0 owner, out[2] max|F| of its modes),
 * waiting only for that stage's copy to the host. */
sk_status sk_stage_stats(sk_plan_t plan, double out[3]);

/* Plan facts: info[0] = M, [1] = N, [2] = nrhs, [3] = device,
 * [4] = grid path supported (1/0), [5] = spectrum leading dimension,
 * [6] = theta-stage split (CTAs per column), [7] = theta-stage threads,
 * [8] = lambda-stage threads, [9] = kernels launched by the last call,
 * [10]/[11] = theta/lambda shared memory per CTA (bytes), [12] = theta chain
 * solver (0 shared-memory walk, 1 fixed segments, 2 12-element register
 * walk), [13] = kernel variants (bit 0 high-occupancy theta kernel, bit 1
 * high-occupancy lambda kernels, bit 2 swizzled theta slots, bit 3 swizzled
 * lambda slots, bit 4 forward lambda rows on CTA pairs, bit 5 inverse lambda
 * rows on CTA pairs, bit 6 theta_sym_kernel (pruned forward transform, paired
 * chains), bit 7 forward lambda rows on 4-CTA clusters (peer stores / opt-in)). */
sk_status sk_plan_info(sk_plan_t plan, long long info[16]);

/* Time one launch of each stage (device events, ms): t[0] lambda_fwd,
 * t[1] theta, t[2] lambda_inv, t[3] coeff solve (last measured). */
sk_status sk_stage_times(sk_plan_t plan, double t[4]);
sk_status sk_enable_stage_timing(sk_plan_t plan, int on);

const char* sk_last_error(void);
const char* sk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SK_POISSON_H */
