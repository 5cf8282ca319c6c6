// Internal declarations shared by the host plan code and the CUDA kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace sk {

// cudaFuncSetAttribute acts on the current device's context: launchers keep
// one bit per device of the kernels they configured, set only after the
// attribute calls returned (two threads may both configure; never neither),
// so a plan on a second device configures its kernels again.
template <class Fn>
inline void configure_on_device(std::atomic<unsigned long long>& done, Fn&& set_attributes) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    set_attributes();
    done.fetch_or(bit, std::memory_order_release);
}

constexpr int kMaxStages = 24;
constexpr int kMaxRanks = 16;

// In-place mixed-radix Cooley-Tukey FFT of length L in shared memory:
// forward = decimation in frequency (natural in -> digit-reversed out),
// inverse = decimation in time (digit-reversed in -> natural out).
// Stage s has radix R[s], sub-block size sz[s] = L/(R[0]..R[s-1]) and
// span[s] = sz[s]/R[s]; its twiddles are omega_sz^(q j) = table index
// q*j*tw[s] of the 2L-th roots (tw[s] = 2L/sz[s]).
struct FftDesc {
    int L = 0;
    int nst = 0;
    int R[kMaxStages] = {};
    int span[kMaxStages] = {};
    int tw[kMaxStages] = {};
    // b / span[s] as ((umulhi(b, mag) + ((b - umulhi) >> sh1)) >> sh2) (Granlund-Montgomery)
    unsigned mag[kMaxStages] = {};
    int sh1[kMaxStages] = {};
    int sh2[kMaxStages] = {};
    // twiddle table for the 2L-th roots exp(-2 pi i m / 2L), m in [0, 2L):
    // T(m) = hi[m >> shift] * lo[m & (B-1)], B = 1 << shift
    int shift = 0;
    int nhi = 0;
    int nlo = 0;
    const double2* hi = nullptr;  // device, nhi entries
    const double2* lo = nullptr;  // device, nlo entries
    const int* rev = nullptr;     // device, L entries: natural index -> DIF output position
};

// Slab decomposition of one right-hand side over P ranks (P = 1 on a single
// GPU).  Physical rows p in [0, M/2] are split by row_b, lambda modes
// k in [0, N/2] by col_b.
struct Slabs {
    int P = 1;
    int rank = 0;
    int row_b[kMaxRanks + 1] = {};
    int col_b[kMaxRanks + 1] = {};
};

// Destinations of a stage's output in other ranks' buffers (device pointers
// valid in this process: CUDA IPC mappings of the peers' allocations).  The
// element with owner index idx and coordinates (a, b) goes to
// base[d] + off[d] + a mul[d] + b, d the rank with bound[d] <= idx < bound[d+1].
struct PeerMap {
    double2* base[kMaxRanks] = {};
    long long off[kMaxRanks] = {};
    int mul[kMaxRanks] = {};
    int bound[kMaxRanks + 1] = {};
    int n = 0;  // 0: the stage writes its own buffer
};

struct GridGeom {
    int M = 0, N = 0;
    int Lt = 0;   // theta FFT length M/2
    int Ll = 0;   // lambda FFT length N/2
    int rows = 0; // M/2 + 1 physical rows
    int cols = 0; // N/2 + 1 lambda modes (k >= 0)
    // The reference's sample_dfs evaluates theta_j = -pi + 2 pi j / M in
    // floating point (sphere_domain.hpp:54) and dfs_extend glides every
    // theta < 0 (sphere_domain.cpp:19-26).  For some M (22, 30, 44, 60, ...)
    // theta_{M/2} rounds to a tiny negative number, so the doubled row j = M/2
    // reads the pole row p = 0 at longitude lambda -+ pi: spectrally s = (-1)^k
    // times its own coefficients.  Replicated when set (sk_pole_glide).
    int pole_glide = 0;
};

}  // namespace sk
