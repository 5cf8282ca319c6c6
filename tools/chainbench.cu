// Chain-solve microbenchmark: cycles per chain solve of the theta kernel's
// solvers on one (lambda mode, parity) column resident in shared memory, one
// CTA per SM.  Usage: chainbench L nthr k variant R0 R1 ...  (variant: 0 smem walk,
// 1 fixed segments, 2 SMAX=12 register walk)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <numeric>

#include "../paper_1510_08094_b200/csrc/grid_kernels.cu"

namespace sk {
template <int VAR>
__global__ void __launch_bounds__(512) chain_bench(FftDesc fd, int kg, const int* rev, const double* piv, int reps,
                                                   long long* cyc) {
    const int L = fd.L;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double* ip = reinterpret_cast<double*>(a + theta_data_slots(L));
    V4* wsc = reinterpret_cast<V4*>(ip + theta_chain_slots(L));
    double2* misc = reinterpret_cast<double2*>(wsc + 32);
    const int tid = threadIdx.x, nthr = blockDim.x;
    Chain cp, cm;
    make_chains(0, L, cp, cm);
    for (int i = tid; i < L; i += nthr) a[i] = make_double2(1e-3 * ((i * 7919) % 1000), 1e-3 * ((i * 104729) % 1000));
    uint32_t pb = 0;
    const double* ipw = pivot_window(ip, piv, 0, cp.tau0, cp.tau0 + cp.n, pb);
    const size_t a0 = static_cast<size_t>(cp.tau0) & ~static_cast<size_t>(1);
    for (uint32_t i = tid; i < pb / 8; i += nthr) ip[i] = piv[a0 + i];
    __syncthreads();
    double fmax_acc = 0.0;
    double2 wsum = make_double2(0.0, 0.0);
    unsigned fh = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if constexpr (VAR == 0) solve_chain(a, rev, ipw, wsc, cp, L, misc[0], fmax_acc, wsum, false, &misc[3]);
        else if constexpr (VAR == 1) {
            if (!solve_chain_fast_dispatch(a, fd.rev, ipw, reinterpret_cast<Aff3*>(wsc), cp, L, misc[0], &fh, &wsum,
                                           false, &misc[3]))
                solve_chain(a, rev, ipw, wsc, cp, L, misc[0], fmax_acc, wsum, false, &misc[3]);
        } else solve_chain_reg<kSegMax>(a, rev, ipw, wsc, cp, L, misc[0], fmax_acc, wsum, false, &misc[3]);
    }
    const long long t1 = clock64();
    if (tid == 0) {
        cyc[blockIdx.x] = t1 - t0;
        misc[5].x = fmax_acc + fh + wsum.x;
    }
}
}  // namespace sk

using namespace sk;
int main(int argc, char** argv) {
    const int L = atoi(argv[1]), nthr = atoi(argv[2]), kg = atoi(argv[3]), var = atoi(argv[4]);
    // a real DIF plan (radices from the command line) and its digit reversal
    std::vector<int> R;
    for (int i = 5; i < argc; ++i) R.push_back(atoi(argv[i]));
    FftDesc fd;
    fd.L = L;
    fd.nst = static_cast<int>(R.size());
    int sz = L;
    for (int st = 0; st < fd.nst; ++st) {
        fd.R[st] = R[st];
        fd.span[st] = sz / R[st];
        sz /= R[st];
    }
    std::vector<int> rev(L);
    for (int k = 0; k < L; ++k) {
        int kk = k, pos = 0;
        for (int st = 0; st < fd.nst; ++st) {
            pos += (kk % fd.R[st]) * fd.span[st];
            kk /= fd.R[st];
        }
        rev[k] = pos;
    }
    int* drev;
    double* dpiv;
    long long* cyc;
    cudaMalloc(&drev, 4 * L);
    cudaMemcpy(drev, rev.data(), 4 * L, cudaMemcpyHostToDevice);
    fd.rev = drev;
    cudaMalloc(&dpiv, 8 * 2 * L * (kg + 1));
    launch_pivot_table(L, 0, kg + 1, dpiv, L, 0);
    cudaMalloc(&cyc, 8 * 148);
    const size_t smem = 200 * 1024;
    const double* prow = dpiv + static_cast<size_t>(kg) * 2 * L;
    const int reps = 20;
    auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<148, nthr, smem>>>(fd, kg, drev, prow, 2, cyc);
        kern<<<148, nthr, smem>>>(fd, kg, drev, prow, reps, cyc);
    };
    if (var == 0) run(chain_bench<0>);
    else if (var == 1) run(chain_bench<1>);
    else run(chain_bench<2>);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<long long> c(148);
    cudaMemcpy(c.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
    double m = 0;
    for (auto v : c) m += v;
    m /= 148;
    printf("L=%d nthr=%d k=%d var=%d cycles/chain=%.0f per element %.3f\n", L, nthr, kg, var, m / reps,
           m / reps / (L / 2));
#ifdef SK_PHASES
    std::vector<unsigned long long> ph(4096 * 24);
    cudaMemcpyFromSymbol(ph.data(), sk::g_phase, 8 * 4096 * 24);
    const char* nm[] = {"loads", "pass1", "scan1", "pass2", "scan2", "pass3"};
    double acc[6] = {0};
    for (int b = 0; b < 148; ++b)
        for (int i = 0; i < 5; ++i) acc[i + 1] += double(ph[b * 24 + 13 + i] - ph[b * 24 + 12 + i]);
    for (int i = 1; i < 6; ++i) printf("   %s %.0f\n", nm[i], acc[i] / 148);
#endif
    return 0;
}
