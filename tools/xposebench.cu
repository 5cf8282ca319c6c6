// Microbenchmark: the memory access patterns of the three grid-path stages
// without their arithmetic, at C3 sizes (R = 10001 physical rows of N = 10000
// reals, C = 5001 lambda modes), to separate pattern cost from compute.
//   copy        contiguous read + write of the same bytes (baseline)
//   fwd_scatter row read contiguous, 16-byte stores to S[k][p] (lambda_fwd today)
//   fwd_tileT   row read, stores to S[k/T][p][k%T] (T consecutive modes per p)
//   inv_gather  16-byte loads of S[k][p] for one p, row stored (lambda_inv today)
//   inv_tileT   loads of S[k/T][p][k%T], row stored
//   col         one CTA per mode: S[k][0..R) loaded and stored back (theta today)
//   col_tileT   one CTA per mode over the tiled layout (stride T*16 bytes)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int R = 10001, N = 10000, C = N / 2 + 1, L = N / 2;

__device__ __forceinline__ size_t sidx(int T, int k, int p) {
    return T == 1 ? (size_t)k * R + p : ((size_t)(k / T) * R + p) * T + (k % T);
}

__global__ void copy_k(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}

template <int T>
__global__ void __launch_bounds__(256) fwd_k(const double* __restrict__ f, double2* __restrict__ S) {
    const int p = blockIdx.x;
    const double2* row = reinterpret_cast<const double2*>(f + (size_t)p * N);
    // per mode one 16-byte value (two consecutive reals of the row as stand-in)
    for (int k = threadIdx.x; k < C; k += blockDim.x) {
        double2 v = row[k < L ? k : 0];
        S[sidx(T, k, p)] = v;
    }
}

template <int T>
__global__ void __launch_bounds__(256) inv_k(const double2* __restrict__ S, double* __restrict__ u) {
    const int p = blockIdx.x;
    double2* row = reinterpret_cast<double2*>(u + (size_t)p * N);
    for (int k = threadIdx.x; k < L; k += blockDim.x) row[k] = S[sidx(T, k, p)];
}

template <int T>
__global__ void __launch_bounds__(512) col_k(double2* __restrict__ S, double2* __restrict__ S2) {
    const int k = blockIdx.x;
    for (int p = threadIdx.x; p < R; p += blockDim.x) S2[sidx(T, k, p)] = S[sidx(T, k, p)];
}

// lambda_fwd store pattern with the kernel's occupancy (80 KB row in shared
// memory, 2 CTAs/SM): (a) one CTA per row, 16-byte stores S[k][p]; (b) a CTA
// pair per row pair exchanging halves through DSMEM, 32-byte stores of
// (p, p+1) per mode.
__global__ void __launch_bounds__(256, 2) fwd_smem_single(const double* __restrict__ f, double2* __restrict__ S) {
    extern __shared__ double2 sm[];
    const int p = blockIdx.x;
    const double2* row = reinterpret_cast<const double2*>(f + (size_t)p * N);
    for (int k = threadIdx.x; k < L; k += blockDim.x) sm[k] = row[k];
    __syncthreads();
    for (int k = threadIdx.x; k < C; k += blockDim.x) S[(size_t)k * R + p] = sm[k < L ? k : 0];
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) fwd_smem_pair(const double* __restrict__ f, double2* __restrict__ S) {
    extern __shared__ double2 sm[];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int r = cl.block_rank();
    const int p = (blockIdx.x >> 1) * 2 + r;
    if (p < R) {
        const double2* row = reinterpret_cast<const double2*>(f + (size_t)p * N);
        for (int k = threadIdx.x; k < L; k += blockDim.x) sm[k] = row[k];
    }
    cl.sync();
    const double2* s0 = cl.map_shared_rank(sm, 0);
    const double2* s1 = cl.map_shared_rank(sm, 1);
    const int p0 = (blockIdx.x >> 1) * 2;
    const int kb = r == 0 ? 0 : C / 2, ke = r == 0 ? C / 2 : C;
    for (int k = kb + threadIdx.x; k < ke; k += blockDim.x) {
        const int kk = k < L ? k : 0;
        const double2 v0 = s0[kk];
        if (p0 + 1 < R) {
            const double2 v1 = s1[kk];
            double4 w = make_double4(v0.x, v0.y, v1.x, v1.y);
            *reinterpret_cast<double4*>(S + (size_t)k * (R + 1) + p0) = w;  // row stride R+1 keeps 32-byte alignment
        } else {
            S[(size_t)k * (R + 1) + p0] = v0;
        }
    }
    cl.sync();
}

int main() {
    double *f, *u;
    double2 *S, *S2;
    const size_t nrow = (size_t)R * N, ns = (size_t)(C + 8) * R;
    CK(cudaMalloc(&f, nrow * 8));
    CK(cudaMalloc(&u, nrow * 8));
    CK(cudaMalloc(&S, ns * 16));
    CK(cudaMalloc(&S2, ns * 16));
    cudaMemset(f, 0, nrow * 8);
    cudaMemset(S, 0, ns * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes_stage = nrow * 8.0 + (double)C * R * 16.0;  // 1.6 GB
    auto run = [&](const char* name, auto launch, double bytes) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        const int it = 10;
        cudaEventRecord(e0);
        for (int i = 0; i < it; ++i) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= it;
        printf("%-14s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / ms / 1e6);
    };
    run("copy", [&] { copy_k<<<148 * 8, 256>>>(S, S2, (size_t)C * R); }, 2.0 * C * R * 16);
    run("fwd_scatter", [&] { fwd_k<1><<<R, 256>>>(f, S); }, bytes_stage);
    run("fwd_tile2", [&] { fwd_k<2><<<R, 256>>>(f, S); }, bytes_stage);
    run("fwd_tile4", [&] { fwd_k<4><<<R, 256>>>(f, S); }, bytes_stage);
    run("fwd_tile8", [&] { fwd_k<8><<<R, 256>>>(f, S); }, bytes_stage);
    run("inv_gather", [&] { inv_k<1><<<R, 256>>>(S, u); }, bytes_stage);
    run("inv_tile2", [&] { inv_k<2><<<R, 256>>>(S, u); }, bytes_stage);
    run("inv_tile4", [&] { inv_k<4><<<R, 256>>>(S, u); }, bytes_stage);
    run("inv_tile8", [&] { inv_k<8><<<R, 256>>>(S, u); }, bytes_stage);
    cudaFuncSetAttribute(fwd_smem_single, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(fwd_smem_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    run("fwd_smem_1", [&] { fwd_smem_single<<<R, 256, 100 * 1024>>>(f, S); }, bytes_stage);
    run("fwd_smem_pair", [&] { fwd_smem_pair<<<(R + 1) / 2 * 2, 256, 100 * 1024>>>(f, S); }, bytes_stage);
    run("col", [&] { col_k<1><<<C, 512>>>(S, S2); }, 2.0 * C * R * 16);
    run("col_tile2", [&] { col_k<2><<<C, 512>>>(S, S2); }, 2.0 * C * R * 16);
    run("col_tile4", [&] { col_k<4><<<C, 512>>>(S, S2); }, 2.0 * C * R * 16);
    run("col_tile8", [&] { col_k<8><<<C, 512>>>(S, S2); }, 2.0 * C * R * 16);
    return 0;
}
