// Microbenchmark: FP64 FMA throughput and latency on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void thr(double* out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void lat(double* out, int iters, long long* cyc) {
    double a = threadIdx.x;
    const double b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lds_lat(double* out, int iters, long long* cyc) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int p = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = idx[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {8, 16, 32, 64}) {
        thr<<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e0);
        thr<<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = double(sms) * warps * 32 * iters * 8;
        printf("warps/SM %2d: %.2f TFLOP/s FP64 (FMA=2), %.1f FMA/clk/SM at %.0f MHz\n", warps, 2 * fmas / ms / 1e9,
               fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
    }
    long long h;
    lat<<<1, 32>>>(out, 10000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", h / 10000.0);
    lds_lat<<<1, 32>>>(out, 10000, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.2f cycles\n", h / 10000.0);
    return 0;
}
