// FFT microbenchmark: cycles per in-place forward+inverse pair of the shared-
// memory engine (fft_dev.cuh) for a given length / radix plan / block size,
// one CTA per SM (smem padded to force it).  Usage: fftbench L nthr R0 R1 ...
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1510_08094_b200/csrc/fft_dev.cuh"

using namespace sk;

__global__ void __launch_bounds__(512) bench(FftDesc d, int reps, long long* cyc, double2* out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* a = reinterpret_cast<double2*>(smem_raw);
    double2* th = a + d.L;
    double2* tl = th + d.nhi;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const Tw T = load_tw(d, th, tl, tid, nthr);
    for (int i = tid; i < d.L; i += nthr) a[i] = make_double2(sin(0.1 * i + blockIdx.x), cos(0.3 * i));
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        fft_forward<false>(a, d, T, tid, nthr);
        fft_inverse<false>(a, d, T, tid, nthr);
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (tid == 0) out[blockIdx.x] = a[1];
}

static void root(long long m, long long n, double& c, double& s) {
    m %= n; if (m < 0) m += n;
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double a = 2.0L * pi * (long double)m / (long double)n;
    c = (double)cosl(a); s = (double)-sinl(a);
}

int main(int argc, char** argv) {
    const int L = atoi(argv[1]), nthr = atoi(argv[2]);
    std::vector<int> R;
    for (int i = 3; i < argc; ++i) R.push_back(atoi(argv[i]));
    FftDesc d;
    d.L = L; d.nst = (int)R.size();
    int sz = L;
    for (int s = 0; s < d.nst; ++s) {
        d.R[s] = R[s]; d.span[s] = sz / R[s]; d.tw[s] = 2 * L / sz;
        const unsigned dv = (unsigned)d.span[s]; int l = 0;
        while ((1ull << l) < dv) ++l;
        d.mag[s] = (unsigned)(((1ull << 32) * ((1ull << l) - dv)) / dv + 1);
        d.sh1[s] = l < 1 ? l : 1; d.sh2[s] = l > 1 ? l - 1 : 0;
        sz /= R[s];
    }
    const long long n2 = 2LL * L; int shift = 0;
    while ((1LL << (2 * shift)) < n2) ++shift;
    const int B = 1 << shift;
    d.shift = shift; d.nlo = B; d.nhi = (int)((n2 + B - 1) / B);
    std::vector<double2> hi(d.nhi), lo(d.nlo);
    for (int h = 0; h < d.nhi; ++h) root((long long)h * B, n2, hi[h].x, hi[h].y);
    for (int l = 0; l < d.nlo; ++l) root(l, n2, lo[l].x, lo[l].y);
    double2 *dh, *dl, *out; long long* cyc;
    cudaMalloc(&dh, 16 * d.nhi); cudaMalloc(&dl, 16 * d.nlo);
    cudaMemcpy(dh, hi.data(), 16 * d.nhi, cudaMemcpyHostToDevice);
    cudaMemcpy(dl, lo.data(), 16 * d.nlo, cudaMemcpyHostToDevice);
    d.hi = dh; d.lo = dl; d.rev = nullptr;
    const int nsm = 148;
    cudaMalloc(&cyc, 8 * nsm); cudaMalloc(&out, 16 * nsm);
    size_t smem = 200 * 1024;  // one CTA per SM
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 20;
    bench<<<nsm, nthr, smem>>>(d, 2, cyc, out);
    bench<<<nsm, nthr, smem>>>(d, reps, cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<long long> c(nsm);
    cudaMemcpy(c.data(), cyc, 8 * nsm, cudaMemcpyDeviceToHost);
    double m = 0; for (auto v : c) m += v; m /= nsm;
    const double per = m / reps / 2;  // cycles per transform
    // DP-op estimate per element handled by the caller
    printf("L=%d nthr=%d plan=", L, nthr);
    for (int r : R) printf("%d ", r);
    printf(" cycles/transform=%.0f  cycles/element=%.3f\n", per, per / L);
    return 0;
}
