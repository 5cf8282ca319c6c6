// ORACLE / TEST INFRASTRUCTURE ONLY — FFTW-API shim over skfft (see fftw3.h).
// Transform tables are cached per (n, sign) so that the reference's
// plan-per-call pattern (fourier.cpp:22-35) does not pay for twiddle set-up on
// every 1D transform, much like FFTW's own ESTIMATE planner + twiddle cache.
#include "fftw3.h"

#include <map>
#include <mutex>
#include <utility>

#include "../skfft.h"

struct fftw_plan_s {
    const skfft_plan* tr;
    double* in;
    double* out;
};

namespace {
std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
std::map<std::pair<int, int>, skfft_plan*>& cache() {
    static std::map<std::pair<int, int>, skfft_plan*> c;
    return c;
}
}  // namespace

extern "C" fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned) {
    const skfft_plan* tr;
    {
        std::lock_guard<std::mutex> lock(cache_mutex());
        auto& c = cache();
        auto key = std::make_pair(n, sign < 0 ? -1 : 1);
        auto it = c.find(key);
        if (it == c.end()) it = c.emplace(key, skfft_plan_create(n, key.second)).first;
        tr = it->second;
    }
    return new fftw_plan_s{tr, reinterpret_cast<double*>(in), reinterpret_cast<double*>(out)};
}

extern "C" void fftw_execute(const fftw_plan p) { skfft_execute(p->tr, p->in, p->out); }

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
