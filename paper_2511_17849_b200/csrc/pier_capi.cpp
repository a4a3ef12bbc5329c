// C-ABI plumbing: thread-local error messages, device queries and the exact
// host-side outer schedule (optim.py:162-219) for C/C++ callers.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <string>

#include "../../include/pier_b200.h"
#include "pier_comm_internal.h"

namespace pier {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int& default_ctas_per_sm() {
    static thread_local int v = 0;  // 0: one tile per CTA (uncapped grid)
    return v;
}

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    // a trapped persistent round leaves a record of the wait that timed out
    return set_error(PIER_ECUDA, std::string(what) + ": " + cudaGetErrorString(e) + round_diag_text());
}

int sm_count() {
    static thread_local int cached_dev = -1;
    static thread_local int cached = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cached;
    if (dev != cached_dev) {
        int c = 0;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && c > 0) cached = c;
        cached_dev = dev;
    }
    return cached;
}

// optim.py:162-163 -- int(math.floor(frac * total)) in binary64
static int64_t floor_frac(double frac, int64_t total) { return (int64_t)std::floor(frac * (double)total); }

}  // namespace pier

extern "C" {

const char* pier_last_error(void) { return pier::g_last_error.c_str(); }

int pier_version(void) { return 100; }  // 0.1.0

unsigned long long pier_launch_count(void) { return pier::g_launches.load(std::memory_order_relaxed); }

int pier_device_sync(void) {
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? PIER_OK : pier::cuda_status(e, "cudaDeviceSynchronize");
}

int pier_device_sm_count(int device) {
    int c = 0;
    if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return c;
}

// optim.py:205-219
double pier_momentum_mu(int64_t t, int64_t T) {
    using pier::floor_frac;
    if (t < 0) return -1.0;
    if (t < floor_frac(0.1, T)) return 0.9;
    if (t < floor_frac(0.15, T)) return 0.99;
    if (t < floor_frac(0.2, T)) return 0.95;
    return 0.9;
}

// optim.py:181-202
int pier_outer_lr(int64_t t, int64_t T, double* out) {
    using pier::floor_frac;
    int64_t a = floor_frac(0.1, T), b = floor_frac(0.2, T), c = floor_frac(0.8, T);
    if (!out) return pier::set_error(PIER_EINVAL, "outer_lr: null out");
    if (t < a) return pier::set_error(PIER_EINVAL, "outer_lr is undefined before the ramp start");
    if (t > T) return pier::set_error(PIER_EINVAL, "outer_lr is undefined past total_iters");
    if (t < b) *out = (double)(t - a) / (double)(b - a);
    else *out = t < c ? 1.1 : 0.9;
    return PIER_OK;
}

}  // extern "C"
