// Shared helpers for the Pier sm_100a kernels: error plumbing, per-op IEEE
// rounding (no FMA contraction, so results match NumPy's one-rounding-per-ufunc
// evaluation bit for bit), 128-bit streaming vector access and launch sizing.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/pier_b200.h"

namespace pier {

// ---- error plumbing (capi.cpp owns the thread-local message) -------------
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

#define PIER_CHECK_CUDA(expr)                                   \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return ::pier::cuda_status(_e, #expr); \
    } while (0)

void count_launch();  // process-wide kernel launch counter (pier_launch_count)

#define PIER_LAUNCH_CHECK(what)          \
    do {                                 \
        ::pier::count_launch();          \
        PIER_CHECK_CUDA(cudaGetLastError()); \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // cached multiprocessor count of the current device

// ---- correctly rounded scalar ops, one rounding each -----------------------
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

// ---- 128-bit vectors ---------------------------------------------------------
template <typename T> struct V16;
template <> struct V16<float> {
    using type = float4;
    static constexpr int W = 4;
};
template <> struct V16<double> {
    using type = double2;
    static constexpr int W = 2;
};

__device__ __forceinline__ float& lane(float4& v, int i) { return (&v.x)[i]; }
__device__ __forceinline__ double& lane(double2& v, int i) { return (&v.x)[i]; }

// streaming (evict-first) loads/stores: every byte is touched exactly once
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, const float4& v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, const double2& v) { __stcs(p, v); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Launch geometry for streaming kernels: 256 threads, UNROLL vectors per
// thread per tile, grid = min(tiles, resident CTAs on all SMs) with a
// grid-stride loop over tiles.
constexpr int kThreads = 256;
int& default_ctas_per_sm();  // 8 unless a pipelined caller shares the GPU (pier_round_p2p)

inline int stream_grid(int64_t nvec, int unroll, int ctas_per_sm = 0) {
    if (ctas_per_sm <= 0) ctas_per_sm = default_ctas_per_sm();
    int64_t tiles = (nvec + (int64_t)kThreads * unroll - 1) / ((int64_t)kThreads * unroll);
    int64_t cap = (int64_t)sm_count() * ctas_per_sm;
    if (tiles < 1) tiles = 1;
    return (int)(tiles < cap ? tiles : cap);
}

}  // namespace pier
