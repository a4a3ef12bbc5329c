// Shared helpers for the Pier sm_100a kernels: error plumbing, per-op IEEE
// rounding (no FMA contraction, so results match NumPy's one-rounding-per-ufunc
// evaluation bit for bit), 128/256-bit streaming vector access and launch sizing.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>
#include <initializer_list>
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

// ---- 256-bit vectors (sm_100: LDG/STG.E.ENL2.256) -------------------------
// Two 128-bit halves; 256-bit accesses reach ~6.9 TB/s where 128-bit ones
// top out near 6.6 on the same kernels (tools/stream_probe.cu).
struct F8 { float4 lo, hi; };
struct D4 { double2 lo, hi; };
template <typename T> struct V32;
template <> struct V32<float> {
    using type = F8;
    static constexpr int W = 8;
};
template <> struct V32<double> {
    using type = D4;
    static constexpr int W = 4;
};

__device__ __forceinline__ float& lane(F8& v, int i) { return i < 4 ? lane(v.lo, i) : lane(v.hi, i - 4); }
__device__ __forceinline__ double& lane(D4& v, int i) { return i < 2 ? lane(v.lo, i) : lane(v.hi, i - 2); }

__device__ __forceinline__ F8 ld_stream(const F8* p) {
    F8 r;
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y),
                   "=f"(r.hi.z), "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ D4 ld_stream(const D4* p) {
    D4 r;
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.lo.x), "=d"(r.lo.y), "=d"(r.hi.x), "=d"(r.hi.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(F8* p, const F8& v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.lo.x), "f"(v.lo.y),
                 "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z), "f"(v.hi.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(D4* p, const D4& v) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.lo.x), "d"(v.lo.y), "d"(v.hi.x),
                 "d"(v.hi.y)
                 : "memory");
}
// write-back store (no evict-first hint): data a peer reads right after stays in L2
__device__ __forceinline__ void st_keep(F8* p, const F8& v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.lo.x), "f"(v.lo.y),
                 "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z), "f"(v.hi.w)
                 : "memory");
}

// write-back store with an L2 evict-last policy (createpolicy.fractional)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_keep_l2(F8* p, const F8& v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p), "f"(v.lo.x),
                 "f"(v.lo.y), "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z), "f"(v.hi.w), "l"(pol)
                 : "memory");
}

// L2-coherent (.cg) access for buffers other GPUs read or write over NVLink
__device__ __forceinline__ float4 ld_cg(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg(float4* p, const float4& v) { __stcg(p, v); }
__device__ __forceinline__ F8 ld_cg(const F8* p) {
    F8 r;
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y),
                   "=f"(r.hi.z), "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_cg(F8* p, const F8& v) {
    asm volatile("st.global.cg.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v.lo.x), "f"(v.lo.y),
                 "f"(v.lo.z), "f"(v.lo.w), "f"(v.hi.x), "f"(v.hi.y), "f"(v.hi.z), "f"(v.hi.w)
                 : "memory");
}
__device__ __forceinline__ void st_keep(float4* p, const float4& v) { *p = v; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

// widest vector every pointer allows: 32, 16 or 0 (scalar) bytes
inline int common_align(std::initializer_list<const void*> ps) {
    bool a32 = true, a16 = true;
    for (const void* p : ps) {
        a32 = a32 && aligned32(p);
        a16 = a16 && aligned16(p);
    }
    return a32 ? 32 : a16 ? 16 : 0;
}

// Launch geometry for streaming kernels: 256 threads, UNROLL vectors per
// thread per tile.  Default: one tile per CTA (the hardware scheduler keeps
// every SM full and there is no tail of long-running CTAs -- measured faster
// than a resident grid striding over the buffer, tools/stream_probe.cu);
// a positive ctas_per_sm caps the grid at that many CTAs per SM with a
// grid-stride loop (callers that share the GPU with a concurrent kernel).
constexpr int kThreads = 256;
int& default_ctas_per_sm();  // 0 = uncapped unless a pipelined caller shares the GPU (pier_round_p2p)

inline int stream_grid(int64_t nvec, int unroll, int ctas_per_sm = 0) {
    if (ctas_per_sm <= 0) ctas_per_sm = default_ctas_per_sm();
    int64_t tiles = (nvec + (int64_t)kThreads * unroll - 1) / ((int64_t)kThreads * unroll);
    if (tiles < 1) tiles = 1;
    int64_t cap = ctas_per_sm > 0 ? (int64_t)sm_count() * ctas_per_sm : (int64_t)0x7fffffff;
    return (int)(tiles < cap ? tiles : cap);
}

}  // namespace pier
