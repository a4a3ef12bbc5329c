// K5-shaped HBM probe (one GPU): does the 11-stream shape of k_adamw_outer
// (read theta,g,m,v,anchor,mom; write theta,m,v,anchor,mom) lose bandwidth
// to the number of concurrent streams, and would interleaving the optimizer
// state (m|v, anchor|mom) or 256-bit accesses recover it?  Same element math
// as K5 (pier_adamw.cuh), -fmad=false like the product.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -I paper_2511_17849_b200/csrc -I include tools/stream_probe.cu -o tools/stream_probe
//   ./tools/stream_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#include "pier_adamw.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

using namespace pier;

__device__ __forceinline__ void step4(float4& a, float4 b, float4& mm, float4& vv, float4& an, float4& mo,
                                      const AdamC<float>& c, float lr, float mu) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        float t = lane(a, w);
        adamw_lane<float>(t, lane(b, w), lane(mm, w), lane(vv, w), c);
        float dl = sub_rn(t, lane(an, w));
        float m2 = add_rn(mul_rn(mu, lane(mo, w)), dl);
        float up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));
        t = add_rn(t, sub_rn(up, dl));
        lane(mo, w) = m2;
        lane(a, w) = t;
        lane(an, w) = t;
    }
}

// V0: six separate arrays (the product layout)
template <int U>
__global__ void __launch_bounds__(256) k_sep(float4* th, const float4* g, float4* m, float4* v, float4* an,
                                             float4* mo, int64_t nv, AdamC<float> c, float lr, float mu) {
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < nv; i0 += (int64_t)gridDim.x * 256 * U) {
        float4 a[U], b[U], mm[U], vv[U], aa[U], oo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) {
                a[k] = __ldcs(th + i); b[k] = __ldcs(g + i); mm[k] = __ldcs(m + i); vv[k] = __ldcs(v + i);
                aa[k] = __ldcs(an + i); oo[k] = __ldcs(mo + i);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) {
                step4(a[k], b[k], mm[k], vv[k], aa[k], oo[k], c, lr, mu);
                __stcs(th + i, a[k]); __stcs(m + i, mm[k]); __stcs(v + i, vv[k]);
                __stcs(an + i, aa[k]); __stcs(mo + i, oo[k]);
            }
        }
    }
}

// V1: m|v and anchor|mom interleaved per float4 (pairs of 16 B)
template <int U>
__global__ void __launch_bounds__(256) k_pair(float4* th, const float4* g, float4* mv, float4* am, int64_t nv,
                                              AdamC<float> c, float lr, float mu) {
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < nv; i0 += (int64_t)gridDim.x * 256 * U) {
        float4 a[U], b[U], mm[U], vv[U], aa[U], oo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) {
                a[k] = __ldcs(th + i); b[k] = __ldcs(g + i);
                mm[k] = __ldcs(mv + 2 * i); vv[k] = __ldcs(mv + 2 * i + 1);
                aa[k] = __ldcs(am + 2 * i); oo[k] = __ldcs(am + 2 * i + 1);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) {
                step4(a[k], b[k], mm[k], vv[k], aa[k], oo[k], c, lr, mu);
                __stcs(th + i, a[k]);
                __stcs(mv + 2 * i, mm[k]); __stcs(mv + 2 * i + 1, vv[k]);
                __stcs(am + 2 * i, aa[k]); __stcs(am + 2 * i + 1, oo[k]);
            }
        }
    }
}

// 256-bit global accesses (ld/st.global.v8.f32, sm_100+)
struct F8 { float4 lo, hi; };
__device__ __forceinline__ F8 ld8(const float4* p) {
    F8 r;
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y), "=f"(r.hi.z),
                   "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float4* p, const F8& r) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.lo.x), "f"(r.lo.y),
                 "f"(r.lo.z), "f"(r.lo.w), "f"(r.hi.x), "f"(r.hi.y), "f"(r.hi.z), "f"(r.hi.w)
                 : "memory");
}

// V2: six separate arrays, 256-bit accesses (two float4 per thread per array)
template <int U>
__global__ void __launch_bounds__(256) k_sep8(float4* th, const float4* g, float4* m, float4* v, float4* an,
                                              float4* mo, int64_t nv, AdamC<float> c, float lr, float mu) {
    const int64_t n8 = nv / 2;
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n8; i0 += (int64_t)gridDim.x * 256 * U) {
        F8 a[U], b[U], mm[U], vv[U], aa[U], oo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
                a[k] = ld8(th + i); b[k] = ld8(g + i); mm[k] = ld8(m + i); vv[k] = ld8(v + i);
                aa[k] = ld8(an + i); oo[k] = ld8(mo + i);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
                step4(a[k].lo, b[k].lo, mm[k].lo, vv[k].lo, aa[k].lo, oo[k].lo, c, lr, mu);
                step4(a[k].hi, b[k].hi, mm[k].hi, vv[k].hi, aa[k].hi, oo[k].hi, c, lr, mu);
                st8(th + i, a[k]); st8(m + i, mm[k]); st8(v + i, vv[k]); st8(an + i, aa[k]); st8(mo + i, oo[k]);
            }
        }
    }
}

// control: K4b shape (read theta,g,m,v; write theta,m,v)
template <int U>
__global__ void __launch_bounds__(256) k_adam(float4* th, const float4* g, float4* m, float4* v, int64_t nv,
                                              AdamC<float> c) {
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < nv; i0 += (int64_t)gridDim.x * 256 * U) {
        float4 a[U], b[U], mm[U], vv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) { a[k] = __ldcs(th + i); b[k] = __ldcs(g + i); mm[k] = __ldcs(m + i); vv[k] = __ldcs(v + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + k * 256;
            if (i < nv) {
#pragma unroll
                for (int w = 0; w < 4; ++w) adamw_lane<float>(lane(a[k], w), lane(b[k], w), lane(mm[k], w), lane(vv[k], w), c);
                __stcs(th + i, a[k]); __stcs(m + i, mm[k]); __stcs(v + i, vv[k]);
            }
        }
    }
}

int main() {
    const int64_t n = 1557611200;  // GPT-2 XL-shaped flat set
    const int64_t nv = n / 4;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float4 *th, *g, *m, *v, *an, *mo, *mv, *am;
    CK(cudaMalloc(&th, n * 4)); CK(cudaMalloc(&g, n * 4)); CK(cudaMalloc(&m, n * 4)); CK(cudaMalloc(&v, n * 4));
    CK(cudaMalloc(&an, n * 4)); CK(cudaMalloc(&mo, n * 4)); CK(cudaMalloc(&mv, n * 8)); CK(cudaMalloc(&am, n * 8));
    CK(cudaMemset(th, 0, n * 4)); CK(cudaMemset(g, 0, n * 4)); CK(cudaMemset(m, 0, n * 4)); CK(cudaMemset(v, 0, n * 4));
    CK(cudaMemset(an, 0, n * 4)); CK(cudaMemset(mo, 0, n * 4)); CK(cudaMemset(mv, 0, n * 8)); CK(cudaMemset(am, 0, n * 8));
    PierAdamW h{1e-4, 0.9, 0.95, 1e-8, 0.1, 100};
    AdamC<float> c = adam_consts<float>(h);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](const char* name, int U, int per_sm, double bytes_per_param, auto launch) {
        int grid = per_sm * sms;
        for (int w = 0; w < 3; ++w) launch(grid);
        cudaEventRecord(e0);
        const int reps = 10;
        for (int r = 0; r < reps; ++r) launch(grid);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        cudaError_t err = cudaGetLastError();
        printf("{\"kernel\": \"%s\", \"U\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"tbs\": %.4f, \"err\": \"%s\"}\n", name,
               U, per_sm, ms, bytes_per_param * n / ms / 1e9, cudaGetErrorString(err));
        fflush(stdout);
    };
    for (int per_sm : {4, 8, 16}) {
        timeit("adamw_4in3out", 4, per_sm, 28, [&](int gr) { k_adam<4><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("k5_sep", 1, per_sm, 44, [&](int gr) { k_sep<1><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_sep", 2, per_sm, 44, [&](int gr) { k_sep<2><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_sep", 4, per_sm, 44, [&](int gr) { k_sep<4><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_pair", 1, per_sm, 44, [&](int gr) { k_pair<1><<<gr, 256>>>(th, g, mv, am, nv, c, 1.1f, 0.9f); });
        timeit("k5_pair", 2, per_sm, 44, [&](int gr) { k_pair<2><<<gr, 256>>>(th, g, mv, am, nv, c, 1.1f, 0.9f); });
        timeit("k5_sep8", 1, per_sm, 44, [&](int gr) { k_sep8<1><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_sep8", 2, per_sm, 44, [&](int gr) { k_sep8<2><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
    }
    return 0;
}
