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
#include <cstdlib>

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

// 256-bit with streaming (evict-first) cache hints
__device__ __forceinline__ F8 ld8cs(const float4* p) {
    F8 r;
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x), "=f"(r.hi.y), "=f"(r.hi.z),
                   "=f"(r.hi.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8cs(float4* p, const F8& r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.lo.x), "f"(r.lo.y),
                 "f"(r.lo.z), "f"(r.lo.w), "f"(r.hi.x), "f"(r.hi.y), "f"(r.hi.z), "f"(r.hi.w)
                 : "memory");
}

template <int U, bool CS>
__global__ void __launch_bounds__(256) k_sep8h(float4* th, const float4* g, float4* m, float4* v, float4* an,
                                               float4* mo, int64_t nv, AdamC<float> c, float lr, float mu) {
    const int64_t n8 = nv / 2;
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n8; i0 += (int64_t)gridDim.x * 256 * U) {
        F8 a[U], b[U], mm[U], vv[U], aa[U], oo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
                if (CS) { a[k] = ld8cs(th + i); b[k] = ld8cs(g + i); mm[k] = ld8cs(m + i); vv[k] = ld8cs(v + i);
                          aa[k] = ld8cs(an + i); oo[k] = ld8cs(mo + i); }
                else { a[k] = ld8(th + i); b[k] = ld8(g + i); mm[k] = ld8(m + i); vv[k] = ld8(v + i);
                       aa[k] = ld8(an + i); oo[k] = ld8(mo + i); }
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
                step4(a[k].lo, b[k].lo, mm[k].lo, vv[k].lo, aa[k].lo, oo[k].lo, c, lr, mu);
                step4(a[k].hi, b[k].hi, mm[k].hi, vv[k].hi, aa[k].hi, oo[k].hi, c, lr, mu);
                if (CS) { st8cs(th + i, a[k]); st8cs(m + i, mm[k]); st8cs(v + i, vv[k]); st8cs(an + i, aa[k]);
                          st8cs(mo + i, oo[k]); }
                else { st8(th + i, a[k]); st8(m + i, mm[k]); st8(v + i, vv[k]); st8(an + i, aa[k]); st8(mo + i, oo[k]); }
            }
        }
    }
}

template <int U, bool CS>
__global__ void __launch_bounds__(256) k_adam8(float4* th, const float4* g, float4* m, float4* v, int64_t nv,
                                               AdamC<float> c) {
    const int64_t n8 = nv / 2;
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n8; i0 += (int64_t)gridDim.x * 256 * U) {
        F8 a[U], b[U], mm[U], vv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
                if (CS) { a[k] = ld8cs(th + i); b[k] = ld8cs(g + i); mm[k] = ld8cs(m + i); vv[k] = ld8cs(v + i); }
                else { a[k] = ld8(th + i); b[k] = ld8(g + i); mm[k] = ld8(m + i); vv[k] = ld8(v + i); }
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = 2 * (i0 + k * 256);
            if (i0 + k * 256 < n8) {
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    adamw_lane<float>(lane(a[k].lo, w), lane(b[k].lo, w), lane(mm[k].lo, w), lane(vv[k].lo, w), c);
                    adamw_lane<float>(lane(a[k].hi, w), lane(b[k].hi, w), lane(mm[k].hi, w), lane(vv[k].hi, w), c);
                }
                if (CS) { st8cs(th + i, a[k]); st8cs(m + i, mm[k]); st8cs(v + i, vv[k]); }
                else { st8(th + i, a[k]); st8(m + i, mm[k]); st8(v + i, vv[k]); }
            }
        }
    }
}

// plain copies: the MEASURED_PEAKS denominator vs 256-bit accesses
template <int U>
__global__ void __launch_bounds__(256) k_copy4(const float4* src, float4* dst, int64_t nv) {
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < nv; i0 += (int64_t)gridDim.x * 256 * U) {
        float4 a[U];
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * 256 < nv) a[k] = __ldcs(src + i0 + k * 256);
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * 256 < nv) __stcs(dst + i0 + k * 256, a[k]);
    }
}
template <int U>
__global__ void __launch_bounds__(256) k_copy8(const float4* src, float4* dst, int64_t nv) {
    const int64_t n8 = nv / 2;
    for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n8; i0 += (int64_t)gridDim.x * 256 * U) {
        F8 a[U];
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * 256 < n8) a[k] = ld8cs(src + 2 * (i0 + k * 256));
#pragma unroll
        for (int k = 0; k < U; ++k) if (i0 + k * 256 < n8) st8cs(dst + 2 * (i0 + k * 256), a[k]);
    }
}

// AdamW with dynamically claimed tiles (atomic counter): does in-order claiming
// recover the one-tile-per-CTA bandwidth inside a persistent grid?
template <int U, int CHUNK>
__global__ void __launch_bounds__(256) k_adam8_dyn(float4* th, const float4* g, float4* m, float4* v, int64_t nv,
                                                   AdamC<float> c, unsigned long long* counter) {
    const int64_t n8 = nv / 2;
    const int64_t tile = 256 * U;
    const int64_t ntiles = (n8 + tile - 1) / tile;
    __shared__ long long s_next;
    for (;;) {
        if (threadIdx.x == 0) s_next = (long long)atomicAdd(counter, (unsigned long long)CHUNK);
        __syncthreads();
        const int64_t first = s_next;
        __syncthreads();
        if (first >= ntiles) break;
        for (int64_t tix = first; tix < first + CHUNK && tix < ntiles; ++tix) {
            const int64_t i0 = tix * tile + threadIdx.x;
            F8 a[U], b[U], mm[U], vv[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = 2 * (i0 + k * 256);
                if (i0 + k * 256 < n8) { a[k] = ld8cs(th + i); b[k] = ld8cs(g + i); mm[k] = ld8cs(m + i); vv[k] = ld8cs(v + i); }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = 2 * (i0 + k * 256);
                if (i0 + k * 256 < n8) {
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        adamw_lane<float>(lane(a[k].lo, w), lane(b[k].lo, w), lane(mm[k].lo, w), lane(vv[k].lo, w), c);
                        adamw_lane<float>(lane(a[k].hi, w), lane(b[k].hi, w), lane(mm[k].hi, w), lane(vv[k].hi, w), c);
                    }
                    st8cs(th + i, a[k]); st8cs(m + i, mm[k]); st8cs(v + i, vv[k]);
                }
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

// realistic magnitudes: the IEEE div/sqrt intrinsics take slow paths on zeros
__global__ void k_fill(float* p, int64_t n, uint32_t seed, float scale, float bias) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
        p[i] = bias + scale * ((float)(h & 0xffffff) / 16777216.0f - 0.5f);
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
    k_fill<<<4 * sms, 256>>>((float*)th, n, 1, 0.2f, 0.f);
    k_fill<<<4 * sms, 256>>>((float*)g, n, 2, 0.02f, 0.f);
    k_fill<<<4 * sms, 256>>>((float*)m, n, 3, 0.002f, 0.f);
    k_fill<<<4 * sms, 256>>>((float*)v, n, 4, 1e-5f, 1e-5f);
    k_fill<<<4 * sms, 256>>>((float*)an, n, 5, 0.2f, 0.f);
    k_fill<<<4 * sms, 256>>>((float*)mo, n, 6, 0.01f, 0.f);
    k_fill<<<4 * sms, 256>>>((float*)mv, 2 * n, 7, 1e-5f, 1e-5f);
    k_fill<<<4 * sms, 256>>>((float*)am, 2 * n, 8, 0.2f, 0.f);
    CK(cudaDeviceSynchronize());
    PierAdamW h{1e-4, 0.9, 0.95, 1e-8, 0.1, 100};
    AdamC<float> c = adam_consts<float>(h);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](const char* name, int U, int per_sm, double bytes_per_param, auto launch) {
        // per_sm <= 0: one tile per CTA (no grid-stride loop)
        int64_t tiles = n / 8 / (256 * U);
        int grid = per_sm > 0 ? per_sm * sms : (int)tiles;
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
    const char* which = getenv("PROBE");
    if (which && which[0] == '3') {
        unsigned long long* ctr;
        CK(cudaMalloc(&ctr, 8));
        for (int per_sm : {2, 3, 4, 8}) {
            timeit("adamw_v8_stride", 2, per_sm, 28, [&](int gr) { k_adam8<2, true><<<gr, 256>>>(th, g, m, v, nv, c); });
            timeit("adamw_v8_stride", 1, per_sm, 28, [&](int gr) { k_adam8<1, true><<<gr, 256>>>(th, g, m, v, nv, c); });
            timeit("adamw_v8_dyn1", 2, per_sm, 28, [&](int gr) { cudaMemsetAsync(ctr, 0, 8); k_adam8_dyn<2, 1><<<gr, 256>>>(th, g, m, v, nv, c, ctr); });
            timeit("adamw_v8_dyn1", 1, per_sm, 28, [&](int gr) { cudaMemsetAsync(ctr, 0, 8); k_adam8_dyn<1, 1><<<gr, 256>>>(th, g, m, v, nv, c, ctr); });
            timeit("adamw_v8_dyn4", 2, per_sm, 28, [&](int gr) { cudaMemsetAsync(ctr, 0, 8); k_adam8_dyn<2, 4><<<gr, 256>>>(th, g, m, v, nv, c, ctr); });
            timeit("adamw_v8_dyn16", 2, per_sm, 28, [&](int gr) { cudaMemsetAsync(ctr, 0, 8); k_adam8_dyn<2, 16><<<gr, 256>>>(th, g, m, v, nv, c, ctr); });
        }
        timeit("adamw_v8_tiles", 1, 0, 28, [&](int gr) { k_adam8<1, true><<<gr, 256>>>(th, g, m, v, nv, c); });
        return 0;
    }
    if (which && which[0] == '2') {
        for (int per_sm : {32, 64, 128, 256, 0}) {
            timeit("copy_v8", 2, per_sm, 8, [&](int gr) { k_copy8<2><<<gr, 256>>>(th, mv, nv); });
            timeit("adamw_v8", 1, per_sm, 28, [&](int gr) { k_adam8<1, true><<<gr, 256>>>(th, g, m, v, nv, c); });
            timeit("adamw_v8", 2, per_sm, 28, [&](int gr) { k_adam8<2, true><<<gr, 256>>>(th, g, m, v, nv, c); });
            timeit("k5_v8", 1, per_sm, 44, [&](int gr) { k_sep8h<1, true><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
            timeit("k5_v8", 2, per_sm, 44, [&](int gr) { k_sep8h<2, true><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
            timeit("k5_v4", 2, per_sm, 44, [&](int gr) { k_sep<2><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        }
        return 0;
    }
    for (int per_sm : {8, 16, 32, 64}) {
        timeit("copy_v4", 4, per_sm, 8, [&](int gr) { k_copy4<4><<<gr, 256>>>(th, mv, nv); });
        timeit("copy_v8", 2, per_sm, 8, [&](int gr) { k_copy8<2><<<gr, 256>>>(th, mv, nv); });
        timeit("adamw_v4", 4, per_sm, 28, [&](int gr) { k_adam<4><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("adamw_v8_na", 1, per_sm, 28, [&](int gr) { k_adam8<1, false><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("adamw_v8_na", 2, per_sm, 28, [&](int gr) { k_adam8<2, false><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("adamw_v8_cs", 1, per_sm, 28, [&](int gr) { k_adam8<1, true><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("adamw_v8_cs", 2, per_sm, 28, [&](int gr) { k_adam8<2, true><<<gr, 256>>>(th, g, m, v, nv, c); });
        timeit("k5_v4", 2, per_sm, 44, [&](int gr) { k_sep<2><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_v8_na", 1, per_sm, 44, [&](int gr) { k_sep8h<1, false><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_v8_na", 2, per_sm, 44, [&](int gr) { k_sep8h<2, false><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_v8_cs", 1, per_sm, 44, [&](int gr) { k_sep8h<1, true><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
        timeit("k5_v8_cs", 2, per_sm, 44, [&](int gr) { k_sep8h<2, true><<<gr, 256>>>(th, g, m, v, an, mo, nv, c, 1.1f, 0.9f); });
    }
    return 0;
}
