// Pier hot-path kernels for sm_100a: pseudo-gradient (K1), fused outer update
// (K3), warmup fold (K3b), gradient norm + clip scale (K4a), fused AdamW (K4b,
// flat / bf16-master / multi-tensor) and the virtual-group left-fold mean (K6).
//
// All of these are elementwise or reductions over flat parameter buffers and
// therefore HBM-bound: no tensor cores, no shared-memory staging (nothing is
// reused), just coalesced 256-bit (32-byte aligned buffers) or 128-bit
// streaming loads/stores with one or more vectors in flight per thread per
// array, one tile per CTA (pier_common.cuh: stream_grid).
//
// Rounding: one IEEE rounding per reference NumPy ufunc, in the reference's
// order (see pier_common.cuh), so f32 results are bitwise equal to the
// reference's float32 arithmetic.  Built with -fmad=false as a second guard.
#include "pier_adamw.cuh"
#include "pier_common.cuh"

#include <cmath>
#include <vector>

namespace pier {

// ===========================================================================
// generic streaming skeleton
// ===========================================================================
// Each CTA owns tiles of kThreads*U vectors; thread t handles vectors
// base + t + k*kThreads (k < U), so each of the U loads is a fully coalesced
// 4 KB (f32x4) warp-row and all U loads are issued before any use.

template <int U, typename F>
__device__ __forceinline__ void for_tiles(int64_t nvec, F&& f) {
    const int64_t tile = (int64_t)kThreads * U;
    for (int64_t base = (int64_t)blockIdx.x * tile; base < nvec; base += (int64_t)gridDim.x * tile)
        f(base + threadIdx.x);
}

// element w of a 256/128-bit vector, or the value itself when the kernel is
// instantiated on scalars (tails and unaligned buffers)
template <typename VT, typename T>
__device__ __forceinline__ T& L(VT& v, int i) {
    if constexpr (sizeof(VT) == sizeof(T)) return v;
    else return lane(v, i);
}

template <typename VT> __device__ __forceinline__ VT ldv(const VT* p) { return __ldcs(p); }
template <typename VT> __device__ __forceinline__ void stv(VT* p, const VT& v) { __stcs(p, v); }
__device__ __forceinline__ F8 ldv(const F8* p) { return ld_stream(p); }
__device__ __forceinline__ D4 ldv(const D4* p) { return ld_stream(p); }
__device__ __forceinline__ void stv(F8* p, const F8& v) { st_stream(p, v); }
__device__ __forceinline__ void stv(D4* p, const D4& v) { st_stream(p, v); }

// ===========================================================================
// K1 pseudo-gradient: delta = theta - anchor   (driver.py:415, :434)
// ===========================================================================
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_pseudograd(const VT* __restrict__ th,
                                                          const VT* __restrict__ an,
                                                          VT* __restrict__ out, int64_t nvec) {
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { a[k] = ldv(th + i); b[k] = ldv(an + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) L<VT, T>(a[k], w) = sub_rn(L<VT, T>(a[k], w), L<VT, T>(b[k], w));
                stv(out + i, a[k]);
            }
        }
    });
}

// ===========================================================================
// a1 fold / a2 outer_step (pure forms, optim.py:243-276)
// ===========================================================================
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_fold(const VT* __restrict__ mom, const VT* __restrict__ d,
                                                    VT* __restrict__ out, int64_t nvec, T mu) {
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { a[k] = ldv(mom + i); b[k] = ldv(d + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    L<VT, T>(a[k], w) = add_rn(mul_rn(mu, L<VT, T>(a[k], w)), L<VT, T>(b[k], w));
                stv(out + i, a[k]);
            }
        }
    });
}

template <typename T, typename VT, int U, bool kAnchor>
__global__ void __launch_bounds__(kThreads) k_outer_pure(const VT* __restrict__ mom, const VT* __restrict__ base,
                                                          const VT* __restrict__ d, VT* __restrict__ th_out,
                                                          VT* __restrict__ mom_out, int64_t nvec, T lr, T mu) {
    // base = anchor (kAnchor) or snapshot
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT m[U], b[U], dd[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { m[k] = ldv(mom + i); b[k] = ldv(base + i); dd[k] = ldv(d + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    T dl = L<VT, T>(dd[k], w);
                    T m2 = add_rn(mul_rn(mu, L<VT, T>(m[k], w)), dl);        // optim.py:270
                    T up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));           // optim.py:271
                    T bs = L<VT, T>(b[k], w);
                    L<VT, T>(b[k], w) = kAnchor ? add_rn(bs, sub_rn(up, dl))  // optim.py:275
                                                : add_rn(bs, up);             // optim.py:273
                    L<VT, T>(m[k], w) = m2;
                }
                stv(th_out + i, b[k]);
                stv(mom_out + i, m[k]);
            }
        }
    });
}

// ===========================================================================
// K3 fused outer update (driver.py:428-440 after the mean) -- one HBM pass
// reads avg(or sum), anchor, mom; writes mom, anchor, theta  (24 B/param f32)
// ===========================================================================
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_outer_update(const VT* avg, VT* __restrict__ anchor,
                                                            VT* __restrict__ mom, VT* th_out, int64_t nvec,
                                                            T lr, T mu, T divisor, int do_div) {
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U], an[U], m[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { a[k] = ldv(avg + i); an[k] = ldv(anchor + i); m[k] = ldv(mom + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    T av = L<VT, T>(a[k], w);
                    if (do_div) av = div_rn(av, divisor);                    // topology.py:121
                    T dl = sub_rn(av, L<VT, T>(an[k], w));                   // driver.py:434
                    T m2 = add_rn(mul_rn(mu, L<VT, T>(m[k], w)), dl);        // optim.py:270
                    T up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));           // optim.py:271
                    T th = add_rn(av, sub_rn(up, dl));                       // optim.py:275
                    L<VT, T>(m[k], w) = m2;
                    L<VT, T>(an[k], w) = th;                                 // driver.py:438
                }
                stv(mom + i, m[k]);
                stv(anchor + i, an[k]);
                stv(th_out + i, an[k]);                                      // driver.py:439-440
            }
        }
    });
}

// ===========================================================================
// K3b warmup fold (driver.py:412-420): mom = mu*mom + (theta-anchor); anchor=theta
// ===========================================================================
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_warmup_fold(const VT* __restrict__ th, VT* __restrict__ anchor,
                                                           VT* __restrict__ mom, int64_t nvec, T mu) {
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT t[U], an[U], m[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { t[k] = ldv(th + i); an[k] = ldv(anchor + i); m[k] = ldv(mom + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    T dl = sub_rn(L<VT, T>(t[k], w), L<VT, T>(an[k], w));       // driver.py:415
                    L<VT, T>(m[k], w) = add_rn(mul_rn(mu, L<VT, T>(m[k], w)), dl);  // optim.py:245
                }
                stv(mom + i, m[k]);
                stv(anchor + i, t[k]);                                        // driver.py:420
            }
        }
    });
}

// ===========================================================================
// K6 left-fold mean over replicas (topology.py:113-122)
// ===========================================================================
template <typename T> struct PartPtrs { const T* p[PIER_MAX_PARTS]; };

template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_mean_left_fold(PartPtrs<T> parts, int nparts, VT* out,
                                                              int64_t nvec, T nf) {
    constexpr int W = sizeof(VT) / sizeof(T);
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT acc[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) acc[k] = ldv(reinterpret_cast<const VT*>(parts.p[0]) + i);
        }
        for (int j = 1; j < nparts; ++j) {
            VT x[U];
            const VT* pj = reinterpret_cast<const VT*>(parts.p[j]);
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = i0 + (int64_t)k * kThreads;
                if (i < nvec) x[k] = ldv(pj + i);
            }
#pragma unroll
            for (int k = 0; k < U; ++k)
#pragma unroll
                for (int w = 0; w < W; ++w) L<VT, T>(acc[k], w) = add_rn(L<VT, T>(acc[k], w), L<VT, T>(x[k], w));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) L<VT, T>(acc[k], w) = div_rn(L<VT, T>(acc[k], w), nf);
                stv(out + i, acc[k]);
            }
        }
    });
}

// ===========================================================================
// K4a gradient square norm -> PierClip  (optim.py:70-79)
// ===========================================================================

// warp_sum / block_sum / clip_finalize / norm_sum_last / norm_epilogue live in
// pier_adamw.cuh (shared with the P2P gradient mean's fused norm)

// Recompute norm / scale from ws->res.sqnorm (after the partial square sums of
// the tensor-parallel shards of one replica were summed into it)
template <typename T>
__global__ void k_clip_finalize(NormWs* ws, double max_norm) {
    if (threadIdx.x == 0 && blockIdx.x == 0) clip_finalize<T>(ws, ws->res.sqnorm, max_norm);
}

template <typename T, typename VT, int U, typename LoadT = T>
__global__ void __launch_bounds__(kThreads) k_sqnorm(const VT* __restrict__ g, int64_t nvec, const LoadT* tail,
                                                      int64_t tail_n, NormWs* ws, double max_norm) {
    constexpr int W = sizeof(VT) / sizeof(T);
    double acc = 0.0;
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT x[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) x[k] = ldv(g + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec)
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    double v = (double)L<VT, T>(x[k], w);
                    acc += v * v;
                }
        }
    });
    if (blockIdx.x == 0)
        for (int64_t i = threadIdx.x; i < tail_n; i += kThreads) {
            double v = (double)tail[i];
            acc += v * v;
        }
    norm_epilogue<T>(ws, acc, max_norm);
}

// bf16 gradients: 8 per 16-byte vector
__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

// VT = uint4 (8 bf16 per 16-byte vector) or F8 (16 bf16 per 32-byte vector: the
// 256-bit accesses take the pass from 5.9 to the copy bandwidth)
__device__ __forceinline__ uint4 ld_bf16v(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ F8 ld_bf16v(const F8* p) { return ld_stream(p); }

template <typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_sqnorm_bf16(const VT* __restrict__ g, int64_t nvec,
                                                           const uint16_t* tail, int64_t tail_n, NormWs* ws,
                                                           double max_norm) {
    constexpr int NW = sizeof(VT) / 4;   // 32-bit words (2 bf16 each) per vector
    double acc = 0.0;
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT x[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) x[k] = ld_bf16v(g + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
                const uint32_t* w = reinterpret_cast<const uint32_t*>(&x[k]);
#pragma unroll
                for (int j = 0; j < NW; ++j) {
                    double lo = (double)__uint_as_float(w[j] << 16);
                    double hi = (double)__uint_as_float(w[j] & 0xffff0000u);
                    acc += lo * lo;
                    acc += hi * hi;
                }
            }
        }
    });
    if (blockIdx.x == 0)
        for (int64_t i = threadIdx.x; i < tail_n; i += kThreads) {
            double v = (double)bf16_bits_to_float(tail[i]);
            acc += v * v;
        }
    norm_epilogue<float>(ws, acc, max_norm);
}

// ===========================================================================
// K4b fused AdamW (optim.py:94-102), clip scale applied in-flight (:78)
// ===========================================================================
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_adamw(VT* __restrict__ th, const VT* __restrict__ g,
                                                     VT* __restrict__ m, VT* __restrict__ v, int64_t nvec,
                                                     AdamC<T> c, const NormWs* ws) {
    constexpr int W = sizeof(VT) / sizeof(T);
    const T s = load_scale<T>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U], b[U], mm[U], vv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) { a[k] = ldv(th + i); b[k] = ldv(g + i); mm[k] = ldv(m + i); vv[k] = ldv(v + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    T gg = L<VT, T>(b[k], w);
                    if (clip) gg = mul_rn(gg, s);                          // optim.py:78
                    adamw_lane<T>(L<VT, T>(a[k], w), gg, L<VT, T>(mm[k], w), L<VT, T>(vv[k], w), c);
                }
                stv(th + i, a[k]);
                stv(m + i, mm[k]);
                stv(v + i, vv[k]);
            }
        }
    });
}

// bf16 live params + fp32 master: 8 params per step (256-bit master/m/v,
// 128-bit bf16 g/theta)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&b);
}

template <int U>
__global__ void __launch_bounds__(kThreads) k_adamw_bf16(F8* __restrict__ master, uint4* __restrict__ th16,
                                                          const uint4* __restrict__ g16, F8* __restrict__ m,
                                                          F8* __restrict__ v, int64_t nvec, AdamC<float> c,
                                                          const NormWs* ws) {
    const float s = load_scale<float>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for_tiles<U>(nvec, [&](int64_t i0) {
        F8 a[U], mm[U], vv[U];
        uint4 gb[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
                a[k] = ld_stream(master + i); gb[k] = __ldcs(g16 + i);
                mm[k] = ld_stream(m + i); vv[k] = ld_stream(v + i);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
                const uint32_t* gw = &gb[k].x;
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    float gf = __uint_as_float((w & 1) ? (gw[w >> 1] & 0xffff0000u) : (gw[w >> 1] << 16));
                    float gg = clip ? mul_rn(gf, s) : gf;
                    adamw_lane<float>(lane(a[k], w), gg, lane(mm[k], w), lane(vv[k], w), c);
                }
                uint4 o;
                o.x = pack_bf16x2(a[k].lo.x, a[k].lo.y);
                o.y = pack_bf16x2(a[k].lo.z, a[k].lo.w);
                o.z = pack_bf16x2(a[k].hi.x, a[k].hi.y);
                o.w = pack_bf16x2(a[k].hi.z, a[k].hi.w);
                st_stream(master + i, a[k]);
                __stcs(th16 + i, o);
                st_stream(m + i, mm[k]);
                st_stream(v + i, vv[k]);
            }
        }
    });
}

// fp32 master -> bf16 live params (RNE), after an outer step on the master
template <int U>
__global__ void __launch_bounds__(kThreads) k_cast_bf16(const F8* __restrict__ src, uint4* __restrict__ dst,
                                                         int64_t nvec, const float* tail_src, uint16_t* tail_dst,
                                                         int64_t tail_n) {
    for_tiles<U>(nvec, [&](int64_t i0) {
        F8 a[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) a[k] = ld_stream(src + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
                uint4 o;
                o.x = pack_bf16x2(a[k].lo.x, a[k].lo.y);
                o.y = pack_bf16x2(a[k].lo.z, a[k].lo.w);
                o.z = pack_bf16x2(a[k].hi.x, a[k].hi.y);
                o.w = pack_bf16x2(a[k].hi.z, a[k].hi.w);
                __stcs(dst + i, o);
            }
        }
    });
    if (blockIdx.x == 0)
        for (int64_t i = threadIdx.x; i < tail_n; i += kThreads) {
            __nv_bfloat16 b = __float2bfloat16_rn(tail_src[i]);
            tail_dst[i] = *reinterpret_cast<uint16_t*>(&b);
        }
}

// scalar tail for the bf16 path
__global__ void k_adamw_bf16_tail(float* master, uint16_t* th16, const uint16_t* g16, float* m, float* v,
                                  int64_t n, AdamC<float> c, const NormWs* ws) {
    const float s = load_scale<float>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        float gg = bf16_bits_to_float(g16[i]);
        if (clip) gg = mul_rn(gg, s);
        float th = master[i], mm = m[i], vv = v[i];
        adamw_lane<float>(th, gg, mm, vv, c);
        master[i] = th;
        m[i] = mm;
        v[i] = vv;
        __nv_bfloat16 b = __float2bfloat16_rn(th);
        th16[i] = *reinterpret_cast<uint16_t*>(&b);
    }
}

// ===========================================================================
// multi-tensor AdamW / norm: one launch over a chunk table
// ===========================================================================
struct MtChunk {
    int32_t tensor;
    int32_t vec_ok;   // widest vector all four pointers allow at this chunk: 32, 16 or 0 bytes
    int64_t start;
    int64_t len;
};

// one AdamW pass over elements [0, n) of a chunk with vector type VT
template <typename T, typename VT>
__device__ __forceinline__ int64_t adamw_chunk_vec(T* th, const T* g, T* m, T* v, int64_t n, const AdamC<T>& c,
                                                   bool clip, T s) {
    constexpr int W = sizeof(VT) / sizeof(T);
    const int64_t nv = n / W;
    for (int64_t i = threadIdx.x; i < nv; i += kThreads) {
        VT a = ldv((VT*)th + i), b = ldv((const VT*)g + i), mm = ldv((VT*)m + i), vv = ldv((VT*)v + i);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            T gg = lane(b, w);
            if (clip) gg = mul_rn(gg, s);
            adamw_lane<T>(lane(a, w), gg, lane(mm, w), lane(vv, w), c);
        }
        stv((VT*)th + i, a);
        stv((VT*)m + i, mm);
        stv((VT*)v + i, vv);
    }
    return nv * W;
}
// 8192-element chunks: AdamW 6.59 -> 6.36 ms and the norm 0.89 -> 0.87 ms over the
// GPT-2 XL list (65536: few long-running CTAs on scattered regions; 2048: the norm's
// per-chunk overhead shows), tools/kernel_census.py --only-mt sweep
constexpr int64_t kMtChunk = 8192;

template <typename T>
__global__ void __launch_bounds__(kThreads) k_adamw_mt(const PierTensorDesc* __restrict__ d,
                                                        const MtChunk* __restrict__ ch, int nch, AdamC<T> c,
                                                        const NormWs* ws) {
    const T s = load_scale<T>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for (int ci = blockIdx.x; ci < nch; ci += gridDim.x) {
        MtChunk k = ch[ci];
        PierTensorDesc t = d[k.tensor];
        T* th = (T*)t.param + k.start;
        const T* g = (const T*)t.grad + k.start;
        T* m = (T*)t.exp_avg + k.start;
        T* v = (T*)t.exp_avg_sq + k.start;
        int64_t done = 0;
        if (k.vec_ok == 32)
            done = adamw_chunk_vec<T, typename V32<T>::type>(th, g, m, v, k.len, c, clip, s);
        else if (k.vec_ok == 16)
            done = adamw_chunk_vec<T, typename V16<T>::type>(th, g, m, v, k.len, c, clip, s);
        for (int64_t i = done + threadIdx.x; i < k.len; i += kThreads) {
            T gg = g[i];
            if (clip) gg = mul_rn(gg, s);
            T a = th[i], mm = m[i], vv = v[i];
            adamw_lane<T>(a, gg, mm, vv, c);
            th[i] = a;
            m[i] = mm;
            v[i] = vv;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_sqnorm_mt(const PierTensorDesc* __restrict__ d,
                                                         const MtChunk* __restrict__ ch, int nch, NormWs* ws,
                                                         double max_norm) {
    using VT = typename V16<T>::type;
    constexpr int W = V16<T>::W;
    double acc = 0.0;
    for (int ci = blockIdx.x; ci < nch; ci += gridDim.x) {
        MtChunk k = ch[ci];
        const T* g = (const T*)d[k.tensor].grad + k.start;
        int64_t nv = k.vec_ok ? k.len / W : 0;   // 16-B vectors suffice for a read-only pass
        // kMtU vectors in flight per thread (one at a time left the pass at 0.93 of
        // the copy bandwidth, profiles/r01_kernel_census_xl.jsonl)
        constexpr int kMtU = 4;
        for (int64_t i0 = threadIdx.x; i0 < nv; i0 += (int64_t)kThreads * kMtU) {
            VT b[kMtU];
#pragma unroll
            for (int u = 0; u < kMtU; ++u) {
                const int64_t i = i0 + (int64_t)u * kThreads;
                if (i < nv) b[u] = ldv((const VT*)g + i);
            }
#pragma unroll
            for (int u = 0; u < kMtU; ++u)
                if (i0 + (int64_t)u * kThreads < nv)
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        double x = (double)lane(b[u], w);
                        acc += x * x;
                    }
        }
        for (int64_t i = nv * W + threadIdx.x; i < k.len; i += kThreads) {
            double x = (double)g[i];
            acc += x * x;
        }
    }
    norm_epilogue<T>(ws, acc, max_norm);
}

// K5: one group (n = 1) at a boundary iteration: the inner AdamW step and the
// outer step in ONE pass (driver.py:395-399 then :428-440).  With one
// participant the mean is a copy (topology.py:113-121: acc/1 is exact), so the
// outer update reads the fresh AdamW result from registers: 44 B/param instead
// of 28 + 24 (theta is neither written nor re-read in between).  Same op
// sequence as k_adamw followed by k_outer_update -> bitwise identical.
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_adamw_outer(VT* __restrict__ th, const VT* __restrict__ g,
                                                           VT* __restrict__ m, VT* __restrict__ v,
                                                           VT* __restrict__ anchor, VT* __restrict__ mom, int64_t nvec,
                                                           AdamC<T> c, const NormWs* ws, T lr, T mu) {
    constexpr int W = sizeof(VT) / sizeof(T);
    const T s = load_scale<T>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U], b[U], mm[U], vv[U], an[U], mo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
                a[k] = ldv(th + i); b[k] = ldv(g + i); mm[k] = ldv(m + i); vv[k] = ldv(v + i);
                an[k] = ldv(anchor + i); mo[k] = ldv(mom + i);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    T gg = L<VT, T>(b[k], w);
                    if (clip) gg = mul_rn(gg, s);                                  // optim.py:78
                    T t = L<VT, T>(a[k], w);
                    adamw_lane<T>(t, gg, L<VT, T>(mm[k], w), L<VT, T>(vv[k], w), c);  // optim.py:94-102
                    T dl = sub_rn(t, L<VT, T>(an[k], w));                          // driver.py:434
                    T m2 = add_rn(mul_rn(mu, L<VT, T>(mo[k], w)), dl);             // optim.py:270
                    T up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));                 // optim.py:271
                    t = add_rn(t, sub_rn(up, dl));                                 // optim.py:275
                    L<VT, T>(mo[k], w) = m2;
                    L<VT, T>(a[k], w) = t;
                }
                stv(th + i, a[k]);
                stv(anchor + i, a[k]);                                             // driver.py:438
                stv(m + i, mm[k]);
                stv(v + i, vv[k]);
                stv(mom + i, mo[k]);
            }
        }
    });
}

// K4c: clipped copy  out = g * scale  (optim.py:78), scale read from the workspace
template <typename T, typename VT, int U>
__global__ void __launch_bounds__(kThreads) k_apply_clip(const VT* __restrict__ g, VT* __restrict__ out,
                                                          int64_t nvec, const NormWs* ws) {
    constexpr int W = sizeof(VT) / sizeof(T);
    const T s = (T)ws->res.scale;
    for_tiles<U>(nvec, [&](int64_t i0) {
        VT a[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) a[k] = ldv(g + i);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = i0 + (int64_t)k * kThreads;
            if (i < nvec) {
#pragma unroll
                for (int w = 0; w < W; ++w) L<VT, T>(a[k], w) = mul_rn(L<VT, T>(a[k], w), s);
                stv(out + i, a[k]);
            }
        }
    });
}

// ===========================================================================
// host-side launchers
// ===========================================================================
constexpr int kU = 4;    // 128-bit vectors in flight per thread per array
constexpr int kU32 = 2;  // 256-bit vectors in flight per thread per array
static int g_k5_unroll = 2;  // K5 256-bit vectors per thread per array (pier_kernel_tune)

template <typename VT_, int U_> struct VecTag {
    using VT = VT_;
    static constexpr int U = U_;
};

// Run a streaming kernel over [0,n): the widest vector body the buffers'
// alignment allows (`align` from common_align: 32 -> 256-bit, 16 -> 128-bit),
// then the same kernel instantiated on scalars for the tail (or for all of an
// unaligned buffer).  lv(VecTag<VT, U>, grid, nvec) launches the body.
template <typename T, int U32 = kU32, typename LaunchVec, typename LaunchScalar>
int run_split(int64_t n, int align, cudaStream_t st, LaunchVec lv, LaunchScalar ls) {
    if (n <= 0) return PIER_OK;
    int64_t done = 0;
    if (align == 32) {
        constexpr int W = V32<T>::W;
        int64_t nvec = n / W;
        if (nvec > 0) {
            lv(VecTag<typename V32<T>::type, U32>{}, stream_grid(nvec, U32), nvec);
            PIER_LAUNCH_CHECK("vector body (256-bit)");
        }
        done = nvec * W;
    } else if (align == 16) {
        constexpr int W = V16<T>::W;
        int64_t nvec = n / W;
        if (nvec > 0) {
            lv(VecTag<typename V16<T>::type, kU>{}, stream_grid(nvec, kU), nvec);
            PIER_LAUNCH_CHECK("vector body (128-bit)");
        }
        done = nvec * W;
    }
    if (done < n) {
        ls(stream_grid(n - done, 1), done, n - done);
        PIER_LAUNCH_CHECK("scalar tail");
    }
    return PIER_OK;
}

#define PIER_VEC_LAMBDA [&](auto tag, int grid, int64_t nvec)
#define PIER_VEC_TYPES using VT = typename decltype(tag)::VT; constexpr int U = decltype(tag)::U

template <typename T>
int pseudograd(const T* th, const T* an, T* out, int64_t n, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || (n > 0 && (!th || !an || !out))) return set_error(PIER_EINVAL, "pseudograd: bad args");
    int al = common_align({th, an, out});
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_pseudograd<T, VT, U><<<grid, kThreads, 0, st>>>((const VT*)th, (const VT*)an, (VT*)out, nvec); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_pseudograd<T, T, 1><<<grid, kThreads, 0, st>>>(th + off, an + off, out + off, cnt); });
}

template <typename T>
int fold_momentum(const T* mom, const T* d, T* out, int64_t n, double mu, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || (n > 0 && (!mom || !d || !out))) return set_error(PIER_EINVAL, "fold_momentum: bad args");
    int al = common_align({mom, d, out});
    T m = (T)mu;
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_fold<T, VT, U><<<grid, kThreads, 0, st>>>((const VT*)mom, (const VT*)d, (VT*)out, nvec, m); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_fold<T, T, 1><<<grid, kThreads, 0, st>>>(mom + off, d + off, out + off, cnt, m); });
}

template <typename T>
int outer_step_pure(const T* mom, const T* snap, const T* d, const T* anchor, T* th_out, T* mom_out,
                    int64_t n, double lr, double mu, void* stream) {
    cudaStream_t st = as_stream(stream);
    const T* base = anchor ? anchor : snap;
    if (n < 0 || (n > 0 && (!mom || !base || !d || !th_out || !mom_out)))
        return set_error(PIER_EINVAL, "outer_step: bad args");
    int al = common_align({mom, base, d, th_out, mom_out});
    T l = (T)lr, m = (T)mu;
    if (anchor)
        return run_split<T>(n, al, st,
            PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
                k_outer_pure<T, VT, U, true><<<grid, kThreads, 0, st>>>((const VT*)mom, (const VT*)base,
                    (const VT*)d, (VT*)th_out, (VT*)mom_out, nvec, l, m); },
            [&](int grid, int64_t off, int64_t cnt) {
                k_outer_pure<T, T, 1, true><<<grid, kThreads, 0, st>>>(mom + off, base + off, d + off,
                    th_out + off, mom_out + off, cnt, l, m); });
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_outer_pure<T, VT, U, false><<<grid, kThreads, 0, st>>>((const VT*)mom, (const VT*)base,
                (const VT*)d, (VT*)th_out, (VT*)mom_out, nvec, l, m); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_outer_pure<T, T, 1, false><<<grid, kThreads, 0, st>>>(mom + off, base + off, d + off,
                th_out + off, mom_out + off, cnt, l, m); });
}

template <typename T>
int outer_update(const T* avg, T* anchor, T* mom, T* th_out, int64_t n, double lr, double mu, int32_t div,
                 void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || div < 1 || (n > 0 && (!avg || !anchor || !mom || !th_out)))
        return set_error(PIER_EINVAL, "outer_update: bad args");
    int al = common_align({avg, anchor, mom, th_out});
    T l = (T)lr, m = (T)mu, dv = (T)div;
    int dd = div > 1;
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_outer_update<T, VT, U><<<grid, kThreads, 0, st>>>((const VT*)avg, (VT*)anchor, (VT*)mom,
                (VT*)th_out, nvec, l, m, dv, dd); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_outer_update<T, T, 1><<<grid, kThreads, 0, st>>>(avg + off, anchor + off, mom + off,
                th_out + off, cnt, l, m, dv, dd); });
}

template <typename T>
int warmup_fold(const T* th, T* anchor, T* mom, int64_t n, double mu, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || (n > 0 && (!th || !anchor || !mom))) return set_error(PIER_EINVAL, "warmup_fold: bad args");
    int al = common_align({th, anchor, mom});
    T m = (T)mu;
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_warmup_fold<T, VT, U><<<grid, kThreads, 0, st>>>((const VT*)th, (VT*)anchor, (VT*)mom, nvec, m); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_warmup_fold<T, T, 1><<<grid, kThreads, 0, st>>>(th + off, anchor + off, mom + off, cnt, m); });
}

template <typename T>
int mean_left_fold(const T* const* parts, int32_t np, T* out, int64_t n, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (np < 1 || np > PIER_MAX_PARTS || !parts || n < 0 || (n > 0 && !out))
        return set_error(PIER_EINVAL, "mean_left_fold: need 1..64 participants");
    PartPtrs<T> pp{};
    int al = common_align({out});
    for (int i = 0; i < np; ++i) {
        if (n > 0 && !parts[i]) return set_error(PIER_EINVAL, "mean_left_fold: null participant");
        pp.p[i] = parts[i];
        int a = common_align({parts[i]});
        al = a < al ? a : al;
    }
    T nf = (T)np;
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_mean_left_fold<T, VT, U><<<grid, kThreads, 0, st>>>(pp, np, (VT*)out, nvec, nf); },
        [&](int grid, int64_t off, int64_t cnt) {
            PartPtrs<T> q = pp;
            for (int i = 0; i < np; ++i) q.p[i] = pp.p[i] + off;
            k_mean_left_fold<T, T, 1><<<grid, kThreads, 0, st>>>(q, np, out + off, cnt, nf); });
}

inline int norm_grid(int64_t nvec, int unroll) {
    int g = stream_grid(nvec, unroll, 4);
    return g > kMaxNormBlocks ? kMaxNormBlocks : g;
}

template <typename T>
int grad_sqnorm(const T* g, int64_t n, double max_norm, void* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || !ws || (n > 0 && !g)) return set_error(PIER_EINVAL, "grad_sqnorm: bad args");
    if (!(max_norm > 0.0)) return set_error(PIER_EINVAL, "grad_sqnorm: clip_norm must be positive");
    NormWs* w = (NormWs*)ws;
    int al = common_align({g});
    if (al == 32) {
        using VT = typename V32<T>::type;
        constexpr int W = V32<T>::W;
        int64_t nvec = n / W, done = nvec * W;
        k_sqnorm<T, VT, kU32><<<norm_grid(nvec > 0 ? nvec : 1, kU32), kThreads, 0, st>>>(
            (const VT*)g, nvec, g + done, n - done, w, max_norm);
    } else if (al == 16) {
        using VT = typename V16<T>::type;
        constexpr int W = V16<T>::W;
        int64_t nvec = n / W, done = nvec * W;
        k_sqnorm<T, VT, kU><<<norm_grid(nvec > 0 ? nvec : 1, kU), kThreads, 0, st>>>(
            (const VT*)g, nvec, g + done, n - done, w, max_norm);
    } else {
        k_sqnorm<T, T, kU><<<norm_grid(n > 0 ? n : 1, kU), kThreads, 0, st>>>(g, n, g, 0, w, max_norm);
    }
    PIER_LAUNCH_CHECK("k_sqnorm");
    return PIER_OK;
}

template <typename T>
int adamw(T* th, const T* g, T* m, T* v, int64_t n, const PierAdamW* hp, const void* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (!hp || n < 0 || (n > 0 && (!th || !g || !m || !v))) return set_error(PIER_EINVAL, "adamw: bad args");
    if (hp->step < 1) return set_error(PIER_EINVAL, "adamw: step must be >= 1 (state.step + 1)");
    AdamC<T> c = adam_consts<T>(*hp);
    const NormWs* w = (const NormWs*)ws;
    int al = common_align({th, g, m, v});
    // one 256-bit vector per array per thread: 6.24 ms vs 6.92 with two at XL (tools/stream_probe.cu)
    return run_split<T, 1>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_adamw<T, VT, U><<<grid, kThreads, 0, st>>>((VT*)th, (const VT*)g, (VT*)m, (VT*)v, nvec, c, w); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_adamw<T, T, 1><<<grid, kThreads, 0, st>>>(th + off, g + off, m + off, v + off, cnt, c, w); });
}

template <typename T>
int adamw_outer(T* th, const T* g, T* m, T* v, T* anchor, T* mom, int64_t n, const PierAdamW* hp, const void* ws,
                double lr, double mu, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (!hp || n < 0 || (n > 0 && (!th || !g || !m || !v || !anchor || !mom)))
        return set_error(PIER_EINVAL, "adamw_outer: bad args");
    if (hp->step < 1) return set_error(PIER_EINVAL, "adamw_outer: step must be >= 1");
    AdamC<T> c = adam_consts<T>(*hp);
    const NormWs* w = (const NormWs*)ws;
    T l = (T)lr, mu_ = (T)mu;
    int al = common_align({th, g, m, v, anchor, mom});
    auto body = PIER_VEC_LAMBDA {
        PIER_VEC_TYPES;
        k_adamw_outer<T, VT, U><<<grid, kThreads, 0, st>>>((VT*)th, (const VT*)g, (VT*)m, (VT*)v, (VT*)anchor,
                                                           (VT*)mom, nvec, c, w, l, mu_);
    };
    auto tail = [&](int grid, int64_t off, int64_t cnt) {
        k_adamw_outer<T, T, 1><<<grid, kThreads, 0, st>>>(th + off, g + off, m + off, v + off, anchor + off,
                                                          mom + off, cnt, c, w, l, mu_);
    };
    if (g_k5_unroll == 1) return run_split<T, 1>(n, al, st, body, tail);
    return run_split<T, 2>(n, al, st, body, tail);
}

template <typename T>
int apply_clip(const T* g, T* out, int64_t n, const void* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || !ws || (n > 0 && (!g || !out))) return set_error(PIER_EINVAL, "apply_clip: bad args");
    const NormWs* w = (const NormWs*)ws;
    int al = common_align({g, out});
    return run_split<T>(n, al, st,
        PIER_VEC_LAMBDA {
            PIER_VEC_TYPES;
            k_apply_clip<T, VT, U><<<grid, kThreads, 0, st>>>((const VT*)g, (VT*)out, nvec, w); },
        [&](int grid, int64_t off, int64_t cnt) {
            k_apply_clip<T, T, 1><<<grid, kThreads, 0, st>>>(g + off, out + off, cnt, w); });
}

}  // namespace pier

// ===========================================================================
// multi-tensor list object
// ===========================================================================
struct PierTensorList {
    int dtype;  // 0 f32, 1 f64
    int nchunks;
    PierTensorDesc* d_desc;
    pier::MtChunk* d_chunks;
};

using namespace pier;

extern "C" {

int pier_pseudograd_f32(const float* a, const float* b, float* o, int64_t n, void* s) { return pseudograd(a, b, o, n, s); }
int pier_pseudograd_f64(const double* a, const double* b, double* o, int64_t n, void* s) { return pseudograd(a, b, o, n, s); }

int pier_fold_momentum_f32(const float* m, const float* d, float* o, int64_t n, double mu, void* s) {
    return fold_momentum(m, d, o, n, mu, s);
}
int pier_fold_momentum_f64(const double* m, const double* d, double* o, int64_t n, double mu, void* s) {
    return fold_momentum(m, d, o, n, mu, s);
}

int pier_outer_step_f32(const float* mom, const float* snap, const float* d, const float* anchor, float* th,
                        float* mo, int64_t n, double lr, double mu, void* s) {
    return outer_step_pure(mom, snap, d, anchor, th, mo, n, lr, mu, s);
}
int pier_outer_step_f64(const double* mom, const double* snap, const double* d, const double* anchor,
                        double* th, double* mo, int64_t n, double lr, double mu, void* s) {
    return outer_step_pure(mom, snap, d, anchor, th, mo, n, lr, mu, s);
}

int pier_outer_update_f32(const float* a, float* an, float* m, float* th, int64_t n, double lr, double mu,
                          int32_t div, void* s) {
    return outer_update(a, an, m, th, n, lr, mu, div, s);
}
int pier_outer_update_f64(const double* a, double* an, double* m, double* th, int64_t n, double lr, double mu,
                          int32_t div, void* s) {
    return outer_update(a, an, m, th, n, lr, mu, div, s);
}

int pier_warmup_fold_f32(const float* th, float* an, float* m, int64_t n, double mu, void* s) {
    return warmup_fold(th, an, m, n, mu, s);
}
int pier_warmup_fold_f64(const double* th, double* an, double* m, int64_t n, double mu, void* s) {
    return warmup_fold(th, an, m, n, mu, s);
}

int pier_mean_left_fold_f32(const float* const* p, int32_t np, float* o, int64_t n, void* s) {
    return mean_left_fold(p, np, o, n, s);
}
int pier_mean_left_fold_f64(const double* const* p, int32_t np, double* o, int64_t n, void* s) {
    return mean_left_fold(p, np, o, n, s);
}

size_t pier_norm_ws_bytes(void) { return sizeof(NormWs); }

int pier_kernel_tune(int ctas_per_sm, int k5_unroll) {
    if (ctas_per_sm > 0) default_ctas_per_sm() = ctas_per_sm;
    else if (ctas_per_sm < 0) default_ctas_per_sm() = 0;
    if (k5_unroll > 0) g_k5_unroll = k5_unroll >= 2 ? 2 : 1;
    return PIER_OK;
}

int pier_clip_finalize(void* ws, double max_norm, int32_t dtype_code, void* stream) {
    if (!ws || !(max_norm > 0.0) || (dtype_code != 0 && dtype_code != 1))
        return set_error(PIER_EINVAL, "clip_finalize: bad args");
    cudaStream_t st = as_stream(stream);
    if (dtype_code == 0) k_clip_finalize<float><<<1, 32, 0, st>>>((NormWs*)ws, max_norm);
    else k_clip_finalize<double><<<1, 32, 0, st>>>((NormWs*)ws, max_norm);
    PIER_LAUNCH_CHECK("k_clip_finalize");
    return PIER_OK;
}

int pier_apply_clip_f32(const float* g, float* out, int64_t n, const void* ws, void* s) {
    return apply_clip(g, out, n, ws, s);
}
int pier_apply_clip_f64(const double* g, double* out, int64_t n, const void* ws, void* s) {
    return apply_clip(g, out, n, ws, s);
}

int pier_grad_sqnorm_f32(const float* g, int64_t n, double mx, void* ws, void* s) { return grad_sqnorm(g, n, mx, ws, s); }
int pier_grad_sqnorm_f64(const double* g, int64_t n, double mx, void* ws, void* s) { return grad_sqnorm(g, n, mx, ws, s); }

int pier_grad_sqnorm_bf16(const uint16_t* g, int64_t n, double max_norm, void* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || !ws || (n > 0 && !g)) return set_error(PIER_EINVAL, "grad_sqnorm_bf16: bad args");
    if (!(max_norm > 0.0)) return set_error(PIER_EINVAL, "grad_sqnorm_bf16: clip_norm must be positive");
    int al = common_align({g});
    if (al == 32) {
        int64_t nvec = n / 16, done = nvec * 16;
        k_sqnorm_bf16<F8, kU32><<<norm_grid(nvec > 0 ? nvec : 1, kU32), kThreads, 0, st>>>(
            (const F8*)g, nvec, g + done, n - done, (NormWs*)ws, max_norm);
    } else {
        int64_t nvec = al ? n / 8 : 0;
        int64_t done = nvec * 8;
        k_sqnorm_bf16<uint4, kU><<<norm_grid(nvec > 0 ? nvec : 1, kU), kThreads, 0, st>>>(
            (const uint4*)g, nvec, g + done, n - done, (NormWs*)ws, max_norm);
    }
    PIER_LAUNCH_CHECK("k_sqnorm_bf16");
    return PIER_OK;
}

int pier_adamw_f32(float* th, const float* g, float* m, float* v, int64_t n, const PierAdamW* hp, const void* ws,
                   void* s) {
    return adamw(th, g, m, v, n, hp, ws, s);
}
int pier_adamw_f64(double* th, const double* g, double* m, double* v, int64_t n, const PierAdamW* hp,
                   const void* ws, void* s) {
    return adamw(th, g, m, v, n, hp, ws, s);
}

int pier_adamw_outer_f32(float* th, const float* g, float* m, float* v, float* anchor, float* mom, int64_t n,
                         const PierAdamW* hp, const void* ws, double lr, double mu, void* s) {
    return adamw_outer(th, g, m, v, anchor, mom, n, hp, ws, lr, mu, s);
}
int pier_adamw_outer_f64(double* th, const double* g, double* m, double* v, double* anchor, double* mom, int64_t n,
                         const PierAdamW* hp, const void* ws, double lr, double mu, void* s) {
    return adamw_outer(th, g, m, v, anchor, mom, n, hp, ws, lr, mu, s);
}

int pier_adamw_bf16_f32(float* master, uint16_t* th16, const uint16_t* g16, float* m, float* v, int64_t n,
                        const PierAdamW* hp, const void* ws, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (!hp || n < 0 || (n > 0 && (!master || !th16 || !g16 || !m || !v)))
        return set_error(PIER_EINVAL, "adamw_bf16: bad args");
    if (hp->step < 1) return set_error(PIER_EINVAL, "adamw_bf16: step must be >= 1");
    AdamC<float> c = adam_consts<float>(*hp);
    // vector body: 32-byte aligned fp32 arrays and 16-byte aligned bf16 arrays
    bool al = common_align({master, m, v}) == 32 && common_align({th16, g16}) >= 16;
    int64_t nvec = al ? n / 8 : 0;
    if (nvec > 0) {
        k_adamw_bf16<1><<<stream_grid(nvec, 1), kThreads, 0, st>>>((F8*)master, (uint4*)th16, (const uint4*)g16,
                                                                    (F8*)m, (F8*)v, nvec, c, (const NormWs*)ws);
        PIER_LAUNCH_CHECK("k_adamw_bf16");
    }
    int64_t done = nvec * 8;
    if (done < n) {
        k_adamw_bf16_tail<<<1, kThreads, 0, st>>>(master + done, th16 + done, g16 + done, m + done, v + done,
                                                  n - done, c, (const NormWs*)ws);
        PIER_LAUNCH_CHECK("k_adamw_bf16_tail");
    }
    return PIER_OK;
}

int pier_cast_bf16(const float* src, uint16_t* dst, int64_t n, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 0 || (n > 0 && (!src || !dst))) return set_error(PIER_EINVAL, "cast_bf16: bad args");
    if (n == 0) return PIER_OK;
    bool al = common_align({src}) == 32 && common_align({dst}) >= 16;
    int64_t nvec = al ? n / 8 : 0;
    int64_t done = nvec * 8;
    k_cast_bf16<2><<<stream_grid(nvec > 0 ? nvec : 1, 2), kThreads, 0, st>>>(
        (const F8*)src, (uint4*)dst, nvec, src + done, dst + done, n - done);
    PIER_LAUNCH_CHECK("k_cast_bf16");
    return PIER_OK;
}

int pier_tensor_list_create(const PierTensorDesc* descs, int32_t nt, int32_t dtype, PierTensorList** out) {
    if (!descs || nt < 1 || !out || (dtype != 0 && dtype != 1))
        return set_error(PIER_EINVAL, "tensor_list_create: bad args");
    const int esz = dtype == 0 ? 4 : 8;
    std::vector<MtChunk> ch;
    for (int t = 0; t < nt; ++t) {
        const PierTensorDesc& d = descs[t];
        if (d.numel < 0) return set_error(PIER_EINVAL, "tensor_list_create: negative numel");
        if (d.numel > 0 && (!d.param || !d.grad || !d.exp_avg || !d.exp_avg_sq))
            return set_error(PIER_EINVAL, "tensor_list_create: null pointer");
        for (int64_t s = 0; s < d.numel; s += kMtChunk) {
            MtChunk c;
            c.tensor = t;
            c.start = s;
            c.len = (d.numel - s) < kMtChunk ? (d.numel - s) : kMtChunk;
            auto at = [&](const void* p) { return (const void*)((const char*)p + s * esz); };
            c.vec_ok = common_align({at(d.param), at(d.grad), at(d.exp_avg), at(d.exp_avg_sq)});
            ch.push_back(c);
        }
    }
    auto* L = new (std::nothrow) PierTensorList{dtype, (int)ch.size(), nullptr, nullptr};
    if (!L) return set_error(PIER_ENOMEM, "tensor_list_create: host alloc");
    if (cudaMalloc(&L->d_desc, sizeof(PierTensorDesc) * nt) != cudaSuccess ||
        cudaMalloc(&L->d_chunks, sizeof(MtChunk) * (ch.empty() ? 1 : ch.size())) != cudaSuccess) {
        cudaFree(L->d_desc);
        delete L;
        return set_error(PIER_ECUDA, "tensor_list_create: cudaMalloc failed");
    }
    cudaMemcpy(L->d_desc, descs, sizeof(PierTensorDesc) * nt, cudaMemcpyHostToDevice);
    if (!ch.empty()) cudaMemcpy(L->d_chunks, ch.data(), sizeof(MtChunk) * ch.size(), cudaMemcpyHostToDevice);
    PIER_CHECK_CUDA(cudaGetLastError());
    *out = L;
    return PIER_OK;
}

int pier_tensor_list_destroy(PierTensorList* L) {
    if (!L) return PIER_OK;
    cudaFree(L->d_desc);
    cudaFree(L->d_chunks);
    delete L;
    return PIER_OK;
}

int pier_grad_sqnorm_mt(const PierTensorList* L, double max_norm, void* ws, void* stream) {
    if (!L || !ws) return set_error(PIER_EINVAL, "grad_sqnorm_mt: bad args");
    if (!(max_norm > 0.0)) return set_error(PIER_EINVAL, "grad_sqnorm_mt: clip_norm must be positive");
    cudaStream_t st = as_stream(stream);
    int grid = L->nchunks < kMaxNormBlocks ? (L->nchunks > 0 ? L->nchunks : 1) : kMaxNormBlocks;
    int cap = sm_count() * 4;
    if (grid > cap) grid = cap;
    if (L->dtype == 0)
        k_sqnorm_mt<float><<<grid, kThreads, 0, st>>>(L->d_desc, L->d_chunks, L->nchunks, (NormWs*)ws, max_norm);
    else
        k_sqnorm_mt<double><<<grid, kThreads, 0, st>>>(L->d_desc, L->d_chunks, L->nchunks, (NormWs*)ws, max_norm);
    PIER_LAUNCH_CHECK("k_sqnorm_mt");
    return PIER_OK;
}

int pier_adamw_mt(const PierTensorList* L, const PierAdamW* hp, const void* ws, void* stream) {
    if (!L || !hp) return set_error(PIER_EINVAL, "adamw_mt: bad args");
    if (hp->step < 1) return set_error(PIER_EINVAL, "adamw_mt: step must be >= 1");
    if (L->nchunks == 0) return PIER_OK;
    cudaStream_t st = as_stream(stream);
    int grid = L->nchunks;   // one chunk per CTA (pier_common.cuh: stream_grid)
    if (L->dtype == 0)
        k_adamw_mt<float><<<grid, kThreads, 0, st>>>(L->d_desc, L->d_chunks, L->nchunks, adam_consts<float>(*hp),
                                                      (const NormWs*)ws);
    else
        k_adamw_mt<double><<<grid, kThreads, 0, st>>>(L->d_desc, L->d_chunks, L->nchunks, adam_consts<double>(*hp),
                                                       (const NormWs*)ws);
    PIER_LAUNCH_CHECK("k_adamw_mt");
    return PIER_OK;
}

}  // extern "C"
