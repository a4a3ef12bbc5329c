// AdamW element math, its host-rounded constants and the norm workspace
// layout -- shared by the standalone kernels (pier_kernels.cu) and the
// persistent round kernel (pier_round.cu).
#pragma once

#include <cmath>

#include "pier_common.cuh"

namespace pier {

// K4a workspace: the clip record, a launch counter and per-block partials
constexpr int kMaxNormBlocks = 2048;
struct NormWs {
    PierClip res;                 // 40 B
    char pad0[64 - sizeof(PierClip)];
    unsigned int done;            // blocks finished in the current launch
    char pad1[60];
    double partial[kMaxNormBlocks];
};
static_assert(sizeof(PierClip) <= 64, "clip record");

template <typename T> struct AdamC {
    T decay, b1, c1, b2, c2, bc1, bc2, eps, lr;
};

// one AdamW element in the reference's op order (optim.py:94-102)
template <typename T>
__device__ __forceinline__ void adamw_lane(T& th, T g, T& m, T& v, const AdamC<T>& c) {
    T t1 = mul_rn(th, c.decay);                                         // optim.py:96
    T m2 = add_rn(mul_rn(c.b1, m), mul_rn(c.c1, g));                    // optim.py:97
    T v2 = add_rn(mul_rn(c.b2, v), mul_rn(c.c2, mul_rn(g, g)));         // optim.py:98
    T mh = div_rn(m2, c.bc1);                                           // optim.py:99
    T den = add_rn(sqrt_rn(div_rn(v2, c.bc2)), c.eps);                  // optim.py:100-101
    th = sub_rn(t1, div_rn(mul_rn(c.lr, mh), den));                     // optim.py:102
    m = m2;
    v = v2;
}

// ---- K4a building blocks (deterministic reductions) -------------------------
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// fixed-shape block reduction -> deterministic
__device__ __forceinline__ double block_sum(double x) {
    __shared__ double red[kThreads / 32];
    x = warp_sum(x);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

template <typename T> __device__ __forceinline__ void clip_finalize(NormWs* ws, double sq, double max_norm);

// reference: norm = float(np.sqrt(np.dot(g, g))) -- for float32 the dot and
// the sqrt are float32, so round the fp64 sum to fp32 before the fp32 sqrt.
template <> __device__ __forceinline__ void clip_finalize<float>(NormWs* ws, double sq, double max_norm) {
    float sq32 = __double2float_rn(sq);
    double norm = (double)__fsqrt_rn(sq32);
    ws->res.sqnorm = sq;
    ws->res.norm = norm;
    int clip = norm > max_norm;
    ws->res.clipped = clip;
    ws->res.scale = clip ? (double)__double2float_rn(max_norm / norm) : 1.0;
    ws->res.nonfinite = !isfinite(sq);
}
template <> __device__ __forceinline__ void clip_finalize<double>(NormWs* ws, double sq, double max_norm) {
    double norm = __dsqrt_rn(sq);
    ws->res.sqnorm = sq;
    ws->res.norm = norm;
    int clip = norm > max_norm;
    ws->res.clipped = clip;
    ws->res.scale = clip ? max_norm / norm : 1.0;
    ws->res.nonfinite = !isfinite(sq);
}

// Every block deposits its partial; the last block to arrive sums them in
// block order (deterministic for a given grid) and re-arms the counter.
// Returns true in thread 0 of the last block, with the total in *sum.
__device__ __forceinline__ bool norm_sum_last(NormWs* ws, double mine, double* sum) {
    __shared__ bool last;
    double b = block_sum(mine);
    if (threadIdx.x == 0) {
        ws->partial[blockIdx.x] = b;
        __threadfence();
        unsigned int prev = atomicAdd(&ws->done, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) s += ((volatile double*)ws->partial)[i];
    s = block_sum(s);
    if (threadIdx.x != 0) return false;
    ws->done = 0;  // re-arm for the next launch on this workspace
    *sum = s;
    return true;
}

template <typename T>
__device__ __forceinline__ void norm_epilogue(NormWs* ws, double mine, double max_norm) {
    double s;
    if (norm_sum_last(ws, mine, &s)) clip_finalize<T>(ws, s, max_norm);
}

template <typename T>
__device__ __forceinline__ T load_scale(const NormWs* ws) {
    return ws ? (T)ws->res.scale : (T)1;
}

template <typename T> AdamC<T> adam_consts(const PierAdamW& h) {
    // exactly the reference's dt(...) roundings (optim.py:96-102); Python's
    // float ** int is C pow(), so the bias corrections agree bit for bit.
    AdamC<T> c;
    c.decay = (T)(1.0 - h.lr * h.weight_decay);
    c.b1 = (T)h.beta1;
    c.c1 = (T)(1.0 - h.beta1);
    c.b2 = (T)h.beta2;
    c.c2 = (T)(1.0 - h.beta2);
    c.bc1 = (T)(1.0 - std::pow(h.beta1, (double)h.step));
    c.bc2 = (T)(1.0 - std::pow(h.beta2, (double)h.step));
    c.eps = (T)h.eps;
    c.lr = (T)h.lr;
    return c;
}

}  // namespace pier
