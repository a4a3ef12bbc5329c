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
