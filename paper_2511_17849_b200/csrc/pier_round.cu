// One persistent kernel per Pier round at an outer-step boundary, n groups
// over NVLink: this group's inner AdamW step AND the cross-group outer step,
// overlapped span by span inside the kernel.
//
// Replaces driver.py:395-399 (apply) followed by driver.py:428-440 (mean of the
// groups, Nesterov outer step, re-anchor, broadcast) for one group per GPU.
//
// The grid (co-resident: cooperative launch) is split in two roles:
//   * AdamW CTAs claim tiles of the local buffer in address order from a
//     counter (K4b math, the clip scale from the K4a workspace) and, once past
//     a span, bump this rank's ready[span] counter with a system-scope release;
//   * exchange CTAs walk the same spans; for span b they wait until EVERY
//     rank's ready[b] shows all its AdamW CTAs done (acquire loads over
//     NVLink), then pull their part of this rank's slice from every rank,
//     fold in ascending rank order (bitwise = topology.py:113-121), apply the
//     fused update with the local anchor/momentum shard and push the result
//     into every rank's buffer.
// At the end every exchange CTA signals a done counter on every rank and
// waits for all of them, so when the kernel returns every remote push into
// this rank's buffer has landed.  HBM-bound AdamW and NVLink-bound exchange
// run concurrently on separate SM partitions with no host or stream
// synchronisation in between.  Counters are monotonic and the wait targets
// are booked per round, so no reset is needed between rounds.  The ranks meet
// at a stream-ordered barrier right before the launch, so the spins only
// cover the round itself; a spin that exceeds the communicator's timeout
// (20 s default, PIER_ROUND_TIMEOUT_S / pier_comm_set_timeout) records which
// counter of which rank it waited on in a host-mapped slot (surfaced by
// pier_last_error) and traps instead of hanging the GPU.  On a virtual group
// (n ranks on one device, pier_vgroup.cpp) all ranks' grids are ONE
// cooperative launch (k_round_multi).  The 7B recipe runs the same kernel
// with bf16 gradients (pier_round_fused_bf16_f32): the AdamW role updates the fp32
// master and the exchange runs on it; the bf16 live copy is refreshed afterwards.
#include <cuda/atomic>

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <string>

#include "pier_adamw.cuh"
#include "pier_comm_internal.h"
#include "pier_common.cuh"

namespace pier {

constexpr int kRoundMaxSpans = 4096;
// AdamW-role CTAs per SM and total exchange-role CTAs (0 = one per SM);
// tools/round_sweep.py at n=2/4: AdamW needs the bandwidth, the NVLink
// exchange saturates with few CTAs (pier_round_split)
static int g_split_a = 3, g_split_b = 0;
// signal block (per rank, mapped into every rank):
//   [0, kMax)        ready[b]: +nA per round that used span b (written by this rank)
//   kSigDone         done: +nB*NR per round (written by every rank)
//   [kSigUses, +kMax] booked totals: sum of nA over earlier rounds that used span
//                    b, and of nB*NR for done (local bookkeeping, identical on
//                    every rank) -> the wait targets, so rounds with different
//                    span counts or CTA splits never desynchronise the counters
constexpr int kSigDone = kRoundMaxSpans;
constexpr int kSigWork = kRoundMaxSpans + 32;   // AdamW tile claims (local): +tiles+nA per round
constexpr int kSigUses = kRoundMaxSpans + 64;
constexpr int kBookWork = kRoundMaxSpans + 1;   // booked claim total, at kSigUses + kBookWork
constexpr size_t kSigBytes = (2 * kRoundMaxSpans + 128) * sizeof(uint32_t);

struct RoundParams {
    float* th[PIER_MAX_RANKS];
    uint32_t* sig[PIER_MAX_RANKS];
    const float* g;
    const uint16_t* g16;          // bf16 gradients (7B recipe) instead of g, or null
    float* m;
    float* v;
    float* anchor;
    float* mom;
    int64_t n_pad, B;
    int rank, nA, nB;
    uint32_t epoch;
    AdamC<float> c;
    const NormWs* ws;
    float lr, mu;
    uint32_t* diag;               // host-mapped timeout record (may be null)
    uint64_t timeout_ns;
};

// every virtual rank's round in one cooperative launch: blocks [v*per, (v+1)*per) are rank v's grid
struct RoundMulti {
    RoundParams p[PIER_MAX_RANKS];
    int per;
};

#ifdef PIER_ROUND_TRACE
// diagnostic build only (-DPIER_ROUND_TRACE): per-span timestamps of exchange CTA 0
__device__ unsigned long long g_trace_ready[kRoundMaxSpans], g_trace_xdone[kRoundMaxSpans];
__device__ unsigned long long g_trace_start, g_trace_adam_end, g_trace_end;
#endif

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// wait until *p >= target (wrap-safe), acquire at system scope.  On timeout:
// record {flag, rank, span, observed, target, kind, peer} in the host-mapped
// diagnostic slot, then trap (a peer never arrived; the context is lost).
__device__ __forceinline__ void wait_geq(uint32_t* p, uint32_t target, const RoundParams& prm, int span, int kind,
                                         int peer) {
    cuda::atomic_ref<uint32_t, cuda::thread_scope_system> a(*p);
    uint64_t t0 = globaltimer();
    uint32_t seen;
    while ((int32_t)((seen = a.load(cuda::memory_order_acquire)) - target) < 0) {
        __nanosleep(64);
        if (globaltimer() - t0 > prm.timeout_ns) {
            if (volatile uint32_t* d = prm.diag) {
                d[1] = (uint32_t)prm.rank;
                d[2] = (uint32_t)span;
                d[3] = seen;
                d[4] = target;
                d[5] = (uint32_t)kind;
                d[6] = (uint32_t)peer;
                __threadfence_system();
                d[0] = 1u;
                __threadfence_system();
            }
            __trap();
        }
    }
}

// 4 co-resident CTAs per SM (64 registers): 3 AdamW + 1 exchange was the
// fastest split at n=2 and n=4 (tools/exp/README.md: round_dyn*); the exchange role
// moves 256-bit vectors at n <= 2, 128-bit above (register budget)
constexpr int kRoundMinCtas = 4;
template <int NR> struct XchgVec {                   // exchange role vector: 256-bit up to 2 peers
    using VT = typename std::conditional<NR <= 2, F8, float4>::type;
};

// one rank's round; bid = this CTA's index in the rank's grid
template <int NR>
__device__ __forceinline__ void round_body(const RoundParams& p, const int bid) {
    const int64_t span = p.B * NR;
    const int r = p.rank;
    if (bid < p.nA) {
        // ---------------- AdamW role: this group's inner step (optim.py:94-102).
        // CTAs claim 2048-element tiles in address order from a local counter
        // (the in-order window of a one-tile-per-CTA launch; a static stride
        // was 0.1-1.1 ms slower per round, tools/exp/README.md: round_dyn).  A CTA that
        // claims a tile in span b' has finished all its tiles of spans < b', so
        // it releases ready[cur..b'-1] then -- each CTA adds exactly 1 per span.
        constexpr int W = 8;
        const float s = load_scale<float>(p.ws);
        const bool clip = p.ws != nullptr && p.ws->res.clipped;
        F8* th = reinterpret_cast<F8*>(p.th[r]);
        const F8* g = reinterpret_cast<const F8*>(p.g);
        const uint4* g16 = reinterpret_cast<const uint4*>(p.g16);   // 8 bf16 per F8 of master
        F8* m = reinterpret_cast<F8*>(p.m);
        F8* v = reinterpret_cast<F8*>(p.v);
        const uint32_t work_base = p.sig[r][kSigUses + kBookWork];
        const int64_t span_v = span / W;                               // vectors per full span
        const uint32_t tiles_full = (uint32_t)((span_v + kThreads - 1) / kThreads);
        const int nspans = (int)((p.n_pad + span - 1) / span);
        const int64_t last_v = (p.n_pad - (int64_t)(nspans - 1) * span) / W;
        const uint32_t total = tiles_full * (uint32_t)(nspans - 1) + (uint32_t)((last_v + kThreads - 1) / kThreads);
        __shared__ uint32_t s_claim;
        int cur = 0;
#ifdef PIER_ROUND_TRACE
        if (bid == 0 && threadIdx.x == 0) {
            g_trace_start = globaltimer();
            g_trace_adam_end = 0;
        }
#endif
        for (;;) {
            if (threadIdx.x == 0) {
                cuda::atomic_ref<uint32_t, cuda::thread_scope_device> w(p.sig[r][kSigWork]);
                s_claim = w.fetch_add(1u, cuda::memory_order_relaxed) - work_base;
            }
            __syncthreads();                 // also: this CTA's stores of its previous tile are done
            const uint32_t t = s_claim;
            __syncthreads();
            const int b = t < total ? (int)(t / tiles_full) : nspans;
            if (b > cur) {
                if (threadIdx.x == 0)
                    for (int q = cur; q < b; ++q) {
                        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> rdy(p.sig[r][q]);
                        rdy.fetch_add(1u, cuda::memory_order_release);
                    }
                cur = b;
            }
            if (t >= total) {
#ifdef PIER_ROUND_TRACE
                if (threadIdx.x == 0) atomicMax(&g_trace_adam_end, (unsigned long long)globaltimer());
#endif
                break;
            }
            const int64_t nv = b == nspans - 1 ? last_v : span_v;
            const int64_t i = (int64_t)(t - (uint32_t)b * tiles_full) * kThreads + threadIdx.x;
            if (i < nv) {
                const int64_t e = (int64_t)b * span_v + i;
                F8 a = ld_stream(th + e), gg, mm = ld_stream(m + e), vv = ld_stream(v + e);
                if (g16 != nullptr) {   // bf16 -> fp32 is exact; element 2j = low half of word j
                    const uint4 gb = __ldcs(g16 + e);
                    const uint32_t* gw = &gb.x;
#pragma unroll
                    for (int w = 0; w < W; ++w)
                        lane(gg, w) = __uint_as_float((w & 1) ? (gw[w >> 1] & 0xffff0000u) : (gw[w >> 1] << 16));
                } else {
                    gg = ld_stream(g + e);
                }
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    float x = lane(gg, w);
                    if (clip) x = mul_rn(x, s);                                         // optim.py:78
                    adamw_lane<float>(lane(a, w), x, lane(mm, w), lane(vv, w), p.c);
                }
                // theta with an L2 evict-last policy: the owner's pull and the result
                // push that overwrites it mostly hit L2 (n=2: 12.67 -> 12.45 ms,
                // tools/exp/README.md: round_l2); m, v stream out evict-first
                st_keep_l2(th + e, a, l2_evict_last_policy());
                st_stream(m + e, mm);
                st_stream(v + e, vv);
            }
        }
        return;
    }
    // ---------------- exchange role: mean of the groups + outer step (driver.py:428-440)
    // One vector per thread per tile; the peers' vectors are loaded QG at a time
    // and folded in ascending rank order as they arrive (the left fold needs
    // only the running sum), so at NR = 8 the role keeps 4 pulls in flight per
    // thread within the 64-register budget of 4 co-resident CTAs per SM.
    using VT = typename XchgVec<NR>::VT;
    constexpr int W = sizeof(VT) / sizeof(float);
    constexpr int QG = NR <= 4 ? NR : 4;
    const int cta = bid - p.nA;
    const uint32_t* booked = p.sig[r] + kSigUses;   // ready/done totals of earlier rounds (local)
    const uint32_t done_target = booked[kRoundMaxSpans] + (uint32_t)(p.nB * NR);
    const float nf = (float)NR;
    int b = 0;
    int64_t sh = 0;
    for (int64_t off = 0; off < p.n_pad; off += span, ++b) {
        const int64_t len = (p.n_pad - off) < span ? (p.n_pad - off) : span;
        const int64_t slice = len / NR, nv = slice / W;
        const int64_t base = off + (int64_t)r * slice;      // this rank's slice of the span
        if (threadIdx.x < NR) wait_geq(&p.sig[threadIdx.x][b], booked[b] + (uint32_t)p.nA, p, b, 0, threadIdx.x);
        __syncthreads();
#ifdef PIER_ROUND_TRACE
        if (cta == 0 && threadIdx.x == 0) g_trace_ready[b] = globaltimer();
#endif
        VT* an = reinterpret_cast<VT*>(p.anchor + sh);
        VT* mo = reinterpret_cast<VT*>(p.mom + sh);
        for (int64_t i = (int64_t)cta * kThreads + threadIdx.x; i < nv; i += (int64_t)p.nB * kThreads) {
            VT x[QG];
#pragma unroll
            for (int q = 0; q < QG; ++q) x[q] = ld_cg(reinterpret_cast<const VT*>(p.th[q] + base) + i);
            VT a4 = ld_stream(an + i), m4 = ld_stream(mo + i);
            float acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                acc[w] = lane(x[0], w);
#pragma unroll
                for (int q = 1; q < QG; ++q) acc[w] = add_rn(acc[w], lane(x[q], w));          // topology.py:113-120
            }
#pragma unroll
            for (int q0 = QG; q0 < NR; q0 += QG) {
#pragma unroll
                for (int q = 0; q < QG && q0 + q < NR; ++q)
                    x[q] = ld_cg(reinterpret_cast<const VT*>(p.th[q0 + q] + base) + i);
#pragma unroll
                for (int w = 0; w < W; ++w)
#pragma unroll
                    for (int q = 0; q < QG && q0 + q < NR; ++q) acc[w] = add_rn(acc[w], lane(x[q], w));
            }
            VT out;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                float av = div_rn(acc[w], nf);                                                 // topology.py:121
                float dl = sub_rn(av, lane(a4, w));                                            // driver.py:434
                float m2 = add_rn(mul_rn(p.mu, lane(m4, w)), dl);                              // optim.py:270
                float up = mul_rn(p.lr, add_rn(mul_rn(p.mu, m2), dl));                         // optim.py:271
                av = add_rn(av, sub_rn(up, dl));                                               // optim.py:275
                lane(m4, w) = m2;
                lane(a4, w) = av;                                                              // driver.py:438
                lane(out, w) = av;
            }
            st_stream(mo + i, m4);
            st_stream(an + i, a4);
#pragma unroll
            for (int q = 0; q < NR; ++q)                                                       // driver.py:439-440
                st_cg(reinterpret_cast<VT*>(p.th[q] + base) + i, out);
        }
        sh += slice;
#ifdef PIER_ROUND_TRACE
        __syncthreads();
        if (cta == 0 && threadIdx.x == 0) g_trace_xdone[b] = globaltimer();
#endif
    }
    // all of this CTA's remote pushes are ordered before its done signals
    __syncthreads();
    if (threadIdx.x < NR) {
        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> d(p.sig[threadIdx.x][kSigDone]);
        d.fetch_add(1u, cuda::memory_order_release);
    }
    if (threadIdx.x == 0) wait_geq(&p.sig[r][kSigDone], done_target, p, b, 1, r);
#ifdef PIER_ROUND_TRACE
    if (cta == 0 && threadIdx.x == 0) g_trace_end = globaltimer();
#endif
    __syncthreads();
    if (cta == 0) {  // every exchange CTA of every rank is past its waits: book this round's targets
        uint32_t* u = p.sig[r] + kSigUses;
        for (int i = threadIdx.x; i < b; i += kThreads) u[i] += (uint32_t)p.nA;
        if (threadIdx.x == 0) {
            u[kRoundMaxSpans] += (uint32_t)(p.nB * NR);
            // every AdamW CTA made its last (failing) claim before releasing the last span
            u[kBookWork] = p.sig[r][kSigWork];
        }
    }
}

template <int NR>
__global__ void __launch_bounds__(kThreads, kRoundMinCtas) k_round(const __grid_constant__ RoundParams p) {
    round_body<NR>(p, (int)blockIdx.x);
}

// virtual groups only: 3 CTAs per SM (80 registers) -- with 4 the eight-way
// parameter switch spills at some team sizes
template <int NR>
__global__ void __launch_bounds__(kThreads, kRoundMinCtas - 1) k_round_multi(const __grid_constant__ RoundMulti m) {
    const int v = (int)blockIdx.x / m.per, bid = (int)blockIdx.x - v * m.per;
    // static indices keep every parameter a constant-bank operand (a dynamic
    // m.p[v] costs registers and spills)
    switch (v) {
        case 0: round_body<NR>(m.p[0], bid); break;
        case 1: round_body<NR>(m.p[1], bid); break;
        case 2: round_body<NR>(m.p[2], bid); break;
        case 3: round_body<NR>(m.p[3], bid); break;
        case 4: round_body<NR>(m.p[4], bid); break;
        case 5: round_body<NR>(m.p[5], bid); break;
        case 6: round_body<NR>(m.p[6], bid); break;
        default: round_body<NR>(m.p[7], bid); break;
    }
}

template <int NR>
int launch_round(const RoundParams& prm, int grid, cudaStream_t st) {
    void* args[] = {(void*)&prm};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_round<NR>, dim3(grid), dim3(kThreads), args, 0, st);
    count_launch();
    if (e != cudaSuccess) return cuda_status(e, "cudaLaunchCooperativeKernel(k_round)");
    return PIER_OK;
}

template <int NR>
int launch_round_multi(const RoundMulti& m, int nv, cudaStream_t st) {
    void* args[] = {(void*)&m};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_round_multi<NR>, dim3(nv * m.per), dim3(kThreads),
                                                args, 0, st);
    count_launch();
    if (e != cudaSuccess) return cuda_status(e, "cudaLaunchCooperativeKernel(k_round_multi)");
    return PIER_OK;
}

template <int NR>
int round_ctas(int* per_sm) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_round<NR>, kThreads, 0);
    if (e != cudaSuccess) return cuda_status(e, "occupancy(k_round)");
    *per_sm = occ;
    return PIER_OK;
}

template <int NR>
int round_multi_ctas(int* per_sm) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_round_multi<NR>, kThreads, 0);
    if (e != cudaSuccess) return cuda_status(e, "occupancy(k_round_multi)");
    *per_sm = occ;
    return PIER_OK;
}

int round_multi_ctas_n(int n, int* per_sm) {
    switch (n) {
        case 2: return round_multi_ctas<2>(per_sm);
        case 3: return round_multi_ctas<3>(per_sm);
        case 4: return round_multi_ctas<4>(per_sm);
        case 5: return round_multi_ctas<5>(per_sm);
        case 6: return round_multi_ctas<6>(per_sm);
        case 7: return round_multi_ctas<7>(per_sm);
        case 8: return round_multi_ctas<8>(per_sm);
        default: return set_error(PIER_EINVAL, "round: teams of 2..8 ranks");
    }
}

int launch_round_multi_n(int NR, const RoundMulti& m, int nv, cudaStream_t st) {
    switch (NR) {
        case 2: return launch_round_multi<2>(m, nv, st);
        case 3: return launch_round_multi<3>(m, nv, st);
        case 4: return launch_round_multi<4>(m, nv, st);
        case 5: return launch_round_multi<5>(m, nv, st);
        case 6: return launch_round_multi<6>(m, nv, st);
        case 7: return launch_round_multi<7>(m, nv, st);
        case 8: return launch_round_multi<8>(m, nv, st);
        default: return set_error(PIER_EINVAL, "round: teams of 2..8 ranks");
    }
}

// Leader of a virtual group's round: every rank's parameters -> ONE cooperative
// launch.  The co-resident budget is split evenly between the ranks; within a
// rank 3/4 of its CTAs run AdamW (the multi-GPU split, pier_round_split).
int launch_virtual_round(void* const* payloads, int nv, cudaStream_t st) {
    RoundMulti m;   // copied into the launch by cudaLaunchCooperativeKernel
    memset(&m, 0, sizeof(m));
    const int NR = ((const RoundParams*)payloads[0])->nA;   // team size, stashed by round_fused
    int occ = 0;
    if (int e = round_multi_ctas_n(NR, &occ)) return e;
    m.per = sm_count() * occ / nv;
    const int nA = (m.per * 3) / 4, nB = m.per - nA;
    if (nA < 1 || nB < 1) return set_error(PIER_EINVAL, "virtual round: too few co-resident CTAs per rank");
    for (int v = 0; v < nv; ++v) {
        m.p[v] = *(const RoundParams*)payloads[v];
        if (m.p[v].nA != NR) return set_error(PIER_EINVAL, "virtual round: every team must have the same size");
        m.p[v].nA = nA;
        m.p[v].nB = nB;
    }
    return launch_round_multi_n(NR, m, nv, st);
}

}  // namespace pier

using namespace pier;

extern "C" {

int pier_round_split(int adamw_ctas_per_sm, int exchange_ctas) {
    if (adamw_ctas_per_sm > 0) g_split_a = adamw_ctas_per_sm;
    if (exchange_ctas >= 0) g_split_b = exchange_ctas;   // 0 = one per SM
    return PIER_OK;
}

}  // extern "C"

namespace pier {
// g (fp32) or g16 (bf16) gradients; everything else shared by both entry points
static int round_fused(PierComm* c, int32_t theta_id, const int32_t* team, int32_t nteam, const float* g,
                       const uint16_t* g16, float* m, float* v, float* anchor_shard, float* mom_shard,
                       int64_t n_padded, int64_t B, const PierAdamW* hp, const void* clip_ws, double lr, double mu,
                       void* stream) {
    if (!c || theta_id < 0 || theta_id >= (int)c->shared.size() || !c->shared[theta_id].local)
        return set_error(PIER_EINVAL, "round_fused: unknown shared buffer");
    if ((!g && !g16) || !m || !v || !anchor_shard || !mom_shard || !hp) return set_error(PIER_EINVAL, "round_fused: null");
    if (common_align({m, v, anchor_shard, mom_shard}) != 32 || (g && !aligned32(g)) || (g16 && !aligned16(g16)))
        return set_error(PIER_EINVAL, "round_fused: buffers must be 32-byte aligned (bf16 gradients 16-byte)");
    if (hp->step < 1) return set_error(PIER_EINVAL, "round_fused: step must be >= 1");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, me = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &me)) return e;
    if (n < 2) return set_error(PIER_EINVAL, "round_fused: a team of 2..8 ranks");
    if (n_padded <= 0 || n_padded % ((int64_t)n * 8) || B <= 0 || B % 8 ||
        (size_t)n_padded * 4 > c->shared[theta_id].bytes)
        return set_error(PIER_EINVAL, "round_fused: bad n_padded / bucket");
    const int64_t span = B * n;
    if ((n_padded + span - 1) / span > kRoundMaxSpans)
        return set_error(PIER_EINVAL, "round_fused: too many spans (raise bucket_elems)");
    if (c->sig_id < 0) return set_error(PIER_EINVAL, "round_fused: communicator has no signal block");
    const PierSharedBuf& sb = c->shared[theta_id];
    const PierSharedBuf& sig = c->shared[c->sig_id];
    RoundParams prm;
    memset(&prm, 0, sizeof(prm));
    for (int q = 0; q < n; ++q) {
        prm.th[q] = (float*)sb.peers[members[q]];
        prm.sig[q] = (uint32_t*)sig.peers[members[q]];
    }
    prm.g = g;
    prm.g16 = g16;
    prm.m = m;
    prm.v = v;
    prm.anchor = anchor_shard;
    prm.mom = mom_shard;
    prm.n_pad = n_padded;
    prm.B = B;
    prm.rank = me;
    prm.c = adam_consts<float>(*hp);
    prm.ws = (const NormWs*)clip_ws;
    prm.lr = (float)lr;
    prm.mu = (float)mu;
    prm.diag = c->diag_dev;
    prm.timeout_ns = c->timeout_ns;
    cudaStream_t st = as_stream(stream);
    if (c->vg) {
        // virtual group: the leader launches every rank's grid as ONE cooperative
        // kernel (nA carries the team size to it; it sets the split)
        prm.nA = n;
        return vg_rendezvous(c, &prm, st, [c](void* const* ps, cudaStream_t ls) {
            return launch_virtual_round(ps, c->nranks, ls);
        });
    }
    int occ = 0;
    int e = 0;
    switch (n) {
        case 2: e = round_ctas<2>(&occ); break;
        case 3: e = round_ctas<3>(&occ); break;
        case 4: e = round_ctas<4>(&occ); break;
        case 5: e = round_ctas<5>(&occ); break;
        case 6: e = round_ctas<6>(&occ); break;
        case 7: e = round_ctas<7>(&occ); break;
        default: e = round_ctas<8>(&occ); break;
    }
    if (e) return e;
    const int sms = sm_count();
    int a = g_split_a, nb = g_split_b > 0 ? g_split_b : sms;
    if (occ < 2) return set_error(PIER_EINVAL, "round_fused: needs 2 co-resident CTAs per SM");
    if (a >= occ) a = occ - 1;                       // leave room for the exchange role
    if (nb > sms * (occ - a)) nb = sms * (occ - a);  // the whole grid must be co-resident
    prm.nA = sms * a;
    prm.nB = nb;
    prm.epoch = ++c->round_epoch;
    const int grid = prm.nA + prm.nB;
    // meet first (1-element all-reduce on this stream): the spin-waits then cover
    // only the round, never another rank's lag in reaching it (a slow data
    // loader, a rank-local checkpoint)
    if (int e2 = barrier(c, st)) return e2;
    switch (n) {
        case 2: return launch_round<2>(prm, grid, st);
        case 3: return launch_round<3>(prm, grid, st);
        case 4: return launch_round<4>(prm, grid, st);
        case 5: return launch_round<5>(prm, grid, st);
        case 6: return launch_round<6>(prm, grid, st);
        case 7: return launch_round<7>(prm, grid, st);
        default: return launch_round<8>(prm, grid, st);
    }
}
}  // namespace pier

extern "C" {

int pier_round_fused_team_f32(PierComm* c, int32_t theta_id, const int32_t* team, int32_t nteam, const float* g,
                              float* m, float* v, float* anchor_shard, float* mom_shard, int64_t n_padded, int64_t B,
                              const PierAdamW* hp, const void* clip_ws, double lr, double mu, void* stream) {
    if (!g) return set_error(PIER_EINVAL, "round_fused: null gradient");
    return round_fused(c, theta_id, team, nteam, g, nullptr, m, v, anchor_shard, mom_shard, n_padded, B, hp, clip_ws,
                       lr, mu, stream);
}

int pier_round_fused_bf16_f32(PierComm* c, int32_t theta_id, const uint16_t* g16, float* m, float* v,
                              float* anchor_shard, float* mom_shard, int64_t n_padded, int64_t B,
                              const PierAdamW* hp, const void* clip_ws, double lr, double mu, void* stream) {
    if (!g16) return set_error(PIER_EINVAL, "round_fused_bf16: null gradient");
    return round_fused(c, theta_id, nullptr, 0, nullptr, g16, m, v, anchor_shard, mom_shard, n_padded, B, hp,
                       clip_ws, lr, mu, stream);
}

size_t pier_round_sig_bytes(void) { return kSigBytes; }

#ifdef PIER_ROUND_TRACE
// out: [start, adam_end, end, ready[0..nspans), xdone[0..nspans)] (ns, globaltimer)
int pier_round_trace(unsigned long long* out, int nspans) {
    if (nspans > kRoundMaxSpans) nspans = kRoundMaxSpans;
    PIER_CHECK_CUDA(cudaMemcpyFromSymbol(out, g_trace_start, 8));
    PIER_CHECK_CUDA(cudaMemcpyFromSymbol(out + 1, g_trace_adam_end, 8));
    PIER_CHECK_CUDA(cudaMemcpyFromSymbol(out + 2, g_trace_end, 8));
    PIER_CHECK_CUDA(cudaMemcpyFromSymbol(out + 3, g_trace_ready, 8 * (size_t)nspans));
    PIER_CHECK_CUDA(cudaMemcpyFromSymbol(out + 3 + nspans, g_trace_xdone, 8 * (size_t)nspans));
    return PIER_OK;
}
#endif

int pier_round_virtual_f32(int32_t n, float* const* theta, const float* const* g, float* const* m_,
                           float* const* v, float* const* anchor_shards, float* const* mom_shards,
                           uint32_t* const* sig, int64_t n_padded, int64_t B, const PierAdamW* hp,
                           const void* const* clip_ws, double lr, double mu, int32_t adamw_ctas,
                           int32_t exchange_ctas, void* const* streams) {
    if (n < 2 || n > PIER_MAX_RANKS || !theta || !g || !m_ || !v || !anchor_shards || !mom_shards || !sig || !hp ||
        !clip_ws || !streams)
        return set_error(PIER_EINVAL, "round_virtual: 2..8 virtual ranks and non-null tables");
    if (adamw_ctas < 1 || exchange_ctas < 1) return set_error(PIER_EINVAL, "round_virtual: CTA counts >= 1");
    if (n_padded <= 0 || n_padded % ((int64_t)n * 8) || B <= 0 || B % 8)
        return set_error(PIER_EINVAL, "round_virtual: bad n_padded / bucket");
    const int64_t span = B * n;
    if ((n_padded + span - 1) / span > kRoundMaxSpans) return set_error(PIER_EINVAL, "round_virtual: too many spans");
    if (hp->step < 1) return set_error(PIER_EINVAL, "round_virtual: step must be >= 1");
    for (int r = 0; r < n; ++r)
        if (!theta[r] || !g[r] || !m_[r] || !v[r] || !anchor_shards[r] || !mom_shards[r] || !sig[r] ||
            common_align({theta[r], g[r], m_[r], v[r], anchor_shards[r], mom_shards[r]}) != 32)
            return set_error(PIER_EINVAL, "round_virtual: buffers must be non-null and 32-byte aligned");
    // ONE cooperative launch over all virtual ranks: co-residency is guaranteed,
    // so the CTAs of one rank may spin on flags another rank's CTAs release
    // a host-mapped timeout record for the harness (once per process) and the
    // PIER_ROUND_TIMEOUT_S spin limit, as on a communicator
    static uint32_t* diag_dev = nullptr;
    static uint64_t timeout_ns = 20ull * 1000000000ull;
    if (!diag_dev) {
        void* h = nullptr;
        PIER_CHECK_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
        memset(h, 0, 64);
        PIER_CHECK_CUDA(cudaHostGetDevicePointer((void**)&diag_dev, h, 0));
        register_diag((volatile uint32_t*)h);
        if (const char* s = getenv("PIER_ROUND_TIMEOUT_S"))
            if (atof(s) > 0) timeout_ns = (uint64_t)(atof(s) * 1e9);
    }
    RoundMulti m;
    memset(&m, 0, sizeof(m));
    int occ = 0;
    if (int e = round_multi_ctas_n(n, &occ)) return e;
    if (n * (adamw_ctas + exchange_ctas) > occ * sm_count())
        return set_error(PIER_EINVAL, "round_virtual: the grids of all virtual ranks must be co-resident");
    m.per = adamw_ctas + exchange_ctas;
    for (int r = 0; r < n; ++r) {
        RoundParams& prm = m.p[r];
        for (int q = 0; q < n; ++q) {
            prm.th[q] = theta[q];
            prm.sig[q] = sig[q];
        }
        prm.g = g[r];
        prm.m = m_[r];
        prm.v = v[r];
        prm.anchor = anchor_shards[r];
        prm.mom = mom_shards[r];
        prm.n_pad = n_padded;
        prm.B = B;
        prm.rank = r;
        prm.c = adam_consts<float>(*hp);
        prm.ws = (const NormWs*)clip_ws[r];
        prm.lr = (float)lr;
        prm.mu = (float)mu;
        prm.nA = adamw_ctas;
        prm.nB = exchange_ctas;
        prm.diag = diag_dev;
        prm.timeout_ns = timeout_ns;
    }
    return launch_round_multi_n(n, m, n, as_stream(streams[0]));
}

int pier_round_fused_f32(PierComm* c, int32_t theta_id, const float* g, float* m, float* v, float* anchor_shard,
                         float* mom_shard, int64_t n_padded, int64_t B, const PierAdamW* hp, const void* clip_ws,
                         double lr, double mu, void* stream) {
    return pier_round_fused_team_f32(c, theta_id, nullptr, 0, g, m, v, anchor_shard, mom_shard, n_padded, B, hp,
                                     clip_ws, lr, mu, stream);
}

}  // extern "C"
