// Fused outer step over NVLink peer memory (one kernel = reduce-scatter +
// outer update + all-gather), the same pattern for the lazy-phase gradient
// mean, and the sharded inner steps (reduce-scatter + norm, AdamW on the
// rank's shard, all-gather; optionally copy-engine pulls behind the backward
// and a copy-engine all-gather behind the next forward) -- see "Lazy phase,
// sharded" below.
//
// Replaces outer_delta_sync / inner_gradient_sync (topology.py:104-132,
// driver.py:385, :428-429) plus the broadcast of the new model
// (driver.py:439-440).  Every rank owns a contiguous slice of the flat buffer
// (same span/slice layout as the NCCL path, see pier_comm.cu).  For each
// 32-byte (or 16-byte) vector of its slice a thread
//   1. loads the vector from EVERY rank's buffer over NVLink, rank 0 first,
//      and sums in ascending rank order -- exactly the reference's left fold
//      `acc = a0; acc += a1; ...; acc /= n` (topology.py:113-121), so the
//      result is bitwise equal to the reference at any group count;
//   2. (outer) applies the fused Nesterov/re-anchor update with the local
//      anchor / momentum shard (optim.py:243-276, driver.py:434-438);
//   3. stores the result into EVERY rank's buffer (the all-gather).
// Wire volume: each link direction carries the peers' pulls of our slices
// plus our pushes of results, 2(n-1)/n * 4N bytes -- the ring RS + AG volume --
// but in ONE pass with no partial-sum round trips through HBM, the update
// fused in, and every result written exactly once per rank.
//
// Cross-GPU ordering: a 1-element ncclAllReduce on the caller's stream before
// the kernel (all ranks finished writing their buffers) and after it (all
// remote stores landed; each block ends with a system-scope fence).  No
// kernel spins on another GPU.
#include <cstring>
#include <vector>

#include "pier_adamw.cuh"
#include "pier_comm_internal.h"
#include "pier_common.cuh"

namespace pier {

struct PeerTable {
    float* p[PIER_MAX_RANKS];
};

// kP2pMeanOwn: the mean of this rank's slice is stored into its own buffer
// only (the reduce-scatter half of the sharded lazy step below)
enum { kP2pMean = 0, kP2pOuter = 1, kP2pMeanOwn = 2 };

// launch tunables (pier_p2p_tune): CTAs per SM, 16-byte vectors per thread
// per rank (0 = auto: 256-bit vectors where aligned), diagnostic flags (bit0
// remote loads, bit1 remote stores)
static int g_ctas_per_sm = 4, g_unroll = 0, g_flags = 3;
// the sharded lazy step's two kernels: 6 CTAs per SM (tools/exp/lazy_sweep.sh, XL:
// n=2 9.62 -> 9.37 ms, n=4 14.08 -> 13.96 vs 4); pier_p2p_tune sets both
static int g_lazy_ctas_per_sm = 6;
// pipelined round: CTAs per SM of its AdamW spans and of its exchange kernels
static int g_round_adamw_ctas = 8, g_round_p2p_ctas = 2;  // tools/round_sweep.py, n=2/4 XL

// One launch covers every span of the buffer: the CTAs walk the spans in
// order and stride over this rank's slice of each (no per-span launch drain;
// spans never wait on each other here -- the NCCL barriers around the launch
// order the ranks).
// Fused norm (MODE == kP2pMean, nws != NULL): the owner also sums the squares
// of the means it produces (fp64); the last CTA sums the CTA partials in order
// and stores this rank's total into slot[r] of every rank's norm slots, which
// k_norm_slots adds up in rank order after the closing barrier -> the clip
// record of the averaged gradient, identical on every rank, without re-reading
// the buffer (optim.py:76 on the result of driver.py:380-393).
struct SlotTable {
    double* p[PIER_MAX_RANKS];
};

template <int MODE, int NR, int U, typename VT>
__global__ void __launch_bounds__(kThreads) k_p2p_reduce(PeerTable peers, PeerTable dsts, int64_t n_pad, int64_t B,
                                                          int r, VT* __restrict__ anchor, VT* __restrict__ mom,
                                                          float lr, float mu, float nf, NormWs* nws,
                                                          SlotTable slots, uint32_t dup) {
    double sq = 0.0;
    constexpr int W = sizeof(VT) / sizeof(float);
    const int64_t span = B * NR;
    const int64_t tile = (int64_t)kThreads * U;
    int64_t sh = 0;  // vector offset of this span's slice in the shard
    for (int64_t off = 0; off < n_pad; off += span) {
        const int64_t len = (n_pad - off) < span ? (n_pad - off) : span;
        const int64_t slice = len / NR, nvec = slice / W;
        const int64_t base = off + (int64_t)r * slice;  // this rank's slice of the span
        for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < nvec; t0 += (int64_t)gridDim.x * tile) {
            // issue every rank's loads first (NR*U vectors in flight per thread) ...
            VT x[NR][U];
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                const VT* src = reinterpret_cast<const VT*>(peers.p[q] + base);
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                    // dup bit q: member q's copy is member q-1's (dp replicas of one group
                    // hold identical params) -- reuse it instead of pulling it again
                    if (i < nvec) x[q][k] = (q > 0 && ((dup >> q) & 1u)) ? x[q > 0 ? q - 1 : 0][k] : ld_cg(src + i);
                }
            }
            VT an[U], m[U];
            if (MODE == kP2pOuter) {
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                    if (i < nvec) { an[k] = ld_stream(anchor + sh + i); m[k] = ld_stream(mom + sh + i); }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                if (i >= nvec) continue;
                VT out;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    // ... then the reference's left fold: acc = a0; acc += a1; ...; acc /= n
                    float acc = lane(x[0][k], w);
#pragma unroll
                    for (int q = 1; q < NR; ++q) acc = add_rn(acc, lane(x[q][k], w));   // topology.py:113-120
                    float av = div_rn(acc, nf);                                         // topology.py:121
                    if (MODE == kP2pOuter) {
                        float dl = sub_rn(av, lane(an[k], w));                          // driver.py:434
                        float m2 = add_rn(mul_rn(mu, lane(m[k], w)), dl);               // optim.py:270
                        float up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));              // optim.py:271
                        av = add_rn(av, sub_rn(up, dl));                                // optim.py:275
                        lane(m[k], w) = m2;
                        lane(an[k], w) = av;                                            // driver.py:438
                    }
                    lane(out, w) = av;
                    if (MODE != kP2pOuter) sq += (double)av * (double)av;
                }
                if (MODE == kP2pOuter) {
                    st_stream(mom + sh + i, m[k]);
                    st_stream(anchor + sh + i, an[k]);
                }
                if (MODE == kP2pMeanOwn) {   // dsts.p[0] = this rank's buffer (a static index: no stack copy)
                    st_cg(reinterpret_cast<VT*>(dsts.p[0] + base) + i, out);
                } else {
#pragma unroll
                    for (int q = 0; q < NR; ++q)                                        // driver.py:439-440
                        st_cg(reinterpret_cast<VT*>(dsts.p[q] + base) + i, out);
                }
            }
        }
        sh += nvec;
    }
    if (MODE != kP2pOuter && nws) {
        double total;
        if (norm_sum_last(nws, sq, &total))
            for (int q = 0; q < NR; ++q) slots.p[q][r] = total;   // this rank's share, to every rank
    }
    __threadfence_system();
}

__global__ void k_norm_slots(const double* slots, int n, NormWs* ws, double max_norm) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < n; ++q) s += slots[q];   // rank order: identical on every rank
        clip_finalize<float>(ws, s, max_norm);
    }
}

// Lazy-phase mean of bf16 gradients (7B recipe: driver.py:380-393 with bf16
// live gradients).  Rank r owns the r-th 1/n of the buffer; for 8 bf16 per
// thread it pulls that vector from every rank, widens each value exactly to
// fp32, folds in ascending rank order in fp32 (topology.py:113-120), divides
// by n (topology.py:121) and rounds ONCE to bf16 (RNE), then pushes the result
// into every rank's buffer.  Replaces an ncclAllReduce(ncclBfloat16, ncclAvg),
// whose bf16 partial sums round at every step and in ring order.
struct BfTable {
    uint16_t* p[PIER_MAX_RANKS];
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// B: this rank's slice of every span of NR*B elements (B = n_pad/NR: one span)
template <int NR, bool OWN>
__global__ void __launch_bounds__(kThreads) k_p2p_mean_bf16(BfTable peers, uint16_t* __restrict__ own,
                                                             int64_t n_pad, int64_t B, int r, NormWs* nws,
                                                             SlotTable slots) {
    const float nf = (float)NR;
    double sq = 0.0;   // fused K4a (nws != NULL): squares of the rounded means this rank owns
    for (int64_t off = 0; off < n_pad; off += B * NR) {
    const int64_t len = (n_pad - off) < B * NR ? (n_pad - off) : B * NR;
    const int64_t slice = len / NR, nvec = slice / 8, base = off + (int64_t)r * slice;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * kThreads) {
        uint4 x[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) x[q] = __ldcg(reinterpret_cast<const uint4*>(peers.p[q] + base) + i);
        uint4 out;
        uint32_t* ow = &out.x;
#pragma unroll
        for (int w = 0; w < 4; ++w) {   // word w: element 2w in the low half, 2w+1 in the high half
            float lo = bf_lo((&x[0].x)[w]), hi = bf_hi((&x[0].x)[w]);
#pragma unroll
            for (int q = 1; q < NR; ++q) {
                lo = add_rn(lo, bf_lo((&x[q].x)[w]));
                hi = add_rn(hi, bf_hi((&x[q].x)[w]));
            }
            const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(div_rn(lo, nf)));
            const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(div_rn(hi, nf)));
            ow[w] = l | (h << 16);
            if (nws) {   // the value every rank will hold, as k_sqnorm_bf16 squares it
                const double a = (double)__uint_as_float(l << 16), b = (double)__uint_as_float(h << 16);
                sq += a * a;
                sq += b * b;
            }
        }
        if (OWN) {   // the reduce-scatter half of the sharded lazy step: our slice only
            __stcg(reinterpret_cast<uint4*>(own + base) + i, out);
        } else {
#pragma unroll
            for (int q = 0; q < NR; ++q) __stcg(reinterpret_cast<uint4*>(peers.p[q] + base) + i, out);
        }
    }
    }
    if (nws) {
        double total;
        if (norm_sum_last(nws, sq, &total))
            for (int q = 0; q < NR; ++q) slots.p[q][r] = total;   // this rank's share, to every rank
    }
    __threadfence_system();
}

// one rank's K4a partial square sum into slot[idx] of every team member
__global__ void k_slot_put(SlotTable dst, int idx, int n, const NormWs* ws) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double v = ws->res.sqnorm;
        for (int q = 0; q < n; ++q) dst.p[q][idx] = v;
        __threadfence_system();
    }
}

struct NormArgs {
    NormWs* ws = nullptr;   // fused norm of the mean (kP2pMean / kP2pMeanOwn)
    SlotTable slots{};
    uint32_t dup = 0;       // members whose copy repeats the previous member's (k_p2p_reduce)
};

template <int MODE, int NR, int U, typename VT>
void launch_vt(int ctas_per_sm, cudaStream_t st, const PeerTable& pt, const PeerTable& dt, int64_t n_pad, int64_t B,
               int r, float* an, float* mo, float lr, float mu, const NormArgs& na) {
    constexpr int W = sizeof(VT) / sizeof(float);
    const int64_t nvec = n_pad / NR / W;  // this rank's shard, in vectors
    int grid = stream_grid(nvec, U, ctas_per_sm);
    if (na.ws && grid > kMaxNormBlocks) grid = kMaxNormBlocks;   // one partial per CTA
    k_p2p_reduce<MODE, NR, U, VT><<<grid, kThreads, 0, st>>>(pt, dt, n_pad, B, r, (VT*)an, (VT*)mo, lr, mu,
                                                             (float)NR, na.ws, na.slots, na.dup);
}

// 256-bit vectors when every address allows it and the registers do (<= 4
// ranks), else 128-bit; g_unroll (pier_p2p_tune) overrides the 128-bit unroll.
// (n_pad, B) with n_pad % (8*NR) == 0 and B % 8 == 0 keep every slice 32-byte aligned.
template <int MODE, int NR>
void launch_p2p(int ctas_per_sm, cudaStream_t st, const PeerTable& pt, const PeerTable& dt, int64_t n_pad, int64_t B,
                int r, float* an, float* mo, float lr, float mu, const NormArgs& na) {
    bool wide = NR <= 4 && g_unroll == 0 && n_pad % (8 * NR) == 0 && B % 8 == 0 &&
                (MODE != kP2pOuter || common_align({an, mo}) == 32);
    for (int q = 0; q < NR && wide; ++q) wide = aligned32(pt.p[q]) && aligned32(dt.p[q]);
    if (wide) {
        if (NR <= 2) launch_vt<MODE, NR, 2, F8>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na);
        else launch_vt<MODE, NR, 1, F8>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na);
        return;
    }
    const int u = g_unroll > 0 ? g_unroll : (NR <= 2 ? 4 : NR <= 4 ? 2 : 1);
    if (u >= 4) launch_vt<MODE, NR, 4, float4>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na);
    else if (u == 2) launch_vt<MODE, NR, 2, float4>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na);
    else launch_vt<MODE, NR, 1, float4>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na);
}

template <int MODE>
int launch_p2p_n(int n, int ctas_per_sm, cudaStream_t st, const PeerTable& pt, const PeerTable& dt, int64_t n_pad,
                 int64_t B, int r, float* an, float* mo, float lr, float mu, const NormArgs& na = NormArgs()) {
    switch (n) {
        case 1: launch_p2p<MODE, 1>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 2: launch_p2p<MODE, 2>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 3: launch_p2p<MODE, 3>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 4: launch_p2p<MODE, 4>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 5: launch_p2p<MODE, 5>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 6: launch_p2p<MODE, 6>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 7: launch_p2p<MODE, 7>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        case 8: launch_p2p<MODE, 8>(ctas_per_sm, st, pt, dt, n_pad, B, r, an, mo, lr, mu, na); break;
        default: return set_error(PIER_EINVAL, "p2p: 1..8 ranks");
    }
    PIER_LAUNCH_CHECK("k_p2p_reduce");
    return PIER_OK;
}

int barrier(PierComm* c, cudaStream_t st) {
    if (c->vg) return vg_rendezvous(c, nullptr, st, nullptr);   // virtual group: host rendezvous + events
    if (c->nranks == 1) return PIER_OK;
    ncclResult_t r = ncclAllReduce(c->d_barrier, c->d_barrier, 1, ncclFloat, ncclSum, c->nccl, st);
    if (r != ncclSuccess) return set_error(PIER_ENCCL, std::string("p2p barrier: ") + ncclGetErrorString(r));
    return PIER_OK;
}

int comm_free_shared_all(PierComm* c) {
    for (auto& b : c->shared) shared_release(c, b);
    return PIER_OK;
}

int resolve_team(const PierComm* c, const int32_t* team, int32_t nteam, int32_t* members, int* n, int* r) {
    if (!team) {  // all ranks
        for (int i = 0; i < c->nranks; ++i) members[i] = i;
        *n = c->nranks;
        *r = c->rank;
        return PIER_OK;
    }
    if (nteam < 1 || nteam > c->nranks || nteam > PIER_MAX_RANKS) return set_error(PIER_EINVAL, "team: bad size");
    *r = -1;
    for (int i = 0; i < nteam; ++i) {
        if (team[i] < 0 || team[i] >= c->nranks || (i > 0 && team[i] <= team[i - 1]))
            return set_error(PIER_EINVAL, "team: ranks must be valid and strictly ascending");
        members[i] = team[i];
        if (team[i] == c->rank) *r = i;
    }
    if (*r < 0) return set_error(PIER_EINVAL, "team: the calling rank is not a member");
    *n = nteam;
    return PIER_OK;
}

// offset: element offset of the region [offset, offset + n_padded) of the
// shared buffer (a multiple of the span B*n); the shards point at the region's
// first slice
NormArgs norm_args(PierComm* c, NormWs* nws, const int32_t* members, int n) {
    NormArgs na;
    if (!nws) return na;
    na.ws = nws;
    for (int q = 0; q < n; ++q) na.slots.p[q] = (double*)c->shared[c->slots_id].peers[members[q]];
    return na;
}

// reps (optional, n entries): the rank whose copy stands in for member q in the fold --
// it must hold the same values (the dp replicas of one group); members sharing a source
// with the member before them are pulled once
int p2p_run(PierComm* c, int mode, int32_t id, float* anchor_shard, float* mom_shard, int64_t n_padded, int64_t B,
            double lr, double mu, void* stream, const int32_t* team = nullptr, int32_t nteam = 0,
            int64_t offset = 0, NormWs* nws = nullptr, double max_norm = 0.0, const int32_t* reps = nullptr) {
    if (!c || id < 0 || id >= (int)c->shared.size() || !c->shared[id].local)
        return set_error(PIER_EINVAL, "p2p: unknown shared buffer");
    // the fused norm of a team's mean is the clip norm only when the team's buffer is
    // the whole model (tp = 1): the replicated mean needs the whole communicator, the
    // sharded step (kP2pMeanOwn) may run over a dp team
    if (nws && (mode == kP2pOuter || (team && mode != kP2pMeanOwn) || !(max_norm > 0.0)))
        return set_error(PIER_EINVAL, "p2p: the fused norm needs the whole-communicator mean and clip_norm > 0");
    if (nws && c->slots_id < 0) return set_error(PIER_EINVAL, "p2p: communicator has no norm slots");
    const PierSharedBuf& sb = c->shared[id];   // (after any allocation: c->shared may have grown)
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4 || offset < 0 || offset % (B * n) ||
        (size_t)(offset + n_padded) * 4 > sb.bytes)
        return set_error(PIER_EINVAL, "p2p: n_padded must be a multiple of 4*nranks, the region span-aligned and "
                                      "inside the shared buffer");
    if (mode == kP2pOuter && (!anchor_shard || !mom_shard)) return set_error(PIER_EINVAL, "p2p: null shard");
    if (mode == kP2pOuter && (!aligned16(anchor_shard) || !aligned16(mom_shard)))
        return set_error(PIER_EINVAL, "p2p: shards must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    PeerTable pt{}, dt{};
    uint32_t dup = 0;
    for (int i = 0; i < n; ++i) {
        int src = members[i];
        if (reps) {
            if (reps[i] < 0 || reps[i] >= c->nranks) return set_error(PIER_EINVAL, "p2p: bad stand-in rank");
            src = reps[i];
            if (i > 0 && reps[i] == reps[i - 1]) dup |= 1u << i;
        }
        pt.p[i] = (float*)((g_flags & 1) ? sb.peers[src] : sb.local) + offset;
        dt.p[i] = (float*)((g_flags & 2) ? sb.peers[members[i]] : sb.local) + offset;
    }
    if (mode == kP2pMeanOwn) dt.p[0] = dt.p[r];
    // whole-communicator barrier (a superset of the team): every team of the
    // job runs its exchange at the same point of the step
    if (int e = barrier(c, st)) return e;
    const int ctas = mode == kP2pMeanOwn ? g_lazy_ctas_per_sm : g_ctas_per_sm;
    NormArgs outer_na;
    outer_na.dup = dup;
    int e = mode == kP2pOuter
                ? launch_p2p_n<kP2pOuter>(n, g_ctas_per_sm, st, pt, dt, n_padded, B, r, anchor_shard, mom_shard,
                                          (float)lr, (float)mu, outer_na)
            : mode == kP2pMeanOwn
                ? launch_p2p_n<kP2pMeanOwn>(n, ctas, st, pt, dt, n_padded, B, r, nullptr, nullptr, 0.f, 0.f,
                                            norm_args(c, nws, members, n))
                : launch_p2p_n<kP2pMean>(n, g_ctas_per_sm, st, pt, dt, n_padded, B, r, nullptr, nullptr, 0.f, 0.f,
                                         norm_args(c, nws, members, n));
    if (e) return e;
    if (int e2 = barrier(c, st)) return e2;
    if (nws) {   // every rank's share has landed in our slots
        k_norm_slots<<<1, 32, 0, st>>>((const double*)c->shared[c->slots_id].local, n, nws, max_norm);
        PIER_LAUNCH_CHECK("k_norm_slots");
    }
    return PIER_OK;
}

template <int NR>
void launch_mean_bf16(const BfTable& t, int64_t n_pad, int64_t B, int r, cudaStream_t st, const NormArgs& na,
                      bool own) {
    const int64_t nvec = n_pad / NR / 8;
    int grid = stream_grid(nvec, 1, own ? g_lazy_ctas_per_sm : g_ctas_per_sm);
    if (na.ws && grid > kMaxNormBlocks) grid = kMaxNormBlocks;   // one partial per CTA
    if (own) k_p2p_mean_bf16<NR, true><<<grid, kThreads, 0, st>>>(t, t.p[r], n_pad, B, r, na.ws, na.slots);
    else k_p2p_mean_bf16<NR, false><<<grid, kThreads, 0, st>>>(t, nullptr, n_pad, B, r, na.ws, na.slots);
}

// own: store the mean of this rank's slices only (the sharded lazy step, slices of
// every span of n*B elements); otherwise into every rank (one span of n_padded)
int mean_p2p_bf16(PierComm* c, int32_t buf_id, int64_t n_padded, NormWs* nws, double max_norm, void* stream,
                  bool own = false, int64_t B = 0) {
    if (!c || buf_id < 0 || buf_id >= (int)c->shared.size() || !c->shared[buf_id].local)
        return set_error(PIER_EINVAL, "allreduce_mean_p2p_bf16: unknown shared buffer");
    if (nws && (!(max_norm > 0.0) || c->slots_id < 0))
        return set_error(PIER_EINVAL, "allreduce_mean_norm_p2p_bf16: clip_norm > 0 and a communicator with slots");
    const PierSharedBuf& sb = c->shared[buf_id];
    const int n = c->nranks;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 8) || (size_t)n_padded * 2 > sb.bytes)
        return set_error(PIER_EINVAL, "allreduce_mean_p2p_bf16: n_padded must be a multiple of 8*nranks inside "
                                      "the shared buffer");
    cudaStream_t st = as_stream(stream);
    if (n == 1) {   // one group: the mean is the buffer itself; the fused norm is plain K4a
        if (nws) return pier_grad_sqnorm_bf16((const uint16_t*)sb.local, n_padded, max_norm, nws, stream);
        return PIER_OK;
    }
    BfTable t{};
    for (int q = 0; q < n; ++q) t.p[q] = (uint16_t*)sb.peers[q];
    int32_t members[PIER_MAX_RANKS];
    for (int q = 0; q < n; ++q) members[q] = q;
    const NormArgs na = norm_args(c, nws, members, n);
    if (!own || B <= 0) B = n_padded / n;
    if (B % 8) return set_error(PIER_EINVAL, "allreduce_mean_p2p_bf16: bucket_elems must be a multiple of 8");
    if (int e = barrier(c, st)) return e;
    switch (n) {
        case 2: launch_mean_bf16<2>(t, n_padded, B, c->rank, st, na, own); break;
        case 3: launch_mean_bf16<3>(t, n_padded, B, c->rank, st, na, own); break;
        case 4: launch_mean_bf16<4>(t, n_padded, B, c->rank, st, na, own); break;
        case 5: launch_mean_bf16<5>(t, n_padded, B, c->rank, st, na, own); break;
        case 6: launch_mean_bf16<6>(t, n_padded, B, c->rank, st, na, own); break;
        case 7: launch_mean_bf16<7>(t, n_padded, B, c->rank, st, na, own); break;
        default: launch_mean_bf16<8>(t, n_padded, B, c->rank, st, na, own); break;
    }
    PIER_LAUNCH_CHECK("k_p2p_mean_bf16");
    if (int e = barrier(c, st)) return e;
    if (nws) {   // every rank's share has landed in our slots: add them in rank order
        k_norm_slots<<<1, 32, 0, st>>>((const double*)c->shared[c->slots_id].local, n, nws, max_norm);
        PIER_LAUNCH_CHECK("k_norm_slots");
    }
    return PIER_OK;
}

// ---- Lazy phase, sharded (driver.py:380-399 for t <= lazy_end) ---------------
// In the lazy phase every replica holds the same theta, m and v and applies
// the same averaged gradient, so the AdamW pass need not run n times: rank r
// updates only ITS shard -- its B-slice of every span of n*B elements (the
// layout of the outer exchange) -- and broadcasts the new theta.
//   1. reduce-scatter: k_p2p_reduce<kP2pMeanOwn> pulls slice r of every span of
//      every rank's gradient, folds in ascending rank order (topology.py:113-121)
//      into this rank's gradient buffer, and sums the squares of the means;
//   2. the ranks' square sums are added in rank order (k_norm_slots) -> the
//      clip record, identical on every rank (optim.py:70-79);
//   3. k_lazy_adamw_push: AdamW (optim.py:94-102) on the shard with the clipped
//      mean, m / v updated in place, the new theta stored into EVERY rank's
//      buffer (the all-gather).
// Bitwise what every replica computes in the reference; the same wire bytes
// as the all-reduce + replicated AdamW (2(n-1)/n * 4N per direction), but the
// 28 B/param AdamW pass shrinks to 28/n B/param and runs under the
// all-gather's NVLink time instead of after it.  m and v of the other slices
// are left stale; pier_gather_p2p_f32 brings them back (once, when the groups
// diverge after the lazy phase).  Overlapped with the backward pass, step 1
// becomes copy-engine pulls of every completed span into a local staging
// buffer (no SMs taken from the backward) and a local fold at the end.

// every W-float vector of rank r's shard: f(e, s) with e its index in the
// buffer and s its index in the shard (the concatenated slices); grid-stride
// within each span of NR*B elements (the last one shorter)
template <int NR, int W, typename F>
__device__ __forceinline__ void for_own_slices(int64_t n_pad, int64_t B, int r, F&& f) {
    const int64_t span = B * NR;
    int64_t sh = 0;
    for (int64_t off = 0; off < n_pad; off += span) {
        const int64_t len = (n_pad - off) < span ? (n_pad - off) : span;
        const int64_t nv = len / NR / W, base = (off + (int64_t)r * (len / NR)) / W;
        for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nv; i += (int64_t)gridDim.x * kThreads)
            f(base + i, sh + i);
        sh += nv;
    }
}

// push = false: the new theta stays in this rank's buffer (the deferred all-gather
// pulls it with the copy engines, span by span, behind the next forward)
template <int NR, typename VT>
__global__ void __launch_bounds__(kThreads) k_lazy_adamw_push(PeerTable th, VT* __restrict__ own,
                                                               const VT* __restrict__ g, VT* __restrict__ m,
                                                               VT* __restrict__ v, int64_t n_pad, int64_t B, int r,
                                                               const AdamC<float> c, const NormWs* ws, bool push) {
    constexpr int W = sizeof(VT) / sizeof(float);
    const float s = load_scale<float>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for_own_slices<NR, W>(n_pad, B, r, [&](int64_t e, int64_t) {
        VT a = ld_stream(own + e), gg = ld_stream(g + e), mm = ld_stream(m + e), vv = ld_stream(v + e);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            float x = lane(gg, w);
            if (clip) x = mul_rn(x, s);                                                    // optim.py:78
            adamw_lane<float>(lane(a, w), x, lane(mm, w), lane(vv, w), c);
        }
        st_stream(m + e, mm);
        st_stream(v + e, vv);
        if (push) {
#pragma unroll
            for (int q = 0; q < NR; ++q) st_cg(reinterpret_cast<VT*>(th.p[q]) + e, a);    // every replica's theta
        } else {
            st_cg(own + e, a);
        }
    });
    __threadfence_system();
}

// all-gather of a shard-sharded buffer: rank r stores its shard into every peer
template <int NR, typename VT>
__global__ void __launch_bounds__(kThreads) k_p2p_push_own(PeerTable buf, const VT* __restrict__ own, int64_t n_pad,
                                                            int64_t B, int r) {
    constexpr int W = sizeof(VT) / sizeof(float);
    for_own_slices<NR, W>(n_pad, B, r, [&](int64_t e, int64_t) {
        const VT x = ld_stream(own + e);
#pragma unroll
        for (int q = 0; q < NR; ++q)
            if (q != r) st_cg(reinterpret_cast<VT*>(buf.p[q]) + e, x);
    });
    __threadfence_system();
}

// the overlapped form's reduce: every rank's copy of our shard sits in the local
// staging buffer (rank q's at q * shard_len, copy-engine pulls) except our own,
// read in place; fold in ascending rank order, store the mean over our shard of
// the gradient and post our square sum into every rank's slot r (as k_p2p_reduce)
template <int NR, typename VT>
__global__ void __launch_bounds__(kThreads) k_fold_staged(VT* __restrict__ g, const VT* __restrict__ staging,
                                                           int64_t shard_v, int64_t n_pad, int64_t B, int r,
                                                           NormWs* nws, SlotTable slots) {
    constexpr int W = sizeof(VT) / sizeof(float);
    const float nf = (float)NR;
    double sq = 0.0;
    for_own_slices<NR, W>(n_pad, B, r, [&](int64_t e, int64_t s) {
        VT x[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) x[q] = q == r ? ld_stream(g + e) : ld_stream(staging + (int64_t)q * shard_v + s);
        VT out;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            float acc = lane(x[0], w);
#pragma unroll
            for (int q = 1; q < NR; ++q) acc = add_rn(acc, lane(x[q], w));                 // topology.py:113-120
            const float av = div_rn(acc, nf);                                               // topology.py:121
            lane(out, w) = av;
            sq += (double)av * (double)av;
        }
        st_stream(g + e, out);
    });
    double total;
    if (norm_sum_last(nws, sq, &total))
        for (int q = 0; q < NR; ++q) slots.p[q][r] = total;   // this rank's share, to every rank
    __threadfence_system();
}

template <int NR, typename VT>
void launch_lazy_vt(int kind, cudaStream_t st, const PeerTable& b, const float* g, float* m, float* v,
                    int64_t n_pad, int64_t B, int r, const AdamC<float>& c, const NormWs* ws, bool push) {
    constexpr int W = sizeof(VT) / sizeof(float);
    const int grid = stream_grid(n_pad / NR / W, 1, g_lazy_ctas_per_sm);
    if (kind == 0)
        k_lazy_adamw_push<NR, VT><<<grid, kThreads, 0, st>>>(b, (VT*)b.p[r], (const VT*)g, (VT*)m, (VT*)v,
                                                             n_pad, B, r, c, ws, push);
    else
        k_p2p_push_own<NR, VT><<<grid, kThreads, 0, st>>>(b, (const VT*)b.p[r], n_pad, B, r);
}

// kind 0: lazy AdamW + push, 1: gather; 256-bit vectors when every address allows
template <int NR>
void launch_lazy_kind(int kind, bool wide, cudaStream_t st, const PeerTable& b, const float* g, float* m, float* v,
                      int64_t n_pad, int64_t B, int r, const AdamC<float>& c, const NormWs* ws, bool push) {
    if (wide) launch_lazy_vt<NR, F8>(kind, st, b, g, m, v, n_pad, B, r, c, ws, push);
    else launch_lazy_vt<NR, float4>(kind, st, b, g, m, v, n_pad, B, r, c, ws, push);
}

int launch_lazy(int kind, int n, bool wide, cudaStream_t st, const PeerTable& b, const float* g, float* m, float* v,
                int64_t n_pad, int64_t B, int r, const AdamC<float>& c = AdamC<float>(),
                const NormWs* ws = nullptr, bool push = true) {
    switch (n) {
        case 2: launch_lazy_kind<2>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 3: launch_lazy_kind<3>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 4: launch_lazy_kind<4>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 5: launch_lazy_kind<5>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 6: launch_lazy_kind<6>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 7: launch_lazy_kind<7>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        case 8: launch_lazy_kind<8>(kind, wide, st, b, g, m, v, n_pad, B, r, c, ws, push); break;
        default: return set_error(PIER_EINVAL, "lazy step: 2..8 ranks");
    }
    PIER_LAUNCH_CHECK(kind == 0 ? "k_lazy_adamw_push" : "k_p2p_push_own");
    return PIER_OK;
}

template <int NR>
void launch_fold_staged_n(bool wide, cudaStream_t st, float* g, const float* staging, int64_t n_pad, int64_t B, int r,
                          const NormArgs& na) {
    const int64_t shard = n_pad / NR;
    if (wide) {
        int grid = stream_grid(shard / 8, 1, g_lazy_ctas_per_sm);
        if (grid > kMaxNormBlocks) grid = kMaxNormBlocks;   // one partial per CTA
        k_fold_staged<NR, F8><<<grid, kThreads, 0, st>>>((F8*)g, (const F8*)staging, shard / 8, n_pad, B, r, na.ws,
                                                          na.slots);
    } else {
        int grid = stream_grid(shard / 4, 1, g_lazy_ctas_per_sm);
        if (grid > kMaxNormBlocks) grid = kMaxNormBlocks;
        k_fold_staged<NR, float4><<<grid, kThreads, 0, st>>>((float4*)g, (const float4*)staging, shard / 4, n_pad, B,
                                                              r, na.ws, na.slots);
    }
}

int launch_fold_staged(int n, bool wide, cudaStream_t st, float* g, const float* staging, int64_t n_pad, int64_t B,
                       int r, const NormArgs& na) {
    switch (n) {
        case 2: launch_fold_staged_n<2>(wide, st, g, staging, n_pad, B, r, na); break;
        case 3: launch_fold_staged_n<3>(wide, st, g, staging, n_pad, B, r, na); break;
        case 4: launch_fold_staged_n<4>(wide, st, g, staging, n_pad, B, r, na); break;
        case 5: launch_fold_staged_n<5>(wide, st, g, staging, n_pad, B, r, na); break;
        case 6: launch_fold_staged_n<6>(wide, st, g, staging, n_pad, B, r, na); break;
        case 7: launch_fold_staged_n<7>(wide, st, g, staging, n_pad, B, r, na); break;
        case 8: launch_fold_staged_n<8>(wide, st, g, staging, n_pad, B, r, na); break;
        default: return set_error(PIER_EINVAL, "lazy fold: 2..8 ranks");
    }
    PIER_LAUNCH_CHECK("k_fold_staged");
    return PIER_OK;
}

// The 7B recipe's sharded lazy step (bf16 live params and gradients, fp32 master /
// m / v): AdamW on this rank's shard of the master with the clipped bf16 mean
// (as k_adamw_bf16: widen exactly, scale in fp32, optim.py:94-102), the master,
// m, v stored locally (the other slices go stale until pier_gather_p2p_f32),
// the RNE bf16 of the new master pushed into EVERY rank's live params.
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&b);
}

template <int NR>
__global__ void __launch_bounds__(kThreads) k_lazy_adamw_push_bf16(BfTable live, F8* __restrict__ master,
                                                                    const uint4* __restrict__ g16, F8* __restrict__ m,
                                                                    F8* __restrict__ v, int64_t n_pad, int64_t B,
                                                                    int r, const AdamC<float> c, const NormWs* ws) {
    const float s = load_scale<float>(ws);
    const bool clip = ws != nullptr && ws->res.clipped;
    for_own_slices<NR, 8>(n_pad, B, r, [&](int64_t e, int64_t) {   // 8 params per vector
        F8 a = ld_stream(master + e), mm = ld_stream(m + e), vv = ld_stream(v + e);
        const uint4 gb = __ldcs(g16 + e);
        const uint32_t* gw = &gb.x;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            float gf = __uint_as_float((w & 1) ? (gw[w >> 1] & 0xffff0000u) : (gw[w >> 1] << 16));
            if (clip) gf = mul_rn(gf, s);                                                   // optim.py:78
            adamw_lane<float>(lane(a, w), gf, lane(mm, w), lane(vv, w), c);
        }
        st_stream(master + e, a);
        st_stream(m + e, mm);
        st_stream(v + e, vv);
        uint4 o;
        o.x = bf16x2_rn(a.lo.x, a.lo.y);
        o.y = bf16x2_rn(a.lo.z, a.lo.w);
        o.z = bf16x2_rn(a.hi.x, a.hi.y);
        o.w = bf16x2_rn(a.hi.z, a.hi.w);
#pragma unroll
        for (int q = 0; q < NR; ++q) __stcg(reinterpret_cast<uint4*>(live.p[q]) + e, o);   // every replica's live params
    });
    __threadfence_system();
}

template <int NR>
void launch_lazy_bf16(cudaStream_t st, const BfTable& live, float* master, const uint16_t* g16, float* m, float* v,
                      int64_t n_pad, int64_t B, int r, const AdamC<float>& c, const NormWs* ws) {
    k_lazy_adamw_push_bf16<NR><<<stream_grid(n_pad / NR / 8, 1, g_lazy_ctas_per_sm), kThreads, 0, st>>>(
        live, (F8*)master, (const uint4*)g16, (F8*)m, (F8*)v, n_pad, B, r, c, ws);
}

// the 7B recipe's overlapped reduce: member q's bf16 copy of our shard sits in
// `staging` at q * shard (copy-engine pulls), our own is read in place; fp32 left
// fold of the bf16 values, one RNE rounding (as k_p2p_mean_bf16), the rounded mean
// stored over our shard of the gradient, its square sum posted to every rank's slot r
template <int NR>
__global__ void __launch_bounds__(kThreads) k_fold_staged_bf16(uint4* __restrict__ g16,
                                                                const uint4* __restrict__ staging, int64_t shard_v,
                                                                int64_t n_pad, int64_t B, int r, NormWs* nws,
                                                                SlotTable slots) {
    const float nf = (float)NR;
    double sq = 0.0;
    for_own_slices<NR, 8>(n_pad, B, r, [&](int64_t e, int64_t s) {
        uint4 x[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) x[q] = q == r ? __ldcs(g16 + e) : __ldcs(staging + (int64_t)q * shard_v + s);
        uint4 out;
        uint32_t* ow = &out.x;
#pragma unroll
        for (int w = 0; w < 4; ++w) {   // word w: element 2w in the low half, 2w+1 in the high half
            float lo = bf_lo((&x[0].x)[w]), hi = bf_hi((&x[0].x)[w]);
#pragma unroll
            for (int q = 1; q < NR; ++q) {
                lo = add_rn(lo, bf_lo((&x[q].x)[w]));                                       // topology.py:113-120
                hi = add_rn(hi, bf_hi((&x[q].x)[w]));
            }
            const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(div_rn(lo, nf)));   // topology.py:121
            const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(div_rn(hi, nf)));
            ow[w] = l | (h << 16);
            const double a = (double)__uint_as_float(l << 16), b = (double)__uint_as_float(h << 16);
            sq += a * a;
            sq += b * b;
        }
        __stcs(g16 + e, out);
    });
    double total;
    if (norm_sum_last(nws, sq, &total))
        for (int q = 0; q < NR; ++q) slots.p[q][r] = total;   // this rank's share, to every rank
    __threadfence_system();
}

int launch_fold_staged_bf16(int n, cudaStream_t st, uint16_t* g16, const uint16_t* staging, int64_t n_pad,
                            int64_t B, int r, const NormArgs& na) {
    const int64_t shard_v = n_pad / n / 8;
    int grid = stream_grid(shard_v, 1, g_lazy_ctas_per_sm);
    if (grid > kMaxNormBlocks) grid = kMaxNormBlocks;   // one partial per CTA
    uint4* g = (uint4*)g16;
    const uint4* sg = (const uint4*)staging;
    switch (n) {
        case 2: k_fold_staged_bf16<2><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 3: k_fold_staged_bf16<3><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 4: k_fold_staged_bf16<4><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 5: k_fold_staged_bf16<5><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 6: k_fold_staged_bf16<6><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 7: k_fold_staged_bf16<7><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        case 8: k_fold_staged_bf16<8><<<grid, kThreads, 0, st>>>(g, sg, shard_v, n_pad, B, r, na.ws, na.slots); break;
        default: return set_error(PIER_EINVAL, "lazy fold bf16: 2..8 ranks");
    }
    PIER_LAUNCH_CHECK("k_fold_staged_bf16");
    return PIER_OK;
}

// the bf16 AdamW + push of the live params over n ranks (step 3 of the 7B recipe's sharded step)
int lazy_adamw_push_bf16(PierComm* c, const PierSharedBuf* lb, float* master, const uint16_t* g16, float* m, float* v,
                         int64_t n_padded, int64_t B, const PierAdamW* hp, void* clip_ws, void* stream) {
    const int n = c->nranks, r = c->rank;
    cudaStream_t st = as_stream(stream);
    BfTable live{};
    for (int q = 0; q < n; ++q) live.p[q] = (uint16_t*)lb->peers[q];
    const AdamC<float> ac = adam_consts<float>(*hp);
    const NormWs* ws = (const NormWs*)clip_ws;
    switch (n) {
        case 2: launch_lazy_bf16<2>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        case 3: launch_lazy_bf16<3>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        case 4: launch_lazy_bf16<4>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        case 5: launch_lazy_bf16<5>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        case 6: launch_lazy_bf16<6>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        case 7: launch_lazy_bf16<7>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
        default: launch_lazy_bf16<8>(st, live, master, g16, m, v, n_padded, B, r, ac, ws); break;
    }
    PIER_LAUNCH_CHECK("k_lazy_adamw_push_bf16");
    return barrier(c, st);
}

// AdamW on this rank's shard + all-gather of theta (step 3 of the sharded lazy
// step), then every push has landed
int lazy_adamw_push(PierComm* c, const PierSharedBuf* tb, const PierSharedBuf* gb, const int32_t* members, int n,
                    int r, float* m, float* v, int64_t n_padded, int64_t B, const PierAdamW* hp, void* clip_ws,
                    void* stream, bool push = true) {
    cudaStream_t st = as_stream(stream);
    PeerTable th{};
    bool wide = n_padded % (8 * n) == 0 && B % 8 == 0 && aligned32(m) && aligned32(v) && aligned32(gb->local);
    for (int q = 0; q < n; ++q) {
        th.p[q] = (float*)tb->peers[members[q]];
        wide = wide && aligned32(th.p[q]);
    }
    if (int e = launch_lazy(0, n, wide, st, th, (const float*)gb->local, m, v, n_padded, B, r,
                            adam_consts<float>(*hp), (const NormWs*)clip_ws, push))
        return e;
    return barrier(c, st);   // pushed: every push landed / deferred: every shard is final
}

// the lazy layout's bucket: B > 0 (a multiple of 4, of 8 for 256-bit access) or
// 0 = one span (the contiguous 1/n slices)
int lazy_bucket(int64_t n_padded, int n, int64_t* B) {
    if (*B == 0) *B = n_padded / n;
    if (*B <= 0 || *B % 4) return set_error(PIER_EINVAL, "lazy step: bucket_elems must be a positive multiple of 4");
    return PIER_OK;
}

const PierSharedBuf* shared_buf(PierComm* c, int32_t id) {
    if (!c || id < 0 || id >= (int)c->shared.size() || !c->shared[id].local) return nullptr;
    return &c->shared[id];
}

}  // namespace pier

using namespace pier;

extern "C" {

int pier_allreduce_mean_p2p_bf16(PierComm* c, int32_t buf_id, int64_t n_padded, void* stream) {
    return mean_p2p_bf16(c, buf_id, n_padded, nullptr, 0.0, stream);
}

int pier_allreduce_mean_norm_p2p_bf16(PierComm* c, int32_t buf_id, int64_t n_padded, double max_norm,
                                      void* clip_ws, void* stream) {
    if (!clip_ws) return set_error(PIER_EINVAL, "allreduce_mean_norm_p2p_bf16: null workspace");
    return mean_p2p_bf16(c, buf_id, n_padded, (NormWs*)clip_ws, max_norm, stream);
}

int pier_norm_allreduce_team(PierComm* c, const int32_t* team, int32_t nteam, void* ws, double max_norm,
                             void* stream) {
    if (!c || !ws || !(max_norm > 0.0)) return set_error(PIER_EINVAL, "norm_allreduce_team: bad args");
    if (c->slots_id < 0) return set_error(PIER_EINVAL, "norm_allreduce_team: communicator has no norm slots");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    cudaStream_t st = as_stream(stream);
    SlotTable dst{};
    for (int q = 0; q < n; ++q) dst.p[q] = (double*)c->shared[c->slots_id].peers[members[q]] + PIER_MAX_RANKS;
    // barrier first: every member consumed the slots of the previous call
    if (int e = barrier(c, st)) return e;
    k_slot_put<<<1, 32, 0, st>>>(dst, r, n, (const NormWs*)ws);
    PIER_LAUNCH_CHECK("k_slot_put");
    if (int e = barrier(c, st)) return e;
    k_norm_slots<<<1, 32, 0, st>>>((const double*)c->shared[c->slots_id].local + PIER_MAX_RANKS, n, (NormWs*)ws,
                                    max_norm);
    PIER_LAUNCH_CHECK("k_norm_slots");
    return PIER_OK;
}

int pier_p2p_tune(int ctas_per_sm, int unroll, int flags) {
    if (ctas_per_sm > 0) g_ctas_per_sm = g_lazy_ctas_per_sm = ctas_per_sm;
    if (unroll >= 0) g_unroll = unroll;
    if (flags >= 0) g_flags = flags & 3;
    return PIER_OK;
}

int pier_round_tune(int adamw_ctas_per_sm, int p2p_ctas_per_sm) {
    if (adamw_ctas_per_sm > 0) g_round_adamw_ctas = adamw_ctas_per_sm;
    if (p2p_ctas_per_sm > 0) g_round_p2p_ctas = p2p_ctas_per_sm;
    return PIER_OK;
}

int pier_round_p2p_f32(PierComm* c, int32_t theta_id, const float* g, float* m, float* v, float* anchor_shard,
                       float* mom_shard, int64_t n_padded, int64_t B, const PierAdamW* hp, const void* clip_ws,
                       double lr, double mu, void* stream) {
    if (!c || theta_id < 0 || theta_id >= (int)c->shared.size() || !c->shared[theta_id].local)
        return set_error(PIER_EINVAL, "round_p2p: unknown shared buffer");
    if (!g || !m || !v || !anchor_shard || !mom_shard || !hp) return set_error(PIER_EINVAL, "round_p2p: null");
    const PierSharedBuf& sb = c->shared[theta_id];
    const int n = c->nranks, r = c->rank;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4 || (size_t)n_padded * 4 > sb.bytes)
        return set_error(PIER_EINVAL, "round_p2p: bad n_padded / bucket");
    cudaStream_t st = as_stream(stream);
    if (!c->ps) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        PIER_CHECK_CUDA(cudaStreamCreateWithPriority(&c->ps, cudaStreamNonBlocking, hi));
    }
    float* theta = (float*)sb.local;
    PeerTable pt{}, dt{};
    for (int i = 0; i < n; ++i) pt.p[i] = dt.p[i] = (float*)sb.peers[i];
    const int64_t span = B * n;
    const int64_t nspans = (n_padded + span - 1) / span;
    while ((int64_t)c->ev_rs.size() < nspans) {
        cudaEvent_t e;
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_rs.push_back(e);
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_k3.push_back(e);
    }
    int64_t sh = 0, b = 0;
    for (int64_t off = 0; off < n_padded; off += span, ++b) {
        int64_t len = (n_padded - off) < span ? (n_padded - off) : span;
        int64_t slice = len / n;
        // this group's inner AdamW on the whole span (driver.py:395-399), on a
        // reduced grid so the exchange kernels find free SMs ...
        int saved = default_ctas_per_sm();
        default_ctas_per_sm() = g_round_adamw_ctas;
        int ea = pier_adamw_f32(theta + off, g + off, m + off, v + off, len, hp, clip_ws, stream);
        default_ctas_per_sm() = saved;
        if (ea) return ea;
        PIER_CHECK_CUDA(cudaEventRecord(c->ev_rs[b], st));
        // ... then, on the exchange stream, once every rank finished that span:
        // pull-fold-update-push (overlaps the AdamW of the next span)
        PIER_CHECK_CUDA(cudaStreamWaitEvent(c->ps, c->ev_rs[b], 0));
        if (int e = barrier(c, c->ps)) return e;
        PeerTable pb{}, db{};  // this span only: a one-span buffer of len elements
        for (int q = 0; q < n; ++q) {
            pb.p[q] = pt.p[q] + off;
            db.p[q] = dt.p[q] + off;
        }
        if (int e = launch_p2p_n<kP2pOuter>(n, g_round_p2p_ctas, c->ps, pb, db, len, slice, r, anchor_shard + sh,
                                            mom_shard + sh, (float)lr, (float)mu))
            return e;
        sh += slice;
    }
    if (int e = barrier(c, c->ps)) return e;
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->ps));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

int pier_comm_alloc_shared(PierComm* c, size_t bytes, void** out_local, int32_t* out_id) {
    if (!c || !out_local || !out_id || bytes == 0) return set_error(PIER_EINVAL, "alloc_shared: bad args");
    if (c->nranks > PIER_MAX_RANKS) return set_error(PIER_EINVAL, "alloc_shared: at most 8 ranks");
    if (!c->d_barrier) {
        PIER_CHECK_CUDA(cudaMalloc(&c->d_barrier, 256));
        PIER_CHECK_CUDA(cudaMemset(c->d_barrier, 0, 256));
    }
    PierSharedBuf b;
    b.bytes = bytes;
    PIER_CHECK_CUDA(cudaMalloc(&b.local, bytes));
    PIER_CHECK_CUDA(cudaMemset(b.local, 0, bytes));
    b.peers[c->rank] = b.local;
    if (c->vg) {
        // virtual group: the peers are the other ranks' allocations on this device;
        // the rendezvous orders every rank's zero-fill before anyone's later work
        void* ptrs[PIER_MAX_RANKS] = {};
        if (int e = vg_rendezvous(c, b.local, nullptr, nullptr, ptrs)) {
            cudaFree(b.local);
            return e;
        }
        for (int r = 0; r < c->nranks; ++r) b.peers[r] = ptrs[r];
        c->shared.push_back(b);
        *out_local = b.local;
        *out_id = (int32_t)c->shared.size() - 1;
        return PIER_OK;
    }
    if (c->nranks > 1) {
        cudaIpcMemHandle_t h;
        PIER_CHECK_CUDA(cudaIpcGetMemHandle(&h, b.local));
        const size_t hs = sizeof(cudaIpcMemHandle_t);
        char* d = nullptr;
        PIER_CHECK_CUDA(cudaMalloc(&d, hs * c->nranks));
        PIER_CHECK_CUDA(cudaMemcpy(d + hs * c->rank, &h, hs, cudaMemcpyHostToDevice));
        ncclResult_t rr = ncclAllGather(d + hs * c->rank, d, hs, ncclChar, c->nccl, c->cs);
        if (rr != ncclSuccess) {
            cudaFree(d);
            return set_error(PIER_ENCCL, std::string("alloc_shared allgather: ") + ncclGetErrorString(rr));
        }
        PIER_CHECK_CUDA(cudaStreamSynchronize(c->cs));
        std::vector<cudaIpcMemHandle_t> all(c->nranks);
        PIER_CHECK_CUDA(cudaMemcpy(all.data(), d, hs * c->nranks, cudaMemcpyDeviceToHost));
        cudaFree(d);
        for (int r = 0; r < c->nranks; ++r) {
            if (r == c->rank) continue;
            PIER_CHECK_CUDA(cudaIpcOpenMemHandle(&b.peers[r], all[r], cudaIpcMemLazyEnablePeerAccess));
        }
    }
    // stream-ordered zero-fill finished everywhere before anyone uses the buffer
    PIER_CHECK_CUDA(cudaDeviceSynchronize());
    c->shared.push_back(b);
    *out_local = b.local;
    *out_id = (int32_t)c->shared.size() - 1;
    return PIER_OK;
}

int pier_comm_free_shared(PierComm* c, int32_t id) {
    if (!c || id < 0 || id >= (int)c->shared.size()) return set_error(PIER_EINVAL, "free_shared: bad id");
    PierSharedBuf& b = c->shared[id];
    if (!b.local) return PIER_OK;
    cudaDeviceSynchronize();
    shared_release(c, b);
    return PIER_OK;
}

int pier_outer_step_p2p_f32(PierComm* c, int32_t theta_id, float* anchor_shard, float* mom_shard,
                            int64_t n_padded, int64_t B, double lr, double mu, void* stream) {
    return p2p_run(c, kP2pOuter, theta_id, anchor_shard, mom_shard, n_padded, B, lr, mu, stream);
}

int pier_p2p_virtual_f32(int32_t n, int32_t outer, float* const* buf, float* const* anchor_shards,
                         float* const* mom_shards, int64_t n_padded, int64_t B, double lr, double mu,
                         void* const* streams) {
    if (n < 1 || n > PIER_MAX_RANKS || !buf || !streams || (outer && (!anchor_shards || !mom_shards)))
        return set_error(PIER_EINVAL, "p2p_virtual: 1..8 virtual ranks and non-null tables");
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4)
        return set_error(PIER_EINVAL, "p2p_virtual: bad n_padded / bucket");
    PeerTable pt{};
    for (int q = 0; q < n; ++q) {
        if (!buf[q]) return set_error(PIER_EINVAL, "p2p_virtual: null buffer");
        pt.p[q] = buf[q];
    }
    // slices are disjoint: rank r pulls and pushes only its own slice of every
    // span, so the n launches may run concurrently once all inputs are final
    for (int r = 0; r < n; ++r) {
        cudaStream_t st = as_stream(streams[r]);
        int e = outer ? launch_p2p_n<kP2pOuter>(n, g_ctas_per_sm, st, pt, pt, n_padded, B, r, anchor_shards[r],
                                                mom_shards[r], (float)lr, (float)mu)
                      : launch_p2p_n<kP2pMean>(n, g_ctas_per_sm, st, pt, pt, n_padded, B, r, nullptr, nullptr, 0.f,
                                               0.f);
        if (e) return e;
    }
    return PIER_OK;
}

int pier_outer_step_p2p_reps_f32(PierComm* c, int32_t theta_id, const int32_t* team, int32_t nteam,
                                 const int32_t* reps, float* anchor_shard, float* mom_shard, int64_t n_padded,
                                 int64_t B, double lr, double mu, void* stream) {
    if (!reps) return set_error(PIER_EINVAL, "outer_step_p2p_reps: null stand-in table");
    return p2p_run(c, kP2pOuter, theta_id, anchor_shard, mom_shard, n_padded, B, lr, mu, stream, team, nteam, 0,
                   nullptr, 0.0, reps);
}

int pier_outer_step_p2p_region_f32(PierComm* c, int32_t theta_id, int64_t offset, int64_t len, float* anchor_shard,
                                   float* mom_shard, int64_t B, double lr, double mu, void* stream) {
    return p2p_run(c, kP2pOuter, theta_id, anchor_shard, mom_shard, len, B, lr, mu, stream, nullptr, 0, offset);
}

int pier_outer_step_p2p_team_f32(PierComm* c, int32_t theta_id, const int32_t* team, int32_t nteam,
                                 float* anchor_shard, float* mom_shard, int64_t n_padded, int64_t B, double lr,
                                 double mu, void* stream) {
    if (!team) return set_error(PIER_EINVAL, "outer_step_p2p_team: null team");
    return p2p_run(c, kP2pOuter, theta_id, anchor_shard, mom_shard, n_padded, B, lr, mu, stream, team, nteam);
}

int pier_allreduce_mean_p2p_team_f32(PierComm* c, int32_t buf_id, const int32_t* team, int32_t nteam,
                                     int64_t n_padded, void* stream) {
    if (!team || nteam < 1) return set_error(PIER_EINVAL, "allreduce_mean_p2p_team: null team");
    int64_t slice = n_padded / nteam;
    return p2p_run(c, kP2pMean, buf_id, nullptr, nullptr, n_padded, slice > 0 ? slice : 4, 0.0, 0.0, stream, team,
                   nteam);
}

int pier_allreduce_mean_norm_p2p_f32(PierComm* c, int32_t buf_id, int64_t n_padded, double max_norm, void* clip_ws,
                                     void* stream) {
    if (!clip_ws) return set_error(PIER_EINVAL, "allreduce_mean_norm_p2p: null workspace");
    int64_t slice = c ? n_padded / (c->nranks > 0 ? c->nranks : 1) : 0;
    return p2p_run(c, kP2pMean, buf_id, nullptr, nullptr, n_padded, slice > 0 ? slice : 4, 0.0, 0.0, stream, nullptr,
                   0, 0, (NormWs*)clip_ws, max_norm);
}

int pier_allreduce_mean_p2p_f32(PierComm* c, int32_t buf_id, int64_t n_padded, void* stream) {
    // one span per rank: the mean needs no shard layout
    int64_t slice = c ? n_padded / (c->nranks > 0 ? c->nranks : 1) : 0;
    return p2p_run(c, kP2pMean, buf_id, nullptr, nullptr, n_padded, slice > 0 ? slice : 4, 0.0, 0.0, stream);
}

int pier_lazy_step_p2p_team_f32(PierComm* c, int32_t theta_id, int32_t grad_id, const int32_t* team, int32_t nteam,
                                const int32_t* norm_team, int32_t n_norm_team, float* m, float* v, int64_t n_padded,
                                int64_t bucket_elems, const PierAdamW* hp, double max_norm, void* clip_ws,
                                void* stream) {
    const PierSharedBuf* tb = shared_buf(c, theta_id);
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!tb || !gb || theta_id == grad_id) return set_error(PIER_EINVAL, "lazy_step_p2p: unknown shared buffers");
    if (!m || !v || !hp || !clip_ws || !(max_norm > 0.0)) return set_error(PIER_EINVAL, "lazy_step_p2p: bad args");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n < 2) return set_error(PIER_EINVAL, "lazy_step_p2p: needs 2..8 ranks (one group: pier_adamw_f32)");
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > tb->bytes ||
        (size_t)n_padded * 4 > gb->bytes)
        return set_error(PIER_EINVAL, "lazy_step_p2p: n_padded must be a multiple of 4*nranks inside the buffers");
    if (!aligned16(m) || !aligned16(v)) return set_error(PIER_EINVAL, "lazy_step_p2p: m, v must be 16-byte aligned");
    if (c->slots_id < 0) return set_error(PIER_EINVAL, "lazy_step_p2p: communicator has no norm slots");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    // 1-2: reduce-scatter of the gradient with the norm of the mean -> clip record on every member
    if (int e = p2p_run(c, kP2pMeanOwn, grad_id, nullptr, nullptr, n_padded, B, 0.0, 0.0, stream, team, nteam, 0,
                        (NormWs*)clip_ws, max_norm))
        return e;
    // tensor parallelism: the other shards of this replica add their square sums -> the global norm
    if (norm_team)
        if (int e = pier_norm_allreduce_team(c, norm_team, n_norm_team, clip_ws, max_norm, stream)) return e;
    // 3: AdamW on this rank's shard + all-gather of theta
    return lazy_adamw_push(c, tb, gb, members, n, r, m, v, n_padded, B, hp, clip_ws, stream);
}

int pier_lazy_step_p2p_f32(PierComm* c, int32_t theta_id, int32_t grad_id, float* m, float* v, int64_t n_padded,
                           int64_t bucket_elems, const PierAdamW* hp, double max_norm, void* clip_ws, void* stream) {
    return pier_lazy_step_p2p_team_f32(c, theta_id, grad_id, nullptr, 0, nullptr, 0, m, v, n_padded, bucket_elems,
                                       hp, max_norm, clip_ws, stream);
}

int pier_lazy_pull_span_p2p_f32(PierComm* c, int32_t grad_id, const int32_t* team, int32_t nteam, float* staging,
                                int64_t n_padded, int64_t bucket_elems, int32_t span, void* stream) {
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!gb || !staging) return set_error(PIER_EINVAL, "lazy_pull_span_p2p: unknown buffer / null staging");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n < 2 || n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > gb->bytes)
        return set_error(PIER_EINVAL, "lazy_pull_span_p2p: 2..8 ranks, n_padded a multiple of 4*nranks");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    const int64_t sp = B * n, off = (int64_t)span * sp;
    if (span < 0 || off >= n_padded) return set_error(PIER_EINVAL, "lazy_pull_span_p2p: span out of range");
    const int64_t len = (n_padded - off) < sp ? (n_padded - off) : sp, slice = len / n;
    cudaStream_t st = as_stream(stream);
    // every rank's gradient of this span is final (whole-communicator barrier: every team
    // of the job pulls the same span at the same point); then the copy engines bring our
    // slice of every member's copy into staging (member q's at q * n_padded/n), no SMs used
    if (int e = barrier(c, st)) return e;
    for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        PIER_CHECK_CUDA(cudaMemcpyAsync(staging + (int64_t)q * (n_padded / n) + (int64_t)span * B,
                                        (const float*)gb->peers[members[q]] + off + (int64_t)r * slice,
                                        (size_t)slice * sizeof(float), cudaMemcpyDefault, st));
    }
    return PIER_OK;
}

int pier_lazy_finish_staged_p2p_f32(PierComm* c, int32_t theta_id, int32_t grad_id, const int32_t* team,
                                    int32_t nteam, const int32_t* norm_team, int32_t n_norm_team,
                                    const float* staging, float* m, float* v, int64_t n_padded,
                                    int64_t bucket_elems, const PierAdamW* hp, double max_norm, void* clip_ws,
                                    int32_t push, void* stream) {
    const PierSharedBuf* tb = shared_buf(c, theta_id);
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!tb || !gb || theta_id == grad_id || !staging)
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p: unknown shared buffers / null staging");
    if (!m || !v || !hp || !clip_ws || !(max_norm > 0.0))
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p: bad args");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n < 2 || n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > tb->bytes ||
        (size_t)n_padded * 4 > gb->bytes || !aligned16(m) || !aligned16(v) || !aligned16(staging))
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p: bad n_padded / alignment");
    if (c->slots_id < 0) return set_error(PIER_EINVAL, "lazy_finish_staged_p2p: communicator has no norm slots");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    cudaStream_t st = as_stream(stream);
    // local fold of the staged copies (+ the norm share posted to every member) ...
    const bool wide = n_padded % (8 * n) == 0 && B % 8 == 0 && aligned32(gb->local) && aligned32(staging);
    if (int e = launch_fold_staged(n, wide, st, (float*)gb->local, staging, n_padded, B, r,
                                   norm_args(c, (NormWs*)clip_ws, members, n)))
        return e;
    // ... every share landed: the clip record (summed over the replica's tensor shards
    // with tensor parallelism); then AdamW on our shard + the all-gather
    if (int e = barrier(c, st)) return e;
    k_norm_slots<<<1, 32, 0, st>>>((const double*)c->shared[c->slots_id].local, n, (NormWs*)clip_ws, max_norm);
    PIER_LAUNCH_CHECK("k_norm_slots");
    if (norm_team)
        if (int e = pier_norm_allreduce_team(c, norm_team, n_norm_team, clip_ws, max_norm, stream)) return e;
    return lazy_adamw_push(c, tb, gb, members, n, r, m, v, n_padded, B, hp, clip_ws, stream, push != 0);
}

int pier_allgather_span_p2p_f32(PierComm* c, int32_t buf_id, const int32_t* team, int32_t nteam, int64_t n_padded,
                                int64_t bucket_elems, int32_t span, void* stream) {
    const PierSharedBuf* b = shared_buf(c, buf_id);
    if (!b) return set_error(PIER_EINVAL, "allgather_span_p2p: unknown shared buffer");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > b->bytes)
        return set_error(PIER_EINVAL, "allgather_span_p2p: n_padded must be a multiple of 4*nranks inside the buffer");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    const int64_t sp = B * n, off = (int64_t)span * sp;
    if (span < 0 || off >= n_padded) return set_error(PIER_EINVAL, "allgather_span_p2p: span out of range");
    const int64_t len = (n_padded - off) < sp ? (n_padded - off) : sp, slice = len / n;
    cudaStream_t st = as_stream(stream);
    for (int q = 0; q < n; ++q) {   // every member's slice of the span into our copy, by the copy engines
        if (q == r) continue;
        const int64_t at = off + (int64_t)q * slice;
        PIER_CHECK_CUDA(cudaMemcpyAsync((float*)b->local + at, (const float*)b->peers[members[q]] + at,
                                        (size_t)slice * sizeof(float), cudaMemcpyDefault, st));
    }
    return PIER_OK;
}

int pier_lazy_step_p2p_bf16(PierComm* c, int32_t master_id, int32_t live_id, int32_t grad_id, float* m, float* v,
                            int64_t n_padded, int64_t bucket_elems, const PierAdamW* hp, double max_norm,
                            void* clip_ws, void* stream) {
    const PierSharedBuf* mb = shared_buf(c, master_id);
    const PierSharedBuf* lb = shared_buf(c, live_id);
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!mb || !lb || !gb || master_id == live_id || master_id == grad_id || live_id == grad_id)
        return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: unknown shared buffers");
    if (!m || !v || !hp || !clip_ws || !(max_norm > 0.0)) return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: bad args");
    const int n = c->nranks, r = c->rank;
    if (n < 2) return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: needs 2..8 ranks");
    if (n_padded <= 0 || n_padded % ((int64_t)n * 8) || (size_t)n_padded * 4 > mb->bytes ||
        (size_t)n_padded * 2 > lb->bytes || (size_t)n_padded * 2 > gb->bytes)
        return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: n_padded must be a multiple of 8*nranks inside the buffers");
    if (common_align({mb->local, m, v}) != 32) return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: 32-byte alignment");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    if (B % 8) return set_error(PIER_EINVAL, "lazy_step_p2p_bf16: bucket_elems must be a multiple of 8");
    // 1-2: reduce-scatter of the bf16 gradients (fp32 left fold, one RNE rounding) with the norm of the mean
    if (int e = mean_p2p_bf16(c, grad_id, n_padded, (NormWs*)clip_ws, max_norm, stream, true, B)) return e;
    // 3: AdamW on this rank's shard of the master + all-gather of the live bf16 params
    return lazy_adamw_push_bf16(c, lb, (float*)mb->local, (const uint16_t*)gb->local, m, v, n_padded, B, hp, clip_ws,
                                stream);
}

// the 7B recipe's step overlapped with the backward: copy-engine pulls of bf16 spans,
// then the staged fold + the norm, AdamW on the master shard, the live params pushed
int pier_lazy_pull_span_p2p_bf16(PierComm* c, int32_t grad_id, uint16_t* staging, int64_t n_padded,
                                 int64_t bucket_elems, int32_t span, void* stream) {
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!gb || !staging) return set_error(PIER_EINVAL, "lazy_pull_span_p2p_bf16: unknown buffer / null staging");
    const int n = c->nranks, r = c->rank;
    if (n < 2 || n_padded <= 0 || n_padded % ((int64_t)n * 8) || (size_t)n_padded * 2 > gb->bytes)
        return set_error(PIER_EINVAL, "lazy_pull_span_p2p_bf16: 2..8 ranks, n_padded a multiple of 8*nranks");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    if (B % 8) return set_error(PIER_EINVAL, "lazy_pull_span_p2p_bf16: bucket_elems must be a multiple of 8");
    const int64_t sp = B * n, off = (int64_t)span * sp;
    if (span < 0 || off >= n_padded) return set_error(PIER_EINVAL, "lazy_pull_span_p2p_bf16: span out of range");
    const int64_t len = (n_padded - off) < sp ? (n_padded - off) : sp, slice = len / n;
    cudaStream_t st = as_stream(stream);
    if (int e = barrier(c, st)) return e;   // every rank's gradient of this span is final
    for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        PIER_CHECK_CUDA(cudaMemcpyAsync(staging + (int64_t)q * (n_padded / n) + (int64_t)span * B,
                                        (const uint16_t*)gb->peers[q] + off + (int64_t)r * slice,
                                        (size_t)slice * sizeof(uint16_t), cudaMemcpyDefault, st));
    }
    return PIER_OK;
}

int pier_lazy_finish_staged_p2p_bf16(PierComm* c, int32_t master_id, int32_t live_id, int32_t grad_id,
                                     const uint16_t* staging, float* m, float* v, int64_t n_padded,
                                     int64_t bucket_elems, const PierAdamW* hp, double max_norm, void* clip_ws,
                                     void* stream) {
    const PierSharedBuf* mb = shared_buf(c, master_id);
    const PierSharedBuf* lb = shared_buf(c, live_id);
    const PierSharedBuf* gb = shared_buf(c, grad_id);
    if (!mb || !lb || !gb || !staging || master_id == live_id || master_id == grad_id || live_id == grad_id)
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: unknown shared buffers / null staging");
    if (!m || !v || !hp || !clip_ws || !(max_norm > 0.0))
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: bad args");
    const int n = c->nranks, r = c->rank;
    if (n < 2 || n_padded <= 0 || n_padded % ((int64_t)n * 8) || (size_t)n_padded * 4 > mb->bytes ||
        (size_t)n_padded * 2 > lb->bytes || (size_t)n_padded * 2 > gb->bytes || !aligned16(staging))
        return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: bad n_padded / alignment");
    if (common_align({mb->local, m, v}) != 32) return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: alignment");
    if (c->slots_id < 0) return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: communicator has no norm slots");
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    if (B % 8) return set_error(PIER_EINVAL, "lazy_finish_staged_p2p_bf16: bucket_elems must be a multiple of 8");
    cudaStream_t st = as_stream(stream);
    int32_t members[PIER_MAX_RANKS];
    for (int q = 0; q < n; ++q) members[q] = q;
    if (int e = launch_fold_staged_bf16(n, st, (uint16_t*)gb->local, staging, n_padded, B, r,
                                        norm_args(c, (NormWs*)clip_ws, members, n)))
        return e;
    if (int e = barrier(c, st)) return e;   // every share landed: the clip record
    k_norm_slots<<<1, 32, 0, st>>>((const double*)c->shared[c->slots_id].local, n, (NormWs*)clip_ws, max_norm);
    PIER_LAUNCH_CHECK("k_norm_slots");
    return lazy_adamw_push_bf16(c, lb, (float*)mb->local, (const uint16_t*)gb->local, m, v, n_padded, B, hp, clip_ws,
                                stream);
}

int pier_gather_p2p_team_f32(PierComm* c, int32_t buf_id, const int32_t* team, int32_t nteam, int64_t n_padded,
                             int64_t bucket_elems, void* stream) {
    const PierSharedBuf* b = shared_buf(c, buf_id);
    if (!b) return set_error(PIER_EINVAL, "gather_p2p: unknown shared buffer");
    int32_t members[PIER_MAX_RANKS];
    int n = 0, r = 0;
    if (int e = resolve_team(c, team, nteam, members, &n, &r)) return e;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > b->bytes)
        return set_error(PIER_EINVAL, "gather_p2p: n_padded must be a multiple of 4*nranks inside the buffer");
    if (n == 1) return PIER_OK;
    int64_t B = bucket_elems;
    if (int e = lazy_bucket(n_padded, n, &B)) return e;
    cudaStream_t st = as_stream(stream);
    PeerTable pt{};
    bool wide = n_padded % (8 * n) == 0 && B % 8 == 0;
    for (int q = 0; q < n; ++q) {
        pt.p[q] = (float*)b->peers[members[q]];
        wide = wide && aligned32(pt.p[q]);
    }
    if (int e = barrier(c, st)) return e;   // every member's shard is final
    if (int e = launch_lazy(1, n, wide, st, pt, nullptr, nullptr, nullptr, n_padded, B, r)) return e;
    return barrier(c, st);                  // every member's pushes have landed
}

int pier_gather_p2p_f32(PierComm* c, int32_t buf_id, int64_t n_padded, int64_t bucket_elems, void* stream) {
    return pier_gather_p2p_team_f32(c, buf_id, nullptr, 0, n_padded, bucket_elems, stream);
}

}  // extern "C"
