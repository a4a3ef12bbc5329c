// Pier round with the NVLink transfers on the copy engines (reduce="p2p",
// round_impl="ce"): this group's AdamW and the fold/update run on the SMs, the
// reduce-scatter and all-gather bytes move as cudaMemcpyAsync pushes between
// peer-mapped buffers.
//
// Why: tools/tma_probe.cu measured the copy engines at 778 GB/s per direction
// with both directions busy, against 665-712 GB/s for SM-issued loads/stores
// (LDG, STG or TMA bulk) -- the exchange is wire-bound from n = 4 on.
//
// Per span b (layout of pier_comm.cu; rank r owns slice r of every span):
//   compute stream : AdamW(b)                                   (K4b)
//   exchange stream: barrier -> [copy streams: push theta[b, slice q] into
//                    rank q's recv slot r] -> barrier -> fold(b): recv slots
//                    and the own slice in ascending rank order (bitwise =
//                    topology.py:113-121) + fused outer update -> [copy
//                    streams: push theta[b, slice r] into every rank]
// and one final barrier.  The barriers are 1-element ncclAllReduces on the
// exchange stream; copies for span b+1 overlap the fold of span b and the
// AdamW of later spans.
#include <cstring>
#include <string>
#include <vector>

#include "pier_comm_internal.h"
#include "pier_common.cuh"

namespace pier {

struct SrcTable {
    const float* p[PIER_MAX_RANKS];
};

template <int NR, int U>
__global__ void __launch_bounds__(kThreads) k_ce_fold(SrcTable src, float4* __restrict__ dst,
                                                       float4* __restrict__ anchor, float4* __restrict__ mom,
                                                       int64_t nvec, float lr, float mu, float nf) {
    const int64_t tile = (int64_t)kThreads * U;
    for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < nvec; t0 += (int64_t)gridDim.x * tile) {
        float4 x[NR][U], a4[U], m4[U];
#pragma unroll
        for (int q = 0; q < NR; ++q)
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                if (i < nvec) x[q][k] = __ldcs(reinterpret_cast<const float4*>(src.p[q]) + i);
            }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
            if (i < nvec) { a4[k] = __ldcs(anchor + i); m4[k] = __ldcs(mom + i); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
            if (i >= nvec) continue;
            float4 out;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                float acc = lane(x[0][k], w);
#pragma unroll
                for (int q = 1; q < NR; ++q) acc = add_rn(acc, lane(x[q][k], w));   // topology.py:113-120
                float av = div_rn(acc, nf);                                         // topology.py:121
                float dl = sub_rn(av, lane(a4[k], w));                              // driver.py:434
                float m2 = add_rn(mul_rn(mu, lane(m4[k], w)), dl);                  // optim.py:270
                float up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));                  // optim.py:271
                av = add_rn(av, sub_rn(up, dl));                                    // optim.py:275
                lane(m4[k], w) = m2;
                lane(a4[k], w) = av;                                                // driver.py:438
                lane(out, w) = av;
            }
            __stcs(mom + i, m4[k]);
            __stcs(anchor + i, a4[k]);
            dst[i] = out;   // stays in L2 for the all-gather copies
        }
    }
}

template <int NR>
void launch_ce_fold(int grid, cudaStream_t st, const SrcTable& s, float* dst, float* an, float* mo, int64_t nvec,
                    float lr, float mu) {
    constexpr int U = NR <= 2 ? 4 : NR <= 4 ? 2 : 1;
    k_ce_fold<NR, U><<<grid, kThreads, 0, st>>>(s, (float4*)dst, (float4*)an, (float4*)mo, nvec, lr, mu, (float)NR);
}

int ce_fold(int n, int grid, cudaStream_t st, const SrcTable& s, float* dst, float* an, float* mo, int64_t nvec,
            float lr, float mu) {
    switch (n) {
        case 2: launch_ce_fold<2>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 3: launch_ce_fold<3>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 4: launch_ce_fold<4>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 5: launch_ce_fold<5>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 6: launch_ce_fold<6>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 7: launch_ce_fold<7>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        case 8: launch_ce_fold<8>(grid, st, s, dst, an, mo, nvec, lr, mu); break;
        default: return set_error(PIER_EINVAL, "ce: 2..8 ranks");
    }
    PIER_LAUNCH_CHECK("k_ce_fold");
    return PIER_OK;
}

int ce_setup(PierComm* c, size_t nevents) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (!c->ps) PIER_CHECK_CUDA(cudaStreamCreateWithPriority(&c->ps, cudaStreamNonBlocking, hi));
    while ((int)c->copy_streams.size() < c->nranks) {
        cudaStream_t s;
        PIER_CHECK_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi));
        c->copy_streams.push_back(s);
    }
    while (c->ce_events.size() < nevents) {
        cudaEvent_t e;
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ce_events.push_back(e);
    }
    return PIER_OK;
}

}  // namespace pier

using namespace pier;

extern "C" {

int pier_round_ce_f32(PierComm* c, int32_t theta_id, int32_t recv_id, const float* g, float* m, float* v,
                      float* anchor_shard, float* mom_shard, int64_t n_padded, int64_t B, const PierAdamW* hp,
                      const void* clip_ws, double lr, double mu, void* stream) {
    if (!c || theta_id < 0 || theta_id >= (int)c->shared.size() || !c->shared[theta_id].local || recv_id < 0 ||
        recv_id >= (int)c->shared.size() || !c->shared[recv_id].local)
        return set_error(PIER_EINVAL, "round_ce: unknown shared buffer");
    if (!g || !m || !v || !anchor_shard || !mom_shard || !hp) return set_error(PIER_EINVAL, "round_ce: null");
    const int n = c->nranks, r = c->rank;
    if (n < 2 || n > PIER_MAX_RANKS) return set_error(PIER_EINVAL, "round_ce: 2..8 ranks");
    const PierSharedBuf& th = c->shared[theta_id];
    const PierSharedBuf& rv = c->shared[recv_id];
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4 || (size_t)n_padded * 4 > th.bytes ||
        (size_t)n_padded * 4 > rv.bytes)
        return set_error(PIER_EINVAL, "round_ce: bad n_padded / bucket / recv size");
    const int64_t span = B * n, shard = n_padded / n;
    const int64_t nspans = (n_padded + span - 1) / span;
    if (int e = ce_setup(c, (size_t)(nspans * (3 + n) + n))) return e;
    cudaStream_t st = as_stream(stream), X = c->ps;
    float* mine = (float*)th.local;
    float* recv = (float*)rv.local;
    size_t ev = 0;
    auto next = [&]() { return c->ce_events[ev++]; };
    int64_t sh = 0;
    for (int64_t off = 0; off < n_padded; off += span) {
        const int64_t len = (n_padded - off) < span ? (n_padded - off) : span;
        const int64_t slice = len / n;
        // this group's AdamW of the span (driver.py:395-399)
        if (int e = pier_adamw_f32(mine + off, g + off, m + off, v + off, len, hp, clip_ws, stream)) return e;
        cudaEvent_t evA = next();
        PIER_CHECK_CUDA(cudaEventRecord(evA, st));
        PIER_CHECK_CUDA(cudaStreamWaitEvent(X, evA, 0));
        if (int e = barrier(c, X)) return e;                       // every rank's span is updated
        cudaEvent_t fork = next();
        PIER_CHECK_CUDA(cudaEventRecord(fork, X));
        // reduce-scatter: push slice q of the span into rank q's recv slot r
        for (int q = 0; q < n; ++q) {
            if (q == r) continue;
            cudaStream_t cq = c->copy_streams[q];
            PIER_CHECK_CUDA(cudaStreamWaitEvent(cq, fork, 0));
            float* dst = (float*)c->shared[recv_id].peers[q] + (int64_t)r * shard + sh;
            PIER_CHECK_CUDA(cudaMemcpyAsync(dst, mine + off + (int64_t)q * slice, slice * 4,
                                            cudaMemcpyDeviceToDevice, cq));
            cudaEvent_t done = next();
            PIER_CHECK_CUDA(cudaEventRecord(done, cq));
            PIER_CHECK_CUDA(cudaStreamWaitEvent(X, done, 0));
        }
        if (int e = barrier(c, X)) return e;                       // every push of the span landed
        SrcTable s{};
        for (int q = 0; q < n; ++q)
            s.p[q] = q == r ? mine + off + (int64_t)r * slice : recv + (int64_t)q * shard + sh;
        if (int e = ce_fold(n, stream_grid(slice / 4, 2, 4), X, s, mine + off + (int64_t)r * slice,
                            anchor_shard + sh, mom_shard + sh, slice / 4, (float)lr, (float)mu))
            return e;
        cudaEvent_t folded = next();
        PIER_CHECK_CUDA(cudaEventRecord(folded, X));
        // all-gather: push the new slice into every rank (driver.py:439-440)
        for (int q = 0; q < n; ++q) {
            if (q == r) continue;
            cudaStream_t cq = c->copy_streams[q];
            PIER_CHECK_CUDA(cudaStreamWaitEvent(cq, folded, 0));
            float* dst = (float*)th.peers[q] + off + (int64_t)r * slice;
            PIER_CHECK_CUDA(cudaMemcpyAsync(dst, mine + off + (int64_t)r * slice, slice * 4,
                                            cudaMemcpyDeviceToDevice, cq));
        }
        sh += slice;
    }
    for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        cudaEvent_t done = next();
        PIER_CHECK_CUDA(cudaEventRecord(done, c->copy_streams[q]));
        PIER_CHECK_CUDA(cudaStreamWaitEvent(X, done, 0));
    }
    if (int e = barrier(c, X)) return e;                           // every all-gather push landed
    PIER_CHECK_CUDA(cudaEventRecord(c->end, X));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

}  // extern "C"
