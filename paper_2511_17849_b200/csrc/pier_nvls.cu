// Outer step through NVLink SHARP (NVLS): the NVSwitch reduces in the fabric.
//
// Same contract as pier_p2p.cu (pull-reduce, fused outer update, broadcast of
// the result; shard layout of pier_comm.cu), but the buffer is an NCCL
// symmetric window with a multicast mapping, so one
//   multimem.ld_reduce.add.v4.f32   (the switch fetches every rank's copy and sums)
// replaces the n peer loads, and one
//   multimem.st.v4.f32              (the switch replicates into every rank)
// replaces the n peer stores.  Per GPU the links carry S + S/n bytes in each
// direction instead of 2(n-1)/n * S for any switch-less exchange: 1.25 S vs
// 1.5 S at n=4, 1.125 S vs 1.75 S at n=8 (S = 4N bytes).
//
// The switch's fp32 summation order is not the reference's left fold, so this
// path is within fp32 tolerance, not bitwise (the p2p path is the bitwise one).
// Cross-rank ordering uses NCCL's device-side LSA barrier (one per CTA index)
// at kernel start and end -- no host round trip.
#include <cuda/atomic>
#include <nccl.h>
#include <nccl_device.h>

#include <cstring>
#include <string>

#include "pier_comm_internal.h"
#include "pier_common.cuh"

namespace pier {

constexpr int kNvlsCtasPerSm = 2;      // grid always fully resident (barriers spin)
constexpr int kNvlsMaxBarriers = 1024;

__device__ __forceinline__ float4 mm_ld_reduce_add(const float4* p) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void mm_st(float4* p, const float4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

enum { kNvlsMean = 0, kNvlsOuter = 1 };

// One launch walks every span of a region of the window (region_bytes:
// its start, n_pad elements, spans of B*nranks) and strides over this rank's
// slice of each; one LSA barrier before and one after.
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_nvls_reduce(ncclDevComm dc, ncclWindow_t win, size_t region_bytes,
                                                           int64_t n_pad, int64_t B, int nranks, int r,
                                                           float4* __restrict__ anchor, float4* __restrict__ mom,
                                                           float lr, float mu, float nf) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);     // every rank's theta is final
    float* mm0 = reinterpret_cast<float*>(ncclGetLsaMultimemPointer(win, region_bytes, dc));
    constexpr int U = 4;  // multicast reductions in flight per thread
    const int64_t tile = (int64_t)kThreads * U;
    const int64_t span = B * nranks;
    int64_t sh = 0;       // vector offset of this span's slice in the shard
    for (int64_t off = 0; off < n_pad; off += span) {
        const int64_t len = (n_pad - off) < span ? (n_pad - off) : span;
        const int64_t slice = len / nranks, nvec = slice / 4;
        float4* mm = reinterpret_cast<float4*>(mm0 + off + (int64_t)r * slice);
        for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < nvec; t0 += (int64_t)gridDim.x * tile) {
            float4 s[U], an[U], m[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                if (i < nvec) s[k] = mm_ld_reduce_add(mm + i);     // sum over ranks, in the switch
            }
            if (MODE == kNvlsOuter) {
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                    if (i < nvec) { an[k] = __ldcs(anchor + sh + i); m[k] = __ldcs(mom + sh + i); }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t i = t0 + threadIdx.x + (int64_t)k * kThreads;
                if (i >= nvec) continue;
                float4 out;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    float av = div_rn(lane(s[k], w), nf);                             // topology.py:121
                    if (MODE == kNvlsOuter) {
                        float dl = sub_rn(av, lane(an[k], w));                        // driver.py:434
                        float m2 = add_rn(mul_rn(mu, lane(m[k], w)), dl);             // optim.py:270
                        float up = mul_rn(lr, add_rn(mul_rn(mu, m2), dl));            // optim.py:271
                        av = add_rn(av, sub_rn(up, dl));                              // optim.py:275
                        lane(m[k], w) = m2;
                        lane(an[k], w) = av;
                    }
                    lane(out, w) = av;
                }
                if (MODE == kNvlsOuter) {
                    __stcs(mom + sh + i, m[k]);
                    __stcs(anchor + sh + i, an[k]);
                }
                mm_st(mm + i, out);                                 // every rank's copy (driver.py:439-440)
            }
        }
        sh += nvec;
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);     // all multicast stores landed
}

int nvls_devcomm(PierComm* c) {
    if (c->devcomm_ok) return PIER_OK;
    ncclDevCommRequirements reqs;
    memset(&reqs, 0, sizeof(reqs));
    reqs.lsaMultimem = true;
    reqs.lsaBarrierCount = kNvlsMaxBarriers;
    ncclResult_t r = ncclDevCommCreate(c->nccl, &reqs, &c->devcomm);
    if (r != ncclSuccess)
        return set_error(PIER_ENCCL, std::string("ncclDevCommCreate(lsaMultimem): ") + ncclGetErrorString(r) +
                                         " -- NVLS multicast unavailable on this system");
    c->devcomm_ok = true;
    return PIER_OK;
}

// region: [region_elems, region_elems + n_pad) of the window, spans of B*nranks
int nvls_launch(PierComm* c, int mode, const PierWindowBuf& wb, int64_t region_elems, int64_t n_pad, int64_t B,
                float* an, float* mo, float lr, float mu, cudaStream_t st) {
    int grid = stream_grid(n_pad / c->nranks / 4, 4, kNvlsCtasPerSm);
    if (grid > kNvlsMaxBarriers) grid = kNvlsMaxBarriers;
    size_t region = (size_t)region_elems * sizeof(float);
    if (mode == kNvlsOuter)
        k_nvls_reduce<kNvlsOuter><<<grid, kThreads, 0, st>>>(c->devcomm, wb.win, region, n_pad, B, c->nranks,
                                                              c->rank, (float4*)an, (float4*)mo, lr, mu,
                                                              (float)c->nranks);
    else
        k_nvls_reduce<kNvlsMean><<<grid, kThreads, 0, st>>>(c->devcomm, wb.win, region, n_pad, B, c->nranks,
                                                             c->rank, nullptr, nullptr, 0.f, 0.f, (float)c->nranks);
    PIER_LAUNCH_CHECK("k_nvls_reduce");
    return PIER_OK;
}

const PierWindowBuf* find_window(PierComm* c, int32_t id) {
    if (!c || id < 0 || id >= (int)c->windows.size() || !c->windows[id].ptr) return nullptr;
    return &c->windows[id];
}

int comm_free_windows(PierComm* c) {
    for (auto& w : c->windows) {
        if (!w.ptr) continue;
        ncclCommWindowDeregister(c->nccl, w.win);
        ncclMemFree(w.ptr);
        w = PierWindowBuf();
    }
    if (c->devcomm_ok) {
        ncclDevCommDestroy(c->nccl, &c->devcomm);
        c->devcomm_ok = false;
    }
    return PIER_OK;
}

}  // namespace pier

using namespace pier;

extern "C" {

int pier_comm_alloc_window(PierComm* c, size_t bytes, void** out_local, int32_t* out_id) {
    if (!c || !out_local || !out_id || bytes == 0) return set_error(PIER_EINVAL, "alloc_window: bad args");
    if (int e = require_nccl(c, "alloc_window")) return e;
    PierWindowBuf w;
    w.bytes = bytes;
    ncclResult_t r = ncclMemAlloc(&w.ptr, bytes);
    if (r != ncclSuccess) return set_error(PIER_ENCCL, std::string("ncclMemAlloc: ") + ncclGetErrorString(r));
    PIER_CHECK_CUDA(cudaMemset(w.ptr, 0, bytes));
    PIER_CHECK_CUDA(cudaDeviceSynchronize());
    r = ncclCommWindowRegister(c->nccl, w.ptr, bytes, &w.win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        ncclMemFree(w.ptr);
        return set_error(PIER_ENCCL, std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r));
    }
    if (int e = nvls_devcomm(c)) return e;
    c->windows.push_back(w);
    *out_local = w.ptr;
    *out_id = (int32_t)c->windows.size() - 1;
    return PIER_OK;
}

int pier_outer_step_nvls_f32(PierComm* c, int32_t win_id, float* anchor_shard, float* mom_shard, int64_t n_padded,
                             int64_t B, double lr, double mu, void* stream) {
    const PierWindowBuf* wb = find_window(c, win_id);
    if (!wb) return set_error(PIER_EINVAL, "outer_step_nvls: unknown window");
    const int n = c->nranks;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4 || (size_t)n_padded * 4 > wb->bytes)
        return set_error(PIER_EINVAL, "outer_step_nvls: bad n_padded / bucket");
    if (!anchor_shard || !mom_shard || !aligned16(anchor_shard) || !aligned16(mom_shard))
        return set_error(PIER_EINVAL, "outer_step_nvls: shards must be non-null and 16-byte aligned");
    return nvls_launch(c, kNvlsOuter, *wb, 0, n_padded, B, anchor_shard, mom_shard, (float)lr, (float)mu,
                       as_stream(stream));
}

int pier_round_nvls_f32(PierComm* c, int32_t theta_win, const float* g, float* m, float* v, float* anchor_shard,
                        float* mom_shard, int64_t n_padded, int64_t B, const PierAdamW* hp, const void* clip_ws,
                        double lr, double mu, void* stream) {
    const PierWindowBuf* wb = find_window(c, theta_win);
    if (!wb) return set_error(PIER_EINVAL, "round_nvls: unknown window");
    if (!g || !m || !v || !anchor_shard || !mom_shard || !hp) return set_error(PIER_EINVAL, "round_nvls: null");
    const int n = c->nranks;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || B <= 0 || B % 4 || (size_t)n_padded * 4 > wb->bytes)
        return set_error(PIER_EINVAL, "round_nvls: bad n_padded / bucket");
    cudaStream_t st = as_stream(stream);
    if (!c->ps) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        PIER_CHECK_CUDA(cudaStreamCreateWithPriority(&c->ps, cudaStreamNonBlocking, hi));
    }
    float* theta = (float*)wb->ptr;
    const int64_t span = B * n;
    const int64_t nspans = (n_padded + span - 1) / span;
    while ((int64_t)c->ev_rs.size() < nspans) {
        cudaEvent_t e;
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_rs.push_back(e);
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_k3.push_back(e);
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->start, st));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(c->ps, c->start, 0));
    int64_t sh = 0, b = 0;
    for (int64_t off = 0; off < n_padded; off += span, ++b) {
        int64_t len = (n_padded - off) < span ? (n_padded - off) : span;
        int64_t slice = len / n;
        if (int e = pier_adamw_f32(theta + off, g + off, m + off, v + off, len, hp, clip_ws, stream)) return e;
        PIER_CHECK_CUDA(cudaEventRecord(c->ev_rs[b], st));
        PIER_CHECK_CUDA(cudaStreamWaitEvent(c->ps, c->ev_rs[b], 0));
        if (int e = nvls_launch(c, kNvlsOuter, *wb, off, len, slice, anchor_shard + sh, mom_shard + sh, (float)lr,
                                (float)mu, c->ps))
            return e;
        sh += slice;
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->ps));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

int pier_allreduce_mean_nvls_f32(PierComm* c, int32_t win_id, int64_t n_padded, void* stream) {
    const PierWindowBuf* wb = find_window(c, win_id);
    if (!wb) return set_error(PIER_EINVAL, "allreduce_mean_nvls: unknown window");
    const int n = c->nranks;
    if (n_padded <= 0 || n_padded % ((int64_t)n * 4) || (size_t)n_padded * 4 > wb->bytes)
        return set_error(PIER_EINVAL, "allreduce_mean_nvls: bad n_padded");
    return nvls_launch(c, kNvlsMean, *wb, 0, n_padded, n_padded / n, nullptr, nullptr, 0.f, 0.f,
                       as_stream(stream));
}

}  // extern "C"
