// Inter-group reduction for the outer step over NCCL (NVLink 5 / NVSwitch),
// one group per GPU, one process per GPU.
//
// Replaces the simulated `outer_delta_sync` (topology.py:104-132, called at
// driver.py:428-429) and the per-worker broadcast of the new model
// (driver.py:439-440).  "Mode B": the parameter buffer is cut into spans of
// nranks*B elements; for span b every rank owns the B-slice at rank*B inside
// the span, so one bucket is ONE contiguous in-place ReduceScatter, the fused
// outer update (K3) on the owned slice, and ONE in-place AllGather.  Rank r's
// anchor / outer-momentum shard is the concatenation of its slices, i.e. each
// GPU keeps only 1/n of the outer state (8N/n bytes), the same partition idea
// as the per-rank HostStore keys of driver.py:318-329.
//
// Pipelining: the comm stream runs RS(0), RS(1), [wait K3(0)] AG(0), RS(2),
// [wait K3(1)] AG(1), ... while K3(b) runs on the caller's stream as soon as
// RS(b) lands, so the HBM pass of the update hides under the NVLink transfer.
// The reduction is an NCCL sum followed by `/ n` inside K3 (topology.py:121):
// bitwise equal to the reference's left fold whenever the sum order agrees
// (always at n <= 2), within fp32 rounding otherwise.
#include <nccl.h>

#include <vector>

#include "pier_common.cuh"

#include <cstring>

#include "pier_comm_internal.h"

namespace {

using namespace pier;

int nccl_status(ncclResult_t r, const char* what) {
    return set_error(PIER_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define PIER_CHECK_NCCL(expr)                                   \
    do {                                                        \
        ncclResult_t _r = (expr);                               \
        if (_r != ncclSuccess) return nccl_status(_r, #expr);   \
    } while (0)

struct Bucket {
    int64_t off;    // start of the span in the full buffer
    int64_t slice;  // elements owned per rank in this span
    int64_t shard;  // offset of this slice inside the rank's shard
};

int layout(int64_t n_padded, int nranks, int64_t B, std::vector<Bucket>& out) {
    if (n_padded <= 0 || B <= 0 || n_padded % ((int64_t)nranks * 4) != 0 || B % 4 != 0)
        return set_error(PIER_EINVAL,
                         "sharded layout: n_padded must be a positive multiple of 4*nranks and bucket_elems of 4");
    out.clear();
    const int64_t span = B * nranks;
    int64_t off = 0, sh = 0;
    while (off < n_padded) {
        int64_t len = (n_padded - off) < span ? (n_padded - off) : span;
        Bucket b{off, len / nranks, sh};
        out.push_back(b);
        off += len;
        sh += b.slice;
    }
    return PIER_OK;
}

int ensure_events(PierComm* c, size_t nb) {
    while (c->ev_rs.size() < nb) {
        cudaEvent_t a, b;
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        c->ev_rs.push_back(a);
        c->ev_k3.push_back(b);
    }
    return PIER_OK;
}

}  // namespace

extern "C" {

int pier_nccl_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int pier_nccl_get_unique_id(void* out) {
    if (!out) return set_error(PIER_EINVAL, "nccl_get_unique_id: null");
    ncclUniqueId id;
    PIER_CHECK_NCCL(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return PIER_OK;
}

int pier_comm_init(const void* uid, int32_t rank, int32_t nranks, PierComm** out) {
    if (!uid || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(PIER_EINVAL, "comm_init: bad rank/nranks");
    auto* c = new (std::nothrow) PierComm();
    if (!c) return set_error(PIER_ENOMEM, "comm_init: host alloc");
    c->rank = rank;
    c->nranks = nranks;
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_status(r, "ncclCommInitRank");
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // the NCCL stream gets the higher priority: the transfer is the critical path
    PIER_CHECK_CUDA(cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi));
    PIER_CHECK_CUDA(cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming));
    PIER_CHECK_CUDA(cudaEventCreateWithFlags(&c->end, cudaEventDisableTiming));
    // the persistent round's signal block, the fused-norm slots and the timeout
    // diagnostic slot: allocated (collectively) here, never inside a hot call
    if (int e = pier::comm_setup(c)) {
        pier_comm_destroy(c);
        return e;
    }
    *out = c;
    return PIER_OK;
}

int pier_comm_destroy(PierComm* c) {
    if (!c) return PIER_OK;
    if (c->cs) cudaStreamSynchronize(c->cs);
    if (c->ps) cudaStreamSynchronize(c->ps);
    pier::comm_free_shared_all(c);
    pier::comm_free_windows(c);
    if (c->diag_host) {
        pier::unregister_diag(c->diag_host);
        cudaFreeHost((void*)c->diag_host);
    }
    pier::vgroup_release(c);
    if (c->ps) cudaStreamDestroy(c->ps);
    if (c->d_barrier) cudaFree(c->d_barrier);
    for (auto e : c->ev_rs) cudaEventDestroy(e);
    for (auto e : c->ev_k3) cudaEventDestroy(e);
    if (c->start) cudaEventDestroy(c->start);
    if (c->end) cudaEventDestroy(c->end);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
    return PIER_OK;
}

int pier_outer_step_sharded_f32(PierComm* c, float* theta, float* anchor_shard, float* mom_shard,
                                int64_t n_padded, int64_t B, double lr, double mu, void* stream) {
    if (!theta || !anchor_shard || !mom_shard) return set_error(PIER_EINVAL, "outer_step_sharded: null");
    if (!c || c->nranks == 1) {  // one group (comm may be NULL): the fused update over the whole buffer
        if (n_padded <= 0) return set_error(PIER_EINVAL, "outer_step_sharded: empty buffer");
        return pier_outer_update_f32(theta, anchor_shard, mom_shard, theta, n_padded, lr, mu, 1, stream);
    }
    if (int e = require_nccl(c, "outer_step_sharded")) return e;
    cudaStream_t st = as_stream(stream);
    std::vector<Bucket> bk;
    if (int e = layout(n_padded, c->nranks, B, bk)) return e;
    if (int e = ensure_events(c, bk.size())) return e;
    const int r = c->rank, n = c->nranks;
    PIER_CHECK_CUDA(cudaEventRecord(c->start, st));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
    auto rs = [&](size_t b) -> int {
        float* span = theta + bk[b].off;
        PIER_CHECK_NCCL(ncclReduceScatter(span, span + (int64_t)r * bk[b].slice, (size_t)bk[b].slice, ncclFloat,
                                          ncclSum, c->nccl, c->cs));
        PIER_CHECK_CUDA(cudaEventRecord(c->ev_rs[b], c->cs));
        return PIER_OK;
    };
    auto ag = [&](size_t b) -> int {
        float* span = theta + bk[b].off;
        PIER_CHECK_CUDA(cudaStreamWaitEvent(c->cs, c->ev_k3[b], 0));
        PIER_CHECK_NCCL(ncclAllGather(span + (int64_t)r * bk[b].slice, span, (size_t)bk[b].slice, ncclFloat,
                                      c->nccl, c->cs));
        return PIER_OK;
    };
    const size_t nb = bk.size();
    if (int e = rs(0)) return e;
    for (size_t b = 0; b < nb; ++b) {
        if (b + 1 < nb)
            if (int e = rs(b + 1)) return e;
        PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->ev_rs[b], 0));
        float* mine = theta + bk[b].off + (int64_t)r * bk[b].slice;
        if (int e = pier_outer_update_f32(mine, anchor_shard + bk[b].shard, mom_shard + bk[b].shard, mine,
                                          bk[b].slice, lr, mu, n, stream))
            return e;
        PIER_CHECK_CUDA(cudaEventRecord(c->ev_k3[b], st));
        if (int e = ag(b)) return e;
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->cs));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

int pier_warmup_fold_sharded_f32(PierComm* c, const float* theta, float* anchor_shard, float* mom_shard,
                                 int64_t n_padded, int64_t B, double mu, void* stream) {
    if (!theta || !anchor_shard || !mom_shard) return set_error(PIER_EINVAL, "warmup_fold_sharded: null");
    if (!c || c->nranks == 1) return pier_warmup_fold_f32(theta, anchor_shard, mom_shard, n_padded, mu, stream);
    std::vector<Bucket> bk;
    if (int e = layout(n_padded, c->nranks, B, bk)) return e;
    for (const Bucket& b : bk) {
        const float* mine = theta + b.off + (int64_t)c->rank * b.slice;
        if (int e = pier_warmup_fold_f32(mine, anchor_shard + b.shard, mom_shard + b.shard, b.slice, mu, stream))
            return e;
    }
    return PIER_OK;
}

int pier_allreduce_mean_f32(PierComm* c, float* buf, int64_t n, int64_t B, void* stream) {
    if (!c || (!buf && n > 0) || n < 0 || B <= 0) return set_error(PIER_EINVAL, "allreduce_mean: bad args");
    if (c->nranks == 1 || n == 0) return PIER_OK;
    if (int e = require_nccl(c, "allreduce_mean")) return e;
    cudaStream_t st = as_stream(stream);
    PIER_CHECK_CUDA(cudaEventRecord(c->start, st));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
    for (int64_t off = 0; off < n; off += B) {
        int64_t len = (n - off) < B ? (n - off) : B;
        PIER_CHECK_NCCL(ncclAllReduce(buf + off, buf + off, (size_t)len, ncclFloat, ncclAvg, c->nccl, c->cs));
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->cs));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

int pier_allreduce_mean_bf16(PierComm* c, uint16_t* buf, int64_t n, int64_t B, void* stream) {
    if (!c || (!buf && n > 0) || n < 0 || B <= 0) return set_error(PIER_EINVAL, "allreduce_mean_bf16: bad args");
    if (c->nranks == 1 || n == 0) return PIER_OK;
    cudaStream_t st = as_stream(stream);
    PIER_CHECK_CUDA(cudaEventRecord(c->start, st));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
    for (int64_t off = 0; off < n; off += B) {
        int64_t len = (n - off) < B ? (n - off) : B;
        PIER_CHECK_NCCL(ncclAllReduce(buf + off, buf + off, (size_t)len, ncclBfloat16, ncclAvg, c->nccl, c->cs));
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->cs));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

int pier_shard_allgather_f32(PierComm* c, const float* shard, float* full, int64_t n_padded, int64_t B,
                             void* stream) {
    if (!c || !shard || !full) return set_error(PIER_EINVAL, "shard_allgather: null");
    cudaStream_t st = as_stream(stream);
    std::vector<Bucket> bk;
    if (int e = layout(n_padded, c->nranks, B, bk)) return e;
    if (c->vg) {   // virtual group: copy every rank's slices straight from its shard
        void* shards[PIER_MAX_RANKS];
        if (int e = vg_rendezvous(c, (void*)shard, st, nullptr, shards)) return e;
        for (const Bucket& b : bk)
            for (int q = 0; q < c->nranks; ++q)
                PIER_CHECK_CUDA(cudaMemcpyAsync(full + b.off + (int64_t)q * b.slice, (const float*)shards[q] + b.shard,
                                                (size_t)b.slice * 4, cudaMemcpyDeviceToDevice, st));
        return barrier(c, st);   // no rank overwrites its shard before every copy ran
    }
    PIER_CHECK_CUDA(cudaEventRecord(c->start, st));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(c->cs, c->start, 0));
    PIER_CHECK_NCCL(ncclGroupStart());
    for (const Bucket& b : bk) {
        ncclResult_t rr = ncclAllGather(shard + b.shard, full + b.off, (size_t)b.slice, ncclFloat, c->nccl, c->cs);
        if (rr != ncclSuccess) {
            ncclGroupEnd();
            return nccl_status(rr, "ncclAllGather");
        }
    }
    PIER_CHECK_NCCL(ncclGroupEnd());
    PIER_CHECK_CUDA(cudaEventRecord(c->end, c->cs));
    PIER_CHECK_CUDA(cudaStreamWaitEvent(st, c->end, 0));
    return PIER_OK;
}

}  // extern "C"
