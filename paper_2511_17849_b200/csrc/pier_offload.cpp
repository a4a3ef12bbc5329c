// Host offload of the outer state (anchor / outer momentum shards) to pinned
// host memory on side streams (K5).
//
// Replaces HostStore (driver.py:115-164) and its park/fetch call sites
// (driver.py:318-329, initial park :307-309).  Same protocol: a slot is
// "live" between park (store) and fetch (load); parking a live slot or
// fetching a dead one is a protocol error (driver.py:136-146).  Unlike the
// reference (which copies synchronously), the D2H/H2D copies run with
// cudaMemcpyAsync on dedicated low-priority streams, ordered against the
// producer / consumer streams by events only, so they overlap the inner loop.
// Parks (D2H) and fetches (H2D) use separate streams and move kChunk pieces:
// the fetch of piece i waits only for the park of piece i, so when a window
// is too short to hide the round trip the fetch runs behind the park in the
// other PCIe direction instead of after it.
#include <cuda_runtime.h>

#include <new>
#include <string>
#include <vector>

#include "../../include/pier_b200.h"

namespace pier {
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
}

#define OFF_CHECK(expr)                                                \
    do {                                                               \
        cudaError_t _e = (expr);                                       \
        if (_e != cudaSuccess) return ::pier::cuda_status(_e, #expr);  \
    } while (0)

constexpr size_t kChunk = (size_t)64 << 20;   // bytes per piece of a park / fetch

struct PierOffload {
    size_t slot_bytes = 0;
    std::vector<void*> host;
    std::vector<size_t> live_bytes;  // 0 = not live
    std::vector<char> live;
    cudaStream_t side = nullptr;     // D2H (park)
    cudaStream_t side_in = nullptr;  // H2D (fetch)
    cudaEvent_t ev_in = nullptr;     // producer / consumer -> side streams
    std::vector<cudaEvent_t> ev_done;               // per slot: last park or fetch complete
    std::vector<std::vector<cudaEvent_t>> ev_piece;  // per slot, per piece: parked
    double to_host = 0, from_host = 0, stores = 0, loads = 0;
};

static size_t npieces(size_t bytes) { return (bytes + kChunk - 1) / kChunk; }

extern "C" {

int pier_offload_create(int32_t nslots, size_t slot_bytes, PierOffload** out) {
    if (nslots < 1 || !out) return pier::set_error(PIER_EINVAL, "offload_create: bad args");
    auto* o = new (std::nothrow) PierOffload();
    if (!o) return pier::set_error(PIER_ENOMEM, "offload_create: host alloc");
    o->slot_bytes = slot_bytes;
    o->host.assign(nslots, nullptr);
    o->live_bytes.assign(nslots, 0);
    o->live.assign(nslots, 0);
    o->ev_done.assign(nslots, nullptr);
    o->ev_piece.assign(nslots, std::vector<cudaEvent_t>(npieces(slot_bytes), nullptr));
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    auto fail = [&](cudaError_t e, const char* what) {
        pier_offload_destroy(o);
        return pier::cuda_status(e, what);
    };
    cudaError_t e = cudaStreamCreateWithPriority(&o->side, cudaStreamNonBlocking, lo);
    if (e != cudaSuccess) return fail(e, "cudaStreamCreate(side)");
    e = cudaStreamCreateWithPriority(&o->side_in, cudaStreamNonBlocking, lo);
    if (e != cudaSuccess) return fail(e, "cudaStreamCreate(side_in)");
    if ((e = cudaEventCreateWithFlags(&o->ev_in, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "event");
    for (int i = 0; i < nslots; ++i) {
        if (slot_bytes && (e = cudaHostAlloc(&o->host[i], slot_bytes, cudaHostAllocPortable)) != cudaSuccess)
            return fail(e, "cudaHostAlloc(pinned slot)");
        if ((e = cudaEventCreateWithFlags(&o->ev_done[i], cudaEventDisableTiming)) != cudaSuccess)
            return fail(e, "event");
        for (auto& ev : o->ev_piece[i])
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "event");
    }
    *out = o;
    return PIER_OK;
}

int pier_offload_destroy(PierOffload* o) {
    if (!o) return PIER_OK;
    if (o->side) cudaStreamSynchronize(o->side);
    if (o->side_in) cudaStreamSynchronize(o->side_in);
    for (void* p : o->host)
        if (p) cudaFreeHost(p);
    for (auto e : o->ev_done)
        if (e) cudaEventDestroy(e);
    for (auto& v : o->ev_piece)
        for (auto e : v)
            if (e) cudaEventDestroy(e);
    if (o->ev_in) cudaEventDestroy(o->ev_in);
    if (o->side) cudaStreamDestroy(o->side);
    if (o->side_in) cudaStreamDestroy(o->side_in);
    delete o;
    return PIER_OK;
}

int pier_offload_park(PierOffload* o, int32_t slot, const void* dev, size_t bytes, void* producer) {
    if (!o || slot < 0 || slot >= (int)o->host.size() || (!dev && bytes))
        return pier::set_error(PIER_EINVAL, "offload_park: bad slot/pointer");
    if (bytes > o->slot_bytes) return pier::set_error(PIER_EINVAL, "offload_park: larger than the slot");
    if (o->live[slot])
        return pier::set_error(PIER_EPROTOCOL, "offload slot " + std::to_string(slot) +
                                                   " stored twice without a reload");
    // the previous fetch of this slot finished reading the host copy before its
    // consumer went on (protocol: load before store), and `producer` is that consumer
    OFF_CHECK(cudaEventRecord(o->ev_in, (cudaStream_t)producer));
    OFF_CHECK(cudaStreamWaitEvent(o->side, o->ev_in, 0));
    for (size_t i = 0, off = 0; off < bytes; ++i, off += kChunk) {
        const size_t len = bytes - off < kChunk ? bytes - off : kChunk;
        OFF_CHECK(cudaMemcpyAsync((char*)o->host[slot] + off, (const char*)dev + off, len, cudaMemcpyDeviceToHost,
                                  o->side));
        OFF_CHECK(cudaEventRecord(o->ev_piece[slot][i], o->side));
    }
    OFF_CHECK(cudaEventRecord(o->ev_done[slot], o->side));
    o->live[slot] = 1;
    o->live_bytes[slot] = bytes;
    o->to_host += (double)bytes;
    o->stores += 1;
    return PIER_OK;
}

int pier_offload_prefetch(PierOffload* o, int32_t slot, void* dev, size_t bytes, void* consumer) {
    if (!o || slot < 0 || slot >= (int)o->host.size() || (!dev && bytes))
        return pier::set_error(PIER_EINVAL, "offload_fetch: bad slot/pointer");
    if (!o->live[slot])
        return pier::set_error(PIER_EPROTOCOL, "offload slot " + std::to_string(slot) + " loaded before being stored");
    if (bytes != o->live_bytes[slot]) return pier::set_error(PIER_EINVAL, "offload_fetch: size differs from park");
    // `dev` may have been (re)allocated on the consumer stream since the park
    OFF_CHECK(cudaEventRecord(o->ev_in, (cudaStream_t)consumer));
    OFF_CHECK(cudaStreamWaitEvent(o->side_in, o->ev_in, 0));
    for (size_t i = 0, off = 0; off < bytes; ++i, off += kChunk) {   // piece i once it is parked
        const size_t len = bytes - off < kChunk ? bytes - off : kChunk;
        OFF_CHECK(cudaStreamWaitEvent(o->side_in, o->ev_piece[slot][i], 0));
        OFF_CHECK(cudaMemcpyAsync((char*)dev + off, (const char*)o->host[slot] + off, len, cudaMemcpyHostToDevice,
                                  o->side_in));
    }
    OFF_CHECK(cudaEventRecord(o->ev_done[slot], o->side_in));
    o->live[slot] = 0;
    o->live_bytes[slot] = 0;
    o->from_host += (double)bytes;
    o->loads += 1;
    return PIER_OK;
}

int pier_offload_wait(PierOffload* o, int32_t slot, void* consumer) {
    if (!o || slot < 0 || slot >= (int)o->host.size()) return pier::set_error(PIER_EINVAL, "offload_wait: bad slot");
    OFF_CHECK(cudaStreamWaitEvent((cudaStream_t)consumer, o->ev_done[slot], 0));
    return PIER_OK;
}

int pier_offload_fetch(PierOffload* o, int32_t slot, void* dev, size_t bytes, void* consumer) {
    if (int e = pier_offload_prefetch(o, slot, dev, bytes, consumer)) return e;
    return pier_offload_wait(o, slot, consumer);
}

int pier_offload_sync(PierOffload* o) {
    if (!o) return pier::set_error(PIER_EINVAL, "offload_sync: null");
    OFF_CHECK(cudaStreamSynchronize(o->side));
    OFF_CHECK(cudaStreamSynchronize(o->side_in));
    return PIER_OK;
}

int pier_offload_counters(const PierOffload* o, double* out5) {
    if (!o || !out5) return pier::set_error(PIER_EINVAL, "offload_counters: null");
    double res = 0;
    for (size_t i = 0; i < o->live.size(); ++i)
        if (o->live[i]) res += (double)o->live_bytes[i];
    out5[0] = o->to_host;
    out5[1] = o->from_host;
    out5[2] = o->stores;
    out5[3] = o->loads;
    out5[4] = res;
    return PIER_OK;
}

void* pier_offload_host_ptr(PierOffload* o, int32_t slot) {
    if (!o || slot < 0 || slot >= (int)o->host.size()) return nullptr;
    return o->host[slot];
}

void* pier_offload_stream(PierOffload* o) { return o ? (void*)o->side : nullptr; }
void* pier_offload_stream_h2d(PierOffload* o) { return o ? (void*)o->side_in : nullptr; }

}  // extern "C"
