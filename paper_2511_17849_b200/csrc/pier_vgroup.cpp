// Virtual groups: n Pier ranks on ONE device, one host thread per rank.
//
// The reference simulates its groups in one process and keeps every
// reduction in ascending rank order with barriers between stages
// (driver.py:476-529, topology.py:104-122).  A virtual group is the same idea
// on one B200: every rank owns its own buffers on the device and drives them
// from its own host thread through the ordinary communicator entry points;
// where the multi-GPU build orders ranks with a 1-element ncclAllReduce, a
// virtual group rendezvous on the host and fences the ranks' streams with
// events.  Kernels that read or write several ranks' buffers (the P2P
// exchanges) run unchanged -- the "peer" pointers are just other allocations
// on the same device -- and the persistent round, whose CTAs spin on flags
// other ranks' CTAs release, is launched ONCE for all ranks as a single
// cooperative kernel (no kernel ever waits on a separately launched one).
//
// A rank that fails aborts the group (pier_vgroup_abort): every rank blocked
// in a rendezvous returns PIER_EABORTED, like the reference's worker failure
// aborting all barriers (driver.py:494-501).
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pier_comm_internal.h"
#include "pier_common.cuh"

struct PierVGroup {
    int n = 0;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;           // completed rendezvous
    bool aborted = false;
    int status = PIER_OK;       // leader status of the last completed rendezvous
    std::string msg;
    std::vector<void*> slots[2];           // payloads, double-buffered by generation parity
    std::vector<cudaEvent_t> ev_in;        // rank q's stream reached the rendezvous
    cudaEvent_t ev_out = nullptr;          // the leader's work is done
    std::atomic<int> refs{0};
};

namespace pier {

int vg_rendezvous(PierComm* c, void* payload, cudaStream_t st, const VgLeader& leader, void** out) {
    PierVGroup* g = c->vg;
    if (!g) return set_error(PIER_EINVAL, "rendezvous: not a virtual group");
    cudaSetDevice(g->device);
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->aborted) return set_error(PIER_EABORTED, "virtual group aborted by a failing rank");
    const uint64_t my = g->gen;
    std::vector<void*>& sl = g->slots[my & 1];
    cudaError_t e = cudaEventRecord(g->ev_in[c->rank], st);
    if (e != cudaSuccess) {   // this rank cannot take part: release everybody
        g->aborted = true;
        g->cv.notify_all();
        return cuda_status(e, "rendezvous: cudaEventRecord");
    }
    sl[c->rank] = payload;
    if (++g->arrived == g->n) {
        // leader: order after every rank's stream, run the collective work, publish
        int rc = PIER_OK;
        for (int q = 0; q < g->n && rc == PIER_OK; ++q) {
            cudaError_t w = cudaStreamWaitEvent(st, g->ev_in[q], 0);
            if (w != cudaSuccess) rc = cuda_status(w, "rendezvous: cudaStreamWaitEvent");
        }
        if (rc == PIER_OK && leader) rc = leader(sl.data(), st);
        if (rc == PIER_OK) {
            cudaError_t w = cudaEventRecord(g->ev_out, st);
            if (w != cudaSuccess) rc = cuda_status(w, "rendezvous: cudaEventRecord(out)");
        }
        g->status = rc;
        g->msg = rc == PIER_OK ? std::string() : std::string(pier_last_error());
        g->arrived = 0;
        ++g->gen;
        g->cv.notify_all();
    } else {
        g->cv.wait(lk, [&] { return g->gen != my || g->aborted; });
        if (g->gen == my) {
            // aborted while waiting: withdraw so a later rendezvous does not count us
            --g->arrived;
            return set_error(PIER_EABORTED, "virtual group aborted by a failing rank");
        }
        if (g->status == PIER_OK) {
            cudaError_t w = cudaStreamWaitEvent(st, g->ev_out, 0);
            if (w != cudaSuccess) return cuda_status(w, "rendezvous: cudaStreamWaitEvent(out)");
        }
    }
    if (out)
        for (int q = 0; q < g->n; ++q) out[q] = sl[q];
    if (g->status != PIER_OK) return set_error(g->status, g->msg);
    return PIER_OK;
}

int require_nccl(const PierComm* c, const char* what) {
    if (c && c->nccl) return PIER_OK;
    return set_error(PIER_EINVAL, std::string(what) + ": needs an NCCL communicator (not available on a virtual "
                                                      "group; use the p2p exchanges)");
}

void shared_release(PierComm* c, PierSharedBuf& b) {
    if (!b.local) return;
    if (!c->vg)
        for (int r = 0; r < c->nranks; ++r)
            if (r != c->rank && b.peers[r]) cudaIpcCloseMemHandle(b.peers[r]);
    cudaFree(b.local);   // virtual peers are the other ranks' own allocations
    b = PierSharedBuf();
}

// ---- round timeout diagnostics ------------------------------------------------
static std::mutex g_diag_mu;
static std::vector<volatile uint32_t*> g_diag;

void register_diag(volatile uint32_t* slot) {
    std::lock_guard<std::mutex> lk(g_diag_mu);
    g_diag.push_back(slot);
}

void unregister_diag(volatile uint32_t* slot) {
    std::lock_guard<std::mutex> lk(g_diag_mu);
    for (auto& s : g_diag)
        if (s == slot) s = nullptr;
}

std::string round_diag_text() {
    std::lock_guard<std::mutex> lk(g_diag_mu);
    std::string out;
    for (volatile uint32_t* d : g_diag) {
        if (!d || d[0] != 1u) continue;
        const char* what = d[5] == 0 ? "ready counter of span" : "done counter (span index = spans walked)";
        out += " [round wait timed out: team rank " + std::to_string(d[1]) + " waited on team rank " +
               std::to_string(d[6]) + "'s " + what + " " + std::to_string(d[2]) + ": observed " +
               std::to_string(d[3]) + " < target " + std::to_string(d[4]) + "]";
    }
    return out;
}

int comm_setup(PierComm* c) {
    // round signal block + fused-norm slots, mapped into every rank (collective)
    void* p = nullptr;
    int32_t id = -1;
    if (int e = pier_comm_alloc_shared(c, pier_round_sig_bytes(), &p, &id)) return e;
    c->sig_id = id;
    if (int e = pier_comm_alloc_shared(c, 2 * PIER_MAX_RANKS * sizeof(double), &p, &id)) return e;
    c->slots_id = id;
    void* h = nullptr;
    PIER_CHECK_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
    memset(h, 0, 64);
    c->diag_host = (volatile uint32_t*)h;
    PIER_CHECK_CUDA(cudaHostGetDevicePointer((void**)&c->diag_dev, h, 0));
    register_diag(c->diag_host);
    if (const char* s = getenv("PIER_ROUND_TIMEOUT_S")) {
        double v = atof(s);
        if (v > 0) c->timeout_ns = (uint64_t)(v * 1e9);
    }
    return PIER_OK;
}

}  // namespace pier

using namespace pier;

extern "C" {

int pier_vgroup_create(int32_t n, PierComm** out) {
    if (n < 1 || n > PIER_MAX_RANKS || !out) return set_error(PIER_EINVAL, "vgroup_create: 1..8 ranks");
    auto* g = new (std::nothrow) PierVGroup();
    if (!g) return set_error(PIER_ENOMEM, "vgroup_create: host alloc");
    g->n = n;
    PIER_CHECK_CUDA(cudaGetDevice(&g->device));
    g->slots[0].assign(n, nullptr);
    g->slots[1].assign(n, nullptr);
    g->ev_in.resize(n);
    for (int q = 0; q < n; ++q) PIER_CHECK_CUDA(cudaEventCreateWithFlags(&g->ev_in[q], cudaEventDisableTiming));
    PIER_CHECK_CUDA(cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming));
    std::vector<PierComm*> cs(n);
    for (int r = 0; r < n; ++r) {
        auto* c = new (std::nothrow) PierComm();
        if (!c) return set_error(PIER_ENOMEM, "vgroup_create: host alloc");
        c->rank = r;
        c->nranks = n;
        c->vg = g;
        g->refs.fetch_add(1);
        PIER_CHECK_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming));
        PIER_CHECK_CUDA(cudaEventCreateWithFlags(&c->end, cudaEventDisableTiming));
        cs[r] = c;
    }
    // the setup allocations are collective: run them with one helper thread per rank
    std::vector<int> rcs(n, PIER_OK);
    std::vector<std::string> msgs(n);
    {
        std::vector<std::thread> th;
        for (int r = 0; r < n; ++r)
            th.emplace_back([&, r] {
                cudaSetDevice(g->device);
                rcs[r] = comm_setup(cs[r]);
                if (rcs[r]) {
                    msgs[r] = pier_last_error();
                    pier_vgroup_abort(cs[r]);
                }
            });
        for (auto& t : th) t.join();
    }
    for (int r = 0; r < n; ++r)
        if (rcs[r]) return set_error(rcs[r], "vgroup_create: " + msgs[r]);
    for (int r = 0; r < n; ++r) out[r] = cs[r];
    return PIER_OK;
}

int pier_vgroup_abort(PierComm* c) {
    if (!c || !c->vg) return set_error(PIER_EINVAL, "vgroup_abort: not a virtual group");
    std::lock_guard<std::mutex> lk(c->vg->mu);
    c->vg->aborted = true;
    c->vg->cv.notify_all();
    return PIER_OK;
}

int pier_comm_is_virtual(const PierComm* c) { return c && c->vg ? 1 : 0; }

int pier_comm_set_timeout(PierComm* c, double seconds) {
    if (!c || !(seconds > 0.0)) return set_error(PIER_EINVAL, "comm_set_timeout: positive seconds");
    c->timeout_ns = (uint64_t)(seconds * 1e9);
    return PIER_OK;
}

int pier_comm_diag(const PierComm* c, uint32_t* out7) {
    if (!c || !out7) return set_error(PIER_EINVAL, "comm_diag: null");
    for (int i = 0; i < 7; ++i) out7[i] = c->diag_host ? c->diag_host[i] : 0u;
    return PIER_OK;
}

}  // extern "C"

namespace pier {
// called by pier_comm_destroy for a virtual handle: drop the group reference
void vgroup_release(PierComm* c) {
    PierVGroup* g = c->vg;
    if (!g) return;
    c->vg = nullptr;
    if (g->refs.fetch_sub(1) == 1) {
        for (auto e : g->ev_in) cudaEventDestroy(e);
        if (g->ev_out) cudaEventDestroy(g->ev_out);
        delete g;
    }
}
}  // namespace pier
