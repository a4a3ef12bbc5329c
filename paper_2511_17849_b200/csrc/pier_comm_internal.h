// Internal definition of the group communicator shared by pier_comm.cu (NCCL
// bucketed path) and pier_p2p.cu (fused peer-memory path).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <functional>
#include <string>
#include <vector>

#define PIER_MAX_RANKS 8

struct PierVGroup;  // n virtual ranks on one device (pier_vgroup.cpp)

// A buffer allocated collectively and mapped into every rank's address space
// (CUDA IPC over NVLink): peers[r] is rank r's copy, peers[rank] our own.
struct PierSharedBuf {
    void* local = nullptr;
    size_t bytes = 0;
    void* peers[PIER_MAX_RANKS] = {};
};

// An NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister) with a
// multicast (NVLS) mapping, used by the in-switch reduction path.
struct PierWindowBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
};

struct PierComm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1;
    cudaStream_t cs = nullptr;          // NCCL stream (bucketed path)
    cudaStream_t ps = nullptr;          // exchange stream of the pipelined p2p round
    cudaEvent_t start = nullptr, end = nullptr;
    std::vector<cudaEvent_t> ev_rs, ev_k3;
    std::vector<PierSharedBuf> shared;  // id -> buffer (freed slots have local == nullptr)
    float* d_barrier = nullptr;         // 1-element buffer for stream-ordered barriers
    std::vector<PierWindowBuf> windows; // NVLS windows
    ncclDevComm devcomm{};              // device communicator (LSA barriers + multimem)
    bool devcomm_ok = false;
    int32_t sig_id = -1;                // shared signal block of the persistent round kernel
    int32_t slots_id = -1;              // shared fp64 slots of the fused-norm gradient mean
    uint32_t round_epoch = 0;           // rounds launched (all ranks advance in lockstep)
    // host-mapped diagnostic slot the round kernel fills before it traps on a
    // timed-out wait: {flag, rank, span, observed, target, kind, peer}; set up at init
    volatile uint32_t* diag_host = nullptr;
    uint32_t* diag_dev = nullptr;
    uint64_t timeout_ns = 20ull * 1000000000ull;  // spin limit of the round kernel's waits
    // virtual group: this handle is one of n ranks living on ONE device, driven
    // by one host thread each; collectives rendezvous on the host instead of NCCL
    PierVGroup* vg = nullptr;
};

namespace pier {
int comm_free_shared_all(PierComm* c);
int comm_free_windows(PierComm* c);
// team = strictly ascending ranks containing the caller (NULL: all ranks) ->
// members[], team size n, the caller's index r
int resolve_team(const PierComm* c, const int32_t* team, int32_t nteam, int32_t* members, int* n, int* r);
// stream-ordered barrier over the whole communicator (1-element ncclAllReduce,
// or the host rendezvous of a virtual group)
int barrier(PierComm* c, cudaStream_t st);
// per-communicator setup shared by pier_comm_init and pier_vgroup_create: the
// round signal block, the fused-norm slots and the diagnostic slot
int comm_setup(PierComm* c);
// nccl-only entry points refuse virtual groups
int require_nccl(const PierComm* c, const char* what);

// Virtual-group rendezvous: every rank of c's group calls it (from its own
// host thread) with a payload pointer.  The LAST rank to arrive waits (on its
// stream) for every rank's stream to reach the call, runs
// `leader(payloads, stream)` -- payloads[q] = rank q's pointer -- and every
// rank's stream then waits for the leader's work.  All ranks return the
// leader's status; `out` (optional, n entries) receives the payloads.  A
// group aborted by pier_vgroup_abort returns PIER_EABORTED everywhere.
using VgLeader = std::function<int(void* const* payloads, cudaStream_t st)>;
int vg_rendezvous(PierComm* c, void* payload, cudaStream_t st, const VgLeader& leader, void** out = nullptr);
// free / close the shared buffers of one handle (IPC peers or virtual peers)
void shared_release(PierComm* c, struct PierSharedBuf& b);
// timed-out round waits recorded in the diagnostic slots (empty when none)
std::string round_diag_text();
void register_diag(volatile uint32_t* slot);
void unregister_diag(volatile uint32_t* slot);
// pier_comm_destroy of a virtual handle: drop its reference on the group
void vgroup_release(PierComm* c);
}
