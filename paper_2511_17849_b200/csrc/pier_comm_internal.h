// Internal definition of the group communicator shared by pier_comm.cu (NCCL
// bucketed path) and pier_p2p.cu (fused peer-memory path).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <vector>

#define PIER_MAX_RANKS 8

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
};

namespace pier {
int comm_free_shared_all(PierComm* c);
int comm_free_windows(PierComm* c);
// team = strictly ascending ranks containing the caller (NULL: all ranks) ->
// members[], team size n, the caller's index r
int resolve_team(const PierComm* c, const int32_t* team, int32_t nteam, int32_t* members, int* n, int* r);
// stream-ordered barrier over the whole communicator (1-element ncclAllReduce)
int barrier(PierComm* c, cudaStream_t st);
}
