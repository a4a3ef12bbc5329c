// Internal definition of the group communicator shared by pier_comm.cu (NCCL
// bucketed path) and pier_p2p.cu (fused peer-memory path).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <vector>

#define PIER_MAX_RANKS 8

// A buffer allocated collectively and mapped into every rank's address space
// (CUDA IPC over NVLink): peers[r] is rank r's copy, peers[rank] our own.
struct PierSharedBuf {
    void* local = nullptr;
    size_t bytes = 0;
    void* peers[PIER_MAX_RANKS] = {};
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
};

namespace pier {
int comm_free_shared_all(PierComm* c);
}
