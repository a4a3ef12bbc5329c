// NVLink pull/push probe (one process, 2 GPUs, peer access): how close do
// SM-driven LDG.128 loads, TMA bulk copies (cp.async.bulk, mbarrier) and the
// copy engines get to the link rate?  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -o tools/tma_probe
//   ./tools/tma_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kThreads = 256;

// LDG pull: every thread loads float4s from the peer buffer, xor-accumulates (keeps loads live)
__global__ void pull_ldg(const float4* __restrict__ src, int64_t nvec, float4* sink) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t i = blockIdx.x * (int64_t)kThreads * 4 + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * kThreads * 4) {
        float4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int64_t j = i + (int64_t)k * kThreads;
            x[k] = j < nvec ? __ldcg(src + j) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) { acc.x += x[k].x; acc.y += x[k].y; acc.z += x[k].z; acc.w += x[k].w; }
    }
    if (acc.x == 12345.f) sink[threadIdx.x] = acc;
}

// LDG push: every thread stores float4s into the peer buffer
__global__ void push_stg(float4* __restrict__ dst, int64_t nvec) {
    float4 v = make_float4(1, 2, 3, 4);
    for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * kThreads)
        __stcg(dst + i, v);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk pull: one elected thread streams CHUNK-byte pieces of the peer buffer
// into a STAGES-deep shared-memory ring, completion tracked by mbarriers.
template <int CHUNK, int STAGES>
__global__ void pull_tma(const char* __restrict__ src, int64_t nbytes, float* sink) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    const int64_t nchunks = nbytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t k = 0;
        uint32_t phase[STAGES] = {0};
        // prologue
        int64_t c = blockIdx.x;
        for (int s = 0; s < STAGES && c < nchunks; ++s, c += gridDim.x) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(CHUNK));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + s * CHUNK)), "l"(src + c * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[s]))
                         : "memory");
        }
        for (int64_t cc = blockIdx.x; cc < nchunks; cc += gridDim.x, ++k) {
            int s = (int)(k % STAGES);
            // wait for stage s
            asm volatile(
                "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
                ::"r"(smem_u32(&bar[s])), "r"(phase[s]));
            phase[s] ^= 1;
            int64_t nxt = cc + (int64_t)STAGES * gridDim.x;
            if (nxt < nchunks) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(CHUNK));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(smem + s * CHUNK)), "l"(src + nxt * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[s]))
                             : "memory");
            }
        }
        if (((float*)smem)[0] == 12345.f) sink[0] = 1.f;
    }
}

// TMA bulk push: shared memory -> peer global, bulk groups
template <int CHUNK, int STAGES>
__global__ void push_tma(char* __restrict__ dst, int64_t nbytes) {
    extern __shared__ __align__(128) char smem[];
    for (int i = threadIdx.x; i < CHUNK * STAGES / 4; i += blockDim.x) ((float*)smem)[i] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int64_t nchunks = nbytes / CHUNK;
    int64_t k = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        int s = (int)(k % STAGES);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst + c * CHUNK), "r"(smem_u32(smem + s * CHUNK)), "r"(CHUNK) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int64_t nbytes = 4ll << 30;
    int nd = 0;
    CK(cudaGetDeviceCount(&nd));
    if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
    char *buf[2], *dst[2];
    float* sink[2];
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&buf[d], nbytes));
        CK(cudaMalloc(&dst[d], nbytes));
        CK(cudaMalloc(&sink[d], 4096));
        CK(cudaMemset(buf[d], 0, nbytes));
        CK(cudaStreamCreate(&st[d]));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
        CK(cudaFuncSetAttribute(pull_tma<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4));
        CK(cudaFuncSetAttribute(push_tma<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4));
    }
    const char* names[] = {"pull_ldg", "push_stg", "pull_tma", "push_tma", "memcpy"};
    for (int kind = 0; kind < 5; ++kind) {
        for (int both = 0; both < 2; ++both) {
            for (int rep = 0; rep < 3; ++rep) {
                for (int d = 0; d <= both; ++d) {
                    CK(cudaSetDevice(d));
                    CK(cudaEventRecord(e0[d], st[d]));
                    const int o = 1 - d;  // peer
                    switch (kind) {
                        case 0: pull_ldg<<<sms * 4, kThreads, 0, st[d]>>>((const float4*)buf[o], nbytes / 16, (float4*)sink[d]); break;
                        case 1: push_stg<<<sms * 4, kThreads, 0, st[d]>>>((float4*)dst[o], nbytes / 16); break;
                        case 2: pull_tma<16384, 4><<<sms * 2, 32, 16384 * 4, st[d]>>>(buf[o], nbytes, sink[d]); break;
                        case 3: push_tma<16384, 4><<<sms * 2, 32, 16384 * 4, st[d]>>>(dst[o], nbytes); break;
                        case 4: CK(cudaMemcpyPeerAsync(dst[o], o, buf[d], d, nbytes, st[d])); break;
                    }
                    CK(cudaGetLastError());
                    CK(cudaEventRecord(e1[d], st[d]));
                }
                for (int d = 0; d <= both; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamSynchronize(st[d])); }
            }
            float ms = 0;
            CK(cudaSetDevice(0));
            CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
            printf("{\"kind\": \"%s\", \"both_directions\": %d, \"ms\": %.3f, \"GBps_per_direction\": %.1f}\n",
                   names[kind], both, ms, nbytes / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
