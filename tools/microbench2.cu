// Microbenchmarks for the tile-ranking design choice:
//  (1) is the return order of same-address shared-memory atomicAdd within one
//      warp instruction ascending in lane id on this GPU?  (checked, not assumed)
//  (2) throughput of ranking rounds: ordered atomicAdd, atomicOr peers, match_any
//  (3) scattered STS throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// (1) ordering check: per trial, each lane draws b in [0,K); per-warp table.
__global__ void k_order(int trials, int K, int mode, unsigned long long* viol, unsigned long long* checked) {
    extern __shared__ uint32_t C[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* T = C + w * 256;
    unsigned long long v = 0, c = 0;
    for (int t = 0; t < trials; ++t) {
        for (int i = lane; i < 256; i += 32) T[i] = (mode == 1) ? (hash32(t * 977 + i) & 1023) : 0;
        __syncwarp();
        uint32_t h = hash32((blockIdx.x * 1315423911u) ^ (threadIdx.x * 2654435761u) ^ (t * 97u));
        uint32_t b = (mode == 2) ? 7 : (h % K);
        bool active = (mode == 3) ? ((h >> 20) & 1) : true;
        uint32_t r = 0;
        if (active) r = atomicAdd(&T[b], 1u);
        __syncwarp();
        // gather all lanes' (b, r, active) and check order
        for (int j = 0; j < 32; ++j) {
            uint32_t bj = __shfl_sync(0xffffffffu, b, j), rj = __shfl_sync(0xffffffffu, r, j);
            bool aj = __shfl_sync(0xffffffffu, active ? 1 : 0, j);
            if (active && aj && j > lane && bj == b) { c++; if (!(rj > r)) v++; }
        }
        __syncwarp();
    }
    atomicAdd(viol, v);
    atomicAdd(checked, c);
}

// (2a) ordered-atomic ranking rounds
__global__ void k_rank_atom(int iters, uint32_t* out) {
    __shared__ uint32_t C[16 * 256];
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) C[i] = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5;
    uint32_t* T = C + w * 256;
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x, acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t b = (v >> 8) & 255u;
        acc += atomicAdd(&T[b], 1u);
        v = v * 1664525u + 1013904223u;
    }
    if (acc == 0x12345) out[0] = acc;
}

// (2b) atomicOr peers + counter ranking rounds (documented-deterministic)
__global__ void k_rank_or(int iters, uint32_t* out) {
    __shared__ uint32_t M[16 * 256];
    __shared__ uint32_t C[16 * 256];
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) { M[i] = 0; C[i] = 0; }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* Mw = M + w * 256; uint32_t* Cw = C + w * 256;
    uint32_t lt = (1u << lane) - 1u;
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x, acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t b = (v >> 8) & 255u;
        atomicOr(&Mw[b], 1u << lane);
        __syncwarp();
        uint32_t peers = Mw[b];
        uint32_t c = Cw[b];
        __syncwarp();
        if ((peers & lt) == 0) { Mw[b] = 0; Cw[b] = c + __popc(peers); }
        __syncwarp();
        acc += c + __popc(peers & lt);
        v = v * 1664525u + 1013904223u;
    }
    if (acc == 0x12345) out[0] = acc;
}

// (3) scattered 4-byte smem stores (random slots in 64 KB) + sequential reads
__global__ void k_sts(int iters, uint32_t* out) {
    extern __shared__ uint32_t S[];
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x, acc = 0;
    for (int i = 0; i < iters; ++i) {
        S[(v >> 8) & 16383u] = v;
        v = v * 1664525u + 1013904223u;
    }
    __syncthreads();
    acc = S[threadIdx.x];
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_lds_seq(int iters, uint32_t* out) {
    extern __shared__ uint32_t S[];
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) S[i] = i;
    __syncthreads();
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) acc += S[(threadIdx.x + i * 512) & 16383u];
    if (acc == 0x12345) out[0] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned long long *viol, *chk; CK(cudaMalloc(&viol, 8)); CK(cudaMalloc(&chk, 8));
    uint32_t* out; CK(cudaMalloc(&out, 16));
    const char* mname[] = {"random b", "random init", "all same", "partial mask"};
    for (int mode = 0; mode < 4; ++mode) for (int K : {2, 4, 16, 256}) {
        cudaMemset(viol, 0, 8); cudaMemset(chk, 0, 8);
        k_order<<<sms * 2, 512, 16 * 256 * 4>>>(2000, K, mode, viol, chk);
        CK(cudaDeviceSynchronize());
        unsigned long long v, c; cudaMemcpy(&v, viol, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&c, chk, 8, cudaMemcpyDeviceToHost);
        printf("order test mode=%s K=%d: same-address lane pairs checked %llu, out-of-lane-order %llu\n", mname[mode], K, c, v);
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms; int iters = 4096;
    double lanes = (double)sms * 4 * 512 * iters;
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(e0); k_rank_atom<<<sms * 4, 512>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    printf("rank via atomicAdd: %.2f lanes/clk/SM\n", lanes / (ms * 1e-3) / sms / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(e0); k_rank_or<<<sms * 4, 512>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    printf("rank via atomicOr peers: %.2f lanes/clk/SM\n", lanes / (ms * 1e-3) / sms / (clk * 1e3));
    cudaFuncSetAttribute(k_sts, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(k_lds_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(e0); k_sts<<<sms * 3, 512, 65536>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    lanes = (double)sms * 3 * 512 * iters;
    printf("scattered STS.32: %.2f lanes/clk/SM\n", lanes / (ms * 1e-3) / sms / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(e0); k_lds_seq<<<sms * 3, 512, 65536>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    printf("sequential LDS.32: %.2f lanes/clk/SM\n", lanes / (ms * 1e-3) / sms / (clk * 1e3));
    return 0;
}
