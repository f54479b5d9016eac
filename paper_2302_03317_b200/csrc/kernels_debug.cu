// Raw-draw dump kernels (test hooks shuf_debug_bucket_draws / _fy_draws):
// the device D4/D5 draws, one thread per output, for parity with the oracle.
#include <cuda_runtime.h>

#include "philox.cuh"
#include "shuf_internal.cuh"

namespace shuf {

__global__ void k_debug_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, BucketParams bp,
                                     uint32_t* out) {
    const PhiloxKey key = make_key(K);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = bucket_draw(key, level, p0 + i, bp);
}

__global__ void k_debug_fy_draws(uint64_t K, const uint64_t* q, const uint32_t* step, uint64_t count, uint32_t* out) {
    const PhiloxKey key = make_key(K);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = fy_draw(key, q[i], step[i]);
}

// Probe: do same-address shared atomicAdds of one warp instruction return in
// ascending lane order?  Random bucket patterns (2..256 distinct values,
// partial masks); counts lane pairs that violate the order.
__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void k_rank_order_probe(uint32_t* viol) {
    __shared__ uint32_t C[16 * 256];
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t* T = C + w * 256;
    uint32_t bad = 0;
    for (uint32_t t = 0; t < 512; ++t) {
        for (uint32_t i = lane; i < 256; i += 32) T[i] = probe_hash(t * 977u + i) & 0xFFu;
        __syncwarp();
        const uint32_t h = probe_hash((blockIdx.x * 1315423911u) ^ (threadIdx.x * 2654435761u) ^ (t * 97u));
        const uint32_t K = 2u << (t & 7u);  // 2 .. 256 distinct addresses
        const uint32_t b = h % K;
        const bool active = (t & 8u) ? ((h >> 20) & 1u) : true;
        uint32_t r = 0;
        if (active) r = atomicAdd(&T[b], (t & 16u) ? (1u << 16) : 1u);
        __syncwarp();
        for (uint32_t j = 0; j < 32; ++j) {
            const uint32_t bj = __shfl_sync(0xFFFFFFFFu, b, j), rj = __shfl_sync(0xFFFFFFFFu, r, j);
            const uint32_t aj = __shfl_sync(0xFFFFFFFFu, active ? 1u : 0u, j);
            if (active && aj && j > lane && bj == b && !(rj > r)) ++bad;
        }
        __syncwarp();
    }
    if (bad) atomicAdd(viol, bad);
}

cudaError_t launch_rank_order_probe(int grid, uint32_t* d_violations, cudaStream_t s) {
    k_rank_order_probe<<<grid, 512, 0, s>>>(d_violations);
    return cudaGetLastError();
}

cudaError_t launch_debug_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k,
                                      uint32_t* d_out, cudaStream_t s) {
    uint64_t blocks = (count + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    k_debug_bucket_draws<<<(unsigned)blocks, 256, 0, s>>>(K, level, p0, count, make_bucket_params(k), d_out);
    return cudaGetLastError();
}

cudaError_t launch_debug_fy_draws(uint64_t K, const uint64_t* d_P, const uint32_t* d_s, uint64_t count,
                                  uint32_t* d_out, cudaStream_t s) {
    uint64_t blocks = (count + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    k_debug_fy_draws<<<(unsigned)blocks, 256, 0, s>>>(K, d_P, d_s, count, d_out);
    return cudaGetLastError();
}

}  // namespace shuf
