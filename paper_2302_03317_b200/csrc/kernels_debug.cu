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

__global__ void k_debug_fy_draws(uint64_t K, const uint64_t* P, const uint32_t* s, uint64_t count, uint32_t* out) {
    const PhiloxKey key = make_key(K);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = fy_draw(key, P[i], s[i]);
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
