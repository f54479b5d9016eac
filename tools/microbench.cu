// Microbenchmarks of the primitives the shuffle kernels are built from, on
// the B200: Philox4x32-10 throughput, warp match_any, shared-memory atomics,
// plain HBM copy.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2302_03317_b200/csrc/philox.cuh"
using namespace shuf;

#define CK(x) do { cudaError_t e = (x); if (e) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_philox(uint64_t groups, uint32_t* out) {
    PhiloxKey key{0x12345678u, 0x9abcdef0u};
    uint32_t acc = 0;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * blockDim.x) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0, 1), key);
        acc ^= w.x ^ w.y ^ w.z ^ w.w;
    }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_match(int iters, uint32_t* out) {
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t b = (v >> 8) & 255u;
        uint32_t m = __match_any_sync(0xFFFFFFFFu, b);
        acc += __popc(m);
        v = v * 1664525u + 1013904223u;
    }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_ballot8(int iters, uint32_t* out) {
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x;
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint32_t b = (v >> 8) & 255u;
        uint32_t m = 0xFFFFFFFFu;
#pragma unroll
        for (int bit = 0; bit < 8; ++bit) {
            uint32_t bb = __ballot_sync(0xFFFFFFFFu, (b >> bit) & 1u);
            m &= ((b >> bit) & 1u) ? bb : ~bb;
        }
        acc += __popc(m);
        v = v * 1664525u + 1013904223u;
    }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_satomic(int iters, uint32_t* out) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t v = (threadIdx.x * 2654435761u) ^ blockIdx.x;
    for (int i = 0; i < iters; ++i) {
        atomicAdd(&h[(v >> 8) & 255u], 1u);
        v = v * 1664525u + 1013904223u;
    }
    __syncthreads();
    if (h[threadIdx.x & 255] == 0x12345) out[0] = 1;
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out; CK(cudaMalloc(&out, 16));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    // Philox
    uint64_t groups = 1ull << 28;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_philox<<<sms * 8, 256>>>(groups, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("philox: %.3f ms for 2^28 calls -> %.3g calls/s (%.2f calls/clk/SM at %d MHz)\n", ms, groups / (ms * 1e-3),
           groups / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_match<<<sms * 8, 256>>>(iters, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double lanes = (double)sms * 8 * 256 * iters;
    printf("match_any(256 values): %.3f ms -> %.2f lane-ops/clk/SM\n", ms, lanes / (ms * 1e-3) / sms / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_ballot8<<<sms * 8, 256>>>(iters, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("8x ballot multisplit: %.3f ms -> %.2f lane-ops/clk/SM\n", ms, lanes / (ms * 1e-3) / sms / (clk * 1e3));
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_satomic<<<sms * 8, 256>>>(iters, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("smem atomicAdd (256 bins): %.3f ms -> %.2f lane-ops/clk/SM\n", ms, lanes / (ms * 1e-3) / sms / (clk * 1e3));
    uint64_t nbytes = 4ull << 30;
    uint4 *a, *b; CK(cudaMalloc(&a, nbytes)); CK(cudaMalloc(&b, nbytes));
    cudaMemset(a, 1, nbytes);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_copy<<<sms * 4, 512>>>(a, b, nbytes / 16);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("copy 4 GiB (uint4 grid-stride): %.3f ms -> %.1f GB/s (read+write)\n", ms, 2.0 * nbytes / (ms * 1e-3) / 1e9);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaMemcpyAsync(b, a, nbytes, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("cudaMemcpy D2D 4 GiB: %.3f ms -> %.1f GB/s (read+write)\n", ms, 2.0 * nbytes / (ms * 1e-3) / 1e9);
    return 0;
}
