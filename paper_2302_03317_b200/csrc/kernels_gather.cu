// Element sizes other than 4, 8 and 16 bytes (the
// element-size sweep of P:600-603 / Fig. 7): D6's permutation does not depend
// on the element size (D6), so the library shuffles the index
// array 0..n-1 (u32, or u64 above 2^32 elements) with the native kernels and
// then moves the elements once: out[i] = in[idx[i]].
#include <cuda_runtime.h>

#include "shuf_internal.cuh"

namespace shuf {

template <typename I>
__global__ void k_iota(I* idx, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        idx[i] = (I)i;
}

// out[i] = in[idx[i]] for elements of eb bytes, moved in units U (16, 4, 2 or
// 1 bytes; eb a multiple of U): thread t copies unit t % (eb/U) of element
// t / (eb/U), so consecutive threads write consecutive units (coalesced).
template <typename I, typename U>
__global__ void k_gather(const unsigned char* __restrict__ in, unsigned char* __restrict__ out,
                         const I* __restrict__ idx, uint64_t n, uint32_t upe) {
    const U* src = reinterpret_cast<const U*>(in);
    U* dst = reinterpret_cast<U*>(out);
    const uint64_t total = n * upe;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = t / upe, u = t - i * upe;
        dst[t] = src[(uint64_t)idx[i] * upe + u];
    }
}

cudaError_t launch_iota(void* idx, uint32_t ieb, uint64_t n, cudaStream_t s, int grid) {
    if (ieb == 4) k_iota<uint32_t><<<grid, 256, 0, s>>>(static_cast<uint32_t*>(idx), n);
    else k_iota<uint64_t><<<grid, 256, 0, s>>>(static_cast<uint64_t*>(idx), n);
    return cudaGetLastError();
}

template <typename I>
static void gather_as(const unsigned char* in, unsigned char* out, const void* idx, uint64_t n, uint32_t eb,
                      cudaStream_t s, int grid) {
    const I* ix = static_cast<const I*>(idx);
    if (eb % 16 == 0) k_gather<I, uint4><<<grid, 256, 0, s>>>(in, out, ix, n, eb / 16);
    else if (eb % 4 == 0) k_gather<I, uint32_t><<<grid, 256, 0, s>>>(in, out, ix, n, eb / 4);
    else if (eb % 2 == 0) k_gather<I, uint16_t><<<grid, 256, 0, s>>>(in, out, ix, n, eb / 2);
    else k_gather<I, unsigned char><<<grid, 256, 0, s>>>(in, out, ix, n, eb);
}

cudaError_t launch_gather(const void* in, void* out, const void* idx, uint32_t ieb, uint64_t n, uint32_t eb,
                          cudaStream_t s, int grid) {
    const unsigned char* i8 = static_cast<const unsigned char*>(in);
    unsigned char* o8 = static_cast<unsigned char*>(out);
    if (ieb == 4) gather_as<uint32_t>(i8, o8, idx, n, eb, s, grid);
    else gather_as<uint64_t>(i8, o8, idx, n, eb, s, grid);
    return cudaGetLastError();
}

}  // namespace shuf
