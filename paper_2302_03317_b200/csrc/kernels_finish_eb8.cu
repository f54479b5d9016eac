// Instantiations of the fused-finish kernels for 8-byte elements (one TU per
// element size so the library builds in parallel).
#include "kernels_finish.cuh"

namespace shuf {

void* finish_children_kernel_eb8(bool seg, bool narrow, bool ord) {
    if (seg) {
        if (ord) return narrow ? (void*)k_finish_segments<8, true, true> : (void*)k_finish_segments<8, false, true>;
        return narrow ? (void*)k_finish_segments<8, true, false> : (void*)k_finish_segments<8, false, false>;
    }
    if (ord) return narrow ? (void*)k_finish_children<8, true, true> : (void*)k_finish_children<8, false, true>;
    return narrow ? (void*)k_finish_children<8, true, false> : (void*)k_finish_children<8, false, false>;
}

void* finish_ip_kernel_eb8(bool narrow, bool ord) {
    if (ord) return narrow ? (void*)k_finish_ipchildren<8, true, true> : (void*)k_finish_ipchildren<8, false, true>;
    return narrow ? (void*)k_finish_ipchildren<8, true, false> : (void*)k_finish_ipchildren<8, false, false>;
}

void* finish_stream_kernel_eb8(bool narrow, bool ord) {
    if (ord) return narrow ? (void*)k_finish_stream<8, true, true> : (void*)k_finish_stream<8, false, true>;
    return narrow ? (void*)k_finish_stream<8, true, false> : (void*)k_finish_stream<8, false, false>;
}

cudaError_t launch_copy_big_eb8(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    k_copy_big<8><<<grid, 256, 0, s>>>(rp, lp);
    return cudaGetLastError();
}

}  // namespace shuf
