// Instantiations of the fused-finish kernels for 4-byte elements (one TU per
// element size so the library builds in parallel).
#include "kernels_finish.cuh"

namespace shuf {

void* finish_children_kernel_eb4(bool seg, bool narrow, bool ord) {
    if (seg) {
        if (ord) return narrow ? (void*)k_finish_segments<4, true, true> : (void*)k_finish_segments<4, false, true>;
        return narrow ? (void*)k_finish_segments<4, true, false> : (void*)k_finish_segments<4, false, false>;
    }
    if (ord) return narrow ? (void*)k_finish_children<4, true, true> : (void*)k_finish_children<4, false, true>;
    return narrow ? (void*)k_finish_children<4, true, false> : (void*)k_finish_children<4, false, false>;
}

void* finish_ip_kernel_eb4(bool narrow, bool ord) {
    if (ord) return narrow ? (void*)k_finish_ipchildren<4, true, true> : (void*)k_finish_ipchildren<4, false, true>;
    return narrow ? (void*)k_finish_ipchildren<4, true, false> : (void*)k_finish_ipchildren<4, false, false>;
}

void* finish_stream_kernel_eb4(bool narrow, bool ord) {
    if (ord) return narrow ? (void*)k_finish_stream<4, true, true> : (void*)k_finish_stream<4, false, true>;
    return narrow ? (void*)k_finish_stream<4, true, false> : (void*)k_finish_stream<4, false, false>;
}

cudaError_t launch_copy_big_eb4(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    k_copy_big<4><<<grid, 256, 0, s>>>(rp, lp);
    return cudaGetLastError();
}

}  // namespace shuf
