// Fused finish: host-side dispatch.  The kernel templates live in
// kernels_finish.cuh and are instantiated per element size in
// kernels_finish_eb{4,8,16}.cu (separate TUs so the library builds in parallel).
#include "kernels_finish.cuh"

namespace shuf {

void* finish_children_kernel_eb4(bool seg, bool narrow, bool ord);
void* finish_children_kernel_eb8(bool seg, bool narrow, bool ord);
void* finish_children_kernel_eb16(bool seg, bool narrow, bool ord);
void* finish_ip_kernel_eb4(bool narrow, bool ord);
void* finish_ip_kernel_eb8(bool narrow, bool ord);
void* finish_ip_kernel_eb16(bool narrow, bool ord);
void* finish_stream_kernel_eb4(bool narrow, bool ord);
void* finish_stream_kernel_eb8(bool narrow, bool ord);
void* finish_stream_kernel_eb16(bool narrow, bool ord);
cudaError_t launch_copy_big_eb4(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_copy_big_eb8(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_copy_big_eb16(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);

uint32_t finish_smem_bytes(uint32_t S_fuse, uint32_t eb, uint32_t k, uint32_t) {
    return finish_layout(S_fuse, eb, k).total;
}
uint32_t finish_stream_smem_bytes(uint32_t S, uint32_t eb, uint32_t k) { return finish_layout(S, eb, k, true).total; }
uint32_t finish_max_elems(uint32_t, uint32_t) { return 65535u; }

static void* fin_stream(uint32_t eb, bool narrow, bool ord) {
    switch (eb) {
    case 4: return finish_stream_kernel_eb4(narrow, ord);
    case 8: return finish_stream_kernel_eb8(narrow, ord);
    default: return finish_stream_kernel_eb16(narrow, ord);
    }
}

cudaError_t configure_finish_stream(uint32_t eb, uint32_t smem) {
    for (int nr = 0; nr < 2; ++nr)
        for (int o = 0; o < 2; ++o) {
            cudaError_t e = cudaFuncSetAttribute(fin_stream(eb, nr, o), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e) return e;
        }
    return cudaSuccess;
}

cudaError_t launch_finish_stream(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = finish_stream_smem_bytes(rp.S_stream, rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(fin_stream(rp.eb, rp.bp.narrow != 0, rp.rank_ordered != 0), dim3(grid), dim3(NTF), args,
                            smem, s);
}
uint32_t finish_smem_budget(uint32_t) { return kSmemLimit; }

static void* fin_fn(uint32_t eb, bool seg, bool narrow, bool ord) {
    switch (eb) {
    case 4: return finish_children_kernel_eb4(seg, narrow, ord);
    case 8: return finish_children_kernel_eb8(seg, narrow, ord);
    default: return finish_children_kernel_eb16(seg, narrow, ord);
    }
}

static void* fin_ip(uint32_t eb, bool narrow, bool ord) {
    switch (eb) {
    case 4: return finish_ip_kernel_eb4(narrow, ord);
    case 8: return finish_ip_kernel_eb8(narrow, ord);
    default: return finish_ip_kernel_eb16(narrow, ord);
    }
}

cudaError_t launch_finish_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k, 1);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(fin_fn(rp.eb, false, rp.bp.narrow != 0, rp.rank_ordered != 0), dim3(grid), dim3(NTF),
                            args, smem, s);
}

cudaError_t launch_finish_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                   cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k, 1);
    void* args[] = {(void*)&rp, (void*)&d_offsets, (void*)&num_segments};
    return cudaLaunchKernel(fin_fn(rp.eb, true, rp.bp.narrow != 0, rp.rank_ordered != 0), dim3(grid), dim3(NTF),
                            args, smem, s);
}

cudaError_t launch_finish_ipchildren(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k, 1);
    void* args[] = {(void*)&rp, (void*)&ip};
    return cudaLaunchKernel(fin_ip(rp.eb, rp.bp.narrow != 0, rp.rank_ordered != 0), dim3(grid), dim3(NTF), args, smem,
                            s);
}

cudaError_t launch_copy_big(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    switch (rp.eb) {
    case 4: return launch_copy_big_eb4(rp, lp, s, grid);
    case 8: return launch_copy_big_eb8(rp, lp, s, grid);
    default: return launch_copy_big_eb16(rp, lp, s, grid);
    }
}

cudaError_t configure_finish(uint32_t) {  // the attribute is the limit: plans of other sizes share the kernels
    for (uint32_t eb : {4u, 8u, 16u})
        for (int seg = 0; seg < 2; ++seg)
            for (int nr = 0; nr < 2; ++nr)
                for (int o = 0; o < 2; ++o) {
                    cudaError_t e = cudaFuncSetAttribute(fin_fn(eb, seg, nr, o),
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
                    if (e) return e;
                    if (seg == 0 && (e = cudaFuncSetAttribute(fin_ip(eb, nr, o),
                                                              cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)))
                        return e;
                }
    return cudaSuccess;
}

cudaError_t occupancy_finish(uint32_t eb, uint32_t smem, int* blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fin_fn(eb, false, true, true), NTF, smem);
}

}  // namespace shuf
