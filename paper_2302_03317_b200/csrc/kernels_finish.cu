// Fused finish: every segment of at most S_fuse elements is finished by one
// CTA in a single HBM round trip -- all of its remaining scatter levels run
// on a u16 index permutation in shared memory, every leaf (<= L elements) is
// Fisher-Yates'd on that permutation (Fig. 1), and the element
// data (staged in shared memory by a bulk async copy that overlaps the index
// work) is gathered once into its final place in ptr.
//
// The permutation never depends on element values (D6), so the
// index work needs no data and hides the load latency.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

struct FinishLayout {
    uint32_t data, idx, tmp, draws, cwb, bst, wsum, front0, front1, misc, bar, total;
};

__host__ __device__ inline FinishLayout finish_layout(uint32_t S, uint32_t eb, uint32_t k) {
    // every region starts 16-byte aligned (bulk-copy target, mbarrier, u64 views)
    FinishLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    f.data = take(S * eb + 32);
    f.bst = take((k + 1) * 4);
    f.wsum = take((kWarps + 1) * 4);
    f.front0 = take(kFrontierCap * 4);
    f.front1 = take(kFrontierCap * 4);
    f.misc = take(16);
    f.bar = take(16);
    f.idx = take(S * 2);
    f.tmp = take(S * 2);
    f.draws = take(S * 2);
    f.cwb = take(k * kWarps * 2);
    f.total = off;
    return f;
}

uint32_t finish_smem_bytes(uint32_t S_fuse, uint32_t eb, uint32_t k) { return finish_layout(S_fuse, eb, k).total; }

struct FinishCtx {
    unsigned char* data;
    uint16_t* idx;
    uint16_t* tmp;
    uint16_t* draws;
    uint16_t* cwb;
    uint32_t* bst;
    uint32_t* wsum;
    uint32_t* front[2];
    uint32_t* misc;
    uint64_t* bar;
    uint32_t phase;
};

// Sequential Fisher-Yates (Fig. 1) on idx[a .. a+m) whose element 0 sits at
// problem-relative position P0: for i = m-1 .. 1, swap(i, fy(P0+i, i+1)).
__device__ void fy_seq(uint16_t* idx, uint32_t a, uint32_t m, uint64_t P0, PhiloxKey key) {
    uint64_t gcur = ~0ull;
    uint4 w = make_uint4(0, 0, 0, 0);
    for (uint32_t i = m; i-- > 1;) {
        const uint64_t P = P0 + i;
        const uint64_t g = P >> 2;
        if (g != gcur) {
            w = fy_group_words(key, g);
            gcur = g;
        }
        const uint32_t j = fy_from_word(word32(w, (uint32_t)(P & 3u)), key, P, i + 1);
        const uint16_t t = idx[a + i];
        idx[a + i] = idx[a + j];
        idx[a + j] = t;
    }
}

// Stable counting scatter of idx[a .. a+m) by the level-`level` draws of
// positions P0 .. P0+m-1 (D6), through tmp.  Leaves bucket starts
// (relative to a) in bst[0..k] on return.
__device__ void smem_scatter(const FinishCtx& c, uint32_t a, uint32_t m, uint64_t P0, uint32_t level, PhiloxKey key,
                             const BucketParams& bp) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t k = bp.k;
    uint16_t* d = c.draws + a;
    draws_to_smem(d, P0, m, key, level, bp);
    for (uint32_t i = tid; i < k * kWarps; i += kThreads) c.cwb[i] = 0;
    __syncthreads();
    const uint32_t qq = ((m + kWarps - 1) / kWarps + 31u) & ~31u;
    const uint32_t wb = warp * qq, we = min(m, wb + qq);
    // count pass
    for (uint32_t e0 = wb; e0 < we; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool valid = e < we;
        const uint32_t b = valid ? d[e] : 0xFFFFu;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
        if (valid && lane == (uint32_t)(__ffs(peers) - 1)) c.cwb[b * kWarps + warp] += (uint16_t)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    block_exclusive_scan(c.cwb, k * kWarps, c.wsum);
    for (uint32_t b = tid; b < k; b += kThreads) c.bst[b] = c.cwb[b * kWarps];
    if (tid == 0) c.bst[k] = m;
    __syncthreads();
    // placement pass
    for (uint32_t e0 = wb; e0 < we; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool valid = e < we;
        const uint32_t b = valid ? d[e] : 0xFFFFu;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
        const uint32_t old = valid ? c.cwb[b * kWarps + warp] : 0u;
        __syncwarp();
        if (valid) {
            if (lane == (uint32_t)(__ffs(peers) - 1)) c.cwb[b * kWarps + warp] = (uint16_t)(old + __popc(peers));
            c.tmp[old + __popc(peers & lanemask_lt())] = c.idx[a + e];
        }
        __syncwarp();
    }
    __syncthreads();
    for (uint32_t i = tid; i < m; i += kThreads) c.idx[a + i] = c.tmp[i];
    __syncthreads();
}

// Finish one segment [start, start+len) of buffer `src` at level `level`
// (problem origin `origin`, key K), writing the result to buf0.
template <int EB>
__device__ void finish_item(const RunParams& rp, FinishCtx& c, const unsigned char* src, uint64_t start, uint32_t len,
                            uint32_t level, uint64_t origin, uint64_t K) {
    using E = typename ElemT<EB>::type;
    const uint32_t tid = threadIdx.x;
    const bool in_place = (src == rp.buf0);
    const bool is_leaf = len <= rp.L;
    const bool scatters = !is_leaf && level < rp.max_levels;
    const bool permutes = scatters || (is_leaf && rp.run_leaves && len >= 2);
    if (in_place && !permutes) return;  // nothing moves
    const PhiloxKey key = make_key(K);
    const uint64_t P0 = start - origin;
    // ---- load: aligned body by one bulk copy, head/tail by 4-byte words
    const uint64_t x0 = start * EB, x1 = (start + len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    if (body && tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(c.bar, (uint32_t)(B - A));
        bulk_g2s(c.data + (A - fl), src + A, (uint32_t)(B - A), c.bar);
    }
    {
        const uint64_t hEnd = body ? A : x1;
        const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
        const uint64_t tBeg = body ? B : x1;
        const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
        if (tid < nh)
            *reinterpret_cast<uint32_t*>(c.data + (x0 - fl) + 4 * tid) =
                *reinterpret_cast<const uint32_t*>(src + x0 + 4 * tid);
        else if (tid >= 32 && tid - 32 < nt)
            *reinterpret_cast<uint32_t*>(c.data + (tBeg - fl) + 4 * (tid - 32)) =
                *reinterpret_cast<const uint32_t*>(src + tBeg + 4 * (tid - 32));
    }
    // ---- index permutation (independent of the data)
    for (uint32_t i = tid; i < len; i += kThreads) c.idx[i] = (uint16_t)i;
    __syncthreads();
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->finished, (unsigned long long)len);
    if (is_leaf) {
        if (permutes && tid == 0) {
            fy_seq(c.idx, 0, len, P0, key);
            atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)len);
        }
    } else if (scatters) {
        uint32_t nf = 1, cur = 0, lv = level;
        // frontier entries: a in the low 16 bits, m in the high 16 bits (S_fuse <= 65535)
        if (tid == 0) c.front[0][0] = (uint32_t)len << 16;
        __syncthreads();
        while (nf > 0) {
            if (tid == 0) c.misc[0] = 0;
            __syncthreads();
            for (uint32_t f = 0; f < nf; ++f) {
                const uint32_t ent = c.front[cur][f];
                const uint32_t a = ent & 0xFFFFu, m = ent >> 16;
                smem_scatter(c, a, m, P0 + a, lv, key, rp.bp);
                if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[lv], (unsigned long long)m);
                for (uint32_t b = tid; b < rp.k; b += kThreads) {
                    const uint32_t ca = a + c.bst[b], cm = c.bst[b + 1] - c.bst[b];
                    if (cm <= rp.L) {
                        if (rp.run_leaves && cm >= 2) {
                            fy_seq(c.idx, ca, cm, P0 + ca, key);
                            atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)cm);
                        }
                    } else if (lv + 1 < rp.max_levels) {
                        const uint32_t slot = atomicAdd(&c.misc[0], 1u);
                        c.front[cur ^ 1][slot] = ca | (cm << 16);
                    }
                }
                __syncthreads();
            }
            nf = c.misc[0];
            cur ^= 1;
            ++lv;
            __syncthreads();
        }
    }
    __syncthreads();
    // ---- wait for the data, gather into the final place
    if (body) {
        mbar_wait(c.bar, c.phase);
        c.phase ^= 1u;
    }
    __syncthreads();
    const unsigned char* din = c.data + (x0 - fl);
    E* out = reinterpret_cast<E*>(rp.buf0) + start;
    for (uint32_t j = tid; j < len; j += kThreads) out[j] = *reinterpret_cast<const E*>(din + (size_t)c.idx[j] * EB);
    __syncthreads();
}

template <int EB>
__device__ void copy_range(const RunParams& rp, const unsigned char* src, uint64_t start, uint64_t len) {
    using E = typename ElemT<EB>::type;
    const E* s = reinterpret_cast<const E*>(src) + start;
    E* d = reinterpret_cast<E*>(rp.buf0) + start;
    for (uint64_t i = threadIdx.x; i < len; i += kThreads) d[i] = s[i];
}

__device__ FinishCtx make_ctx(const RunParams& rp, unsigned char* sm) {
    const FinishLayout f = finish_layout(rp.S_fuse, rp.eb, rp.k);
    FinishCtx c;
    c.data = sm + f.data;
    c.idx = reinterpret_cast<uint16_t*>(sm + f.idx);
    c.tmp = reinterpret_cast<uint16_t*>(sm + f.tmp);
    c.draws = reinterpret_cast<uint16_t*>(sm + f.draws);
    c.cwb = reinterpret_cast<uint16_t*>(sm + f.cwb);
    c.bst = reinterpret_cast<uint32_t*>(sm + f.bst);
    c.wsum = reinterpret_cast<uint32_t*>(sm + f.wsum);
    c.front[0] = reinterpret_cast<uint32_t*>(sm + f.front0);
    c.front[1] = reinterpret_cast<uint32_t*>(sm + f.front1);
    c.misc = reinterpret_cast<uint32_t*>(sm + f.misc);
    c.bar = reinterpret_cast<uint64_t*>(sm + f.bar);
    c.phase = 0;
    if (threadIdx.x == 0) {
        mbar_init(c.bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    return c;
}

__device__ __forceinline__ void child_of(const SegDesc& sg, const uint64_t* __restrict__ prefix, uint32_t k, uint32_t b,
                                         uint64_t& start, uint64_t& len) {
    const uint64_t base0 = prefix[sg.cbase];
    const uint64_t s0 = prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
    const uint64_t s1 = (b + 1 < k) ? prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
    start = sg.start + s0;
    len = s1 - s0;
}

// Children of the level-l segments (they sit in the level's output buffer).
template <int EB>
__global__ void __launch_bounds__(kThreads, 1) k_finish_children(RunParams rp, LevelParams lp) {
    extern __shared__ __align__(16) unsigned char sm[];
    FinishCtx c = make_ctx(rp, sm);
    const uint32_t groups = (rp.k + kFinishBucketGroup - 1) / kFinishBucketGroup;
    const uint64_t units = (uint64_t)lp.ctr->nseg * groups;
    const uint32_t next = lp.level + 1;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const uint32_t s = (uint32_t)(u / groups);
        const uint32_t b0 = (uint32_t)(u % groups) * kFinishBucketGroup;
        const SegDesc sg = lp.segs[s];
        for (uint32_t b = b0; b < min(rp.k, b0 + kFinishBucketGroup); ++b) {
            uint64_t start, len;
            child_of(sg, lp.prefix, rp.k, b, start, len);
            if (len == 0) continue;
            if (len > rp.S_fuse) {
                if (next >= rp.max_levels && lp.dst != rp.buf0) {  // debug level limit: state -> ptr
                    copy_range<EB>(rp, lp.dst, start, len);
                    __syncthreads();
                }
                continue;
            }
            finish_item<EB>(rp, c, lp.dst, start, (uint32_t)len, next, sg.origin, sg.key);
        }
    }
}

// Segments given by offsets (segmented mode at level 0, or the single
// problem when n <= S_fuse).  They sit in ptr.
template <int EB>
__global__ void __launch_bounds__(kThreads, 1) k_finish_segments(RunParams rp, const uint64_t* __restrict__ off,
                                                                  uint64_t nsegs) {
    extern __shared__ __align__(16) unsigned char sm[];
    FinishCtx c = make_ctx(rp, sm);
    const uint64_t units = (nsegs + kSegGroup - 1) / kSegGroup;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        for (uint64_t s = u * kSegGroup; s < min(nsegs, (u + 1) * kSegGroup); ++s) {
            const uint64_t a = off[s], b = off[s + 1];
            if (b <= a || b - a > rp.S_fuse) continue;
            finish_item<EB>(rp, c, rp.buf0, a, (uint32_t)(b - a), 0u, a, rp.seed + s * 0x9E3779B97F4A7C15ull);
        }
    }
}

cudaError_t launch_finish_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k);
    switch (rp.eb) {
    case 4: k_finish_children<4><<<grid, kThreads, smem, s>>>(rp, lp); break;
    case 8: k_finish_children<8><<<grid, kThreads, smem, s>>>(rp, lp); break;
    default: k_finish_children<16><<<grid, kThreads, smem, s>>>(rp, lp); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_finish_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                   cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k);
    switch (rp.eb) {
    case 4: k_finish_segments<4><<<grid, kThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    case 8: k_finish_segments<8><<<grid, kThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    default: k_finish_segments<16><<<grid, kThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    }
    return cudaGetLastError();
}

cudaError_t configure_finish(uint32_t smem) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_finish_children<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_children<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_children<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_segments<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_segments<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    return cudaFuncSetAttribute(k_finish_segments<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

cudaError_t occupancy_finish(uint32_t eb, uint32_t smem, int* blocks) {
    switch (eb) {
    case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<4>, kThreads, smem);
    case 8: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<8>, kThreads, smem);
    default: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<16>, kThreads, smem);
    }
}

}  // namespace shuf
