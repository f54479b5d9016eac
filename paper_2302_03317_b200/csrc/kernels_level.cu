// HBM-resident ("global") scatter level: init, histogram, decoupled-lookback
// scan and segment planner (the stable scatter itself: kernels_scatter.cu).
//
// One level l over the active segments computes, for every segment s of
// length m at [a, a+m) (D6, P:140-142 with pi stable):
//   c_b = #{i : bucket(l, i) = b},  o_b = a + sum_{b'<b} c_b',
//   OUT[o_b++] = IN[i] for ascending i.
// Segments are cut into chunks of C elements; a CTA owns a chunk and walks
// it tile by tile in order, so the destination of (segment, bucket, chunk)
// is the exclusive prefix of the counts flattened in (segment, bucket,
// chunk) order (k_scan), and within a chunk a per-bucket running offset plus
// the stable in-tile rank gives every element's destination.
#include <cuda_runtime.h>

#include <cstdlib>
#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

__device__ __forceinline__ void latch_error(Header* h, uint32_t code) { atomicCAS(&h->error, 0u, code); }

__device__ __forceinline__ uint64_t gtid() { return (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ uint64_t gstride() { return (uint64_t)gridDim.x * blockDim.x; }

// ------------------------------------------------------------------ init --
__global__ void k_init_single(RunParams rp, LevelParams lp0) {
    const uint64_t n = rp.n;
    if (gtid() == 0) {
        rp.hdr->root_off[0] = 0;
        rp.hdr->root_off[1] = n;
    }
    if (!(n > rp.S_fuse && rp.max_levels > 0)) return;
    const uint64_t nch = (n + rp.chunk - 1) / rp.chunk;
    if (gtid() == 0) {
        SegDesc sd;
        sd.start = 0;
        sd.len = n;
        sd.origin = 0;
        sd.key = rp.seed;  // K(seed, 0) = seed (D2)
        sd.cbase = 0;
        sd.nchunks = (uint32_t)nch;
        sd.pad = 0;
        lp0.segs[0] = sd;
        lp0.ctr->nseg = 1;
        lp0.ctr->nchunk = (uint32_t)nch;
    }
    for (uint64_t j = gtid(); j < nch; j += gstride()) lp0.chunks[j] = ChunkDesc{0u, (uint32_t)j};
}

__global__ void k_init_segmented(RunParams rp, LevelParams lp0, const uint64_t* __restrict__ off, uint64_t nsegs) {
    if (gtid() == 0 && (off[0] != 0 || off[nsegs] != rp.n)) latch_error(rp.hdr, 1u /*SHUF_ERR_INVALID_ARG*/);
    for (uint64_t s = gtid(); s < nsegs; s += gstride()) {
        const uint64_t a = off[s], b = off[s + 1];
        if (b < a) {
            latch_error(rp.hdr, 1u);
            continue;
        }
        const uint64_t len = b - a;
        if (!(len > rp.S_fuse && rp.max_levels > 0)) continue;
        const uint64_t nch = (len + rp.chunk - 1) / rp.chunk;
        const uint32_t si = atomicAdd(&lp0.ctr->nseg, 1u);
        const uint32_t cb = atomicAdd(&lp0.ctr->nchunk, (uint32_t)nch);
        if (si >= lp0.max_segs || cb + nch > lp0.max_chunks) {
            latch_error(rp.hdr, 4u /*SHUF_ERR_SCRATCH*/);
            continue;
        }
        SegDesc sd;
        sd.start = a;
        sd.len = len;
        // user segment s: K(seed, s), positions segment-relative (D7); a sharded
        // rank's level-0 children: K(seed, 0), global positions (NEXT-3)
        sd.origin = rp.shard ? 0ull - rp.seg_base : a;
        sd.key = rp.shard ? rp.seed : rp.seed + s * 0x9E3779B97F4A7C15ull;
        sd.cbase = (uint64_t)cb * rp.k;
        sd.nchunks = (uint32_t)nch;
        sd.pad = 0;
        lp0.segs[si] = sd;
        for (uint64_t c = 0; c < nch; ++c) lp0.chunks[cb + c] = ChunkDesc{si, (uint32_t)c};
    }
}

// Sharded level 0 (NEXT-3): the rank's input slice [0, m) holds the global
// level-0 positions [pos0, pos0 + m) of the one problem (K(seed, 0)); it is
// scattered as one segment whatever its length (the whole problem exceeds L).
__global__ void k_init_shard(RunParams rp, LevelParams lp0, uint64_t m, uint64_t pos0) {
    const uint64_t nch = (m + rp.chunk - 1) / rp.chunk;
    if (gtid() == 0) {
        SegDesc sd;
        sd.start = 0;
        sd.len = m;
        sd.origin = 0ull - pos0;
        sd.key = rp.seed;  // K(seed, 0) (D2)
        sd.cbase = 0;
        sd.nchunks = (uint32_t)nch;
        sd.pad = 0;
        lp0.segs[0] = sd;
        lp0.ctr->nseg = 1;
        lp0.ctr->nchunk = (uint32_t)nch;
        if (nch > lp0.max_chunks) latch_error(rp.hdr, 4u /*SHUF_ERR_SCRATCH*/);
    }
    for (uint64_t j = gtid(); j < nch && j < lp0.max_chunks; j += gstride()) lp0.chunks[j] = ChunkDesc{0u, (uint32_t)j};
}

// counts[b] = |child b| of the sharded level-0 segment (after k_scan).
__global__ void k_shard_counts(RunParams rp, LevelParams lp, uint64_t* __restrict__ counts) {
    const SegDesc sg = lp.segs[0];
    const uint64_t base0 = lp.prefix[sg.cbase];
    for (uint64_t b = gtid(); b < rp.k; b += gstride()) {
        const uint64_t s0 = lp.prefix[sg.cbase + b * sg.nchunks] - base0;
        const uint64_t s1 = (b + 1 < rp.k) ? lp.prefix[sg.cbase + (b + 1) * sg.nchunks] - base0 : sg.len;
        counts[b] = s1 - s0;
    }
}

// ------------------------------------------------------------- histogram --
// counts[cbase + b*nchunks + c] = #{p in chunk c : bucket(l, p) = b}.
// Regenerates the draws from Philox counters; reads no element data.
// (Replicating the counters per lane to avoid bank conflicts was measured
// slower: 1.18 vs 1.06 ms on HOT -- the kernel is ALU-bound on Philox.)
// LANES (k <= 256): every lane counts into its own column of the table,
// hist[b*32 + lane] -- the 32 atomics of one warp instruction hit 32 distinct
// banks (random buckets into one k-entry table conflict ~3.5-way); the
// columns are summed per bucket at the end of the chunk (rotated so a warp's
// 32 threads read 32 distinct banks).  SHUF_HIST_LANES=0 keeps one k-entry table.
static bool hist_lanes(uint32_t k) {
    static const int on = [] {
        const char* e = std::getenv("SHUF_HIST_LANES");
        return e ? std::atoi(e) : 1;
    }();
    return on != 0 && k <= 256;
}
uint32_t hist_smem_bytes(uint32_t k) { return hist_lanes(k) ? k * 32u * 4u : k * 4u; }

template <bool LANES>
__global__ void __launch_bounds__(kThreads) k_hist(RunParams rp, LevelParams lp) {
    extern __shared__ uint32_t hist[];
    const uint32_t nchunk = lp.ctr->nchunk;
    const uint64_t E = (uint64_t)nchunk * rp.k;
    const uint64_t ntiles = (E + kScanTile - 1) / kScanTile;
    for (uint64_t t = gtid(); t < ntiles; t += gstride()) lp.status[t] = 0;
    if (gtid() == 0) {
        lp.ctr->scan_ticket = 0;
        lp.ctr->nfuse = 0;
        lp.ctr->nstream = 0;
        // (the next level's segment counters are reset by k_scan: this kernel may
        // run while the previous level's kernels still read that slot)
    }
    const uint32_t k = rp.k;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t col = LANES ? lane : 0u, cs = LANES ? 5u : 0u;  // counter of bucket b: hist[(b << cs) | col]
    const BucketParams bp = rp.bp;
    const uint32_t sh = bp.narrow ? 4u : 3u, dpg = 1u << sh;
    for (uint32_t b = threadIdx.x; b < (k << cs); b += kThreads) hist[b] = 0;
    __syncthreads();
    for (uint32_t j = blockIdx.x; j < nchunk; j += gridDim.x) {
        const ChunkDesc ch = lp.chunks[j];
        const SegDesc sg = lp.segs[ch.seg];
        const uint64_t q0 = sg.start + (uint64_t)ch.c * rp.chunk;
        const uint64_t q1 = min(sg.start + sg.len, q0 + rp.chunk);
        const uint64_t P0 = q0 - sg.origin, P1 = q1 - sg.origin;
        const PhiloxKey key = make_key(sg.key);
        const uint64_t g0 = P0 >> sh, ng = ((P1 - 1) >> sh) - g0 + 1;
        for (uint64_t t = threadIdx.x; t < ng; t += kThreads) {
            const uint64_t g = g0 + t;
            const uint4 w = bucket_group_words(key, lp.level, g);
            const uint64_t pb = g << sh;
            if (pb >= P0 && pb + dpg <= P1) {
                if (bp.narrow) {
                    // the 16 draws are the bytes of the group's words shifted right by
                    // 8 - log2 k (masked per byte): one byte extract each
                    const uint32_t msk = (0xFFu >> bp.shift) * 0x01010101u;
                    const uint32_t pw[4] = {(w.x >> bp.shift) & msk, (w.y >> bp.shift) & msk,
                                            (w.z >> bp.shift) & msk, (w.w >> bp.shift) & msk};
#pragma unroll
                    for (uint32_t jj = 0; jj < 16; ++jj)
                        atomicAdd(&hist[(__byte_perm(pw[jj >> 2], 0u, 0x4440u | (jj & 3u)) << cs) | col], 1u);
                } else {
#pragma unroll
                    for (uint32_t jj = 0; jj < 8; ++jj)
                        atomicAdd(&hist[(bucket_from_group(w, jj, key, lp.level, pb + jj, bp) << cs) | col], 1u);
                }
            } else {
                for (uint32_t jj = 0; jj < dpg; ++jj) {
                    const uint64_t p = pb + jj;
                    if (p >= P0 && p < P1)
                        atomicAdd(&hist[(bucket_from_group(w, jj, key, lp.level, p, bp) << cs) | col], 1u);
                }
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < k; b += kThreads) {
            uint32_t c;
            if (LANES) {  // sum bucket b's 32 columns and clear them for the next chunk
                c = 0;
#pragma unroll 8
                for (uint32_t i = 0; i < 32; ++i) {
                    const uint32_t x = (b << 5) | ((i + b) & 31u);
                    c += hist[x];
                    hist[x] = 0;
                }
            } else {
                c = hist[b];
                hist[b] = 0;
            }
            lp.counts[sg.cbase + (uint64_t)b * sg.nchunks + ch.c] = c;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ scan --
// Single-pass exclusive scan (decoupled lookback, Merrill & Garland) of the
// u32 counts into u64 prefixes.  Tiles are claimed in order through a ticket
// so every predecessor of a claimed tile is owned by a running CTA.
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t warp_inclusive_sum64(uint64_t v) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= (uint32_t)o) v += t;
    }
    return v;
}

__global__ void __launch_bounds__(kThreads) k_scan(RunParams rp, LevelParams lp) {
    __shared__ uint64_t wsum[kWarps + 1];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_excl;
    constexpr uint32_t PER = kScanTile / kThreads;  // 8
    const uint64_t E = (uint64_t)lp.ctr->nchunk * rp.k;
    const uint64_t ntiles = (E + kScanTile - 1) / kScanTile;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (blockIdx.x == 0 && tid == 0) {  // the next level's list, filled by k_plan after this kernel
        lp.nctr->nseg = 0;
        lp.nctr->nchunk = 0;
    }
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(&lp.ctr->scan_ticket, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint64_t base = (uint64_t)tile * kScanTile + (uint64_t)tid * PER;
        uint32_t v[PER];
        uint64_t s = 0;
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            v[i] = (base + i < E) ? lp.counts[base + i] : 0u;
            s += v[i];
        }
        const uint64_t incl = warp_inclusive_sum64(s);
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint64_t x = lane < (uint32_t)kWarps ? wsum[lane] : 0ull;
            uint64_t xi = warp_inclusive_sum64(x);
            if (lane < (uint32_t)kWarps) wsum[lane] = xi - x;
            if (lane == kWarps - 1) wsum[kWarps] = xi;
        }
        __syncthreads();
        const uint64_t agg = wsum[kWarps];
        if (warp == 0) {
            uint64_t excl = 0;
            if (tile == 0) {
                if (lane == 0) st_release_u64(&lp.status[0], kFlagInc | agg);
            } else {
                if (lane == 0) st_release_u64(&lp.status[tile], kFlagAgg | agg);
                int64_t j = (int64_t)tile - 1;
                for (;;) {
                    const int64_t idx = j - (int64_t)lane;
                    uint64_t st = kFlagInc;  // before tile 0: inclusive zero
                    if (idx >= 0) {
                        do {
                            st = ld_acquire_u64(&lp.status[idx]);
                        } while ((st >> 62) == 0);
                    }
                    const uint32_t incmask = __ballot_sync(0xFFFFFFFFu, (st >> 62) == 2);
                    uint64_t val = st & kValMask;
                    if (incmask) {
                        const uint32_t p = __ffs(incmask) - 1;
                        if (lane > p) val = 0;
                    }
                    // reduce over the warp
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
                    excl += val;
                    if (incmask) break;
                    j -= 32;
                }
                if (lane == 0) st_release_u64(&lp.status[tile], kFlagInc | (excl + agg));
            }
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        uint64_t run = s_excl + wsum[warp] + incl - s;
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            if (base + i < E) lp.prefix[base + i] = run;
            run += v[i];
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------- planner --
// Child b of segment s: [start_s + P(s,b,0) - P(s,0,0), next).
// Children longer than S_fuse become segments of level l+1 (chunked);
// shorter ones are finished in shared memory by k_finish_children.
__device__ __forceinline__ void child_range(const SegDesc& sg, const uint64_t* __restrict__ prefix, uint32_t k,
                                            uint32_t b, uint64_t& start, uint64_t& len) {
    const uint64_t base0 = prefix[sg.cbase];
    const uint64_t s0 = prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
    const uint64_t s1 = (b + 1 < k) ? prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
    start = sg.start + s0;
    len = s1 - s0;
}

__global__ void k_plan(RunParams rp, LevelParams lp) {
    const uint64_t nchild = (uint64_t)lp.ctr->nseg * rp.k;
    const uint32_t next = lp.level + 1;
    for (uint64_t i = gtid(); i < nchild; i += gstride()) {
        const uint32_t s = (uint32_t)(i / rp.k), b = (uint32_t)(i % rp.k);
        const SegDesc sg = lp.segs[s];
        uint64_t start, len;
        child_range(sg, lp.prefix, rp.k, b, start, len);
        if (len <= rp.S_fuse) {  // finished by k_finish_children (or the leaf kernel)
            if (rp.max_fused && len > rp.L) {
                const bool permutes = next < rp.max_levels;  // not a leaf: another level to run
                if (permutes || lp.dst != rp.buf0) {
                    const uint32_t at = atomicAdd(&lp.ctr->nfuse, 1u);
                    if (at < rp.max_fused) rp.fused[at] = (uint32_t)i;
                    else latch_error(rp.hdr, 4u);
                }
            }
            continue;
        }
        if (rp.S_stream && len <= rp.S_stream) {  // k_finish_stream takes it (single buffer)
            atomicAdd(&lp.ctr->nstream, 1u);
            continue;
        }
        if (next >= rp.max_levels) continue;  // debug level limit: copied out by k_finish_children
        if (next >= rp.planned_levels) {
            latch_error(rp.hdr, 5u /*SHUF_ERR_DEPTH*/);
            continue;
        }
        const uint64_t nch = (len + rp.chunk - 1) / rp.chunk;
        const uint32_t si = atomicAdd(&lp.nctr->nseg, 1u);
        const uint32_t cb = atomicAdd(&lp.nctr->nchunk, (uint32_t)nch);
        if (si >= lp.max_segs || cb + nch > lp.max_chunks) {
            latch_error(rp.hdr, 4u);
            continue;
        }
        SegDesc nd;
        nd.start = start;
        nd.len = len;
        nd.origin = sg.origin;
        nd.key = sg.key;
        nd.cbase = (uint64_t)cb * rp.k;
        nd.nchunks = (uint32_t)nch;
        nd.pad = 0;
        lp.nsegs[si] = nd;
        for (uint64_t c = 0; c < nch; ++c) lp.nchunks[cb + c] = ChunkDesc{si, (uint32_t)c};
    }
}

// --------------------------------------------------------------- launchers --
cudaError_t launch_init(const RunParams& rp, const LevelParams& lp0, cudaStream_t s, int grid) {
    k_init_single<<<grid, 256, 0, s>>>(rp, lp0);
    return cudaGetLastError();
}

cudaError_t launch_init_segmented(const RunParams& rp, const LevelParams& lp0, const uint64_t* d_offsets,
                                  uint64_t num_segments, cudaStream_t s, int grid) {
    k_init_segmented<<<grid, 256, 0, s>>>(rp, lp0, d_offsets, num_segments);
    return cudaGetLastError();
}

cudaError_t launch_init_shard(const RunParams& rp, const LevelParams& lp0, uint64_t m, uint64_t pos0, cudaStream_t s,
                              int grid) {
    k_init_shard<<<grid, 256, 0, s>>>(rp, lp0, m, pos0);
    return cudaGetLastError();
}

cudaError_t launch_shard_counts(const RunParams& rp, const LevelParams& lp, uint64_t* counts, cudaStream_t s) {
    k_shard_counts<<<(rp.k + 255) / 256, 256, 0, s>>>(rp, lp, counts);
    return cudaGetLastError();
}

cudaError_t launch_hist(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    if (hist_lanes(rp.k)) k_hist<true><<<grid, kThreads, hist_smem_bytes(rp.k), s>>>(rp, lp);
    else k_hist<false><<<grid, kThreads, hist_smem_bytes(rp.k), s>>>(rp, lp);
    return cudaGetLastError();
}

cudaError_t launch_scan(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    k_scan<<<grid, kThreads, 0, s>>>(rp, lp);
    return cudaGetLastError();
}

cudaError_t launch_plan(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    k_plan<<<grid, 256, 0, s>>>(rp, lp);
    return cudaGetLastError();
}

cudaError_t occupancy_level(uint32_t eb, uint32_t k, int* hist, int* scan, int* scatter) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit))) return e;
    if ((e = cudaFuncSetAttribute(k_hist<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(hist, hist_lanes(k) ? (const void*)k_hist<true>
                                                                               : (const void*)k_hist<false>,
                                                           kThreads, hist_smem_bytes(k))))
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(scan, k_scan, kThreads, 0))) return e;
    return occupancy_scatter(eb, k, scatter);
}

}  // namespace shuf
