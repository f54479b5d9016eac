// HBM-resident stable scatter of one level:
// for every segment s of the level, OUT[o_b++] = IN[i] for ascending i with
// b = bucket(l, i) (D6; P:140-142 with pi stable).
//
// A CTA owns chunks (contiguous runs of C elements of one segment; k_scan
// gave each (segment, bucket, chunk) its destination) and walks each chunk
// tile by tile in order, keeping per bucket the running destination of the
// chunk's next element.  Per tile of T elements (double-buffered: the next
// tile's bulk async copy, TMA engine, is in flight while this one is
// processed):
//   1. draws + counts: warp w owns a contiguous run of the tile's Philox
//      groups (D4: 16 draws per call for power-of-two k <= 256), writes the
//      draws to shared memory and counts its elements per bucket in its own
//      table (unordered shared reductions);
//   2. scan: bucket starts of the tile and per-warp slot bases;
//   3. place: every thread reads its elements into registers, then writes
//      each to its slot in the same buffer -- warp w walks its elements in
//      rounds of 32 in position order and one ordered shared atomic on its
//      own table returns the slot (stable; the documented __match_any_sync
//      path when the probe in shuf_api.cu did not verify the order);
//   4. copy-out: slot s of the tile goes to dst[delta[b] + s] (b = bucket of
//      the slot, delta[b] = running[b] - tile start of run b): consecutive
//      lanes write consecutive slots, i.e. whole runs, coalesced.
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

constexpr uint32_t kSW = 8;  // warps per CTA: 256 threads, 2 CTAs per SM (32 KiB tiles)

template <int EB>
struct SCfg {
    static constexpr uint32_t T = kScatterTileBytes / EB;  // elements per tile (32 KiB)
};

// Draw storage of a tile: one 16-byte slot per Philox group (+1 for the
// misaligned head), u8 draws for power-of-two k <= 256, u16 otherwise.
template <int EB>
__host__ __device__ inline uint32_t scatter_draw_bytes(bool narrow) {
    return (SCfg<EB>::T / (narrow ? 16 : 8) + 2) * 16;
}

struct SLayout {
    uint32_t buf0, buf1, draws, slotb, tab, bst, run, delta, wsum, bar, total;
};

template <int EB>
__host__ __device__ inline SLayout s_layout(uint32_t k) {
    SLayout L;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    L.buf0 = take(SCfg<EB>::T * EB + 16);
    L.buf1 = take(SCfg<EB>::T * EB + 16);
    const bool narrow = (k & (k - 1)) == 0 && k <= 256;
    L.draws = take(scatter_draw_bytes<EB>(narrow));
    L.slotb = take((narrow ? 1u : 2u) * SCfg<EB>::T);  // bucket of every slot (u8 / u16)
    L.tab = take(kSW * (narrow ? k : (k + 1) / 2) * 4);  // u32 counters (narrow k) or packed u16 pairs
    L.bst = take((k + 1) * 4);
    L.run = take(k * 8);
    L.delta = take(k * 8);  // destination minus slot: u32 relative to the segment start (mod 2^32),
                            // u64 absolute for segments longer than 2^32 elements
    L.wsum = take((kSW + 1) * 4);
    L.bar = take(16);
    L.total = off;
    return L;
}

uint32_t scatter_smem_bytes(uint32_t eb, uint32_t k) {
    switch (eb) {
    case 4: return s_layout<4>(k).total;
    case 8: return s_layout<8>(k).total;
    default: return s_layout<16>(k).total;
    }
}

struct STile {
    uint32_t chunk;   // chunk index (>= nchunk: none)
    uint32_t seg;     // segment index
    uint64_t q0, q1;  // element range of the chunk's remaining part
};

__device__ __forceinline__ STile s_first_tile(const LevelParams& lp, const RunParams& rp, uint32_t j,
                                              uint32_t nchunk) {
    STile t;
    t.chunk = j;
    t.seg = 0;
    t.q0 = t.q1 = 0;
    if (j >= nchunk) return t;
    const ChunkDesc ch = lp.chunks[j];
    const SegDesc& sg = lp.segs[ch.seg];
    t.seg = ch.seg;
    t.q0 = sg.start + (uint64_t)ch.c * rp.chunk;
    t.q1 = min(sg.start + sg.len, t.q0 + rp.chunk);
    return t;
}

// Tile [q0, q0+cnt) -> buf: aligned body by one bulk copy (mbarrier bar),
// the unaligned head/tail words by threads 32..95.  Element e sits at byte
// ((q0*EB) & 15) + e*EB of buf.
template <int EB>
__device__ __forceinline__ void s_issue_load(uint64_t q0, uint32_t cnt, const unsigned char* src, unsigned char* buf,
                                             uint64_t* bar) {
    const uint32_t tid = threadIdx.x;
    const uint64_t x0 = q0 * EB, x1 = (q0 + cnt) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    if (tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, body ? (uint32_t)(B - A) : 0u);
        if (body) bulk_g2s(buf + (A - fl), src + A, (uint32_t)(B - A), bar);
    }
    const uint64_t hEnd = body ? A : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
    const uint64_t tBeg = body ? B : x1;
    const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
    if (tid >= 32 && tid - 32 < nh)
        *reinterpret_cast<uint32_t*>(buf + (x0 - fl) + 4 * (tid - 32)) =
            *reinterpret_cast<const uint32_t*>(src + x0 + 4 * (tid - 32));
    else if (tid >= 64 && tid - 64 < nt)
        *reinterpret_cast<uint32_t*>(buf + (tBeg - fl) + 4 * (tid - 64)) =
            *reinterpret_cast<const uint32_t*>(src + tBeg + 4 * (tid - 64));
}

template <int EB, bool ORD, bool NARROW>
__global__ void __launch_bounds__(kSW * 32, 2) k_scatter(RunParams rp, LevelParams lp) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    constexpr uint32_t T = SCfg<EB>::T;
    constexpr uint32_t sh = NARROW ? 4u : 3u, dpg = 1u << sh;
    constexpr uint32_t R = (T / dpg / kSW + 1) * dpg / 32 + 1;  // rounds per warp (upper bound)
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t k = rp.k, kw = NARROW ? k : (k + 1) >> 1;  // table words per warp
    const SLayout Ly = s_layout<EB>(k);
    unsigned char* draws = sm + Ly.draws;
    uint32_t* tab = reinterpret_cast<uint32_t*>(sm + Ly.tab);
    uint32_t* bst = reinterpret_cast<uint32_t*>(sm + Ly.bst);
    uint64_t* running = reinterpret_cast<uint64_t*>(sm + Ly.run);
    uint32_t* delta = reinterpret_cast<uint32_t*>(sm + Ly.delta);
    uint64_t* delta64 = reinterpret_cast<uint64_t*>(sm + Ly.delta);
    D* slotb = reinterpret_cast<D*>(sm + Ly.slotb);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + Ly.wsum);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Ly.bar);
    const BucketParams bp = rp.bp;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t nchunk = lp.ctr->nchunk;
    if (blockIdx.x >= nchunk) return;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned char* __restrict__ src = lp.src;
    unsigned char* __restrict__ dstb = lp.dst;
    uint32_t ph0 = 0, ph1 = 0;
    uint32_t* Tw = tab + warp * kw;

    STile cur = s_first_tile(lp, rp, blockIdx.x, nchunk);
    uint32_t cnt = (uint32_t)min((uint64_t)T, cur.q1 - cur.q0);
    s_issue_load<EB>(cur.q0, cnt, src, sm + Ly.buf0, &bar[0]);
    unsigned long long scattered = cur.q1 - cur.q0;
    bool new_chunk = true;
    const bool dbgc = (rp.dbg & 1u) && blockIdx.x == 0 && tid == 0 && lp.level == 0;
    for (uint32_t it = 0; cur.chunk < nchunk; ++it) {
        const bool dbg = dbgc && it < 40;
        if (dbg) rp.hdr->sclk[it * 6 + 0] = clock64();
        // ---- next tile of this CTA's sequence -> the other buffer (free since
        //      the previous iteration's copy-out)
        STile nxt = cur;
        nxt.q0 = cur.q0 + cnt;
        const bool next_chunk = nxt.q0 >= cur.q1;
        if (next_chunk) {
            nxt = s_first_tile(lp, rp, cur.chunk + gridDim.x, nchunk);
            if (nxt.chunk < nchunk) scattered += nxt.q1 - nxt.q0;
        }
        const uint32_t ncnt = (uint32_t)min((uint64_t)T, nxt.q1 - nxt.q0);
        unsigned char* buf = sm + ((it & 1u) ? Ly.buf1 : Ly.buf0);
        if (nxt.chunk < nchunk)
            s_issue_load<EB>(nxt.q0, ncnt, src, sm + ((it & 1u) ? Ly.buf0 : Ly.buf1), &bar[(it & 1u) ^ 1u]);
        const SegDesc sg = lp.segs[cur.seg];
        if (new_chunk) {
            const ChunkDesc ch = lp.chunks[cur.chunk];
            const uint64_t base0 = lp.prefix[sg.cbase];
            for (uint32_t b = tid; b < k; b += kSW * 32)
                running[b] = sg.start + lp.prefix[sg.cbase + (uint64_t)b * sg.nchunks + ch.c] - base0;
        }
        // ---- 1. draws + per-warp counts
        const uint64_t P0 = cur.q0 - sg.origin;
        const uint64_t g0 = P0 >> sh;
        const uint32_t doff = (uint32_t)(P0 & (dpg - 1));
        const uint32_t ng = (uint32_t)(((P0 + cnt - 1) >> sh) - g0 + 1);
        const uint32_t qg = (ng + kSW - 1) / kSW;
        {
            const PhiloxKey key = make_key(sg.key);
            for (uint32_t i = lane; i < kw; i += 32) Tw[i] = 0;
            __syncwarp();
            const uint32_t t1 = min(ng, (warp + 1) * qg);
            for (uint32_t t = warp * qg + lane; t < t1; t += 32) {
                const uint64_t g = g0 + t;
                const uint4 w4 = bucket_group_words(key, lp.level, g);
                uint4 packed;
                if (NARROW) {
                    const uint32_t msk = (0xFFu >> bp.shift) * 0x01010101u;
                    packed = make_uint4((w4.x >> bp.shift) & msk, (w4.y >> bp.shift) & msk, (w4.z >> bp.shift) & msk,
                                        (w4.w >> bp.shift) & msk);
                } else {
                    const uint64_t pb = g << sh;
                    uint32_t bb[8];
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j) {
                        const bool in = pb + j >= P0 && pb + j < P0 + cnt;
                        bb[j] = in ? bucket_from_group(w4, j, key, lp.level, pb + j, bp) : 0u;
                    }
                    packed = make_uint4(bb[0] | (bb[1] << 16), bb[2] | (bb[3] << 16), bb[4] | (bb[5] << 16),
                                        bb[6] | (bb[7] << 16));
                }
                *reinterpret_cast<uint4*>(draws + (size_t)t * 16) = packed;
                const int32_t e0 = (int32_t)(t * dpg) - (int32_t)doff;
                const uint32_t pw4[4] = {packed.x, packed.y, packed.z, packed.w};
                if (e0 >= 0 && e0 + (int32_t)dpg <= (int32_t)cnt) {  // whole group inside the tile
#pragma unroll
                    for (uint32_t j = 0; j < dpg; ++j) {
                        if (NARROW) {
                            atomicAdd(&Tw[__byte_perm(pw4[j >> 2], 0u, 0x4440u | (j & 3u))], 1u);
                        } else {
                            const uint32_t b = (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                            atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
                        }
                    }
                } else {
#pragma unroll
                    for (uint32_t j = 0; j < dpg; ++j) {
                        const int32_t e = e0 + (int32_t)j;
                        if (e >= 0 && e < (int32_t)cnt) {
                            if (NARROW) {
                                atomicAdd(&Tw[(pw4[j >> 2] >> ((j & 3u) * 8u)) & 0xFFu], 1u);
                            } else {
                                const uint32_t b = (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                                atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
                            }
                        }
                    }
                }
            }
        }
        if (dbg) rp.hdr->sclk[it * 6 + 1] = clock64();
        // ---- wait for this tile's data, publish the counts
        if (it & 1u) {
            mbar_wait(&bar[1], ph1);
            ph1 ^= 1u;
        } else {
            mbar_wait(&bar[0], ph0);
            ph0 ^= 1u;
        }
        __syncthreads();
        if (dbg) rp.hdr->sclk[it * 6 + 2] = clock64();
        // ---- 2. scan: (bucket, warp)-major exclusive prefix of the counts ->
        //      per-warp slot bases; bst = bucket starts of the tile
        if (NARROW) scan_counters32<kSW * 32>(tab, kSW, k, bst, wsum);
        else scan_counters<kSW * 32>(tab, kSW, k, bst, wsum);
        __syncthreads();
        if (dbg) rp.hdr->sclk[it * 6 + 3] = clock64();
        // ---- 3. place: values to registers, then each to its slot in buf
        {
            E* el = reinterpret_cast<E*>(buf + ((cur.q0 * EB) & 15u));
            const D* dp = reinterpret_cast<const D*>(draws) + doff;
            // this warp's elements [e_lo, e_hi), walked in rounds of 32 in position order
            const int32_t eb0 = (int32_t)(warp * qg * dpg) - (int32_t)doff;
            const uint32_t e_lo = eb0 > 0 ? (uint32_t)eb0 : 0u;
            const int32_t ehi = min((int32_t)((warp + 1) * qg * dpg) - (int32_t)doff, (int32_t)cnt);
            const uint32_t len = ehi > (int32_t)e_lo ? (uint32_t)ehi - e_lo : 0u;
            const E* ew = el + e_lo;
            const D* dw = dp + e_lo;
            E v[R];
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint32_t i = r * 32 + lane;
                v[r] = ew[i < len ? i : 0];
            }
            __syncthreads();  // every element has been read out of buf
#pragma unroll
            for (uint32_t r = 0; r < R; ++r) {
                const uint32_t i = r * 32 + lane;
                if (r * 32 >= len) break;  // warp-uniform
                const bool valid = i < len;
                const uint32_t b = valid ? (uint32_t)dw[i] : 0u;
                uint32_t slot;
                if (NARROW) {
                    if (ORD) {
                        slot = atomicAdd(&Tw[b], valid ? 1u : 0u);
                    } else {
                        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, valid ? b : 0xFFFFFFFFu);
                        const uint32_t old = valid ? Tw[b] : 0u;
                        __syncwarp();
                        if (valid && (peers & lanemask_lt()) == 0) Tw[b] = old + (uint32_t)__popc(peers);
                        __syncwarp();
                        slot = old + __popc(peers & lanemask_lt());
                    }
                } else if (ORD) {
                    const uint32_t shb = (b & 1u) << 4;
                    slot = (atomicAdd(&Tw[b >> 1], valid ? (1u << shb) : 0u) >> shb) & 0xFFFFu;
                } else {
                    slot = warp_rank(Tw, b, valid, false);
                }
                if (ORD && r == 0 && warp == 0) check_rank_order(b, valid, slot, &rp.hdr->error);
                if (valid) {
                    el[slot] = v[r];
                    slotb[slot] = (D)b;
                }
            }
        }
        // destinations of the tile's runs: dst index of slot s = delta[b] + s
        // a segment of <= 2^32 elements: every destination minus the segment
        // start fits 32 bits, so delta is kept modulo 2^32 (half the lookup
        // bytes in the copy-out); longer segments keep 64-bit deltas
        const bool wide = (sg.len >> 32) != 0 || (rp.dbg & 64u);  // SHUF_DBG=64: test hook forcing the 64-bit path
        for (uint32_t b = tid; b < k; b += kSW * 32) {
            if (wide) delta64[b] = running[b] - bst[b];
            else delta[b] = (uint32_t)(running[b] - sg.start) - bst[b];
            running[b] += bst[b + 1] - bst[b];
        }
        __syncthreads();
        if (dbg) rp.hdr->sclk[it * 6 + 4] = clock64();
        // ---- 4. copy-out: slot s -> dst[delta[bucket(s)] + s]; consecutive
        //      lanes take consecutive slots, so each warp store covers the
        //      1-3 runs that meet its 32 slots (coalesced)
        {
            const E* el = reinterpret_cast<const E*>(buf + ((cur.q0 * EB) & 15u));
            if (!wide) {
                E* dst = reinterpret_cast<E*>(dstb) + sg.start;
#pragma unroll 4
                for (uint32_t x = tid; x < cnt; x += kSW * 32) dst[(uint32_t)(delta[slotb[x]] + x)] = el[x];
            } else {
                E* dst = reinterpret_cast<E*>(dstb);
                for (uint32_t x = tid; x < cnt; x += kSW * 32) dst[delta64[slotb[x]] + x] = el[x];
            }
        }
        __syncthreads();
        if (dbg) rp.hdr->sclk[it * 6 + 5] = clock64();
        new_chunk = next_chunk;
        cur = nxt;
        cnt = ncnt;
    }
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->scattered_hbm[lp.level], scattered);
}

// Kernel selection: element size x ranking mode x lane width.
template <int EB>
static void* scatter_fn(bool ord, bool narrow) {
    if (ord) return narrow ? (void*)k_scatter<EB, true, true> : (void*)k_scatter<EB, true, false>;
    return narrow ? (void*)k_scatter<EB, false, true> : (void*)k_scatter<EB, false, false>;
}

static void* scatter_kernel(uint32_t eb, bool ord, bool narrow) {
    switch (eb) {
    case 4: return scatter_fn<4>(ord, narrow);
    case 8: return scatter_fn<8>(ord, narrow);
    default: return scatter_fn<16>(ord, narrow);
    }
}

cudaError_t launch_scatter(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = scatter_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(scatter_kernel(rp.eb, rp.rank_ordered != 0, rp.bp.narrow != 0), dim3(grid),
                            dim3(kSW * 32), args, smem, s);
}

cudaError_t configure_scatter(uint32_t) {  // the attribute is the limit: plans with other sizes share the kernels
    cudaError_t e;
    for (uint32_t eb : {4u, 8u, 16u})
        for (int o = 0; o < 2; ++o)
            for (int nr = 0; nr < 2; ++nr)
                if ((e = cudaFuncSetAttribute(scatter_kernel(eb, o, nr), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kSmemLimit)))
                    return e;
    return cudaSuccess;
}

cudaError_t occupancy_scatter(uint32_t eb, uint32_t k, int* blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, scatter_kernel(eb, true, true), kSW * 32,
                                                         scatter_smem_bytes(eb, k));
}

}  // namespace shuf
