// HBM-resident stable scatter of one level:
// for every segment s of the level, OUT[o_b++] = IN[i] for ascending i with
// b = bucket(l, i) (D6; P:140-142 with pi stable).
//
// A CTA owns chunks (contiguous runs of C elements of one segment; k_scan
// gave each (segment, bucket, chunk) its destination) and walks each chunk
// tile by tile in order, keeping per bucket the running destination of the
// chunk's next element.  NW warps; warp w owns elements [w*R*32, (w+1)*R*32)
// of a tile of T elements (R rounds of 32 consecutive elements, lane order =
// position order).  Separate buffers for the raw tile (bulk async copy, TMA
// engine) and the bucket-sorted tile, so no element is held in registers
// across a barrier.  Per tile t, three CTA barriers:
//
//   B(t)   scan: (bucket, warp)-major exclusive prefix of the counts -> per-
//          warp slot bases, tile bucket starts, run destinations delta
//          and the run map of the sorted tile: the non-empty buckets in order
//          are runs 0, 1, ..; rdelta[r] = destination minus slot of run r;
//          winfo[w] = (bit i set iff slot 32w+i starts a run) | (number of
//          runs started before slot 32w) << 32
//   C(t)   rank + place: each round reads 32 draws and 32 elements of the raw
//          tile, takes every element's slot with one ordered shared atomic on
//          the warp's table (whose entries the scan set to the warp's first
//          slot per bucket) and stores the element at that slot
//   ---- barrier: raw tile consumed -> bulk load of tile t+1 into it
//   D(t)   copy-out: window w of 32 slots, slot x = 32w + lane ->
//          dst[rdelta[run(x)] + x], run(x) = winfo.base + popc(winfo.bits &
//          lanemask_le) - 1: one broadcast load per window instead of a
//          bucket byte stored per slot; consecutive lanes take consecutive
//          slots, i.e. whole bucket runs (coalesced)
//   A(t+1) draws + counts of the next tile (D4 Philox: positions only, no
//          data): lane-owned Philox groups -> draw buffer, per-warp counts
//   ---- barrier
//
// (plus the two barriers inside the scan).  Full tiles take an unrolled path
// with compile-time offsets (every element valid); a chunk's last partial
// tile takes the checked path.
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

// Tile geometry: 32 KiB tiles, 8 warps (R = T/256 rounds each), 2 CTAs per
// SM.  Measured on HOT: 16 warps per tile, 16 KiB tiles (8 or
// 16 warps), 24 KiB tiles x 3 CTAs/SM, 4 warps x 3 CTAs/SM and packed u16
// counters were all slower -- the per-warp tables (zeroed and scanned every
// tile, NW * k entries) cost more than the extra warps hide.
template <int EB, bool NARROW>
struct SCfg {
    static constexpr uint32_t T = scatter_tile_bytes(EB) / EB;  // elements per tile
    static constexpr uint32_t NW = 8;
    static constexpr uint32_t NT = NW * 32u;
    static constexpr uint32_t R = T / (NW * 32u);     // rounds per warp
    static constexpr uint32_t sh = NARROW ? 4u : 3u;  // log2 draws per Philox group
    static constexpr uint32_t dpg = 1u << sh;
    static constexpr bool P16 = !NARROW;              // counters as packed u16 pairs (k > 256), else u32
#ifndef SHUF_SCATTER_MINB
#define SHUF_SCATTER_MINB 2
#endif
    static constexpr int MINB = NARROW ? SHUF_SCATTER_MINB : 1;
};

struct SLayout {
    uint32_t raw, sorted, draws, tab, bst, rix, winfo, run, delta, wsum, bar, total;
};

template <int EB, bool NARROW>
__host__ __device__ inline SLayout s_layout(uint32_t k) {
    using C = SCfg<EB, NARROW>;
    SLayout L;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    L.raw = take(C::T * EB + 16);
    L.sorted = take(C::T * EB);
    L.draws = take((C::T / C::dpg + 2) * 16);
    L.tab = take(C::NW * (C::P16 ? (k + 1) / 2 : k) * 4);  // u32 counters or packed u16 pairs
    L.bst = take((k + 1) * 4);
    L.rix = take(k * 4);             // run index of every bucket
    L.winfo = take(C::T / 32 * 8);   // per 32-slot window: run-start bits | runs before << 32
    L.run = take(k * 8);
    L.delta = take(k * 8);  // per run: destination minus slot, u32 relative to the segment start
                            // (mod 2^32), u64 absolute for segments longer than 2^32 elements
    L.wsum = take((C::NW + 1) * 4);
    L.bar = take(16);
    L.total = off;
    return L;
}

static bool is_narrow(uint32_t k) { return (k & (k - 1)) == 0 && k <= 256; }

uint32_t scatter_smem_bytes(uint32_t eb, uint32_t k) {
    const bool nr = is_narrow(k);
    switch (eb) {
    case 4: return nr ? s_layout<4, true>(k).total : s_layout<4, false>(k).total;
    case 8: return nr ? s_layout<8, true>(k).total : s_layout<8, false>(k).total;
    default: return nr ? s_layout<16, true>(k).total : s_layout<16, false>(k).total;
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

// A: draws of the tile at problem positions [P0, P0+cnt) -> draw buffer
// (16-byte group t holds the draws of positions ((P0 >> sh) + t) << sh ..),
// and warp w's per-bucket counts of its element range (unordered shared
// reductions on the warp's own table).
template <int EB, bool NARROW>
__device__ __forceinline__ void s_draw_count(const BucketParams& bp, PhiloxKey key, uint32_t level, uint64_t P0,
                                             uint32_t cnt, unsigned char* draws, uint32_t* Tw, uint32_t kw,
                                             uint32_t warp, uint32_t lane) {
    using C = SCfg<EB, NARROW>;
    constexpr uint32_t sh = C::sh, dpg = C::dpg;
    for (uint32_t i = lane; i < kw; i += 32) Tw[i] = 0;
    __syncwarp();
    const uint32_t doff = (uint32_t)(P0 & (dpg - 1));
    const int32_t e_lo = (int32_t)(warp * C::R * 32u);
    const int32_t e_hi = min(e_lo + (int32_t)(C::R * 32u), (int32_t)cnt);
    if (e_hi <= e_lo) return;
    // element e lies in group (e + doff) >> sh
    const uint32_t t0 = (uint32_t)(e_lo + (int32_t)doff) >> sh;
    const uint32_t t1 = (uint32_t)(e_hi - 1 + (int32_t)doff) >> sh;  // inclusive
    const uint64_t g0 = P0 >> sh;
    for (uint32_t t = t0 + lane; t <= t1; t += 32) {
        const uint4 w4 = bucket_group_words(key, level, g0 + t);
        const int32_t es = (int32_t)(t * dpg) - (int32_t)doff;  // element index of the group's lane 0
        uint4 packed;
        if (NARROW) {
            const uint32_t msk = (0xFFu >> bp.shift) * 0x01010101u;
            packed = make_uint4((w4.x >> bp.shift) & msk, (w4.y >> bp.shift) & msk, (w4.z >> bp.shift) & msk,
                                (w4.w >> bp.shift) & msk);
        } else {
            const uint64_t pb = (g0 + t) << sh;
            uint32_t bb[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const int32_t e = es + (int32_t)j;
                bb[j] = (e >= 0 && e < (int32_t)cnt) ? bucket_from_group(w4, j, key, level, pb + j, bp) : 0u;
            }
            packed = make_uint4(bb[0] | (bb[1] << 16), bb[2] | (bb[3] << 16), bb[4] | (bb[5] << 16),
                                bb[6] | (bb[7] << 16));
        }
        // a group straddling two warp ranges is written by the warp it starts in
        if (es >= e_lo || warp == 0) *reinterpret_cast<uint4*>(draws + (size_t)t * 16) = packed;
        const uint32_t pw4[4] = {packed.x, packed.y, packed.z, packed.w};
        if (es >= e_lo && es + (int32_t)dpg <= e_hi) {  // whole group in this warp's range
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const uint32_t b = NARROW ? __byte_perm(pw4[j >> 2], 0u, 0x4440u | (j & 3u))
                                          : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                if (C::P16) atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
                else atomicAdd(&Tw[b], 1u);
            }
        } else {
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const int32_t e = es + (int32_t)j;
                if (e >= e_lo && e < e_hi) {
                    const uint32_t b = NARROW ? (pw4[j >> 2] >> ((j & 3u) * 8u)) & 0xFFu
                                              : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                    if (C::P16) atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
                    else atomicAdd(&Tw[b], 1u);
                }
            }
        }
    }
}

// C: rank + place of warp w's rounds.  FULL: cnt == T (no checks).
template <int EB, bool NARROW, bool ORD, bool FULL>
__device__ __forceinline__ void s_place(const unsigned char* raw, uint64_t q0, const unsigned char* draws,
                                        uint32_t doff, uint32_t cnt, unsigned char* sorted, uint32_t* Tw,
                                        uint32_t warp, uint32_t lane, uint32_t* err) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    using C = SCfg<EB, NARROW>;
    const uint32_t e0 = warp * C::R * 32u;
    const E* el = reinterpret_cast<const E*>(raw + ((q0 * EB) & 15u)) + e0 + lane;
    const D* dp = reinterpret_cast<const D*>(draws) + doff + e0 + lane;
    E* so = reinterpret_cast<E*>(sorted);
    const int32_t wrem = (int32_t)cnt - (int32_t)e0;  // elements of this warp's range in the tile
#pragma unroll
    for (uint32_t r = 0; r < C::R; ++r) {
        if (!FULL && (int32_t)(r * 32u) >= wrem) break;  // warp-uniform
        const bool valid = FULL || (int32_t)(r * 32u + lane) < wrem;
        const uint32_t b = valid ? (uint32_t)dp[r * 32u] : 0u;
        const E v = el[(FULL || valid) ? r * 32u : 0u];
        uint32_t slot;
        if (!C::P16) {
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
        if (ORD && r == 0 && warp == 0) check_rank_order(b, valid, slot, err);
        if (valid) so[slot] = v;
    }
}

template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(SCfg<EB, NARROW>::NT, SCfg<EB, NARROW>::MINB)
    k_scatter(RunParams rp, LevelParams lp) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    using C = SCfg<EB, NARROW>;
    constexpr uint32_t T = C::T, NT = C::NT;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t k = rp.k, kw = C::P16 ? (k + 1) >> 1 : k;  // table words per warp
    const SLayout Ly = s_layout<EB, NARROW>(k);
    unsigned char* raw = sm + Ly.raw;
    unsigned char* sorted = sm + Ly.sorted;
    unsigned char* draws = sm + Ly.draws;
    uint32_t* rix = reinterpret_cast<uint32_t*>(sm + Ly.rix);
    uint64_t* winfo = reinterpret_cast<uint64_t*>(sm + Ly.winfo);
    uint32_t* tab = reinterpret_cast<uint32_t*>(sm + Ly.tab);
    uint32_t* bst = reinterpret_cast<uint32_t*>(sm + Ly.bst);
    uint64_t* running = reinterpret_cast<uint64_t*>(sm + Ly.run);
    uint32_t* delta = reinterpret_cast<uint32_t*>(sm + Ly.delta);
    uint64_t* delta64 = reinterpret_cast<uint64_t*>(sm + Ly.delta);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + Ly.wsum);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Ly.bar);
    const BucketParams bp = rp.bp;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t nchunk = lp.ctr->nchunk;
    if (blockIdx.x >= nchunk) return;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned char* __restrict__ src = lp.src;
    unsigned char* __restrict__ dstb = lp.dst;
    uint32_t ph = 0;
    uint32_t* Tw = tab + warp * kw;

    // ---- prologue: tile 0's load, draws + counts
    STile cur = s_first_tile(lp, rp, blockIdx.x, nchunk);
    uint32_t cnt = (uint32_t)min((uint64_t)T, cur.q1 - cur.q0);
    unsigned long long scattered = cur.q1 - cur.q0;
    s_issue_load<EB>(cur.q0, cnt, src, raw, &bar[0]);
    SegDesc sg = lp.segs[cur.seg];
    s_draw_count<EB, NARROW>(bp, make_key(sg.key), lp.level, cur.q0 - sg.origin, cnt, draws, Tw, kw, warp, lane);
    bool new_chunk = true;
    __syncthreads();
    for (;;) {
        // ---- B: scan of the counts of tile `cur` -> slot bases, bucket starts, run destinations
        if (new_chunk) {
            const ChunkDesc ch = lp.chunks[cur.chunk];
            const uint64_t base0 = lp.prefix[sg.cbase];
            for (uint32_t b = tid; b < k; b += NT)
                running[b] = sg.start + lp.prefix[sg.cbase + (uint64_t)b * sg.nchunks + ch.c] - base0;
        }
        for (uint32_t w = tid; w < T / 32; w += NT) winfo[w] = 0;  // ordered before the run bits by the scan's barriers
        if (!C::P16) scan_counters32<NT>(tab, C::NW, k, bst, wsum, rix);
        else scan_counters<NT>(tab, C::NW, k, bst, wsum, rix);
        // a segment of <= 2^32 elements: every destination minus the segment
        // start fits 32 bits, so delta is kept modulo 2^32 (half the lookup
        // bytes in the copy-out); longer segments keep 64-bit deltas
        const bool wide = (sg.len >> 32) != 0 || (rp.dbg & 64u);  // SHUF_DBG=64: test hook forcing the 64-bit path
        for (uint32_t b = tid; b < k; b += NT) {
            const uint32_t s0 = bst[b], s1 = bst[b + 1];
            if (s1 > s0) {  // run r = rix[b]: slots [s0, s1)
                const uint32_t r = rix[b];
                if (wide) delta64[r] = running[b] - s0;
                else delta[r] = (uint32_t)(running[b] - sg.start) - s0;
                atomicOr(reinterpret_cast<uint32_t*>(&winfo[s0 >> 5]), 1u << (s0 & 31u));
                // windows whose first slot lies in the run
                for (uint32_t w = (s0 + 31u) >> 5; (w << 5) < s1; ++w)
                    reinterpret_cast<uint32_t*>(&winfo[w])[1] = r + ((w << 5) == s0 ? 0u : 1u);
                running[b] += s1 - s0;
            }
        }
        // ---- C: rank + place (the tile's data must have landed)
        mbar_wait(&bar[0], ph);
        ph ^= 1u;
        const uint32_t doff = (uint32_t)((cur.q0 - sg.origin) & (C::dpg - 1));
        if (cnt == T)
            s_place<EB, NARROW, ORD, true>(raw, cur.q0, draws, doff, cnt, sorted, Tw, warp, lane, &rp.hdr->error);
        else
            s_place<EB, NARROW, ORD, false>(raw, cur.q0, draws, doff, cnt, sorted, Tw, warp, lane, &rp.hdr->error);
        __syncthreads();  // raw consumed; sorted, run map and delta complete
        // ---- next tile of this CTA's sequence: load it into the raw buffer
        STile nxt = cur;
        nxt.q0 = cur.q0 + cnt;
        const bool next_chunk = nxt.q0 >= cur.q1;
        if (next_chunk) {
            nxt = s_first_tile(lp, rp, cur.chunk + gridDim.x, nchunk);
            if (nxt.chunk < nchunk) scattered += nxt.q1 - nxt.q0;
        }
        const uint32_t ncnt = (uint32_t)min((uint64_t)T, nxt.q1 - nxt.q0);
        if (nxt.chunk < nchunk) s_issue_load<EB>(nxt.q0, ncnt, src, raw, &bar[0]);
        // ---- D: copy-out of tile `cur`: slot x -> dst[delta[run(x)] + x]
        {
            const E* so = reinterpret_cast<const E*>(sorted);
            const uint32_t le = lanemask_le();
            if (!wide) {
                E* dst = reinterpret_cast<E*>(dstb) + sg.start;
                if (cnt == T) {
#pragma unroll 8
                    for (uint32_t j = 0; j < T / NT; ++j) {
                        const uint32_t x = tid + j * NT;
                        const uint64_t wi = winfo[x >> 5];
                        const uint32_t r = (uint32_t)(wi >> 32) + __popc((uint32_t)wi & le) - 1u;
                        dst[(uint32_t)(delta[r] + x)] = so[x];
                    }
                } else {
                    for (uint32_t x = tid; x < ((cnt + 31u) & ~31u); x += NT) {
                        const uint64_t wi = winfo[x >> 5];
                        const uint32_t r = (uint32_t)(wi >> 32) + __popc((uint32_t)wi & le) - 1u;
                        if (x < cnt) dst[(uint32_t)(delta[r] + x)] = so[x];
                    }
                }
            } else {
                E* dst = reinterpret_cast<E*>(dstb);
                for (uint32_t x = tid; x < ((cnt + 31u) & ~31u); x += NT) {
                    const uint64_t wi = winfo[x >> 5];
                    const uint32_t r = (uint32_t)(wi >> 32) + __popc((uint32_t)wi & le) - 1u;
                    if (x < cnt) dst[delta64[r] + x] = so[x];
                }
            }
        }
        if (nxt.chunk >= nchunk) break;
        // ---- A: draws + counts of the next tile (positions only)
        const SegDesc nsg = next_chunk ? lp.segs[nxt.seg] : sg;
        s_draw_count<EB, NARROW>(bp, make_key(nsg.key), lp.level, nxt.q0 - nsg.origin, ncnt, draws, Tw, kw, warp,
                                 lane);
        __syncthreads();  // copy-out done (sorted, run map, delta free); counts complete
        new_chunk = next_chunk;
        cur = nxt;
        cnt = ncnt;
        sg = nsg;
    }
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->scattered_hbm[lp.level], scattered);
}

// Kernel selection: element size x ranking mode x lane width.
template <int EB>
static void* scatter_fn(bool ord, bool narrow) {
    if (ord) return narrow ? (void*)k_scatter<EB, true, true> : (void*)k_scatter<EB, false, true>;
    return narrow ? (void*)k_scatter<EB, true, false> : (void*)k_scatter<EB, false, false>;
}

static void* scatter_kernel(uint32_t eb, bool ord, bool narrow) {
    switch (eb) {
    case 4: return scatter_fn<4>(ord, narrow);
    case 8: return scatter_fn<8>(ord, narrow);
    default: return scatter_fn<16>(ord, narrow);
    }
}

static uint32_t scatter_threads(uint32_t, uint32_t) { return SCfg<4, true>::NT; }

cudaError_t launch_scatter(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = scatter_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(scatter_kernel(rp.eb, rp.rank_ordered != 0, rp.bp.narrow != 0), dim3(grid),
                            dim3(scatter_threads(rp.eb, rp.k)), args, smem, s);
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
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, scatter_kernel(eb, true, is_narrow(k)),
                                                         scatter_threads(eb, k), scatter_smem_bytes(eb, k));
}

}  // namespace shuf
