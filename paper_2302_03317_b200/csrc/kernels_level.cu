// HBM-resident ("global") scatter level: init, histogram, decoupled-lookback
// scan, segment planner and the TMA-staged stable scatter.
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
        sd.origin = a;
        sd.key = rp.seed + s * 0x9E3779B97F4A7C15ull;  // K(seed, s) (D2)
        sd.cbase = (uint64_t)cb * rp.k;
        sd.nchunks = (uint32_t)nch;
        sd.pad = 0;
        lp0.segs[si] = sd;
        for (uint64_t c = 0; c < nch; ++c) lp0.chunks[cb + c] = ChunkDesc{si, (uint32_t)c};
    }
}

// ------------------------------------------------------------- histogram --
// counts[cbase + b*nchunks + c] = #{p in chunk c : bucket(l, p) = b}.
// Regenerates the draws from Philox counters; reads no element data.
__global__ void __launch_bounds__(kThreads) k_hist(RunParams rp, LevelParams lp) {
    extern __shared__ uint32_t hist[];
    const uint32_t nchunk = lp.ctr->nchunk;
    const uint64_t E = (uint64_t)nchunk * rp.k;
    const uint64_t ntiles = (E + kScanTile - 1) / kScanTile;
    for (uint64_t t = gtid(); t < ntiles; t += gstride()) lp.status[t] = 0;
    if (gtid() == 0) {
        lp.ctr->scan_ticket = 0;
        lp.nctr->nseg = 0;
        lp.nctr->nchunk = 0;
    }
    const uint32_t k = rp.k;
    const BucketParams bp = rp.bp;
    const uint32_t sh = bp.narrow ? 4u : 3u, dpg = 1u << sh;
    for (uint32_t j = blockIdx.x; j < nchunk; j += gridDim.x) {
        for (uint32_t b = threadIdx.x; b < k; b += kThreads) hist[b] = 0;
        __syncthreads();
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
#pragma unroll
                    for (uint32_t jj = 0; jj < 16; ++jj) atomicAdd(&hist[lane8(w, jj) >> bp.shift], 1u);
                } else {
#pragma unroll
                    for (uint32_t jj = 0; jj < 8; ++jj)
                        atomicAdd(&hist[bucket_from_group(w, jj, key, lp.level, pb + jj, bp)], 1u);
                }
            } else {
                for (uint32_t jj = 0; jj < dpg; ++jj) {
                    const uint64_t p = pb + jj;
                    if (p >= P0 && p < P1) atomicAdd(&hist[bucket_from_group(w, jj, key, lp.level, p, bp)], 1u);
                }
            }
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < k; b += kThreads)
            lp.counts[sg.cbase + (uint64_t)b * sg.nchunks + ch.c] = hist[b];
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
        if (len <= rp.S_fuse) continue;  // finished by k_finish_children
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

// ---------------------------------------------------------------- scatter --
// Per CTA: a sequence of tiles (chunks blockIdx.x, +gridDim.x, ..., each walked
// tile by tile in order).  Tile t lands in buffer t&1 by one bulk async copy
// issued while tile t-1 is processed.  Each warp loads its 32-element rounds
// into registers and ranks them (block_ops.cuh); the (bucket, warp) counters
// are scanned into tile-local bases; the elements are written back into the
// same buffer in bucket-major stable order together with their bucket byte;
// then every thread copies slots s = tid, tid+512, ... to
// dst[running[b] - bst[b] + s] (consecutive lanes -> consecutive addresses
// inside a bucket run).
template <int EB>
struct ScatterCfg {
    static constexpr uint32_t T = 32768 / EB;       // elements per tile (32 KiB)
    static constexpr uint32_t Q = T / kWarps;        // elements per warp
    static constexpr uint32_t R = Q / 32;            // rounds per warp
    static constexpr uint32_t BUF = T * EB + 16;
};

struct ScatterLayout {
    uint32_t buf0, buf1, draws, slotb, C, bst, delta, running, wsum, bar, total;
};

template <int EB>
__host__ __device__ inline ScatterLayout scatter_layout(uint32_t k) {
    ScatterLayout L;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    constexpr uint32_t T = ScatterCfg<EB>::T;
    L.buf0 = take(ScatterCfg<EB>::BUF);
    L.buf1 = take(ScatterCfg<EB>::BUF);
    L.draws = take(draw_bytes(T));
    const bool narrow = (k & (k - 1)) == 0 && k <= 256;  // u8 bucket ids (make_bucket_params)
    L.slotb = take(narrow ? T : 2 * T);
    L.C = take(kWarps * ((k + 1) / 2) * 4);
    L.bst = take((k + 1) * 4);
    L.delta = take(k * 8);
    L.running = take(k * 8);
    L.wsum = take((kWarps + 1) * 4);
    L.bar = take(16);
    L.total = off;
    return L;
}

struct TileRef {
    uint32_t chunk;   // chunk index (>= nchunk: none)
    uint32_t seg;     // segment index
    uint64_t q0, q1;  // element range of the chunk's remaining part
};

__device__ __forceinline__ TileRef first_tile(const LevelParams& lp, const RunParams& rp, uint32_t j, uint32_t nchunk) {
    TileRef t;
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

template <int EB>
__device__ __forceinline__ void issue_tile_load(uint64_t q0, uint32_t cnt, const unsigned char* src,
                                                unsigned char* buf, uint64_t* bar) {
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

template <bool ORD>
__device__ __forceinline__ uint32_t rank_in_warp(uint32_t* Cw, uint32_t b, bool valid) {
    if (ORD) {
        const uint32_t sh = (b & 1u) << 4;
        const uint32_t old = valid ? atomicAdd(&Cw[b >> 1], 1u << sh) : 0u;
        return (old >> sh) & 0xFFFFu;
    } else {
        return warp_rank(Cw, b, valid, false);
    }
}

// Rank + place one tile (FULL: cnt == T, no bounds checks).
template <int EB, bool ORD, bool NARROW, bool FULL>
__device__ __forceinline__ void rank_place(unsigned char* buf, uint32_t in_off, uint32_t cnt, const DrawView& dv,
                                           uint32_t* C, uint32_t kw, uint32_t k, uint32_t* bst, uint32_t* wsum,
                                           unsigned char* slotb) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t Q = ScatterCfg<EB>::Q, R = ScatterCfg<EB>::R;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned char* tin = buf + in_off;
    uint32_t* Cw = C + warp * kw;
    E v[R];
    uint32_t rk[R];
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t e = warp * Q + r * 32 + lane;
        const bool valid = FULL || e < cnt;
        uint32_t b = 0;
        if (valid) {
            v[r] = *reinterpret_cast<const E*>(tin + e * EB);
            b = NARROW ? (uint32_t)dv.d[e + dv.off] : (uint32_t)reinterpret_cast<const uint16_t*>(dv.d)[e + dv.off];
        }
        rk[r] = (b << 16) | rank_in_warp<ORD>(Cw, b, valid);
    }
    __syncthreads();
    scan_counters<kThreads>(C, kWarps, k, bst, wsum);
    E* stage = reinterpret_cast<E*>(buf);
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t e = warp * Q + r * 32 + lane;
        if (FULL || e < cnt) {
            const uint32_t b = rk[r] >> 16;
            const uint32_t slot = ((Cw[b >> 1] >> ((b & 1u) << 4)) & 0xFFFFu) + (rk[r] & 0xFFFFu);
            stage[slot] = v[r];
            if (NARROW) slotb[slot] = (unsigned char)b;
            else reinterpret_cast<uint16_t*>(slotb)[slot] = (uint16_t)b;
        }
    }
}

template <int EB, bool ORD, bool NARROW>
__global__ void __launch_bounds__(kThreads, 2) k_scatter(RunParams rp, LevelParams lp) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t T = ScatterCfg<EB>::T;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const ScatterLayout Ly = scatter_layout<EB>(k);
    unsigned char* dsm = sm + Ly.draws;
    unsigned char* slotb = sm + Ly.slotb;
    uint32_t* C = reinterpret_cast<uint32_t*>(sm + Ly.C);
    uint32_t* bst = reinterpret_cast<uint32_t*>(sm + Ly.bst);
    uint64_t* delta = reinterpret_cast<uint64_t*>(sm + Ly.delta);
    uint64_t* running = reinterpret_cast<uint64_t*>(sm + Ly.running);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + Ly.wsum);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Ly.bar);

    const uint32_t tid = threadIdx.x;
    const uint32_t nchunk = lp.ctr->nchunk;
    if (blockIdx.x >= nchunk) return;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned char* __restrict__ src = lp.src;
    E* __restrict__ dst = reinterpret_cast<E*>(lp.dst);
    uint32_t ph0 = 0, ph1 = 0;

    TileRef cur = first_tile(lp, rp, blockIdx.x, nchunk);
    uint32_t cnt = (uint32_t)min((uint64_t)T, cur.q1 - cur.q0);
    issue_tile_load<EB>(cur.q0, cnt, src, sm + Ly.buf0, &bar[0]);
    unsigned long long scattered = cur.q1 - cur.q0;
    bool new_chunk = true;
    for (uint32_t it = 0; cur.chunk < nchunk; ++it) {
        // ---- prefetch the next tile of this CTA's sequence into the other buffer
        TileRef nxt = cur;
        nxt.q0 = cur.q0 + cnt;
        const bool next_chunk = nxt.q0 >= cur.q1;
        if (next_chunk) {
            nxt = first_tile(lp, rp, cur.chunk + gridDim.x, nchunk);
            if (nxt.chunk < nchunk) scattered += nxt.q1 - nxt.q0;
        }
        const uint32_t ncnt = (uint32_t)min((uint64_t)T, nxt.q1 - nxt.q0);
        unsigned char* buf = sm + ((it & 1u) ? Ly.buf1 : Ly.buf0);
        if (nxt.chunk < nchunk)
            issue_tile_load<EB>(nxt.q0, ncnt, src, sm + ((it & 1u) ? Ly.buf0 : Ly.buf1), &bar[(it & 1u) ^ 1u]);
        const SegDesc sg = lp.segs[cur.seg];
        if (new_chunk) {
            const ChunkDesc ch = lp.chunks[cur.chunk];
            const uint64_t base0 = lp.prefix[sg.cbase];
            for (uint32_t b = tid; b < k; b += kThreads)
                running[b] = sg.start + lp.prefix[sg.cbase + (uint64_t)b * sg.nchunks + ch.c] - base0;
        }
        // ---- draws of the tile's positions, zero the counters, wait for the data
        const DrawView dv = draws_to_smem<kThreads>(dsm, cur.q0 - sg.origin, cnt, make_key(sg.key), lp.level, rp.bp);
        for (uint32_t i = tid; i < kWarps * kw; i += kThreads) C[i] = 0;
        if (it & 1u) {
            mbar_wait(&bar[1], ph1);
            ph1 ^= 1u;
        } else {
            mbar_wait(&bar[0], ph0);
            ph0 ^= 1u;
        }
        __syncthreads();
        const uint32_t in_off = (uint32_t)((cur.q0 * EB) & 15u);
        if (cnt == T) rank_place<EB, ORD, NARROW, true>(buf, in_off, cnt, dv, C, kw, k, bst, wsum, slotb);
        else rank_place<EB, ORD, NARROW, false>(buf, in_off, cnt, dv, C, kw, k, bst, wsum, slotb);
        for (uint32_t b = tid; b < k; b += kThreads) {
            delta[b] = running[b] - bst[b];
            running[b] += bst[b + 1] - bst[b];
        }
        __syncthreads();
        // ---- copy out: slot s goes to dst[running[b] - bst[b] + s]
        const E* stage = reinterpret_cast<const E*>(buf);
        if (cnt == T) {
#pragma unroll 4
            for (uint32_t s = tid; s < T; s += kThreads) {
                const uint32_t b = NARROW ? (uint32_t)slotb[s] : (uint32_t)reinterpret_cast<const uint16_t*>(slotb)[s];
                dst[delta[b] + s] = stage[s];
            }
        } else {
            for (uint32_t s = tid; s < cnt; s += kThreads) {
                const uint32_t b = NARROW ? (uint32_t)slotb[s] : (uint32_t)reinterpret_cast<const uint16_t*>(slotb)[s];
                dst[delta[b] + s] = stage[s];
            }
        }
        __syncthreads();
        new_chunk = next_chunk;
        cur = nxt;
        cnt = ncnt;
    }
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->scattered_hbm[lp.level], scattered);
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

cudaError_t launch_hist(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    k_hist<<<grid, kThreads, rp.k * sizeof(uint32_t), s>>>(rp, lp);
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

uint32_t scatter_smem_bytes(uint32_t eb, uint32_t k) {
    switch (eb) {
    case 4: return scatter_layout<4>(k).total;
    case 8: return scatter_layout<8>(k).total;
    default: return scatter_layout<16>(k).total;
    }
}

// Kernel selection: element size x ranking mode x lane width.
template <int EB>
static void* scatter_fn(bool ord, bool narrow) {
    if (ord) return narrow ? (void*)k_scatter<EB, true, true> : (void*)k_scatter<EB, true, false>;
    return narrow ? (void*)k_scatter<EB, false, true> : (void*)k_scatter<EB, false, false>;
}

static void* scatter_kernel(const RunParams& rp) {
    const bool ord = rp.rank_ordered != 0, nar = rp.bp.narrow != 0;
    switch (rp.eb) {
    case 4: return scatter_fn<4>(ord, nar);
    case 8: return scatter_fn<8>(ord, nar);
    default: return scatter_fn<16>(ord, nar);
    }
}

cudaError_t launch_scatter(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = scatter_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(scatter_kernel(rp), dim3(grid), dim3(kThreads), args, smem, s);
}

cudaError_t configure_scatter(uint32_t smem) {
    cudaError_t e;
    for (int eb : {4, 8, 16})
        for (int o = 0; o < 2; ++o)
            for (int nr = 0; nr < 2; ++nr) {
                void* f = eb == 4 ? scatter_fn<4>(o, nr) : (eb == 8 ? scatter_fn<8>(o, nr) : scatter_fn<16>(o, nr));
                if ((e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
            }
    return cudaSuccess;
}

cudaError_t occupancy_level(uint32_t eb, uint32_t k, int* hist, int* scan, int* scatter) {
    cudaError_t e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(hist, k_hist, kThreads, k * sizeof(uint32_t)))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(scan, k_scan, kThreads, 0))) return e;
    const uint32_t smem = scatter_smem_bytes(eb, k);
    void* f = eb == 4 ? scatter_fn<4>(true, true) : (eb == 8 ? scatter_fn<8>(true, true) : scatter_fn<16>(true, true));
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(scatter, f, kThreads, smem);
}

}  // namespace shuf
