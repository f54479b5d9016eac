// CTA-wide building blocks shared by the scatter and finish kernels:
// draw generation into shared memory, stable in-warp ranking, the
// bucket-major scan of per-warp counters.  (CUDA path only.)
//
// Stable ranking.  A warp walks its sub-tile in rounds of
// 32 consecutive elements, lane order = position order.  Each lane adds 1 to
// its bucket's counter in the warp's own counter table with ONE shared-memory
// atomicAdd; the value returned is the element's rank among the warp's
// elements of that bucket so far.  This is stable because same-address
// atomics of one warp instruction return in ascending lane order on this GPU:
// the PTX ISA leaves that order unspecified, so the library checks it at
// setup with a probe kernel (k_rank_order_probe) and otherwise uses the
// documented __match_any_sync path (rank = count + popc(peers & lanemask_lt)).
// Counters are u16 halves of u32 words (bucket b -> word b>>1, half b&1).
#pragma once
#include <cstdint>

#include "philox.cuh"
#include "ptx.cuh"
#include "shuf_internal.cuh"

namespace shuf {

template <int EB> struct ElemT;
template <> struct ElemT<4> { using type = uint32_t; };
template <> struct ElemT<8> { using type = uint2; };
template <> struct ElemT<16> { using type = uint4; };

__device__ __forceinline__ uint32_t warp_inclusive_sum(uint32_t v) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= (uint32_t)o) v += t;
    }
    return v;
}

// Self-check of the ordered-atomic ranking (see the top of this file): the
// lanes of one warp instruction that share a bucket must have received
// consecutive slots in lane order.  One __match_any_sync per call (slow, ~60
// SM-cycles), so callers sample it -- one round per tile / item.  A violation
// latches SHUF_ERR_RANK_ORDER (7) in *err: the output is then not D6's.
__device__ __forceinline__ void check_rank_order(uint32_t b, bool valid, uint32_t slot, uint32_t* err) {
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, valid ? b : 0xFFFFFFFFu);
    const uint32_t lower = peers & lanemask_lt();
    const int src = lower ? 31 - __clz(lower) : (int)(threadIdx.x & 31u);
    const uint32_t prev = __shfl_sync(0xFFFFFFFFu, slot, src);
    if (valid && lower && prev + 1u != slot) atomicCAS(err, 0u, 7u);
}

// Exclusive scan over one value per thread; returns the thread's exclusive
// prefix, *total gets the block total.  wsum: shared scratch of NT/32+1 words.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_sum(uint32_t v, uint32_t* wsum, uint32_t* total) {
    constexpr int NW = NT / 32;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t incl = warp_inclusive_sum(v);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = lane < (uint32_t)NW ? wsum[lane] : 0u;
        const uint32_t xi = warp_inclusive_sum(x);
        if (lane < (uint32_t)NW) wsum[lane] = xi - x;
        if (lane == NW - 1) wsum[NW] = xi;
    }
    __syncthreads();
    const uint32_t r = wsum[warp] + incl - v;
    *total = wsum[NW];
    __syncthreads();
    return r;
}

// Draw array in shared memory for positions [P0, P0+m): index of position p
// is p - base with base = P0 rounded down to a Philox group; narrow draws
// are u8, wide draws u16.  One Philox call per group, stored with one
// 16-byte store when the group lies inside the range.
struct DrawView {
    unsigned char* d;
    uint32_t off;     // P0 - base
    uint32_t narrow;
    __device__ __forceinline__ uint32_t at(uint32_t e) const {
        return narrow ? (uint32_t)d[e + off] : (uint32_t)reinterpret_cast<const uint16_t*>(d)[e + off];
    }
};

template <int NT>
__device__ __forceinline__ DrawView draws_to_smem(unsigned char* d, uint64_t P0, uint32_t m, PhiloxKey key,
                                                  uint32_t level, const BucketParams& bp) {
    const uint32_t sh = bp.narrow ? 4u : 3u, dpg = 1u << sh;
    const uint64_t g0 = P0 >> sh;
    DrawView v{d, (uint32_t)(P0 - (g0 << sh)), bp.narrow};
    if (m == 0) return v;
    const uint32_t ng = (uint32_t)(((P0 + m - 1) >> sh) - g0 + 1);
    for (uint32_t t = threadIdx.x; t < ng; t += NT) {
        const uint64_t g = g0 + t;
        const uint4 w = bucket_group_words(key, level, g);
        const uint64_t pb = g << sh;
        if (bp.narrow && bp.shift == 0) {  // k = 256: the lanes are the buckets
            *reinterpret_cast<uint4*>(d + (size_t)t * 16) = w;
        } else if (bp.narrow) {
            const uint32_t s = bp.shift, msk = (0xFFu >> s) * 0x01010101u;
            *reinterpret_cast<uint4*>(d + (size_t)t * 16) =
                make_uint4((w.x >> s) & msk, (w.y >> s) & msk, (w.z >> s) & msk, (w.w >> s) & msk);
        } else {
            uint32_t b[8];
            if (pb >= P0 && pb + dpg <= P0 + m) {
#pragma unroll
                for (uint32_t j = 0; j < 8; ++j) b[j] = bucket_from_group(w, j, key, level, pb + j, bp);
            } else {
#pragma unroll
                for (uint32_t j = 0; j < 8; ++j)
                    b[j] = (pb + j >= P0 && pb + j < P0 + m) ? bucket_from_group(w, j, key, level, pb + j, bp) : 0u;
            }
            *reinterpret_cast<uint4*>(d + (size_t)t * 16) =
                make_uint4(b[0] | (b[1] << 16), b[2] | (b[3] << 16), b[4] | (b[5] << 16), b[6] | (b[7] << 16));
        }
    }
    return v;
}

// Bytes of draw storage for m positions (plus one group of slack on each side).
__host__ __device__ inline uint32_t draw_bytes(uint32_t m) { return 2u * (m + 32u); }

// Stable rank of this lane's element among the warp's elements of bucket b
// processed so far; Cw = the warp's packed u16 counters.  All 32 lanes call.
__device__ __forceinline__ uint32_t warp_rank(uint32_t* Cw, uint32_t b, bool valid, bool ordered) {
    if (ordered) {
        if (!valid) return 0u;
        const uint32_t sh = (b & 1u) << 4;
        const uint32_t old = atomicAdd(&Cw[b >> 1], 1u << sh);
        return (old >> sh) & 0xFFFFu;
    }
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, valid ? b : 0xFFFFFFFFu);
    uint32_t old = 0;
    if (valid) old = (Cw[b >> 1] >> ((b & 1u) << 4)) & 0xFFFFu;
    __syncwarp();
    if (valid && (peers & lanemask_lt()) == 0)
        atomicAdd(&Cw[b >> 1], (uint32_t)__popc(peers) << ((b & 1u) << 4));
    __syncwarp();
    return old + __popc(peers & lanemask_lt());
}

// C holds nw packed-u16 counter tables of k entries (table w at C + w*kw,
// kw = ceil(k/2) words).  Replace every count by its exclusive prefix in
// (bucket, warp) order and write bucket starts to bst[0..k] (bst[k] = total).
// With rix != nullptr also rix[b] = the number of non-empty buckets before b
// (the run index of bucket b; the total must stay below 2^16: the two
// prefixes share one scan).  Each thread owns a contiguous run of words.  All
// NT threads call.
template <int NT>
__device__ __forceinline__ void scan_counters(uint32_t* C, uint32_t nw, uint32_t k, uint32_t* bst, uint32_t* wsum,
                                              uint32_t* rix = nullptr) {
    const uint32_t kw = (k + 1) >> 1;
    const uint32_t per = (kw + NT - 1) / NT;
    const uint32_t x0 = threadIdx.x * per, x1 = min(kw, x0 + per);
    uint32_t mine = 0, ne = 0;
    for (uint32_t x = x0; x < x1; ++x) {
        uint32_t t0 = 0, t1 = 0;
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t c = C[w * kw + x];
            t0 += c & 0xFFFFu;
            t1 += c >> 16;
        }
        mine += t0 + t1;
        ne += (t0 != 0) + (t1 != 0);
    }
    uint32_t total;
    const uint32_t pre = block_exclusive_sum<NT>(rix ? mine | (ne << 16) : mine, wsum, &total);
    uint32_t run = rix ? pre & 0xFFFFu : pre, rr = pre >> 16;
    for (uint32_t x = x0; x < x1; ++x) {
        uint32_t t0 = 0, t1 = 0;
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t c = C[w * kw + x];
            t0 += c & 0xFFFFu;
            t1 += c >> 16;
        }
        bst[2 * x] = run;
        if (2 * x + 1 < k) bst[2 * x + 1] = run + t0;
        if (rix) {
            rix[2 * x] = rr;
            rr += t0 != 0;
            if (2 * x + 1 < k) rix[2 * x + 1] = rr;
            rr += t1 != 0;
        }
        uint32_t r0 = run, r1 = run + t0;
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t c = C[w * kw + x];
            C[w * kw + x] = (r0 & 0xFFFFu) | (r1 << 16);
            r0 += c & 0xFFFFu;
            r1 += c >> 16;
        }
        run += t0 + t1;
    }
    if (threadIdx.x == 0) bst[k] = rix ? total & 0xFFFFu : total;
    __syncthreads();
}

// As scan_counters for unpacked u32 counters: C holds nw tables of k words
// (table w at C + w*k).
template <int NT>
__device__ __forceinline__ void scan_counters32(uint32_t* C, uint32_t nw, uint32_t k, uint32_t* bst, uint32_t* wsum,
                                                uint32_t* rix = nullptr) {
    const uint32_t per = (k + NT - 1) / NT;
    const uint32_t x0 = threadIdx.x * per, x1 = min(k, x0 + per);
    uint32_t mine = 0, ne = 0;
    for (uint32_t x = x0; x < x1; ++x) {
        uint32_t c = 0;
        for (uint32_t w = 0; w < nw; ++w) c += C[w * k + x];
        mine += c;
        ne += c != 0;
    }
    uint32_t total;
    const uint32_t pre = block_exclusive_sum<NT>(rix ? mine | (ne << 16) : mine, wsum, &total);
    uint32_t run = rix ? pre & 0xFFFFu : pre, rr = pre >> 16;
    for (uint32_t x = x0; x < x1; ++x) {
        bst[x] = run;
        const uint32_t r0 = run;
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t c = C[w * k + x];
            C[w * k + x] = run;
            run += c;
        }
        if (rix) {
            rix[x] = rr;
            rr += run != r0;
        }
    }
    if (threadIdx.x == 0) bst[k] = rix ? total & 0xFFFFu : total;
    __syncthreads();
}

// ---------------------------------------------------- Fisher-Yates ------
// One Fisher-Yates step (Fig. 1): swap(A[i], A[j]), j = fy(q, i) from the
// 16-bit lane v of the step's Philox group (D5, Lemire16).
template <typename E>
__device__ __forceinline__ void fy_step(E* A, uint32_t i, uint32_t v, PhiloxKey key, uint64_t q) {
    const uint32_t s = i + 1, mm = v * s;
    uint32_t j = mm >> 16;
    if (__builtin_expect((mm & 0xFFFFu) < s, 0)) j = fy16_from_lane(v, key, q, i);  // exact rejection test
    const E t = A[i];
    A[i] = A[j];
    A[j] = t;
}

// Partners j_i of the 8 steps i = 8g .. 8g+7 of a leaf (D5: 16-bit lane i&7
// of the group's Philox block, Lemire16), packed 16 bits per step.  The
// multiply-shift candidate is exact unless its low half is below s; those
// rare steps take the exact test (and the retry stream) out of line.
static __device__ __noinline__ uint4 fy_group_fixup(uint4 pj, uint32_t rej, uint4 w, PhiloxKey key, uint64_t q,
                                                    uint32_t g) {
    uint32_t p[4] = {pj.x, pj.y, pj.z, pj.w};
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
    for (uint32_t jj = 0; jj < 8; ++jj) {
        if (!((rej >> jj) & 1u)) continue;
        const uint32_t v = (wv[jj >> 1] >> ((jj & 1u) * 16u)) & 0xFFFFu;
        const uint32_t j = fy16_from_lane(v, key, q, g * 8u + jj);
        const uint32_t sh = (jj & 1u) * 16u;
        p[jj >> 1] = (p[jj >> 1] & ~(0xFFFFu << sh)) | (j << sh);
    }
    return make_uint4(p[0], p[1], p[2], p[3]);
}

__device__ __forceinline__ uint4 fy_group_partners(uint4 w, PhiloxKey key, uint64_t q, uint32_t g) {
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
    uint32_t p[4] = {0u, 0u, 0u, 0u};
    uint32_t rej = 0;
#pragma unroll
    for (uint32_t jj = 0; jj < 8; ++jj) {
        const uint32_t i = g * 8u + jj, s = i + 1;
        const uint32_t v = (wv[jj >> 1] >> ((jj & 1u) * 16u)) & 0xFFFFu;
        const uint32_t mm = v * s;
        p[jj >> 1] |= (mm >> 16) << ((jj & 1u) * 16u);
        rej |= (((mm & 0xFFFFu) < s) && i >= 1) ? (1u << jj) : 0u;
    }
    uint4 pj = make_uint4(p[0], p[1], p[2], p[3]);
    if (__builtin_expect(rej != 0, 0)) pj = fy_group_fixup(pj, rej, w, key, q, g);
    return pj;
}

// The swaps of one group, steps 8g+7 .. 8g (those in [lo, hi] only when CHECK).
template <typename E, bool CHECK>
__device__ __forceinline__ void fy_group_swaps(E* A, uint32_t g, uint4 pj, uint32_t lo, uint32_t hi) {
    const uint32_t pv[4] = {pj.x, pj.y, pj.z, pj.w};
#pragma unroll
    for (int32_t jj = 7; jj >= 0; --jj) {
        const uint32_t i = g * 8u + (uint32_t)jj;
        if (CHECK && !(i >= lo && i <= hi)) continue;
        if (!CHECK && jj == 0 && g == 0) continue;
        const uint32_t j = (pv[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu;
        const E t = A[i];
        A[i] = A[j];
        A[j] = t;
    }
}

// Fisher-Yates (Fig. 1) of the leaf A[0 .. cm) whose first
// element is problem position q: for i = cm-1 .. 1, swap(i, fy(q, i)) with
// the partner drawn for (leaf id q, step i) (D5): one Philox call per 8
// steps, so every lane of a warp (each on its own leaf) draws in lockstep.
// Partners come a group at a time (branch-free but for rare rejections);
// the next group's Philox block is computed one group ahead.
template <int EB>
__device__ __forceinline__ void fy_leaf(unsigned char* el, uint32_t c, uint32_t cm, uint64_t q, PhiloxKey key) {
    using E = typename ElemT<EB>::type;
    if (cm < 2) return;
    E* A = reinterpret_cast<E*>(el) + c;
    const uint32_t gt = (cm - 1) >> 3;
    uint4 wn = fy16_group_words(key, q, gt);
    {  // top group: steps cm-1 .. max(8*gt, 1)
        const uint4 pj = fy_group_partners(wn, key, q, gt);
        if (gt >= 1) wn = fy16_group_words(key, q, gt - 1);
        fy_group_swaps<E, true>(A, gt, pj, 1u, cm - 1);
    }
    for (int32_t g = (int32_t)gt - 1; g >= 1; --g) {  // full groups
        const uint4 pj = fy_group_partners(wn, key, q, (uint32_t)g);
        wn = fy16_group_words(key, q, (uint32_t)g - 1u);
        fy_group_swaps<E, false>(A, (uint32_t)g, pj, 0u, 0u);
    }
    if (gt >= 1) {  // group 0: steps 7 .. 1
        const uint4 pj = fy_group_partners(wn, key, q, 0u);
        fy_group_swaps<E, false>(A, 0u, pj, 0u, 0u);
    }
}

}  // namespace shuf
