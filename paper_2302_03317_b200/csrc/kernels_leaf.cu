// Leaf kernel: Fisher-Yates (Fig. 1) of every
// leaf -- a segment of at most L elements -- with one thread per leaf and
// many leaves in flight per SM.
//
// Leaves come in units of up to 32 consecutive children of one segment of a
// level (children b = 32g .. 32g+31; a level's children of at most L
// elements are leaves, D6), or of up to 32 consecutive user segments at
// level 0 (D7).  A warp takes a unit and processes its leaves in batches
// that fit the warp's shared-memory slot: lane x owns leaf x of the batch,
// loads it with one bulk async copy (TMA engine; <= 3 unaligned words at
// each end by 4-byte asynchronous copies), runs Fisher-Yates on it with the
// D5 draws of (leaf id = problem position of the leaf start, step), and
// stores it back to ptr the same way.  No CTA barriers: warps are
// independent, so the leaf chains of up to 32 x (warps per SM) leaves hide
// each other's latency.
#include <cuda_runtime.h>

#include <cstdlib>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char lsm[];

constexpr uint32_t kLeafThreads = 128;  // 4 warps per CTA
constexpr uint32_t kLeafWarps = kLeafThreads / 32;

// Slot bytes per warp: at least 16 KiB, and room for one leaf of L elements
// plus its u16 Fisher-Yates partners (the warp-cooperative path).
__host__ __device__ inline uint32_t leaf_slot_bytes(uint32_t eb, uint32_t L) {
    uint32_t s = ((L * eb + 32 + 15) & ~15u) + ((2 * L + 15) & ~15u) + ((L + 15) & ~15u);
    return s < 16384u ? 16384u : s;
}

// Fisher-Yates (Fig. 1) of ONE long leaf A[0..m) by a whole warp, bit for bit
// the sequential result: the partners j_i (D5) are precomputed into P; then
// in rounds the lanes take steps i = top, top-1, .., top-31 and the longest
// prefix of them that touches pairwise distinct positions runs at once --
// lane l conflicts if another lane shares its partner (every lane writes its
// id to M[j], then reads it back: a different id means a shared partner --
// of lanes sharing one, every loser of the store is flagged, and the prefix
// ends before the first flagged lane, at least one step) or if an
// earlier lane's partner is l's own position i_l (that lane sets bit l of
// a warp OR-reduction; an earlier lane's i can never be l's partner, as
// j_l <= i_l).  Lane 0's step is always safe alone, so every
// round makes progress.
template <int EB>
__device__ __forceinline__ void fy_leaf_warp(unsigned char* el, uint16_t* P, unsigned char* M, uint32_t m, uint64_t q,
                                             PhiloxKey key) {
    using E = typename ElemT<EB>::type;
    const uint32_t lane = threadIdx.x & 31u;
    if (m < 2) return;
    const uint32_t ng = ((m - 1) >> 3) + 1;
    // Steps whose multiply-shift candidate may be rejected (low half < s:
    // probability s/2^16, a few % on long leaves) go to a list in M and are
    // settled afterwards by all lanes at once (exact test: 2^16 mod s, retry
    // stream) -- inline, the rare lane's modulo and retry held the whole warp.
    uint32_t* ncand = reinterpret_cast<uint32_t*>(M);
    uint32_t* cand = ncand + 4;
    const uint32_t cap = (m >> 2) - 4;  // M holds >= m bytes; long leaves only (m > 512)
    if (lane == 0) *ncand = 0;
    __syncwarp();
    for (uint32_t g = lane; g < ng; g += 32) {
        const uint4 w = fy16_group_words(key, q, g);
        const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (uint32_t jj = 0; jj < 8; ++jj) {
            const uint32_t i = g * 8u + jj;
            if (i >= 1 && i < m) {
                const uint32_t v = (wv[jj >> 1] >> ((jj & 1u) * 16u)) & 0xFFFFu;
                const uint32_t sb = i + 1, mm = v * sb;
                P[i] = (uint16_t)(mm >> 16);
                if (__builtin_expect((mm & 0xFFFFu) < sb, 0)) {
                    const uint32_t x = atomicAdd(ncand, 1u);
                    if (x < cap) cand[x] = i | (v << 16);
                    else P[i] = (uint16_t)fy16_from_lane(v, key, q, i);
                }
            }
        }
    }
    __syncwarp();
    const uint32_t nc = min(*ncand, cap);
    for (uint32_t x = lane; x < nc; x += 32) {
        const uint32_t e = cand[x], i = e & 0xFFFFu;
        P[i] = (uint16_t)fy16_from_lane(e >> 16, key, q, i);
    }
    __syncwarp();
    E* A = reinterpret_cast<E*>(el);
    int32_t top = (int32_t)m - 1;
    const uint32_t Ms = smem_u32(M);
    while (top >= 1) {
        const int32_t i = top - (int32_t)lane;
        const bool valid = i >= 1;
        const uint32_t j = valid ? (uint32_t)P[i] : 0u;
        // both operands load before the conflict test (off the round's critical
        // path); only the lanes that run use them, and no running lane's
        // positions are touched by another running lane this round
        const E a = A[valid ? i : 0], b = A[j];
        // every lane marks its own position, then its partner: a lane whose own
        // mark was overwritten is the partner of an earlier lane; a lane whose
        // partner mark was overwritten shares its partner
        if (valid) sts_u8(Ms + (uint32_t)i, lane);
        __syncwarp();
        if (valid) sts_u8(Ms + j, lane);
        __syncwarp();
        const uint32_t mj = lds_u8(Ms + j), mi = lds_u8(Ms + (valid ? (uint32_t)i : 0u));  // both loads in flight
        const bool conflict = valid & ((mj != lane) | (mi != lane));
        const uint32_t cmask = __ballot_sync(0xFFFFFFFFu, conflict);
        // Which of two same-address stores to M survives is unspecified: of lanes
        // sharing a partner at least every loser is flagged, so the prefix ends
        // before the first of them; if that is lane 0 it runs alone (a single step
        // is always safe), which also guarantees progress.
        const uint32_t c = cmask ? max((uint32_t)(__ffs(cmask) - 1), 1u) : min(32u, (uint32_t)top);
        if (lane < c) {
            A[i] = b;
            A[j] = a;
        }
        __syncwarp();
        top -= (int32_t)c;
    }
}
// Warps per leaf CTA (1..4): the count that puts the most warps on an SM
// (228 KiB of shared memory, 1 KiB reserved per CTA), the larger CTA on a
// tie.  E.g. u32 with L = 4096 (28.7 KiB slots): 4-warp CTAs fit once per SM
// (4 warps), 1-warp CTAs 7 times (7 warps); 16-byte elements with L = 4096
// (a 64 KiB slot) get 1-warp CTAs, 3 per SM.  SHUF_LEAF_WARPS=w forces w.
uint32_t leaf_warps(uint32_t eb, uint32_t L) {
    static const int forced = [] {
        const char* e = std::getenv("SHUF_LEAF_WARPS");
        return e ? std::atoi(e) : 0;
    }();
    const uint32_t per = leaf_slot_bytes(eb, L) + 16;
    if (forced >= 1 && forced <= (int)kLeafWarps && forced * per <= kSmemLimit) return (uint32_t)forced;
    constexpr uint32_t kSmSmem = 228u * 1024u, kCtaReserve = 1024u;
    uint32_t best = 1, best_warps = 0;
    for (uint32_t w = 1; w <= kLeafWarps; ++w) {
        if (w * per > kSmemLimit) break;
        uint32_t ctas = kSmSmem / (w * per + kCtaReserve);
        if (ctas > 32u) ctas = 32u;
        if (ctas * w >= best_warps) {
            best_warps = ctas * w;
            best = w;
        }
    }
    return best;
}
uint32_t leaf_smem_bytes(uint32_t eb, uint32_t L) { return leaf_warps(eb, L) * (leaf_slot_bytes(eb, L) + 16); }
uint32_t leaf_warps_per_cta(uint32_t eb, uint32_t L) { return leaf_warps(eb, L); }
// Leaf warps resident on an SM with slots for leaves of L elements.
uint32_t leaf_warps_per_sm(uint32_t eb, uint32_t L) {
    const uint32_t w = leaf_warps(eb, L);
    uint32_t ctas = (228u * 1024u) / (w * (leaf_slot_bytes(eb, L) + 16) + 1024u);
    if (ctas > 32u) ctas = 32u;
    return ctas * w;
}

struct Leaf {
    uint64_t start, len, origin, key;
};

// Units of U leaves per warp: U = 32 (lane x owns leaf x of the unit) when
// leaves are short, U = 1 when a leaf of the launch's expected length `avg`
// already takes the warp-cooperative path (fewer than 8 fit the slot) -- then
// one long leaf per warp-unit spreads the long leaves over all warps instead
// of 32 of them over one warp.  `avg` comes from the host: the expected child
// length of the level (n / k^(l+1)) or the mean user-segment length.
uint32_t leaf_unit(uint32_t eb, uint32_t L, uint64_t avg) {
    if (avg > L) avg = L;
    return 8u * ((uint32_t)avg * eb + 32u) > leaf_slot_bytes(eb, L) ? 1u : 32u;
}

// Leaf `lane` of unit u of a level's children: children U*g .. U*g+U-1 of
// segment s, u = s * ceil(k/U) + g.
struct ChildLeaves {
    const LevelParams* lp;
    uint32_t k, groups, U;
    __device__ __forceinline__ uint64_t units() const { return (uint64_t)lp->ctr->nseg * groups; }
    __device__ __forceinline__ Leaf get(uint64_t u, uint32_t lane) const {
        Leaf f{0, 0, 0, 0};
        const uint32_t s = (uint32_t)(u / groups), b = (uint32_t)(u % groups) * U + lane;
        if (lane < U && b < k) {
            const SegDesc sg = lp->segs[s];
            const uint64_t base0 = lp->prefix[sg.cbase];
            const uint64_t s0 = lp->prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
            const uint64_t s1 = (b + 1 < k) ? lp->prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
            f.start = sg.start + s0;
            f.len = s1 - s0;
            f.origin = sg.origin;
            f.key = sg.key;
        }
        return f;
    }
};

// User segments U*u .. U*u+U-1 (segmented mode at level 0, or the root).
struct SegLeaves {
    const uint64_t* off;
    uint64_t nsegs, seed;
    uint32_t U;
    uint32_t shard;     // RunParams::shard: key K(seed, 0), origin -base
    uint64_t base;
    __device__ __forceinline__ uint64_t units() const { return (nsegs + U - 1) / U; }
    __device__ __forceinline__ Leaf get(uint64_t u, uint32_t lane) const {
        Leaf f{0, 0, 0, 0};
        const uint64_t s = u * U + lane;
        if (lane < U && s < nsegs) {
            f.start = off[s];
            const uint64_t e = off[s + 1];
            f.len = e > f.start ? e - f.start : 0;
            f.origin = shard ? 0ull - base : f.start;
            f.key = shard ? seed : seed + s * 0x9E3779B97F4A7C15ull;  // K(seed, s) (D2)
        }
        return f;
    }
};

// Leaf `lane` of unit u of the recorded fused items: children 32g .. 32g+31
// of item r, u = r * ceil(k/32) + g (records: shuf_internal.cuh).
struct ItemLeaves {
    const unsigned char* items;
    const uint64_t* nitems;
    uint32_t k, groups, stride;
    __device__ __forceinline__ uint64_t units() const { return *nitems * groups; }
    __device__ __forceinline__ Leaf get(uint64_t u, uint32_t lane) const {
        Leaf f{0, 0, 0, 0};
        const uint64_t r = u / groups;
        const uint32_t b = (uint32_t)(u % groups) * 32u + lane;
        if (b < k) {
            const unsigned char* rec = items + r * stride;
            const uint16_t* o = reinterpret_cast<const uint16_t*>(rec + 24);
            const uint32_t s0 = o[b], s1 = o[b + 1];
            f.start = reinterpret_cast<const uint64_t*>(rec)[0] + s0;
            f.len = s1 - s0;
            f.origin = reinterpret_cast<const uint64_t*>(rec)[1];
            f.key = reinterpret_cast<const uint64_t*>(rec)[2];
        }
        return f;
    }
};

// Leaf `lane` of unit u of an in-place level batch: children 32g .. 32g+31 of
// batch segment s (bucket starts from the batch table S), in place.
struct IpChildLeaves {
    const IpParams* ip;
    uint32_t k, groups;
    uint64_t seed;
    __device__ __forceinline__ uint64_t units() const { return (uint64_t)ip->nseg * groups; }
    __device__ __forceinline__ Leaf get(uint64_t u, uint32_t lane) const {
        Leaf f{0, 0, 0, 0};
        const uint32_t s = (uint32_t)(u / groups), b = (uint32_t)(u % groups) * 32u + lane;
        if (b < k) {
            const uint64_t* S = ip->S + (uint64_t)s * (k + 1);
            const uint64_t s0 = S[b], s1 = S[b + 1];
            f.start = ip->segs[s].start + s0;
            f.len = s1 - s0;
            f.origin = 0;
            f.key = seed;
        }
        return f;
    }
};

// Leaf `lane` of unit u of an IpSc batch (kernels_ipsc.cu): children
// 32g .. 32g+31 of batch segment s, final bucket starts S[s * (k+1) + b].
struct IpscLeaves {
    const uint64_t* S;
    uint32_t nseg, k, groups;
    uint64_t seed;
    __device__ __forceinline__ uint64_t units() const { return (uint64_t)nseg * groups; }
    __device__ __forceinline__ Leaf get(uint64_t u, uint32_t lane) const {
        Leaf f{0, 0, 0, 0};
        const uint32_t s = (uint32_t)(u / groups), b = (uint32_t)(u % groups) * 32u + lane;
        if (b < k) {
            const uint64_t* T = S + (uint64_t)s * (k + 1) + b;
            f.start = T[0];
            f.len = T[1] - T[0];
            f.origin = 0;
            f.key = seed;  // K(seed, 0) (D2); positions are problem-relative
        }
        return f;
    }
};

template <int EB, class Src>
__device__ __forceinline__ void run_leaves(const RunParams& rp, const unsigned char* src, const Src& ls,
                                           uint32_t slot_bytes, uint32_t len_lo = 0u, uint32_t len_hi = 0xFFFFFFFFu,
                                           unsigned long long* ticket = nullptr) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned char* slot = lsm + warp * (slot_bytes + 16);
    uint64_t* bar = reinterpret_cast<uint64_t*>(slot + slot_bytes);
    if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;
    const uint64_t units = ls.units();
    const bool copy_out = src != rp.buf0;
    unsigned long long fyn = 0, fin = 0;
    const uint32_t nw = blockDim.x >> 5;  // leaf_warps()
    // warp-units by a fixed stride, or (ticket != nullptr) the next one from a global counter:
    // with leaves of very different lengths the stride leaves some warps far behind
    unsigned long long tk = 0;
    if (ticket && lane == 0) tk = atomicAdd(ticket, 1ull);
    uint64_t u = ticket ? __shfl_sync(0xFFFFFFFFu, tk, 0) : (uint64_t)blockIdx.x * nw + warp;
    for (; u < units;) {
        if (ticket && lane == 0) tk = atomicAdd(ticket, 1ull);  // the next unit's ticket, in flight during this unit
        const uint64_t ustep = (uint64_t)gridDim.x * nw;
        const Leaf lf = ls.get(u, lane);
        const uint64_t start = lf.start, len = lf.len, origin = lf.origin, key = lf.key;
        const bool pass = len > len_lo && len <= len_hi;  // this launch's length class
        const bool fy = len >= 2 && len <= rp.L && rp.run_leaves && pass;
        const bool mine = len >= 1 && len <= rp.L && (fy || copy_out) && pass;
        if (mine) fin += len;
        // long leaves (fewer than 8 fit the slot) run one at a time with the
        // whole warp (fy_leaf_warp); the others one thread per leaf
        const uint32_t need = mine ? (((uint32_t)len * EB + 32 + 15) & ~15u) : 0u;
        const bool big = fy && need * 8u > slot_bytes;
        uint32_t todo = __ballot_sync(0xFFFFFFFFu, mine && !big);
        uint32_t todo_big = __ballot_sync(0xFFFFFFFFu, big);
        while (todo | todo_big) {
            uint32_t off = 0;  // my slot offset if I am in the batch
            bool inb = false;
            const bool coop = todo == 0;  // this batch: one long leaf, the whole warp
            if (!coop) {
                // the batch: the longest run of pending short leaves (in lane order) that fits
                const uint32_t first = __ffs(todo) - 1;
                const uint32_t pend = (todo >> lane) & 1u;
                const uint32_t v = pend && lane >= first ? need : 0u;
                const uint32_t incl = warp_inclusive_sum(v);
                inb = pend && lane >= first && incl <= slot_bytes;
                off = incl - v;
                todo &= ~__ballot_sync(0xFFFFFFFFu, inb);
            } else {
                const uint32_t L0 = __ffs(todo_big) - 1;
                inb = lane == L0;
                todo_big &= ~(1u << L0);
            }
            // ---- load: aligned body by one bulk copy per leaf, ends by 4-byte copies
            uint64_t x0 = 0, x1 = 0, A = 0, B = 0;
            uint32_t body = 0;
            if (inb) {
                x0 = start * EB;
                x1 = (start + len) * EB;
                A = (x0 + 15) & ~15ull;
                B = x1 & ~15ull;
                body = B > A ? (uint32_t)(B - A) : 0u;
            }
            uint32_t tot = body;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
            unsigned char* lb = slot + off;  // leaf buffer: element e at lb + (x0 & 15) + e*EB
            if (lane == 0) mbar_arrive_expect_tx(bar, tot);
            __syncwarp();
            if (inb) {
                if (body) {
                    fence_proxy_async();
                    bulk_g2s(lb + (A - (x0 & ~15ull)), src + A, body, bar);
                }
                const uint64_t hEnd = body ? A : x1, tBeg = body ? B : x1;
                for (uint64_t x = x0; x < hEnd; x += 4)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(lb + (x - (x0 & ~15ull)))),
                                 "l"(src + x)
                                 : "memory");
                for (uint64_t x = tBeg; x < x1; x += 4)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(lb + (x - (x0 & ~15ull)))),
                                 "l"(src + x)
                                 : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            mbar_wait(bar, phase);
            phase ^= 1u;
            // ---- Fisher-Yates of my leaf (D5 draws keyed by the leaf start)
            if (coop) {
                const uint32_t L0 = __ffs(__ballot_sync(0xFFFFFFFFu, inb)) - 1;
                const uint32_t m = (uint32_t)__shfl_sync(0xFFFFFFFFu, len, L0);
                const uint64_t q = __shfl_sync(0xFFFFFFFFu, start - origin, L0);
                const uint64_t K = __shfl_sync(0xFFFFFFFFu, key, L0);
                const uint32_t a0 = __shfl_sync(0xFFFFFFFFu, (uint32_t)(x0 & 15u), L0);
                uint16_t* P = reinterpret_cast<uint16_t*>(slot + ((m * EB + 32 + 15) & ~15u));
                unsigned char* M = reinterpret_cast<unsigned char*>(P) + ((2 * m + 15) & ~15u);
                fy_leaf_warp<EB>(slot + a0, P, M, m, q, make_key(K));
                if (inb) fyn += len;
            } else if (inb && fy) {
                fy_leaf<EB>(lb + (x0 & 15u), 0u, (uint32_t)len, start - origin, make_key(key));
                fyn += len;
            }
            // ---- store: aligned body by one bulk copy, ends by words; every lane
            //      that wrote the slot orders its writes before the bulk store
            fence_proxy_async();
            __syncwarp();
            if (inb) {
                if (body) {
                    bulk_s2g(rp.buf0 + A, lb + (A - (x0 & ~15ull)), body);
                    bulk_commit();
                }
                const uint64_t hEnd = body ? A : x1, tBeg = body ? B : x1;
                for (uint64_t x = x0; x < hEnd; x += 4)
                    *reinterpret_cast<uint32_t*>(rp.buf0 + x) =
                        *reinterpret_cast<const uint32_t*>(lb + (x - (x0 & ~15ull)));
                for (uint64_t x = tBeg; x < x1; x += 4)
                    *reinterpret_cast<uint32_t*>(rp.buf0 + x) =
                        *reinterpret_cast<const uint32_t*>(lb + (x - (x0 & ~15ull)));
                bulk_wait_read0();  // the slot is read out before the next batch reuses it
            }
            __syncwarp();
        }
        u = ticket ? __shfl_sync(0xFFFFFFFFu, tk, 0) : u + ustep;
    }
    for (int o = 16; o > 0; o >>= 1) {
        fyn += __shfl_xor_sync(0xFFFFFFFFu, fyn, o);
        fin += __shfl_xor_sync(0xFFFFFFFFu, fin, o);
    }
    if (lane == 0) {
        if (fyn) atomicAdd((unsigned long long*)&rp.hdr->fy_elems, fyn);
        if (fin) atomicAdd((unsigned long long*)&rp.hdr->leafed, fin);
    }
    bulk_wait0();
}

template <int EB>
__global__ void __launch_bounds__(kLeafThreads) k_leaf_children(RunParams rp, LevelParams lp) {
    const uint32_t U = lp.leaf_unit;
    const ChildLeaves ls{&lp, rp.k, (rp.k + U - 1) / U, U};
    const uint32_t hi = lp.leaf_hi ? lp.leaf_hi : rp.L;
    run_leaves<EB>(rp, lp.dst, ls, leaf_slot_bytes(EB, hi), lp.leaf_lo, hi);
}

template <int EB>
__global__ void __launch_bounds__(kLeafThreads) k_leaf_segments(RunParams rp, const uint64_t* __restrict__ off,
                                                                 uint64_t nsegs, uint32_t U, uint32_t lo, uint32_t hi,
                                                                 unsigned long long* ticket) {
    const SegLeaves ls{off, nsegs, rp.seed, U, rp.shard, rp.seg_base};
    run_leaves<EB>(rp, rp.buf0, ls, leaf_slot_bytes(EB, hi), lo, hi, ticket);  // segments with lo < length <= hi
}

template <int EB>
__global__ void __launch_bounds__(kLeafThreads) k_leaf_items(RunParams rp) {
    const ItemLeaves ls{rp.items, &rp.hdr->nitems, rp.k, (rp.k + 31) / 32, item_rec_stride(rp.k)};
    run_leaves<EB>(rp, rp.buf0, ls, leaf_slot_bytes(EB, rp.L));
}

template <int EB>
__global__ void __launch_bounds__(kLeafThreads) k_leaf_ipchildren(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    const IpChildLeaves ls{&ip, rp.k, (rp.k + 31) / 32, rp.seed};
    run_leaves<EB>(rp, rp.buf0, ls, leaf_slot_bytes(EB, rp.L));
}

template <int EB>
__global__ void __launch_bounds__(kLeafThreads) k_leaf_ipsc(RunParams rp, const uint64_t* __restrict__ S, uint32_t nseg) {
    const IpscLeaves ls{S, nseg, rp.k, (rp.k + 31) / 32, rp.seed};
    run_leaves<EB>(rp, rp.buf0, ls, leaf_slot_bytes(EB, rp.L));
}

// mode: 0 children, 1 segments, 2 items, 3 in-place children, 4 IpSc children
static void* leaf_fn(uint32_t eb, int mode) {
    if (mode == 4) return eb == 4 ? (void*)k_leaf_ipsc<4> : eb == 8 ? (void*)k_leaf_ipsc<8> : (void*)k_leaf_ipsc<16>;
    if (mode == 3) return eb == 4 ? (void*)k_leaf_ipchildren<4> : eb == 8 ? (void*)k_leaf_ipchildren<8>
                                                                        : (void*)k_leaf_ipchildren<16>;
    switch (eb) {
    case 4: return mode == 1 ? (void*)k_leaf_segments<4> : mode == 2 ? (void*)k_leaf_items<4> : (void*)k_leaf_children<4>;
    case 8: return mode == 1 ? (void*)k_leaf_segments<8> : mode == 2 ? (void*)k_leaf_items<8> : (void*)k_leaf_children<8>;
    default:
        return mode == 1 ? (void*)k_leaf_segments<16> : mode == 2 ? (void*)k_leaf_items<16> : (void*)k_leaf_children<16>;
    }
}

cudaError_t configure_leaf(uint32_t eb, uint32_t L) {
    (void)L;  // the attribute is the limit: plans of other sizes share the kernels
    for (int mode = 0; mode < 5; ++mode) {
        cudaError_t e = cudaFuncSetAttribute(leaf_fn(eb, mode), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
        if (e) return e;
    }
    return cudaSuccess;
}

cudaError_t occupancy_leaf(uint32_t eb, uint32_t L, int* blocks) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, leaf_fn(eb, 0), 32 * leaf_warps(eb, L),
                                                         leaf_smem_bytes(eb, L));
}

cudaError_t launch_leaf_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp, (void*)&lp};
    const uint32_t hi = lp.leaf_hi ? lp.leaf_hi : rp.L;  // the slots hold leaves of hi elements
    return cudaLaunchKernel(leaf_fn(rp.eb, 0), dim3(grid), dim3(32 * leaf_warps(rp.eb, hi)), args,
                            leaf_smem_bytes(rp.eb, hi), s);
}

cudaError_t launch_leaf_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                 cudaStream_t s, int grid, uint32_t lo, uint32_t hi, unsigned long long* ticket) {
    if (hi == 0) hi = rp.L;  // the slots hold segments of hi elements
    uint64_t avg = num_segments ? rp.n / num_segments : 0;
    if (avg > hi) avg = hi;
    uint32_t U = leaf_unit(rp.eb, hi, avg);
    void* args[] = {(void*)&rp, (void*)&d_offsets, (void*)&num_segments, (void*)&U, (void*)&lo, (void*)&hi,
                    (void*)&ticket};
    return cudaLaunchKernel(leaf_fn(rp.eb, 1), dim3(grid), dim3(32 * leaf_warps(rp.eb, hi)), args,
                            leaf_smem_bytes(rp.eb, hi), s);
}

cudaError_t launch_leaf_items(const RunParams& rp, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp};
    return cudaLaunchKernel(leaf_fn(rp.eb, 2), dim3(grid), dim3(32 * leaf_warps(rp.eb, rp.L)), args, leaf_smem_bytes(rp.eb, rp.L), s);
}

cudaError_t launch_leaf_ipsc(const RunParams& rp, const uint64_t* S, uint32_t nseg, cudaStream_t s, int grid) {
    if (nseg == 0) return cudaSuccess;
    void* args[] = {(void*)&rp, (void*)&S, (void*)&nseg};
    return cudaLaunchKernel(leaf_fn(rp.eb, 4), dim3(grid), dim3(32 * leaf_warps(rp.eb, rp.L)), args, leaf_smem_bytes(rp.eb, rp.L), s);
}

cudaError_t launch_leaf_ipchildren(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp, (void*)&ip};
    return cudaLaunchKernel(leaf_fn(rp.eb, 3), dim3(grid), dim3(32 * leaf_warps(rp.eb, rp.L)), args, leaf_smem_bytes(rp.eb, rp.L), s);
}

}  // namespace shuf
