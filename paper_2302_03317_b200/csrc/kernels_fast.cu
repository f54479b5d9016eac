// Fast fused finish for the common shape of the recursion (SURVEY 8(a) a7+a8):
// a child of the last HBM level ("item") that needs exactly ONE more scatter
// level, after which every grandchild is a leaf (<= L) -- e.g. the HOT run's
// 65 536 children of ~16 K u32 that split into ~64-element leaves.
//
// One CTA of 1024 threads per SM, warp-specialised and software-pipelined
// over the CTA's items.  Two item buffers in shared memory:
// IN (the item as loaded by one bulk async copy, TMA engine) and LV (the item
// grouped into its leaves).  Per item i, three phases separated by CTA
// barriers:
//   A  rank warps (8..31): the level's bucket draws of item i (D4, Philox)
//        -> shared memory, and per-warp bucket counts.
//      FY warps (0..7): Fisher-Yates (Fig. 1) of every leaf of
//        item i-1 in place in LV -- one thread per leaf, partners
//        precomputed -- then one bulk async store of LV to ptr.
//   B  rank warps: scan of the counts -> bucket (leaf) starts and per-warp
//        bases.  FY warps: wait until LV has been read out.
//   C  all warps: stable placement IN -> LV (warp w walks its elements in
//        rounds of 32 in position order; one ordered shared atomic on its
//        own table gives each element its slot, D6), then the Fisher-Yates
//        partners of item i's leaves (D5) -> jb.  The load of item i+1 into
//        IN is issued at the start of the next phase A.
// Items of another shape (a grandchild > L or > 256 elements, a leaf-only
// child, more than SMAX elements) are flagged and finished by the general
// kernel (kernels_finish.cu) right after.
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char xsm[];

constexpr int XNT = 1024;           // threads per CTA
constexpr uint32_t XFYT = 256;      // Fisher-Yates threads (warps 0..7)
constexpr uint32_t XRW = 24;        // rank warps (8..31): draws, counts, scan
constexpr uint32_t XRT = XRW * 32;  // 768 rank threads
constexpr uint32_t XPW = XNT / 32;  // placing warps: all 32 (per-warp rank tables)
constexpr uint32_t XBYTES = 73728;  // item buffer (72 KiB)

template <int EB>
struct XCfg {
    static constexpr uint32_t SMAX = XBYTES / EB;  // largest item of the fast path
};

uint32_t fast_max_elems(uint32_t eb) { return XBYTES / eb; }

struct XItem {
    uint64_t start, origin, key;
    uint64_t child;  // child index c = s*k + b (for the deferral flag)
    uint32_t len, valid;
};

struct XCtl {
    XItem cur, nxt, fy;
    uint64_t bar;     // mbarrier of the IN load
    uint32_t cursor;  // this CTA's next candidate child index
    uint32_t defer;   // cur is handed to the general kernel
    uint32_t phase;   // parity of the IN mbarrier
    uint32_t dbg_it;  // items processed (phase clocks of the first ones, CTA 0)
    unsigned long long st_fin, st_fy;
};

struct XLayout {
    uint32_t in, lv, draws, jb, T, bst, wsum, total;
};

__host__ __device__ inline XLayout fast_layout(uint32_t eb, uint32_t k) {
    XLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    const uint32_t smax = XBYTES / eb;
    const bool narrow = (k & (k - 1)) == 0 && k <= 256;
    take(sizeof(XCtl));
    f.in = take(XBYTES + 32);
    f.lv = take(XBYTES + 32);
    f.draws = take((narrow ? 1u : 2u) * smax + 64);
    f.jb = take(smax + 4 * k + 16);  // Fisher-Yates partners (u8) of the item awaiting FY
    f.T = take(XPW * ((k + 1) / 2) * 4);
    f.bst = take((k + 1) * 4);
    f.wsum = take((XNT / 32 + 1) * 4);
    f.total = off;
    return f;
}

uint32_t fast_smem_bytes(uint32_t eb, uint32_t k) { return fast_layout(eb, k).total; }

__device__ __forceinline__ void bar_named(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Barriers: 0 = whole CTA, 1 = FY warps (256), 2 = rank warps (768).
__device__ __forceinline__ void bar_cta() { bar_named(0, XNT); }
__device__ __forceinline__ void bar_fy() { bar_named(1, XFYT); }
__device__ __forceinline__ void bar_rank() { bar_named(2, XRT); }

// 4-byte asynchronous global -> shared copy (the unaligned head/tail words of
// an item; completion by cp.async.wait_all).
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Element ranges of the placing warps.  The item's positions [P0, P0+m)
// cover ng Philox groups of dpg draws; warp w owns groups [w*qg, (w+1)*qg),
// i.e. elements e in [w*qg*dpg - doff, (w+1)*qg*dpg - doff) clipped to
// [0, m).  Rank warp rw generates and counts the groups of placing warps
// rw and rw + 24.
template <bool NARROW>
struct XRange {
    static constexpr uint32_t sh = NARROW ? 4u : 3u, dpg = 1u << sh;
    uint32_t m, doff, ng, qg;
    uint64_t g0;
    __device__ __forceinline__ XRange(uint64_t P0, uint32_t len) {
        m = len;
        g0 = P0 >> sh;
        doff = (uint32_t)(P0 & (dpg - 1));
        ng = (uint32_t)(((P0 + m - 1) >> sh) - g0 + 1);
        qg = (ng + XPW - 1) / XPW;
    }
    __device__ __forceinline__ int32_t ebase(uint32_t w) const { return (int32_t)(w * qg * dpg) - (int32_t)doff; }
    __device__ __forceinline__ int32_t eend(uint32_t w) const {
        const int32_t x = (int32_t)((w + 1) * qg * dpg) - (int32_t)doff;
        return x < (int32_t)m ? x : (int32_t)m;
    }
};

// Child c = s*k + b of the level's segments: [start, start+len).
// (c < 2^32: nseg * k <= max_segs * k is bounded by the scratch layout.)
__device__ __forceinline__ void child_of(const LevelParams& lp, uint32_t k, uint32_t c, uint64_t& start, uint64_t& len,
                                         SegDesc& sg) {
    sg = lp.segs[c / k];
    const uint32_t b = c % k;
    const uint64_t base0 = lp.prefix[sg.cbase];
    const uint64_t s0 = lp.prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
    const uint64_t s1 = (b + 1 < k) ? lp.prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
    start = sg.start + s0;
    len = s1 - s0;
}

// Next child of this CTA's stride sequence that the fast path takes; flags
// every child of at most S_fuse elements on the way (1: general kernel).
template <int EB>
__device__ __forceinline__ XItem find_next(const RunParams& rp, const LevelParams& lp, uint32_t nchild,
                                           uint32_t& cursor) {
    XItem it;
    it.valid = 0;
    const uint32_t lvl = lp.level + 1;
    for (uint32_t c = cursor; c < nchild; c += gridDim.x) {
        uint64_t start, len;
        SegDesc sg;
        child_of(lp, rp.k, c, start, len, sg);
        if (len == 0 || len > rp.S_fuse) continue;  // empty, or an HBM segment of the next level
        const bool leaf = len <= rp.L;
        const bool permutes = (!leaf && lvl < rp.max_levels) || (leaf && rp.run_leaves && len >= 2);
        if (!permutes) {  // nothing to do unless it must be copied to ptr
            rp.flags[c] = (lp.dst == rp.buf0) ? 0 : 1;
            continue;
        }
        if (leaf || len > XCfg<EB>::SMAX || lvl + 1 > rp.max_levels || !rp.run_leaves) {
            rp.flags[c] = 1;
            continue;
        }
        rp.flags[c] = 0;
        it.start = start;
        it.origin = sg.origin;
        it.key = sg.key;
        it.len = (uint32_t)len;
        it.child = c;
        it.valid = 1;
        cursor = c + gridDim.x;
        return it;
    }
    cursor = 0xFFFFFFFFu;
    return it;
}

// Shared-memory views (byte offsets into the dynamic window).
template <int EB>
struct XView {
    XLayout Ly;
    __device__ __forceinline__ explicit XView(uint32_t k) { Ly = fast_layout(EB, k); }
    __device__ __forceinline__ XCtl* ctl() const { return reinterpret_cast<XCtl*>(xsm); }
    __device__ __forceinline__ unsigned char* in() const { return xsm + Ly.in; }
    __device__ __forceinline__ unsigned char* lv() const { return xsm + Ly.lv; }
    __device__ __forceinline__ unsigned char* draws() const { return xsm + Ly.draws; }
    __device__ __forceinline__ unsigned char* jb() const { return xsm + Ly.jb; }
    __device__ __forceinline__ uint32_t* T() const { return reinterpret_cast<uint32_t*>(xsm + Ly.T); }
    __device__ __forceinline__ uint32_t* bst() const { return reinterpret_cast<uint32_t*>(xsm + Ly.bst); }
    __device__ __forceinline__ uint32_t* wsum() const { return reinterpret_cast<uint32_t*>(xsm + Ly.wsum); }
};

// Element e of an item lives at byte ((start*EB) & 15) + e*EB of IN / LV, so
// its 16-byte-aligned body maps to a 16-byte-aligned shared address.
template <int EB>
__device__ __forceinline__ unsigned char* item_base(unsigned char* buf, uint64_t start) {
    return buf + ((start * EB) & 15u);
}

// Leaf b's partner slot in jb: 4-aligned and disjoint from its neighbours'.
__device__ __forceinline__ uint32_t jslot(uint32_t s0, uint32_t b) { return (s0 + 3u + 4u * b) & ~3u; }

// Start of phase A (thread 0 and rank threads 0..7): the load of item `it`
// into IN: the aligned body by one bulk async copy, the <= 3 unaligned words
// at each end by 4-byte asynchronous copies.
template <int EB>
__device__ __forceinline__ void issue_in_load(const XView<EB>& V, const XItem& it, const unsigned char* src) {
    const uint32_t tid = threadIdx.x;
    const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    unsigned char* buf = V.in();
    XCtl* ctl = V.ctl();
    if (tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&ctl->bar, body ? (uint32_t)(B - A) : 0u);
        if (body) bulk_g2s(buf + (A - fl), src + A, (uint32_t)(B - A), &ctl->bar);
        return;
    }
    const uint64_t hEnd = body ? A : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
    const uint64_t tBeg = body ? B : x1;
    const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
    const uint32_t rt = tid - XFYT;  // 0..7
    if (rt < 4) {
        if (rt < nh) cp_async4(buf + (x0 - fl) + 4 * rt, src + x0 + 4 * rt);
    } else if (rt - 4 < nt) {
        cp_async4(buf + (tBeg - fl) + 4 * (rt - 4), src + tBeg + 4 * (rt - 4));
    }
}

// ---------------------------------------------------------------- FY ---
// Phase C tail (all warps): partners j_i, i = 1 .. mb-1 of every leaf of the
// item just placed (D5: leaf id = problem position of the leaf start, one
// Philox block per 8 steps, Lemire16), packed 4 per word.  Thread t takes
// leaf t % k and every (1024/k)-th group of it.
template <int EB>
__device__ __forceinline__ void partner_phase(const RunParams& rp, const XView<EB>& V) {
    XCtl* ctl = V.ctl();
    const uint32_t k = rp.k, tid = threadIdx.x;
    const uint64_t P0 = ctl->cur.start - ctl->cur.origin;
    const PhiloxKey key = make_key(ctl->cur.key);
    const uint32_t per = XNT / k >= 2 ? XNT / k : 1;  // threads per leaf
    if (per > 1 && tid >= per * k) return;
    const uint32_t sub = per > 1 ? tid / k : 0;
    const uint32_t bstep = per > 1 ? k : XNT;
    for (uint32_t b = per > 1 ? tid % k : tid; b < k; b += bstep) {
        const uint32_t s0 = V.bst()[b], mb = V.bst()[b + 1] - s0;
        if (mb < 2) continue;
        const uint64_t qq = P0 + s0;
        uint32_t* jw = reinterpret_cast<uint32_t*>(V.jb() + jslot(s0, b));
        const uint32_t ngr = ((mb - 1) >> 3) + 1;
        for (uint32_t g = sub; g < ngr; g += per) {
            const uint4 w4 = fy16_group_words(key, qq, g);
            const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
            uint32_t pk[2] = {0u, 0u};
#pragma unroll
            for (uint32_t jj = 0; jj < 8; ++jj) {
                const uint32_t i = g * 8u + jj;
                const uint32_t vv = (wv[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu;
                const uint32_t sb = i + 1, mm = vv * sb;
                uint32_t j = mm >> 16;
                if (__builtin_expect((mm & 0xFFFFu) < sb, 0) && i >= 1 && i < mb) j = fy16_from_lane(vv, key, qq, i);
                pk[jj >> 2] |= (j & 0xFFu) << ((jj & 3u) * 8u);
            }
            jw[2 * g] = pk[0];
            jw[2 * g + 1] = pk[1];
        }
    }
}

// Phase A (FY warps): Fisher-Yates of every leaf of the previous item, in
// place in LV, then its bulk store.
template <int EB>
__device__ __forceinline__ void fy_phase(const RunParams& rp, const XView<EB>& V) {
    using E = typename ElemT<EB>::type;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, k = rp.k;
    XCtl* ctl = V.ctl();
    const uint64_t fstart = ctl->fy.start;
    E* lv0 = reinterpret_cast<E*>(item_base<EB>(V.lv(), fstart));
    uint32_t fyn = 0;
    for (uint32_t b = tid; b < k; b += XFYT) {
        const uint32_t s0 = V.bst()[b], mb = V.bst()[b + 1] - s0;
        if (mb < 2) continue;
        fyn += mb;
        E* A = lv0 + s0;
        // Fig. 1: for i = mb-1 .. 1 swap(A[i], A[j_i]).  The loads of step
        // i-1 are issued before the stores of step i and patched when step i
        // wrote the same place (j_i == i-1, or j_{i-1} == j_i); A[i] is never
        // read again after step i.
        const uint32_t* jw = reinterpret_cast<const uint32_t*>(V.jb() + jslot(s0, b));
        uint32_t i = mb - 1;
        uint32_t jc = (jw[i >> 2] >> ((i & 3u) * 8u)) & 0xFFu;
        E x = A[i], y = A[jc];
        for (; i >= 2; --i) {
            const uint32_t jn = (jw[(i - 1) >> 2] >> (((i - 1) & 3u) * 8u)) & 0xFFu;
            E xn = A[i - 1];
            E yn = A[jn];
            A[jc] = x;
            A[i] = y;
            if (jc == i - 1) xn = x;
            if (jn == jc) yn = x;
            x = xn;
            y = yn;
            jc = jn;
        }
        A[jc] = x;  // step 1
        A[1] = y;
    }
    for (int o = 16; o > 0; o >>= 1) fyn += __shfl_xor_sync(0xFFFFFFFFu, fyn, o);
    if (lane == 0 && fyn) atomicAdd(&ctl->st_fy, (unsigned long long)fyn);
    bar_fy();
    // LV holds the finished item: bulk store of the aligned body + head/tail words
    const uint64_t x0 = fstart * EB, x1 = (fstart + ctl->fy.len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A0 = (x0 + 15) & ~15ull, B0 = x1 & ~15ull;
    const bool body = B0 > A0;
    if (tid == 0 && body) {
        fence_proxy_async();
        bulk_s2g(rp.buf0 + A0, V.lv() + (A0 - fl), (uint32_t)(B0 - A0));
        bulk_commit();
    }
    const uint64_t hEnd = body ? A0 : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
    const uint64_t tBeg = body ? B0 : x1;
    const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
    if (tid >= 32 && tid - 32 < nh)
        *reinterpret_cast<uint32_t*>(rp.buf0 + x0 + 4 * (tid - 32)) =
            *reinterpret_cast<const uint32_t*>(V.lv() + (x0 - fl) + 4 * (tid - 32));
    else if (tid >= 64 && tid - 64 < nt)
        *reinterpret_cast<uint32_t*>(rp.buf0 + tBeg + 4 * (tid - 64)) =
            *reinterpret_cast<const uint32_t*>(V.lv() + (tBeg - fl) + 4 * (tid - 64));
}

// -------------------------------------------------------------- rank ---
// Phase A (rank warps): draws of item i -> smem (indexed by group) and the
// per-placing-warp bucket counts (rank warp rw does placing warps rw, rw+24).
template <int EB, bool NARROW>
__device__ __forceinline__ void draw_count_phase(const RunParams& rp, const XView<EB>& V, uint32_t lvl) {
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t rt = threadIdx.x - XFYT, lane = rt & 31u, rw = rt >> 5;
    XCtl* ctl = V.ctl();
    const BucketParams bp = rp.bp;
    const uint64_t P0 = ctl->cur.start - ctl->cur.origin;
    const XRange<NARROW> xr(P0, ctl->cur.len);
    const uint32_t m = xr.m;
    const PhiloxKey key = make_key(ctl->cur.key);
    constexpr uint32_t sh = XRange<NARROW>::sh, dpg = XRange<NARROW>::dpg;
    for (uint32_t pw = rw; pw < XPW; pw += XRW) {
        uint32_t* Tw = V.T() + pw * kw;
        for (uint32_t i = lane; i < kw; i += 32) Tw[i] = 0;
        __syncwarp();
        const uint32_t t1 = min(xr.ng, (pw + 1) * xr.qg);
        for (uint32_t t = pw * xr.qg + lane; t < t1; t += 32) {
            const uint64_t g = xr.g0 + t;
            const uint4 w4 = bucket_group_words(key, lvl, g);
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
                    const bool in = pb + j >= P0 && pb + j < P0 + m;
                    bb[j] = in ? bucket_from_group(w4, j, key, lvl, pb + j, bp) : 0u;
                }
                packed = make_uint4(bb[0] | (bb[1] << 16), bb[2] | (bb[3] << 16), bb[4] | (bb[5] << 16),
                                    bb[6] | (bb[7] << 16));
            }
            *reinterpret_cast<uint4*>(V.draws() + (size_t)t * 16) = packed;
            const int32_t e0 = (int32_t)(t * dpg) - (int32_t)xr.doff;
            const uint32_t pw4[4] = {packed.x, packed.y, packed.z, packed.w};
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const int32_t e = e0 + (int32_t)j;
                const uint32_t b =
                    NARROW ? (pw4[j >> 2] >> ((j & 3u) * 8u)) & 0xFFu : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                if (e >= 0 && e < (int32_t)m) atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
            }
        }
    }
}

// Exclusive sum over the 768 rank threads (rt = rank thread index).
__device__ __forceinline__ uint32_t rank_exclusive_sum(uint32_t v, uint32_t rt, uint32_t* wsum) {
    constexpr uint32_t NW = XRW;
    const uint32_t lane = rt & 31u, w = rt >> 5;
    const uint32_t incl = warp_inclusive_sum(v);
    if (lane == 31) wsum[w] = incl;
    bar_rank();
    if (w == 0) {
        const uint32_t x = lane < NW ? wsum[lane] : 0u;
        const uint32_t xi = warp_inclusive_sum(x);
        if (lane < NW) wsum[lane] = xi - x;
    }
    bar_rank();
    return wsum[w] + incl - v;
}

// Phase B (rank warps): bucket starts and per-warp slot bases; flags the
// item for the general kernel if a leaf is too long for this kernel.
template <int EB>
__device__ __forceinline__ void scan_phase(const RunParams& rp, const XView<EB>& V) {
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t rt = threadIdx.x - XFYT;
    XCtl* ctl = V.ctl();
    uint32_t* T = V.T();
    const uint32_t b0 = 2 * rt;  // rank thread rt owns buckets 2rt, 2rt+1
    uint32_t c0 = 0, c1 = 0;
    if (b0 < k) {
#pragma unroll 4
        for (uint32_t w = 0; w < XPW; ++w) {
            const uint32_t c = T[w * kw + rt];
            c0 += c & 0xFFFFu;
            c1 += c >> 16;
        }
        if (b0 + 1 >= k) c1 = 0;
    }
    const uint32_t lim = rp.L < 256u ? rp.L : 256u;  // leaves <= L, partners fit u8
    if (c0 > lim || c1 > lim) atomicOr(&ctl->defer, 1u);
    const uint32_t ex = rank_exclusive_sum(c0 + c1, rt, V.wsum());  // (its barriers publish defer)
    const bool big = ctl->defer != 0;
    if (b0 < k) {
        V.bst()[b0] = ex;
        if (b0 + 1 < k) V.bst()[b0 + 1] = ex + c0;
    }
    if (rt == 0) V.bst()[k] = ctl->cur.len;
    if (!big) {
        if (b0 < k) {
            // per-warp slot bases: T[w][b] = bst[b] + sum_{w'<w} cnt[w'][b]
            uint32_t r0 = ex, r1 = ex + c0;
#pragma unroll 4
            for (uint32_t w = 0; w < XPW; ++w) {
                const uint32_t c = T[w * kw + rt];
                T[w * kw + rt] = (r0 & 0xFFFFu) | (r1 << 16);
                r0 += c & 0xFFFFu;
                r1 += c >> 16;
            }
        }
    } else if (rt == 0) {
        rp.flags[ctl->cur.child] = 1;  // hand the item to the general kernel
    }
}

// Phase C (all warps): stable placement IN -> LV.  Warp w walks its elements
// in rounds of 32 in position order; the ordered shared atomic on its own
// table returns each element's slot (bucket start + rank, D6 stable).
template <int EB, bool NARROW>
__device__ __forceinline__ void place_phase(const XView<EB>& V, uint32_t kw) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    XCtl* ctl = V.ctl();
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint64_t start = ctl->cur.start;
    const XRange<NARROW> xr(start - ctl->cur.origin, ctl->cur.len);
    const int32_t eb0 = xr.ebase(w), ee = xr.eend(w);
    const D* dp = reinterpret_cast<const D*>(V.draws()) + xr.doff;
    const E* in = reinterpret_cast<const E*>(item_base<EB>(V.in(), start));
    E* lv = reinterpret_cast<E*>(item_base<EB>(V.lv(), start));
    uint32_t* Tw = V.T() + w * kw;
#pragma unroll 4
    for (int32_t e0 = eb0; e0 < ee; e0 += 32) {
        const int32_t e = e0 + (int32_t)lane;
        const bool valid = e >= 0 && e < ee;
        const int32_t es = valid ? e : 0;
        const uint32_t b = valid ? (uint32_t)dp[es] : 0u;
        const E x = in[es];
        const uint32_t shb = (b & 1u) << 4;
        const uint32_t slot = (atomicAdd(&Tw[b >> 1], valid ? (1u << shb) : 0u) >> shb) & 0xFFFFu;
        if (valid) lv[slot] = x;
    }
}

// ------------------------------------------------------------- loops ---
template <int EB, bool NARROW>
__device__ __forceinline__ void run(const RunParams& rp, const LevelParams& lp, const XView<EB>& V, uint32_t nchild) {
    XCtl* ctl = V.ctl();
    const uint32_t kw = (rp.k + 1) >> 1, tid = threadIdx.x;
    const bool is_fy = tid < XFYT;
    const unsigned char* src = lp.dst;  // the level's output buffer holds the children
    const uint32_t lvl = lp.level + 1;
    for (;;) {
        if (!ctl->cur.valid && !ctl->fy.valid) break;
        const bool have = ctl->cur.valid != 0;
        const bool dbg = blockIdx.x == 0 && tid == XFYT && ctl->dbg_it < 40;
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 0] = clock64();
        // ---- phase A
        if (have && (tid == 0 || (tid >= XFYT && tid < XFYT + 8))) issue_in_load<EB>(V, ctl->cur, src);
        if (is_fy) {
            if (ctl->fy.valid) fy_phase<EB>(rp, V);
            if (blockIdx.x == 0 && tid == 0 && ctl->dbg_it < 40) rp.hdr->clk[ctl->dbg_it * 6 + 1] = clock64();
        } else {
            if (have) draw_count_phase<EB, NARROW>(rp, V, lvl);
            if (tid == XFYT) {  // the next item
                if (have) ctl->nxt = find_next<EB>(rp, lp, nchild, ctl->cursor);
                else ctl->nxt.valid = 0;
            }
            if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 2] = clock64();
        }
        bar_cta();
        // ---- phase B
        if (is_fy) {
            if (tid == 0) bulk_wait_read0();  // LV is read out before placement rewrites it
        } else if (have) {
            scan_phase<EB>(rp, V);
        }
        if (have && tid >= XFYT && tid < XFYT + 8) cp_async_wait_all();
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 3] = clock64();
        bar_cta();
        // ---- phase C
        const bool placed = have && ctl->defer == 0;
        if (have) mbar_wait(&ctl->bar, ctl->phase);  // IN has arrived
        if (placed) place_phase<EB, NARROW>(V, kw);
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 4] = clock64();
        if (placed) partner_phase<EB>(rp, V);
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 5] = clock64();
        bar_cta();
        if (tid == XFYT) {
            ctl->dbg_it++;
            if (have) ctl->phase ^= 1u;
            if (placed) ctl->st_fin += ctl->cur.len;
            ctl->fy = ctl->cur;
            if (!placed) ctl->fy.valid = 0;
            ctl->cur = ctl->nxt;
            ctl->defer = 0;
        }
        bar_cta();
    }
    if (tid == 0) bulk_wait0();
}

template <int EB, bool NARROW>
__global__ void __launch_bounds__(XNT, 1) k_finish_fast(RunParams rp, LevelParams lp) {
    const XView<EB> V(rp.k);
    XCtl* ctl = V.ctl();
    const uint32_t nchild = lp.ctr->nseg * rp.k;
    if (threadIdx.x == 0) {
        ctl->cursor = blockIdx.x;
        ctl->fy.valid = 0;
        ctl->defer = 0;
        ctl->phase = 0;
        ctl->dbg_it = 0;
        ctl->st_fin = 0;
        ctl->st_fy = 0;
        mbar_init(&ctl->bar, 1);
        fence_mbar_init();
        ctl->cur = find_next<EB>(rp, lp, nchild, ctl->cursor);
    }
    __syncthreads();
    run<EB, NARROW>(rp, lp, V, nchild);
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t lvl = lp.level + 1;
        atomicAdd((unsigned long long*)&rp.hdr->finished, ctl->st_fin);
        atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[lvl < kMaxLevels ? lvl : 0], ctl->st_fin);
        atomicAdd((unsigned long long*)&rp.hdr->fy_elems, ctl->st_fy);
    }
}

template <int EB>
static void* fast_fn(bool narrow) {
    return narrow ? (void*)k_finish_fast<EB, true> : (void*)k_finish_fast<EB, false>;
}
static void* fast_kernel(uint32_t eb, bool narrow) {
    switch (eb) {
    case 4: return fast_fn<4>(narrow);
    case 8: return fast_fn<8>(narrow);
    default: return fast_fn<16>(narrow);
    }
}

cudaError_t configure_fast(uint32_t eb, uint32_t k) {
    const uint32_t smem = fast_smem_bytes(eb, k);
    if (smem > kSmemLimit) return cudaErrorInvalidValue;
    for (int nr = 0; nr < 2; ++nr) {
        cudaError_t e = cudaFuncSetAttribute(fast_kernel(eb, nr != 0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem);
        if (e) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_finish_fast(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = fast_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(fast_kernel(rp.eb, rp.bp.narrow != 0), dim3(grid), dim3(XNT), args, smem, s);
}

}  // namespace shuf
