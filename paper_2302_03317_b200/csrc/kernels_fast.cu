// Pipelined fused finish for the common shape of the recursion (SURVEY 8(a)
// a7+a8): a child of the last HBM level ("item") that needs exactly ONE more
// scatter level, after which every grandchild is a leaf -- e.g. the HOT
// run's 65 536 children of ~16 K u32 that split into ~64-element leaves.
//
// The general finish (kernels_finish.cu) runs each item's phases back to
// back with the whole CTA: while one thread per leaf runs Fisher-Yates, three
// quarters of the CTA wait at a barrier.  Here the CTA is
// split into three warp groups that work on different items at once, with
// two item buffers and mbarrier hand-offs (no CTA-wide barrier in the loop):
//   S (warps 9..31, 736 threads): item t+1 -- draws (D4) + per-warp counts,
//       bucket starts and per-warp bases, then the stable in-place scatter
//       inside its buffer (every thread holds its elements in registers
//       across a group barrier; one ordered shared atomic per element
//       returns its slot);
//   F (warps 0..7, 256 threads): item t -- Fisher-Yates (Fig. 1)
//       of every leaf, one thread per leaf, in place (D5 draws);
//   C (warp 8): stores item t (bulk async copy, TMA engine) once F is done,
//       finds the next item and loads it into the freed buffer.
// Items of another shape (a grandchild > L, a leaf-only child, more than
// SMAX elements) are flagged and finished by the general kernel right after.
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char xsm[];

constexpr int XNT = 1024;
constexpr uint32_t XF = 256;             // F: threads 0..255
constexpr uint32_t XC = 256;             // C: warp 8 (threads 256..287)
constexpr uint32_t XS0 = 288;            // S: threads 288..1023
constexpr uint32_t XSN = XNT - XS0;      // 736
constexpr uint32_t XSW = XSN / 32;       // 23 warps
constexpr uint32_t XBUF = 71680;         // bytes per item buffer (70 KiB)
constexpr uint32_t XIN = XBUF - 16;      // largest item in bytes (alignment slack)
constexpr uint32_t kBarS = 1, kBarF = 2; // named barriers

template <int EB>
struct XCfg {
    static constexpr uint32_t SMAX = XIN / EB;                         // largest item
    static constexpr uint32_t R = (SMAX + 16 * XSW) / (32 * XSW) + 2;  // rounds per S warp
};

struct XItem {
    uint64_t start, origin, key;
    uint64_t child;  // child index c = s*k + b (for the deferral flag)
    uint32_t len, valid;
};

constexpr uint32_t XD = 4;  // descriptor ring: item t uses descriptor slot t % XD and buffer t % 2

struct XCtl {
    XItem item[XD];
    uint64_t desc[XD];                      // mbarrier per descriptor slot: published by C
    uint64_t full[2], ready[2], fydone[2];  // mbarriers per buffer
    uint32_t defer[XD];
    uint32_t cursor;
    uint32_t dbg_s, dbg_f;
    unsigned long long st_fin, st_fy;
};

struct XLayout {
    uint32_t buf0, buf1, draws, T, perm, bst0, bst1, wsum, total;
};

__host__ __device__ inline XLayout fast_layout(uint32_t eb, uint32_t k) {
    XLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    const uint32_t smax = XIN / eb;
    const bool narrow = (k & (k - 1)) == 0 && k <= 256;
    take(sizeof(XCtl));
    f.buf0 = take(XBUF);
    f.buf1 = take(XBUF);
    f.draws = take((narrow ? 1u : 2u) * (smax + 64));
    f.T = take(XSW * (narrow ? k : (k + 1) / 2) * 4);  // narrow: u32 counters, else packed u16
    f.perm = take(XD * k * 2);        // per descriptor slot: FY thread -> leaf
    f.bst0 = take(XD * (k + 1) * 4);  // per descriptor slot: bucket starts
    f.bst1 = f.bst0;
    f.wsum = take((XSW + 2 + 32) * 4);
    f.total = off;
    return f;
}

uint32_t fast_smem_bytes(uint32_t eb, uint32_t k) { return fast_layout(eb, k).total; }

__device__ __forceinline__ void bar_group(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Exclusive sum over the S group (one value per S thread; sid = 0..XSN-1).
__device__ __forceinline__ uint32_t s_exclusive_sum(uint32_t v, uint32_t* wsum, uint32_t* total, uint32_t sid) {
    const uint32_t lane = sid & 31u, warp = sid >> 5;
    const uint32_t incl = warp_inclusive_sum(v);
    if (lane == 31) wsum[warp] = incl;
    bar_group(kBarS, XSN);
    if (warp == 0) {
        const uint32_t x = lane < XSW ? wsum[lane] : 0u;
        const uint32_t xi = warp_inclusive_sum(x);
        if (lane < XSW) wsum[lane] = xi - x;
        if (lane == XSW - 1) wsum[XSW] = xi;
    }
    bar_group(kBarS, XSN);
    const uint32_t r = wsum[warp] + incl - v;
    *total = wsum[XSW];
    bar_group(kBarS, XSN);
    return r;
}

// Warp element ranges of the S group: the item's positions [P0, P0+m)
// cover ng Philox groups of dpg draws; S warp w owns groups [w*qg, (w+1)*qg).
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
        qg = (ng + XSW - 1) / XSW;
    }
};

// Child c = s*k + b of the level's segments: [start, start+len).
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

// Where the items come from: the children of a stable-mode level (in its
// output buffer; the stride sequence runs over the fused list when k_plan
// wrote one) or of an in-place level batch (in ptr, bucket starts from the
// batch table S).
struct XSrc {
    const LevelParams* lp;     // stable mode, or nullptr
    const IpParams* ip;        // in-place mode
    const unsigned char* src;  // buffer holding the children
    uint32_t lvl;              // level of the children
    uint32_t nchild;           // length of the stride sequence
    bool copy;                 // src != ptr: non-permuting children must still be copied
    bool list;                 // the sequence runs over rp.fused
    __device__ __forceinline__ void child(const RunParams& rp, uint32_t c, uint64_t& start, uint64_t& len,
                                          uint64_t& origin, uint64_t& key) const {
        if (lp) {
            SegDesc sg;
            child_of(*lp, rp.k, c, start, len, sg);
            origin = sg.origin;
            key = sg.key;
        } else {
            const uint32_t s = c / rp.k, b = c % rp.k;
            const uint64_t* S = ip->S + (uint64_t)s * (rp.k + 1);
            const uint64_t s0 = S[b];
            start = ip->segs[s].start + s0;
            len = S[b + 1] - s0;
            origin = 0;
            key = rp.seed;  // K(seed, 0) (D2)
        }
    }
};

template <int EB>
struct XView {
    XLayout Ly;
    uint32_t k;
    __device__ __forceinline__ explicit XView(uint32_t kk) : k(kk) { Ly = fast_layout(EB, kk); }
    __device__ __forceinline__ XCtl* ctl() const { return reinterpret_cast<XCtl*>(xsm); }
    __device__ __forceinline__ unsigned char* buf(uint32_t i) const { return xsm + (i ? Ly.buf1 : Ly.buf0); }
    __device__ __forceinline__ unsigned char* draws() const { return xsm + Ly.draws; }
    __device__ __forceinline__ uint32_t* T() const { return reinterpret_cast<uint32_t*>(xsm + Ly.T); }
    __device__ __forceinline__ uint32_t* bst(uint32_t d) const {  // d: descriptor slot
        return reinterpret_cast<uint32_t*>(xsm + Ly.bst0) + d * (k + 1);
    }
    __device__ __forceinline__ uint32_t* wsum() const { return reinterpret_cast<uint32_t*>(xsm + Ly.wsum); }
    __device__ __forceinline__ uint16_t* perm(uint32_t i) const {
        return reinterpret_cast<uint16_t*>(xsm + Ly.perm) + i * k;
    }
};

// Element e of an item sits at byte ((start*EB) & 15) + e*EB of its buffer,
// so the 16-byte-aligned body of the item maps to an aligned address.
template <int EB>
__device__ __forceinline__ unsigned char* item_base(unsigned char* buf, uint64_t start) {
    return buf + ((start * EB) & 15u);
}

// ---------------------------------------------------------------- C ------
// Store item `it` from buffer bi (warp C; lane 0 the bulk body, lanes 1..6
// the <= 3 unaligned words at each end); returns when the buffer is free.
template <int EB>
__device__ __forceinline__ void c_store(const RunParams& rp, const XView<EB>& V, const XItem& it, uint32_t bi) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    const unsigned char* ob = V.buf(bi);
    if (lane == 0 && body) {
        fence_proxy_async();
        bulk_s2g(rp.buf0 + A, ob + (A - fl), (uint32_t)(B - A));
        bulk_commit();
    }
    const uint64_t hEnd = body ? A : x1, tBeg = body ? B : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2), nt = (uint32_t)((x1 - tBeg) >> 2);
    if (lane >= 1 && lane <= 3 && lane - 1 < nh)
        *reinterpret_cast<uint32_t*>(rp.buf0 + x0 + 4 * (lane - 1)) =
            *reinterpret_cast<const uint32_t*>(ob + (x0 - fl) + 4 * (lane - 1));
    if (lane >= 4 && lane <= 6 && lane - 4 < nt)
        *reinterpret_cast<uint32_t*>(rp.buf0 + tBeg + 4 * (lane - 4)) =
            *reinterpret_cast<const uint32_t*>(ob + (tBeg - fl) + 4 * (lane - 4));
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
}

// find_next with the 32 lanes of warp C examining 32 children of the CTA's
// stride sequence at once (the first taker wins; children before it are
// flagged, the ones after it are examined again next time).
template <int EB>
__device__ __forceinline__ void find_next_warp(const RunParams& rp, const XSrc& xs, uint32_t nchild, XCtl* ctl,
                                               uint32_t ds) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lvl = xs.lvl;
    uint32_t cursor = ctl->cursor;
    for (;;) {
        if (cursor >= nchild) break;
        const uint64_t c64 = (uint64_t)cursor + (uint64_t)lane * gridDim.x;
        // with the fused list (k_plan) the stride sequence runs over its entries
        const uint32_t c = (xs.list && c64 < nchild) ? rp.fused[c64] : (uint32_t)c64;
        bool take = false;
        int flag = -1;  // -1: leave the flag alone, 0 / 1: write it
        uint64_t start = 0, len = 0, origin = 0, key = 0;
        if (c64 < nchild) {
            xs.child(rp, c, start, len, origin, key);
            const bool leaf = len <= rp.L;
            if (len == 0 || len > rp.S_fuse || (leaf && rp.leafk)) {
                // empty, an HBM segment of the next level, or the leaf kernel's
            } else {
                const bool permutes = (!leaf && lvl < rp.max_levels) || (leaf && rp.run_leaves && len >= 2);
                if (!permutes) flag = xs.copy ? 1 : 0;
                else if (leaf || len > XCfg<EB>::SMAX || lvl + 1 > rp.max_levels || !rp.run_leaves) flag = 1;
                else take = true;
            }
        }
        const uint32_t tk = __ballot_sync(0xFFFFFFFFu, take);
        const uint32_t first = tk ? (uint32_t)(__ffs(tk) - 1) : 32u;
        if (lane < first && flag >= 0) rp.flags[c] = (unsigned char)flag;
        if (tk) {
            if (lane == first) {
                rp.flags[c] = 0;
                XItem& it = ctl->item[ds];
                it.start = start;
                it.origin = origin;
                it.key = key;
                it.len = (uint32_t)len;
                it.child = c;
                it.valid = 1;
                ctl->cursor = (uint32_t)c64 + gridDim.x;
            }
            __syncwarp();
            return;
        }
        cursor += 32u * gridDim.x;
    }
    if (lane == 0) {
        ctl->item[ds].valid = 0;
        ctl->cursor = 0xFFFFFFFFu;
    }
    __syncwarp();
}

// Find the next item into descriptor slot ds and publish it (warp C).
template <int EB>
__device__ __forceinline__ void c_find(const RunParams& rp, const XSrc& xs, const XView<EB>& V, uint32_t nchild,
                                       uint32_t ds) {
    XCtl* ctl = V.ctl();
    find_next_warp<EB>(rp, xs, nchild, ctl, ds);
    if ((threadIdx.x & 31u) == 0) mbar_arrive1(&ctl->desc[ds]);  // release: the descriptor is written
    __syncwarp();
}

// Start the load of the item in descriptor slot ds into buffer bi (warp C);
// an invalid item completes the buffer's phase with no bytes.
template <int EB>
__device__ __forceinline__ void c_load(const XSrc& xs, const XView<EB>& V, uint32_t ds, uint32_t bi) {
    const uint32_t lane = threadIdx.x & 31u;
    XCtl* ctl = V.ctl();
    const XItem it = ctl->item[ds];
    unsigned char* buf = V.buf(bi);
    const unsigned char* src = xs.src;
    uint32_t bytes = 0;
    uint64_t A = 0, fl = 0;
    if (it.valid) {
        const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
        fl = x0 & ~15ull;
        A = (x0 + 15) & ~15ull;
        const uint64_t B = x1 & ~15ull;
        const bool body = B > A;
        bytes = body ? (uint32_t)(B - A) : 0u;
        const uint64_t hEnd = body ? A : x1, tBeg = body ? B : x1;
        const uint32_t nh = (uint32_t)((hEnd - x0) >> 2), nt = (uint32_t)((x1 - tBeg) >> 2);
        if (lane >= 1 && lane <= 3 && lane - 1 < nh)
            *reinterpret_cast<uint32_t*>(buf + (x0 - fl) + 4 * (lane - 1)) =
                *reinterpret_cast<const uint32_t*>(src + x0 + 4 * (lane - 1));
        if (lane >= 4 && lane <= 6 && lane - 4 < nt)
            *reinterpret_cast<uint32_t*>(buf + (tBeg - fl) + 4 * (lane - 4)) =
                *reinterpret_cast<const uint32_t*>(src + tBeg + 4 * (lane - 4));
    }
    __syncwarp();
    if (lane == 0) {
        __threadfence_block();
        fence_proxy_async();
        mbar_arrive_expect_tx(&ctl->full[bi], bytes);
        if (bytes) bulk_g2s(buf + (A - fl), src + A, bytes, &ctl->full[bi]);
    }
    __syncwarp();
}

// ---------------------------------------------------------------- S ------
// Draws of the item -> smem (indexed by Philox group) and each S warp's
// bucket counts (packed u16 halves).
template <int EB, bool NARROW>
__device__ __forceinline__ void s_count(const RunParams& rp, const XView<EB>& V, const XItem& it, uint32_t lvl,
                                        uint32_t w) {
    const uint32_t k = rp.k, kw = NARROW ? k : (k + 1) >> 1, lane = threadIdx.x & 31u;
    const BucketParams bp = rp.bp;
    const uint64_t P0 = it.start - it.origin;
    const XRange<NARROW> xr(P0, it.len);
    const uint32_t m = xr.m;
    const PhiloxKey key = make_key(it.key);
    constexpr uint32_t sh = XRange<NARROW>::sh, dpg = XRange<NARROW>::dpg;
    uint32_t* Tw = V.T() + w * kw;
    for (uint32_t i = lane; i < kw; i += 32) Tw[i] = 0;
    __syncwarp();
    const uint32_t t1 = min(xr.ng, (w + 1) * xr.qg);
    for (uint32_t t = w * xr.qg + lane; t < t1; t += 32) {
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
        if (e0 >= 0 && e0 + (int32_t)dpg <= (int32_t)m) {
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const uint32_t b = NARROW ? __byte_perm(pw4[j >> 2], 0u, 0x4440u | (j & 3u))
                                          : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                if (NARROW) atomicAdd(&Tw[b], 1u);
                else atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
            }
        } else {
            for (uint32_t j = 0; j < dpg; ++j) {
                const int32_t e = e0 + (int32_t)j;
                const uint32_t b =
                    NARROW ? (pw4[j >> 2] >> ((j & 3u) * 8u)) & 0xFFu : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                if (e >= 0 && e < (int32_t)m) {
                    if (NARROW) atomicAdd(&Tw[b], 1u);
                    else atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
                }
            }
        }
    }
}

// Bucket starts -> bst (k+1 entries), per-warp slot bases into T, and the
// FY thread -> leaf map; returns 1 if some bucket exceeds L (the item then
// goes to the general kernel).
template <int EB, bool NARROW>
__device__ __forceinline__ uint32_t s_scan(const RunParams& rp, const XView<EB>& V, uint32_t* bst, uint16_t* perm,
                                           uint64_t start, uint32_t m, uint32_t sid) {
    const uint32_t k = rp.k;
    uint32_t* T = V.T();
    uint32_t mine = 0, big = 0;
    uint32_t x0, x1;
    if (NARROW) {  // u32 counters: thread owns buckets [x0, x1)
        const uint32_t per = (k + XSN - 1) / XSN;
        x0 = min(k, sid * per);
        x1 = min(k, x0 + per);
        for (uint32_t x = x0; x < x1; ++x) {
            uint32_t c = 0;
            for (uint32_t w = 0; w < XSW; ++w) c += T[w * k + x];
            big |= c > rp.L;
            mine += c;
        }
    } else {  // packed u16 counters: thread owns words [x0, x1)
        const uint32_t kw = (k + 1) >> 1;
        const uint32_t per = (kw + XSN - 1) / XSN;
        x0 = min(kw, sid * per);
        x1 = min(kw, x0 + per);
        for (uint32_t x = x0; x < x1; ++x) {
            uint32_t c0 = 0, c1 = 0;
            for (uint32_t w = 0; w < XSW; ++w) {
                const uint32_t c = T[w * kw + x];
                c0 += c & 0xFFFFu;
                c1 += c >> 16;
            }
            big |= (c0 > rp.L) | (c1 > rp.L);
            mine += c0 + c1;
        }
    }
    uint32_t total;
    uint32_t run = s_exclusive_sum(mine, V.wsum(), &total, sid);
    if (NARROW) {
        for (uint32_t x = x0; x < x1; ++x) {
            bst[x] = run;
            for (uint32_t w = 0; w < XSW; ++w) {
                const uint32_t c = T[w * k + x];
                T[w * k + x] = run;
                run += c;
            }
        }
    } else {
        const uint32_t kw = (k + 1) >> 1;
        for (uint32_t x = x0; x < x1; ++x) {
            uint32_t r0 = run, t0 = 0;
            for (uint32_t w = 0; w < XSW; ++w) t0 += T[w * kw + x] & 0xFFFFu;
            uint32_t r1 = run + t0;
            bst[2 * x] = r0;
            if (2 * x + 1 < k) bst[2 * x + 1] = r1;
            for (uint32_t w = 0; w < XSW; ++w) {
                const uint32_t c = T[w * kw + x];
                T[w * kw + x] = (r0 & 0xFFFFu) | (r1 << 16);
                r0 += c & 0xFFFFu;
                r1 += c >> 16;
            }
            run = r1;
        }
    }
    if (sid == 0) bst[k] = m;
    // any bucket > L anywhere in the group? (wsum[XSW] held the total: reused as the flag)
    const bool anyw = __any_sync(0xFFFFFFFFu, big != 0);
    uint32_t* cls = V.wsum();  // 32 class counters live past the XSW+1 scan words
    if ((sid & 31u) == 0 && anyw) cls[XSW] = 0xFFFFFFFFu;
    if (sid < 32) cls[XSW + 1 + sid] = 0;
    bar_group(kBarS, XSN);
    const uint32_t defer = cls[XSW] == 0xFFFFFFFFu ? 1u : 0u;
    // FY thread -> leaf map: with u32 elements and k <= 256 (k % 32 == 0),
    // leaves are dealt to the FY warps by the bank their Fisher-Yates steps
    // start from, so a warp's lanes touch A[i] in (mostly) distinct banks;
    // otherwise thread f takes leaf f.
    const bool deal = EB == 4 && k <= XF && (k & 31u) == 0;  // positions p -> FY threads [0, k), bijective
    uint32_t c = 0, rk = 0;
    const uint32_t w0 = (uint32_t)((start * EB) & 15u) >> 2;  // word offset of element 0
    if (deal && sid < k) {
        // fy_leaf walks i = 8g + jj with the warp's lanes in lockstep over (group
        // iteration n, jj), g = gt - n, gt = (cm - 1) >> 3: lane banks differ iff
        // (start + 8 gt) mod 32 differ
        const uint32_t s0 = bst[sid], cm = bst[sid + 1] - s0;
        c = (w0 + s0 + 8u * ((cm ? cm - 1u : 0u) >> 3)) & 31u;
        rk = atomicAdd(&cls[XSW + 1 + c], 1u);
    }
    bar_group(kBarS, XSN);
    if (sid < 32) {
        const uint32_t n = cls[XSW + 1 + sid];
        const uint32_t incl = warp_inclusive_sum(n);
        cls[XSW + 1 + sid] = incl - n;
    }
    bar_group(kBarS, XSN);
    if (sid < k) {
        if (deal) {
            const uint32_t W = (k + 31) >> 5;  // FY warps in use
            const uint32_t p = cls[XSW + 1 + c] + rk;  // position in bank order
            // position p -> FY thread (warp p % W, lane p / W)
            perm[(p % W) * 32u + p / W] = (uint16_t)sid;
        } else {
            perm[sid] = (uint16_t)sid;
        }
    }
    bar_group(kBarS, XSN);
    return defer;
}

// Stable in-place scatter of the item inside its buffer: every S thread
// holds its elements in registers across a group barrier, then each takes
// its slot with one ordered shared atomic (warp rounds in position order).
template <int EB, bool NARROW, bool ORD>
__device__ __forceinline__ void s_place(const XView<EB>& V, const XItem& it, unsigned char* base, uint32_t w,
                                        uint32_t* err) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    constexpr uint32_t R = XCfg<EB>::R;
    const uint32_t lane = threadIdx.x & 31u, kw = NARROW ? V.k : (V.k + 1) >> 1;
    const XRange<NARROW> xr(it.start - it.origin, it.len);
    const int32_t eb0 = (int32_t)(w * xr.qg * xr.dpg) - (int32_t)xr.doff;
    const uint32_t e_lo = eb0 > 0 ? (uint32_t)eb0 : 0u;
    const int32_t ehi = min((int32_t)((w + 1) * xr.qg * xr.dpg) - (int32_t)xr.doff, (int32_t)xr.m);
    const uint32_t len = ehi > (int32_t)e_lo ? (uint32_t)ehi - e_lo : 0u;
    E* el = reinterpret_cast<E*>(base);
    const D* dp = reinterpret_cast<const D*>(V.draws()) + xr.doff + e_lo;
    uint32_t* Tw = V.T() + w * kw;
    E v[R];
    const uint32_t ilast = len ? len - 1 : 0u;
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = r * 32u + lane;
        v[r] = el[e_lo + (i < len ? i : ilast)];  // unconditional: keeps v[] in registers
    }
    bar_group(kBarS, XSN);
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        if (r * 32u >= len) break;  // warp-uniform
        const uint32_t i = r * 32u + lane;
        const bool valid = i < len;
        const uint32_t b = valid ? (uint32_t)dp[i] : 0u;
        uint32_t slot;
        if (ORD && NARROW) {
            slot = atomicAdd(&Tw[valid ? b : (lane < kw ? lane : 0u)], valid ? 1u : 0u);  // idle lanes: +0, spread over banks
        } else if (ORD) {
            const uint32_t shb = (b & 1u) << 4;
            slot = (atomicAdd(&Tw[valid ? b >> 1 : (lane < kw ? lane : 0u)], valid ? (1u << shb) : 0u) >> shb) & 0xFFFFu;
        } else if (NARROW) {
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, valid ? b : 0xFFFFFFFFu);
            slot = valid ? Tw[b] + __popc(peers & lanemask_lt()) : 0u;
            __syncwarp();
            if (valid && (peers & lanemask_lt()) == 0) Tw[b] += __popc(peers);
            __syncwarp();
        } else {
            slot = warp_rank(Tw, b, valid, false);
        }
        if (ORD && r == 0 && w == 0) check_rank_order(b, valid, slot, err);
        if (valid) el[slot] = v[r];
    }
}

// ------------------------------------------------------------- kernel ---
template <int EB, bool NARROW, bool ORD>
__device__ __forceinline__ void run_fast(const RunParams& rp, const XSrc& xs) {
    const XView<EB> V(rp.k);
    XCtl* ctl = V.ctl();
    const uint32_t tid = threadIdx.x, k = rp.k;
    const uint32_t nchild = xs.nchild;
    const uint32_t lvl = xs.lvl;
    if (tid == 0) {
        ctl->cursor = blockIdx.x;
        ctl->dbg_s = ctl->dbg_f = 0;
        ctl->st_fin = ctl->st_fy = 0;
        for (int i = 0; i < 2; ++i) {
            mbar_init(&ctl->full[i], 1);
            mbar_init(&ctl->ready[i], 1);
            mbar_init(&ctl->fydone[i], 1);
        }
        for (uint32_t d = 0; d < XD; ++d) {
            mbar_init(&ctl->desc[d], 1);
            ctl->defer[d] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    const bool dbgcta = (rp.dbg & 4u) && blockIdx.x == 0;
    if (tid >= XC && tid < XS0) {
        // ---------------- C: loads and stores
        // descriptors run up to 4 items ahead of the stores, loads 2 ahead
        for (uint32_t d = 0; d < XD; ++d) {
            c_find<EB>(rp, xs, V, nchild, d);
            if (d < 2) c_load<EB>(xs, V, d, d);
        }
        for (uint32_t t = 0;; ++t) {
            const uint32_t bi = t & 1u, ds = t % XD;
            mbar_wait(&ctl->fydone[bi], (t >> 1) & 1u);
            const XItem it = ctl->item[ds];
            if (!it.valid) break;
            if (!ctl->defer[ds]) {
                c_store<EB>(rp, V, it, bi);
                if (tid == XC) ctl->st_fin += it.len;
            }
            __syncwarp();
            c_load<EB>(xs, V, (t + 2) % XD, bi);  // buffer bi is free: item t+2
            c_find<EB>(rp, xs, V, nchild, ds);    // descriptor slot ds is free: item t+4
        }
        if (tid == XC) bulk_wait0();
    } else if (tid >= XS0) {
        // ---------------- S: draws, counts, scan, in-place stable scatter
        const uint32_t sid = tid - XS0, w = sid >> 5;
        for (uint32_t t = 0;; ++t) {
            const uint32_t bi = t & 1u, ds = t % XD;
            // draws, counts and scan need only the descriptor: they overlap the load
            mbar_wait(&ctl->desc[ds], (t / XD) & 1u);
            const XItem it = ctl->item[ds];
            const bool dbg = dbgcta && sid == 0 && ctl->dbg_s < 40;
            if (dbg) rp.hdr->clk[ctl->dbg_s * 6 + 0] = clock64();
            uint32_t defer = 1;
            if (it.valid && (rp.dbg & 16u)) {  // timing experiment: S does no work (F runs alone)
                if (sid < k) V.perm(ds)[sid] = (uint16_t)sid;
                for (uint32_t b = sid; b <= k; b += XSN) V.bst(ds)[b] = (uint32_t)((uint64_t)b * it.len / k);
                defer = 0;
                mbar_wait(&ctl->full[bi], (t >> 1) & 1u);
            } else if (it.valid) {
                s_count<EB, NARROW>(rp, V, it, lvl, w);
                bar_group(kBarS, XSN);
                defer = s_scan<EB, NARROW>(rp, V, V.bst(ds), V.perm(ds), it.start, it.len, sid);
                if (dbg) rp.hdr->clk[ctl->dbg_s * 6 + 1] = clock64();
                mbar_wait(&ctl->full[bi], (t >> 1) & 1u);  // the item's data
                if (!defer) s_place<EB, NARROW, ORD>(V, it, item_base<EB>(V.buf(bi), it.start), w, &rp.hdr->error);
                else if (sid == 0) rp.flags[it.child] = 1;  // the general kernel takes it
            } else {
                mbar_wait(&ctl->full[bi], (t >> 1) & 1u);
            }
            fence_proxy_async();  // placement writes, before C's bulk store of a finished item
            bar_group(kBarS, XSN);
            if (sid == 0) {
                ctl->defer[ds] = defer;
                if (dbg) rp.hdr->clk[ctl->dbg_s++ * 6 + 2] = clock64();
                mbar_arrive1(&ctl->ready[bi]);
            }
            if (!it.valid) break;
        }
    } else {
        // ---------------- F: Fisher-Yates of every leaf of item t
        unsigned long long fyn = 0;
        for (uint32_t t = 0;; ++t) {
            const uint32_t bi = t & 1u, ds = t % XD;
            mbar_wait(&ctl->ready[bi], (t >> 1) & 1u);
            const XItem it = ctl->item[ds];
            const bool dbg = dbgcta && tid == 0 && ctl->dbg_f < 40;
            if (dbg) rp.hdr->clk[ctl->dbg_f * 6 + 3] = clock64();
            if (it.valid && !ctl->defer[ds] && !(rp.dbg & 8u)) {  // dbg 8: timing experiment, no FY
                const uint32_t* bst = V.bst(ds);
                unsigned char* base = item_base<EB>(V.buf(bi), it.start);
                const uint64_t P0 = it.start - it.origin;
                const PhiloxKey key = make_key(it.key);
                const uint16_t* perm = V.perm(ds);
                for (uint32_t f = tid; f < k; f += XF) {
                    const uint32_t b = (k <= XF) ? perm[f] : f;
                    const uint32_t s0 = bst[b], cm = bst[b + 1] - s0;
                    if (cm >= 2) {
                        fy_leaf<EB>(base, s0, cm, P0 + s0, key);
                        fyn += cm;
                    }
                }
            }
            fence_proxy_async();  // every writer of the buffer orders its writes before C's bulk store
            bar_group(kBarF, XF);
            if (tid == 0) {
                if (dbg) rp.hdr->clk[ctl->dbg_f++ * 6 + 4] = clock64();
                mbar_arrive1(&ctl->fydone[bi]);
            }
            if (!it.valid) break;
        }
        for (int o = 16; o > 0; o >>= 1) fyn += __shfl_xor_sync(0xFFFFFFFFu, fyn, o);
        if ((tid & 31u) == 0 && fyn) atomicAdd(&ctl->st_fy, fyn);
    }
    __syncthreads();
    if (tid == 0) {
        atomicAdd((unsigned long long*)&rp.hdr->finished, ctl->st_fin);
        atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[lvl < kMaxLevels ? lvl : 0], ctl->st_fin);
        atomicAdd((unsigned long long*)&rp.hdr->fy_elems, ctl->st_fy);
    }
}

template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(XNT, 1) k_finish_fast(RunParams rp, LevelParams lp) {
    XSrc xs;
    xs.lp = &lp;
    xs.ip = nullptr;
    xs.src = lp.dst;
    xs.lvl = lp.level + 1;
    xs.list = rp.max_fused != 0;
    xs.nchild = xs.list ? lp.ctr->nfuse : lp.ctr->nseg * rp.k;
    xs.copy = lp.dst != rp.buf0;
    run_fast<EB, NARROW, ORD>(rp, xs);
}

// Children of an in-place level batch (kernels_inplace.cu), in place in ptr.
template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(XNT, 1) k_finish_fast_ip(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    XSrc xs;
    xs.lp = nullptr;
    xs.ip = &ip;
    xs.src = rp.buf0;
    xs.lvl = ip.level + 1;
    xs.list = false;
    xs.nchild = ip.nseg * rp.k;
    xs.copy = false;
    run_fast<EB, NARROW, ORD>(rp, xs);
}

template <int EB>
static void* fast_fn(bool narrow, bool ord, bool ip) {
    if (ip) {
        if (ord) return narrow ? (void*)k_finish_fast_ip<EB, true, true> : (void*)k_finish_fast_ip<EB, false, true>;
        return narrow ? (void*)k_finish_fast_ip<EB, true, false> : (void*)k_finish_fast_ip<EB, false, false>;
    }
    if (ord) return narrow ? (void*)k_finish_fast<EB, true, true> : (void*)k_finish_fast<EB, false, true>;
    return narrow ? (void*)k_finish_fast<EB, true, false> : (void*)k_finish_fast<EB, false, false>;
}
static void* fast_kernel(uint32_t eb, bool narrow, bool ord, bool ip = false) {
    switch (eb) {
    case 4: return fast_fn<4>(narrow, ord, ip);
    case 8: return fast_fn<8>(narrow, ord, ip);
    default: return fast_fn<16>(narrow, ord, ip);
    }
}

cudaError_t configure_fast(uint32_t eb, uint32_t k) {
    const uint32_t smem = fast_smem_bytes(eb, k);
    if (smem > kSmemLimit) return cudaErrorInvalidValue;
    for (int nr = 0; nr < 2; ++nr)
        for (int o = 0; o < 2; ++o)
            for (int ip = 0; ip < 2; ++ip) {
                cudaError_t e = cudaFuncSetAttribute(fast_kernel(eb, nr != 0, o != 0, ip != 0),
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
                if (e) return e;
            }
    return cudaSuccess;
}

cudaError_t launch_finish_fast(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = fast_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&lp};
    return cudaLaunchKernel(fast_kernel(rp.eb, rp.bp.narrow != 0, rp.rank_ordered != 0), dim3(grid), dim3(XNT), args,
                            smem, s);
}

cudaError_t launch_finish_fast_ip(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    const uint32_t smem = fast_smem_bytes(rp.eb, rp.k);
    void* args[] = {(void*)&rp, (void*)&ip};
    return cudaLaunchKernel(fast_kernel(rp.eb, rp.bp.narrow != 0, rp.rank_ordered != 0, true), dim3(grid), dim3(XNT),
                            args, smem, s);
}

}  // namespace shuf
