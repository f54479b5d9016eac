// Fast fused finish for the common shape of the recursion (SURVEY 8(a) a7+a8):
// a child of the last HBM level ("item") that needs exactly ONE more scatter
// level, after which every grandchild is a leaf (<= L and <= 256 elements)
// -- e.g. the HOT run's 65 536 children of ~16 K u32 that split into
// ~64-element leaves.
//
// One CTA of 1024 threads per SM and two item buffers whose roles alternate
// (DESIGN.md 6.3).  Item t arrives (bulk async copy, TMA engine) in buffer
// I = t & 1; per item, in phases separated by CTA barriers:
//   1. draws + counts: the level's bucket draws (D4, Philox) -> shared
//      memory; warp w owns a run of Philox groups and counts them per bucket;
//   2. scan: bucket (= leaf) starts, 32-leaf column groups, per-warp row
//      bases;  (the load of item t has been in flight since item t-1)
//   3. placement I -> C (the other buffer) in COLUMN layout: leaf b's r-th
//      element at C[32 (G(b) + r) + (b & 31)]; warp w walks its elements in
//      rounds of 32 in position order and one ordered shared atomic on its
//      own table returns the row (stable, D6);
//   4. Fisher-Yates partners of every leaf (D5), all threads;
//   5. Fisher-Yates (Fig. 1), one thread per leaf (warps 0..7):
//      the 32 leaves of a warp sit in 32 banks of C, so each step's loads and
//      store are conflict-free; position i is final after step i and goes
//      straight to the contiguous item layout in I (the input is dead);
//   6. one bulk async store of I to ptr; the load of item t+1 into C (free
//      again) is issued.
// Items of another shape (a grandchild > L or > 256 elements, a leaf-only
// child, more than SMAX elements, column overflow) are flagged and finished
// by the general kernel (kernels_finish.cu) right after.
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char xsm[];

constexpr int XNT = 1024;          // threads per CTA
constexpr uint32_t XW = XNT / 32;  // 32 warps: draws, counts, placement
constexpr uint32_t XFYT = 256;     // Fisher-Yates threads (warps 0..7)
constexpr uint32_t XBUF = 86016;   // bytes per item buffer (contiguous item / column layout)
constexpr uint32_t XIN = 69632;    // bytes of the largest item the fast path takes (68 KiB)

template <int EB>
struct XCfg {
    static constexpr uint32_t SMAX = XIN / EB;               // largest item
    static constexpr uint32_t COLCAP = XBUF / EB / 32 * 32;  // column-layout capacity (elements)
};

uint32_t fast_max_elems(uint32_t eb) { return XIN / eb; }

struct XItem {
    uint64_t start, origin, key;
    uint64_t child;  // child index c = s*k + b (for the deferral flag)
    uint32_t len, valid;
};

struct XCtl {
    XItem cur, nxt, nxt2;  // item t, t+1 (counted during FY(t)), t+2 (searched during FY(t))
    uint64_t bar[2];  // mbarriers of the two buffers' loads
    uint32_t ph[2];   // their parities
    uint32_t cursor;  // this CTA's next candidate child index
    uint32_t defer;   // cur is handed to the general kernel
    uint32_t gh[33];  // per 32-leaf group: longest leaf
    uint32_t dbg_it;  // items processed (phase clocks of the first ones, CTA 0)
    unsigned long long st_fin, st_fy;
};

struct XLayout {
    uint32_t buf0, buf1, draws, jb, T, meta, wsum, total, jbbytes;
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
    f.jbbytes = XBUF / eb + ((k + 31) / 32 + 1) * 256;  // partner words, column layout (4 steps per word)
    f.jb = take(f.jbbytes);
    f.T = take(XW * ((k + 1) / 2) * 4);
    f.meta = take(((k + 1) + 33 + 33) * 4);  // bst[k+1], gb[33], gj[33]
    f.wsum = take((XNT / 32 + 1) * 4);
    f.total = off;
    return f;
}

uint32_t fast_smem_bytes(uint32_t eb, uint32_t k) { return fast_layout(eb, k).total; }

// 4-byte asynchronous global -> shared copy (the unaligned head/tail words of
// an item; completion by cp.async.wait_all).
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Warp element ranges.  The item's positions [P0, P0+m) cover ng Philox
// groups of dpg draws; warp w owns groups [w*qg, (w+1)*qg), i.e. elements
// e in [w*qg*dpg - doff, (w+1)*qg*dpg - doff) clipped to [0, m).
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
        qg = (ng + XW - 1) / XW;
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
    uint32_t k;
    __device__ __forceinline__ explicit XView(uint32_t kk) : k(kk) { Ly = fast_layout(EB, kk); }
    __device__ __forceinline__ XCtl* ctl() const { return reinterpret_cast<XCtl*>(xsm); }
    __device__ __forceinline__ unsigned char* buf(uint32_t i) const { return xsm + (i ? Ly.buf1 : Ly.buf0); }
    __device__ __forceinline__ unsigned char* draws() const { return xsm + Ly.draws; }
    __device__ __forceinline__ uint32_t* jb() const { return reinterpret_cast<uint32_t*>(xsm + Ly.jb); }
    __device__ __forceinline__ uint32_t* T() const { return reinterpret_cast<uint32_t*>(xsm + Ly.T); }
    __device__ __forceinline__ uint32_t* bst() const { return reinterpret_cast<uint32_t*>(xsm + Ly.meta); }
    __device__ __forceinline__ uint32_t* gb() const { return bst() + k + 1; }       // element rows of group g
    __device__ __forceinline__ uint32_t* gj() const { return bst() + k + 1 + 33; }  // partner-word rows of group g
    __device__ __forceinline__ uint32_t* wsum() const { return reinterpret_cast<uint32_t*>(xsm + Ly.wsum); }
};

// Element e of an item in contiguous layout sits at byte ((start*EB) & 15) +
// e*EB of its buffer, so the 16-byte-aligned body maps to an aligned address.
template <int EB>
__device__ __forceinline__ unsigned char* item_base(unsigned char* buf, uint64_t start) {
    return buf + ((start * EB) & 15u);
}

// The load of item `it` into buffer bi: the aligned body by one bulk async
// copy (thread 0), the <= 3 unaligned words at each end by 4-byte
// asynchronous copies (threads 32..39, which wait for them before phase 3).
template <int EB>
__device__ __forceinline__ void issue_load(const XView<EB>& V, const XItem& it, const unsigned char* src, uint32_t bi) {
    const uint32_t tid = threadIdx.x;
    const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    unsigned char* buf = V.buf(bi);
    XCtl* ctl = V.ctl();
    if (tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&ctl->bar[bi], body ? (uint32_t)(B - A) : 0u);
        if (body) bulk_g2s(buf + (A - fl), src + A, (uint32_t)(B - A), &ctl->bar[bi]);
        return;
    }
    const uint64_t hEnd = body ? A : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
    const uint64_t tBeg = body ? B : x1;
    const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
    const uint32_t r = tid - 32;  // 0..7
    if (r < 4) {
        if (r < nh) cp_async4(buf + (x0 - fl) + 4 * r, src + x0 + 4 * r);
    } else if (r - 4 < nt) {
        cp_async4(buf + (tBeg - fl) + 4 * (r - 4), src + tBeg + 4 * (r - 4));
    }
}

// ---- phase 1: draws of the item -> smem (indexed by Philox group) and each
// warp's bucket counts (its groups are its elements).
// Warps [w0, w0 + nw) do it for all 32 placing warps' ranges (w = w0 + i,
// w0 + i + nw, ...).
template <int EB, bool NARROW>
__device__ __forceinline__ void draw_count_phase(const RunParams& rp, const XView<EB>& V, const XItem& it,
                                                 uint32_t lvl, uint32_t w0, uint32_t nw) {
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t lane = threadIdx.x & 31u;
    const BucketParams bp = rp.bp;
    const uint64_t P0 = it.start - it.origin;
    const XRange<NARROW> xr(P0, it.len);
    const uint32_t m = xr.m;
    const PhiloxKey key = make_key(it.key);
    constexpr uint32_t sh = XRange<NARROW>::sh, dpg = XRange<NARROW>::dpg;
    for (uint32_t w = (threadIdx.x >> 5) - w0; w < XW; w += nw) {
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
        // counter of bucket b: 16-bit half (b & 1) of word b >> 1 of the warp's table
        if (e0 >= 0 && e0 + (int32_t)dpg <= (int32_t)m) {  // whole group (all but <= 2 per item)
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const uint32_t b = NARROW ? __byte_perm(pw4[j >> 2], 0u, 0x4440u | (j & 3u))
                                          : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
            }
        } else {
            for (uint32_t j = 0; j < dpg; ++j) {
                const int32_t e = e0 + (int32_t)j;
                const uint32_t b =
                    NARROW ? (pw4[j >> 2] >> ((j & 3u) * 8u)) & 0xFFu : (pw4[j >> 1] >> ((j & 1u) * 16u)) & 0xFFFFu;
                if (e >= 0 && e < (int32_t)m) atomicAdd(&Tw[b >> 1], 1u << ((b & 1u) << 4));
            }
        }
    }
    }
}

// ---- phase 2: bucket starts, 32-leaf column groups (element rows gb and
// partner-word rows gj), per-warp row bases; flags the item for the general
// kernel if it does not fit.
template <int EB>
__device__ __forceinline__ void scan_phase(const RunParams& rp, const XView<EB>& V) {
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    XCtl* ctl = V.ctl();
    uint32_t* T = V.T();
    uint32_t* bst = V.bst();
    uint32_t* gb = V.gb();
    uint32_t* gj = V.gj();
    const uint32_t b0 = 2 * tid;  // thread tid owns buckets 2tid, 2tid+1 (k <= 1024 < 2 x 1024)
    uint32_t c0 = 0, c1 = 0;
    if (b0 < k) {
#pragma unroll 8
        for (uint32_t w = 0; w < XW; ++w) {
            const uint32_t c = T[w * kw + tid];
            c0 += c & 0xFFFFu;
            c1 += c >> 16;
        }
        if (b0 + 1 >= k) c1 = 0;
    }
    uint32_t total;
    const uint32_t ex = block_exclusive_sum<XNT>(c0 + c1, V.wsum(), &total);
    if (b0 < k) {
        bst[b0] = ex;
        if (b0 + 1 < k) bst[b0 + 1] = ex + c0;
    }
    if (tid == 0) bst[k] = ctl->cur.len;
    // rows of each 32-leaf group (16 threads) = its longest leaf
    uint32_t gm = c0 > c1 ? c0 : c1;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        const uint32_t t2 = __shfl_xor_sync(0xFFFFFFFFu, gm, o);
        gm = gm > t2 ? gm : t2;
    }
    if ((tid & 15u) == 0 && (tid >> 4) < 33) ctl->gh[tid >> 4] = gm;
    __syncthreads();
    if (warp == 0) {
        const uint32_t ngr = (k + 31) >> 5;
        const uint32_t h = lane < ngr ? ctl->gh[lane] : 0u;
        const uint32_t hj = ((h + 7) >> 3) * 2;  // partner words: 2 per 8-step Philox group
        const uint32_t incl = warp_inclusive_sum(h), inclj = warp_inclusive_sum(hj);
        if (lane < ngr) {
            gb[lane] = incl - h;
            gj[lane] = inclj - hj;
        }
        const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, h);
        if (lane == 31)
            ctl->defer = (mx > rp.L || mx > 256u || incl * 32u > XCfg<EB>::COLCAP || inclj * 128u > V.Ly.jbbytes)
                             ? 1u
                             : 0u;
    }
    __syncthreads();
    if (ctl->defer == 0) {
        // per-warp row bases: T[w][b] = gb(b / 32) + sum_{w'<w} cnt[w'][b]
        if (b0 < k) {
            uint32_t r0 = gb[b0 >> 5], r1 = gb[(b0 + 1) >> 5];
#pragma unroll 8
            for (uint32_t w = 0; w < XW; ++w) {
                const uint32_t c = T[w * kw + tid];
                T[w * kw + tid] = (r0 & 0xFFFFu) | (r1 << 16);
                r0 += c & 0xFFFFu;
                r1 += c >> 16;
            }
        }
    } else if (tid == 0) {
        rp.flags[ctl->cur.child] = 1;  // hand the item to the general kernel
    }
}

// ---- phase 3: placement, contiguous buffer bi -> column layout in bc.
template <int EB, bool NARROW>
__device__ __forceinline__ void place_phase(const XView<EB>& V, uint32_t kw, uint32_t bi, uint32_t bc) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    XCtl* ctl = V.ctl();
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint64_t start = ctl->cur.start;
    const XRange<NARROW> xr(start - ctl->cur.origin, ctl->cur.len);
    const int32_t eb0 = (int32_t)(w * xr.qg * xr.dpg) - (int32_t)xr.doff;
    const uint32_t e_lo = eb0 > 0 ? (uint32_t)eb0 : 0u;
    const int32_t ehi = min((int32_t)((w + 1) * xr.qg * xr.dpg) - (int32_t)xr.doff, (int32_t)xr.m);
    const uint32_t len = ehi > (int32_t)e_lo ? (uint32_t)ehi - e_lo : 0u;
    const E* in = reinterpret_cast<const E*>(item_base<EB>(V.buf(bi), start)) + e_lo;
    const D* dp = reinterpret_cast<const D*>(V.draws()) + xr.doff + e_lo;
    E* col = reinterpret_cast<E*>(V.buf(bc));
    uint32_t* Tw = V.T() + w * kw;
    // whole rounds of 32 in position order, then the partial last one
    const uint32_t nfull = len & ~31u;
#pragma unroll 4
    for (uint32_t i0 = 0; i0 < nfull; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t b = dp[i];
        const E x = in[i];
        const uint32_t shb = (b & 1u) << 4;
        const uint32_t row = (atomicAdd(&Tw[b >> 1], 1u << shb) >> shb) & 0xFFFFu;
        col[row * 32u + (b & 31u)] = x;
    }
    if (nfull < len) {
        const uint32_t i = nfull + lane;
        const bool valid = i < len;
        const uint32_t ii = valid ? i : nfull;
        const uint32_t b = valid ? (uint32_t)dp[ii] : 0u;
        const E x = in[ii];
        const uint32_t shb = (b & 1u) << 4;
        const uint32_t row = (atomicAdd(&Tw[b >> 1], valid ? (1u << shb) : 0u) >> shb) & 0xFFFFu;
        if (valid) col[row * 32u + (b & 31u)] = x;
    }
}

// Exact Lemire16 decision for the steps flagged by the cheap pre-check
// (low part < s), with the retry stream of D5 (out of line: rare).
static __device__ __noinline__ void partner_fixup(uint32_t (&pk)[2], uint32_t rej, const uint32_t (&wv)[4],
                                                  PhiloxKey key, uint64_t qq, uint32_t g, uint32_t mb) {
    for (uint32_t jj = 0; jj < 8; ++jj) {
        const uint32_t i = g * 8u + jj;
        if (!((rej >> jj) & 1u) || i < 1 || i >= mb) continue;
        const uint32_t vv = (wv[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu;
        const uint32_t j = fy16_from_lane(vv, key, qq, i);
        pk[jj >> 2] = (pk[jj >> 2] & ~(0xFFu << ((jj & 3u) * 8u))) | ((j & 0xFFu) << ((jj & 3u) * 8u));
    }
}

// ---- phase 4: partners j_i, i = 1 .. mb-1 of every leaf (D5: leaf id =
// problem position of the leaf start, one Philox block per 8 steps,
// Lemire16), packed 4 per word, in the leaves' column layout: word w (steps
// 4w .. 4w+3) of leaf b at jb[32 (gj(b/32) + w) + (b & 31)].  Thread t takes
// leaf t % k and every (1024/k)-th Philox group of it.
template <int EB>
__device__ __forceinline__ void partner_phase(const RunParams& rp, const XView<EB>& V) {
    XCtl* ctl = V.ctl();
    const uint32_t k = rp.k, tid = threadIdx.x;
    const uint32_t* bst = V.bst();
    const uint32_t* gj = V.gj();
    const uint64_t P0 = ctl->cur.start - ctl->cur.origin;
    const PhiloxKey key = make_key(ctl->cur.key);
    const uint32_t per = XNT / k >= 2 ? XNT / k : 1;  // threads per leaf
    if (per > 1 && tid >= per * k) return;
    const uint32_t sub = per > 1 ? tid / k : 0;
    const uint32_t bstep = per > 1 ? k : XNT;
    for (uint32_t b = per > 1 ? tid % k : tid; b < k; b += bstep) {
        const uint32_t s0 = bst[b], mb = bst[b + 1] - s0;
        if (mb < 2) continue;
        const uint64_t qq = P0 + s0;
        uint32_t* jw = V.jb() + gj[b >> 5] * 32u + (b & 31u);
        const uint32_t ngr = ((mb - 1) >> 3) + 1;
        for (uint32_t g = sub; g < ngr; g += per) {
            const uint4 w4 = fy16_group_words(key, qq, g);
            const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
            uint32_t pk[2] = {0u, 0u};
            uint32_t rej = 0;  // steps whose 16-bit lane Lemire may reject (rare)
#pragma unroll
            for (uint32_t jj = 0; jj < 8; ++jj) {
                const uint32_t i = g * 8u + jj;
                const uint32_t vv = (wv[jj >> 1] >> ((jj & 1) * 16)) & 0xFFFFu;
                const uint32_t sb = i + 1, mm = vv * sb;
                rej |= ((mm & 0xFFFFu) < sb ? 1u : 0u) << jj;
                pk[jj >> 2] |= ((mm >> 16) & 0xFFu) << ((jj & 3u) * 8u);
            }
            if (__builtin_expect(rej != 0, 0)) partner_fixup(pk, rej, wv, key, qq, g, mb);
            jw[(2 * g) * 32u] = pk[0];
            jw[(2 * g + 1) * 32u] = pk[1];
        }
    }
}

// ---- phase 5: Fisher-Yates of every leaf (threads 0..255), column layout in
// bc -> final elements to the contiguous item layout in bi.
template <int EB>
__device__ __forceinline__ uint32_t fy_phase(const RunParams& rp, const XView<EB>& V, uint32_t bi, uint32_t bc) {
    using E = typename ElemT<EB>::type;
    const uint32_t tid = threadIdx.x, k = rp.k;
    XCtl* ctl = V.ctl();
    const uint32_t* bst = V.bst();
    const uint32_t* gb = V.gb();
    const uint32_t* gj = V.gj();
    E* col0 = reinterpret_cast<E*>(V.buf(bc));
    E* out0 = reinterpret_cast<E*>(item_base<EB>(V.buf(bi), ctl->cur.start));
    uint32_t fyn = 0;
    for (uint32_t b = tid; b < k; b += XFYT) {
        const uint32_t s0 = bst[b], mb = bst[b + 1] - s0;
        if (mb == 0) continue;
        E* c = col0 + gb[b >> 5] * 32u + (b & 31u);  // leaf element t at c[32 t]
        E* o = out0 + s0;
        if (mb >= 2) {
            fyn += mb;
            // Fig. 1 for i = mb-1 .. 1: swap(A[i], A[j_i]).  Position i is final
            // after step i: it goes to o[i], and A[i] is never read again.
            // Software-pipelined: the loads of step i-1 are issued before the
            // store of step i and patched when step i wrote the same place
            // (j_i == i-1, or j_{i-1} == j_i).
            const uint32_t* jw = V.jb() + gj[b >> 5] * 32u + (b & 31u);
            uint32_t i = mb - 1;
            uint32_t word = jw[(i >> 2) * 32u];
            uint32_t jc = (word >> ((i & 3u) * 8u)) & 0xFFu;
            E x = c[i * 32u], y = c[jc * 32u];
            for (; i >= 2; --i) {
                const uint32_t in = i - 1;
                if ((in & 3u) == 3u) word = jw[(in >> 2) * 32u];
                const uint32_t jn = (word >> ((in & 3u) * 8u)) & 0xFFu;
                E xn = c[in * 32u];
                E yn = c[jn * 32u];
                c[jc * 32u] = x;
                o[i] = y;
                xn = (jc == in) ? x : xn;
                yn = (jn == jc) ? x : yn;
                x = xn;
                y = yn;
                jc = jn;
            }
            c[jc * 32u] = x;  // step 1
            o[1] = y;
        }
        o[0] = c[0];
    }
    return fyn;
}

// ------------------------------------------------------------- loop ---
template <int EB, bool NARROW>
__device__ __forceinline__ void run(const RunParams& rp, const LevelParams& lp, const XView<EB>& V, uint32_t nchild) {
    XCtl* ctl = V.ctl();
    const uint32_t k = rp.k, kw = (k + 1) >> 1, tid = threadIdx.x;
    const unsigned char* src = lp.dst;  // the level's output buffer holds the children
    const uint32_t lvl = lp.level + 1;
    // prologue: load + draws/counts of the first item, search of the second
    if (ctl->cur.valid) {
        if (tid == 0 || (tid >= 32 && tid < 40)) issue_load<EB>(V, ctl->cur, src, 0);
        draw_count_phase<EB, NARROW>(rp, V, ctl->cur, lvl, 0, XW);
    }
    if (tid == 64) ctl->nxt = find_next<EB>(rp, lp, nchild, ctl->cursor);
    __syncthreads();
    for (uint32_t t = 0; ctl->cur.valid; ++t) {
        const uint32_t bi = t & 1u, bc = bi ^ 1u;
        const bool dbg = blockIdx.x == 0 && tid == 0 && ctl->dbg_it < 40;
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 0] = clock64();
        // 2. scan (the counts are in the tables); the load of this item and
        //    the read-out of bc's previous contents complete
        if (tid >= 32 && tid < 40) cp_async_wait_all();
        scan_phase<EB>(rp, V);
        if (tid == 0) bulk_wait_read0();
        mbar_wait(&ctl->bar[bi], ctl->ph[bi]);
        __syncthreads();
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 1] = clock64();
        const bool placed = ctl->defer == 0;
        // 3. placement bi -> bc (column layout)
        if (placed) place_phase<EB, NARROW>(V, kw, bi, bc);
        __syncthreads();
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 2] = clock64();
        // 4. partners
        if (placed) partner_phase<EB>(rp, V);
        __syncthreads();
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 3] = clock64();
        // 5. Fisher-Yates bc -> bi (warps 0..7) | draws + counts of the next
        //    item and the search of the one after it (warps 8..31)
        if (tid < XFYT) {
            if (placed) {
                uint32_t fyn = fy_phase<EB>(rp, V, bi, bc);
                for (int o = 16; o > 0; o >>= 1) fyn += __shfl_xor_sync(0xFFFFFFFFu, fyn, o);
                if ((tid & 31u) == 0 && fyn) atomicAdd(&ctl->st_fy, (unsigned long long)fyn);
            }
            if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 4] = clock64();
        } else {
            const XItem nx = ctl->nxt;
            if (nx.valid) draw_count_phase<EB, NARROW>(rp, V, nx, lvl, XFYT / 32, XW - XFYT / 32);
            if (tid == XFYT) ctl->nxt2 = nx.valid ? find_next<EB>(rp, lp, nchild, ctl->cursor) : XItem{};
        }
        __syncthreads();
        if (dbg) rp.hdr->clk[ctl->dbg_it * 6 + 5] = clock64();
        // 6. store bi (aligned body: bulk async copy; head/tail words by threads
        //    32..95), load the next item into bc (free again)
        if (placed) {
            const uint64_t x0 = ctl->cur.start * EB, x1 = (ctl->cur.start + ctl->cur.len) * EB;
            const uint64_t fl = x0 & ~15ull;
            const uint64_t A0 = (x0 + 15) & ~15ull, B0 = x1 & ~15ull;
            const bool body = B0 > A0;
            unsigned char* ob = V.buf(bi);
            if (tid == 0 && body) {
                fence_proxy_async();
                bulk_s2g(rp.buf0 + A0, ob + (A0 - fl), (uint32_t)(B0 - A0));
                bulk_commit();
            }
            const uint64_t hEnd = body ? A0 : x1;
            const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
            const uint64_t tBeg = body ? B0 : x1;
            const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
            if (tid >= 32 && tid - 32 < nh)
                *reinterpret_cast<uint32_t*>(rp.buf0 + x0 + 4 * (tid - 32)) =
                    *reinterpret_cast<const uint32_t*>(ob + (x0 - fl) + 4 * (tid - 32));
            else if (tid >= 64 && tid - 64 < nt)
                *reinterpret_cast<uint32_t*>(rp.buf0 + tBeg + 4 * (tid - 64)) =
                    *reinterpret_cast<const uint32_t*>(ob + (tBeg - fl) + 4 * (tid - 64));
        }
        __syncthreads();  // head/tail words of the store are out
        const XItem nx = ctl->nxt;
        if (nx.valid && (tid == 0 || (tid >= 32 && tid < 40))) issue_load<EB>(V, nx, src, bc);
        if (tid == 0) {
            ctl->dbg_it++;
            ctl->ph[bi] ^= 1u;
            if (placed) ctl->st_fin += ctl->cur.len;
        }
        __syncthreads();
        if (tid == 0) {
            ctl->cur = ctl->nxt;
            ctl->nxt = ctl->nxt2;
            ctl->defer = 0;
        }
        __syncthreads();
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
        ctl->defer = 0;
        ctl->ph[0] = ctl->ph[1] = 0;
        ctl->dbg_it = 0;
        ctl->st_fin = 0;
        ctl->st_fy = 0;
        mbar_init(&ctl->bar[0], 1);
        mbar_init(&ctl->bar[1], 1);
        fence_mbar_init();
        ctl->cur = find_next<EB>(rp, lp, nchild, ctl->cursor);
        ctl->nxt.valid = 0;
        ctl->nxt2.valid = 0;
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
