// Kernel templates of the fused finish (instantiated per element size in
// kernels_finish_eb{4,8,16}.cu; dispatch in kernels_finish.cu).
//
// Fused finish: every segment of at most S_fuse elements is finished by one
// CTA in a single HBM round trip -- all of its remaining scatter levels run
// in shared memory (same draws, same stable order as the HBM levels), every
// leaf (<= L elements) is Fisher-Yates'd (Fig. 1), and the
// finished segment goes back to ptr with one bulk async store.
//
// One CTA of 1024 threads per SM, two data buffers in shared memory: the
// item arrives in IN (bulk async copy), the stable scatter writes it to OUT,
// and as soon as IN has been consumed the next item's copy is issued, so the
// load overlaps this item's Fisher-Yates phase and store.  Every
// shared-memory pointer is derived from the one extern array `fsm`, so all
// accesses compile to LDS/STS/ATOMS.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char fsm[];

constexpr int NTF = 1024;                       // threads per finish CTA
constexpr uint32_t kUnit = kFinishBucketGroup;  // children per work unit

// Warps that rank: all 32 while their per-warp counter tables stay small
// (Wr * k/2 words <= 4096), fewer for large k.
__host__ __device__ inline uint32_t finish_rank_warps(uint32_t k) {
    const uint32_t kw = (k + 1) / 2 > 0 ? (k + 1) / 2 : 1;
    const uint32_t w = 4096u / kw;
    return w > 32u ? 32u : (w < 1 ? 1u : w);
}

struct Item {
    uint64_t start;
    uint32_t len;
    uint32_t level;
    uint64_t origin;
    uint64_t key;
};

// Per-CTA control block (shared memory offset 0): iterator state and the
// current/next item, written by warp 0 and read by everyone.
struct FinCtl {
    Item items[2];
    uint32_t have[2];
    uint32_t phase;      // mbarrier phase of the IN buffer
    uint32_t nfront;     // children queued for the next in-smem level
    uint64_t u, units;   // iterator: work-unit cursor / count
    uint32_t b, bend;    // iterator: child cursor within the unit
    uint64_t seg_start, seg_origin, seg_key;
    uint64_t ub[kUnit + 1];  // unit child boundaries (relative to seg_start)
    uint64_t rec;            // item record index (defer mode)
    uint32_t dbg_it;         // items processed by CTA 0 (phase clocks, SHUF_DBG=2)
    unsigned long long st_finished, st_smem[32];
};

struct FinishLayout {
    uint32_t in, out, draws, C, bst, wsum, front0, front1, bar, total;
};

// stream: the single-buffer layout of k_finish_stream (the item's first
// in-smem level reads it straight from the level's output buffer: no IN).
__host__ __device__ inline FinishLayout finish_layout(uint32_t S, uint32_t eb, uint32_t k, bool stream = false) {
    FinishLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    take(sizeof(FinCtl));  // offset 0
    f.in = take(stream ? 16u : S * eb + 32);
    f.out = take(S * eb + 32);
    f.draws = take(2 * S + 64);  // bucket draws (u8 / u16)
    f.C = take(finish_rank_warps(k) * ((k + 1) / 2) * 4);
    f.bst = take((k + 1) * 4);
    f.wsum = take((NTF / 32 + 1) * 4);
    f.front0 = take(kFrontierCap * 4);
    f.front1 = take(kFrontierCap * 4);
    f.bar = take(16);
    f.total = off;
    return f;
}


// ------------------------------------------------------ smem accessors ----
struct Fin {
    FinishLayout f;
    __device__ __forceinline__ explicit Fin(const RunParams& rp) : f(finish_layout(rp.S_fuse, rp.eb, rp.k)) {}
    __device__ __forceinline__ Fin(const RunParams& rp, bool stream)
        : f(finish_layout(stream ? rp.S_stream : rp.S_fuse, rp.eb, rp.k, stream)) {}
    __device__ __forceinline__ FinCtl* ctl() const { return reinterpret_cast<FinCtl*>(fsm); }
    __device__ __forceinline__ unsigned char* in() const { return fsm + f.in; }
    __device__ __forceinline__ unsigned char* out() const { return fsm + f.out; }
    __device__ __forceinline__ unsigned char* draws() const { return fsm + f.draws; }
    __device__ __forceinline__ uint32_t* C() const { return reinterpret_cast<uint32_t*>(fsm + f.C); }
    __device__ __forceinline__ uint32_t* bst() const { return reinterpret_cast<uint32_t*>(fsm + f.bst); }
    __device__ __forceinline__ uint32_t* wsum() const { return reinterpret_cast<uint32_t*>(fsm + f.wsum); }
    __device__ __forceinline__ uint32_t* front(uint32_t i) const {
        return reinterpret_cast<uint32_t*>(fsm + (i ? f.front1 : f.front0));
    }
    __device__ __forceinline__ uint64_t* bar() const { return reinterpret_cast<uint64_t*>(fsm + f.bar); }
};

__device__ __forceinline__ bool item_permutes(const RunParams& rp, uint32_t len, uint32_t level) {
    const bool leaf = len <= rp.L;
    return (!leaf && level < rp.max_levels) || (leaf && rp.run_leaves && len >= 2);
}

// ---- load / store of one item (aligned body by bulk copy, head/tail words).
// Element i of an item lives at byte ((start*EB) & 15) + i*EB of a buffer,
// so the aligned body maps to a 16-byte-aligned shared address.
template <int EB>
__device__ __forceinline__ void item_load(const Item& it, const unsigned char* src, unsigned char* buf, uint64_t* bar) {
    const uint32_t tid = threadIdx.x;
    const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
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

template <int EB>
__device__ __forceinline__ void item_store(const Item& it, unsigned char* dst, const unsigned char* buf) {
    const uint32_t tid = threadIdx.x;
    fence_proxy_async();  // every thread that wrote buf orders its writes before the bulk store
    __syncthreads();
    const uint64_t x0 = it.start * EB, x1 = (it.start + it.len) * EB;
    const uint64_t fl = x0 & ~15ull;
    const uint64_t A = (x0 + 15) & ~15ull, B = x1 & ~15ull;
    const bool body = B > A;
    if (tid == 0 && body) {
        fence_proxy_async();
        bulk_s2g(dst + A, buf + (A - fl), (uint32_t)(B - A));
        bulk_commit();
    }
    const uint64_t hEnd = body ? A : x1;
    const uint32_t nh = (uint32_t)((hEnd - x0) >> 2);
    const uint64_t tBeg = body ? B : x1;
    const uint32_t nt = (uint32_t)((x1 - tBeg) >> 2);
    if (tid >= 32 && tid - 32 < nh)
        *reinterpret_cast<uint32_t*>(dst + x0 + 4 * (tid - 32)) =
            *reinterpret_cast<const uint32_t*>(buf + (x0 - fl) + 4 * (tid - 32));
    else if (tid >= 64 && tid - 64 < nt)
        *reinterpret_cast<uint32_t*>(dst + tBeg + 4 * (tid - 64)) =
            *reinterpret_cast<const uint32_t*>(buf + (tBeg - fl) + 4 * (tid - 64));
}

// ---------------------------------------------------- one smem level ----
// Stable scatter of src[a .. a+m) into dst[a .. a+m) (element a at problem
// position P0a).  Pass 1 counts buckets per warp; the counters become
// (bucket, warp) bases; pass 2 re-walks the same rounds and takes each
// element's slot with one ordered shared atomic on the base (block_ops.cuh).
// Warp w owns elements [w*q, (w+1)*q); its round r is w*q + 32r + lane.
// bst gets the bucket starts (relative to a).
template <int EB, bool NARROW, bool ORD>
__device__ __forceinline__ void smem_level(const RunParams& rp, const Fin& F, const unsigned char* src,
                                           unsigned char* dst, uint32_t a, uint32_t m, uint64_t P0a, uint32_t level,
                                           PhiloxKey key, bool wait_in) {
    using E = typename ElemT<EB>::type;
    using D = typename std::conditional<NARROW, unsigned char, uint16_t>::type;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t Wr = finish_rank_warps(k);
    const DrawView dv = draws_to_smem<NTF>(F.draws(), P0a, m, key, level, rp.bp);
    uint32_t* C = F.C();
    for (uint32_t i = tid; i < Wr * kw; i += NTF) C[i] = 0;
    FinCtl* ctl = F.ctl();
    if (wait_in) mbar_wait(F.bar(), ctl->phase);
    __syncthreads();
    if (wait_in && tid == 0) ctl->phase ^= 1u;
    const uint32_t q = (((m + Wr - 1) / Wr) + 31u) & ~31u;
    const uint32_t e0 = warp * q + lane;
    const uint32_t lim = (warp < Wr && e0 < m) ? min(m - e0, q - lane) : 0u;  // round r valid iff 32r < lim
    // per-lane bases, computed once; draw offset of position a = P0a mod group
    const uint32_t doff = (uint32_t)(P0a & (NARROW ? 15u : 7u));
    const D* dp = reinterpret_cast<const D*>(fsm + F.f.draws) + doff + e0;
    const E* sp = reinterpret_cast<const E*>(src) + a + e0;
    E* D0 = reinterpret_cast<E*>(dst) + a;
    uint32_t* Cw = C + warp * kw;
    // Rounds are warp-uniform loops (bound q) with the per-lane validity as a
    // predicate (an invalid lane adds 0), so every round is exactly one warp
    // instruction per atomic: the ordered-atomic ranking relies on lane
    // order within an instruction and on program order between rounds.
    if (ORD) {
        if (warp < Wr) {
#pragma unroll 4
            for (uint32_t o = 0; o < q; o += 32) {
                const bool valid = o < lim;
                // an invalid lane may sit past the draws of this range: force bucket 0
                const uint32_t b = valid ? (uint32_t)dp[o] : 0u;
                atomicAdd(&Cw[b >> 1], valid ? (1u << ((b & 1u) << 4)) : 0u);
            }
        }
    } else if (warp < Wr) {  // documented path: match-based counts, whole warp per round
        for (uint32_t o = 0; o < q; o += 32) {
            const bool valid = o < lim;
            const uint32_t b = valid ? (uint32_t)dp[o] : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
            if (valid && (peers & lanemask_lt()) == 0)
                atomicAdd(&Cw[b >> 1], (uint32_t)__popc(peers) << ((b & 1u) << 4));
        }
    }
    __syncthreads();
    scan_counters<NTF>(C, Wr, k, F.bst(), F.wsum());
    if (ORD) {
        if (warp < Wr) {
#pragma unroll 4
            for (uint32_t o = 0; o < q; o += 32) {
                const bool valid = o < lim;
                const uint32_t b = valid ? (uint32_t)dp[o] : 0u;
                const uint32_t sh = (b & 1u) << 4;
                // predicated: an invalid lane's address may lie past the shared window
                const E x = valid ? sp[o] : E{};
                const uint32_t slot = (atomicAdd(&Cw[b >> 1], valid ? (1u << sh) : 0u) >> sh) & 0xFFFFu;
                if (valid) D0[slot] = x;
            }
        }
    } else if (warp < Wr) {
        for (uint32_t o = 0; o < q; o += 32) {
            const bool valid = o < lim;
            const uint32_t b = valid ? (uint32_t)dp[o] : 0u;
            const uint32_t slot = warp_rank(Cw, b, valid, false);
            if (valid) D0[slot] = sp[o];
        }
    }
    if (tid == 0) {
        if (level < 32) ctl->st_smem[level] += m;
        else atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[level], (unsigned long long)m);
    }
    __syncthreads();
}

// After a level over [a, a+m) of `el`: FY the children that are leaves (one
// thread per leaf), queue the longer ones for the next level (ctl->nfront).
template <int EB>
__device__ __forceinline__ void handle_children(const RunParams& rp, const Fin& F, unsigned char* el, uint32_t a,
                                                uint32_t m, uint64_t P0, uint32_t level, PhiloxKey key,
                                                uint32_t* fnext, uint32_t& fy_local) {
    const uint32_t* bst = F.bst();
    for (uint32_t b = threadIdx.x; b < rp.k; b += NTF) {
        const uint32_t ca = a + bst[b], cm = bst[b + 1] - bst[b];
        if (cm <= rp.L) {
            if (rp.run_leaves && cm >= 2) {
                fy_leaf<EB>(el, ca, cm, P0 + ca, key);
                fy_local += cm;
            }
        } else if (level + 1 < rp.max_levels) {
            const uint32_t slot = atomicAdd(&F.ctl()->nfront, 1u);
            fnext[slot] = ca | (cm << 16);
        }
    }
}

// 1 if some child of the last level is longer than L (all threads call).
__device__ __forceinline__ bool any_big_child(const RunParams& rp, const Fin& F) {
    const uint32_t* bst = F.bst();
    bool big = false;
    for (uint32_t b = threadIdx.x; b < rp.k; b += NTF) big |= (bst[b + 1] - bst[b] > rp.L);
    return __syncthreads_or(big) != 0;
}

// Process the item whose data is (arriving) in IN; it leaves through OUT (or
// IN for leaf-only items).  Issues the load of `next` into IN as soon as IN
// is free.
template <int EB, bool NARROW, bool ORD>
__device__ __forceinline__ void process_item(const RunParams& rp, const Fin& F, const Item& it, const Item* next,
                                             const unsigned char* src, uint32_t& fy_local) {
    using E = typename ElemT<EB>::type;
    const uint32_t tid = threadIdx.x;
    const uint32_t off = (uint32_t)((it.start * EB) & 15u);
    unsigned char* in = F.in() + off;
    unsigned char* out = F.out() + off;
    const PhiloxKey key = make_key(it.key);
    const uint64_t P0 = it.start - it.origin;
    const uint32_t m = it.len;
    const bool leaf = m <= rp.L;
    FinCtl* ctl = F.ctl();
    if (tid == 0) ctl->st_finished += m;
    const bool dbg = (rp.dbg & 2u) && blockIdx.x == 0 && tid == 0 && ctl->dbg_it < 40;
    long long* clk = rp.hdr->clk + (dbg ? ctl->dbg_it * 6 : 0);
    if (dbg) clk[0] = clock64();
    if (!leaf && it.level < rp.max_levels) {
        // OUT was last read by the previous item's bulk store
        if (tid == 0) bulk_wait_read0();
        smem_level<EB, NARROW, ORD>(rp, F, in, out, 0, m, P0, it.level, key, true);
        if (dbg) clk[1] = clock64();
        const bool big = any_big_child(rp, F);
        const bool deep = big && it.level + 1 < rp.max_levels;
        if (!deep && next) item_load<EB>(*next, src, F.in(), F.bar());  // IN is free: overlap the next load
        if (tid == 0) {
            ctl->nfront = 0;
            if (rp.defer && !big) ctl->rec = atomicAdd((unsigned long long*)&rp.hdr->nitems, 1ull);
        }
        __syncthreads();
        if (rp.defer && !big) {
            // every child is a leaf: record the item; the leaf kernel runs Fisher-Yates on them
            unsigned char* r = rp.items + ctl->rec * item_rec_stride(rp.k);
            if (tid == 0) {
                reinterpret_cast<uint64_t*>(r)[0] = it.start;
                reinterpret_cast<uint64_t*>(r)[1] = it.origin;
                reinterpret_cast<uint64_t*>(r)[2] = it.key;
            }
            for (uint32_t b = tid; b <= rp.k; b += NTF) reinterpret_cast<uint16_t*>(r + 24)[b] = (uint16_t)F.bst()[b];
        } else {
            if (dbg) clk[2] = clock64();
            handle_children<EB>(rp, F, out, 0, m, P0, it.level, key, F.front(0), fy_local);
        }
        __syncthreads();
        if (dbg) clk[3] = clock64();
        uint32_t nf = ctl->nfront, cur = 0, lv = it.level + 1;
        __syncthreads();
        while (nf > 0) {  // deeper in-smem levels (rare when S_fuse / k << L): OUT -> IN -> OUT
            if (tid == 0) ctl->nfront = 0;
            __syncthreads();
            for (uint32_t f = 0; f < nf; ++f) {
                const uint32_t ent = F.front(cur)[f];
                const uint32_t a = ent & 0xFFFFu, mm = ent >> 16;
                smem_level<EB, NARROW, ORD>(rp, F, out, in, a, mm, P0 + a, lv, key, false);
                for (uint32_t x = tid; x < mm; x += NTF)
                    reinterpret_cast<E*>(out)[a + x] = reinterpret_cast<const E*>(in)[a + x];
                __syncthreads();
                handle_children<EB>(rp, F, out, a, mm, P0, lv, key, F.front(cur ^ 1u), fy_local);
                __syncthreads();
            }
            nf = ctl->nfront;
            cur ^= 1u;
            ++lv;
            __syncthreads();
        }
        if (deep && next) item_load<EB>(*next, src, F.in(), F.bar());
        __syncthreads();
        item_store<EB>(it, rp.buf0, F.out());
        if (dbg) {
            clk[4] = clock64();
            ctl->dbg_it++;
        }
    } else {
        // leaf-only (or level-limited) item: in place in IN
        const bool fy = leaf && rp.run_leaves && m >= 2;
        mbar_wait(F.bar(), ctl->phase);
        __syncthreads();
        if (tid == 0) {
            ctl->phase ^= 1u;
            if (fy) {
                fy_leaf<EB>(in, 0, m, P0, key);
                fy_local += m;
            }
        }
        __syncthreads();
        item_store<EB>(it, rp.buf0, F.in());
        if (next) {
            if (tid == 0) bulk_wait_read0();  // IN must be read out before it is reloaded
            __syncthreads();
            item_load<EB>(*next, src, F.in(), F.bar());
        }
    }
}

__device__ __forceinline__ void fin_init(const Fin& F) {
    if (threadIdx.x == 0) {
        mbar_init(F.bar(), 1);
        fence_mbar_init();
        FinCtl* c = F.ctl();
        c->phase = 0;
        c->dbg_it = 0;
        c->st_finished = 0;
        for (int i = 0; i < 32; ++i) c->st_smem[i] = 0;
    }
}

// Item loop.  Warp 0 advances the iterator (state in the control block) and
// publishes items; everyone reads the current item from smem.
template <int EB, bool NARROW, bool ORD, class It>
__device__ __forceinline__ void run_items(const RunParams& rp, const Fin& F, const It& iter, const unsigned char* src) {
    const uint32_t tid = threadIdx.x;
    FinCtl* ctl = F.ctl();
    if (tid < 32) iter.next(ctl, 0);
    __syncthreads();
    if (!ctl->have[0]) return;
    uint32_t fy_local = 0;
    item_load<EB>(ctl->items[0], src, F.in(), F.bar());
    for (uint32_t t = 0;; ++t) {
        const uint32_t slot = t & 1u;
        if (tid < 32) iter.next(ctl, slot ^ 1u);
        __syncthreads();
        const Item cur = ctl->items[slot];
        const bool hn = ctl->have[slot ^ 1u] != 0;
        process_item<EB, NARROW, ORD>(rp, F, cur, hn ? &ctl->items[slot ^ 1u] : nullptr, src, fy_local);
        if (!hn) break;
    }
    // flush the measurement counters: one global atomic per warp / per CTA
    for (int o = 16; o > 0; o >>= 1) fy_local += __shfl_xor_sync(0xFFFFFFFFu, fy_local, o);
    if ((tid & 31u) == 0 && fy_local) atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)fy_local);
    if (tid == 0) {
        atomicAdd((unsigned long long*)&rp.hdr->finished, ctl->st_finished);
        for (uint32_t l = 0; l < 32; ++l)
            if (ctl->st_smem[l]) atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[l], ctl->st_smem[l]);
        bulk_wait0();
    }
}

// Children of the level-l segments (in the level's output buffer).  Called
// by all 32 lanes of warp 0; lane 0 publishes items[slot] / have[slot].
struct ChildIter {
    const RunParams* rp;
    const LevelParams* lp;
    uint32_t groups;
    bool stream = false;  // k_finish_stream: the children with S_fuse < len <= S_stream
    __device__ __forceinline__ void load_unit(FinCtl* ctl) const {  // warp 0, all lanes
        const uint32_t lane = threadIdx.x & 31u;
        const SegDesc sg = lp->segs[(uint32_t)(ctl->u / groups)];
        const uint32_t b0 = (uint32_t)(ctl->u % groups) * kUnit;
        const uint32_t bend = min(rp->k, b0 + kUnit);
        const uint64_t base0 = lp->prefix[sg.cbase];
        if (lane <= bend - b0) {
            const uint32_t b = b0 + lane;
            ctl->ub[lane] = (b < rp->k) ? lp->prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0 : sg.len;
        }
        if (lane == 0) {
            ctl->b = b0;
            ctl->bend = bend;
            ctl->seg_start = sg.start;
            ctl->seg_origin = sg.origin;
            ctl->seg_key = sg.key;
        }
        __syncwarp();
    }
    __device__ __forceinline__ void next(FinCtl* ctl, uint32_t slot) const {  // warp 0, all lanes
        const uint32_t lane = threadIdx.x & 31u;
        const uint32_t lvl = lp->level + 1;
        while (ctl->u < ctl->units) {
            const uint32_t b0 = (uint32_t)(ctl->u % groups) * kUnit;
            for (uint32_t b = ctl->b; b < ctl->bend; ++b) {
                const uint64_t s0 = ctl->ub[b - b0], len = ctl->ub[b - b0 + 1] - s0;
                if (stream) {
                    if (len <= rp->S_fuse || len > rp->S_stream || lvl >= rp->max_levels) continue;
                } else {
                    if (len == 0 || len > rp->S_fuse) continue;
                    if (rp->leafk && len <= rp->L) continue;  // the leaf kernel's
                    if (lp->dst == rp->buf0 && !item_permutes(*rp, (uint32_t)len, lvl)) continue;
                    // children finished by k_finish_fast carry flag 0
                    if (rp->fast && rp->flags[(ctl->u / groups) * rp->k + b] == 0) continue;
                }
                __syncwarp();
                if (lane == 0) {
                    Item& it = ctl->items[slot];
                    it.start = ctl->seg_start + s0;
                    it.len = (uint32_t)len;
                    it.level = lvl;
                    it.origin = ctl->seg_origin;
                    it.key = ctl->seg_key;
                    ctl->have[slot] = 1;
                    ctl->b = b + 1;
                }
                __syncwarp();
                return;
            }
            __syncwarp();
            if (lane == 0) ctl->u += gridDim.x;
            __syncwarp();
            if (ctl->u < ctl->units) load_unit(ctl);
        }
        __syncwarp();
        if (lane == 0) ctl->have[slot] = 0;
        __syncwarp();
    }
};

// The level's fused list (k_plan): child indices c = s*k + b with
// L < len <= S_fuse (the leaf kernel takes the shorter ones).
struct ListIter {
    const RunParams* rp;
    const LevelParams* lp;
    __device__ __forceinline__ void next(FinCtl* ctl, uint32_t slot) const {  // warp 0, all lanes
        const uint32_t lane = threadIdx.x & 31u;
        // 32 entries of this CTA's stride sequence at once: the first one not
        // taken by k_finish_fast (flag 0) is the next item
        uint64_t u = ctl->u;
        uint32_t c = 0;
        bool found = false;
        while (u < ctl->units) {
            const uint64_t ul = u + (uint64_t)lane * gridDim.x;
            const uint32_t cl = ul < ctl->units ? rp->fused[ul] : 0u;
            const bool want = ul < ctl->units && !(rp->fast && rp->flags[cl] == 0);
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, want);
            if (bal) {
                const uint32_t f = __ffs(bal) - 1;
                c = __shfl_sync(0xFFFFFFFFu, cl, f);
                u += (uint64_t)(f + 1) * gridDim.x;
                found = true;
                break;
            }
            u += 32ull * gridDim.x;
        }
        __syncwarp();
        if (lane == 0) {
            ctl->u = u;
            ctl->have[slot] = 0;
            const uint32_t k = rp->k;
            if (found) {
                const SegDesc sg = lp->segs[c / k];
                const uint32_t b = c % k;
                const uint64_t base0 = lp->prefix[sg.cbase];
                const uint64_t s0 = lp->prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
                const uint64_t s1 = (b + 1 < k) ? lp->prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
                Item& it = ctl->items[slot];
                it.start = sg.start + s0;
                it.len = (uint32_t)(s1 - s0);
                it.level = lp->level + 1;
                it.origin = sg.origin;
                it.key = sg.key;
                ctl->have[slot] = 1;
            }
        }
        __syncwarp();
    }
};

template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(NTF, 1) k_finish_children(RunParams rp, LevelParams lp) {
    if (rp.max_fused) {  // iterate the fused list
        const uint64_t units = lp.ctr->nfuse;
        if (blockIdx.x >= units) return;
        const Fin F(rp);
        fin_init(F);
        if (threadIdx.x == 0) {
            F.ctl()->u = blockIdx.x;
            F.ctl()->units = units;
        }
        __syncthreads();
        ListIter iter{&rp, &lp};
        run_items<EB, NARROW, ORD>(rp, F, iter, lp.dst);
        return;
    }
    const uint32_t groups = (rp.k + kUnit - 1) / kUnit;
    const uint64_t units = (uint64_t)lp.ctr->nseg * groups;
    if (blockIdx.x >= units) return;
    const Fin F(rp);
    fin_init(F);
    ChildIter iter{&rp, &lp, groups};
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            F.ctl()->u = blockIdx.x;
            F.ctl()->units = units;
        }
        __syncwarp();
        iter.load_unit(F.ctl());
    }
    __syncthreads();
    run_items<EB, NARROW, ORD>(rp, F, iter, lp.dst);
}

// Children of an in-place level batch (kernels_inplace.cu): bucket starts
// from the batch's table S, in place in ptr.  Same protocol as ChildIter.
struct IpChildIter {
    const RunParams* rp;
    const IpParams* ip;
    uint32_t groups;
    __device__ __forceinline__ void load_unit(FinCtl* ctl) const {  // warp 0, all lanes
        const uint32_t lane = threadIdx.x & 31u, k = rp->k;
        const uint32_t s = (uint32_t)(ctl->u / groups);
        const uint32_t b0 = (uint32_t)(ctl->u % groups) * kUnit;
        const uint32_t bend = min(k, b0 + kUnit);
        if (lane <= bend - b0) ctl->ub[lane] = ip->S[(uint64_t)s * (k + 1) + b0 + lane];
        if (lane == 0) {
            ctl->b = b0;
            ctl->bend = bend;
            ctl->seg_start = ip->segs[s].start;
            ctl->seg_origin = 0;
            ctl->seg_key = rp->seed;  // K(seed, 0) (D2)
        }
        __syncwarp();
    }
    __device__ __forceinline__ void next(FinCtl* ctl, uint32_t slot) const {  // warp 0, all lanes
        const uint32_t lane = threadIdx.x & 31u;
        const uint32_t lvl = ip->level + 1;
        while (ctl->u < ctl->units) {
            const uint32_t b0 = (uint32_t)(ctl->u % groups) * kUnit;
            for (uint32_t b = ctl->b; b < ctl->bend; ++b) {
                const uint64_t s0 = ctl->ub[b - b0], len = ctl->ub[b - b0 + 1] - s0;
                if (len == 0 || len > rp->S_fuse) continue;
                if (rp->leafk && len <= rp->L) continue;
                if (!item_permutes(*rp, (uint32_t)len, lvl)) continue;
                // children taken by k_finish_fast_ip carry flag 0
                if (rp->fast && rp->flags[(ctl->u / groups) * rp->k + b] == 0) continue;
                __syncwarp();
                if (lane == 0) {
                    Item& it = ctl->items[slot];
                    it.start = ctl->seg_start + s0;
                    it.len = (uint32_t)len;
                    it.level = lvl;
                    it.origin = ctl->seg_origin;
                    it.key = ctl->seg_key;
                    ctl->have[slot] = 1;
                    ctl->b = b + 1;
                }
                __syncwarp();
                return;
            }
            __syncwarp();
            if (lane == 0) ctl->u += gridDim.x;
            __syncwarp();
            if (ctl->u < ctl->units) load_unit(ctl);
        }
        __syncwarp();
        if (lane == 0) ctl->have[slot] = 0;
        __syncwarp();
    }
};

template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(NTF, 1) k_finish_ipchildren(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    const uint32_t groups = (rp.k + kUnit - 1) / kUnit;
    const uint64_t units = (uint64_t)ip.nseg * groups;
    if (blockIdx.x >= units) return;
    const Fin F(rp);
    fin_init(F);
    IpChildIter iter{&rp, &ip, groups};
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            F.ctl()->u = blockIdx.x;
            F.ctl()->units = units;
        }
        __syncwarp();
        iter.load_unit(F.ctl());
    }
    __syncthreads();
    run_items<EB, NARROW, ORD>(rp, F, iter, rp.buf0);
}

// Segments given by offsets (segmented mode at level 0, or the single problem
// when n <= S_fuse).  They sit in ptr.
struct SegIter {
    const RunParams* rp;
    const uint64_t* off;
    // warp 0, all lanes: the lanes look at the CTA's next 32 segments at once (in the segmented mode
    // most segments are the leaf kernel's; one lane walking them paid two dependent global loads each)
    __device__ __forceinline__ void next(FinCtl* ctl, uint32_t slot) const {
        const uint32_t lane = threadIdx.x & 31u;
        uint64_t u = ctl->u;
        const uint64_t units = ctl->units;
        bool found = false;
        uint64_t si = 0, a = 0, b = 0;
        while (u < units) {
            const uint64_t s = u + (uint64_t)lane * gridDim.x;
            uint64_t sa = 0, sb = 0;
            bool ok = false;
            if (s < units) {
                sa = off[s];
                sb = off[s + 1];
                ok = sb > sa && sb - sa <= rp->S_fuse && !(rp->leafk && sb - sa <= rp->L) &&  // not the leaf kernel's
                     item_permutes(*rp, (uint32_t)(sb - sa), rp->first_level);
            }
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
            if (m) {
                const int f = __ffs(m) - 1;
                si = __shfl_sync(0xFFFFFFFFu, s, f);
                a = __shfl_sync(0xFFFFFFFFu, sa, f);
                b = __shfl_sync(0xFFFFFFFFu, sb, f);
                u = si + gridDim.x;
                found = true;
                break;
            }
            u += 32ull * gridDim.x;
        }
        __syncwarp();  // every lane has read ctl->u
        if (lane == 0) {
            ctl->u = u;
            ctl->have[slot] = found ? 1u : 0u;
            if (found) {
                Item& it = ctl->items[slot];
                it.start = a;
                it.len = (uint32_t)(b - a);
                it.level = rp->first_level;
                it.origin = rp->shard ? 0ull - rp->seg_base : a;
                it.key = rp->shard ? rp->seed : rp->seed + si * 0x9E3779B97F4A7C15ull;  // K(seed, s) (D2)
            }
        }
        __syncwarp();
    }
};

template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(NTF, 1)
    k_finish_segments(RunParams rp, const uint64_t* __restrict__ off, uint64_t nsegs) {
    if (blockIdx.x >= nsegs) return;
    const Fin F(rp);
    fin_init(F);
    if (threadIdx.x == 0) {
        F.ctl()->u = blockIdx.x;
        F.ctl()->units = nsegs;
    }
    __syncthreads();
    SegIter iter{&rp, off};
    run_items<EB, NARROW, ORD>(rp, F, iter, rp.buf0);
}

// Single-buffer finish of the children with S_fuse < len <= S_stream (items
// too long for IN + OUT): the item's in-smem level reads its elements straight
// from the level's output buffer (coalesced, in position order) and places
// them into OUT; its children are leaves (the plan enables the stream only when
// len / k stays far below L), Fisher-Yates'd in OUT; OUT goes to
// ptr with one bulk store.  A child longer than L (not seen in any plan that
// enables the stream: > 12 sigma) latches SHUF_ERR_DEPTH.
template <int EB, bool NARROW, bool ORD>
__global__ void __launch_bounds__(NTF, 1) k_finish_stream(RunParams rp, LevelParams lp) {
    const uint32_t groups = (rp.k + kUnit - 1) / kUnit;
    const uint64_t units = (uint64_t)lp.ctr->nseg * groups;
    if (blockIdx.x >= units || lp.ctr->nstream == 0) return;
    const Fin F(rp, true);
    fin_init(F);
    ChildIter iter{&rp, &lp, groups};
    iter.stream = true;
    FinCtl* ctl = F.ctl();
    const uint32_t tid = threadIdx.x;
    if (tid < 32) {
        if (tid == 0) {
            ctl->u = blockIdx.x;
            ctl->units = units;
        }
        __syncwarp();
        iter.load_unit(ctl);
    }
    __syncthreads();
    uint32_t fy_local = 0;
    for (;;) {
        if (tid < 32) iter.next(ctl, 0);
        __syncthreads();
        if (!ctl->have[0]) break;
        const Item it = ctl->items[0];
        const uint32_t off = (uint32_t)((it.start * EB) & 15u);
        unsigned char* out = F.out() + off;
        const PhiloxKey key = make_key(it.key);
        const uint64_t P0 = it.start - it.origin;
        if (tid == 0) {
            ctl->st_finished += it.len;
            bulk_wait_read0();  // OUT was last read by the previous item's bulk store
        }
        __syncthreads();
        smem_level<EB, NARROW, ORD>(rp, F, lp.dst + it.start * EB, out, 0, it.len, P0, it.level, key, false);
        if (tid == 0) ctl->nfront = 0;
        __syncthreads();
        handle_children<EB>(rp, F, out, 0, it.len, P0, it.level, key, F.front(0), fy_local);
        __syncthreads();
        if (tid == 0 && ctl->nfront) atomicCAS(&rp.hdr->error, 0u, 5u /*SHUF_ERR_DEPTH*/);
        item_store<EB>(it, rp.buf0, F.out());  // (fences every writer, then one bulk store)
    }
    for (int o = 16; o > 0; o >>= 1) fy_local += __shfl_xor_sync(0xFFFFFFFFu, fy_local, o);
    if ((tid & 31u) == 0 && fy_local) atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)fy_local);
    if (tid == 0) {
        atomicAdd((unsigned long long*)&rp.hdr->finished, ctl->st_finished);
        for (uint32_t l = 0; l < 32; ++l)
            if (ctl->st_smem[l]) atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[l], ctl->st_smem[l]);
        bulk_wait0();
    }
}

// Debug level limit: children longer than S_fuse produced by the last level
// that ran are copied (unchanged) from the level's output buffer to ptr.
template <int EB>
__global__ void k_copy_big(RunParams rp, LevelParams lp) {
    using E = typename ElemT<EB>::type;
    const uint64_t nchild = (uint64_t)lp.ctr->nseg * rp.k;
    for (uint64_t i = blockIdx.x; i < nchild; i += gridDim.x) {
        const SegDesc sg = lp.segs[i / rp.k];
        const uint32_t b = (uint32_t)(i % rp.k);
        const uint64_t base0 = lp.prefix[sg.cbase];
        const uint64_t s0 = lp.prefix[sg.cbase + (uint64_t)b * sg.nchunks] - base0;
        const uint64_t s1 = (b + 1 < rp.k) ? lp.prefix[sg.cbase + (uint64_t)(b + 1) * sg.nchunks] - base0 : sg.len;
        if (s1 - s0 <= rp.S_fuse) continue;
        const E* s = reinterpret_cast<const E*>(lp.dst) + sg.start + s0;
        E* d = reinterpret_cast<E*>(rp.buf0) + sg.start + s0;
        for (uint64_t x = threadIdx.x; x < s1 - s0; x += blockDim.x) d[x] = s[x];
    }
}

}  // namespace shuf
