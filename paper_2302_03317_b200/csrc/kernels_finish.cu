// Fused finish: every segment of at most S_fuse elements is finished by one
// CTA in a single HBM round trip -- all of its remaining scatter levels run
// in shared memory (same draws, same stable order as the HBM levels), every
// leaf (<= L elements) is Fisher-Yates'd in place (Fig. 1), and
// the finished segment goes back to ptr with one bulk async store.
//
// Items are pipelined: while item t is processed in buffer t&1, item t+1 is
// already being loaded into the other buffer by the bulk-copy engine.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

constexpr int kFinThreads = 1024;
constexpr int kFinWarps = kFinThreads / 32;

template <int EB> struct FinCfg;
template <> struct FinCfg<4> { static constexpr uint32_t RMAX = 18; };
template <> struct FinCfg<8> { static constexpr uint32_t RMAX = 12; };
template <> struct FinCfg<16> { static constexpr uint32_t RMAX = 6; };

__host__ __device__ inline uint32_t finish_rank_warps(uint32_t k) {
    uint32_t w = 16384u / k;
    return w > (uint32_t)kFinWarps ? (uint32_t)kFinWarps : (w < 1 ? 1u : w);
}

__host__ __device__ inline uint32_t finish_rmax(uint32_t eb) {
    return eb == 4 ? FinCfg<4>::RMAX : (eb == 8 ? FinCfg<8>::RMAX : FinCfg<16>::RMAX);
}

struct FinishLayout {
    uint32_t buf[2], draws, C, bst, wsum, front0, front1, misc, bar, ctl, total;
};

__host__ __device__ inline FinishLayout finish_layout(uint32_t S, uint32_t eb, uint32_t k, uint32_t nbuf) {
    FinishLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    f.buf[0] = take(S * eb + 32);
    f.buf[1] = nbuf > 1 ? take(S * eb + 32) : f.buf[0];
    f.draws = take(draw_bytes(S));
    f.C = take(finish_rank_warps(k) * ((k + 1) / 2) * 4);
    f.bst = take((k + 1) * 4);
    f.wsum = take((kFinWarps + 1) * 4);
    f.front0 = take(kFrontierCap * 4);
    f.front1 = take(kFrontierCap * 4);
    f.misc = take(64);
    f.bar = take(16);
    f.ctl = take(256);
    f.total = off;
    return f;
}

uint32_t finish_smem_bytes(uint32_t S_fuse, uint32_t eb, uint32_t k, uint32_t nbuf) {
    return finish_layout(S_fuse, eb, k, nbuf).total;
}

uint32_t finish_max_elems(uint32_t eb, uint32_t k) { return finish_rmax(eb) * finish_rank_warps(k) * 32u; }

struct Item {
    uint64_t start;
    uint32_t len;
    uint32_t level;
    uint64_t origin;
    uint64_t key;
};

// Per-CTA control block in shared memory: the current and next item and the
// iterator state are kept here (written by thread 0) so that the 1024
// threads' registers stay free for the ranking rounds.
struct FinCtl {
    Item items[2];
    uint32_t have[2];
    uint64_t u, units;   // iterator: unit cursor / count
    uint32_t b, bend;    // iterator: bucket cursor within the unit
    uint32_t phase[2];   // mbarrier phase per buffer
};

struct FinCtx {
    unsigned char* sm;
    FinishLayout f;
    __device__ __forceinline__ unsigned char* buf(uint32_t i) const { return sm + f.buf[i]; }
    __device__ __forceinline__ unsigned char* draws() const { return sm + f.draws; }
    __device__ __forceinline__ uint32_t* C() const { return reinterpret_cast<uint32_t*>(sm + f.C); }
    __device__ __forceinline__ uint32_t* bst() const { return reinterpret_cast<uint32_t*>(sm + f.bst); }
    __device__ __forceinline__ uint32_t* wsum() const { return reinterpret_cast<uint32_t*>(sm + f.wsum); }
    __device__ __forceinline__ uint32_t* front(uint32_t i) const {
        return reinterpret_cast<uint32_t*>(sm + (i ? f.front1 : f.front0));
    }
    __device__ __forceinline__ uint32_t* misc() const { return reinterpret_cast<uint32_t*>(sm + f.misc); }
    __device__ __forceinline__ uint64_t* bar() const { return reinterpret_cast<uint64_t*>(sm + f.bar); }
    __device__ __forceinline__ FinCtl* ctl() const { return reinterpret_cast<FinCtl*>(sm + f.ctl); }
};

__device__ __forceinline__ bool item_permutes(const RunParams& rp, uint32_t len, uint32_t level) {
    const bool leaf = len <= rp.L;
    return (!leaf && level < rp.max_levels) || (leaf && rp.run_leaves && len >= 2);
}

// ---- load / store of one item (aligned body by bulk copy, head/tail words)
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

// Sequential Fisher-Yates (Fig. 1) on the elements el[a .. a+m) whose
// element 0 sits at problem-relative position P0: for i = m-1 .. 1,
// swap(i, fy(P0+i, i+1)).
template <int EB>
__device__ void fy_seq(unsigned char* el, uint32_t a, uint32_t m, uint64_t P0, PhiloxKey key) {
    using E = typename ElemT<EB>::type;
    E* A = reinterpret_cast<E*>(el) + a;
    uint64_t gcur = ~0ull;
    uint4 w = make_uint4(0, 0, 0, 0);
    for (uint32_t i = m; i-- > 1;) {
        const uint64_t P = P0 + i;
        const uint64_t g = P >> 3;
        if (g != gcur) {
            w = fy16_group_words(key, g);
            gcur = g;
        }
        const uint32_t j = fy16_from_lane(lane16(w, (uint32_t)(P & 7u)), key, P, i + 1);
        const E t = A[i];
        A[i] = A[j];
        A[j] = t;
    }
}

// One stable scatter level in shared memory over el[a .. a+m), element a at
// problem-relative position P0a: ranks in registers, then written back in
// place in bucket-major order.  Leaves bucket starts (relative to a) in bst.
template <int EB>
__device__ void smem_level(const RunParams& rp, const FinCtx& c, unsigned char* el, uint32_t a, uint32_t m, uint64_t P0a,
                           uint32_t level, PhiloxKey key, int wait_buf) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t RMAX = FinCfg<EB>::RMAX;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t k = rp.k, kw = (k + 1) >> 1;
    const uint32_t Wr = finish_rank_warps(k);
    const DrawView dv = draws_to_smem<kFinThreads>(c.draws(), P0a, m, key, level, rp.bp);
    uint32_t* C = c.C();
    for (uint32_t i = tid; i < Wr * kw; i += kFinThreads) C[i] = 0;
    if (wait_buf >= 0) mbar_wait(&c.bar()[wait_buf], c.ctl()->phase[wait_buf]);
    __syncthreads();
    if (wait_buf >= 0 && tid == 0) c.ctl()->phase[wait_buf] ^= 1u;
    const uint32_t q = (((m + Wr - 1) / Wr) + 31u) & ~31u;
    const uint32_t R = q >> 5;
    E* A = reinterpret_cast<E*>(el) + a;
    E v[RMAX];
    uint32_t rk[(RMAX + 1) / 2];  // two u16 ranks per register; buckets re-read from the draws
    uint32_t* Cw = C + warp * kw;
    const bool ordered = rp.rank_ordered != 0;
    if (warp < Wr) {
#pragma unroll
        for (uint32_t r = 0; r < RMAX; ++r) {
            if (r < R) {
                const uint32_t e = warp * q + r * 32 + lane;
                const bool valid = e < m;
                uint32_t b = 0;
                if (valid) {
                    v[r] = A[e];
                    b = dv.at(e);
                }
                const uint32_t rank = warp_rank(Cw, b, valid, ordered);
                if (r & 1u) rk[r >> 1] |= rank << 16;
                else rk[r >> 1] = rank;
            }
        }
    }
    __syncthreads();
    scan_counters<kFinThreads>(C, Wr, k, c.bst(), c.wsum());
    if (warp < Wr) {
#pragma unroll
        for (uint32_t r = 0; r < RMAX; ++r) {
            const uint32_t e = warp * q + r * 32 + lane;
            if (r < R && e < m) {
                const uint32_t b = dv.at(e);
                const uint32_t base = (Cw[b >> 1] >> ((b & 1u) << 4)) & 0xFFFFu;
                A[base + ((rk[r >> 1] >> ((r & 1u) << 4)) & 0xFFFFu)] = v[r];
            }
        }
    }
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->scattered_smem[level], (unsigned long long)m);
    __syncthreads();
}

// After smem_level over [a, a+m) at `level`: FY the children that are leaves,
// queue the others for level+1 (count in misc[0]).
template <int EB>
__device__ __forceinline__ void handle_children(const RunParams& rp, const FinCtx& c, unsigned char* el, uint32_t a,
                                                uint64_t P0, uint32_t level, PhiloxKey key, uint32_t* fnext) {
    const uint32_t* bst = c.bst();
    for (uint32_t b = threadIdx.x; b < rp.k; b += kFinThreads) {
        const uint32_t ca = a + bst[b], cm = bst[b + 1] - bst[b];
        if (cm <= rp.L) {
            if (rp.run_leaves && cm >= 2) {
                fy_seq<EB>(el, ca, cm, P0 + ca, key);
                atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)cm);
            }
        } else if (level + 1 < rp.max_levels) {
            const uint32_t slot = atomicAdd(&c.misc()[0], 1u);
            fnext[slot] = ca | (cm << 16);
        }
    }
}

// Process one loaded (or loading) item in buffer bi and store it to buf0.
template <int EB>
__device__ void process_item(const RunParams& rp, const FinCtx& c, const Item& it, uint32_t bi) {
    const uint32_t tid = threadIdx.x;
    unsigned char* el = c.buf(bi) + ((it.start * EB) & 15u);
    const PhiloxKey key = make_key(it.key);
    const uint64_t P0 = it.start - it.origin;
    const uint32_t m = it.len;
    const bool leaf = m <= rp.L;
    uint32_t* misc = c.misc();
    if (tid == 0) atomicAdd((unsigned long long*)&rp.hdr->finished, (unsigned long long)m);
    if (!leaf && it.level < rp.max_levels) {
        if (tid == 0) misc[0] = 0;
        smem_level<EB>(rp, c, el, 0, m, P0, it.level, key, (int)bi);
        handle_children<EB>(rp, c, el, 0, P0, it.level, key, c.front(0));
        __syncthreads();
        uint32_t nf = misc[0], cur = 0, lv = it.level + 1;
        __syncthreads();
        while (nf > 0) {  // deeper in-smem levels (rare when S_fuse / k << L)
            if (tid == 0) misc[0] = 0;
            __syncthreads();
            for (uint32_t f = 0; f < nf; ++f) {
                const uint32_t ent = c.front(cur)[f];
                const uint32_t a = ent & 0xFFFFu, mm = ent >> 16;
                smem_level<EB>(rp, c, el, a, mm, P0 + a, lv, key, -1);
                handle_children<EB>(rp, c, el, a, P0, lv, key, c.front(cur ^ 1u));
                __syncthreads();
            }
            nf = misc[0];
            cur ^= 1u;
            ++lv;
            __syncthreads();
        }
    } else {
        mbar_wait(&c.bar()[bi], c.ctl()->phase[bi]);
        __syncthreads();
        if (tid == 0) {
            c.ctl()->phase[bi] ^= 1u;
            if (leaf && rp.run_leaves && m >= 2) {
                fy_seq<EB>(el, 0, m, P0, key);
                atomicAdd((unsigned long long*)&rp.hdr->fy_elems, (unsigned long long)m);
            }
        }
    }
    __syncthreads();
    item_store<EB>(it, rp.buf0, c.buf(bi));
}

__device__ FinCtx make_fin_ctx(const RunParams& rp, unsigned char* sm) {
    FinCtx c;
    c.sm = sm;
    c.f = finish_layout(rp.S_fuse, rp.eb, rp.k, rp.fin_nbuf);
    if (threadIdx.x == 0) {
        mbar_init(&c.bar()[0], 1);
        mbar_init(&c.bar()[1], 1);
        fence_mbar_init();
        c.ctl()->phase[0] = c.ctl()->phase[1] = 0;
    }
    return c;
}

// Pipelined item loop.  Thread 0 advances the iterator (state in the control
// block) and publishes items; everyone reads the current item from smem.
template <int EB, class It>
__device__ void run_items(const RunParams& rp, const FinCtx& c, const It& iter, const unsigned char* src) {
    const uint32_t tid = threadIdx.x;
    FinCtl* ctl = c.ctl();
    if (tid == 0) ctl->have[0] = iter.next(ctl, ctl->items[0]) ? 1u : 0u;
    __syncthreads();
    if (!ctl->have[0]) return;
    item_load<EB>(ctl->items[0], src, c.buf(0), &c.bar()[0]);
    const uint32_t nbuf = rp.fin_nbuf;
    for (uint32_t t = 0;; ++t) {
        const uint32_t slot = t & 1u;
        if (tid == 0) ctl->have[slot ^ 1u] = iter.next(ctl, ctl->items[slot ^ 1u]) ? 1u : 0u;
        __syncthreads();
        const Item cur = ctl->items[slot];
        const bool hn = ctl->have[slot ^ 1u] != 0;
        const uint32_t bi = (nbuf > 1) ? slot : 0u;
        if (hn && nbuf > 1) {
            // buffer bi^1 was stored by item t-1: wait until that store has read it
            if (tid == 0) bulk_wait_read0();
            __syncthreads();
            item_load<EB>(ctl->items[slot ^ 1u], src, c.buf(bi ^ 1u), &c.bar()[bi ^ 1u]);
        }
        process_item<EB>(rp, c, cur, bi);
        if (!hn) break;
        if (nbuf == 1) {
            if (tid == 0) bulk_wait_read0();
            __syncthreads();
            item_load<EB>(ctl->items[slot ^ 1u], src, c.buf(0), &c.bar()[0]);
        }
    }
    if (tid == 0) bulk_wait0();
}

// Children of the level-l segments (in the level's output buffer).
struct ChildIter {
    const RunParams* rp;
    const LevelParams* lp;
    uint32_t groups;
    __device__ void load_unit(FinCtl* ctl) const {
        ctl->b = (uint32_t)(ctl->u % groups) * kFinishBucketGroup;
        ctl->bend = min(rp->k, ctl->b + kFinishBucketGroup);
    }
    __device__ bool next(FinCtl* ctl, Item& it) const {
        while (ctl->u < ctl->units) {
            const SegDesc sg = lp->segs[(uint32_t)(ctl->u / groups)];
            const uint64_t base0 = lp->prefix[sg.cbase];
            while (ctl->b < ctl->bend) {
                const uint32_t bb = ctl->b++;
                const uint64_t s0 = lp->prefix[sg.cbase + (uint64_t)bb * sg.nchunks] - base0;
                const uint64_t s1 =
                    (bb + 1 < rp->k) ? lp->prefix[sg.cbase + (uint64_t)(bb + 1) * sg.nchunks] - base0 : sg.len;
                const uint64_t len = s1 - s0;
                if (len == 0 || len > rp->S_fuse) continue;
                const uint32_t lvl = lp->level + 1;
                if (lp->dst == rp->buf0 && !item_permutes(*rp, (uint32_t)len, lvl)) continue;
                it.start = sg.start + s0;
                it.len = (uint32_t)len;
                it.level = lvl;
                it.origin = sg.origin;
                it.key = sg.key;
                return true;
            }
            ctl->u += gridDim.x;
            if (ctl->u < ctl->units) load_unit(ctl);
        }
        return false;
    }
};

template <int EB>
__global__ void __launch_bounds__(kFinThreads, 1) k_finish_children(RunParams rp, LevelParams lp) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t groups = (rp.k + kFinishBucketGroup - 1) / kFinishBucketGroup;
    const uint64_t units = (uint64_t)lp.ctr->nseg * groups;
    if (blockIdx.x >= units) return;
    const FinCtx c = make_fin_ctx(rp, sm);
    ChildIter iter;
    iter.rp = &rp;
    iter.lp = &lp;
    iter.groups = groups;
    if (threadIdx.x == 0) {
        c.ctl()->u = blockIdx.x;
        c.ctl()->units = units;
        iter.load_unit(c.ctl());
    }
    __syncthreads();
    run_items<EB>(rp, c, iter, lp.dst);
}

// Segments given by offsets (segmented mode at level 0, or the single problem
// when n <= S_fuse).  They sit in ptr.
struct SegIter {
    const RunParams* rp;
    const uint64_t* off;
    __device__ bool next(FinCtl* ctl, Item& it) const {
        while (ctl->u < ctl->units) {
            const uint64_t si = ctl->u;
            ctl->u += gridDim.x;
            const uint64_t a = off[si], b = off[si + 1];
            if (b <= a || b - a > rp->S_fuse) continue;
            if (!item_permutes(*rp, (uint32_t)(b - a), 0u)) continue;
            it.start = a;
            it.len = (uint32_t)(b - a);
            it.level = 0;
            it.origin = a;
            it.key = rp->seed + si * 0x9E3779B97F4A7C15ull;  // K(seed, s) (D2)
            return true;
        }
        return false;
    }
};

template <int EB>
__global__ void __launch_bounds__(kFinThreads, 1) k_finish_segments(RunParams rp, const uint64_t* __restrict__ off,
                                                                     uint64_t nsegs) {
    extern __shared__ __align__(16) unsigned char sm[];
    if (blockIdx.x >= nsegs) return;
    const FinCtx c = make_fin_ctx(rp, sm);
    SegIter iter;
    iter.rp = &rp;
    iter.off = off;
    if (threadIdx.x == 0) {
        c.ctl()->u = blockIdx.x;
        c.ctl()->units = nsegs;
    }
    __syncthreads();
    run_items<EB>(rp, c, iter, rp.buf0);
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

cudaError_t launch_finish_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k, rp.fin_nbuf);
    switch (rp.eb) {
    case 4: k_finish_children<4><<<grid, kFinThreads, smem, s>>>(rp, lp); break;
    case 8: k_finish_children<8><<<grid, kFinThreads, smem, s>>>(rp, lp); break;
    default: k_finish_children<16><<<grid, kFinThreads, smem, s>>>(rp, lp); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_copy_big(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid) {
    switch (rp.eb) {
    case 4: k_copy_big<4><<<grid, 256, 0, s>>>(rp, lp); break;
    case 8: k_copy_big<8><<<grid, 256, 0, s>>>(rp, lp); break;
    default: k_copy_big<16><<<grid, 256, 0, s>>>(rp, lp); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_finish_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                   cudaStream_t s, int grid) {
    const uint32_t smem = finish_smem_bytes(rp.S_fuse, rp.eb, rp.k, rp.fin_nbuf);
    switch (rp.eb) {
    case 4: k_finish_segments<4><<<grid, kFinThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    case 8: k_finish_segments<8><<<grid, kFinThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    default: k_finish_segments<16><<<grid, kFinThreads, smem, s>>>(rp, d_offsets, num_segments); break;
    }
    return cudaGetLastError();
}

cudaError_t configure_finish(uint32_t smem) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_finish_children<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_children<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_children<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_segments<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    if ((e = cudaFuncSetAttribute(k_finish_segments<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    return cudaFuncSetAttribute(k_finish_segments<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

cudaError_t occupancy_finish(uint32_t eb, uint32_t smem, int* blocks) {
    switch (eb) {
    case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<4>, kFinThreads, smem);
    case 8: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<8>, kFinThreads, smem);
    default: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k_finish_children<16>, kFinThreads, smem);
    }
}

}  // namespace shuf
