// The paper's own In-Place ScatterShuffle on the GPU (SURVEY 8(f) NEXT-2,
// DESIGN.md D10 and section 6.3): one IpSc per segment [a, a+m) longer than L
// at every level (Fig. 2), made deterministic by counter-based
// draws so that the result equals the oracle (oracle_ipsc_shuffle) bit for bit.
//
//   ParRoughScatter  the k equal buckets are halved
//     recursively to depth t = min(11, floor(log2(m / k^2))) (base case
//     N0 = k^2); heap node v, children 2v / 2v+1.  k_ipsc_rs runs
//     RoughScatter on a leaf subtask (all staged) or, after
//     merging the two children bucket by bucket ("swapping the staged items of
//     the first half to the second half"), on an inner node.  One CTA
//     per node; only the staged starts s_i live in the node table (b_i and
//     e_i are the node's bucket bounds, recomputed from the split rule).
//   FineScatter  k_ipsc_fine, one CTA per segment: the
//     multinomial final sizes from R uniform draws, TwoSweep
//      boundary by boundary, and the stash shuffle.
//
// RoughScatter as a parallel computation.  A step draws a partner bucket j
// (a function of (node, step) only) and moves the element at s_0 (the
// "hand") to s_j, s_j++ (j = 0: the hand stays, s_0++).  So step t places
// the hand h_t at P_t = s_{j_t} + #{earlier steps with the same j}, and the
// next hand is the element found at Q_{t+1} = P_t (j_t != 0: swapped in) or
// P_t + 1 (j_t = 0: the next staged slot of bucket 0).  Every P_t and every
// Q_t is read before it is written and never read again, so a CTA runs NT
// steps at once: draws, per-bucket ranks (match_any within a warp + per-warp
// counts), the first step that fills a bucket (stop), all reads of the next
// hands, then all writes.  At the stop the last hand (if j != 0) lands at
// s_0.  This is the sequential RoughScatter, bit for bit.
//
// The stash shuffle.  "Compact the staged items into X[a..a+R), shuffle,
// undo the swaps" leaves every non-staged item where it was and
// gives the staged position p_t the item of p_{phi(t)}, phi the Fisher-Yates
// permutation of [0, R).  So Fisher-Yates runs directly on the virtual array
// V[t] = X[p_t] (p_t from the staged ranges), with the same draws: exact.  A
// CTA runs it in rounds: steps i = top, top-1, .. take their partners j_i, and
// the longest prefix of them touching pairwise distinct positions (a step
// conflicts when an earlier one in the round has the same partner or has the
// step's own index as partner -- found with a shared-memory hash table) runs
// at once.
#include <cuda_runtime.h>

#include <cstdlib>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

enum : uint32_t { TAG_IPSC_RS = 7u, TAG_IPSC_FM = 8u, TAG_IPSC_FY = 9u };

// D10 draw: the first of the four words of Philox(K, (c0, c1, lo32 a,
// tag | level << 8 | (hi32 a & 0xFFFF) << 16)) that Lemire32 accepts for the
// bound (threshold 2^32 mod bound), else (w0 * bound) >> 32.
__device__ __forceinline__ uint32_t ipsc_draw(PhiloxKey key, uint32_t tag, uint32_t c0, uint32_t c1, uint32_t level,
                                              uint64_t a, uint32_t bound) {
    const uint4 w = philox4x32_10(
        make_uint4(c0, c1, (uint32_t)a, tag | (level << 8) | (((uint32_t)(a >> 32) & 0xFFFFu) << 16)), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t M = (uint64_t)ws[q] * bound;
        const uint32_t lo = (uint32_t)M;
        if (lo >= bound || lo >= (0u - bound) % bound) return (uint32_t)(M >> 32);
    }
    return (uint32_t)(((uint64_t)w.x * bound) >> 32);
}

// Bucket i's range in heap node v of the segment [a, a+m): bucket i of the
// root is [a + floor(i m / k), a + floor((i+1) m / k)) ("equal sizes up to
// rounding"); node 2v takes [lo, lo + floor((hi-lo)/2)), 2v+1 the rest.
__device__ __forceinline__ void node_range(uint64_t a, uint64_t m, uint32_t k, uint32_t i, uint32_t v, uint64_t& lo,
                                           uint64_t& hi) {
    lo = a + ((uint64_t)i * m) / k;
    hi = a + ((uint64_t)(i + 1) * m) / k;
    const int d = 31 - __clz(v);
    for (int bit = d - 1; bit >= 0; --bit) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if ((v >> bit) & 1u) lo = mid;
        else hi = mid;
    }
}

__device__ __forceinline__ void ipsc_latch(Header* h, uint32_t code) { atomicCAS(&h->error, 0u, code); }

// Swap X[p + x] <-> X[q - x] for x in [0, n) (MIRROR), or X[p + x] <-> X[p + x + q]
// (stride q >= n), by threads gt = 0.. of a group of G.  The pairs are
// disjoint, so each thread keeps four in flight (memory-level parallelism).
template <typename E, bool MIRROR>
__device__ __forceinline__ void pair_swaps(E* X, uint64_t p, uint64_t q, uint64_t n, uint32_t gt, uint32_t G) {
    auto other = [&](uint64_t x) { return MIRROR ? q - x : p + x + q; };
    uint64_t x = gt;
    for (; x + 3ull * G < n; x += 4ull * G) {
        E a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = X[p + x + u * (uint64_t)G];
            b[u] = X[other(x + u * (uint64_t)G)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            X[p + x + u * (uint64_t)G] = b[u];
            X[other(x + u * (uint64_t)G)] = a[u];
        }
    }
    for (; x < n; x += G) {
        const E t0 = X[p + x];
        X[p + x] = X[other(x)];
        X[other(x)] = t0;
    }
}


// ---------------------------------------------------------- RoughScatter --
// Shared scratch of one RoughScatter run by NT threads taking U steps each
// per round: s_i, e_i, two per-warp count tables [NT/32][k] (u8), hands
// [U NT + 1].
template <int EB, int NT, int U>
struct RsScratch {
    static constexpr uint32_t TB = NT / 32u;  // count-table rows
    uint64_t* sp;
    uint64_t* se;
    unsigned char* cnt;
    typename ElemT<EB>::type* hand;
    __host__ __device__ static uint32_t cnt_bytes(uint32_t k) { return (2u * TB * k + 15u) / 16u * 16u; }
    __host__ __device__ static uint32_t bytes(uint32_t k) { return 16u * k + cnt_bytes(k) + (U * NT + 1u) * EB; }
    __device__ RsScratch(unsigned char* base, uint32_t k)
        : sp(reinterpret_cast<uint64_t*>(base)),
          se(reinterpret_cast<uint64_t*>(base) + k),
          cnt(base + 16u * k),
          hand(reinterpret_cast<typename ElemT<EB>::type*>(base + 16u * k + cnt_bytes(k))) {}
};

// Node v of the segment [a, a+m): MERGE -> merge the children's halves
// (staged starts sl, sr), then RoughScatter; the node's staged starts go to
// out (which may alias sr: read before written).  X: absolute positions
// (global memory, or a shared-memory view shifted by -a).  All NT threads.
// A round takes U sub-rounds of NT consecutive steps: their positions (ranks
// against the pointers the previous sub-round advanced), then ONE batch of
// hand reads for all U NT steps, then the writes -- one memory round trip
// per U NT steps.
template <int EB, int NT, int U, bool MERGE>
__device__ void rs_node(typename ElemT<EB>::type* X, const IpscParams& P, uint64_t a, uint64_t m, uint32_t v,
                        const uint64_t* sl, const uint64_t* sr, uint64_t* out, const RsScratch<EB, NT, U>& R,
                        uint32_t* s_stop) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t TB = RsScratch<EB, NT, U>::TB;
    const uint32_t k = P.k, tid = threadIdx.x, lane = tid & 31u, w = tid >> 5;
    uint64_t* sp = R.sp;
    uint64_t* se = R.se;
    unsigned char* cnt = R.cnt;
    E* hand = R.hand;
    for (uint32_t i = tid; i < k; i += NT) {
        uint64_t lo, hi;
        node_range(a, m, k, i, v, lo, hi);
        se[i] = hi;
        sp[i] = MERGE ? sl[i] + (sr[i] - (lo + (hi - lo) / 2)) : lo;  // (b, s1 + B, e') / all staged
    }
    for (uint32_t x = tid; x < 2u * TB * k; x += NT) cnt[x] = 0;
    if (MERGE) {  // staged items of the first half <-> placed items of the second half, per bucket
        for (uint32_t i = 0; i < k; ++i) {
            uint64_t lo, hi;
            node_range(a, m, k, i, v, lo, hi);
            const uint64_t mid = lo + (hi - lo) / 2, s1 = sl[i], s2 = sr[i];
            const uint64_t A = mid - s1, B = s2 - mid, mn = A < B ? A : B;
            pair_swaps<E, true>(X, s1, s2 - 1, mn, tid, NT);
        }
    }
    __syncthreads();
    int full = 0;
    for (uint32_t i = tid; i < k; i += NT) full |= (sp[i] == se[i]);
    if (!__syncthreads_or(full)) {
        const PhiloxKey key = make_key(P.seed);
        if (tid == 0) hand[0] = X[sp[0]];
        const uint32_t lt = (1u << lane) - 1u;
        for (uint32_t base = 0;; base += U * NT) {
            uint64_t pos[U];
            uint32_t jj[U];
            if (tid == 0) {
                *s_stop = U * NT;
                if (base) hand[0] = hand[U * NT];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                unsigned char* tab = cnt + (u & 1) * TB * k;
                const uint32_t step = u * NT + tid;
                const uint32_t j = ipsc_draw(key, TAG_IPSC_RS, base + step, v, P.level, a, k);
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, j);
                const uint32_t lead = __ffs(peers) - 1;
                if (lane == lead) tab[w * k + j] = (unsigned char)__popc(peers);
                __syncthreads();  // (also: the previous sub-round's pointer updates are visible)
                uint64_t pre = __popc(peers & lt);
                for (uint32_t q = 0; q < w; ++q) pre += tab[q * k + j];
                pos[u] = sp[j] + pre;
                jj[u] = j;
                if (pos[u] + 1 == se[j] && step < *s_stop) atomicMin(s_stop, step);
                __syncthreads();
                const bool active = step <= *s_stop;
                const uint32_t pa = peers & __ballot_sync(0xFFFFFFFFu, active);
                if (lane == lead) {
                    tab[w * k + j] = 0;
                    if (pa) atomicAdd(reinterpret_cast<unsigned long long*>(&sp[j]), (unsigned long long)__popc(pa));
                }
            }
            const uint32_t T = *s_stop;  // (fixed since the last sub-round's second barrier)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t step = u * NT + tid;
                if (step <= T && !(step == T && jj[u] == 0)) hand[step + 1] = X[jj[u] ? pos[u] : pos[u] + 1];
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t step = u * NT + tid;
                if (step <= T) X[pos[u]] = hand[step];
                if (step == T && jj[u] != 0) X[sp[0]] = hand[T + 1];  // the last hand lands at s_0 (staged)
            }
            if (T < U * NT) break;
            __syncthreads();
        }
    }
    __syncthreads();
    for (uint32_t i = tid; i < k; i += NT) out[i] = sp[i];
    __syncthreads();
}

// One CTA per work item (segment, heap node v) of a batch, in HBM.
// RoughScatter of node v by ONE warp (many nodes per launch): rounds of U
// sub-rounds of 32 steps; ranks by match_any, the stop by a ballot, the hand
// chain by shuffles -- no CTA barriers.  Per warp shared state: the node's
// staged starts s0_i at the round's start (u64), placed counts c_i and
// remaining capacities cap_i (u32).
template <typename E>
__device__ __forceinline__ E shfl_elem(E x, uint32_t src_lane_or_delta, bool up) {
    constexpr int W = sizeof(E) / 4;
    uint32_t w[W];
    memcpy(w, &x, sizeof(E));
#pragma unroll
    for (int q = 0; q < W; ++q)
        w[q] = up ? __shfl_up_sync(0xFFFFFFFFu, w[q], src_lane_or_delta) : __shfl_sync(0xFFFFFFFFu, w[q], src_lane_or_delta);
    E y;
    memcpy(&y, w, sizeof(E));
    return y;
}

template <int EB, int U, bool MERGE>
__device__ void rs_node_warp(typename ElemT<EB>::type* X, const IpscParams& P, uint64_t a, uint64_t m, uint32_t v,
                             const uint64_t* sl, const uint64_t* sr, uint64_t* out, uint64_t* s0, uint32_t* c,
                             uint32_t* cap) {
    using E = typename ElemT<EB>::type;
    const uint32_t k = P.k, lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    int full = 0;
    for (uint32_t i = lane; i < k; i += 32) {
        uint64_t lo, hi;
        node_range(a, m, k, i, v, lo, hi);
        const uint64_t st = MERGE ? sl[i] + (sr[i] - (lo + (hi - lo) / 2)) : lo;
        s0[i] = st;
        c[i] = 0;
        cap[i] = (uint32_t)(hi - st);
        full |= hi == st;
    }
    if (MERGE) {  // staged items of the first half <-> placed items of the second half, bucket by bucket
        for (uint32_t i = 0; i < k; ++i) {
            uint64_t lo, hi;
            node_range(a, m, k, i, v, lo, hi);
            const uint64_t mid = lo + (hi - lo) / 2, s1 = sl[i], s2 = sr[i];
            const uint64_t A = mid - s1, B = s2 - mid, mn = A < B ? A : B;
            pair_swaps<E, true>(X, s1, s2 - 1, mn, lane, 32u);
        }
    }
    __syncwarp();
    if (!__any_sync(0xFFFFFFFFu, full)) {
        const PhiloxKey key = make_key(P.seed);
        const uint32_t nbits = 32u - __clz(k - 1u);  // <= 10 (k <= 1024)
        E carry = X[s0[0]];  // the first hand (all lanes)
        for (uint32_t base = 0;; base += 32u * U) {
            // draws of the round's U x 32 steps and the ballots of their bits: lanes of
            // sub-round u' holding value x = AND_b (x_b ? bal[u'][b] : ~bal[u'][b])
            uint32_t jj[U], bal[U][10];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                jj[u] = ipsc_draw(key, TAG_IPSC_RS, base + 32u * u + lane, v, P.level, a, k);
#pragma unroll
                for (int b = 0; b < 10; ++b) bal[u][b] = (uint32_t)b < nbits ? __ballot_sync(0xFFFFFFFFu, (jj[u] >> b) & 1u) : 0u;
            }
            uint32_t eq[U][U], rank[U], cj[U], capj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint32_t r = 0;
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    uint32_t msk = 0xFFFFFFFFu;
#pragma unroll
                    for (int b = 0; b < 10; ++b)
                        if ((uint32_t)b < nbits) msk &= ((jj[u] >> b) & 1u) ? bal[q][b] : ~bal[q][b];
                    eq[u][q] = msk;
                    if (q < u) r += __popc(msk);
                    else if (q == u) r += __popc(msk & lt);
                }
                rank[u] = r;  // earlier steps of the round with my partner
                cj[u] = c[jj[u]];
                capj[u] = cap[jj[u]];
            }
            uint32_t T = 32u * U;  // first step of the round that fills its bucket
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t fm = __ballot_sync(0xFFFFFFFFu, cj[u] + rank[u] + 1u == capj[u]);
                if (T == 32u * U && fm) T = 32u * u + __ffs(fm) - 1;
            }
            uint64_t pos[U];
#pragma unroll
            for (int u = 0; u < U; ++u) pos[u] = s0[jj[u]] + cj[u] + rank[u];
            __syncwarp();
#pragma unroll
            for (int u = 0; u < U; ++u) {  // the first occurrence of a partner in the round adds its active steps
                if (rank[u] == 0 && 32u * u + lane <= T) {
                    uint32_t n = 0;
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const uint32_t act = T >= 32u * q + 31u ? 0xFFFFFFFFu
                                             : T < 32u * q     ? 0u
                                                               : (2u << (T - 32u * q)) - 1u;
                        n += __popc(eq[u][q] & act);
                    }
                    c[jj[u]] += n;
                }
            }
            E val[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t st = 32u * u + lane;
                if (st <= T && !(st == T && jj[u] == 0)) val[u] = X[jj[u] ? pos[u] : pos[u] + 1];
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t st = 32u * u + lane;
                E h = shfl_elem(val[u], 1, true);
                const E prev = u == 0 ? carry : shfl_elem(val[u > 0 ? u - 1 : 0], 31, false);
                if (lane == 0) h = prev;
                if (st <= T) X[pos[u]] = h;
            }
            if (T < 32u * U) {
                const uint32_t ut = T / 32u;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if ((uint32_t)u == ut && lane == (T & 31u) && jj[u] != 0)
                        X[s0[0] + c[0]] = val[u];  // the last hand lands at s_0 (staged)
                break;
            }
            carry = shfl_elem(val[U - 1], 31, false);
        }
    }
    __syncwarp();
    for (uint32_t i = lane; i < k; i += 32) out[i] = s0[i] + c[i];
    __syncwarp();
}

constexpr uint32_t kRsWarpThreads = 256;

template <int EB, bool MERGE>
__global__ void __launch_bounds__(kRsWarpThreads) k_ipsc_rs_warp(IpscParams P, uint32_t nwork) {
    constexpr int U = 4;
    extern __shared__ __align__(16) unsigned char ism[];
    const uint32_t k = P.k, warp = threadIdx.x >> 5, nw = kRsWarpThreads / 32u;
    uint64_t* s0 = reinterpret_cast<uint64_t*>(ism) + (uint64_t)warp * 2u * k;  // [s0 k u64 | c k u32 | cap k u32]
    uint32_t* c = reinterpret_cast<uint32_t*>(s0 + k);
    uint32_t* cap = c + k;
    for (uint32_t x = blockIdx.x * nw + warp; x < nwork; x += gridDim.x * nw) {
        const uint2 wi = P.work[x];
        const IpscSeg sg = P.segs[wi.x];
        const uint32_t v = wi.y;
        uint64_t* T = P.s_tab + sg.node_base * k;
        rs_node_warp<EB, U, MERGE>(reinterpret_cast<typename ElemT<EB>::type*>(P.X), P, sg.a, sg.m, v,
                                   T + (uint64_t)(2 * v - 1) * k, T + (uint64_t)(2 * v) * k, T + (uint64_t)(v - 1) * k,
                                   s0, c, cap);
    }
}

constexpr int kRsU = 4;  // steps per thread per round in HBM

// Persistent: a few CTAs per SM walk the work list, so that the bucket
// cursors in flight (k per node) keep their sectors in L2.
template <int EB, int NT, bool MERGE>
__global__ void __launch_bounds__(NT) k_ipsc_rs(IpscParams P, uint32_t nwork) {
    extern __shared__ __align__(16) unsigned char ism[];
    __shared__ uint32_t s_stop;
    const uint32_t k = P.k;
    const RsScratch<EB, NT, kRsU> R(ism, k);
    for (uint32_t x = blockIdx.x; x < nwork; x += gridDim.x) {
        const uint2 wi = P.work[x];
        const IpscSeg sg = P.segs[wi.x];
        const uint32_t v = wi.y;
        uint64_t* T = P.s_tab + sg.node_base * k;
        rs_node<EB, NT, kRsU, MERGE>(reinterpret_cast<typename ElemT<EB>::type*>(P.X), P, sg.a, sg.m, v,
                                     T + (uint64_t)(2 * v - 1) * k, T + (uint64_t)(2 * v) * k,
                                     T + (uint64_t)(v - 1) * k, R, &s_stop);
    }
}

// ----------------------------------------------------------- FineScatter --
__device__ __forceinline__ uint32_t fy_hash(uint32_t x, uint32_t H) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    return x & (H - 1u);
}

// Virtual index t of the staged items -> position (staged ranges in bucket order).
__device__ __forceinline__ uint64_t staged_pos(const uint64_t* cum, const uint64_t* s, uint32_t k, uint64_t t) {
    uint32_t lo = 0, hi = k;  // largest i with cum[i] <= t (the non-empty range holding t)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] <= t) lo = mid;
        else hi = mid;
    }
    return s[lo] + (t - cum[lo]);
}

// Shared scratch of FineScatter: b, s, e, n^f, D, cum[k+1] (u64), counts
// (u32), hash keys/values [H] (u64), H = 2 NT (at most half full).
template <int NT>
struct FineScratch {
    static constexpr uint32_t H = 2u * NT;
    uint64_t *b, *s, *e, *nf, *cum, *hkey, *hval;
    int64_t* Dp;
    uint32_t* cnt;
    __host__ __device__ static uint32_t bytes(uint32_t k) { return 8u * (6u * k + 1u) + 4u * (k + 1u) + 16u * H + 16u; }
    __device__ FineScratch(unsigned char* base, uint32_t k) {
        b = reinterpret_cast<uint64_t*>(base);
        s = b + k;
        e = s + k;
        nf = e + k;
        Dp = reinterpret_cast<int64_t*>(nf + k);
        cum = reinterpret_cast<uint64_t*>(Dp + k);
        cnt = reinterpret_cast<uint32_t*>(cum + k + 1);
        hkey = reinterpret_cast<uint64_t*>(cnt + k + (k & 1u));
        hval = hkey + H;
    }
};

// One TwoSweep boundary move of x slots with stride P (see k_ipsc_fine):
// sweep 1 (DOWN) over [c - x, c + P), sweep 2 (UP) over [c, c + P + x); lanes
// gt = 0.. of a group of G threads take the residue classes.
template <typename E, bool DOWN>
__device__ __forceinline__ void sweep_move(E* X, uint64_t c, uint64_t x, uint64_t Pp, uint32_t gt, uint32_t G) {
    if (Pp == 0) return;
    if (x <= Pp) {  // every class holds two elements: x disjoint swaps at distance P
        pair_swaps<E, false>(X, DOWN ? c - x : c, Pp, x, gt, G);
        return;
    }
    const uint64_t nr = Pp < x ? Pp : x;  // here x > P: chains of C + 1 >= 3 elements
    const bool n32 = ((x | Pp) >> 32) == 0;
    for (uint64_t r = gt; r < nr; r += G) {
        const uint64_t C = (n32 ? (uint64_t)((uint32_t)(x - 1 - r) / (uint32_t)Pp) : (x - 1 - r) / Pp) + 1;
        if (DOWN) {  // unit u swaps (c-1-u, c-1-u+P): each class's top element drops to its bottom
            const uint64_t q0 = c - x + r;
            const E top = X[q0 + C * Pp];
            for (uint64_t jj = C; jj-- > 0;) X[q0 + (jj + 1) * Pp] = X[q0 + jj * Pp];
            X[q0] = top;
        } else {     // unit u swaps (c+u, c+u+P): each class's bottom element rises to its top
            const uint64_t q0 = c + r;
            const E bot = X[q0];
            for (uint64_t jj = 1; jj <= C; ++jj) X[q0 + (jj - 1) * Pp] = X[q0 + jj * Pp];
            X[q0 + C * Pp] = bot;
        }
    }
}

// FineScatter of the segment [a, a+m) whose root staged starts are s_root:
// writes the final bucket starts S[0..k] (S[k] = a + m).  All NT threads.
// WARP_SWEEP: TwoSweep by warp 0 alone (data in shared memory: cheap steps).
template <int EB, int NT, bool WARP_SWEEP>
__device__ void fine_seg(typename ElemT<EB>::type* X, const IpscParams& P, uint64_t a, uint64_t m, const uint64_t* s_root,
                         uint64_t* S, const FineScratch<NT>& F, unsigned long long* s_R, uint32_t* s_prefix) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t H = FineScratch<NT>::H;
    const uint32_t k = P.k, tid = threadIdx.x;
    uint64_t *b = F.b, *s = F.s, *e = F.e, *nf = F.nf, *cum = F.cum, *hkey = F.hkey, *hval = F.hval;
    int64_t* Dp = F.Dp;
    uint32_t* cnt = F.cnt;
    const PhiloxKey key = make_key(P.seed);
    if (tid == 0) *s_R = 0;
    __syncthreads();
    unsigned long long myR = 0;
    for (uint32_t i = tid; i < k; i += NT) {
        uint64_t lo, hi;
        node_range(a, m, k, i, 1u, lo, hi);
        b[i] = lo;
        e[i] = hi;
        s[i] = s_root[i];
        cnt[i] = 0;
        myR += hi - s[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) myR += __shfl_xor_sync(0xFFFFFFFFu, myR, o);
    if ((tid & 31u) == 0 && myR) atomicAdd(s_R, myR);
    for (uint32_t x = tid; x < H; x += NT) {
        hkey[x] = 0;
        hval[x] = 0;
    }
    __syncthreads();
    const uint64_t R = *s_R;
    if (R > 0xFFFFFFFFull) {
        if (tid == 0) ipsc_latch(P.hdr, 8u /*SHUF_ERR_INTERNAL*/);
        return;
    }
    // final sizes n^f_i = n_i + N'_i, N' ~ multinomial(R, 1/k) from R uniform draws
    for (uint32_t r = tid; r < (uint32_t)R; r += NT)
        atomicAdd(&cnt[ipsc_draw(key, TAG_IPSC_FM, r, 0u, P.level, a, k)], 1u);
    __syncthreads();
    // D_i = sum_{j<=i} (n^f_j - c_j)  (Lemma 4): warp 0 scans, lane l owning buckets [l*per, (l+1)*per)
    if (tid < 32) {
        const uint32_t per = (k + 31u) >> 5, i0 = tid * per, i1 = min(k, i0 + per);
        int64_t part = 0;
        for (uint32_t i = i0; i < i1; ++i) {
            nf[i] = s[i] - b[i] + cnt[i];
            part += (int64_t)nf[i] - (int64_t)(e[i] - b[i]);
        }
        int64_t incl = part;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= (uint32_t)o) incl += t;
        }
        int64_t D = incl - part;
        for (uint32_t i = i0; i < i1; ++i) {
            D += (int64_t)nf[i] - (int64_t)(e[i] - b[i]);
            Dp[i] = D;
        }
    }
    __syncthreads();
    const bool tk = P.clk && blockIdx.x == 0 && tid == 0 && *s_R == R && WARP_SWEEP;
    if (tk && P.clk[2] == 0) P.clk[2] = clock64();
    // TwoSweep.  Boundary i makes ONE move: sweep 1 (ascending) when
    // D_i < 0, sweep 2 (descending) when D_i > 0, at c = b_{i+1}, with stride
    // P = s_{i+1} - b_{i+1} -- values of the state before the sweeps, since only
    // the boundary's own move changes them; afterwards b_{i+1} = s_{i+1} - P =
    // b_{i+1} + D_i and e_i = b_{i+1}.  The data order between the moves is
    // kept by a group barrier after each.
    if (!WARP_SWEEP || tid < 32) {
        const uint32_t G = WARP_SWEEP ? 32u : NT, gt = tid;
        for (uint32_t i = 0; i + 1 < k; ++i) {  // sweep 1: -D_i slots of B_i's end -> B_{i+1}
            const int64_t xd = -Dp[i];
            if (xd <= 0) continue;
            sweep_move<E, true>(X, b[i + 1], (uint64_t)xd, s[i + 1] - b[i + 1], gt, G);
            if (WARP_SWEEP) __syncwarp();
            else __syncthreads();
        }
        for (uint32_t i = k - 1; i-- > 0;) {  // sweep 2: D_i slots of B_{i+1}'s start -> B_i
            const int64_t xd = Dp[i];
            if (xd <= 0) continue;
            sweep_move<E, false>(X, b[i + 1], (uint64_t)xd, s[i + 1] - b[i + 1], gt, G);
            if (WARP_SWEEP) __syncwarp();
            else __syncthreads();
        }
    }
    __syncthreads();
    for (uint32_t i = tid; i + 1 < k; i += NT) {
        b[i + 1] += (uint64_t)Dp[i];
        s[i + 1] += (uint64_t)Dp[i];
    }
    __syncthreads();
    for (uint32_t i = tid; i + 1 < k; i += NT) e[i] = b[i + 1];
    __syncthreads();
    if (tk && P.clk[3] == 0) P.clk[3] = clock64();
    if (tid < 32) {  // cum = exclusive prefix of the staged counts (warp 0), and the final sizes reached
        const uint32_t per = (k + 31u) >> 5, i0 = tid * per, i1 = min(k, i0 + per);
        uint64_t part = 0;
        for (uint32_t i = i0; i < i1; ++i) {
            if (s[i] < b[i] || s[i] > e[i] || e[i] - b[i] != nf[i]) ipsc_latch(P.hdr, 8u);
            part += e[i] - s[i];
        }
        uint64_t incl = part;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= (uint32_t)o) incl += t;
        }
        uint64_t t = incl - part;
        for (uint32_t i = i0; i < i1; ++i) {
            cum[i] = t;
            t += e[i] - s[i];
        }
        if (tid == 31) {
            cum[k] = incl;
            if (incl != R) ipsc_latch(P.hdr, 8u);
        }
    }
    __syncthreads();
    // stash shuffle: Fisher-Yates on V[t] = X[p_t], rounds of conflict-free prefixes
    uint64_t top = R ? R - 1 : 0;
    constexpr bool kWarpFy = true;  // shared-memory data: warp-0 rounds (CTA rounds measured 1.8x slower, r03g)
    if (WARP_SWEEP && kWarpFy) {  // warp 0, rounds of <= 32 steps; conflicts found by match_any and an OR-reduction
        // positions p_t - a as u16 in the (here unused) hash region when they fit
        uint16_t* posT = reinterpret_cast<uint16_t*>(hkey);
        const bool tab = R <= 8u * H && m <= 65536u;
        if (tab)
            for (uint32_t t = tid; t < (uint32_t)R; t += NT) posT[t] = (uint16_t)(staged_pos(cum, s, k, t) - a);
        __syncthreads();
        if (tid < 32) {
            const uint32_t lane = tid, lt = (1u << lane) - 1u;
            uint32_t tp = (uint32_t)top;
            uint32_t jn = tp >= lane + 1 ? ipsc_draw(key, TAG_IPSC_FY, tp - lane, 0u, P.level, a, tp - lane + 1) : 0u;
            while (tp >= 1) {
                const bool valid = tp >= lane + 1;
                const uint32_t i = valid ? tp - lane : 0u;
                const uint32_t j = valid ? jn : 0u;
                // the draws of the next 32 steps, assuming this round runs all 32 (the usual case)
                const uint32_t tq = tp >= 32u ? tp - 32u : 0u;
                const uint32_t jspec = tq >= lane + 1 ? ipsc_draw(key, TAG_IPSC_FY, tq - lane, 0u, P.level, a, tq - lane + 1) : 0u;
                // (j <= i < R < 2^31: idle lanes match nothing)
                bool conflict = (__match_any_sync(0xFFFFFFFFu, valid ? j : 0xFFFFFFFFu - lane) & lt) != 0;
                // an earlier step's partner is my own index: lane l' with j = tp - l (l > l') hits lane l
                const uint32_t d = tp - j;
                const uint32_t hit = __reduce_or_sync(0xFFFFFFFFu, valid && d < 32u && d > lane ? 1u << d : 0u);
                conflict |= (hit >> lane) & 1u;
                const uint32_t cm = __ballot_sync(0xFFFFFFFFu, valid && conflict);
                const uint32_t nv = __popc(__ballot_sync(0xFFFFFFFFu, valid));
                const uint32_t pre = cm ? (uint32_t)(__ffs(cm) - 1) : nv;
                if (valid && lane < pre && i != j) {
                    const uint64_t pi = tab ? a + posT[i] : staged_pos(cum, s, k, i);
                    const uint64_t pj = tab ? a + posT[j] : staged_pos(cum, s, k, j);
                    const E t0 = X[pi];
                    X[pi] = X[pj];
                    X[pj] = t0;
                }
                __syncwarp();
                tp -= pre;
                if (pre == 32u) jn = jspec;
                else if (tp >= lane + 1) jn = ipsc_draw(key, TAG_IPSC_FY, tp - lane, 0u, P.level, a, tp - lane + 1);
            }
        }
        top = 0;
        __syncthreads();
        if (tk && P.clk[4] == 0) P.clk[4] = clock64();
    }
    // CTA rounds of up to NT steps (32-bit tables in the hash region, reset every
    // round): hk/hv = open-addressing map partner -> min order; win[d] = min order
    // of a step whose partner is the round's index top - d.
    uint32_t* hk = reinterpret_cast<uint32_t*>(hkey);
    uint32_t* hv = hk + H;
    uint32_t* win = hv + H;
    for (uint32_t x = tid; x < H; x += NT) {
        hk[x] = 0xFFFFFFFFu;
        hv[x] = 0xFFFFFFFFu;
    }
    for (uint32_t x = tid; x < NT; x += NT) win[x] = 0xFFFFFFFFu;
    __syncthreads();
    while (top >= 1) {
        const uint32_t o = tid;
        const bool valid = top >= (uint64_t)o + 1;
        const uint32_t i = valid ? (uint32_t)(top - o) : 0u;
        const uint32_t j = valid ? ipsc_draw(key, TAG_IPSC_FY, i, 0u, P.level, a, i + 1) : 0u;
        if (tid == 0) *s_prefix = (uint32_t)(top < NT ? top : NT);
        uint32_t hslot = 0;
        if (valid) {
            const uint64_t d = top - j;
            if (d < NT && d > o) atomicMin(&win[d], o);
            uint32_t h = fy_hash(j, H);
            for (;;) {
                const uint32_t prev = atomicCAS(&hk[h], 0xFFFFFFFFu, j);
                if (prev == 0xFFFFFFFFu || prev == j) break;
                h = (h + 1) & (H - 1u);
            }
            atomicMin(&hv[h], o);
            hslot = h;
        }
        __syncthreads();
        if (valid && (win[o] < o || hv[hslot] < o)) atomicMin(s_prefix, o);
        __syncthreads();
        const uint32_t pre = *s_prefix;
        if (valid && o < pre && i != j) {
            const uint64_t pi = staged_pos(cum, s, k, i), pj = staged_pos(cum, s, k, j);
            const E t0 = X[pi];
            X[pi] = X[pj];
            X[pj] = t0;
        }
        if (valid) {
            hk[hslot] = 0xFFFFFFFFu;
            hv[hslot] = 0xFFFFFFFFu;
        }
        win[o] = 0xFFFFFFFFu;
        __syncthreads();
        top -= pre;
    }
    for (uint32_t i = tid; i < k; i += NT) S[i] = b[i];
    if (tid == 0) S[k] = a + m;
    __syncthreads();
}

constexpr uint32_t kFineThreads = 1024;

template <int EB>
__global__ void __launch_bounds__(kFineThreads) k_ipsc_fine(IpscParams P) {
    extern __shared__ __align__(16) unsigned char ism[];
    __shared__ unsigned long long s_R;
    __shared__ uint32_t s_prefix;
    const IpscSeg sg = P.segs[blockIdx.x];
    const FineScratch<kFineThreads> F(ism, P.k);
    fine_seg<EB, kFineThreads, false>(reinterpret_cast<typename ElemT<EB>::type*>(P.X), P, sg.a, sg.m,
                                      P.s_tab + sg.node_base * P.k, P.S + (uint64_t)blockIdx.x * (P.k + 1), F, &s_R,
                                      &s_prefix);
}

// ------------------------------------------------------- small segments --
// A segment of at most `cap` elements runs its whole IpSc level in shared
// memory: load, ParRoughScatter's tree in post-order (a completed left child
// waits in the slot of its depth), FineScatter, Fisher-Yates of the children
// of at most L elements (D5, Fig. 1), store; longer children join the next
// level's list.  One CTA per segment (persistent over the level's list).
constexpr uint32_t kSmallThreads = 512;

__host__ __device__ inline uint32_t ipsc_small_fixed(uint32_t k, uint32_t eb, uint32_t tmax) {
    const uint32_t rs = 16u * k + (2u * (kSmallThreads / 32u) * k + 15u) / 16u * 16u + (kSmallThreads + 1u) * eb;
    const uint32_t fine = FineScratch<kSmallThreads>::bytes(k);
    return (tmax + 2u) * k * 8u + (rs > fine ? rs : fine) + 8u * (k + 1u) + 64u;
}

template <int EB>
__global__ void __launch_bounds__(kSmallThreads, 2) k_ipsc_small(IpscParams P, const uint64_t* __restrict__ list,
                                                              uint32_t count, uint32_t cap, uint32_t tmax) {
    using E = typename ElemT<EB>::type;
    constexpr uint32_t NT = kSmallThreads;
    extern __shared__ __align__(16) unsigned char ism[];
    __shared__ uint32_t s_stop, s_prefix;
    __shared__ unsigned long long s_R;
    const uint32_t k = P.k, tid = threadIdx.x;
    E* data = reinterpret_cast<E*>(ism);
    uint64_t* slots = reinterpret_cast<uint64_t*>(ism + ((uint64_t)cap * EB + 15u) / 16u * 16u);  // [tmax + 2][k]
    unsigned char* scr = reinterpret_cast<unsigned char*>(slots + (uint64_t)(tmax + 2u) * k);
    const uint32_t rsb = RsScratch<EB, NT, 1>::bytes(k), fb = FineScratch<NT>::bytes(k);
    uint64_t* Sb = reinterpret_cast<uint64_t*>(scr + ((rsb > fb ? rsb : fb) + 15u) / 16u * 16u);
    const RsScratch<EB, NT, 1> R(scr, k);
    const FineScratch<NT> F(scr, k);
    E* G = reinterpret_cast<E*>(P.X);
    for (uint32_t si = blockIdx.x; si < count; si += gridDim.x) {
        const uint64_t a = list[2 * (uint64_t)si], m = list[2 * (uint64_t)si + 1];
        if (m > cap) continue;  // the HBM kernels' segment
        const bool tk = P.clk && blockIdx.x == 0 && tid == 0 && si == 0;
        if (tk) P.clk[0] = clock64();
        for (uint64_t x = tid; x < m; x += NT) data[x] = G[a + x];
        __syncthreads();
        E* X = reinterpret_cast<E*>(reinterpret_cast<uintptr_t>(data) - a * EB);  // absolute positions
        // ParRoughScatter tree, post-order over the leaves v = 2^t .. 2^(t+1)-1
        uint32_t t = 0;
        while (t < 11u && (m >> (t + 1)) >= (uint64_t)k * k) ++t;
        uint64_t* cur = slots + (uint64_t)(tmax + 1u) * k;
        for (uint32_t v = 1u << t; v < (2u << t); ++v) {
            rs_node<EB, NT, 1, false>(X, P, a, m, v, nullptr, nullptr, cur, R, &s_stop);
            uint32_t u = v, d = t;
            while (u & 1u && u > 1u) {  // a right child completes its parent
                rs_node<EB, NT, 1, true>(X, P, a, m, u >> 1, slots + (uint64_t)d * k, cur, cur, R, &s_stop);
                u >>= 1;
                --d;
            }
            if (u > 1u)  // a left child waits for its sibling
                for (uint32_t i = tid; i < k; i += NT) slots[(uint64_t)d * k + i] = cur[i];
            __syncthreads();
        }
        if (tk) P.clk[1] = clock64();
        fine_seg<EB, NT, true>(X, P, a, m, cur, Sb, F, &s_R, &s_prefix);
        if (tk) P.clk[5] = clock64();
        // children: Fisher-Yates leaves in shared memory, longer ones to the next level
        const PhiloxKey key = make_key(P.seed);
        for (uint32_t c = tid; c < k; c += NT) {
            const uint64_t st = Sb[c], len = Sb[c + 1] - st;
            if (len > P.L) {
                const uint32_t at = atomicAdd(P.next_cnt, 1u);
                if (at >= P.max_next) {
                    ipsc_latch(P.hdr, 4u /*SHUF_ERR_SCRATCH*/);
                } else {
                    P.next[2 * (uint64_t)at] = st;
                    P.next[2 * (uint64_t)at + 1] = len;
                }
            } else if (P.run_leaves && len >= 2) {
                for (uint32_t i = (uint32_t)len - 1; i >= 1; --i) {
                    const uint32_t jj = fy_draw(key, st, i);
                    const E t0 = X[st + i];
                    X[st + i] = X[st + jj];
                    X[st + jj] = t0;
                }
            }
        }
        __syncthreads();
        if (tk) P.clk[6] = clock64();
        for (uint64_t x = tid; x < m; x += NT) G[a + x] = data[x];
        __syncthreads();
        if (tk) P.clk[7] = clock64();
    }
}

// Children of the batch's segments: longer than L -> the next level's list
// (the leaf kernel takes the others, kernels_leaf.cu IpscLeaves).
__global__ void k_ipsc_children(IpscParams P, uint32_t nseg) {
    const uint32_t k = P.k;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < (uint64_t)nseg * k;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t* S = P.S + (x / k) * (k + 1) + (x % k);
        const uint64_t st = S[0], len = S[1] - S[0];
        if (len <= P.L) continue;
        const uint32_t at = atomicAdd(P.next_cnt, 1u);
        if (at >= P.max_next) {
            ipsc_latch(P.hdr, 4u /*SHUF_ERR_SCRATCH*/);
            continue;
        }
        P.next[2 * (uint64_t)at] = st;
        P.next[2 * (uint64_t)at + 1] = len;
    }
}

// ------------------------------------------------------------- launchers --
template <int EB, int NT, bool MERGE>
static cudaError_t rs_launch(const IpscParams& P, uint32_t nwork, uint32_t grid, cudaStream_t s) {
    const uint32_t sm = RsScratch<EB, NT, kRsU>::bytes(P.k) + 16u;
    cudaError_t e = cudaFuncSetAttribute(k_ipsc_rs<EB, NT, MERGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!e)  // all of the SM's shared memory: several CTAs per SM (the default carveout fits one)
        e = cudaFuncSetAttribute(k_ipsc_rs<EB, NT, MERGE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e) return e;
    k_ipsc_rs<EB, NT, MERGE><<<nwork < grid ? nwork : grid, NT, sm, s>>>(P, nwork);
    return cudaGetLastError();
}

template <int EB, bool MERGE>
static cudaError_t rs_warp_launch(const IpscParams& P, uint32_t nwork, cudaStream_t s) {
    const uint32_t sm = (kRsWarpThreads / 32u) * 16u * P.k;
    cudaError_t e = cudaFuncSetAttribute(k_ipsc_rs_warp<EB, MERGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!e) e = cudaFuncSetAttribute(k_ipsc_rs_warp<EB, MERGE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e) return e;
    const uint32_t nw = kRsWarpThreads / 32u;
    k_ipsc_rs_warp<EB, MERGE><<<(nwork + nw - 1) / nw, kRsWarpThreads, sm, s>>>(P, nwork);
    return cudaGetLastError();
}

template <int EB>
static cudaError_t rs_launch_eb(const IpscParams& P, uint32_t nwork, bool merge, bool wide, uint32_t grid,
                                cudaStream_t s) {
    if (wide) return merge ? rs_launch<EB, 1024, true>(P, nwork, nwork, s) : rs_launch<EB, 1024, false>(P, nwork, nwork, s);
    static const int mode = [] {  // SHUF_IPSC_RSMODE (experiments): 0 = one warp per node, 1 = persistent
        const char* e = std::getenv("SHUF_IPSC_RSMODE");  // 256-thread CTAs (default), 2 = 1024-thread CTAs
        return e ? std::atoi(e) : 1;
    }();
    if (mode == 1) return merge ? rs_launch<EB, 256, true>(P, nwork, grid, s) : rs_launch<EB, 256, false>(P, nwork, grid, s);
    if (mode == 2) return merge ? rs_launch<EB, 1024, true>(P, nwork, grid, s) : rs_launch<EB, 1024, false>(P, nwork, grid, s);
    return merge ? rs_warp_launch<EB, true>(P, nwork, s) : rs_warp_launch<EB, false>(P, nwork, s);
}

// wide: one 1024-thread CTA per node (few nodes); otherwise `grid` persistent 256-thread CTAs walking the
// work list in order (measured faster than one warp per node, r03n/r03o).
cudaError_t launch_ipsc_rs(const IpscParams& P, uint32_t eb, uint32_t nwork, bool merge, bool wide, uint32_t grid,
                           cudaStream_t s) {
    if (nwork == 0) return cudaSuccess;
    switch (eb) {
    case 4: return rs_launch_eb<4>(P, nwork, merge, wide, grid, s);
    case 8: return rs_launch_eb<8>(P, nwork, merge, wide, grid, s);
    default: return rs_launch_eb<16>(P, nwork, merge, wide, grid, s);
    }
}

cudaError_t launch_ipsc_fine(const IpscParams& P, uint32_t eb, uint32_t nseg, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    const uint32_t sm = FineScratch<kFineThreads>::bytes(P.k);
    void* fn = eb == 4 ? (void*)k_ipsc_fine<4> : eb == 8 ? (void*)k_ipsc_fine<8> : (void*)k_ipsc_fine<16>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!e) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e) return e;
    void* args[] = {(void*)&P};
    return cudaLaunchKernel(fn, dim3(nseg), dim3(kFineThreads), args, sm, s);
}

cudaError_t launch_ipsc_children(const IpscParams& P, uint32_t nseg, cudaStream_t s, int grid) {
    if (nseg == 0) return cudaSuccess;
    k_ipsc_children<<<grid, 256, 0, s>>>(P, nseg);
    return cudaGetLastError();
}

// Largest small-segment capacity (elements) whose CTA fits the opt-in shared memory.
uint32_t ipsc_small_cap(uint32_t k, uint32_t eb, uint32_t* tmax_out) {
    uint32_t cap = 0, tmax = 0;
    for (uint32_t c = (kSmemLimit / eb) & ~15u; c >= 16u; c -= 16u) {
        uint32_t t = 0;
        while (t < 11u && (c >> (t + 1)) >= k * k) ++t;
        if (((uint64_t)c * eb + 15u) / 16u * 16u + ipsc_small_fixed(k, eb, t) <= kSmemLimit) {
            cap = c;
            tmax = t;
            break;
        }
    }
    *tmax_out = tmax;
    return cap;
}

cudaError_t launch_ipsc_small(const IpscParams& P, uint32_t eb, const uint64_t* list, uint32_t count, uint32_t cap,
                              uint32_t tmax, cudaStream_t s, int grid) {
    if (count == 0 || cap == 0) return cudaSuccess;
    const uint32_t sm = ((cap * eb + 15u) / 16u * 16u) + ipsc_small_fixed(P.k, eb, tmax);
    void* fn = eb == 4 ? (void*)k_ipsc_small<4> : eb == 8 ? (void*)k_ipsc_small<8> : (void*)k_ipsc_small<16>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!e) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e) return e;
    if (grid > (int)count) grid = (int)count;
    void* args[] = {(void*)&P, (void*)&list, (void*)&count, (void*)&cap, (void*)&tmax};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kSmallThreads), args, sm, s);
}

}  // namespace shuf
