// In-place mode (secondary; BJ "in-place"; motivation
// P:32-36): one HBM scatter level over segments longer than S_fuse
// with O(k * stripes * B) auxiliary memory instead of an n-element
// ping-pong buffer.  NOT stable and NOT deterministic (the order inside a
// bucket depends on atomics); the bucket of every element is still the D4
// draw at its position at that level, so the level-0 bucket multisets equal
// the stable mode's, and segments <= S_fuse / leaves run the stable, in-place
// finish and leaf kernels.
//
// The block scheme (the in-place samplesort idea; blocks of B elements,
// B*eb = 128 bytes):
//  P0 k_ip_stripes   cut every segment of the batch into stripes of Z
//                    elements (block-aligned relative to the segment start);
//  P1 k_ip_classify  a CTA walks its stripe tile by tile, appends elements to
//                    per-bucket carry buffers in shared memory and writes every
//                    full block back into the stripe's own, already consumed
//                    block slots (tagging the slot with its bucket); the
//                    leftovers (< B per bucket) go to the stripe's partial
//                    buffers in aux;
//  k_ip_plan         bucket starts S_d, block region [ceil(S_d/B),
//                    ceil(S_{d+1}/B)) and the (write, read) pointer pair of
//                    every region;
//  P2 k_ip_permute   every thread takes unprocessed blocks from the top of a
//                    region (read pointer) and places each at the write
//                    pointer of its bucket's region, swapping out the block
//                    found there while that slot is still unprocessed, waiting
//                    on the slot's tag while a reader still copies it, and
//                    diverting a block that would cross its bucket's end to a
//                    per-(segment, bucket) overflow block;
//  P3 k_ip_fill      the head of each bucket (up to its first block slot) and
//                    the tail after its last in-place block are filled from
//                    the overflow block and the stripes' partial buffers;
//                    children longer than S_fuse join the next level's list.
// Children of at most S_fuse elements are then finished in place by the
// fused finish / leaf kernels (kernels_finish.cu, kernels_leaf.cu) through
// the per-batch bucket-start table S.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

extern __shared__ __align__(16) unsigned char ism[];

constexpr uint32_t kIpThreads = 512;   // P1
constexpr uint32_t kIpTileBytes = 32768;
constexpr uint16_t kTagEmpty = 0xFFFFu;
constexpr uint16_t kTagRead = 0xFFFEu;
constexpr uint64_t kRBias = 1ull << 31;

template <int EB> struct IpCfg {
    static constexpr uint32_t B = kIpBlockBytes / EB;  // elements per block
    static constexpr uint32_t T = kIpTileBytes / EB;   // elements per P1 tile
    static constexpr uint32_t R = T / kIpThreads;      // elements per thread per tile
};

struct IpLayout {
    uint32_t carry, el, draws, ccnt, cnt, nf, fcount, tb, fb, blk, wsum, total;
};

__host__ __device__ inline IpLayout ip_layout(uint32_t eb, uint32_t k) {
    IpLayout f;
    uint32_t off = 0;
    auto take = [&off](uint32_t bytes) {
        const uint32_t at = off;
        off = (off + bytes + 15u) & ~15u;
        return at;
    };
    const uint32_t B = kIpBlockBytes / eb, T = kIpTileBytes / eb;
    f.carry = take(k * kIpBlockBytes);
    f.el = take(kIpTileBytes);
    f.draws = take(draw_bytes(T));
    f.ccnt = take(k * 4);
    f.cnt = take(k * 4);
    f.nf = take(k * 4);
    f.fcount = take(k * 4);
    f.tb = take((k + 1) * 4);
    f.fb = take((k + 1) * 4);
    f.blk = take((T / B + k + 1) * 4);
    f.wsum = take((kIpThreads / 32 + 1) * 4);
    f.total = off;
    return f;
}

uint32_t ip_classify_smem_bytes(uint32_t eb, uint32_t k) { return ip_layout(eb, k).total; }

// Exclusive scan of in[0..k) into out[0..k], out[k] = total (all NT threads).
template <int NT>
__device__ __forceinline__ void scan_k(const uint32_t* in, uint32_t* out, uint32_t k, uint32_t* wsum) {
    const uint32_t per = (k + NT - 1) / NT;
    const uint32_t x0 = min(k, threadIdx.x * per), x1 = min(k, x0 + per);
    uint32_t mine = 0;
    for (uint32_t x = x0; x < x1; ++x) mine += in[x];
    uint32_t total;
    uint32_t run = block_exclusive_sum<NT>(mine, wsum, &total);
    for (uint32_t x = x0; x < x1; ++x) {
        const uint32_t c = in[x];
        out[x] = run;
        run += c;
    }
    if (threadIdx.x == 0) out[k] = total;
    __syncthreads();
}

// ------------------------------------------------------------------ P0 ----
// One CTA: stripe counts and bases of the batch's segments, stripe -> segment.
__global__ void __launch_bounds__(256) k_ip_stripes(IpParams ip) {
    ip = ip_resolve(ip);
    __shared__ uint32_t wsum[256 / 32 + 1];
    uint32_t base = 0;
    for (uint32_t s0 = 0; s0 < ip.nseg; s0 += 256) {
        const uint32_t s = s0 + threadIdx.x;
        uint32_t nz = 0;
        if (s < ip.nseg) nz = (uint32_t)((ip.segs[s].len + ip.Z - 1) / ip.Z);
        uint32_t total;
        const uint32_t ex = block_exclusive_sum<256>(nz, wsum, &total);
        if (s < ip.nseg) {
            ip.segs[s].zbase = base + ex;
            ip.segs[s].nz = nz;
            for (uint32_t z = 0; z < nz; ++z) ip.zseg[base + ex + z] = s;
        }
        base += total;
    }
}

// ------------------------------------------------------------------ P1 ----
template <int EB>
__global__ void __launch_bounds__(kIpThreads) k_ip_classify(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    using E = typename ElemT<EB>::type;
    constexpr uint32_t B = IpCfg<EB>::B, T = IpCfg<EB>::T, R = IpCfg<EB>::R;
    const uint32_t tid = threadIdx.x, k = rp.k;
    const IpLayout L = ip_layout(EB, k);
    E* carry = reinterpret_cast<E*>(ism + L.carry);
    E* el = reinterpret_cast<E*>(ism + L.el);
    uint32_t* ccnt = reinterpret_cast<uint32_t*>(ism + L.ccnt);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(ism + L.cnt);
    uint32_t* nf = reinterpret_cast<uint32_t*>(ism + L.nf);
    uint32_t* fcount = reinterpret_cast<uint32_t*>(ism + L.fcount);
    uint32_t* tb = reinterpret_cast<uint32_t*>(ism + L.tb);
    uint32_t* fb = reinterpret_cast<uint32_t*>(ism + L.fb);
    uint32_t* blk = reinterpret_cast<uint32_t*>(ism + L.blk);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(ism + L.wsum);
    E* ptr = reinterpret_cast<E*>(rp.buf0);
    const PhiloxKey key = make_key(rp.seed);
    for (uint32_t b = tid; b < k; b += kIpThreads) ccnt[b] = cnt[b] = fcount[b] = 0;
    __syncthreads();
    for (uint32_t z = blockIdx.x; z < ip.nstripes; z += gridDim.x) {
        const uint32_t s = ip.zseg[z];
        const IpSeg sg = ip.segs[s];
        const uint64_t zrel = (uint64_t)(z - sg.zbase) * ip.Z;
        const uint64_t zs = sg.start + zrel, ze = min(sg.start + sg.len, zs + ip.Z);
        const uint64_t slot0 = zrel / B;  // first block slot of the stripe (segment-relative)
        const uint64_t nslots = (ze - zs) / B;
        const uint64_t tag0 = sg.start / B + slot0;
        uint64_t W = 0;  // blocks written so far
        for (uint64_t t0 = zs; t0 < ze; t0 += T) {
            const uint32_t m = (uint32_t)min((uint64_t)T, ze - t0);
            const DrawView dv = draws_to_smem<kIpThreads>(ism + L.draws, t0, m, key, ip.level, rp.bp);
            __syncthreads();
            uint32_t bb[R], rr[R];
            E vv[R];
#pragma unroll
            for (uint32_t i = 0; i < R; ++i) {
                const uint32_t e = tid + i * kIpThreads;
                if (e < m) {
                    bb[i] = dv.at(e);
                    vv[i] = ptr[t0 + e];
                    rr[i] = atomicAdd(&cnt[bb[i]], 1u);
                }
            }
            __syncthreads();
            for (uint32_t b = tid; b < k; b += kIpThreads) nf[b] = (ccnt[b] + cnt[b]) / B;
            __syncthreads();
            scan_k<kIpThreads>(cnt, tb, k, wsum);
            scan_k<kIpThreads>(nf, fb, k, wsum);
            for (uint32_t b = tid; b < k; b += kIpThreads)
                for (uint32_t i = 0; i < nf[b]; ++i) blk[fb[b] + i] = b | (i << 16);
#pragma unroll
            for (uint32_t i = 0; i < R; ++i) {
                const uint32_t e = tid + i * kIpThreads;
                if (e < m) el[tb[bb[i]] + rr[i]] = vv[i];
            }
            __syncthreads();
            // full blocks -> the stripe's next block slots (all already consumed)
            const uint32_t NF = fb[k];
            for (uint32_t x = tid; x < NF * B; x += kIpThreads) {
                const uint32_t q = x / B, e = x % B;
                const uint32_t bi = blk[q], b = bi & 0xFFFFu, idx = (bi >> 16) * B + e;
                const uint32_t c = ccnt[b];
                const E v = idx < c ? carry[b * B + idx] : el[tb[b] + idx - c];
                ptr[sg.start + (slot0 + W + q) * B + e] = v;
            }
            for (uint32_t q = tid; q < NF; q += kIpThreads) ip.tags[tag0 + W + q] = (uint16_t)(blk[q] & 0xFFFFu);
            __syncthreads();
            // leftovers -> carry buffers
#pragma unroll
            for (uint32_t i = 0; i < R; ++i) {
                const uint32_t e = tid + i * kIpThreads;
                if (e < m) {
                    const uint32_t b = bb[i], idx = ccnt[b] + rr[i], f = nf[b] * B;
                    if (idx >= f) carry[b * B + idx - f] = vv[i];
                }
            }
            __syncthreads();
            for (uint32_t b = tid; b < k; b += kIpThreads) {
                ccnt[b] = ccnt[b] + cnt[b] - nf[b] * B;
                fcount[b] += nf[b];
                cnt[b] = 0;
            }
            W += NF;
            __syncthreads();
        }
        // stripe end: partial buffers, bucket totals, empty slots
        for (uint32_t x = tid; x < k * B; x += kIpThreads) {
            const uint32_t b = x / B, e = x % B;
            if (e < ccnt[b]) reinterpret_cast<E*>(ip.part)[((uint64_t)z * k + b) * B + e] = carry[x];
        }
        for (uint32_t b = tid; b < k; b += kIpThreads) {
            ip.pcnt[(uint64_t)z * k + b] = ccnt[b];
            if (fcount[b] || ccnt[b]) {
                atomicAdd((unsigned long long*)&ip.N[(uint64_t)s * k + b], (unsigned long long)fcount[b] * B + ccnt[b]);
                atomicAdd(&ip.F[(uint64_t)s * k + b], fcount[b]);
            }
        }
        for (uint64_t q = W + tid; q < nslots; q += kIpThreads) ip.tags[tag0 + q] = kTagEmpty;
        __syncthreads();
        for (uint32_t b = tid; b < k; b += kIpThreads) ccnt[b] = fcount[b] = 0;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- plan ----
// CTA per batch segment (grid-stride): S[s][0..k] (segment-relative bucket
// starts), and the (write, read) pointers of every bucket's block region.
__global__ void __launch_bounds__(256) k_ip_plan(RunParams rp, IpParams ip, uint32_t B) {
    ip = ip_resolve(ip);
    __shared__ unsigned long long wsum[256 / 32 + 1];
    __shared__ uint32_t work[kMaxK];
    const uint32_t k = rp.k, tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    for (uint32_t s = blockIdx.x; s < ip.nseg; s += gridDim.x) {
    const IpSeg sg = ip.segs[s];
    const uint64_t* N = ip.N + (uint64_t)s * k;
    uint64_t* S = ip.S + (uint64_t)s * (k + 1);
    const uint32_t per = (k + 255) / 256;
    const uint32_t x0 = min(k, tid * per), x1 = min(k, x0 + per);
    unsigned long long mine = 0;
    for (uint32_t x = x0; x < x1; ++x) mine += N[x];
    unsigned long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        unsigned long long r = 0;
        for (int w = 0; w < 8; ++w) {
            const unsigned long long c = wsum[w];
            wsum[w] = r;
            r += c;
        }
        wsum[8] = r;
    }
    __syncthreads();
    unsigned long long run = wsum[warp] + incl - mine;
    for (uint32_t x = x0; x < x1; ++x) {
        S[x] = run;
        run += N[x];
    }
    if (tid == 0) {
        S[k] = sg.len;
        if (wsum[8] != sg.len) atomicCAS(&rp.hdr->error, 0u, 7u);  // internal: counts lost
    }
    __syncthreads();
    const uint64_t nfb = sg.len / B;
    for (uint32_t d = tid; d < k; d += 256) {
        const uint64_t w = (S[d] + B - 1) / B;
        const uint64_t re = min((S[d + 1] + B - 1) / B, nfb);
        const uint64_t r = re + kRBias - 1;  // biased: may sit below w
        ip.wr[(uint64_t)s * k + d] = (w << 32) | (r & 0xFFFFFFFFull);
        work[d] = re > w ? (uint32_t)(re - w) : 0u;
    }
    __syncthreads();
    if (tid == 0) {  // per-segment prefix of the slots to read (k_ip_permute spreads its workers by it)
        uint64_t run = 0;
        for (uint32_t d = 0; d < k; ++d) {
            run += work[d];
            ip.regpre[(uint64_t)s * k + d] = (uint32_t)run;
        }
        ip.segtot[s] = run;
    }
    __syncthreads();
    }
}

// ------------------------------------------------------------------ P2 ----
// Every lane is a worker with at most one 128-byte block in hand; a warp
// moves its lanes' blocks together, one coalesced 128-byte load or store
// per block (32 lanes x 4 bytes), staging the blocks in hand in shared
// memory (hand: 32 blocks per warp; tmp: the blocks swapped out).
constexpr uint32_t kIpPermThreads = 256;
constexpr uint32_t kIpPermSmem = (kIpPermThreads / 32) * 32 * kIpBlockBytes + (kIpBatchCap + 1) * 8;  // ~40 KiB

template <int EB>
__global__ void __launch_bounds__(kIpPermThreads) k_ip_permute(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    constexpr uint32_t B = IpCfg<EB>::B;
    constexpr uint32_t W = kIpBlockBytes / 4;  // 32 words per block
    const uint32_t k = rp.k, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    unsigned char* base = rp.buf0;
    uint32_t* hand = reinterpret_cast<uint32_t*>(ism) + warp * (32 * W);
    uint64_t* segpre = reinterpret_cast<uint64_t*>(ism + (kIpPermThreads / 32) * 32 * kIpBlockBytes);
    const uint64_t P = (uint64_t)ip.nseg * k;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    // workers spread over the regions in proportion to their unprocessed slots:
    // worker g starts in the region holding slot g * G / T of the batch
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (uint32_t s = 0; s < ip.nseg; ++s) {
            segpre[s] = run;
            run += ip.segtot[s];
        }
        segpre[ip.nseg] = run;
    }
    __syncthreads();
    const uint64_t G = segpre[ip.nseg];
    bool done = G == 0;
    uint64_t p = 0;
    if (!done) {
        const uint64_t g = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * G / T;
        uint32_t lo = 0, hi = ip.nseg - 1;  // last segment with segpre <= g
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) / 2;
            if (segpre[mid] <= g) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t s = lo;
        const uint32_t gl = (uint32_t)(g - segpre[s]);
        const uint32_t* rp0 = ip.regpre + (uint64_t)s * k;
        uint32_t a = 0, b = k - 1;  // first region with inclusive prefix > gl
        while (a < b) {
            const uint32_t mid = (a + b) / 2;
            if (rp0[mid] > gl) b = mid;
            else a = mid + 1;
        }
        p = (uint64_t)s * k + a;
    }
    bool have = false;
    uint32_t t = 0;  // bucket of the block in hand
    for (;;) {
        // ---- A: lanes without a block claim the top unprocessed slot of a region
        bool need_load = false;
        const uint32_t* src = nullptr;
        uint64_t tagi = 0;
        if (!have && !done) {
            for (;;) {
                unsigned long long* wrp = (unsigned long long*)&ip.wr[p];
                const unsigned long long cur = *(volatile unsigned long long*)wrp;
                bool claimed = false;
                uint64_t slot = 0;
                if ((cur & 0xFFFFFFFFull) >= (cur >> 32) + kRBias) {
                    const unsigned long long old = atomicAdd(wrp, ~0ull);  // read -= 1
                    const uint64_t ow = old >> 32, orb = old & 0xFFFFFFFFull;
                    if (orb >= ow + kRBias) {
                        claimed = true;
                        slot = orb - kRBias;
                    }
                }
                if (!claimed) {  // region exhausted: sweep the pairs once more through the cursor
                    const uint64_t np = atomicAdd(ip.cursor, 1ull);
                    if (np >= P) {
                        done = true;
                        break;
                    }
                    p = np;
                    continue;
                }
                const IpSeg sg = ip.segs[(uint32_t)(p / k)];
                tagi = sg.start / B + slot;
                const uint32_t tg = ip.tags[tagi];
                if (tg == kTagEmpty) continue;
                t = tg;
                src = reinterpret_cast<const uint32_t*>(base + (sg.start + slot * B) * EB);
                need_load = true;
                break;
            }
        }
        const uint32_t ldm = __ballot_sync(0xFFFFFFFFu, need_load);
        for (uint32_t m = ldm; m; m &= m - 1) {
            const uint32_t q = __ffs(m) - 1;
            const uint32_t* sq = reinterpret_cast<const uint32_t*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)src, q));
            hand[q * W + lane] = sq[lane];
        }
        __syncwarp();
        if (need_load) {
            __threadfence();
            *(volatile uint16_t*)&ip.tags[tagi] = kTagRead;
            have = true;
        }
        // ---- B: place each block in hand at the write pointer of its bucket's region
        bool swap = false, store = false;
        uint32_t* dst = nullptr;
        const uint32_t* ssrc = nullptr;
        uint32_t t2 = 0;
        if (have) {
            const uint32_t s = (uint32_t)(p / k);
            const IpSeg sg = ip.segs[s];
            const uint64_t q = (uint64_t)s * k + t;
            const unsigned long long old = atomicAdd((unsigned long long*)&ip.wr[q], 1ull << 32);
            const uint64_t ow = old >> 32, orb = old & 0xFFFFFFFFull;
            const bool owned = orb >= ow + kRBias;  // slot ow still unprocessed: ours
            const uint64_t bend = ip.S[(uint64_t)s * (k + 1) + t + 1];
            const uint64_t ti = sg.start / B + ow;
            uint32_t* slotp = reinterpret_cast<uint32_t*>(base + (sg.start + ow * B) * EB);
            const bool overflow = (ow + 1) * B > bend;
            if (owned) {
                t2 = ip.tags[ti];
                if (t2 != kTagEmpty) {
                    swap = true;
                    ssrc = slotp;
                }
            } else if (!overflow) {
                // a reader claimed the slot: wait until its block has been copied out
                for (;;) {
                    const uint16_t tv = *(volatile uint16_t*)&ip.tags[ti];
                    if (tv == kTagRead || tv == kTagEmpty) break;
                    __nanosleep(32);
                }
                __threadfence();
            }
            if (overflow) {  // the block would cross its bucket's end: overflow block of (s, bucket)
                dst = reinterpret_cast<uint32_t*>(ip.ovfd + q * kIpBlockBytes);
                ip.ovf[q] = 1u;
            } else {
                dst = slotp;
            }
            store = true;
        }
        // blocks swapped out are read before the stores, into registers (lane l
        // holds word l of every swapped block: tr[q] for the block of lane q)
        const uint32_t swm = __ballot_sync(0xFFFFFFFFu, swap);
        uint32_t tr[32];
        if (swm) {
#pragma unroll
            for (uint32_t q = 0; q < 32; ++q) {
                const uint32_t* sq =
                    reinterpret_cast<const uint32_t*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)ssrc, q));
                if ((swm >> q) & 1u) tr[q] = sq[lane];
            }
        }
        const uint32_t stm = __ballot_sync(0xFFFFFFFFu, store);
        for (uint32_t m = stm; m; m &= m - 1) {
            const uint32_t q = __ffs(m) - 1;
            uint32_t* dq = reinterpret_cast<uint32_t*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)dst, q));
            dq[lane] = hand[q * W + lane];
        }
        __syncwarp();
        if (swm) {
#pragma unroll
            for (uint32_t q = 0; q < 32; ++q)
                if ((swm >> q) & 1u) hand[q * W + lane] = tr[q];
        }
        __syncwarp();
        if (have) {
            if (swap) t = t2;
            else have = false;
        }
        if (__ballot_sync(0xFFFFFFFFu, have || !done) == 0) break;
    }
}

// ------------------------------------------------------------------ P3 ----
// Warp per (segment, bucket): fill head and tail from the overflow block and
// the stripes' partial buffers; queue children longer than S_fuse.
template <int EB>
__global__ void __launch_bounds__(256) k_ip_fill(RunParams rp, IpParams ip) {
    ip = ip_resolve(ip);
    using E = typename ElemT<EB>::type;
    constexpr uint32_t B = IpCfg<EB>::B;
    const uint32_t k = rp.k, lane = threadIdx.x & 31u;
    E* ptr = reinterpret_cast<E*>(rp.buf0);
    const uint64_t P = (uint64_t)ip.nseg * k;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t q = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); q < P; q += warps) {
        const uint32_t s = (uint32_t)(q / k), d = (uint32_t)(q % k);
        const IpSeg sg = ip.segs[s];
        const uint64_t Sd = ip.S[(uint64_t)s * (k + 1) + d], Sd1 = ip.S[(uint64_t)s * (k + 1) + d + 1];
        const uint32_t o = ip.ovf[q];
        const uint64_t Fp = ip.F[q] - o;  // blocks placed in place
        const uint64_t H = (Sd + B - 1) / B * B;
        const uint64_t hend = min(H, Sd1);
        const uint64_t tstart = max(hend, min(H + Fp * B, Sd1));
        const uint64_t hlen = hend - Sd;
        auto dest = [&](uint64_t idx) -> uint64_t { return sg.start + (idx < hlen ? Sd + idx : tstart + (idx - hlen)); };
        uint64_t base = 0;
        if (o) {
            for (uint32_t e = lane; e < B; e += 32) ptr[dest(e)] = reinterpret_cast<const E*>(ip.ovfd)[q * B + e];
            base = B;
        }
        for (uint32_t z0 = 0; z0 < sg.nz; z0 += 32) {
            const uint32_t z = sg.zbase + z0 + lane;
            const uint32_t c = (z0 + lane < sg.nz) ? ip.pcnt[(uint64_t)z * k + d] : 0u;
            const uint32_t incl = warp_inclusive_sum(c);
            const uint64_t my = base + incl - c;
            const E* src = reinterpret_cast<const E*>(ip.part) + ((uint64_t)z * k + d) * B;
            for (uint32_t e = 0; e < c; ++e) ptr[dest(my + e)] = src[e];
            base += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        if (lane == 0) {
            if (base != (hend - Sd) + (Sd1 - tstart)) atomicCAS(&rp.hdr->error, 0u, 7u);  // internal check
            const uint64_t len = Sd1 - Sd;
            if (len > rp.S_fuse && ip.level + 1 < rp.max_levels) {
                const uint32_t at = atomicAdd(ip.nnext, 1u);
                if (at < ip.max_next) ip.next[at] = IpSeg{sg.start + Sd, len, 0u, 0u};
                else atomicCAS(&rp.hdr->error, 0u, 7u);
            }
            ip.N[q] = 0;
            ip.F[q] = 0;
            ip.ovf[q] = 0;
        }
    }
}

// ------------------------------------------------ device-driven loop ----
// The level loop of the in-place mode runs on the device (shuf_api.cu builds a
// CUDA graph: WHILE(levels){ k_ip_level_plan; WHILE(batches){ batch kernels;
// k_ip_batch_next }; k_ip_level_next }).  No host round trip per level.

// Level 0: the root segment, loop state.
__global__ void k_ip_init(IpParams ip, Header* hdr, uint64_t n, IpState init) {
    hdr->root_off[0] = 0;
    hdr->root_off[1] = n;
    ip.segbase[0][0] = IpSeg{0, n, 0u, 0u};
    IpState* st = ip.state;
    *st = init;
    st->level = 0;
    st->cur = 0;
    st->batch = 0;
    st->nbatch = 0;
    st->nseg = 1;
}

// Cut the level's segment list into batches: with P_s the exclusive prefix of
// the segments' stripe counts, segment s goes to batch floor(P_s / C).  A
// segment has at most C stripes (shuf_api.cu chooses Z so), so a batch holds
// fewer than 2C <= cap stripes and segments; batch indices a long segment
// jumps over stay empty (their kernels return at once).
__global__ void __launch_bounds__(1024) k_ip_level_plan(RunParams rp, IpParams ip, cudaGraphConditionalHandle hb) {
    __shared__ uint32_t wsum[1024 / 32 + 1];
    __shared__ unsigned long long tot;
    IpState* st = ip.state;
    const uint32_t cur = st->cur, tid = threadIdx.x;
    const IpSeg* segs = ip.segbase[cur];
    uint32_t nseg = st->level == 0 ? 1u : ip.nnext_base[cur];
    if (nseg > ip.max_next) {  // list overflow (cannot happen with the planned capacity)
        if (tid == 0) atomicCAS(&rp.hdr->error, 0u, 7u);
        nseg = 0;
    }
    const uint32_t C = st->C;
    // total stripes -> number of batches
    if (tid == 0) tot = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (uint32_t x = tid; x < nseg; x += 1024) mine += (segs[x].len + ip.Z - 1) / ip.Z;
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    if ((tid & 31u) == 0 && mine) atomicAdd(&tot, mine);
    __syncthreads();
    uint32_t nb = (uint32_t)((tot + C - 1) / C);
    if (nb > st->max_batches) {
        if (tid == 0) atomicCAS(&rp.hdr->error, 0u, 7u);
        nb = 0;
        nseg = 0;
    }
    for (uint32_t b = tid; b < nb; b += 1024) st->batches[b] = IpBatch{0u, 0u, 0u, 0xFFFFFFFFu};
    __syncthreads();
    uint32_t base = 0;
    for (uint32_t s0 = 0; s0 < nseg; s0 += 1024) {
        const uint32_t s = s0 + tid;
        const uint32_t nz = s < nseg ? (uint32_t)((segs[s].len + ip.Z - 1) / ip.Z) : 0u;
        uint32_t total;
        const uint32_t ex = block_exclusive_sum<1024>(nz, wsum, &total);
        if (s < nseg) {
            const uint32_t b = (base + ex) / C;
            atomicMin(&st->batches[b].first, s);
            atomicAdd(&st->batches[b].nz, nz);
        }
        base += total;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t nxt = nseg;
        for (int32_t b = (int32_t)nb - 1; b >= 0; --b) {
            IpBatch& bt = st->batches[b];
            if (bt.first == 0xFFFFFFFFu) {
                bt.s0 = nxt;
                bt.nseg = 0;
            } else {
                bt.s0 = bt.first;
                bt.nseg = nxt - bt.first;
                nxt = bt.first;
            }
        }
        st->nbatch = nb;
        st->batch = 0;
        st->nseg = nseg;
        ip.nnext_base[cur ^ 1u] = 0;
        *ip.cursor = 0;
        cudaGraphSetConditional(hb, nb > 0 ? 1u : 0u);
    }
}

__global__ void k_ip_batch_next(IpParams ip, cudaGraphConditionalHandle hb) {
    IpState* st = ip.state;
    const uint32_t b = ++st->batch;
    *ip.cursor = 0;
    cudaGraphSetConditional(hb, b < st->nbatch ? 1u : 0u);
}

__global__ void k_ip_level_next(RunParams rp, IpParams ip, cudaGraphConditionalHandle hl) {
    IpState* st = ip.state;
    const uint32_t nn = ip.nnext_base[st->cur ^ 1u];
    st->cur ^= 1u;
    st->level += 1;
    bool more = nn > 0;
    if (more && st->level >= kMaxLevels) {
        atomicCAS(&rp.hdr->error, 0u, 5u);  // SHUF_ERR_DEPTH
        more = false;
    }
    cudaGraphSetConditional(hl, more ? 1u : 0u);
}

cudaError_t launch_ip_init(const IpParams& ip, Header* hdr, uint64_t n, const IpState& init, cudaStream_t s) {
    k_ip_init<<<1, 1, 0, s>>>(ip, hdr, n, init);
    return cudaGetLastError();
}
cudaError_t launch_ip_level_plan(const RunParams& rp, const IpParams& ip, cudaGraphConditionalHandle hb,
                                 cudaStream_t s) {
    k_ip_level_plan<<<1, 1024, 0, s>>>(rp, ip, hb);
    return cudaGetLastError();
}
cudaError_t launch_ip_batch_next(const IpParams& ip, cudaGraphConditionalHandle hb, cudaStream_t s) {
    k_ip_batch_next<<<1, 1, 0, s>>>(ip, hb);
    return cudaGetLastError();
}
cudaError_t launch_ip_level_next(const RunParams& rp, const IpParams& ip, cudaGraphConditionalHandle hl,
                                 cudaStream_t s) {
    k_ip_level_next<<<1, 1, 0, s>>>(rp, ip, hl);
    return cudaGetLastError();
}

// ------------------------------------------------------------- dispatch ---
__global__ void k_ip_root(Header* hdr, uint64_t n) {
    hdr->root_off[0] = 0;
    hdr->root_off[1] = n;
}

cudaError_t launch_ip_root(Header* hdr, uint64_t n, cudaStream_t s) {
    k_ip_root<<<1, 1, 0, s>>>(hdr, n);
    return cudaGetLastError();
}

static void* ip_fn(uint32_t eb, int which) {
    switch (eb) {
    case 4: return which == 0 ? (void*)k_ip_classify<4> : which == 1 ? (void*)k_ip_permute<4> : (void*)k_ip_fill<4>;
    case 8: return which == 0 ? (void*)k_ip_classify<8> : which == 1 ? (void*)k_ip_permute<8> : (void*)k_ip_fill<8>;
    default:
        return which == 0 ? (void*)k_ip_classify<16> : which == 1 ? (void*)k_ip_permute<16> : (void*)k_ip_fill<16>;
    }
}

cudaError_t configure_inplace(uint32_t eb, uint32_t k) {
    cudaError_t e = cudaFuncSetAttribute(ip_fn(eb, 0), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e) return e;
    return cudaFuncSetAttribute(ip_fn(eb, 1), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
}

cudaError_t occupancy_inplace(uint32_t eb, uint32_t k, int* classify, int* permute) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(classify, ip_fn(eb, 0), kIpThreads,
                                                                  ip_classify_smem_bytes(eb, k));
    if (e) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(permute, ip_fn(eb, 1), kIpPermThreads, kIpPermSmem);
}

cudaError_t launch_ip_stripes(const IpParams& ip, cudaStream_t s) {
    k_ip_stripes<<<1, 256, 0, s>>>(ip);
    return cudaGetLastError();
}

cudaError_t launch_ip_classify(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp, (void*)&ip};
    const int g = ip.state ? grid : (int)min((uint64_t)grid, (uint64_t)ip.nstripes);  // device-resolved batch: any size
    return cudaLaunchKernel(ip_fn(rp.eb, 0), dim3(g), dim3(kIpThreads), args, ip_classify_smem_bytes(rp.eb, rp.k), s);
}

cudaError_t launch_ip_plan(const RunParams& rp, const IpParams& ip, cudaStream_t s) {
    k_ip_plan<<<ip.state ? kIpBatchCap : ip.nseg, 256, 0, s>>>(rp, ip, kIpBlockBytes / rp.eb);
    return cudaGetLastError();
}

cudaError_t launch_ip_permute(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp, (void*)&ip};
    return cudaLaunchKernel(ip_fn(rp.eb, 1), dim3(grid), dim3(kIpPermThreads), args, kIpPermSmem, s);
}

cudaError_t launch_ip_fill(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid) {
    void* args[] = {(void*)&rp, (void*)&ip};
    const uint64_t warps = (uint64_t)ip.nseg * rp.k;
    const int g = ip.state ? grid : (int)min((uint64_t)grid, (warps + 7) / 8);
    return cudaLaunchKernel(ip_fn(rp.eb, 2), dim3(g), dim3(256), args, 0, s);
}

}  // namespace shuf
