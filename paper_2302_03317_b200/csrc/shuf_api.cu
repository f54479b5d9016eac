// C ABI of libshuf.so (include/shuf.h): plan, scratch layout, stream-ordered
// level loop.  No host synchronisation and no allocation inside shuf_run /
// shuf_segmented: every level's work list lives on the device and each
// kernel is a persistent grid that reads its own work count.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/shuf.h"
#include "philox.cuh"
#include "shuf_internal.cuh"

using namespace shuf;

// Byte offsets of the in-place mode's auxiliary buffer (kernels_inplace.cu).
struct IpAuxLayout {
    uint64_t header, ctr, state, batches, segs[2], zseg, N, F, S, wr, regpre, segtot, ovf, ovfd, pcnt, part, tags, flags,
        total;
    uint64_t Z, max_segs, max_batches;
    uint32_t cap, C;
};

struct shuf_plan_s {
    uint64_t n;
    uint32_t eb, k, L;
    uint64_t seed;
    uint32_t S_fuse, chunk, levels, fin_nbuf;
    uint32_t S_stream;  // children with S_fuse < len <= S_stream: k_finish_stream (0: none)
    int defer_planned;  // SHUF_DEFER=1 at plan time: item records are laid out
    ScratchLayout lay;  // shuf_run's layout (one level-0 segment)
    IpAuxLayout ipl;
    // device setup (lazily, first run)
    bool dev_ready;
    int sms;
    int grid_hist, grid_scan, grid_scatter, grid_finish, grid_small, grid_fast, grid_leaf;
    int fast, leafk, defer;
    int hist_overlap;             // 1: level l+1's histogram runs on side_stream during level l's scatter
    double leaf_sigma;            // small-slot leaf pass: slots hold avg + leaf_sigma * sqrt(avg) elements (< 0: off)
    cudaStream_t side_stream;
    cudaEvent_t ev_fork, ev_join;
    bool ip_ready;
    int grid_ipc, grid_ipp;
    // in-place mode: the device-driven level loop as an instantiated CUDA graph,
    // cached for the (ptr, aux, max_levels, run_leaves) it was built for
    cudaGraphExec_t ip_exec;
    cudaStream_t ip_cap_stream;
    void *ip_ptr, *ip_aux;
    uint32_t ip_maxlv;
    int ip_leaves;
    uint64_t ip_nodes;
    // elem_bytes outside {4, 8, 16}: the gather route (kernels_gather.cu) --
    // `idx` shuffles the index array 0..n-1, then the elements move once
    struct shuf_plan_s* idx;
    int rank_ordered;
    uint32_t finish_smem, scatter_smem;
    int last_cuda_error;
    uint64_t last_launches;
    Header* last_hdr;
};

static thread_local shuf_status g_last_status = SHUF_OK;

static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Largest S with finish_smem_bytes(S) <= the opt-in shared-memory limit,
// capped by the ranking registers (finish_max_elems), u16 tile-local
// offsets, and in-smem frontiers (<= S/(L+1) entries <= kFrontierCap).
static uint32_t pick_s_fuse_nbuf(uint32_t eb, uint32_t k, uint32_t L, uint32_t nbuf) {
    uint32_t lo = 1, hi = 65535;
    while (lo < hi) {
        uint32_t mid = (lo + hi + 1) / 2;
        if (finish_smem_bytes(mid, eb, k, nbuf) <= finish_smem_budget(eb)) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t rmax = finish_max_elems(eb, k);
    if (rmax < lo) lo = rmax;
    uint64_t cap = (uint64_t)kFrontierCap * ((uint64_t)L + 1);
    if (cap < lo) lo = (uint32_t)cap;
    return lo;
}

static uint32_t pick_s_fuse(uint32_t eb, uint32_t k, uint32_t L, uint32_t* nbuf) {
    const uint32_t s2 = pick_s_fuse_nbuf(eb, k, L, 2), s1 = pick_s_fuse_nbuf(eb, k, L, 1);
    // double-buffer the items unless that costs more than 10% of the fusable size
    *nbuf = (10ull * s2 >= 9ull * s1) ? 2u : 1u;
    return *nbuf == 2 ? s2 : s1;
}

// Global levels needed until the largest segment fits S_fuse, with a
// 6-sigma binomial margin per level, plus one spare level (a rarer outlier
// child simply takes the spare level; only one that outlives the spare
// level too raises SHUF_ERR_DEPTH).
static uint32_t plan_levels(uint64_t n, uint32_t k, uint32_t S_fuse, uint32_t S_eff) {
    if (n <= S_fuse) return 0;
    double m = (double)n;
    uint32_t g = 0;
    while (m > S_eff && g < kMaxLevels) {
        ++g;
        double mu = m / k;
        m = mu + 6.0 * std::sqrt(mu) + 32.0;
        if (m >= (double)n) m = (double)n;  // k small: still shrinks in expectation
        if (g > 200) break;
    }
    return g + 1 > kMaxLevels ? kMaxLevels : g + 1;
}

// Upper bounds on the segments and chunks of every planned level (DESIGN.md
// 5).  A single shuffle starts from one segment; level l+1's segments are
// the children of level l's longer than S_fuse.  Each child of a parent of
// mean size m is Binomial(m, 1/k): with p = P(child > S_fuse) (normal
// approximation) the bound is E + 6 sqrt(E) + 4 for E = N p, N the number
// of children, capped by N and by n / (S_fuse + 1).  Segmented mode starts
// from up to segs0 user segments of unknown lengths, so every level takes the
// worst case min(N, n / (S_fuse + 1) + 1).  A level beyond its bound latches
// SHUF_ERR_SCRATCH (k_plan / k_init_segmented).
static void level_caps(uint64_t n, uint32_t k, uint32_t S, uint64_t C, uint32_t levels, uint64_t segs0,
                       bool segmented, uint64_t* segcap, uint64_t* chunkcap) {
    const double worst = (double)(n / ((uint64_t)S + 1) + 1);
    double cnt = (double)segs0, mean = segs0 ? (double)n / (double)segs0 : 0.0;
    for (uint32_t l = 0; l < levels; ++l) {
        double segs, elems;
        if (l == 0) {
            segs = cnt;
            elems = (double)n;
        } else {
            const double N = cnt * k;
            if (segmented) {
                segs = N < worst ? N : worst;
                elems = (double)n;
            } else {
                const double mu = mean / k, sd = std::sqrt(mean * (1.0 / k) * (1.0 - 1.0 / k)) + 1e-9;
                const double z = ((double)S + 0.5 - mu) / sd;
                const double pr = 0.5 * std::erfc(z / std::sqrt(2.0));
                const double E = N * pr;
                segs = std::ceil(E + 6.0 * std::sqrt(E) + 4.0);
                if (segs > N) segs = N;
                if (segs > worst) segs = worst;
                const double big = mu + 6.0 * sd + 32.0;
                elems = segs * (big > S + 1.0 ? big : S + 1.0);
                if (elems > (double)n) elems = (double)n;
                mean = mu > S + 1.0 ? mu : S + 1.0;
            }
        }
        if (segs < 1) segs = 1;
        cnt = segs;
        segcap[l] = (uint64_t)segs;
        chunkcap[l] = (uint64_t)(elems / (double)C) + (uint64_t)segs + 1;
    }
}

// Scratch layout for up to segs0 level-0 segments (1 for shuf_run,
// min(num_segments, n / (S_fuse + 1) + 1) for shuf_segmented).
static ScratchLayout compute_layout(const shuf_plan_s* p, uint64_t segs0, bool segmented) {
    ScratchLayout l{};
    const uint64_t n = p->n;
    std::vector<uint64_t> sc(p->levels + 1, 0), cc(p->levels + 1, 0);
    const uint32_t S_eff = p->S_stream ? p->S_stream : p->S_fuse;  // children above it take another HBM level
    if (p->levels) level_caps(n, p->k, S_eff, p->chunk, p->levels, segs0, segmented, sc.data(), cc.data());
    for (int s = 0; s < 2; ++s) {
        l.seg_cap[s] = l.chunk_cap[s] = 1;
        for (uint32_t lv = (uint32_t)s; lv < p->levels; lv += 2) {
            if (sc[lv] > l.seg_cap[s]) l.seg_cap[s] = sc[lv];
            if (cc[lv] > l.chunk_cap[s]) l.chunk_cap[s] = cc[lv];
        }
        l.entry_cap[s] = l.chunk_cap[s] * p->k;
        l.tile_cap[s] = (l.entry_cap[s] + kScanTile - 1) / kScanTile + 1;
    }
    uint64_t off = 0;
    l.pingpong = off;
    off = align_up(off + n * p->eb + 16, 256);
    l.header = off;
    off = align_up(off + sizeof(Header), 256);
    for (int s = 0; s < 2; ++s) {
        l.segs[s] = off;
        off = align_up(off + l.seg_cap[s] * sizeof(SegDesc), 256);
        l.chunks[s] = off;
        off = align_up(off + l.chunk_cap[s] * sizeof(ChunkDesc), 256);
        l.counts[s] = off;
        off = align_up(off + l.entry_cap[s] * 4, 256);
        l.prefix[s] = off;
        off = align_up(off + l.entry_cap[s] * 8, 256);
        l.status[s] = off;
        off = align_up(off + l.tile_cap[s] * 8, 256);
    }
    const uint64_t maxseg = l.seg_cap[0] > l.seg_cap[1] ? l.seg_cap[0] : l.seg_cap[1];
    l.flags = off;
    off = align_up(off + maxseg * p->k, 256);
    l.max_items = p->defer_planned ? n / ((uint64_t)p->L + 1) + 1 : 0;
    l.items = off;
    off = align_up(off + l.max_items * item_rec_stride(p->k), 256);
    l.max_fused = n / ((uint64_t)p->L + 1) + 1;
    l.fused = off;
    off = align_up(off + l.max_fused * 4, 256);
    l.total = off;
    l.meta = l.total - (n * p->eb);
    return l;
}

// In-place aux: batches of < 2C <= cap stripes / segments; stripes of Z
// elements (a multiple of the block and of the classify tile) chosen so that
// one segment never has more than C stripes (k_ip_level_plan).
static void compute_ip_layout(shuf_plan_s* p) {
    IpAuxLayout& l = p->ipl;
    const uint64_t n = p->n, k = p->k;
    const uint64_t B = kIpBlockBytes / p->eb;
    // batch capacity: the per-(stripe|segment, bucket) buffers (~2 blocks + 32 B each) stay within
    // ~2.5 % of the data plus 16 MiB, and between 64 and kIpBatchCap entries (aux total < 5 % of the data
    // above 1 GiB, tests/test_library_cpu.py)
    const uint64_t per = k * (2 * kIpBlockBytes + 32);
    uint64_t capb = (n * p->eb / 40 + (16ull << 20)) / per;
    capb = capb < 64 ? 64 : (capb > kIpBatchCap ? kIpBatchCap : capb);
    l.C = (uint32_t)(capb / 2);
    l.Z = align_up((n + l.C - 1) / l.C, 4096);
    if (l.Z < 65536) l.Z = 65536;
    l.max_segs = n / ((uint64_t)p->S_fuse + 1) + 1;
    uint64_t cap = n / l.Z + l.max_segs + 1;
    l.cap = (uint32_t)(cap < capb ? cap : capb);
    if (l.cap < l.C) l.C = l.cap;
    l.max_batches = (n / l.Z + l.max_segs + 1) / l.C + 2;
    uint64_t off = 0;
    auto take = [&off](uint64_t bytes) {
        const uint64_t at = off;
        off = align_up(off + bytes, 256);
        return at;
    };
    l.header = take(sizeof(Header));
    l.ctr = take(sizeof(IpCounters));
    l.state = take(sizeof(IpState));
    l.batches = take(l.max_batches * sizeof(IpBatch));
    l.segs[0] = take(l.max_segs * sizeof(IpSeg));
    l.segs[1] = take(l.max_segs * sizeof(IpSeg));
    l.zseg = take((uint64_t)l.cap * 4);
    l.N = take((uint64_t)l.cap * k * 8);
    l.F = take((uint64_t)l.cap * k * 4);
    l.S = take((uint64_t)l.cap * (k + 1) * 8);
    l.wr = take((uint64_t)l.cap * k * 8);
    l.regpre = take((uint64_t)l.cap * k * 4);
    l.segtot = take((uint64_t)l.cap * 8);
    l.ovf = take((uint64_t)l.cap * k * 4);
    l.ovfd = take((uint64_t)l.cap * k * kIpBlockBytes);
    l.pcnt = take((uint64_t)l.cap * k * 4);
    l.part = take((uint64_t)l.cap * k * kIpBlockBytes);
    l.tags = take((n / B + 2) * 2);
    l.flags = take((uint64_t)l.cap * k);  // per batch child: 1 = the general finish takes it
    l.total = off;
}

extern "C" shuf_plan_t shuf_plan(uint64_t n, uint32_t elem_bytes, uint32_t k, uint32_t L, uint64_t seed) {
    g_last_status = SHUF_OK;
    if (elem_bytes > kMaxGatherElem) {
        g_last_status = SHUF_ERR_UNSUPPORTED;
        return nullptr;
    }
    if (elem_bytes != 0 && !(elem_bytes == 4 || elem_bytes == 8 || elem_bytes == 16)) {
        // gather route: D6's permutation of n elements does not depend on their size
        shuf_plan_s* ix = shuf_plan(n, n <= 0xFFFFFFFFull ? 4u : 8u, k, L, seed);
        if (!ix) return nullptr;
        shuf_plan_s* p = new (std::nothrow) shuf_plan_s();
        if (!p) {
            shuf_destroy(ix);
            g_last_status = SHUF_ERR_INVALID_ARG;
            return nullptr;
        }
        p->n = n;
        p->eb = elem_bytes;
        p->k = k;
        p->L = L;
        p->seed = seed;
        p->S_fuse = ix->S_fuse;
        p->chunk = ix->chunk;
        p->levels = ix->levels;
        p->idx = ix;
        return p;
    }
    if (elem_bytes == 0 || k < 2 || k > 65536 || L < 1) {
        g_last_status = SHUF_ERR_INVALID_ARG;
        return nullptr;
    }
    if (k > kMaxK) {
        g_last_status = SHUF_ERR_UNSUPPORTED;
        return nullptr;
    }
    uint32_t nbuf = 1;
    uint32_t S = pick_s_fuse(elem_bytes, k, L, &nbuf);
    {  // SHUF_SFUSE=<elements>: a smaller fusable size (e.g. L: every level in HBM)
        const char* sf = std::getenv("SHUF_SFUSE");
        const long v = sf ? std::atol(sf) : 0;
        if (v >= (long)L && v < (long)S) S = (uint32_t)v;
    }
    if (L > S) {
        g_last_status = SHUF_ERR_UNSUPPORTED;
        return nullptr;
    }
    shuf_plan_s* p = new (std::nothrow) shuf_plan_s();
    if (!p) {
        g_last_status = SHUF_ERR_INVALID_ARG;
        return nullptr;
    }
    p->n = n;
    p->eb = elem_bytes;
    p->k = k;
    p->L = L;
    p->seed = seed;
    p->S_fuse = S;
    p->fin_nbuf = nbuf;
    const uint32_t T = scatter_tile_bytes(elem_bytes) / elem_bytes;  // scatter tile (kernels_scatter.cu SCfg)
    // chunks per level: at most 4096 (balanced over the persistent grid), and
    // few enough that a level's count + prefix tables (12 B per (bucket,
    // chunk)) stay within ~0.5 % of the data each
    uint64_t target = (n * (uint64_t)elem_bytes) / (2400ull * k);
    if (target < 1) target = 1;
    if (target > 4096) target = 4096;
    uint64_t C = (n + target - 1) / target;
    {  // SHUF_CHUNK=<elements>: another chunk size (test hook: the result must not depend on it)
        const char* ce = std::getenv("SHUF_CHUNK");
        const long long v = ce ? std::atoll(ce) : 0;
        if (v > 0) C = (uint64_t)v;
    }
    C = align_up(C < T ? T : C, T);
    if (C > 0x40000000ull) C = 0x40000000ull;
    p->chunk = (uint32_t)C;
    {  // single-buffer streaming finish (k_finish_stream) for children too long for the fused size,
       // when their own children stay far below L (> 12 sigma); SHUF_STREAM=0 disables it
        uint32_t Ss = 0;
        for (uint32_t c = 65535u; c > S; c -= 64u)
            if (finish_stream_smem_bytes(c, elem_bytes, k) <= kSmemLimit) {
                Ss = c;
                break;
            }
        const double mc = (double)Ss / k;
        const char* se = std::getenv("SHUF_STREAM");
        const bool on = !(se && se[0] == '0') && Ss >= S + S / 8 && mc + 12.0 * std::sqrt(mc) + 32.0 <= (double)L;
        p->S_stream = on ? Ss : 0u;
    }
    p->levels = plan_levels(n, k, S, p->S_stream ? p->S_stream : S);
    {  // SHUF_LEVELS=<n>: fewer planned HBM levels (test hook for the device depth check)
        const char* le = std::getenv("SHUF_LEVELS");
        const long v = le ? std::atol(le) : -1;
        if (v >= 0 && (uint32_t)v < p->levels) p->levels = (uint32_t)v;
    }
    {
        const char* df = std::getenv("SHUF_DEFER");
        p->defer_planned = (df && df[0] == '1') ? 1 : 0;
    }
    p->lay = compute_layout(p, n > S ? 1 : 0, false);
    compute_ip_layout(p);
    return p;
}

extern "C" shuf_status shuf_last_status(void) { return g_last_status; }

// Gather route scratch: [index plan's scratch | index array | staging buffer].
static uint64_t gather_extra(const shuf_plan_s* p) {
    return align_up(p->n * p->idx->eb, 256) + align_up(p->n * p->eb, 256);
}

extern "C" shuf_status shuf_scratch_bytes(shuf_plan_t p, uint64_t* bytes) {
    if (!p || !bytes) return SHUF_ERR_INVALID_ARG;
    *bytes = p->idx ? align_up(p->idx->lay.total, 256) + gather_extra(p) : p->lay.total;
    return SHUF_OK;
}

extern "C" uint32_t shuf_planned_levels(shuf_plan_t p) { return p ? p->levels : 0; }
extern "C" int shuf_last_cuda_error(shuf_plan_t p) { return p ? p->last_cuda_error : 0; }
extern "C" uint64_t shuf_last_launch_count(shuf_plan_t p) { return p ? p->last_launches : 0; }

static shuf_status cuda_fail(shuf_plan_s* p, cudaError_t e) {
    if (p) p->last_cuda_error = (int)e;
    return SHUF_ERR_CUDA;
}

// One-time (per process) check that same-address shared atomics of a warp
// return in lane order (block_ops.cuh); SHUF_RANK_MODE=match|atomic overrides.
static int g_rank_ordered = -1;
static std::mutex g_probe_mu;

static cudaError_t probe_rank_order(int sms, int* ordered) {
    std::lock_guard<std::mutex> lk(g_probe_mu);
    if (g_rank_ordered >= 0) {
        *ordered = g_rank_ordered;
        return cudaSuccess;
    }
    const char* env = std::getenv("SHUF_RANK_MODE");
    if (env && std::strcmp(env, "match") == 0) {
        g_rank_ordered = 0;
    } else if (env && std::strcmp(env, "atomic") == 0) {
        g_rank_ordered = 1;
    } else {
        uint32_t* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(uint32_t));
        if (e) return e;
        uint32_t h = 0;
        if (!(e = cudaMemset(d, 0, sizeof(uint32_t))) && !(e = launch_rank_order_probe(sms, d, 0)) &&
            !(e = cudaDeviceSynchronize()))
            e = cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
        cudaFree(d);
        if (e) return e;
        g_rank_ordered = (h == 0) ? 1 : 0;
    }
    *ordered = g_rank_ordered;
    return cudaSuccess;
}

extern "C" int shuf_rank_mode(void) { return g_rank_ordered; }

static cudaError_t device_setup(shuf_plan_s* p) {
    if (p->dev_ready) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    if ((e = cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = probe_rank_order(p->sms, &p->rank_ordered))) return e;
    p->finish_smem = finish_smem_bytes(p->S_fuse, p->eb, p->k, p->fin_nbuf);
    p->scatter_smem = scatter_smem_bytes(p->eb, p->k);
    if ((e = configure_finish(p->finish_smem))) return e;
    if (p->S_stream && (e = configure_finish_stream(p->eb, finish_stream_smem_bytes(p->S_stream, p->eb, p->k)))) return e;
    if ((e = configure_scatter(p->scatter_smem))) return e;
    // pipelined finish (kernels_fast.cu) for single-level items; SHUF_FAST_FINISH=0
    // leaves every item to the general finish kernel
    {
        const char* ff = std::getenv("SHUF_FAST_FINISH");
        p->fast = (p->k <= kMaxK && !(ff && ff[0] == '0') &&
                   fast_smem_bytes(p->eb, p->k) <= kSmemLimit)
                      ? 1
                      : 0;
        if (p->fast && (e = configure_fast(p->eb, p->k))) return e;
    }
    // leaf kernel (kernels_leaf.cu): SHUF_LEAF=0 keeps leaves in the finish kernel
    {
        const char* lf = std::getenv("SHUF_LEAF");
        p->leafk = (lf && lf[0] == '0') ? 0 : 1;
        if (p->leafk && leaf_smem_bytes(p->eb, p->L) > kSmemLimit) p->leafk = 0;
        if (p->leafk && (e = configure_leaf(p->eb, p->L))) return e;
        // SHUF_DEFER=1: fused items whose children are all leaves leave them to the leaf kernel
        // (one more HBM round trip; measured slower on HOT)
        const char* df = std::getenv("SHUF_DEFER");
        p->defer = (p->leafk && p->defer_planned && df && df[0] == '1') ? 1 : 0;
    }
    // the next level's histogram (reads no data: positions only) on a side
    // stream, overlapping the current level's scatter (SHUF_HIST_OVERLAP=1; off by
    // default: the scatter holds every register of the SM, so the two do not co-run)
    {  // SHUF_LEAF_SIGMA: 12 by default; 0 sends about half of the leaves to the second pass (tests); -1 = one pass
        const char* ls = std::getenv("SHUF_LEAF_SIGMA");
        p->leaf_sigma = ls ? std::atof(ls) : 12.0;
    }
    {
        const char* ho = std::getenv("SHUF_HIST_OVERLAP");
        p->hist_overlap = (ho && ho[0] == '1') ? 1 : 0;  // measured: no gain
        if (p->hist_overlap) {
            if ((e = cudaStreamCreateWithFlags(&p->side_stream, cudaStreamNonBlocking))) return e;
            if ((e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming))) return e;
            if ((e = cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming))) return e;
        }
    }
    // persistent grids: SM count x resident CTAs per SM
    int oh = 1, os = 1, osc = 1, of = 1, ol = 1;
    if ((e = occupancy_level(p->eb, p->k, &oh, &os, &osc))) return e;
    if ((e = occupancy_finish(p->eb, p->finish_smem, &of))) return e;
    if (p->leafk && (e = occupancy_leaf(p->eb, p->L, &ol))) return e;
    auto clamp1 = [](int v) { return v < 1 ? 1 : v; };
    p->grid_hist = p->sms * clamp1(oh);
    p->grid_scan = p->sms * clamp1(os);
    p->grid_scatter = p->sms * clamp1(osc);
    p->grid_finish = p->sms * clamp1(of);
    p->grid_small = p->sms * 4;
    p->grid_fast = p->sms;
    p->grid_leaf = p->sms * clamp1(ol);
    {  // SHUF_GRID=<ctas>: cap every persistent grid (test hook: the result must not depend on it)
        const char* ge = std::getenv("SHUF_GRID");
        const int g = ge ? std::atoi(ge) : 0;
        if (g > 0) {
            int* grids[] = {&p->grid_hist, &p->grid_scan, &p->grid_scatter, &p->grid_finish, &p->grid_small,
                            &p->grid_fast, &p->grid_leaf};
            for (int* q : grids)
                if (*q > g) *q = g;
        }
    }
    p->dev_ready = true;
    return cudaSuccess;
}

// Level l's tables (slot l & 1) and the next level's (slot ^ 1).  max_segs /
// max_chunks bound the slot a kernel WRITES: the next level's for k_plan,
// level 0's own for the init kernels (init = true).
static LevelParams level_params(const ScratchLayout& l, unsigned char* sc, unsigned char* buf0, uint32_t level,
                                bool init = false) {
    Header* hdr = reinterpret_cast<Header*>(sc + l.header);
    const int s = (int)(level & 1u), t = s ^ 1;
    LevelParams lp;
    lp.level = level;
    lp.slot = s;
    lp.segs = reinterpret_cast<SegDesc*>(sc + l.segs[s]);
    lp.chunks = reinterpret_cast<ChunkDesc*>(sc + l.chunks[s]);
    lp.counts = reinterpret_cast<uint32_t*>(sc + l.counts[s]);
    lp.prefix = reinterpret_cast<uint64_t*>(sc + l.prefix[s]);
    lp.status = reinterpret_cast<uint64_t*>(sc + l.status[s]);
    lp.ctr = &hdr->lv[s];
    lp.nsegs = reinterpret_cast<SegDesc*>(sc + l.segs[t]);
    lp.nchunks = reinterpret_cast<ChunkDesc*>(sc + l.chunks[t]);
    lp.nctr = &hdr->lv[t];
    lp.max_segs = init ? l.seg_cap[s] : l.seg_cap[t];
    lp.max_chunks = init ? l.chunk_cap[s] : l.chunk_cap[t];
    unsigned char* buf1 = sc + l.pingpong;
    lp.src = (level & 1u) ? buf1 : buf0;
    lp.dst = (level & 1u) ? buf0 : buf1;
    lp.leaf_unit = 32;
    lp.leaf_lo = lp.leaf_hi = 0;
    return lp;
}

static shuf_status check_run_args(shuf_plan_s* p, void* ptr, void* scratch, uint64_t scratch_bytes,
                                  uint64_t need = ~0ull) {
    if (!p) return SHUF_ERR_INVALID_ARG;
    if (p->n > 1 && (!ptr || !scratch)) return SHUF_ERR_INVALID_ARG;
    if (((uintptr_t)ptr & 15u) || ((uintptr_t)scratch & 15u)) return SHUF_ERR_ALIGNMENT;
    if (p->n > 1 && scratch_bytes < (need == ~0ull ? p->lay.total : need)) return SHUF_ERR_SCRATCH;
    return SHUF_OK;
}

// Layout of a segmented run: up to min(num_segments, n / (S_fuse + 1) + 1)
// level-0 segments longer than S_fuse, worst case at every level.
static uint64_t seg0_bound(const shuf_plan_s* p, uint64_t num_segments) {
    const uint64_t w = p->n / ((uint64_t)p->S_fuse + 1) + 1;
    return num_segments < w ? num_segments : w;
}

extern "C" shuf_status shuf_scratch_bytes_segmented(shuf_plan_t p, uint64_t num_segments, uint64_t* bytes) {
    if (!p || !bytes) return SHUF_ERR_INVALID_ARG;
    if (p->idx) {
        *bytes = align_up(compute_layout(p->idx, seg0_bound(p->idx, num_segments), true).total, 256) + gather_extra(p);
        return SHUF_OK;
    }
    *bytes = compute_layout(p, seg0_bound(p, num_segments), true).total;
    return SHUF_OK;
}


// Optional per-launch CUDA-event bracketing (shuf_profile_run only).
struct Prof {
    cudaStream_t st;
    std::vector<int> cls;
    std::vector<cudaEvent_t> ev;  // 2 per launch
    cudaError_t mark(int c, bool begin) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreate(&e);
        if (r) return r;
        ev.push_back(e);
        if (begin) cls.push_back(c);
        return cudaEventRecord(e, st);
    }
    ~Prof() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

#define LAUNCH(cls_, expr)                                  \
    do {                                                    \
        if (prof && (e = prof->mark(cls_, true))) return cuda_fail(p, e);  \
        if ((e = (expr))) return cuda_fail(p, e);           \
        if (prof && (e = prof->mark(cls_, false))) return cuda_fail(p, e); \
        ++launches;                                         \
    } while (0)

// A sharded rank's slice (NEXT-3): n elements at global positions [base, ..),
// segments that are children at first_level of the one problem, laid out in
// the plan's shard layout (shard_layout).
struct ShardOpts {
    uint64_t n, base;
    uint32_t first_level;
    ScratchLayout lay;
};

// Layout shared by shuf_shard_scatter (one level-0 slice of <= n elements) and
// shuf_shard_continue (<= k segments of <= n elements in total).
static ScratchLayout shard_layout(const shuf_plan_s* p) {
    shuf_plan_s q = *p;
    if (q.levels < 1) q.levels = 1;
    return compute_layout(&q, seg0_bound(&q, p->k), true);
}

extern "C" shuf_status shuf_scratch_bytes_shard(shuf_plan_t p, uint64_t* bytes) {
    if (!p || !bytes) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;
    *bytes = shard_layout(p).total;
    return SHUF_OK;
}

static RunParams base_params(const shuf_plan_s* p, const ScratchLayout& lay, unsigned char* sc, unsigned char* buf0,
                             uint32_t max_levels, int run_leaves) {
    RunParams rp{};
    rp.buf0 = buf0;
    rp.buf1 = sc + lay.pingpong;
    rp.hdr = reinterpret_cast<Header*>(sc + lay.header);
    rp.n = p->n;
    rp.eb = p->eb;
    rp.k = p->k;
    rp.L = p->L;
    rp.S_fuse = p->S_fuse;
    rp.S_stream = p->S_stream;
    rp.chunk = p->chunk;
    rp.max_levels = max_levels;
    rp.planned_levels = p->levels;
    rp.run_leaves = run_leaves;
    rp.bp = make_bucket_params(p->k);
    rp.seed = p->seed;
    rp.rank_ordered = (uint32_t)p->rank_ordered;
    rp.fin_nbuf = p->fin_nbuf;
    rp.fast = (uint32_t)p->fast;
    rp.leafk = (uint32_t)p->leafk;
    rp.defer = (uint32_t)p->defer;
    rp.items = sc + lay.items;
    rp.fused = reinterpret_cast<uint32_t*>(sc + lay.fused);
    rp.max_fused = p->leafk ? lay.max_fused : 0;  // the list holds children > L only
    {
        const char* dbg = std::getenv("SHUF_DBG");
        rp.dbg = dbg ? (uint32_t)std::atoi(dbg) : 0u;
    }
    rp.flags = sc + lay.flags;
    return rp;
}

// Enqueue the whole shuffle.  segmented: d_offsets != nullptr; a sharded
// rank's continuation: so != nullptr (with d_offsets).
static shuf_status enqueue(shuf_plan_s* p, void* ptr, const uint64_t* d_offsets, uint64_t nsegs, void* scratch,
                           cudaStream_t st, uint32_t max_levels, int run_leaves, Prof* prof = nullptr,
                           const ShardOpts* so = nullptr) {
    p->last_launches = 0;
    cudaError_t e = device_setup(p);
    if (e) return cuda_fail(p, e);
    unsigned char* sc = static_cast<unsigned char*>(scratch);
    unsigned char* buf0 = static_cast<unsigned char*>(ptr);
    const ScratchLayout lay = so ? so->lay : d_offsets ? compute_layout(p, seg0_bound(p, nsegs), true) : p->lay;
    Header* hdr = reinterpret_cast<Header*>(sc + lay.header);
    p->last_hdr = hdr;
    RunParams rp = base_params(p, lay, sc, buf0, max_levels, run_leaves);
    const uint32_t lv0 = so ? so->first_level : 0u;
    if (so) {
        rp.n = so->n;
        rp.shard = 1;
        rp.first_level = lv0;
        rp.seg_base = so->base;
        rp.planned_levels = p->levels + lv0;
    }
    uint64_t launches = 0;
    if ((e = cudaMemsetAsync(hdr, 0, sizeof(Header), st))) return cuda_fail(p, e);
    const LevelParams lp0 = level_params(lay, sc, buf0, 0, true);
    if (d_offsets) {
        LAUNCH(SHUF_K_INIT, launch_init_segmented(rp, lp0, d_offsets, nsegs, st, p->grid_small));
        LAUNCH(SHUF_K_FINISH, launch_finish_segments(rp, d_offsets, nsegs, st, p->grid_finish));
        if (p->leafk) {
            // Long segments (one per warp): length classes (0, L/2], (L/2, 3L/4], (3L/4, L], each pass
            // with slots for its class -- the shorter classes put more warps on an SM -- and warp-units
            // handed out by a ticket counter (a fixed stride plus the class filter left warps unevenly
            // loaded, r06i).  The host does not know the lengths; a pass that finds no segment of its
            // class only reads offsets.  SHUF_LEAF_SIGMA=-1: one pass, fixed stride.
            uint32_t cuts[3] = {0, 0, p->L};
            int nc = 1;
            const uint64_t avg = nsegs ? rp.n / nsegs : 0;
            const bool classes = !so && p->leaf_sigma >= 0.0 && nsegs >= 1024 &&
                                 leaf_unit(p->eb, p->L, avg > p->L ? p->L : avg) == 1;
            if (classes) {
                uint32_t prev = p->L;
                for (uint32_t c : {(3 * p->L / 4 + 63) & ~63u, (p->L / 2 + 63) & ~63u}) {
                    if (c >= 512 && c < prev && leaf_warps_per_sm(p->eb, c) > leaf_warps_per_sm(p->eb, prev)) {
                        cuts[2 - nc] = c;
                        ++nc;
                        prev = c;
                    }
                }
            }
            uint32_t lo = 0;
            for (int i = 3 - nc; i < 3; ++i) {
                const uint32_t hi = cuts[i];
                const int g = hi == p->L ? p->grid_leaf
                                         : p->sms * (int)(leaf_warps_per_sm(p->eb, hi) / leaf_warps_per_cta(p->eb, hi));
                LAUNCH(SHUF_K_LEAF, launch_leaf_segments(rp, d_offsets, nsegs, st, g, lo, hi,
                                                         classes ? &hdr->leaf_ticket[i] : nullptr));
                lo = hi;
            }
        }
    } else {
        LAUNCH(SHUF_K_INIT, launch_init(rp, lp0, st, p->grid_small));
        if (p->n <= p->S_fuse) {
            if (p->leafk && p->n <= p->L) LAUNCH(SHUF_K_LEAF, launch_leaf_segments(rp, hdr->root_off, 1, st, 1));
            else LAUNCH(SHUF_K_FINISH, launch_finish_segments(rp, hdr->root_off, 1, st, 1));
        }
    }
    const uint32_t lim = max_levels > lv0 ? max_levels - lv0 : 0u;
    const uint32_t G = p->levels < lim ? p->levels : lim;
    // level l+1's histogram needs only k_plan(l)'s list, so it is forked onto
    // the side stream before level l's scatter and joined before scan(l+1)
    // (fork/join inside the call: still stream-ordered for the caller)
    const bool overlap = p->hist_overlap && !prof;
    for (uint32_t lv = 0; lv < G; ++lv) {
        LevelParams lp = level_params(lay, sc, buf0, lv);
        lp.level = lv + lv0;  // draws are keyed by the problem's level; buffers and slots by lv
        {  // expected child length of the level: (n / segments) / k^(lv+1)
            double avg = (double)rp.n / (double)(d_offsets ? (nsegs ? nsegs : 1) : 1);
            for (uint32_t i = 0; i <= lv; ++i) avg /= (double)p->k;
            lp.leaf_unit = leaf_unit(p->eb, p->L, (uint64_t)avg);
            // Single shuffle, long leaves (one per warp) expected well below L: a
            // first leaf pass whose slots hold avg + leaf_sigma * sqrt(avg) elements
            // (child lengths are binomial: sigma < sqrt(avg)) when that puts more
            // warps on an SM, then the full-slot pass for longer leaves (normally none).
            if (!d_offsets && p->leaf_sigma >= 0.0 && avg <= (double)p->L && lp.leaf_unit == 1) {
                uint64_t cand = (uint64_t)(avg + p->leaf_sigma * std::sqrt(avg)) + 1;
                cand = (cand + 63) & ~63ull;
                if (cand < p->L && leaf_unit(p->eb, (uint32_t)cand, (uint64_t)avg) == 1 &&
                    leaf_warps_per_sm(p->eb, (uint32_t)cand) > leaf_warps_per_sm(p->eb, p->L))
                    lp.leaf_hi = (uint32_t)cand;
            }
        }
        if (overlap && lv > 0) {
            if ((e = cudaStreamWaitEvent(st, p->ev_join, 0))) return cuda_fail(p, e);
        } else {
            LAUNCH(SHUF_K_HIST, launch_hist(rp, lp, st, p->grid_hist));
        }
        LAUNCH(SHUF_K_SCAN, launch_scan(rp, lp, st, p->grid_scan));
        LAUNCH(SHUF_K_PLAN, launch_plan(rp, lp, st, p->grid_small));
        if (overlap && lv + 1 < G) {
            if ((e = cudaEventRecord(p->ev_fork, st))) return cuda_fail(p, e);
            if ((e = cudaStreamWaitEvent(p->side_stream, p->ev_fork, 0))) return cuda_fail(p, e);
            LevelParams ln = level_params(lay, sc, buf0, lv + 1);
            ln.level = lv + 1 + lv0;
            LAUNCH(SHUF_K_HIST, launch_hist(rp, ln, p->side_stream, p->grid_hist));
            if ((e = cudaEventRecord(p->ev_join, p->side_stream))) return cuda_fail(p, e);
        }
        LAUNCH(SHUF_K_SCATTER, launch_scatter(rp, lp, st, p->grid_scatter));
        if (p->fast) LAUNCH(SHUF_K_FINISH, launch_finish_fast(rp, lp, st, p->grid_fast));
        LAUNCH(SHUF_K_FINISH, launch_finish_children(rp, lp, st, p->grid_finish));
        if (p->S_stream) LAUNCH(SHUF_K_FINISH, launch_finish_stream(rp, lp, st, p->sms));
        if (p->leafk) {
            if (lp.leaf_hi) {
                const uint32_t wps = leaf_warps_per_sm(p->eb, lp.leaf_hi), wpc = leaf_warps_per_cta(p->eb, lp.leaf_hi);
                LAUNCH(SHUF_K_LEAF, launch_leaf_children(rp, lp, st, p->sms * (int)(wps / wpc)));
                LevelParams rest = lp;
                rest.leaf_lo = lp.leaf_hi;
                rest.leaf_hi = 0;
                rest.leaf_unit = 32;  // normally no leaf at all: look at 32 children per warp-unit
                LAUNCH(SHUF_K_LEAF, launch_leaf_children(rp, rest, st, p->grid_leaf));
            } else {
                LAUNCH(SHUF_K_LEAF, launch_leaf_children(rp, lp, st, p->grid_leaf));
            }
        }
        if (lv + lv0 + 1 == max_levels) LAUNCH(SHUF_K_FINISH, launch_copy_big(rp, lp, st, p->grid_small));
    }
    // leaves of the recorded fused items (all levels; they sit in ptr)
    if (p->defer && (d_offsets || p->n > p->L)) LAUNCH(SHUF_K_LEAF, launch_leaf_items(rp, st, p->grid_leaf));
    p->last_launches = launches;
    return SHUF_OK;
}

// The gather route: iota -> the index plan's shuffle (single, segmented or
// level-limited) -> out[i] = in[idx[i]] into the staging buffer -> copy back.
static shuf_status gather_route(shuf_plan_s* p, void* ptr, const uint64_t* d_offsets, uint64_t nsegs, void* scratch,
                                uint64_t scratch_bytes, cudaStream_t st, uint32_t max_levels, int run_leaves,
                                Prof* prof) {
    shuf_plan_s* ix = p->idx;
    const uint64_t sub = align_up(d_offsets ? compute_layout(ix, seg0_bound(ix, nsegs), true).total : ix->lay.total, 256);
    if (scratch_bytes < sub + gather_extra(p)) return SHUF_ERR_SCRATCH;
    unsigned char* sc = static_cast<unsigned char*>(scratch);
    unsigned char* idxa = sc + sub;
    unsigned char* stage = idxa + align_up(p->n * ix->eb, 256);
    cudaError_t e = device_setup(ix);
    if (e) return cuda_fail(p, e);
    const int grid = ix->sms * 8;
    if ((e = launch_iota(idxa, ix->eb, p->n, st, grid))) return cuda_fail(p, e);
    shuf_status r = enqueue(ix, idxa, d_offsets, nsegs, sc, st, max_levels, run_leaves, prof);
    if (r) {
        p->last_cuda_error = ix->last_cuda_error;
        return r;
    }
    if ((e = launch_gather(ptr, stage, idxa, ix->eb, p->n, p->eb, st, grid))) return cuda_fail(p, e);
    if ((e = cudaMemcpyAsync(ptr, stage, p->n * p->eb, cudaMemcpyDeviceToDevice, st))) return cuda_fail(p, e);
    p->last_hdr = ix->last_hdr;
    p->last_launches = ix->last_launches + 2;
    return SHUF_OK;
}

extern "C" shuf_status shuf_run(shuf_plan_t p, void* ptr, void* scratch, uint64_t scratch_bytes, void* stream) {
    shuf_status s = check_run_args(p, ptr, scratch, scratch_bytes, p && p->idx ? 0 : ~0ull);
    if (s) return s;
    if (p->n <= 1) {
        p->last_launches = 0;
        return SHUF_OK;
    }
    if (p->idx)
        return gather_route(p, ptr, nullptr, 0, scratch, scratch_bytes, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu,
                            1, nullptr);
    return enqueue(p, ptr, nullptr, 0, scratch, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu, 1);
}

// ---------------------------------------------------------------- IpSc ---
// NEXT-2 (kernels_ipsc.cu): the paper's In-Place ScatterShuffle, level by
// level; the host plans batches of segments whose ParRoughScatter trees fit
// the node table, and reads each level's segment list back (one sync/level).
struct IpscLayout {
    uint64_t header, root, segs[2], cnt, bsegs, work, stab, S, total;
    uint64_t max_segs, max_bseg, E;
};

static uint32_t ipsc_depth_host(uint64_t m, uint32_t k) {
    const uint64_t n0 = (uint64_t)k * k;
    uint32_t t = 0;
    while (t < 11u && (m >> (t + 1)) >= n0) ++t;
    return t;
}

static IpscLayout ipsc_layout(const shuf_plan_s* p) {
    IpscLayout l{};
    const uint64_t n = p->n, k = p->k;
    l.max_segs = n / ((uint64_t)p->L + 1) + 1;
    const uint64_t root_entries = ((2ull << ipsc_depth_host(n, p->k)) - 1) * k;
    uint64_t E = l.max_segs * k;
    if (E > (1ull << 21)) E = 1ull << 21;
    if (E < root_entries) E = root_entries;
    l.E = E;
    l.max_bseg = E / k;
    uint64_t off = 0;
    auto take = [&off](uint64_t bytes) {
        const uint64_t at = off;
        off = align_up(off + bytes, 256);
        return at;
    };
    l.header = take(sizeof(Header));
    l.root = take(16);
    l.segs[0] = take(l.max_segs * 16);
    l.segs[1] = take(l.max_segs * 16);
    l.cnt = take(8);
    l.bsegs = take(l.max_bseg * sizeof(IpscSeg));
    l.work = take(l.max_bseg * 8);
    l.stab = take(E * 8);
    l.S = take(l.max_bseg * (k + 1) * 8);
    l.total = off;
    return l;
}

extern "C" shuf_status shuf_aux_bytes_ipsc(shuf_plan_t p, uint64_t* bytes) {
    if (!p || !bytes) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;
    *bytes = ipsc_layout(p).total;
    return SHUF_OK;
}

static shuf_status enqueue_ipsc(shuf_plan_s* p, void* ptr, void* aux, cudaStream_t st, uint32_t max_levels,
                                int run_leaves) {
    p->last_launches = 0;
    cudaError_t e = device_setup(p);
    if (e) return cuda_fail(p, e);
    if (leaf_smem_bytes(p->eb, p->L) > kSmemLimit) return SHUF_ERR_UNSUPPORTED;
    if (!p->leafk) {
        if ((e = configure_leaf(p->eb, p->L))) return cuda_fail(p, e);
        int ol = 1;
        if ((e = occupancy_leaf(p->eb, p->L, &ol))) return cuda_fail(p, e);
        p->grid_leaf = p->sms * (ol < 1 ? 1 : ol);
    }
    const IpscLayout l = ipsc_layout(p);
    unsigned char* ax = static_cast<unsigned char*>(aux);
    Header* hdr = reinterpret_cast<Header*>(ax + l.header);
    p->last_hdr = hdr;
    RunParams rp{};
    rp.buf0 = static_cast<unsigned char*>(ptr);
    rp.hdr = hdr;
    rp.n = p->n;
    rp.eb = p->eb;
    rp.k = p->k;
    rp.L = p->L;
    rp.S_fuse = p->S_fuse;
    rp.chunk = p->chunk;
    rp.max_levels = max_levels;
    rp.planned_levels = kMaxLevels;
    rp.run_leaves = run_leaves;
    rp.bp = make_bucket_params(p->k);
    rp.seed = p->seed;
    uint64_t launches = 0;
    Prof* prof = nullptr;
    if ((e = cudaMemsetAsync(hdr, 0, sizeof(Header), st))) return cuda_fail(p, e);
    const uint64_t n = p->n, k = p->k;
    if (n <= p->L) {  // the whole array is one leaf (Fig. 2)
        if (run_leaves && n >= 2) {
            const uint64_t root[2] = {0, n};
            uint64_t* d_root = reinterpret_cast<uint64_t*>(ax + l.root);
            if ((e = cudaMemcpyAsync(d_root, root, sizeof root, cudaMemcpyHostToDevice, st))) return cuda_fail(p, e);
            LAUNCH(SHUF_K_LEAF, launch_leaf_segments(rp, d_root, 1, st, 1));
        }
        p->last_launches = launches;
        return SHUF_OK;
    }
    IpscParams P{};
    P.X = static_cast<unsigned char*>(ptr);
    P.k = p->k;
    P.L = p->L;
    P.seed = p->seed;
    P.segs = reinterpret_cast<const IpscSeg*>(ax + l.bsegs);
    P.s_tab = reinterpret_cast<uint64_t*>(ax + l.stab);
    P.S = reinterpret_cast<uint64_t*>(ax + l.S);
    P.next_cnt = reinterpret_cast<uint32_t*>(ax + l.cnt);
    P.max_next = l.max_segs;
    P.hdr = hdr;
    P.run_leaves = (uint32_t)run_leaves;
    if (const char* dbg = std::getenv("SHUF_DBG"))
        if (std::atoi(dbg) & 128) P.clk = hdr->clk;
    // RoughScatter: 8 persistent CTAs per SM (HOT: 1/2/3/4/6/8 per SM -> 248/213/206/203/199/196 ms, r03n/r03o)
    int rs_per_sm = 8;  // SHUF_IPSC_RSGRID=<CTAs per SM> (experiments)
    if (const char* g = std::getenv("SHUF_IPSC_RSGRID")) rs_per_sm = std::atoi(g);
    uint32_t tsmall = 0;  // (the capacity's tree depth; launches size their own)
    const uint32_t cap = std::getenv("SHUF_IPSC_NOSMALL") ? 0u : ipsc_small_cap(p->k, p->eb, &tsmall);
    IpscSeg* d_bsegs = reinterpret_cast<IpscSeg*>(ax + l.bsegs);
    uint2* d_work = reinterpret_cast<uint2*>(ax + l.work);
    std::vector<uint64_t> cur = {0, n}, nxt;
    std::vector<IpscSeg> bs;
    std::vector<uint2> work;
    std::vector<uint32_t> wofs;
    {
        uint64_t* l0 = reinterpret_cast<uint64_t*>(ax + l.segs[0]);
        if ((e = cudaMemcpyAsync(l0, cur.data(), 16, cudaMemcpyHostToDevice, st))) return cuda_fail(p, e);
    }
    for (uint32_t lv = 0; !cur.empty() && lv < max_levels; ++lv) {
        if (lv > 255) return SHUF_ERR_DEPTH;
        const int slot = (lv + 1) & 1;
        P.level = lv;
        P.next = reinterpret_cast<uint64_t*>(ax + l.segs[slot]);
        if ((e = cudaMemsetAsync(P.next_cnt, 0, 4, st))) return cuda_fail(p, e);
        const size_t nseg = cur.size() / 2;
        // segments of at most `cap` elements: one fused shared-memory launch over the level's list
        // (shared memory sized for the longest of them: more CTAs per SM when they are short)
        size_t nsmall = 0;
        uint64_t mmax = 0;
        for (size_t q = 0; q < nseg; ++q)
            if (cur[2 * q + 1] <= cap) {
                ++nsmall;
                if (cur[2 * q + 1] > mmax) mmax = cur[2 * q + 1];
            }
        if (nsmall) {
            uint32_t tl = 0;
            while (tl < 11u && (mmax >> (tl + 1)) >= k * k) ++tl;
            LAUNCH(SHUF_K_FINISH, launch_ipsc_small(P, p->eb, reinterpret_cast<const uint64_t*>(ax + l.segs[lv & 1]),
                                                    (uint32_t)nseg, (uint32_t)((mmax + 15) & ~15ull), tl, st,
                                                    4 * p->sms));
        }
        for (size_t s0 = 0; s0 < nseg;) {
            // batch: segments while their node tables fit E entries
            bs.clear();
            uint64_t entries = 0;
            uint32_t tmax = 0;
            size_t s1 = s0;
            for (; s1 < nseg; ++s1) {
                IpscSeg g{};
                g.a = cur[2 * s1];
                g.m = cur[2 * s1 + 1];
                if (g.m <= cap) continue;  // the shared-memory kernel's
                g.t = ipsc_depth_host(g.m, p->k);
                const uint64_t nodes = (2ull << g.t) - 1;
                if (!bs.empty() && (entries + nodes * k > l.E || bs.size() >= l.max_bseg)) break;
                g.node_base = entries / k;
                entries += nodes * k;
                if (g.t > tmax) tmax = g.t;
                bs.push_back(g);
            }
            // work lists: leaf subtasks, then the inner nodes depth by depth (deepest first)
            work.clear();
            wofs.clear();
            for (int d = (int)tmax; d >= 0; --d) {
                wofs.push_back((uint32_t)work.size());
                for (uint32_t si = 0; si < bs.size(); ++si) {
                    const uint32_t t = bs[si].t;
                    if (d == (int)tmax) {  // first launch: every segment's leaves
                        for (uint32_t v = 1u << t; v < (2u << t); ++v) work.push_back(make_uint2(si, v));
                    } else if ((uint32_t)d < t) {
                        for (uint32_t v = 1u << d; v < (2u << d); ++v) work.push_back(make_uint2(si, v));
                    }
                }
            }
            wofs.push_back((uint32_t)work.size());
            s0 = s1;
            if (bs.empty()) continue;
            if (work.size() > l.max_bseg) return SHUF_ERR_SCRATCH;  // (nodes <= E / k = max_bseg)
            if ((e = cudaMemcpyAsync(d_bsegs, bs.data(), bs.size() * sizeof(IpscSeg), cudaMemcpyHostToDevice, st)))
                return cuda_fail(p, e);
            if ((e = cudaMemcpyAsync(d_work, work.data(), work.size() * sizeof(uint2), cudaMemcpyHostToDevice, st)))
                return cuda_fail(p, e);
            for (size_t q = 0; q + 1 < wofs.size(); ++q) {
                const uint32_t nw = wofs[q + 1] - wofs[q];
                P.work = d_work + wofs[q];
                const bool wide = nw < (uint32_t)p->sms;
                LAUNCH(SHUF_K_SCATTER, launch_ipsc_rs(P, p->eb, nw, q > 0, wide, (uint32_t)rs_per_sm * (uint32_t)p->sms, st));
            }
            LAUNCH(SHUF_K_FINISH, launch_ipsc_fine(P, p->eb, (uint32_t)bs.size(), st));
            LAUNCH(SHUF_K_PLAN, launch_ipsc_children(P, (uint32_t)bs.size(), st, p->grid_small));
            if (run_leaves) LAUNCH(SHUF_K_LEAF, launch_leaf_ipsc(rp, P.S, (uint32_t)bs.size(), st, p->grid_leaf));
        }
        uint32_t cnt = 0, err = 0;
        if ((e = cudaMemcpyAsync(&cnt, P.next_cnt, 4, cudaMemcpyDeviceToHost, st))) return cuda_fail(p, e);
        if ((e = cudaMemcpyAsync(&err, &hdr->error, 4, cudaMemcpyDeviceToHost, st))) return cuda_fail(p, e);
        if ((e = cudaStreamSynchronize(st))) return cuda_fail(p, e);
        if (err) break;  // reported by shuf_last_device_error
        nxt.resize(2 * (size_t)cnt);
        if (cnt && (e = cudaMemcpy(nxt.data(), P.next, nxt.size() * 8, cudaMemcpyDeviceToHost))) return cuda_fail(p, e);
        cur.swap(nxt);
    }
    p->last_launches = launches;
    return SHUF_OK;
}

static shuf_status check_ipsc_args(shuf_plan_s* p, void* ptr, void* aux, uint64_t aux_bytes) {
    if (!p) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;
    if (p->n > 1 && (!ptr || !aux)) return SHUF_ERR_INVALID_ARG;
    if (((uintptr_t)ptr & 15u) || ((uintptr_t)aux & 15u)) return SHUF_ERR_ALIGNMENT;
    if (p->n > 1 && aux_bytes < ipsc_layout(p).total) return SHUF_ERR_SCRATCH;
    return SHUF_OK;
}

extern "C" shuf_status shuf_run_ipsc(shuf_plan_t p, void* ptr, void* aux, uint64_t aux_bytes, void* stream) {
    shuf_status s = check_ipsc_args(p, ptr, aux, aux_bytes);
    if (s) return s;
    if (p->n <= 1) return SHUF_OK;
    return enqueue_ipsc(p, ptr, aux, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu, 1);
}

extern "C" shuf_status shuf_debug_ipsc_levels(shuf_plan_t p, void* ptr, void* aux, uint64_t aux_bytes, void* stream,
                                              uint32_t max_levels, int run_leaves) {
    shuf_status s = check_ipsc_args(p, ptr, aux, aux_bytes);
    if (s) return s;
    if (p->n <= 1) return SHUF_OK;
    return enqueue_ipsc(p, ptr, aux, static_cast<cudaStream_t>(stream), max_levels, run_leaves ? 1 : 0);
}

// ------------------------------------------------------------ in-place ---
extern "C" shuf_status shuf_aux_bytes_inplace(shuf_plan_t p, uint64_t* bytes) {
    if (!p || !bytes) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;  // the in-place mode moves 4/8/16-byte elements only
    *bytes = p->ipl.total;
    return SHUF_OK;
}

// The in-place mode: its level loop runs on the device -- one launch of a
// cached CUDA graph whose two nested WHILE nodes (levels, batches) are driven
// by k_ip_level_plan / k_ip_batch_next / k_ip_level_next; no host
// synchronisation and no host round trip per level.
static shuf_status enqueue_inplace(shuf_plan_s* p, void* ptr, void* aux, cudaStream_t st, uint32_t max_levels,
                                   int run_leaves) {
    p->last_launches = 0;
    cudaError_t e = device_setup(p);
    if (e) return cuda_fail(p, e);
    if (!p->ip_ready) {
        if ((e = configure_inplace(p->eb, p->k))) return cuda_fail(p, e);
        if (!p->leafk && (e = configure_leaf(p->eb, p->L))) return cuda_fail(p, e);
        int oc = 1, op = 1;
        if ((e = occupancy_inplace(p->eb, p->k, &oc, &op))) return cuda_fail(p, e);
        p->grid_ipc = p->sms * (oc < 1 ? 1 : oc);
        p->grid_ipp = p->sms * (op < 1 ? 1 : op);
        if (p->grid_leaf == 0) {
            int ol = 1;
            if ((e = occupancy_leaf(p->eb, p->L, &ol))) return cuda_fail(p, e);
            p->grid_leaf = p->sms * (ol < 1 ? 1 : ol);
        }
        p->ip_ready = true;
    }
    const IpAuxLayout& l = p->ipl;
    unsigned char* ax = static_cast<unsigned char*>(aux);
    Header* hdr = reinterpret_cast<Header*>(ax + l.header);
    IpCounters* ctr = reinterpret_cast<IpCounters*>(ax + l.ctr);
    p->last_hdr = hdr;
    RunParams rp{};
    rp.buf0 = static_cast<unsigned char*>(ptr);
    rp.buf1 = nullptr;
    rp.hdr = hdr;
    rp.n = p->n;
    rp.eb = p->eb;
    rp.k = p->k;
    rp.L = p->L;
    rp.S_fuse = p->S_fuse;
    rp.S_stream = p->S_stream;
    rp.chunk = p->chunk;
    rp.max_levels = max_levels;
    rp.planned_levels = p->levels;
    rp.run_leaves = run_leaves;
    rp.bp = make_bucket_params(p->k);
    rp.seed = p->seed;
    rp.rank_ordered = (uint32_t)p->rank_ordered;
    rp.fin_nbuf = p->fin_nbuf;
    rp.fast = (uint32_t)p->fast;
    rp.leafk = 1;
    rp.defer = 0;
    rp.items = nullptr;
    rp.flags = ax + l.flags;
    rp.fused = nullptr;
    rp.max_fused = 0;
    rp.dbg = 0;
    uint64_t launches = 0;
    Prof* prof = nullptr;
    if (p->n <= p->S_fuse || max_levels == 0) {
        if ((e = cudaMemsetAsync(ax, 0, l.segs[0], st))) return cuda_fail(p, e);  // header, counters, state
        LAUNCH(SHUF_K_INIT, launch_ip_root(hdr, p->n, st));
        if (p->n <= p->S_fuse) {
            if (p->n <= p->L) LAUNCH(SHUF_K_LEAF, launch_leaf_segments(rp, hdr->root_off, 1, st, 1));
            else LAUNCH(SHUF_K_FINISH, launch_finish_segments(rp, hdr->root_off, 1, st, 1));
        }
        p->last_launches = launches;
        return SHUF_OK;
    }
    if (!p->ip_exec || p->ip_ptr != ptr || p->ip_aux != aux || p->ip_maxlv != max_levels || p->ip_leaves != run_leaves) {
        if (p->ip_exec) {
            cudaGraphExecDestroy(p->ip_exec);
            p->ip_exec = nullptr;
        }
        IpParams ip{};
        ip.Z = l.Z;
        ip.zseg = reinterpret_cast<uint32_t*>(ax + l.zseg);
        ip.N = reinterpret_cast<uint64_t*>(ax + l.N);
        ip.F = reinterpret_cast<uint32_t*>(ax + l.F);
        ip.S = reinterpret_cast<uint64_t*>(ax + l.S);
        ip.wr = reinterpret_cast<uint64_t*>(ax + l.wr);
        ip.regpre = reinterpret_cast<uint32_t*>(ax + l.regpre);
        ip.segtot = reinterpret_cast<uint64_t*>(ax + l.segtot);
        ip.ovf = reinterpret_cast<uint32_t*>(ax + l.ovf);
        ip.ovfd = ax + l.ovfd;
        ip.pcnt = reinterpret_cast<uint32_t*>(ax + l.pcnt);
        ip.part = ax + l.part;
        ip.tags = reinterpret_cast<uint16_t*>(ax + l.tags);
        ip.max_next = l.max_segs;
        ip.cursor = &ctr->cursor;
        ip.state = reinterpret_cast<IpState*>(ax + l.state);
        ip.segbase[0] = reinterpret_cast<IpSeg*>(ax + l.segs[0]);
        ip.segbase[1] = reinterpret_cast<IpSeg*>(ax + l.segs[1]);
        ip.nnext_base = ctr->nnext;
        if (!p->ip_cap_stream && (e = cudaStreamCreateWithFlags(&p->ip_cap_stream, cudaStreamNonBlocking)))
            return cuda_fail(p, e);
        cudaStream_t cs = p->ip_cap_stream;
        IpState st0{};
        st0.C = l.C;
        st0.max_batches = (uint32_t)l.max_batches;
        st0.batches = reinterpret_cast<IpBatch*>(ax + l.batches);
        // Graph: memsets, init; WHILE(levels) { level_plan; WHILE(batches) { batch kernels; batch_next };
        // level_next }.  Built by stream capture; the WHILE nodes are added mid-capture.
        cudaGraph_t g = nullptr, bl = nullptr, bb = nullptr;
        cudaGraphConditionalHandle hl = 0, hb = 0;
        auto fail = [&](cudaError_t err) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(cs, &junk);
            if (junk) cudaGraphDestroy(junk);
            if (g) cudaGraphDestroy(g);
            return cuda_fail(p, err);
        };
        auto add_while = [&](cudaGraphConditionalHandle h, cudaGraph_t* body) -> cudaError_t {
            cudaStreamCaptureStatus cst;
            cudaGraph_t cg = nullptr;
            const cudaGraphNode_t* deps = nullptr;
            size_t nd = 0;
            cudaError_t err = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &cg, &deps, &nd);
            if (err) return err;
            cudaGraphNodeParams cp{};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            if ((err = cudaGraphAddNode(&node, cg, deps, nd, &cp))) return err;
            *body = cp.conditional.phGraph_out[0];
            return cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies);
        };
        uint64_t nodes = 0;
        if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed))) return cuda_fail(p, e);
        if ((e = cudaMemsetAsync(ax, 0, l.segs[0], cs))) return fail(e);  // header, counters, state, batches
        if ((e = cudaMemsetAsync(ax + l.N, 0, l.S - l.N, cs))) return fail(e);          // N, F
        if ((e = cudaMemsetAsync(ax + l.ovf, 0, l.ovfd - l.ovf, cs))) return fail(e);
        if ((e = launch_ip_init(ip, hdr, p->n, st0, cs))) return fail(e);  // (kernel argument: no host memory in the graph)
        {
            cudaStreamCaptureStatus cst;
            if ((e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &g))) return fail(e);
            if ((e = cudaGraphConditionalHandleCreate(&hl, g, 1, cudaGraphCondAssignDefault))) return fail(e);
        }
        if ((e = add_while(hl, &bl))) return fail(e);
        if ((e = cudaStreamEndCapture(cs, &g))) return fail(e);
        // level body
        if ((e = cudaGraphConditionalHandleCreate(&hb, bl, 0, cudaGraphCondAssignDefault))) return fail(e);
        if ((e = cudaStreamBeginCaptureToGraph(cs, bl, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
            return fail(e);
        if ((e = launch_ip_level_plan(rp, ip, hb, cs))) return fail(e);
        if ((e = add_while(hb, &bb))) return fail(e);
        if ((e = launch_ip_level_next(rp, ip, hl, cs))) return fail(e);
        {
            cudaGraph_t out = nullptr;
            if ((e = cudaStreamEndCapture(cs, &out))) return fail(e);
        }
        // batch body
        if ((e = cudaStreamBeginCaptureToGraph(cs, bb, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
            return fail(e);
        if ((e = launch_ip_stripes(ip, cs))) return fail(e);
        if ((e = launch_ip_classify(rp, ip, cs, p->grid_ipc))) return fail(e);
        if ((e = launch_ip_plan(rp, ip, cs))) return fail(e);
        if ((e = launch_ip_permute(rp, ip, cs, p->grid_ipp))) return fail(e);
        if ((e = launch_ip_fill(rp, ip, cs, p->grid_ipp))) return fail(e);
        nodes = 6;
        if (p->fast) {
            if ((e = launch_finish_fast_ip(rp, ip, cs, p->grid_fast))) return fail(e);
            ++nodes;
        }
        if ((e = launch_finish_ipchildren(rp, ip, cs, p->grid_finish))) return fail(e);
        if ((e = launch_leaf_ipchildren(rp, ip, cs, p->grid_leaf))) return fail(e);
        if ((e = launch_ip_batch_next(ip, hb, cs))) return fail(e);
        {
            cudaGraph_t out = nullptr;
            if ((e = cudaStreamEndCapture(cs, &out))) return fail(e);
        }
        e = cudaGraphInstantiate(&p->ip_exec, g, 0);
        cudaGraphDestroy(g);
        if (e) {
            p->ip_exec = nullptr;
            return cuda_fail(p, e);
        }
        p->ip_ptr = ptr;
        p->ip_aux = aux;
        p->ip_maxlv = max_levels;
        p->ip_leaves = run_leaves;
        p->ip_nodes = nodes + 2;  // + init, plan, next per level / batch (counted by the caller as launches)
    }
    if ((e = cudaGraphLaunch(p->ip_exec, st))) return cuda_fail(p, e);
    p->last_launches = p->ip_nodes;
    return SHUF_OK;
}

static shuf_status check_inplace_args(shuf_plan_s* p, void* ptr, void* aux, uint64_t aux_bytes) {
    if (!p) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;
    if (p->n > 1 && (!ptr || !aux)) return SHUF_ERR_INVALID_ARG;
    if (((uintptr_t)ptr & 15u) || ((uintptr_t)aux & 15u)) return SHUF_ERR_ALIGNMENT;
    if (p->n > 1 && aux_bytes < p->ipl.total) return SHUF_ERR_SCRATCH;
    return SHUF_OK;
}

extern "C" shuf_status shuf_run_inplace(shuf_plan_t p, void* ptr, void* aux, uint64_t aux_bytes, void* stream) {
    shuf_status s = check_inplace_args(p, ptr, aux, aux_bytes);
    if (s) return s;
    if (p->n <= 1) return SHUF_OK;
    return enqueue_inplace(p, ptr, aux, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu, 1);
}

extern "C" shuf_status shuf_debug_inplace_levels(shuf_plan_t p, void* ptr, void* aux, uint64_t aux_bytes,
                                                 void* stream, uint32_t max_levels, int run_leaves) {
    shuf_status s = check_inplace_args(p, ptr, aux, aux_bytes);
    if (s) return s;
    if (p->n <= 1) return SHUF_OK;
    return enqueue_inplace(p, ptr, aux, static_cast<cudaStream_t>(stream), max_levels, run_leaves ? 1 : 0);
}

extern "C" shuf_status shuf_debug_run_levels(shuf_plan_t p, void* ptr, void* scratch, uint64_t scratch_bytes,
                                             void* stream, uint32_t max_levels, int run_leaves) {
    shuf_status s = check_run_args(p, ptr, scratch, scratch_bytes, p && p->idx ? 0 : ~0ull);
    if (s) return s;
    if (p->n <= 1) return SHUF_OK;
    if (p->idx)
        return gather_route(p, ptr, nullptr, 0, scratch, scratch_bytes, static_cast<cudaStream_t>(stream), max_levels,
                            run_leaves ? 1 : 0, nullptr);
    return enqueue(p, ptr, nullptr, 0, scratch, static_cast<cudaStream_t>(stream), max_levels, run_leaves ? 1 : 0);
}

extern "C" shuf_status shuf_segmented(shuf_plan_t p, void* ptr, const uint64_t* d_offsets, uint64_t num_segments,
                                      void* scratch, uint64_t scratch_bytes, void* stream) {
    shuf_status s = check_run_args(p, ptr, scratch, scratch_bytes,
                                   p && !p->idx ? compute_layout(p, seg0_bound(p, num_segments), true).total : 0);
    if (s) return s;
    if (!d_offsets) return SHUF_ERR_INVALID_ARG;
    if ((uintptr_t)d_offsets & 7u) return SHUF_ERR_ALIGNMENT;
    if (num_segments == 0 || p->n == 0) {
        p->last_launches = 0;
        return SHUF_OK;
    }
    if (p->idx)
        return gather_route(p, ptr, d_offsets, num_segments, scratch, scratch_bytes, static_cast<cudaStream_t>(stream),
                            0xFFFFFFFFu, 1, nullptr);
    return enqueue(p, ptr, d_offsets, num_segments, scratch, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu, 1);
}

// ------------------------------------------------------------- sharded ---
// NEXT-3: one problem of N elements sharded over ranks.  Rank r
// scatters its input slice at level 0 (shuf_shard_scatter), the runs of each
// bucket go to the bucket's owner (the caller's exchange, NCCL), and every
// owner finishes its buckets as level-1 segments (shuf_shard_continue).
static shuf_status check_shard_args(shuf_plan_s* p, const void* a, const void* b, void* scratch,
                                    uint64_t scratch_bytes, uint64_t m) {
    if (!p) return SHUF_ERR_INVALID_ARG;
    if (p->idx) return SHUF_ERR_UNSUPPORTED;  // elem_bytes in {4, 8, 16}
    if (m > p->n) return SHUF_ERR_INVALID_ARG;
    if (m && (!a || !b || !scratch)) return SHUF_ERR_INVALID_ARG;
    if (((uintptr_t)a & 15u) || ((uintptr_t)b & 7u) || ((uintptr_t)scratch & 15u)) return SHUF_ERR_ALIGNMENT;
    if (m && scratch_bytes < shard_layout(p).total) return SHUF_ERR_SCRATCH;
    return SHUF_OK;
}

extern "C" shuf_status shuf_shard_scatter(shuf_plan_t p, const void* in, uint64_t m, uint64_t pos0, void* out,
                                          uint64_t* d_counts, void* scratch, uint64_t scratch_bytes, void* stream) {
    shuf_status s = check_shard_args(p, in, d_counts, scratch, scratch_bytes, m);
    if (s) return s;
    if (m && (!out || ((uintptr_t)out & 15u))) return out ? SHUF_ERR_ALIGNMENT : SHUF_ERR_INVALID_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = device_setup(p);
    if (e) return cuda_fail(p, e);
    if (m == 0) {
        if (d_counts && (e = cudaMemsetAsync(d_counts, 0, (size_t)p->k * 8, st))) return cuda_fail(p, e);
        p->last_launches = 0;
        return SHUF_OK;
    }
    unsigned char* sc = static_cast<unsigned char*>(scratch);
    unsigned char* buf0 = static_cast<unsigned char*>(const_cast<void*>(in));
    const ScratchLayout lay = shard_layout(p);
    RunParams rp = base_params(p, lay, sc, buf0, 1u, 0);
    rp.n = m;
    rp.shard = 1;
    rp.seg_base = pos0;
    rp.planned_levels = 1;
    p->last_hdr = rp.hdr;
    uint64_t launches = 0;
    Prof* prof = nullptr;
    if ((e = cudaMemsetAsync(rp.hdr, 0, sizeof(Header), st))) return cuda_fail(p, e);
    LAUNCH(SHUF_K_INIT, launch_init_shard(rp, level_params(lay, sc, buf0, 0, true), m, pos0, st, p->grid_small));
    LevelParams lp = level_params(lay, sc, buf0, 0);
    lp.dst = static_cast<unsigned char*>(out);
    LAUNCH(SHUF_K_HIST, launch_hist(rp, lp, st, p->grid_hist));
    LAUNCH(SHUF_K_SCAN, launch_scan(rp, lp, st, p->grid_scan));
    LAUNCH(SHUF_K_SCATTER, launch_scatter(rp, lp, st, p->grid_scatter));
    LAUNCH(SHUF_K_PLAN, launch_shard_counts(rp, lp, d_counts, st));
    p->last_launches = launches;
    return SHUF_OK;
}

extern "C" shuf_status shuf_shard_continue(shuf_plan_t p, void* ptr, uint64_t m, const uint64_t* d_offsets,
                                           uint64_t num_segments, uint64_t base, uint32_t first_level, void* scratch,
                                           uint64_t scratch_bytes, void* stream) {
    shuf_status s = check_shard_args(p, ptr, d_offsets, scratch, scratch_bytes, m);
    if (s) return s;
    if (first_level > kMaxLevels || (m && num_segments == 0)) return SHUF_ERR_INVALID_ARG;
    if (m <= 1 || num_segments == 0) {
        p->last_launches = 0;
        return SHUF_OK;
    }
    ShardOpts so;
    so.n = m;
    so.base = base;
    so.first_level = first_level;
    so.lay = shard_layout(p);
    return enqueue(p, ptr, d_offsets, num_segments, scratch, static_cast<cudaStream_t>(stream), 0xFFFFFFFFu, 1,
                   nullptr, &so);
}

extern "C" shuf_status shuf_profile_run(shuf_plan_t p, void* ptr, const uint64_t* d_offsets, uint64_t num_segments,
                                        void* scratch, uint64_t scratch_bytes, void* stream, float* ms_by_class,
                                        uint32_t* launches_by_class) {
    shuf_status s = check_run_args(p, ptr, scratch, scratch_bytes,
                                   p && p->idx ? 0
                                   : p && d_offsets ? compute_layout(p, seg0_bound(p, num_segments), true).total
                                                    : ~0ull);
    if (s) return s;
    if (!ms_by_class || !launches_by_class) return SHUF_ERR_INVALID_ARG;
    for (int c = 0; c < SHUF_K_CLASSES; ++c) {
        ms_by_class[c] = 0.f;
        launches_by_class[c] = 0;
    }
    if (p->n <= 1 || (d_offsets && num_segments == 0)) return SHUF_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Prof prof;
    prof.st = st;
    s = p->idx ? gather_route(p, ptr, d_offsets, num_segments, scratch, scratch_bytes, st, 0xFFFFFFFFu, 1, &prof)
               : enqueue(p, ptr, d_offsets, num_segments, scratch, st, 0xFFFFFFFFu, 1, &prof);
    if (s) return s;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e) return cuda_fail(p, e);
    for (size_t i = 0; i < prof.cls.size(); ++i) {
        float ms = 0.f;
        if ((e = cudaEventElapsedTime(&ms, prof.ev[2 * i], prof.ev[2 * i + 1]))) return cuda_fail(p, e);
        ms_by_class[prof.cls[i]] += ms;
        launches_by_class[prof.cls[i]] += 1;
    }
    return SHUF_OK;
}

extern "C" shuf_status shuf_debug_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k,
                                               uint32_t* d_out, void* stream) {
    if (k < 2 || k > 65536 || (!d_out && count)) return SHUF_ERR_INVALID_ARG;
    if (count == 0) return SHUF_OK;
    cudaError_t e = launch_debug_bucket_draws(K, level, p0, count, k, d_out, static_cast<cudaStream_t>(stream));
    return e ? SHUF_ERR_CUDA : SHUF_OK;
}

extern "C" shuf_status shuf_sim_rough_scatter(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t* d_T,
                                              uint64_t* d_M, void* stream) {
    if (k < 2 || k > 65536 || n < k || (runs && (!d_T || !d_M))) return SHUF_ERR_INVALID_ARG;
    if (((uintptr_t)d_T & 7u) || ((uintptr_t)d_M & 7u)) return SHUF_ERR_ALIGNMENT;
    if (k > 32768) {  // packed u16 counters: every final bucket count must stay below 2^16
        const double m = (double)n / k;
        if (m + 8.0 * std::sqrt(m) + 64.0 >= 65536.0) return SHUF_ERR_UNSUPPORTED;
    }
    if (runs == 0) return SHUF_OK;
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!e) e = launch_sim_rough(n, k, seed, runs, d_T, d_M, sms * 8, static_cast<cudaStream_t>(stream));
    return e ? SHUF_ERR_CUDA : SHUF_OK;
}

extern "C" shuf_status shuf_debug_fy_draws(uint64_t K, const uint64_t* d_P, const uint32_t* d_s, uint64_t count,
                                           uint32_t* d_out, void* stream) {
    if (count && (!d_P || !d_s || !d_out)) return SHUF_ERR_INVALID_ARG;
    if (count == 0) return SHUF_OK;
    cudaError_t e = launch_debug_fy_draws(K, d_P, d_s, count, d_out, static_cast<cudaStream_t>(stream));
    return e ? SHUF_ERR_CUDA : SHUF_OK;
}

extern "C" shuf_status shuf_last_device_error(shuf_plan_t p, void* stream) {
    if (!p) return SHUF_ERR_INVALID_ARG;
    if (!p->last_hdr) return SHUF_OK;
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e) return cuda_fail(p, e);
    uint32_t err = 0;
    if ((e = cudaMemcpy(&err, &p->last_hdr->error, sizeof err, cudaMemcpyDeviceToHost))) return cuda_fail(p, e);
    if (err) {
        uint32_t zero = 0;
        cudaMemcpy(&p->last_hdr->error, &zero, sizeof zero, cudaMemcpyHostToDevice);
    }
    return (shuf_status)err;
}

extern "C" shuf_status shuf_last_run_stats(shuf_plan_t p, void* stream, uint64_t* out, uint32_t count) {
    if (!p || !out) return SHUF_ERR_INVALID_ARG;
    for (uint32_t i = 0; i < count; ++i) out[i] = 0;
    if (!p->last_hdr) return SHUF_OK;
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e) return cuda_fail(p, e);
    Header h;
    if ((e = cudaMemcpy(&h, p->last_hdr, sizeof h, cudaMemcpyDeviceToHost))) return cuda_fail(p, e);
    // layout: [0] finished, [1] fy_elems, [2 + 2l] hbm(l), [3 + 2l] smem(l)
    if (count > 0) out[0] = h.finished;
    if (count > 1) out[1] = h.fy_elems;
    for (uint32_t l = 0; l < kMaxLevels; ++l) {
        if (2 + 2 * l < count) out[2 + 2 * l] = h.scattered_hbm[l];
        if (3 + 2 * l < count) out[3 + 2 * l] = h.scattered_smem[l];
    }
    if (count > 514) out[514] = h.leafed;
    return SHUF_OK;
}

extern "C" void shuf_destroy(shuf_plan_t p) {
    if (p && p->dev_ready && p->hist_overlap) {
        cudaStreamDestroy(p->side_stream);
        cudaEventDestroy(p->ev_fork);
        cudaEventDestroy(p->ev_join);
    }
    if (p && p->ip_exec) cudaGraphExecDestroy(p->ip_exec);
    if (p && p->idx) shuf_destroy(p->idx);
    if (p && p->ip_cap_stream) cudaStreamDestroy(p->ip_cap_stream);
    delete p;
}

extern "C" const char* shuf_status_string(shuf_status s) {
    switch (s) {
    case SHUF_OK: return "ok";
    case SHUF_ERR_INVALID_ARG: return "invalid argument";
    case SHUF_ERR_UNSUPPORTED: return "unsupported on the device path";
    case SHUF_ERR_ALIGNMENT: return "pointer not 16-byte aligned";
    case SHUF_ERR_SCRATCH: return "scratch buffer too small";
    case SHUF_ERR_DEPTH: return "more scatter levels than planned";
    case SHUF_ERR_CUDA: return "CUDA error";
    case SHUF_ERR_RANK_ORDER: return "ordered-atomic ranking self-check failed (use SHUF_RANK_MODE=match)";
    case SHUF_ERR_INTERNAL: return "IpSc device self-check failed";
    }
    return "unknown status";
}

// Debug: phase clocks recorded by CTA 0 of the finish kernels / the level-0 scatter (SHUF_DBG).
extern "C" shuf_status shuf_debug_clocks(shuf_plan_t p, void* stream, long long* out, uint32_t count) {
    if (!p || !out) return SHUF_ERR_INVALID_ARG;
    if (!p->last_hdr) return SHUF_OK;
    cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e) return cuda_fail(p, e);
    if (count > 512) count = 512;  // [0, 256): finish, [256, 512): level-0 scatter
    if ((e = cudaMemcpy(out, p->last_hdr->clk, count * sizeof(long long), cudaMemcpyDeviceToHost))) return cuda_fail(p, e);
    return SHUF_OK;
}
