// Internal descriptors, scratch layout and kernel entry points of libshuf.
// DESIGN.md section 4 describes the pipeline; section 5 the HBM layout.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "philox.cuh"

namespace shuf {

// ----------------------------------------------------------- constants ----
constexpr int kWarps = 16;                 // warps per CTA in the ranking kernels
constexpr int kThreads = kWarps * 32;      // 512
constexpr uint32_t kMaxK = 1024;           // device bucket-count limit
constexpr uint32_t kMaxGatherElem = 256;   // largest element (bytes); sizes other than 4/8/16 take the gather route
constexpr uint32_t kScanTile = 4096;       // entries per decoupled-lookback tile
constexpr uint32_t kSmemLimit = 227 * 1024;
constexpr uint32_t kFinishBucketGroup = 16; // children per finish work unit
constexpr uint32_t kMaxLevels = 256;
constexpr uint32_t kScatterTileBytes = 32768; // HBM scatter tile (kernels_scatter.cu); chunks are multiples of it
#ifndef SHUF_TILE16
#define SHUF_TILE16 65536
#endif
#ifndef SHUF_TILE8
#define SHUF_TILE8 32768
#endif
// Tile bytes per element size: 16-byte records take 64 KiB tiles (4096 records: with k = 1024,
// config 4, 32 KiB tiles leave ~2 records per bucket run; scatter 138.8 -> 126.0 ms, r04h).
__host__ __device__ constexpr uint32_t scatter_tile_bytes(uint32_t eb) {
    return eb == 16 ? SHUF_TILE16 : eb == 8 ? SHUF_TILE8 : kScatterTileBytes;
}
constexpr uint32_t kFrontierCap = 256;      // pending in-smem sub-segments per level
constexpr uint32_t kIpBlockBytes = 128;     // in-place mode block (kernels_inplace.cu)
constexpr uint32_t kIpBatchCap = 2048;      // in-place mode: stripes (and segments) per batch

// ---------------------------------------------------------- descriptors ---
// A segment processed by an HBM-resident ("global") scatter level.
struct SegDesc {
    uint64_t start;   // first element (absolute index into the buffer)
    uint64_t len;     // elements
    uint64_t origin;  // absolute index of the problem's position 0 (D7)
    uint64_t key;     // K(seed, s)
    uint64_t cbase;   // first count entry of this segment's (bucket, chunk) block
    uint32_t nchunks; // chunks of this segment
    uint32_t pad;
};

// Chunk j of a level: chunk c of segment seg, positions
// [start + c*C, min(start + len, start + (c+1)*C)).
struct ChunkDesc {
    uint32_t seg;
    uint32_t c;
};

// Per-level (two slots, by level parity) device counters.
struct LevelCounters {
    uint32_t nseg;
    uint32_t nchunk;
    uint32_t scan_ticket;
    uint32_t nfuse;    // children of this level in the fused list (RunParams::fused)
    uint32_t nstream;  // children of this level for k_finish_stream
    uint32_t pad;
};

struct Header {
    LevelCounters lv[2];
    uint64_t root_off[2];  // {0, n}: the single problem as a one-segment batch
    uint32_t error;        // latched shuf_status detected on the device
    uint32_t pad0;
    // work tickets of the segmented mode's leaf passes (one per pass; zeroed with the header):
    // warps take the next warp-unit from the pass's counter instead of a fixed stride
    unsigned long long leaf_ticket[3];
    // measurement counters (one atomic per chunk / per shared-memory scatter)
    uint64_t scattered_hbm[kMaxLevels];   // elements scattered through HBM at level l
    uint64_t scattered_smem[kMaxLevels];  // elements scattered in shared memory at level l
    uint64_t finished;                    // elements written by the fused finish
    uint64_t fy_elems;                    // elements in Fisher-Yates leaves
    uint64_t leafed;                      // elements written by the leaf kernel
    uint64_t nitems;                      // fused items recorded for the leaf kernel (RunParams::items)
    long long clk[256];                   // phase timestamps of CTA 0 of the fast finish (shuf_debug_clocks)
    long long sclk[256];                  // phase timestamps of CTA 0 of the level-0 HBM scatter
};

// Byte offsets of every region inside the caller's scratch buffer.  The
// per-level tables are sized from the planned structure (shuf_api.cu
// level_caps): slot s holds the levels l with l & 1 == s, so its capacity is
// the largest bound among them.  A level that would overflow its slot latches
// SHUF_ERR_SCRATCH on the device.
struct ScratchLayout {
    uint64_t pingpong;  // n * eb
    uint64_t header;
    uint64_t segs[2];
    uint64_t chunks[2];
    uint64_t counts[2];  // u32 per (bucket, chunk)
    uint64_t prefix[2];  // u64 per (bucket, chunk)
    uint64_t status[2];  // u64 per scan tile
    uint64_t flags;      // u8 per child of a level: 1 = finished by the general finish kernel
    uint64_t items;      // item records (item_rec_stride bytes each), max_items of them (SHUF_DEFER=1 only)
    uint64_t max_items;
    uint64_t fused;      // u32 child indices of the current level that the finish kernels take
    uint64_t max_fused;
    uint64_t total;
    uint64_t seg_cap[2], chunk_cap[2], entry_cap[2], tile_cap[2];
    uint64_t meta;       // total - pingpong bytes: the metadata
};

// Everything a kernel needs about the run (passed by value).
struct RunParams {
    unsigned char* buf0;  // ptr (level-0 input, final output)
    unsigned char* buf1;  // ping-pong buffer in scratch
    Header* hdr;
    uint64_t n;
    uint32_t eb;
    uint32_t k;
    uint32_t L;
    uint32_t S_fuse;      // max elements of a segment finished in shared memory
    uint32_t chunk;       // C: elements per chunk (multiple of the tile)
    uint32_t max_levels;  // debug level limit (0xFFFFFFFF = none)
    uint32_t planned_levels;
    int run_leaves;
    BucketParams bp;
    uint64_t seed;
    uint32_t rank_ordered;  // 1: ordered shared atomics verified on this GPU (block_ops.cuh)
    uint32_t fin_nbuf;      // finish-kernel data buffers (2 = items double-buffered)
    uint32_t fast;          // 1: k_finish_fast runs first; the general finish takes flagged children only
    unsigned char* flags;   // per-child flags of the current level (ScratchLayout::flags)
    uint32_t dbg;           // timing experiments only (SHUF_DBG): skip parts of the fast finish
    uint32_t leafk;         // 1: leaves of HBM levels / user segments go to the leaf kernel (kernels_leaf.cu)
    uint32_t defer;         // 1: the finish leaves the leaves of single-level items to the leaf kernel
    unsigned char* items;   // item records: {start, origin, key} + u16 bucket starts [0, k]
    uint32_t* fused;        // with the leaf kernel: the level's children that need the finish kernels
    uint64_t max_fused;     // (k_plan writes them; 0: the finish kernels scan every child)
    // Sharded problem (NEXT-3, shuf_shard_*): buf0 holds a contiguous slice of one
    // problem of global positions [seg_base, seg_base + n); its segments are
    // children at level first_level, keyed K(seed, 0), positions global.
    uint32_t S_stream;      // children with S_fuse < len <= S_stream: k_finish_stream (0: none)
    uint32_t shard;         // 1: the above; 0: single problem / user segments (D7)
    uint32_t first_level;   // level of the initial segments (0 unless shard)
    uint64_t seg_base;      // global position of buf0[0] (shard only)
};

// Item record of a fused item whose children are all leaves (defer mode):
// u64 start, origin, key, then k+1 u16 child starts relative to start.
__host__ __device__ inline uint32_t item_rec_stride(uint32_t k) { return (24u + 2u * (k + 1u) + 15u) & ~15u; }

struct LevelParams {
    uint32_t level;     // l
    int slot;           // l & 1
    SegDesc* segs;
    ChunkDesc* chunks;
    uint32_t* counts;
    uint64_t* prefix;
    uint64_t* status;
    LevelCounters* ctr;
    // next level (slot ^ 1)
    SegDesc* nsegs;
    ChunkDesc* nchunks;
    LevelCounters* nctr;
    uint64_t max_segs, max_chunks;
    unsigned char* src;  // level input buffer
    unsigned char* dst;  // level output buffer
    uint32_t leaf_unit;  // leaves per warp-unit of k_leaf_children (1 or 32, leaf_unit())
    // k_leaf_children takes the leaves with leaf_lo < length <= leaf_hi; its warp
    // slots hold a leaf of leaf_hi elements (leaf_hi = 0: L).  A level whose
    // expected leaf length is well below L runs a first pass with small slots
    // (more warps per SM) and a second pass with full slots for the outliers.
    uint32_t leaf_lo, leaf_hi;
};

// ------------------------------------------------------- in-place mode ---
// A segment of an in-place HBM level (kernels_inplace.cu); zbase/nz: its
// stripes within the batch.
struct IpSeg {
    uint64_t start, len;
    uint32_t zbase, nz;
};

struct IpCounters {
    uint32_t nnext[2];  // next-level list lengths (by level parity)
    unsigned long long cursor;  // k_ip_permute pair cursor
};

// One batch of an in-place level: segments [s0, s0+nseg) of the level's
// list, nz stripes.
struct IpBatch {
    uint32_t s0, nseg, nz, first;  // first: scratch of k_ip_level_plan
};

// Device-resident loop state of the in-place mode.  The whole level loop runs
// on the device (a CUDA graph with two nested conditional WHILE nodes, levels
// and batches; shuf_api.cu): every batch kernel resolves its batch from here.
struct IpState {
    uint32_t level, cur, batch, nbatch;  // cur: parity of the level's segment list
    uint32_t nseg;                       // segments of the current level
    uint32_t C;                          // stripe window per batch (batches hold < 2C stripes)
    uint32_t max_batches, pad;
    IpBatch* batches;
};

// One batch of segments of one in-place level.  With `state` set, the
// fields marked (*) are resolved on the device from the loop state at the
// start of every kernel (ip_resolve); the host fills the rest.
struct IpParams {
    IpSeg* segs;              // (*) the batch's segments
    uint32_t nseg;            // (*) segments in the batch
    uint32_t nstripes;        // (*) stripes in the batch
    uint32_t level;           // (*)
    uint32_t pad;
    uint64_t Z;               // stripe length (elements, multiple of the block)
    uint32_t* zseg;           // stripe -> batch segment
    uint64_t* N;              // [nseg*k] elements per (segment, bucket)
    uint32_t* F;              // [nseg*k] full blocks per (segment, bucket)
    uint64_t* S;              // [nseg*(k+1)] bucket starts (segment-relative)
    uint64_t* wr;             // [nseg*k] packed (write << 32 | read + 2^31) block pointers
    uint32_t* regpre;         // [nseg*k] inclusive prefix of the regions' unprocessed slots (per segment)
    uint64_t* segtot;         // [nseg] unprocessed slots per segment
    uint32_t* ovf;            // [nseg*k] 1: the overflow block of (segment, bucket) is used
    unsigned char* ovfd;      // [nseg*k] overflow blocks
    uint32_t* pcnt;           // [nstripes*k] partial counts
    unsigned char* part;      // [nstripes*k] partial buffers (one block each)
    uint16_t* tags;           // per block slot: bucket / empty / read
    IpSeg* next;              // (*) next level's list
    uint32_t* nnext;          // (*)
    uint64_t max_next;
    unsigned long long* cursor;
    IpState* state;           // device loop state
    IpSeg* segbase[2];        // the two level lists (by parity)
    uint32_t* nnext_base;     // their lengths (IpCounters::nnext)
};

#ifdef __CUDACC__
__device__ __forceinline__ IpParams ip_resolve(IpParams ip) {
    if (!ip.state) return ip;
    const IpState* st = ip.state;
    const uint32_t cur = st->cur;
    const IpBatch bt = st->batches[st->batch];
    ip.segs = ip.segbase[cur] + bt.s0;
    ip.nseg = bt.nseg;
    ip.nstripes = bt.nz;
    ip.level = st->level;
    ip.next = ip.segbase[cur ^ 1u];
    ip.nnext = ip.nnext_base + (cur ^ 1u);
    return ip;
}
#endif

// In-place ScatterShuffle of the paper (NEXT-2, kernels_ipsc.cu): one batch
// of segments of a level; heap node v of segment s has node slot
// segs[s].node_base + v - 1 in the s-table (k staged starts per slot).
struct IpscSeg {
    uint64_t a, m;       // [a, a+m) at the batch's level
    uint64_t node_base;  // first node slot
    uint32_t t, pad;     // ParRoughScatter depth
};

struct IpscParams {
    unsigned char* X;
    uint32_t k, L, level, run_leaves;
    uint64_t seed;
    const IpscSeg* segs;
    const uint2* work;   // (segment, heap node) per CTA of an RoughScatter launch
    uint64_t* s_tab;     // node slot * k + i
    uint64_t* S;         // final bucket starts, segment * (k + 1) + i
    uint64_t* next;      // next level's (start, len) list
    uint32_t* next_cnt;
    uint64_t max_next;
    Header* hdr;
    long long* clk;      // SHUF_DBG & 128: phase clocks of CTA 0's first small segment (hdr->clk)
};

// ------------------------------------------------------ host launchers ---
cudaError_t launch_ipsc_rs(const IpscParams& P, uint32_t eb, uint32_t nwork, bool merge, bool wide, uint32_t grid,
                           cudaStream_t s);
cudaError_t launch_ipsc_fine(const IpscParams& P, uint32_t eb, uint32_t nseg, cudaStream_t s);
cudaError_t launch_ipsc_children(const IpscParams& P, uint32_t nseg, cudaStream_t s, int grid);
uint32_t ipsc_small_cap(uint32_t k, uint32_t eb, uint32_t* tmax);
cudaError_t launch_ipsc_small(const IpscParams& P, uint32_t eb, const uint64_t* list, uint32_t count, uint32_t cap,
                              uint32_t tmax, cudaStream_t s, int grid);
cudaError_t launch_leaf_ipsc(const RunParams& rp, const uint64_t* S, uint32_t nseg, cudaStream_t s, int grid);
cudaError_t launch_init(const RunParams& rp, const LevelParams& lp0, cudaStream_t s, int grid);
cudaError_t launch_init_segmented(const RunParams& rp, const LevelParams& lp0, const uint64_t* d_offsets,
                                  uint64_t num_segments, cudaStream_t s, int grid);
cudaError_t launch_init_shard(const RunParams& rp, const LevelParams& lp0, uint64_t m, uint64_t pos0, cudaStream_t s,
                              int grid);
cudaError_t launch_shard_counts(const RunParams& rp, const LevelParams& lp, uint64_t* counts, cudaStream_t s);
cudaError_t launch_hist(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_scan(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_scatter(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_plan(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_finish_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_finish_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                   cudaStream_t s, int grid);
uint32_t finish_smem_bytes(uint32_t S_fuse, uint32_t eb, uint32_t k, uint32_t nbuf);
uint32_t finish_max_elems(uint32_t eb, uint32_t k);
uint32_t finish_stream_smem_bytes(uint32_t S, uint32_t eb, uint32_t k);
cudaError_t configure_finish_stream(uint32_t eb, uint32_t smem);
cudaError_t launch_finish_stream(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
uint32_t finish_smem_budget(uint32_t eb);
cudaError_t launch_finish_fast(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_finish_fast_ip(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t configure_fast(uint32_t eb, uint32_t k);
uint32_t fast_smem_bytes(uint32_t eb, uint32_t k);
uint32_t leaf_unit(uint32_t eb, uint32_t L, uint64_t avg);
uint32_t leaf_warps_per_sm(uint32_t eb, uint32_t L);
uint32_t leaf_warps_per_cta(uint32_t eb, uint32_t L);
cudaError_t launch_leaf_children(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
// segments with lo < length <= hi (hi = 0: L), warp slots sized for hi elements
cudaError_t launch_leaf_segments(const RunParams& rp, const uint64_t* d_offsets, uint64_t num_segments,
                                 cudaStream_t s, int grid, uint32_t lo = 0, uint32_t hi = 0,
                                 unsigned long long* ticket = nullptr);
cudaError_t launch_leaf_items(const RunParams& rp, cudaStream_t s, int grid);
cudaError_t configure_leaf(uint32_t eb, uint32_t L);
cudaError_t occupancy_leaf(uint32_t eb, uint32_t L, int* blocks);
uint32_t leaf_smem_bytes(uint32_t eb, uint32_t L);
cudaError_t launch_ip_root(Header* hdr, uint64_t n, cudaStream_t s);
cudaError_t launch_ip_init(const IpParams& ip, Header* hdr, uint64_t n, const IpState& init, cudaStream_t s);
cudaError_t launch_ip_level_plan(const RunParams& rp, const IpParams& ip, cudaGraphConditionalHandle hb, cudaStream_t s);
cudaError_t launch_ip_batch_next(const IpParams& ip, cudaGraphConditionalHandle hb, cudaStream_t s);
cudaError_t launch_ip_level_next(const RunParams& rp, const IpParams& ip, cudaGraphConditionalHandle hl,
                                 cudaStream_t s);
cudaError_t launch_ip_stripes(const IpParams& ip, cudaStream_t s);
cudaError_t launch_ip_classify(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t launch_ip_plan(const RunParams& rp, const IpParams& ip, cudaStream_t s);
cudaError_t launch_ip_permute(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t launch_ip_fill(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t launch_finish_ipchildren(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t launch_leaf_ipchildren(const RunParams& rp, const IpParams& ip, cudaStream_t s, int grid);
cudaError_t configure_inplace(uint32_t eb, uint32_t k);
cudaError_t occupancy_inplace(uint32_t eb, uint32_t k, int* classify, int* permute);
uint32_t ip_classify_smem_bytes(uint32_t eb, uint32_t k);
cudaError_t launch_iota(void* idx, uint32_t ieb, uint64_t n, cudaStream_t s, int grid);
cudaError_t launch_gather(const void* in, void* out, const void* idx, uint32_t ieb, uint64_t n, uint32_t eb,
                          cudaStream_t s, int grid);
cudaError_t launch_copy_big(const RunParams& rp, const LevelParams& lp, cudaStream_t s, int grid);
cudaError_t launch_rank_order_probe(int grid, uint32_t* d_violations, cudaStream_t s);
uint32_t scatter_smem_bytes(uint32_t eb, uint32_t k);
cudaError_t configure_scatter(uint32_t smem);
cudaError_t occupancy_scatter(uint32_t eb, uint32_t k, int* blocks);
cudaError_t configure_finish(uint32_t smem);
cudaError_t occupancy_level(uint32_t eb, uint32_t k, int* hist, int* scan, int* scatter);
cudaError_t occupancy_finish(uint32_t eb, uint32_t smem, int* blocks);
cudaError_t launch_sim_rough(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t* T, uint64_t* M, int grid,
                             cudaStream_t s);
cudaError_t launch_debug_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k,
                                      uint32_t* d_out, cudaStream_t s);
cudaError_t launch_debug_fy_draws(uint64_t K, const uint64_t* d_P, const uint32_t* d_s, uint64_t count,
                                  uint32_t* d_out, cudaStream_t s);

}  // namespace shuf
