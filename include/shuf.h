/*
 * include/shuf.h -- C ABI of libshuf.so, the B200 (sm_100a) deterministic
 * ScatterShuffle hot path.
 *
 * What it computes (PAPER.md = arXiv 2302.03317 text):
 *   A uniformly random permutation of an array of n elements by recursive
 *   ScatterShuffle: every element of a segment draws a uniform
 *   bucket id in [0,k), the segment is grouped by bucket with a
 *   STABLE permutation ("some permutation pi that sorts A"),
 *   recursion continues on every bucket longer than L, and buckets of at most
 *   L elements ("leaves") are finished by Fisher-Yates exactly as Fig. 1
 *   (P:107-110).  Every draw is a counter-based Philox4x32-10 draw mapped to
 *   [0,s) by Lemire's method -- DESIGN.md D1-D5 -- so the result is
 *   a pure function of (n, k, L, seed) and equals the CPU oracle bit for bit.
 *
 * Conventions for every entry point:
 *   - Device pointers are CUDA device addresses (e.g. torch .data_ptr()),
 *     16-byte aligned; host pointers are plain host memory.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     All device work is enqueued on it; no call synchronises the stream
 *     unless its comment says so.  No call allocates device memory except
 *     shuf_plan (a few hundred bytes of plan metadata).
 *   - The caller owns ptr, scratch, offsets and the stream.  The plan owns
 *     only its own metadata.  A plan may be used by one stream at a time.
 *   - Errors: argument errors are returned synchronously and nothing is
 *     enqueued.  CUDA launch errors return SHUF_ERR_CUDA.  Errors detected on
 *     the device (depth bound exceeded, scratch too small) are latched in the
 *     plan's device status word and read by shuf_last_device_error() (which
 *     synchronises).  There is no CPU fallback: without a CUDA device every
 *     compute entry point returns SHUF_ERR_CUDA.
 */
#ifndef SHUF_H
#define SHUF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct shuf_plan_s *shuf_plan_t;

typedef enum {
    SHUF_OK = 0,
    SHUF_ERR_INVALID_ARG = 1, /* n/k/L/elem_bytes/offsets outside the domain     */
    SHUF_ERR_UNSUPPORTED = 2, /* valid for the oracle, not supported on device   */
    SHUF_ERR_ALIGNMENT = 3,   /* ptr/scratch/offsets not 16-byte aligned         */
    SHUF_ERR_SCRATCH = 4,     /* scratch_bytes smaller than shuf_scratch_bytes() */
    SHUF_ERR_DEPTH = 5,       /* more levels than planned (device-detected)      */
    SHUF_ERR_CUDA = 6,        /* a CUDA runtime error; see shuf_last_cuda_error  */
    SHUF_ERR_RANK_ORDER = 7,  /* device self-check: same-address shared atomics of
                                 one warp instruction did not return in lane order
                                 (DESIGN.md 6); rerun with SHUF_RANK_MODE=match   */
    SHUF_ERR_INTERNAL = 8     /* device self-check of the IpSc mode failed (a
                                 final bucket size not reached, or R >= 2^32)      */
} shuf_status;

/* Create a plan for shuffling n elements of elem_bytes bytes each with k
 * buckets per scatter level, leaves of at most L elements, and seed `seed`
 * (D2: the single-problem key is K = seed).
 * Domain: elem_bytes in {4, 8, 16}; 2 <= k <= 1024 on the device (any k;
 * powers of two <= 256 take the 8-bit-lane shift path of P:99; larger k
 * return SHUF_ERR_UNSUPPORTED); 1 <= L <= the fused size S_fuse (about 20 K
 * 4-byte, 11 K 8-byte or 6 K 16-byte elements; larger L return
 * SHUF_ERR_UNSUPPORTED).  n may be 0 or 1 (no-ops); n is 64-bit.  For
 * shuf_segmented, n is the total number of elements over all segments.
 * Returns NULL on error; the reason is in shuf_last_status(). */
shuf_plan_t shuf_plan(uint64_t n, uint32_t elem_bytes, uint32_t k, uint32_t L, uint64_t seed);

/* Status of the last shuf_plan call on this thread. */
shuf_status shuf_last_status(void);

/* Bytes of device scratch shuf_run needs for this plan: one ping-pong buffer
 * of n*elem_bytes plus per-level metadata sized from the planned recursion
 * (<= 1 % of n*elem_bytes for inputs of 256 MB and more, a few
 * hundred KB at most below that).  The per-level tables are sized for the
 * planned structure with a 6-sigma margin; a run whose level would exceed
 * them (astronomically rare for random draws) latches SHUF_ERR_SCRATCH on
 * the device -- read it with shuf_last_device_error.  Writes *bytes. */
shuf_status shuf_scratch_bytes(shuf_plan_t p, uint64_t *bytes);

/* Bytes of device scratch shuf_segmented needs for num_segments segments of
 * this plan's n elements in total: the worst case of min(num_segments,
 * n / (S_fuse + 1) + 1) segments longer than the fused size at every level
 * (segment lengths are device data, unknown at plan time). */
shuf_status shuf_scratch_bytes_segmented(shuf_plan_t p, uint64_t num_segments, uint64_t *bytes);

/* Shuffle ptr[0..n) in place (result in ptr) using `scratch` (device, at
 * least shuf_scratch_bytes).  Stream-ordered, no host synchronisation, no
 * allocation.  The permutation is DESIGN.md D6 with K = seed.  Errors the
 * device detects after the call returned (SHUF_ERR_DEPTH, SHUF_ERR_SCRATCH;
 * the output is then incomplete) are only reported by shuf_last_device_error:
 * callers MUST check it after synchronising before using the result. */
shuf_status shuf_run(shuf_plan_t p, void *ptr, void *scratch, uint64_t scratch_bytes, void *stream);

/* Segmented batch shuffle (D7): segment s = ptr[off[s] .. off[s+1])
 * is shuffled independently with key K(seed, s) = seed + s*0x9E3779B97F4A7C15
 * and segment-relative positions.  d_offsets: DEVICE array of num_segments+1
 * ascending uint64, d_offsets[0] = 0, d_offsets[num_segments] = n (the plan's
 * n); empty segments allowed.  The offsets are not validated on the device
 * beyond the plan's bounds.  scratch: at least shuf_scratch_bytes_segmented
 * (p, num_segments) bytes.  Device errors as for shuf_run. */
shuf_status shuf_segmented(shuf_plan_t p, void *ptr, const uint64_t *d_offsets, uint64_t num_segments,
                           void *scratch, uint64_t scratch_bytes, void *stream);

/* Sharded single shuffle (data sets approaching memory
 * size, P:9).  ONE problem of N elements (D6 with K = seed) is split over G
 * ranks: rank r holds the global positions [lo_r, hi_r).  D6's level 0 is the
 * only step that crosses ranks (the stable bucket grouping of the
 * whole array); every later level and leaf stays inside one bucket.
 *   1. shuf_shard_scatter: the rank's slice in[0..m) (global positions
 *      [pos0, pos0+m)) is grouped by its level-0 draws, stably, into out[0..m)
 *      (bucket-major, position order inside a bucket) and d_counts[b] (DEVICE,
 *      k uint64) receives the slice's count of bucket b.  The slice is
 *      scattered whatever its length: the caller only shards problems with
 *      N > L (otherwise D6 has no level 0 and the whole array is one leaf).
 *   2. The caller exchanges the runs (all-to-all-v over NCCL,
 *      paper_2302_03317_b200/sharded.py): bucket b's final place in the
 *      global level-0 output is o_b + sum over source ranks s' < s of their
 *      counts of b, so an owner of buckets [b0, b1) receives them in
 *      (bucket, source rank) order -- exactly D6's stable order.
 *   3. shuf_shard_continue: ptr[0..m) holds global positions [base, base+m)
 *      of the level-first_level input, cut into num_segments consecutive
 *      segments d_offsets[0..num_segments] (DEVICE, ascending, 0 .. m), each
 *      a child (bucket) at level first_level (= 1) of the one problem: D6
 *      continues on each with key K(seed, 0) and global positions, in place.
 * The concatenation of all ranks' ptr is D6's output of the whole problem,
 * bit for bit.  The plan's n is a CAPACITY: m <= n for both calls (its level
 * count and chunk size come from n).  scratch: shuf_scratch_bytes_shard bytes
 * (16-byte aligned), one buffer serves both calls; in/out/ptr 16-byte aligned;
 * elem_bytes must be 4, 8 or 16 (else SHUF_ERR_UNSUPPORTED).  Stream-ordered,
 * no host synchronisation, no allocation; device errors via
 * shuf_last_device_error. */
shuf_status shuf_scratch_bytes_shard(shuf_plan_t p, uint64_t *bytes);
shuf_status shuf_shard_scatter(shuf_plan_t p, const void *in, uint64_t m, uint64_t pos0, void *out,
                               uint64_t *d_counts, void *scratch, uint64_t scratch_bytes, void *stream);
shuf_status shuf_shard_continue(shuf_plan_t p, void *ptr, uint64_t m, const uint64_t *d_offsets,
                                uint64_t num_segments, uint64_t base, uint32_t first_level, void *scratch,
                                uint64_t scratch_bytes, void *stream);

/* The paper's own In-Place ScatterShuffle (D10
 * and 6.3; IpSc = RoughScatter P:262-265 in ParRoughScatter's split/merge tree
 * P:479-491, then FineScatter P:357-425, at every level of Fig. 2).
 * Shuffles ptr[0..n) IN PLACE with an auxiliary DEVICE buffer `aux` of
 * shuf_aux_bytes_ipsc() bytes: the staged start of every (ParRoughScatter
 * node, bucket) of one batch of segments -- O(k * subtasks) words, the paper's
 * O(k [log_k n + P]) bound (Theorem) with a batch of at most
 * max(2^21, k * nodes of the root) entries -- plus the levels' segment lists
 * (16 bytes per segment longer than L).  Deterministic and reproducible: the
 * result equals the oracle's D10 (oracle_ipsc_shuffle) bit for bit -- a
 * different permutation from shuf_run's D6 (another algorithm), equally
 * uniform.  NOT allocation-free on the host side: the level loop plans
 * batches on the host and SYNCHRONISES the stream once per level.  ptr and
 * aux 16-byte aligned; elem_bytes 4, 8 or 16 (else SHUF_ERR_UNSUPPORTED).
 * Device self-check failures return SHUF_ERR_INTERNAL. */
shuf_status shuf_aux_bytes_ipsc(shuf_plan_t p, uint64_t *bytes);
shuf_status shuf_run_ipsc(shuf_plan_t p, void *ptr, void *aux, uint64_t aux_bytes, void *stream);
/* Tests only: IpSc on levels < max_levels (segments of that level left as they
 * are), Fisher-Yates leaves only if run_leaves -- the oracle's max_levels mode. */
shuf_status shuf_debug_ipsc_levels(shuf_plan_t p, void *ptr, void *aux, uint64_t aux_bytes, void *stream,
                                   uint32_t max_levels, int run_leaves);

/* In-place mode (the paper's in-place motivation P:32-36,
 * P:39-43).  Shuffles ptr[0..n) using an auxiliary DEVICE buffer `aux` of
 * shuf_aux_bytes_inplace() bytes, about 2 bytes per 128-byte block of ptr plus
 * O(k * 2048 * 128 B) for bucket buffers -- under 5 % of n*elem_bytes above
 * 1 GiB
 * instead of shuf_run's n*elem_bytes ping-pong buffer.  Each level longer than
 * the fused size classifies elements into 128-byte blocks in place, permutes
 * the blocks into their buckets' regions and fills the bucket heads and tails
 * from the leftover buffers (the block scheme of in-place samplesort).
 * Element buckets are the D4 draws at their positions at that level, so the
 * level-0 bucket contents equal shuf_run's; within a bucket the order depends
 * on atomics: the result is a uniformly random permutation but NOT
 * reproducible and NOT equal to shuf_run's.  Segments of at most the fused
 * size and leaves run the same (deterministic) in-place finish and leaf
 * kernels as shuf_run.  Stream-ordered, no host synchronisation: the level
 * loop runs on the device as one launch of a CUDA graph with conditional
 * WHILE nodes (levels, batches of segments) that the plan builds on the first
 * call for a given (ptr, aux) and caches; calls with other buffers rebuild it.
 * ptr and aux must be 16-byte aligned; aux is overwritten; no allocation of
 * device memory (the graph itself is host-side driver state). */
shuf_status shuf_aux_bytes_inplace(shuf_plan_t p, uint64_t *bytes);
shuf_status shuf_run_inplace(shuf_plan_t p, void *ptr, void *aux, uint64_t aux_bytes, void *stream);

/* Test hook: the in-place mode with only levels l < max_levels and leaves
 * Fisher-Yates'd only if run_leaves != 0 (max_levels = 1, run_leaves = 0
 * leaves each level-0 bucket, in arbitrary order, at its bucket range). */
shuf_status shuf_debug_inplace_levels(shuf_plan_t p, void *ptr, void *aux, uint64_t aux_bytes, void *stream,
                                      uint32_t max_levels, int run_leaves);

/* Test hook: like shuf_run, but only scatter levels l < max_levels run (in
 * HBM or in shared memory alike) and leaves are Fisher-Yates'd only if
 * run_leaves != 0; the state reached is left in ptr.  Equals the oracle's
 * level-limited mode (oracle_shuffle(..., max_levels, run_leaves)). */
shuf_status shuf_debug_run_levels(shuf_plan_t p, void *ptr, void *scratch, uint64_t scratch_bytes, void *stream,
                                  uint32_t max_levels, int run_leaves);

/* Test hook (raw-draw parity): out[i] = D4 bucket draw at (level, p0 + i)
 * under key K for bucket count k; d_out is a device array of count uint32. */
shuf_status shuf_debug_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k,
                                    uint32_t *d_out, void *stream);

/* Test hook: out[x] = D5 Fisher-Yates partner of step d_i[x] (bound
 * d_i[x]+1) of the leaf starting at problem position d_q[x], under key K;
 * device arrays of count elements. */
shuf_status shuf_debug_fy_draws(uint64_t K, const uint64_t *d_q, const uint32_t *d_i, uint64_t count,
                                uint32_t *d_out, void *stream);

/* Kernel classes reported by shuf_profile_run. */
enum {
    SHUF_K_INIT = 0,    /* work-list initialisation                         */
    SHUF_K_HIST = 1,    /* per-chunk bucket histogram (draws only, no data)  */
    SHUF_K_SCAN = 2,    /* decoupled-lookback exclusive scan of the counts   */
    SHUF_K_PLAN = 3,    /* next-level segment planner                        */
    SHUF_K_SCATTER = 4, /* HBM stable scatter                                */
    SHUF_K_FINISH = 5,  /* fused shared-memory finish (levels + FY leaves)   */
    SHUF_K_LEAF = 6,    /* leaf kernel: FY of HBM-level leaves / short segments */
    SHUF_K_CLASSES = 7
};

/* Measurement hook: enqueue the same work as shuf_run (d_offsets == NULL) or
 * shuf_segmented, bracket every kernel launch with CUDA events on `stream`,
 * SYNCHRONISE the stream, and write per-class summed milliseconds and launch
 * counts to host arrays of SHUF_K_CLASSES entries.  Allocates events. */
shuf_status shuf_profile_run(shuf_plan_t p, void *ptr, const uint64_t *d_offsets, uint64_t num_segments,
                             void *scratch, uint64_t scratch_bytes, void *stream, float *ms_by_class,
                             uint32_t *launches_by_class);

/* Measurement counters of the last run on this plan (synchronises):
 * out[0] = elements written by the fused finish, out[1] = elements in
 * Fisher-Yates leaves, out[2+2l] = elements scattered through HBM at level l,
 * out[3+2l] = elements scattered in shared memory at level l (l < 256),
 * out[514] = elements written by the leaf kernel.
 * Writes min(count, 515) entries; the rest are zero. */
shuf_status shuf_last_run_stats(shuf_plan_t p, void *stream, uint64_t *out, uint32_t count);

/* Debug (timing experiments; recorded only when the environment variable
 * SHUF_DBG selects them): phase timestamps (clock64) of CTA 0 of the finish
 * kernels during the last run on this plan (6 per item; SHUF_DBG=4 the
 * pipelined finish's S/F groups, SHUF_DBG=2 the general finish) in
 * out[0, 256) and of CTA 0 of the level-0 HBM scatter (6 per tile,
 * SHUF_DBG=1) in out[256, 512); writes min(count, 512) values.
 * Synchronises. */
shuf_status shuf_debug_clocks(shuf_plan_t p, void *stream, long long *out, uint32_t count);

/* Synchronise `stream` and return the plan's latched device error (SHUF_OK
 * if none), clearing it. */
shuf_status shuf_last_device_error(shuf_plan_t p, void *stream);

/* Hidden-constant simulation (section 7,
 * P:773-788, of Lemma 2 P:284-296 and Lemma 4 / Corollary 5 P:392-416),
 * DESIGN.md D9.  For run r = 0 .. runs-1 with key K(seed, r): RoughScatter
 * on n items into k buckets of capacities c_i = floor((i+1)n/k)
 * - floor(i n/k), iteration t placing one item into bucket D4 draw (level 0,
 * position t), stopping when a bucket is full; d_T[r] = items placed T (the
 * Lemma-2 remainder is R = n - T).  The remaining draws t = T .. n-1 complete
 * the final sizes n^f; d_M[r] = sum_i |D_i| with D_i the prefix sums of
 * n^f_i - c_i (TwoSweep's swaps, Lemma 4).  d_T, d_M: DEVICE arrays of runs
 * uint64, 8-byte aligned, owned by the caller.  2 <= k <= 2^16 and n >= k
 * (SHUF_ERR_INVALID_ARG); k > 2^15 needs n/k well below 2^16
 * (SHUF_ERR_UNSUPPORTED).  Stream-ordered; exact integers (bit-identical to
 * the oracle's oracle_sim_rough_scatter). */
shuf_status shuf_sim_rough_scatter(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t *d_T,
                                   uint64_t *d_M, void *stream);

/* The cudaError_t behind the last SHUF_ERR_CUDA returned for this plan. */
int shuf_last_cuda_error(shuf_plan_t p);

/* Number of kernel launches the last shuf_run/shuf_segmented enqueued. */
uint64_t shuf_last_launch_count(shuf_plan_t p);

/* Which in-warp ranking the device path uses (block_ops.cuh): 1 = one
 * shared-memory atomicAdd per element (same-address atomics of a warp
 * instruction return in lane order -- verified by a probe kernel at the
 * first run, since the PTX ISA leaves that order unspecified), 0 = the
 * documented __match_any_sync path, -1 = not probed yet.  The environment
 * variable SHUF_RANK_MODE=atomic|match forces one of them. */
int shuf_rank_mode(void);

/* Planned number of HBM (global) scatter levels for this plan. */
uint32_t shuf_planned_levels(shuf_plan_t p);

void shuf_destroy(shuf_plan_t p);
const char *shuf_status_string(shuf_status s);

#ifdef __cplusplus
}
#endif
#endif /* SHUF_H */
