// CTA-wide building blocks shared by the scatter and finish kernels:
// draw generation into shared memory, warp match/ballot stable ranking,
// block exclusive scan.  (CUDA path only; the oracle never includes this.)
#pragma once
#include <cstdint>

#include "philox.cuh"
#include "ptx.cuh"
#include "shuf_internal.cuh"

namespace shuf {

// Element vector types by element size.
template <int EB> struct ElemT;
template <> struct ElemT<4> { using type = uint32_t; };
template <> struct ElemT<8> { using type = uint2; };
template <> struct ElemT<16> { using type = uint4; };

__device__ __forceinline__ uint32_t warp_inclusive_sum(uint32_t v) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= (uint32_t)o) v += t;
    }
    return v;
}

// Exclusive scan of a[0..N) (in shared memory) in place; returns the total.
// `wsum` is shared scratch of at least kWarps+1 words.  All threads call it.
template <typename T>
__device__ uint32_t block_exclusive_scan(T* a, uint32_t N, uint32_t* wsum) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t per = (N + kThreads - 1) / kThreads;
    const uint32_t beg = min(N, tid * per), end = min(N, beg + per);
    uint32_t s = 0;
    for (uint32_t i = beg; i < end; ++i) s += a[i];
    uint32_t incl = warp_inclusive_sum(s);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < (uint32_t)kWarps ? wsum[lane] : 0u;
        uint32_t vi = warp_inclusive_sum(v);
        if (lane < (uint32_t)kWarps) wsum[lane] = vi - v;
        if (lane == kWarps - 1) wsum[kWarps] = vi;
    }
    __syncthreads();
    uint32_t run = wsum[warp] + incl - s;
    for (uint32_t i = beg; i < end; ++i) {
        T t = a[i];
        a[i] = (T)run;
        run += t;
    }
    const uint32_t total = wsum[kWarps];
    __syncthreads();
    return total;
}

// D4 draws of the problem-relative positions [P0, P0 + m) into d[0..m)
// (one Philox call per 8 consecutive positions, blocked by thread).
__device__ __forceinline__ void draws_to_smem(uint16_t* d, uint64_t P0, uint32_t m, PhiloxKey key, uint32_t level,
                                              BucketParams bp) {
    if (m == 0) return;
    const uint64_t g0 = P0 >> 3, g1 = (P0 + m - 1) >> 3;
    const uint32_t ng = (uint32_t)(g1 - g0 + 1);
    for (uint32_t t = threadIdx.x; t < ng; t += kThreads) {
        const uint64_t g = g0 + t;
        const uint4 w = bucket_group_words(key, level, g);
        const uint64_t pbase = g << 3;
        if (pbase >= P0 && pbase + 8 <= P0 + m) {
            // full group: 8 draws
            uint32_t b[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) b[j] = bucket_from_lane(lane16(w, j), key, level, pbase + j, bp);
            uint16_t* out = d + (pbase - P0);
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) out[j] = (uint16_t)b[j];
        } else {
            for (uint32_t j = 0; j < 8; ++j) {
                const uint64_t p = pbase + j;
                if (p >= P0 && p < P0 + m) d[p - P0] = (uint16_t)bucket_from_lane(lane16(w, j), key, level, p, bp);
            }
        }
    }
}

}  // namespace shuf
