// Hidden-constant simulation (section 7,
// P:773-788): Lemma 2 bounds the items RoughScatter leaves staged
// by R <= sqrt(2 n k log k), Corollary 5 TwoSweep's swaps
// M = sum_i |D_i| (Lemma 4) by O(k sqrt(n k log k)).  One run per
// key K(seed, r) (D2), D9:
//
//   RoughScatter: bucket capacities c_i = floor((i+1)n/k) -
//   floor(i n/k) ("equal sizes n/k up to rounding"); iteration t
//   draws j_t = bucket(0, t) (D4) and places an item into B_j; it stops when
//   B_j is full.  T = items placed, R = n - T.
//   Completion: the R staged items draw j_t for
//   t = T .. n-1; n^f_i = #{t < n : j_t = i}; d_i = n^f_i - c_i,
//   D_i = d_0 + .. + d_i, M = sum_i |D_i|.
//
// One CTA per run.  The draw sequence is walked in tiles of 256 Philox groups
// with unordered shared counters; the tile in which some bucket reaches its
// capacity is undone and replayed in position order by one warp (exact
// in-round ranks from __match_any_sync, no reliance on atomic ordering) to find
// the first full bucket; the remaining tiles only count.  All integer: T and M
// equal the oracle's (oracle_sim_rough_scatter) bit for bit.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "shuf_internal.cuh"

namespace shuf {

constexpr uint32_t kSimThreads = 256;

// c_j = floor((j+1) n / k) - floor(j n / k) with n = q k + r: j q + floor(j r / k) terms.
__device__ __forceinline__ uint64_t sim_cap(uint32_t j, uint64_t q, uint32_t r, uint32_t k) {
    const uint64_t a = (uint64_t)j * q + ((uint64_t)j * r) / k;
    const uint64_t b = (uint64_t)(j + 1) * q + ((uint64_t)(j + 1) * r) / k;
    return b - a;
}

// Counter j: u32 word j, or (P16, k > 32768) the u16 half j & 1 of word j >> 1.
template <bool P16>
__device__ __forceinline__ uint32_t sim_add(uint32_t* cnt, uint32_t j, uint32_t v) {
    if (!P16) return atomicAdd(&cnt[j], v);
    const uint32_t shb = (j & 1u) << 4;
    return (atomicAdd(&cnt[j >> 1], v << shb) >> shb) & 0xFFFFu;
}
template <bool P16>
__device__ __forceinline__ uint32_t sim_get(const uint32_t* cnt, uint32_t j) {
    if (!P16) return cnt[j];
    return (cnt[j >> 1] >> ((j & 1u) << 4)) & 0xFFFFu;
}

template <bool NARROW, bool P16>
__global__ void __launch_bounds__(kSimThreads) k_sim_rough(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs,
                                                           uint64_t* __restrict__ outT, uint64_t* __restrict__ outM) {
    extern __shared__ uint32_t cnt[];  // k counters: u32, or packed u16 pairs (P16)
    __shared__ unsigned long long s_T;
    __shared__ unsigned long long wsum[kSimThreads / 32 + 1];
    constexpr uint32_t dpg = NARROW ? 16u : 8u, sh = NARROW ? 4u : 3u;
    constexpr uint64_t TT = (uint64_t)kSimThreads * dpg;  // positions per tile
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const BucketParams bp = make_bucket_params(k);
    const uint64_t q = n / k;
    const uint32_t r = (uint32_t)(n % k);
    for (uint32_t run = blockIdx.x; run < runs; run += gridDim.x) {
        const PhiloxKey key = make_key(seed + (uint64_t)run * 0x9E3779B97F4A7C15ull);  // K(seed, run) (D2)
        for (uint32_t i = tid; i < (P16 ? (k + 1) / 2 : k); i += kSimThreads) cnt[i] = 0;
        if (tid == 0) s_T = n;
        __syncthreads();
        bool found = false;
        for (uint64_t t0 = 0; t0 < n; t0 += TT) {
            // ---- unordered counts of the tile; a thread that fills a bucket flags the tile
            const uint64_t g = (t0 >> sh) + tid;
            const uint4 w = bucket_group_words(key, 0u, g);
            uint32_t bj[dpg];
            bool hit = false;
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j) {
                const uint64_t p = (g << sh) + j;
                bj[j] = p < n ? bucket_from_group(w, j, key, 0u, p, bp) : 0xFFFFFFFFu;
                if (p < n) {
                    const uint32_t old = sim_add<P16>(cnt, bj[j], 1u);
                    if (!found && old + 1u == sim_cap(bj[j], q, r, k)) hit = true;
                }
            }
            if (found) continue;  // uniform: set after a barrier
            if (!__syncthreads_or(hit)) continue;
            // ---- a bucket filled inside this tile: undo it and replay it in position order
#pragma unroll
            for (uint32_t j = 0; j < dpg; ++j)
                if (bj[j] != 0xFFFFFFFFu) sim_add<P16>(cnt, bj[j], 0xFFFFFFFFu);  // -1 (mod 2^16 per half)
            __syncthreads();
            if (warp == 0) {
                bool done = false;
                for (uint64_t pb = t0; pb < min(n, t0 + TT); pb += 32) {
                    const uint64_t p = pb + lane;
                    const bool valid = p < n;
                    const uint32_t b = valid ? bucket_draw(key, 0u, p, bp) : 0xFFFFFFFFu;
                    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, b);
                    const uint32_t below = __popc(peers & lanemask_lt());
                    const uint32_t old = valid ? sim_get<P16>(cnt, b) : 0u;
                    __syncwarp();
                    if (valid && below == 0) sim_add<P16>(cnt, b, (uint32_t)__popc(peers));
                    __syncwarp();
                    const bool fills = valid && !done && old + below + 1u == sim_cap(b, q, r, k);
                    const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fills);
                    if (fm) {
                        if (lane == __ffs(fm) - 1) s_T = p + 1;
                        done = true;
                    }
                }
                if (!done && lane == 0) s_T = ~0ull;  // internal: the flagged tile filled nothing
            }
            found = true;
            __syncthreads();
        }
        __syncthreads();  // every count in (tiles after the fill run without barriers)
        // ---- M = sum_i |D_i|: each thread a contiguous range of buckets
        const uint32_t per = (k + kSimThreads - 1) / kSimThreads;
        const uint32_t x0 = min(k, tid * per), x1 = min(k, x0 + per);
        long long mine = 0;
        for (uint32_t x = x0; x < x1; ++x) mine += (long long)sim_get<P16>(cnt, x) - (long long)sim_cap(x, q, r, k);
        long long incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        if (lane == 31) wsum[warp] = (unsigned long long)incl;
        __syncthreads();
        if (tid == 0) {
            long long run_ = 0;
            for (uint32_t w8 = 0; w8 < kSimThreads / 32; ++w8) {
                const long long c = (long long)wsum[w8];
                wsum[w8] = (unsigned long long)run_;
                run_ += c;
            }
        }
        __syncthreads();
        long long D = (long long)wsum[warp] + incl - mine;
        unsigned long long m = 0;
        for (uint32_t x = x0; x < x1; ++x) {
            D += (long long)sim_get<P16>(cnt, x) - (long long)sim_cap(x, q, r, k);
            m += (unsigned long long)(D < 0 ? -D : D);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
        __syncthreads();
        if (lane == 0) wsum[warp] = m;
        __syncthreads();
        if (tid == 0) {
            unsigned long long tot = 0;
            for (uint32_t w8 = 0; w8 < kSimThreads / 32; ++w8) tot += wsum[w8];
            outT[run] = s_T;
            outM[run] = tot;
        }
        __syncthreads();
    }
}

// k <= 2^15: u32 counters; up to 2^16: packed u16 (every count < 2^16 needs
// n / k well below 2^16, checked by the caller).
cudaError_t launch_sim_rough(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t* T, uint64_t* M, int grid,
                             cudaStream_t s) {
    const bool narrow = (k & (k - 1)) == 0 && k <= 256, p16 = k > 32768;
    const uint32_t smem = p16 ? (k + 1) / 2 * 4u : k * 4u;
    void* fn = narrow ? (void*)k_sim_rough<true, false>
                      : (p16 ? (void*)k_sim_rough<false, true> : (void*)k_sim_rough<false, false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    void* args[] = {(void*)&n, (void*)&k, (void*)&seed, (void*)&runs, (void*)&T, (void*)&M};
    const int g = (int)min((uint64_t)grid, (uint64_t)runs);
    return cudaLaunchKernel(fn, dim3(g), dim3(kSimThreads), args, smem, s);
}

}  // namespace shuf
