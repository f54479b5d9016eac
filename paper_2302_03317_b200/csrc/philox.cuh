// Device-side random draws of the deterministic ScatterShuffle definition
// (D1-D5).  Written for sm_100a; shares nothing with the
// CPU oracle (oracle/), which implements the same definition independently.
//
//   D1 Philox4x32-10: 10 rounds; round function
//        (x0,x1,x2,x3) <- (hi(M1*x2)^x1^k0, lo(M1*x2), hi(M0*x0)^x3^k1, lo(M0*x0))
//      with M0 = 0xD2511F53, M1 = 0xCD9E8D57; key bumped by the Weyl
//      constants (0x9E3779B9, 0xBB67AE85) before rounds 2..10.
//   D4 bucket draw at (level l, problem-relative position p):
//      k a power of two <= 256 ("narrow"): 8-bit lane p&15 of
//        Philox(K, (p>>4, l, SC=1)) shifted right by 8 - log2 k;
//      otherwise ("wide"): 16-bit lane p&7 of Philox(K, (p>>3, l, SC=1)),
//        Lemire with threshold 2^16 mod k, retries from
//        Philox(K, (p, l | a<<8, SC_RETRY=3)).w0 & 0xFFFF.
//   D5 FY draw for step i (bound s = i+1) of the leaf starting at q:
//      s <= 2^16: 16-bit lane i&7 of Philox(K, (q, i>>3, FY16=2)), Lemire16,
//        retries from Philox(K, (q, i, FY16_RETRY=4 | a<<8)).w0 & 0xFFFF;
//      s >  2^16: word i&3 of Philox(K, (q, i>>2, FY32=5)), Lemire32,
//        retries from Philox(K, (q, i, FY32_RETRY=6 | a<<8)).w0.
//   Fig. 1: partner = gen_index(rng, i+1), i.e. s = i + 1.
#pragma once
#include <cstdint>

namespace shuf {

struct PhiloxKey {
    uint32_t k0, k1;
};

__device__ __forceinline__ PhiloxKey make_key(uint64_t K) { return {(uint32_t)K, (uint32_t)(K >> 32)}; }

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, PhiloxKey key) {
    uint32_t k0 = key.k0, k1 = key.k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

enum : uint32_t {
    TAG_SC = 1u,
    TAG_FY16 = 2u,
    TAG_SC_RETRY = 3u,
    TAG_FY16_RETRY = 4u,
    TAG_FY32 = 5u,
    TAG_FY32_RETRY = 6u
};

// Bucket-draw parameters for one k.
struct BucketParams {
    uint32_t k;
    uint32_t narrow;  // 1: power of two <= 256 -> 16 draws per call, 8-bit lanes
    uint32_t shift;   // narrow: 8 - log2 k; wide power of two: 16 - log2 k; else 0xFFFFFFFF
    uint32_t t;       // wide, general k: 2^16 mod k
};

__host__ __device__ inline BucketParams make_bucket_params(uint32_t k) {
    BucketParams bp;
    bp.k = k;
    bp.t = 65536u % k;
    uint32_t b = 0;
    while ((1u << b) < k) ++b;
    const bool pow2 = (k & (k - 1)) == 0;
    bp.narrow = (pow2 && k <= 256u) ? 1u : 0u;
    bp.shift = pow2 ? (bp.narrow ? 8u - b : 16u - b) : 0xFFFFFFFFu;
    return bp;
}

__host__ __device__ inline uint32_t draws_per_group(const BucketParams& bp) { return bp.narrow ? 16u : 8u; }

// The 128 bits of group g at level l (both lane widths use this counter).
__device__ __forceinline__ uint4 bucket_group_words(PhiloxKey key, uint32_t level, uint64_t g) {
    return philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), level, TAG_SC), key);
}

// Slow path of D4 (wide, non-power-of-two k): retry stream.
__device__ __forceinline__ uint32_t bucket_retry(PhiloxKey key, uint32_t level, uint64_t p, uint32_t k,
                                                     uint32_t t) {
    for (uint32_t a = 1;; ++a) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)(p >> 32), level | (a << 8), TAG_SC_RETRY), key);
        uint32_t m = (w.x & 0xFFFFu) * k;
        if ((m & 0xFFFFu) >= t) return m >> 16;
    }
}

__device__ __forceinline__ uint32_t word_of(uint4 w, uint32_t i) {
    return (i < 2) ? ((i == 0) ? w.x : w.y) : ((i == 2) ? w.z : w.w);
}

__device__ __forceinline__ uint32_t lane8(uint4 w, uint32_t j) { return (word_of(w, j >> 2) >> ((j & 3u) * 8u)) & 0xFFu; }
__device__ __forceinline__ uint32_t lane16(uint4 w, uint32_t j) {
    return (word_of(w, j >> 1) >> ((j & 1u) * 16u)) & 0xFFFFu;
}

// Bucket of lane j of group g (position p = g*dpg + j).
__device__ __forceinline__ uint32_t bucket_from_group(uint4 w, uint32_t j, PhiloxKey key, uint32_t level, uint64_t p,
                                                      const BucketParams& bp) {
    if (bp.narrow) return lane8(w, j) >> bp.shift;
    const uint32_t v = lane16(w, j);
    if (bp.shift != 0xFFFFFFFFu) return v >> bp.shift;
    const uint32_t m = v * bp.k;
    if ((m & 0xFFFFu) >= bp.t) return m >> 16;
    return bucket_retry(key, level, p, bp.k, bp.t);
}

// D4 for a single position (off the hot loops).
__device__ __forceinline__ uint32_t bucket_draw(PhiloxKey key, uint32_t level, uint64_t p, const BucketParams& bp) {
    const uint32_t sh = bp.narrow ? 4u : 3u;
    const uint4 w = bucket_group_words(key, level, p >> sh);
    return bucket_from_group(w, (uint32_t)(p & ((1u << sh) - 1u)), key, level, p, bp);
}

// ---------------------------------------------------------------- D5 ----
// Partner of step i (bound s = i+1) of the leaf starting at problem-relative
// position q, keyed by (seed, leaf id q, step i).
__device__ __forceinline__ uint4 fy16_group_words(PhiloxKey key, uint64_t q, uint32_t grp) {
    return philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), grp, TAG_FY16), key);
}

__device__ __forceinline__ uint32_t fy16_retry(PhiloxKey key, uint64_t q, uint32_t i) {
    const uint32_t s = i + 1, t = 65536u % s;
    for (uint32_t a = 1;; ++a) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), i, TAG_FY16_RETRY | (a << 8)), key);
        const uint32_t m = (w.x & 0xFFFFu) * s;
        if ((m & 0xFFFFu) >= t) return m >> 16;
    }
}

// Lemire16 on lane v for step i (s = i+1 <= 2^16); the modulo is only
// evaluated when the cheap pre-check (low part < s) cannot rule rejection out.
__device__ __forceinline__ uint32_t fy16_from_lane(uint32_t v, PhiloxKey key, uint64_t q, uint32_t i) {
    const uint32_t s = i + 1;
    const uint32_t m = v * s;
    const uint32_t lo = m & 0xFFFFu;
    if (lo < s && lo < 65536u % s) return fy16_retry(key, q, i);
    return m >> 16;
}

static __device__ __noinline__ uint32_t fy32_draw(PhiloxKey key, uint64_t q, uint32_t i) {
    const uint32_t s = i + 1;
    const uint32_t t = (uint32_t)(0x100000000ull % s);
    uint4 w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), i >> 2, TAG_FY32), key);
    uint64_t M = (uint64_t)word_of(w, i & 3u) * s;
    for (uint32_t a = 1; (uint32_t)M < t; ++a) {
        w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), i, TAG_FY32_RETRY | (a << 8)), key);
        M = (uint64_t)w.x * s;
    }
    return (uint32_t)(M >> 32);
}

// D5 for a single step (off the hot loops).
__device__ __forceinline__ uint32_t fy_draw(PhiloxKey key, uint64_t q, uint32_t i) {
    if (i >= 65536u) return fy32_draw(key, q, i);
    const uint4 w = fy16_group_words(key, q, i >> 3);
    return fy16_from_lane(lane16(w, i & 7u), key, q, i);
}

}  // namespace shuf
