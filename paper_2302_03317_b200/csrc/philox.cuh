// Device-side random draws of the deterministic ScatterShuffle definition
// (D1-D5).  Written for sm_100a; shares nothing with the
// CPU oracle (oracle/), which implements the same definition independently.
//
//   D1 Philox4x32-10: 10 rounds; round function
//        (x0,x1,x2,x3) <- (hi(M1*x2)^x1^k0, lo(M1*x2), hi(M0*x0)^x3^k1, lo(M0*x0))
//      with M0 = 0xD2511F53, M1 = 0xCD9E8D57; key bumped by the Weyl
//      constants (0x9E3779B9, 0xBB67AE85) before rounds 2..10.
//   D4 bucket draw at (level l, problem-relative position p): 16-bit lane
//      p&7 of Philox(K, (p>>3, l, SC=1)), Lemire with threshold 2^16 mod k;
//      retries from Philox(K, (p, l | a<<8, SC_RETRY=3)).w0.
//   D5 FY draw at (position P, bound s): 32-bit word P&3 of
//      Philox(K, (P>>2, 0, FY=2)), Lemire with threshold 2^32 mod s;
//      retries from Philox(K, (P, a, FY_RETRY=4)).w0.
//   Paper: Lemire bounded integers P:99-100; FY partner draw Fig. 1 P:109.
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

enum : uint32_t { TAG_SC = 1u, TAG_FY = 2u, TAG_SC_RETRY = 3u, TAG_FY_RETRY = 4u };

// Bucket-draw parameters for one k (power of two or general).
struct BucketParams {
    uint32_t k;
    uint32_t t;      // 2^16 mod k (0 for powers of two: no rejection)
    uint32_t shift;  // 16 - log2(k) when k is a power of two, else 0xFFFFFFFF
};

__host__ __device__ inline BucketParams make_bucket_params(uint32_t k) {
    BucketParams bp;
    bp.k = k;
    bp.t = 65536u % k;
    bp.shift = 0xFFFFFFFFu;
    if ((k & (k - 1)) == 0) {
        uint32_t b = 0;
        while ((1u << b) < k) ++b;
        bp.shift = 16u - b;
    }
    return bp;
}

// The 8 primary 16-bit lanes of group g at level l.
__device__ __forceinline__ uint4 bucket_group_words(PhiloxKey key, uint32_t level, uint64_t g) {
    return philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), level, TAG_SC), key);
}

// Slow path of D4: retry stream for a rejected position.
static __device__ __noinline__ uint32_t bucket_retry(PhiloxKey key, uint32_t level, uint64_t p, BucketParams bp) {
    for (uint32_t a = 1;; ++a) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)(p >> 32), level | (a << 8), TAG_SC_RETRY), key);
        uint32_t m = (w.x & 0xFFFFu) * bp.k;
        if ((m & 0xFFFFu) >= bp.t) return m >> 16;
    }
}

// Map one primary 16-bit lane v (of position p) to a bucket.
__device__ __forceinline__ uint32_t bucket_from_lane(uint32_t v, PhiloxKey key, uint32_t level, uint64_t p,
                                                     BucketParams bp) {
    if (bp.shift != 0xFFFFFFFFu) return v >> bp.shift;
    uint32_t m = v * bp.k;
    if ((m & 0xFFFFu) >= bp.t) return m >> 16;
    return bucket_retry(key, level, p, bp);
}

__device__ __forceinline__ uint32_t lane16(uint4 w, uint32_t j) {
    uint32_t word = (j < 4) ? ((j < 2) ? w.x : w.y) : ((j < 6) ? w.z : w.w);
    return (word >> ((j & 1u) * 16u)) & 0xFFFFu;
}

// D4 for a single position (used off the hot loops).
__device__ __forceinline__ uint32_t bucket_draw(PhiloxKey key, uint32_t level, uint64_t p, BucketParams bp) {
    uint4 w = bucket_group_words(key, level, p >> 3);
    return bucket_from_lane(lane16(w, (uint32_t)(p & 7u)), key, level, p, bp);
}

// D5 slow path.
static __device__ __noinline__ uint32_t fy_retry(PhiloxKey key, uint64_t P, uint32_t s) {
    const uint32_t t = (uint32_t)(0x100000000ull % s);
    for (uint32_t a = 1;; ++a) {
        uint4 w = philox4x32_10(make_uint4((uint32_t)P, (uint32_t)(P >> 32), a, TAG_FY_RETRY), key);
        uint64_t M = (uint64_t)w.x * s;
        if ((uint32_t)M >= t) return (uint32_t)(M >> 32);
    }
}

// Lemire on one primary word w of position P; the 2^32 mod s threshold is
// only evaluated when the cheap pre-check lo < s fails to rule rejection out.
__device__ __forceinline__ uint32_t fy_from_word(uint32_t w, PhiloxKey key, uint64_t P, uint32_t s) {
    uint64_t M = (uint64_t)w * s;
    uint32_t lo = (uint32_t)M;
    if (lo < s) {
        const uint32_t t = (uint32_t)(0x100000000ull % s);
        if (lo < t) return fy_retry(key, P, s);
    }
    return (uint32_t)(M >> 32);
}

__device__ __forceinline__ uint4 fy_group_words(PhiloxKey key, uint64_t g) {
    return philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), 0u, TAG_FY), key);
}

__device__ __forceinline__ uint32_t word32(uint4 w, uint32_t j) {
    return (j < 2) ? ((j == 0) ? w.x : w.y) : ((j == 2) ? w.z : w.w);
}

__device__ __forceinline__ uint32_t fy_draw(PhiloxKey key, uint64_t P, uint32_t s) {
    uint4 w = fy_group_words(key, P >> 2);
    return fy_from_word(word32(w, (uint32_t)(P & 3u)), key, P, s);
}

}  // namespace shuf
