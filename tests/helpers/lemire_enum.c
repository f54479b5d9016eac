/* Test helper: exhaustive enumeration of the oracle's 32-bit Lemire acceptance
 * over ALL 2^32 words w for one bound s.  counts[j] = #{w : accepted with draw j},
 * *rejected = #{w : rejected}.  Calls the oracle's exported function; holds no
 * Lemire arithmetic of its own. */
#include <stdint.h>
typedef int (*accept_fn)(uint32_t, uint32_t, uint32_t *);
void lemire32_enumerate(accept_fn f, uint32_t s, uint64_t *counts, uint64_t *rejected) {
    uint64_t rej = 0;
    uint32_t w = 0;
    do {
        uint32_t out;
        if (f(w, s, &out)) {
            if (out < s) counts[out]++;
            else counts[s]++; /* out of range: recorded in the guard slot */
        } else {
            rej++;
        }
    } while (++w != 0);
    *rejected = rej;
}
void lemire16_enumerate(accept_fn f, uint32_t k_lo, uint32_t k_hi, uint64_t *bad) {
    /* for every k in [k_lo, k_hi]: every bucket gets floor(2^16/k) words and
     * (2^16 mod k) words are rejected; *bad counts the k that violate it */
    static uint32_t cnt[65537];
    uint64_t nbad = 0;
    for (uint32_t k = k_lo; k <= k_hi; k++) {
        for (uint32_t b = 0; b <= k; b++) cnt[b] = 0;
        uint32_t rej = 0;
        for (uint32_t v = 0; v < 65536u; v++) {
            uint32_t out;
            if (f(v, k, &out)) cnt[out < k ? out : k]++;
            else rej++;
        }
        int ok = (rej == 65536u % k) && cnt[k] == 0;
        for (uint32_t b = 0; b < k && ok; b++) ok = (cnt[b] == 65536u / k);
        if (!ok) nbad++;
    }
    *bad = nbad;
}
