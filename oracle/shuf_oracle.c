/*
 * oracle/shuf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded C implementation of the deterministic
 * ScatterShuffle definition D1-D7 in DESIGN.md section 2.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2302_03317_b200/csrc/).
 *
 * Citations: "P:n" = line n of the paper text (arXiv 2302.03317, PAPER.md);
 * "S:n" = line n of SPEC.md.
 *
 *   D1 Philox4x32-10 ........ (the counter-based generator named by the task's
 *                              north star; the paper's own RNG is Pcg64Mcg)
 *   D4 bucket draw .......... Lemire bounded integer, "sampling an
 *                              integer from [0,s) with s=2^k ... shifting and
 *                              masking"; rejection for general s (Lemire 2019);
 *                              8-bit lanes (16 draws per Philox call) for
 *                              power-of-two k <= 256, 16-bit lanes otherwise
 *   D5 Fisher-Yates draw .... Fig. 1: gen_index(rng, i+1),
 *                              "partner from [0..i]", keyed by (leaf, step)
 *   D6 recursion ............ ScatterShuffle, IpSc "groups X by A
 *                              ... with some permutation pi that sorts A"
 *                               with pi chosen stable; recursion and
 *                              FY base case per Fig. 2
 *   D7 segmented ............ independent problems, key K(seed, s)
 *
 * Parity pins (tests/test_oracle_*.py): Philox against cuRAND's host-compiled
 * Philox4x32-10; Lemire by exhaustive enumeration; the stable scatter against
 * numpy.argsort(kind="stable"); FY against the S:116 stub trace; uniformity by
 * the n! census; bucket sizes against the multinomial moments.
 * The counter layout itself (which counter feeds which draw) is a convention
 * of DESIGN.md and is "parity unpinned beyond self-consistency".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "shuf_oracle.h"

/* ---------------------------------------------------------------- D1 ---- */
/* Philox4x32-10 (Salmon et al., SC'11): ten rounds; before every round after
 * the first the key is bumped by the Weyl constants.                         */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
        uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0;
        uint32_t h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
        uint32_t y0 = h1 ^ x1 ^ k0;
        uint32_t y1 = l1;
        uint32_t y2 = h0 ^ x3 ^ k1;
        uint32_t y3 = l0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* ---------------------------------------------------------------- D2 ---- */
uint64_t oracle_problem_key(uint64_t seed, uint64_t s)
{
    return seed + s * 0x9E3779B97F4A7C15ull; /* mod 2^64 */
}

static void key_words(uint64_t K, uint32_t key[2])
{
    key[0] = (uint32_t)K;
    key[1] = (uint32_t)(K >> 32);
}

/* ------------------------------------------------------------- Lemire ---- */
/* Lemire's multiply-shift with rejection on a w-bit word v, bound s.
 * Accept iff the low w bits of v*s are >= t = 2^w mod s; the draw is then the
 * high part of v*s.  Returns 1 and writes *out on acceptance, 0 on rejection. */
int oracle_lemire16_accept(uint32_t v, uint32_t s, uint32_t *out)
{
    uint32_t t = 65536u % s;
    uint32_t m = v * s; /* v < 2^16, s <= 2^16: fits in 32 bits */
    if ((m & 0xFFFFu) >= t) {
        *out = m >> 16;
        return 1;
    }
    return 0;
}

int oracle_lemire32_accept(uint32_t w, uint32_t s, uint32_t *out)
{
    uint32_t t = (uint32_t)((4294967296ull) % s);
    uint64_t M = (uint64_t)w * s;
    if ((uint32_t)M >= t) {
        *out = (uint32_t)(M >> 32);
        return 1;
    }
    return 0;
}

/* ---------------------------------------------------------------- D4 ---- */
#define TAG_SC 1u
#define TAG_FY16 2u
#define TAG_SC_RETRY 3u
#define TAG_FY16_RETRY 4u
#define TAG_FY32 5u
#define TAG_FY32_RETRY 6u

/* log2(k) if k is a power of two <= 256 (8-bit lanes), else -1 (16-bit lanes) */
static int narrow_shift(uint32_t k)
{
    if (k > 256u || (k & (k - 1u)) != 0)
        return -1;
    int b = 0;
    while ((1u << b) < k)
        b++;
    return b;
}

/* D4: bucket of problem-relative position p at level `level`.
 * Power-of-two k <= 256: 16 draws per Philox call, 8-bit lane p&15 of
 *   Philox(K, (p>>4, level, SC)), bucket = lane >> (8 - log2 k) (shift only).
 * Otherwise: 8 draws per call, 16-bit lane p&7 of Philox(K, (p>>3, level, SC)),
 *   Lemire with rejection; retries from Philox(K, (p, level|a<<8, SC_RETRY)). */
uint32_t oracle_bucket_draw(uint64_t K, uint32_t level, uint64_t p, uint32_t k, uint64_t *rejections)
{
    uint32_t key[2], ctr[4], w[4], out;
    key_words(K, key);
    int b = narrow_shift(k);
    if (b >= 0) {
        uint64_t g = p >> 4;
        ctr[0] = (uint32_t)g;
        ctr[1] = (uint32_t)(g >> 32);
        ctr[2] = level;
        ctr[3] = TAG_SC;
        oracle_philox4x32_10(ctr, key, w);
        uint32_t j = (uint32_t)(p & 15u);
        uint32_t v = (w[j >> 2] >> (8u * (j & 3u))) & 0xFFu;
        return v >> (8 - b);
    }
    uint64_t g = p >> 3;
    ctr[0] = (uint32_t)g;
    ctr[1] = (uint32_t)(g >> 32);
    ctr[2] = level;
    ctr[3] = TAG_SC;
    oracle_philox4x32_10(ctr, key, w);
    uint32_t j = (uint32_t)(p & 7u);
    uint32_t v = (w[j >> 1] >> (16u * (j & 1u))) & 0xFFFFu;
    if (oracle_lemire16_accept(v, k, &out))
        return out;
    for (uint32_t a = 1;; a++) {
        if (rejections)
            (*rejections)++;
        ctr[0] = (uint32_t)p;
        ctr[1] = (uint32_t)(p >> 32);
        ctr[2] = level | (a << 8);
        ctr[3] = TAG_SC_RETRY;
        oracle_philox4x32_10(ctr, key, w);
        v = w[0] & 0xFFFFu;
        if (oracle_lemire16_accept(v, k, &out))
            return out;
    }
}

/* ---------------------------------------------------------------- D5 ---- */
/* D5: Fisher-Yates partner for step i (bound s = i+1) of the leaf whose first
 * element is problem-relative position q -- keyed by (seed, leaf id, step)
 * (Fig. 1: gen_index(rng, i+1), "partner from [0..i]").
 * s <= 2^16: 16-bit lane i&7 of Philox(K, (q, i>>3, FY16)), Lemire16.
 * s >  2^16: 32-bit word i&3 of Philox(K, (q, i>>2, FY32)), Lemire32.
 * Retry a >= 1: Philox(K, (q, i, TAG_RETRY | a<<8)).w0 (low 16 bits for
 * 16-bit lanes), TAG_RETRY = FY16_RETRY or FY32_RETRY. */
uint32_t oracle_fy_draw(uint64_t K, uint64_t q, uint32_t i, uint64_t *rejections)
{
    uint32_t key[2], ctr[4], w[4], out;
    const uint32_t s = i + 1u;
    key_words(K, key);
    ctr[0] = (uint32_t)q;
    ctr[1] = (uint32_t)(q >> 32);
    if (s <= 65536u) {
        ctr[2] = i >> 3;
        ctr[3] = TAG_FY16;
        oracle_philox4x32_10(ctr, key, w);
        uint32_t j = i & 7u;
        uint32_t v = (w[j >> 1] >> (16u * (j & 1u))) & 0xFFFFu;
        if (oracle_lemire16_accept(v, s, &out))
            return out;
        for (uint32_t a = 1;; a++) {
            if (rejections)
                (*rejections)++;
            ctr[2] = i;
            ctr[3] = TAG_FY16_RETRY | (a << 8);
            oracle_philox4x32_10(ctr, key, w);
            if (oracle_lemire16_accept(w[0] & 0xFFFFu, s, &out))
                return out;
        }
    }
    ctr[2] = i >> 2;
    ctr[3] = TAG_FY32;
    oracle_philox4x32_10(ctr, key, w);
    if (oracle_lemire32_accept(w[i & 3u], s, &out))
        return out;
    for (uint32_t a = 1;; a++) {
        if (rejections)
            (*rejections)++;
        ctr[2] = i;
        ctr[3] = TAG_FY32_RETRY | (a << 8);
        oracle_philox4x32_10(ctr, key, w);
        if (oracle_lemire32_accept(w[0], s, &out))
            return out;
    }
}

/* batch dumps (raw-draw parity with the device) */
void oracle_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k, uint32_t *out)
{
    for (uint64_t i = 0; i < count; i++)
        out[i] = oracle_bucket_draw(K, level, p0 + i, k, NULL);
}

void oracle_fy_draws(uint64_t K, const uint64_t *q, const uint32_t *i, uint64_t count, uint32_t *out)
{
    for (uint64_t x = 0; x < count; x++)
        out[x] = oracle_fy_draw(K, q[x], i[x], NULL);
}

/* --------------------------------------------------------- elements ---- */
static void elem_copy(unsigned char *dst, const unsigned char *src, uint32_t eb)
{
    switch (eb) {
    case 4: memcpy(dst, src, 4); break;
    case 8: memcpy(dst, src, 8); break;
    case 16: memcpy(dst, src, 16); break;
    default: memcpy(dst, src, eb); break;
    }
}

static void elem_swap(unsigned char *a, unsigned char *b, uint32_t eb)
{
    unsigned char t[64];
    unsigned char *tmp = eb <= sizeof t ? t : (unsigned char *)malloc(eb);
    elem_copy(tmp, a, eb);
    elem_copy(a, b, eb);
    elem_copy(b, tmp, eb);
    if (tmp != t)
        free(tmp);
}

/* FY with explicitly given partners j[i] (i = m-1 .. 1; j[0] unused):
 * Fig. 1 with the generator replaced by a stub, for the S:116 trace test.   */
void oracle_fy_with_draws(void *data, uint64_t m, uint32_t eb, const uint32_t *j)
{
    unsigned char *A = (unsigned char *)data;
    for (uint64_t i = m; i-- > 1;)
        elem_swap(A + i * eb, A + (uint64_t)j[i] * eb, eb);
}

/* ---------------------------------------------------------------- D6 ---- */
typedef struct {
    unsigned char *A;   /* the problem's array (positions are relative to A) */
    unsigned char *T;   /* temporary of the same size                        */
    uint16_t *ids;      /* bucket ids of the current segment                 */
    uint32_t eb, k, L;
    uint64_t K;
    uint32_t max_levels;
    int run_leaves;
    oracle_stats *st;
} ctx_t;

/* Fig. 1: for i = m-1 down to 1: swap(A[q+i], A[q + gen_index(i+1)]),
 * the draw keyed by (leaf id q, step i) (D5).                                */
static void fy_leaf(ctx_t *c, uint64_t q, uint64_t m)
{
    uint64_t *rej = c->st ? &c->st->fy_rejections : NULL;
    for (uint64_t i = m; i-- > 1;) {
        uint32_t j = oracle_fy_draw(c->K, q, (uint32_t)i, rej);
        elem_swap(c->A + (q + i) * c->eb, c->A + (q + j) * c->eb, c->eb);
    }
}

/* Fig. 2 with the scatter replaced by the stable counting
 * scatter of D6.  Segment [a, a+m) at level `level`.                         */
static int shuffle_rec(ctx_t *c, uint64_t a, uint64_t m, uint32_t level)
{
    if (m <= c->L) { /* base case: FY */
        if (c->run_leaves) {
            fy_leaf(c, a, m);
            if (c->st)
                c->st->leaves++;
        }
        return 0;
    }
    if (level >= c->max_levels)
        return 0; /* level-limited debug mode: leave the segment as it is */
    if (level > 255)
        return ORACLE_ERR_DEPTH;
    if (c->st) {
        c->st->scatter_elems[level] += m;
        if (level + 1 > c->st->levels)
            c->st->levels = level + 1;
    }
    uint32_t k = c->k, eb = c->eb;
    uint64_t *cnt = (uint64_t *)calloc(k, sizeof(uint64_t));
    uint64_t *o = (uint64_t *)malloc(k * sizeof(uint64_t));
    if (!cnt || !o) {
        free(cnt);
        free(o);
        return ORACLE_ERR_NOMEM;
    }
    uint64_t *rej = c->st ? &c->st->bucket_rejections : NULL;
    /* A_i: i.i.d. uniform bucket per element */
    for (uint64_t i = 0; i < m; i++) {
        uint32_t b = oracle_bucket_draw(c->K, level, a + i, k, rej);
        c->ids[a + i] = (uint16_t)b;
        cnt[b]++;
    }
    /* o_b = a + sum_{b'<b} c_b' */
    uint64_t acc = a;
    for (uint32_t b = 0; b < k; b++) {
        o[b] = acc;
        acc += cnt[b];
    }
    /* stable: ascending i, OUT[o_b++] = IN[i] */
    for (uint64_t i = 0; i < m; i++) {
        uint32_t b = c->ids[a + i];
        elem_copy(c->T + o[b] * eb, c->A + (a + i) * eb, eb);
        o[b]++;
    }
    memcpy(c->A + a * eb, c->T + a * eb, m * eb);
    /* recurse on the buckets */
    int rc = 0;
    uint64_t start = a;
    for (uint32_t b = 0; b < k && rc == 0; b++) {
        rc = shuffle_rec(c, start, cnt[b], level + 1);
        start += cnt[b];
    }
    free(cnt);
    free(o);
    return rc;
}

static int check_args(uint32_t eb, uint32_t k, uint32_t L)
{
    if (eb == 0 || k < 2 || k > 65536u || L < 1)
        return ORACLE_ERR_INVALID_ARG;
    return 0;
}

int oracle_shuffle(void *data, uint64_t n, uint32_t eb, uint32_t k, uint32_t L, uint64_t seed,
                   uint32_t max_levels, int run_leaves, oracle_stats *st)
{
    int rc = check_args(eb, k, L);
    if (rc)
        return rc;
    if (st)
        memset(st, 0, sizeof *st);
    if (n == 0)
        return 0;
    ctx_t c;
    c.A = (unsigned char *)data;
    c.T = (unsigned char *)malloc(n * eb);
    c.ids = (uint16_t *)malloc(n * sizeof(uint16_t));
    if (!c.T || !c.ids) {
        free(c.T);
        free(c.ids);
        return ORACLE_ERR_NOMEM;
    }
    c.eb = eb; c.k = k; c.L = L;
    c.K = oracle_problem_key(seed, 0);
    c.max_levels = max_levels;
    c.run_leaves = run_leaves;
    c.st = st;
    rc = shuffle_rec(&c, 0, n, 0);
    free(c.T);
    free(c.ids);
    return rc;
}

/* ---------------------------------------------------------------- D7 ---- */
int oracle_segmented(void *data, const uint64_t *offsets, uint64_t num_segments, uint32_t eb, uint32_t k,
                     uint32_t L, uint64_t seed, uint32_t max_levels, int run_leaves, oracle_stats *st)
{
    int rc = check_args(eb, k, L);
    if (rc)
        return rc;
    if (st)
        memset(st, 0, sizeof *st);
    if (offsets[0] != 0)
        return ORACLE_ERR_INVALID_ARG;
    uint64_t maxlen = 0;
    for (uint64_t s = 0; s < num_segments; s++) {
        if (offsets[s + 1] < offsets[s])
            return ORACLE_ERR_INVALID_ARG;
        uint64_t len = offsets[s + 1] - offsets[s];
        if (len > maxlen)
            maxlen = len;
    }
    if (maxlen == 0)
        return 0;
    ctx_t c;
    c.T = (unsigned char *)malloc(maxlen * eb);
    c.ids = (uint16_t *)malloc(maxlen * sizeof(uint16_t));
    if (!c.T || !c.ids) {
        free(c.T);
        free(c.ids);
        return ORACLE_ERR_NOMEM;
    }
    c.eb = eb; c.k = k; c.L = L;
    c.max_levels = max_levels;
    c.run_leaves = run_leaves;
    c.st = st;
    for (uint64_t s = 0; s < num_segments && rc == 0; s++) {
        c.A = (unsigned char *)data + offsets[s] * eb; /* segment-relative positions */
        c.K = oracle_problem_key(seed, s);
        rc = shuffle_rec(&c, 0, offsets[s + 1] - offsets[s], 0);
    }
    free(c.T);
    free(c.ids);
    return rc;
}
