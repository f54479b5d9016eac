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
/* The primary bucket draws of 8 or 16 consecutive positions share one Philox
 * block; remembering the last block (same key and counter => same output)
 * only saves recomputation -- results are those of oracle_philox4x32_10.  */
static void philox_memo(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    static _Thread_local uint32_t mc[4], mk[2], mo[4];
    static _Thread_local int have = 0;
    if (!(have && mc[0] == ctr[0] && mc[1] == ctr[1] && mc[2] == ctr[2] && mc[3] == ctr[3] && mk[0] == key[0] &&
          mk[1] == key[1])) {
        oracle_philox4x32_10(ctr, key, mo);
        memcpy(mc, ctr, sizeof mc);
        memcpy(mk, key, sizeof mk);
        have = 1;
    }
    memcpy(out, mo, sizeof mo);
}

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
        philox_memo(ctr, key, w);
        uint32_t j = (uint32_t)(p & 15u);
        uint32_t v = (w[j >> 2] >> (8u * (j & 3u))) & 0xFFu;
        return v >> (8 - b);
    }
    uint64_t g = p >> 3;
    ctr[0] = (uint32_t)g;
    ctr[1] = (uint32_t)(g >> 32);
    ctr[2] = level;
    ctr[3] = TAG_SC;
    philox_memo(ctr, key, w);
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

/* ------------------------------------------------- D6 point queries ---- */
/* pi(j) for selected output positions j of the single shuffle D6 (key
 * K = seed), without materialising the n-element array: the recursion of D6
 * is walked only into the segments that contain a queried position.  Used to
 * check the GPU output at BASELINE.json's full sizes on sampled positions.
 *
 * In segment [a, a+m) at level l (m > L): c_b and o_b exactly as D6; the
 * output position j lies in child b with o_b <= j < o_b + c_b; after the
 * child has resolved j to a position x of the child's INPUT range (= this
 * level's output range), the element there is the (x - o_b)-th element, in
 * ascending i, of bucket b of this segment's input (stability):
 * one pass over i finds it.  A leaf (m <= L) runs Fig. 1 on the index array
 * 0..m-1 with the D5 draws of leaf id a, and x = a + idx[j - a].            */
typedef struct {
    uint64_t j;     /* queried output position                              */
    uint64_t x;     /* resolved position in the current segment's input     */
    uint32_t b;     /* child bucket at the current level                    */
    uint32_t pad;
    uint64_t r;     /* rank of x within child b                             */
} oq_t;

typedef struct {
    uint64_t K;
    uint32_t k, L;
    /* one-group memo of the last Philox call, so a pass over a range costs
     * one generator call per group like the definition's lane layout       */
    uint32_t level;
    uint64_t g;
    int have;
} oq_ctx;

static uint32_t oq_bucket(oq_ctx *c, uint32_t level, uint64_t p)
{
    /* plain D4 (oracle_bucket_draw), evaluated position by position */
    (void)c;
    return oracle_bucket_draw(c->K, level, p, c->k, NULL);
}

static int oq_cmp_br(const void *x, const void *y)
{
    const oq_t *a = *(const oq_t *const *)x, *b = *(const oq_t *const *)y;
    if (a->b != b->b)
        return a->b < b->b ? -1 : 1;
    if (a->r != b->r)
        return a->r < b->r ? -1 : 1;
    return 0;
}

/* resolve every query of q[0..nq) (all inside [a, a+m)) to x = input position */
static int oq_rec(oq_ctx *c, uint64_t a, uint64_t m, uint32_t level, oq_t **q, uint64_t nq)
{
    if (nq == 0)
        return 0;
    if (m <= c->L) { /* leaf: Fig. 1 on indices */
        uint32_t *idx = (uint32_t *)malloc((m ? m : 1) * sizeof(uint32_t));
        if (!idx)
            return ORACLE_ERR_NOMEM;
        for (uint64_t t = 0; t < m; t++)
            idx[t] = (uint32_t)t;
        for (uint64_t i = m; i-- > 1;) {
            uint32_t jj = oracle_fy_draw(c->K, a, (uint32_t)i, NULL);
            uint32_t tmp = idx[i];
            idx[i] = idx[jj];
            idx[jj] = tmp;
        }
        for (uint64_t s = 0; s < nq; s++)
            q[s]->x = a + idx[q[s]->j - a];
        free(idx);
        return 0;
    }
    if (level > 255)
        return ORACLE_ERR_DEPTH;
    uint32_t k = c->k;
    uint64_t *cnt = (uint64_t *)calloc(k, sizeof(uint64_t));
    uint64_t *o = (uint64_t *)malloc(k * sizeof(uint64_t));
    oq_t **tmpq = (oq_t **)malloc(nq * sizeof(oq_t *));
    uint64_t *ptr = (uint64_t *)malloc((k + 1) * sizeof(uint64_t));
    uint32_t *lb = (uint32_t *)malloc(nq * sizeof(uint32_t)); /* this level's child of each query */
    if (!cnt || !o || !tmpq || !ptr || !lb) {
        free(cnt); free(o); free(tmpq); free(ptr); free(lb);
        return ORACLE_ERR_NOMEM;
    }
    for (uint64_t i = 0; i < m; i++)
        cnt[oq_bucket(c, level, a + i)]++;
    uint64_t acc = a;
    for (uint32_t b = 0; b < k; b++) {
        o[b] = acc;
        acc += cnt[b];
    }
    /* child of every query: largest b with o_b <= j and c_b > 0 */
    for (uint64_t s = 0; s < nq; s++) {
        uint32_t b = 0;
        for (uint32_t bb = 0; bb < k; bb++)
            if (cnt[bb] > 0 && o[bb] <= q[s]->j)
                b = bb;
        lb[s] = b;
    }
    /* recurse child by child (queries grouped by child) */
    int rc = 0;
    for (uint32_t b = 0; b < k && rc == 0; b++) {
        uint64_t nb = 0;
        for (uint64_t s = 0; s < nq; s++)
            if (lb[s] == b)
                tmpq[nb++] = q[s];
        if (nb)
            rc = oq_rec(c, o[b], cnt[b], level + 1, tmpq, nb);
    }
    if (rc == 0) {
        /* x is now a position of this level's output range, in child b */
        for (uint64_t s = 0; s < nq; s++) {
            q[s]->b = lb[s];
            q[s]->r = q[s]->x - o[lb[s]];
            tmpq[s] = q[s];
        }
        qsort(tmpq, nq, sizeof(oq_t *), oq_cmp_br);
        /* ptr[b] = first query of bucket b in the sorted list */
        uint64_t s = 0;
        for (uint32_t b = 0; b <= k; b++) {
            while (s < nq && tmpq[s]->b < b)
                s++;
            ptr[b] = s;
        }
        uint64_t *seen = cnt; /* reuse: occurrences of bucket b so far */
        memset(seen, 0, k * sizeof(uint64_t));
        for (uint64_t i = 0; i < m; i++) {
            uint32_t b = oq_bucket(c, level, a + i);
            while (ptr[b] < nq && tmpq[ptr[b]]->b == b && tmpq[ptr[b]]->r == seen[b]) {
                tmpq[ptr[b]]->x = a + i; /* the r-th element of bucket b (stable) */
                ptr[b]++;
            }
            seen[b]++;
        }
    }
    free(cnt); free(o); free(tmpq); free(ptr); free(lb);
    return rc;
}

int oracle_points(uint64_t n, uint32_t k, uint32_t L, uint64_t seed, const uint64_t *js, uint64_t count,
                  uint64_t *out)
{
    int rc = check_args(1, k, L);
    if (rc)
        return rc;
    if (count == 0)
        return 0;
    oq_t *qs = (oq_t *)calloc(count, sizeof(oq_t));
    oq_t **qp = (oq_t **)malloc(count * sizeof(oq_t *));
    if (!qs || !qp) {
        free(qs); free(qp);
        return ORACLE_ERR_NOMEM;
    }
    for (uint64_t s = 0; s < count; s++) {
        if (js[s] >= n) {
            free(qs); free(qp);
            return ORACLE_ERR_INVALID_ARG;
        }
        qs[s].j = js[s];
        qp[s] = &qs[s];
    }
    oq_ctx c;
    memset(&c, 0, sizeof c);
    c.K = oracle_problem_key(seed, 0);
    c.k = k;
    c.L = L;
    rc = oq_rec(&c, 0, n, 0, qp, count);
    for (uint64_t s = 0; rc == 0 && s < count; s++)
        out[s] = qs[s].x;
    free(qs); free(qp);
    return rc;
}

/* ------------------------------------------------- D9 (NEXT-1) -- */
/* Hidden-constant simulation of Lemma 2 and Corollary 5 / Lemma
 * 4, one run per key K(seed, r) (D2), r = 0 .. runs-1:
 *
 *   RoughScatter on n items and k buckets of capacities
 *   c_i = floor((i+1) n / k) - floor(i n / k) ("equal sizes n/k up to
 *   rounding"): in iteration t = 0, 1, ... draw the partner bucket
 *   j_t uniformly from [0, k) -- here the D4 bucket draw at level 0 and
 *   position t (the path's own generator) -- and place one item into B_j
 *   (s_j += 1); stop as soon as B_j is full (s_j = c_j).  T = number of
 *   placed items, R = n - T the items left staged (Lemma 2).
 *
 *   Final bucket sizes ("run the balls-into-bins experiment to
 *   completion"): the remaining R items draw j_t for t = T .. n-1
 *   the same way, n^f_i = #{t < n : j_t = i}.  d_i = n^f_i - c_i (deviation
 *   from the initial estimate), D_i = d_0 + ... + d_i, and TwoSweep performs
 *   M = sum_i |D_i| swaps (Lemma 4).
 *
 * Writes T[r] and M[r].  Returns 0, or ERR_INVALID_ARG for k < 2, k > 2^16
 * or n < k (every bucket needs capacity >= 1).                               */
int oracle_sim_rough_scatter(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t *T, uint64_t *M)
{
    if (k < 2 || k > 65536u || n < k) return ORACLE_ERR_INVALID_ARG;
    uint64_t *s = (uint64_t *)malloc((size_t)k * sizeof(uint64_t));
    if (!s) return ORACLE_ERR_NOMEM;
    for (uint32_t r = 0; r < runs; ++r) {
        const uint64_t K = oracle_problem_key(seed, r);
        memset(s, 0, (size_t)k * sizeof(uint64_t));
        uint64_t t = 0, stop = n;
        for (; t < n; ++t) {                        /* RoughScatter iterations */
            const uint32_t j = oracle_bucket_draw(K, 0, t, k, NULL);
            const uint64_t cj = (uint64_t)(((unsigned __int128)(j + 1) * n) / k) -
                                (uint64_t)(((unsigned __int128)j * n) / k);
            s[j] += 1;
            if (s[j] == cj) {                       /* B_j is full: stop */
                stop = t + 1;
                ++t;
                break;
            }
        }
        for (; t < n; ++t) s[oracle_bucket_draw(K, 0, t, k, NULL)] += 1; /* the staged rest */
        int64_t D = 0;
        uint64_t m = 0;
        for (uint32_t i = 0; i < k; ++i) {
            const uint64_t ci = (uint64_t)(((unsigned __int128)(i + 1) * n) / k) -
                                (uint64_t)(((unsigned __int128)i * n) / k);
            D += (int64_t)s[i] - (int64_t)ci;
            m += (uint64_t)(D < 0 ? -D : D);
        }
        T[r] = stop;
        M[r] = m;
    }
    free(s);
    return 0;
}

/* ------------------------------------------- D10 (NEXT-2) -- */
/* The paper's own In-Place ScatterShuffle, made deterministic with
 * counter-based draws (D10).  Per segment [a, a+m) at level l with
 * m > L (Fig. 2):
 *   buckets   k contiguous buckets of capacities c_i = floor((i+1)m/k) -
 *             floor(im/k) ("equal sizes n/k up to rounding"), each a
 *             triple (b_i, s_i, e_i): [b, s) placed, [s, e) staged;
 *   ParRough the buckets are split in halves recursively to
 *             depth t = min(11, floor(log2(m / k^2))) (base case N0 = k^2,
 *             P:506; at most 2^11 subtasks); heap-numbered nodes, root
 *             1, children 2v, 2v+1 taking [lo, lo + floor((hi-lo)/2)) and the
 *             rest of every bucket range of v.  Post-order: a leaf starts
 *             all-staged; an inner node first merges its children bucket by
 *             bucket ("swapping the staged items of the first half to the
 *             second half"): with A = e - s staged in the first half
 *             and B = s' - b' placed in the second, swap X[s + x] <-> X[s' - 1
 *             - x] for x < min(A, B) -> (b, s + B, e').  Then, unless a bucket
 *             is full, RoughScatter: repeat { j = draw(RS, step, v)
 *             in [0, k); swap X[s_0] <-> X[s_j] (skipped if j = 0); s_j++;
 *             stop if s_j = e_j }.
 *   Fine at the root: n_i = s_i - b_i placed, R = sum of
 *             the staged; N' = counts of R uniform draws draw(FM, r) (a
 *             multinomial(R, 1/k) variate); n^f_i = n_i + N'_i;
 *             TwoSweep with D_i = sum_{j<=i} (n^f_j - c_j):
 *             ascending i = 0..k-2, -D_i > 0 times B_i's last (staged) slot
 *             moves to B_{i+1} (e_i--, b_{i+1}--, then X[b_{i+1}] <->
 *             X[s_{i+1} - 1] if B_{i+1} has placed items, s_{i+1}--);
 *             descending i = k-2..0, D_i > 0 times B_{i+1}'s first slot moves
 *             to B_i (X[b_{i+1}] <-> X[s_{i+1}] if B_{i+1} has placed items,
 *             b_{i+1}++, s_{i+1}++, e_i++).  Stash: with p_0 < .. < p_{R-1}
 *             the staged positions, swap X[a+t] <-> X[p_t] for t = 0..R-1,
 *             Fisher-Yates X[a .. a+R) with partners draw(FY, i) in [0, i],
 *             undo the swaps for t = R-1..0.
 *   recurse   on the k final buckets at level l+1; a segment of at
 *             most L elements is a Fisher-Yates leaf (D5, as D6).
 * draw(tag, c0, c1): words w0..w3 of Philox(K, (c0, c1, lo32 a, tag | l << 8 |
 * (hi32 a & 0xFFFF) << 16)); the first word Lemire32 accepts for the bound, or
 * (w0 * bound) >> 32 if all four reject (probability < 2^-64).  Tags RS = 7,
 * FM = 8, FY = 9 (D3 holds 1..6).                                  */
#define IPSC_RS 7u
#define IPSC_FM 8u
#define IPSC_FY 9u
#define IPSC_TMAX 11u

uint32_t oracle_ipsc_draw(uint64_t K, uint32_t tag, uint32_t c0, uint32_t c1, uint32_t level, uint64_t a,
                          uint32_t bound)
{
    uint32_t key[2], ctr[4], w[4], out = 0;
    key_words(K, key);
    ctr[0] = c0;
    ctr[1] = c1;
    ctr[2] = (uint32_t)a;
    ctr[3] = tag | (level << 8) | (((uint32_t)(a >> 32) & 0xFFFFu) << 16);
    oracle_philox4x32_10(ctr, key, w);
    for (int q = 0; q < 4; ++q)
        if (oracle_lemire32_accept(w[q], bound, &out)) return out;
    return (uint32_t)(((uint64_t)w[0] * bound) >> 32);
}

uint32_t oracle_ipsc_depth(uint64_t m, uint32_t k)
{
    const uint64_t n0 = (uint64_t)k * k;
    uint32_t t = 0;
    while (t < IPSC_TMAX && (m >> (t + 1)) >= n0) ++t;
    return t;
}

typedef struct {
    unsigned char *A;
    uint32_t eb, k, L;
    uint64_t K;
    uint32_t max_levels;
    int run_leaves;
    uint64_t *b, *s, *e;   /* scratch triples: nodes x k (node v at index (v-1) * k) */
    oracle_ipsc_stats *st;
    uint64_t *sizes0;      /* optional: the root segment's final bucket sizes */
} ipsc_ctx;

static void ipsc_swap(ipsc_ctx *c, uint64_t x, uint64_t y)
{
    if (x != y) elem_swap(c->A + x * c->eb, c->A + y * c->eb, c->eb);
}

/* RoughScatter on node v's triples. */
static void ipsc_rough(ipsc_ctx *c, uint64_t *b, uint64_t *s, uint64_t *e, uint32_t v, uint32_t level, uint64_t a)
{
    (void)b;
    for (uint32_t i = 0; i < c->k; ++i)
        if (s[i] == e[i]) return; /* a full bucket: nothing to do */
    for (uint32_t step = 0;; ++step) {
        const uint32_t j = oracle_ipsc_draw(c->K, IPSC_RS, step, v, level, a, c->k);
        if (j != 0) ipsc_swap(c, s[0], s[j]);
        s[j] += 1;
        if (c->st) c->st->rough_steps += 1;
        if (s[j] == e[j]) return;
    }
}

/* Node v (depth d of t) over bucket ranges [lo_i, hi_i): result triples in node v's slot. */
static void ipsc_node(ipsc_ctx *c, uint32_t v, uint32_t d, uint32_t t, const uint64_t *lo, const uint64_t *hi,
                      uint32_t level, uint64_t a)
{
    const uint32_t k = c->k;
    uint64_t *b = c->b + (uint64_t)(v - 1) * k, *s = c->s + (uint64_t)(v - 1) * k, *e = c->e + (uint64_t)(v - 1) * k;
    if (d == t) {
        for (uint32_t i = 0; i < k; ++i) {
            b[i] = lo[i];
            s[i] = lo[i];
            e[i] = hi[i];
        }
    } else {
        uint64_t *mid = (uint64_t *)calloc((size_t)k, sizeof(uint64_t));
        if (!mid) abort();
        for (uint32_t i = 0; i < k; ++i) mid[i] = lo[i] + (hi[i] - lo[i]) / 2;
        ipsc_node(c, 2 * v, d + 1, t, lo, mid, level, a);
        ipsc_node(c, 2 * v + 1, d + 1, t, mid, hi, level, a);
        free(mid);
        const uint64_t *b1 = c->b + (uint64_t)(2 * v - 1) * k, *s1 = c->s + (uint64_t)(2 * v - 1) * k,
                       *e1 = c->e + (uint64_t)(2 * v - 1) * k;
        const uint64_t *b2 = c->b + (uint64_t)(2 * v) * k, *s2 = c->s + (uint64_t)(2 * v) * k,
                       *e2 = c->e + (uint64_t)(2 * v) * k;
        for (uint32_t i = 0; i < k; ++i) {
            const uint64_t A = e1[i] - s1[i], B = s2[i] - b2[i], mn = A < B ? A : B;
            for (uint64_t x = 0; x < mn; ++x) ipsc_swap(c, s1[i] + x, s2[i] - 1 - x);
            if (c->st) c->st->merge_swaps += mn;
            b[i] = b1[i];
            s[i] = s1[i] + B;
            e[i] = e2[i];
        }
    }
    ipsc_rough(c, b, s, e, v, level, a);
}

/* FineScatter at the root; writes the final bucket sizes to nf. */
static int ipsc_fine(ipsc_ctx *c, uint64_t *b, uint64_t *s, uint64_t *e, uint64_t *nf, uint32_t level, uint64_t a)
{
    const uint32_t k = c->k;
    uint64_t R = 0;
    for (uint32_t i = 0; i < k; ++i) {
        R += e[i] - s[i];
        nf[i] = s[i] - b[i];
    }
    if (R > 0xFFFFFFFFull) return ORACLE_ERR_INVALID_ARG;
    for (uint64_t r = 0; r < R; ++r) nf[oracle_ipsc_draw(c->K, IPSC_FM, (uint32_t)r, 0u, level, a, k)] += 1;
    {   /* Lemma 4: sum_i |D_i| from the capacities and the final sizes (the TwoSweep count below must match) */
        int64_t D = 0;
        for (uint32_t i = 0; i < k; ++i) {
            D += (int64_t)nf[i] - (int64_t)(e[i] - b[i]);
            if (c->st) c->st->dsum += (uint64_t)(D < 0 ? -D : D);
        }
    }
    /* TwoSweep: D_i = sum_{j<=i} (n^f_j - c_j); across the boundary of
     * buckets i and i+1, -D_i > 0 items move right in the ascending sweep (the
     * excess of B_i beyond what the buckets left of it still need, C_i) and
     * D_i > 0 items move left in the descending sweep: sum_i |D_i| transfers. */
    int64_t *Dp = (int64_t *)malloc((size_t)k * sizeof(int64_t));
    if (!Dp) return ORACLE_ERR_NOMEM;
    {
        int64_t D = 0;
        for (uint32_t i = 0; i < k; ++i) {
            D += (int64_t)nf[i] - (int64_t)(e[i] - b[i]);
            Dp[i] = D;
        }
    }
    for (uint32_t i = 0; i + 1 < k; ++i) /* sweep 1: B_i's last staged slot -> B_{i+1} */
        for (int64_t x = -Dp[i]; x > 0; --x) {
            e[i] -= 1;
            b[i + 1] -= 1;
            if (s[i + 1] > b[i + 1] + 1) ipsc_swap(c, b[i + 1], s[i + 1] - 1);
            s[i + 1] -= 1;
            if (c->st) c->st->transfers += 1;
        }
    for (uint32_t i = k - 1; i-- > 0;) /* sweep 2: B_{i+1}'s first slot -> B_i */
        for (int64_t x = Dp[i]; x > 0; --x) {
            if (s[i + 1] > b[i + 1]) ipsc_swap(c, b[i + 1], s[i + 1]);
            b[i + 1] += 1;
            s[i + 1] += 1;
            e[i] += 1;
            if (c->st) c->st->transfers += 1;
        }
    free(Dp);
    for (uint32_t i = 0; i < k; ++i)
        if (e[i] - b[i] != nf[i] || s[i] > e[i] || s[i] < b[i]) return ORACLE_ERR_INVALID_ARG; /* internal */
    /* stash shuffle: compact, Fisher-Yates, undo */
    uint64_t t = 0;
    for (uint32_t i = 0; i < k; ++i)
        for (uint64_t p = s[i]; p < e[i]; ++p) ipsc_swap(c, a + t++, p);
    for (uint64_t i = R; i-- > 1;)
        ipsc_swap(c, a + i, a + oracle_ipsc_draw(c->K, IPSC_FY, (uint32_t)i, 0u, level, a, (uint32_t)(i + 1)));
    for (uint32_t i = k; i-- > 0;)
        for (uint64_t p = e[i]; p-- > s[i];) ipsc_swap(c, a + --t, p);
    if (c->st) c->st->staged += R;
    return 0;
}

static int ipsc_rec(ipsc_ctx *c, uint64_t a, uint64_t m, uint32_t level)
{
    if (m <= c->L) {
        if (c->run_leaves && m >= 2) {
            for (uint64_t i = m; i-- > 1;) {
                const uint32_t j = oracle_fy_draw(c->K, a, (uint32_t)i, NULL);
                ipsc_swap(c, a + i, a + j);
            }
            if (c->st) c->st->leaves += 1;
        }
        return 0;
    }
    if (level >= c->max_levels) return 0;
    if (level > 255) return ORACLE_ERR_DEPTH;
    const uint32_t k = c->k, t = oracle_ipsc_depth(m, k);
    uint64_t *lo = (uint64_t *)malloc((size_t)k * sizeof(uint64_t)), *hi = (uint64_t *)malloc((size_t)k * sizeof(uint64_t));
    uint64_t *nf = (uint64_t *)malloc((size_t)k * sizeof(uint64_t));
    if (!lo || !hi || !nf) return ORACLE_ERR_NOMEM;
    for (uint32_t i = 0; i < k; ++i) {
        lo[i] = a + (uint64_t)(((unsigned __int128)i * m) / k);
        hi[i] = a + (uint64_t)(((unsigned __int128)(i + 1) * m) / k);
    }
    ipsc_node(c, 1, 0, t, lo, hi, level, a);
    int rc = ipsc_fine(c, c->b, c->s, c->e, nf, level, a);
    if (c->st) c->st->segments += 1;
    if (!rc && level == 0 && c->sizes0) memcpy(c->sizes0, nf, (size_t)k * sizeof(uint64_t));
    free(lo);
    free(hi);
    uint64_t start = a;
    for (uint32_t i = 0; i < k && !rc; ++i) {
        rc = ipsc_rec(c, start, nf[i], level + 1);
        start += nf[i];
    }
    free(nf);
    return rc;
}

int oracle_ipsc_shuffle(void *data, uint64_t n, uint32_t eb, uint32_t k, uint32_t L, uint64_t seed,
                        uint32_t max_levels, int run_leaves, oracle_ipsc_stats *st, uint64_t *sizes0)
{
    if (eb == 0 || k < 2 || k > 65536u || L < 1 || n >= (1ull << 48)) return ORACLE_ERR_INVALID_ARG;
    ipsc_ctx c;
    memset(&c, 0, sizeof c);
    c.A = (unsigned char *)data;
    c.eb = eb;
    c.k = k;
    c.L = L;
    c.K = oracle_problem_key(seed, 0);
    c.max_levels = max_levels;
    c.run_leaves = run_leaves;
    c.st = st;
    c.sizes0 = sizes0;
    if (st) memset(st, 0, sizeof *st);
    const uint64_t nodes = 2ull << oracle_ipsc_depth(n, k);  /* the root segment needs the deepest tree */
    c.b = (uint64_t *)malloc(nodes * k * sizeof(uint64_t));
    c.s = (uint64_t *)malloc(nodes * k * sizeof(uint64_t));
    c.e = (uint64_t *)malloc(nodes * k * sizeof(uint64_t));
    int rc = (!c.b || !c.s || !c.e) ? ORACLE_ERR_NOMEM : ipsc_rec(&c, 0, n, 0);
    free(c.b);
    free(c.s);
    free(c.e);
    return rc;
}
