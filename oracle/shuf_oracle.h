/*
 * oracle/shuf_oracle.h -- TEST INFRASTRUCTURE ONLY (see shuf_oracle.c).
 * Never included by the CUDA path.
 */
#ifndef SHUF_ORACLE_H
#define SHUF_ORACLE_H
#include <stdint.h>

#define ORACLE_ERR_INVALID_ARG 1
#define ORACLE_ERR_DEPTH 5
#define ORACLE_ERR_NOMEM 7

typedef struct {
    uint32_t levels;                /* number of scatter levels that ran       */
    uint32_t pad;
    uint64_t scatter_elems[257];    /* n_l: elements scattered at level l       */
    uint64_t leaves;                /* leaves finished by Fisher-Yates          */
    uint64_t bucket_rejections;     /* D4 retry draws                           */
    uint64_t fy_rejections;         /* D5 retry draws                           */
} oracle_stats;

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t oracle_problem_key(uint64_t seed, uint64_t s);
int oracle_lemire16_accept(uint32_t v, uint32_t s, uint32_t *out);
int oracle_lemire32_accept(uint32_t w, uint32_t s, uint32_t *out);
uint32_t oracle_bucket_draw(uint64_t K, uint32_t level, uint64_t p, uint32_t k, uint64_t *rejections);
uint32_t oracle_fy_draw(uint64_t K, uint64_t q, uint32_t i, uint64_t *rejections);
void oracle_bucket_draws(uint64_t K, uint32_t level, uint64_t p0, uint64_t count, uint32_t k, uint32_t *out);
void oracle_fy_draws(uint64_t K, const uint64_t *q, const uint32_t *i, uint64_t count, uint32_t *out);
void oracle_fy_with_draws(void *data, uint64_t m, uint32_t eb, const uint32_t *j);
int oracle_shuffle(void *data, uint64_t n, uint32_t eb, uint32_t k, uint32_t L, uint64_t seed,
                   uint32_t max_levels, int run_leaves, oracle_stats *st);
int oracle_segmented(void *data, const uint64_t *offsets, uint64_t num_segments, uint32_t eb, uint32_t k,
                     uint32_t L, uint64_t seed, uint32_t max_levels, int run_leaves, oracle_stats *st);

int oracle_points(uint64_t n, uint32_t k, uint32_t L, uint64_t seed, const uint64_t *js, uint64_t count,
                  uint64_t *out);
int oracle_sim_rough_scatter(uint64_t n, uint32_t k, uint64_t seed, uint32_t runs, uint64_t *T, uint64_t *M);

/* D10 (NEXT-2): the paper's In-Place ScatterShuffle (RoughScatter, ParRoughScatter
 * merges, FineScatter with TwoSweep and the stash shuffle), deterministic draws. */
typedef struct {
    uint64_t segments;     /* IpSc segments processed                          */
    uint64_t rough_steps;  /* RoughScatter iterations (all nodes)              */
    uint64_t merge_swaps;  /* ParRoughScatter merge swaps                      */
    uint64_t staged;       /* sum of R (items left staged for FineScatter)     */
    uint64_t transfers;    /* TwoSweep unit transfers                          */
    uint64_t dsum;         /* sum over segments of sum_i |D_i| (Lemma 4)       */
    uint64_t leaves;       /* Fisher-Yates leaves                              */
} oracle_ipsc_stats;
uint32_t oracle_ipsc_draw(uint64_t K, uint32_t tag, uint32_t c0, uint32_t c1, uint32_t level, uint64_t a,
                          uint32_t bound);
uint32_t oracle_ipsc_depth(uint64_t m, uint32_t k);
int oracle_ipsc_shuffle(void *data, uint64_t n, uint32_t eb, uint32_t k, uint32_t L, uint64_t seed,
                        uint32_t max_levels, int run_leaves, oracle_ipsc_stats *st, uint64_t *sizes0);

#endif
