/*
 * oracle/oracle.h -- interface of the CPU oracle (TEST INFRASTRUCTURE ONLY;
 * see the header of oracle.c for who may use it and what it follows).
 * This header is private to oracle/: the product path never includes it.
 */
#ifndef EGO_ORACLE_H
#define EGO_ORACLE_H
#include <stdint.h>

#define OG_OK 0
#define OG_EINVAL (-1)
#define OG_ERANGE (-2)

typedef struct {
    int32_t n_vt;
    const int64_t *vt_count;          /* N_t per vertex type */
    int32_t n_rel;
    const int32_t *rel_src_vt;        /* s(r) */
    const int32_t *rel_dst_vt;        /* t(r) */
    const int64_t *const *indptr;     /* per r: global in-CSC over dst tids, N_{t(r)}+1 */
    const int32_t *const *indices;    /* per r: src tids */
} og_graph;

typedef struct og_result og_result;

void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t og_key32(uint64_t seed, uint32_t h, uint32_t r, uint64_t v, uint64_t j);

/* fanouts: n_hops x n_rel, row = hop from the seeds; -1 = all, 0 = none. */
int og_sample(const og_graph *g, const int64_t *seeds, int64_t n_seeds, int32_t n_hops,
              const int32_t *fanouts, uint64_t rng_seed, og_result **out);
/* ids = input vertices of one type u (gids in [off_u, off_u + n_u)); rows = all
 * N_u feature rows of type u; out = n * row_bytes. */
int og_gather(const int64_t *ids, int64_t n, int64_t off_u, int64_t n_u,
              const void *rows, int64_t row_bytes, void *out);
void og_free(og_result *res);

/* Link-prediction targets (see oracle.c): negatives, the seed set (distinct endpoints,
 * ascending) and every pair in local ids.  Sampling then runs og_sample on the seeds. */
int og_lp_targets(const og_graph *g, const int64_t *src, const int64_t *dst, int64_t n_pos, int32_t rel,
                  int32_t n_neg, uint64_t neg_seed, int64_t *neg_dst, int64_t *seeds, int64_t *n_seeds,
                  int32_t *pairs);

/* level 0 = seeds per type (F_0); level h+1 = S_h (src nodes of block h). */
int64_t og_n_nodes(const og_result *res, int32_t level, int32_t u);
const int64_t *og_nodes(const og_result *res, int32_t level, int32_t u);
int og_block(const og_result *res, int32_t h, int32_t r, int64_t *n_dst, int64_t *nnz,
             const int32_t **indptr, const int32_t **indices, const int64_t **eids,
             const int64_t **src_gid);
#endif
