/*
 * oracle/oracle.c -- plain, slow, single-threaded CPU ORACLE for mini-batch
 * ego-network generation (DistDGLv2, arxiv 2112.15345).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this file.
 * The product path (paper_2112_15345_b200/) never links, imports or executes
 * it, and shares no code, header, helper, table or constant generator with
 * it.  Nothing here is blocked, fused or reordered beyond what the cited
 * passage states.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * What it computes, step by step in the paper's order (the readings of the
 * paper that the text leaves open are listed in DESIGN.md §3):
 *
 *   homogenized IDs: gid = off[t] + tid, type-contiguous         P:409-415 §4.1.1
 *   type-specific IDs (tid) address per-type feature rows        P:474-475 §4.1.4
 *   F_0 = seeds split per vertex type, caller order
 *   for hop h = 0..L-1                                           P:694-700 §4.2.2
 *     for every relation r, every dst v in F_h[t(r)]:
 *       "randomly pick at most K (fanout) neighbor vertices"     P:282-285 §3.2
 *       d <= k (or k = -1): all in-edges; else the k smallest
 *       composites (key32(seed,h,r,v,j) << 32 | j), emitted in ascending j
 *     "compute the frontier (the unique set of vertices)"        P:698-700 §4.2.2
 *       new[u] = sorted unique(srcs of type u) \ F_h[u];  S[u] = F_h[u] ++ new[u]
 *     "graph compaction ... relabel vertices and edges"
 *       block h: dst = F_h, src = S, per relation CSC over F_h with local src ids
 *     F_{h+1} = S
 *   features of the input vertices S_{L-1}[u]                    P:563-565 §4.2.1
 *
 * key32(seed,h,r,v,j) = Philox4x32-10(ctr = {j>>2, lo32(v), hi32(v), (h<<16)|r},
 *                                     key = {lo32(seed), hi32(seed)}).word[j & 3]
 * (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ---------------------------------------------------------------- Philox */

/* Philox4x32 with R = 10 rounds; multipliers and Weyl key increments of the
 * published generator.  One round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 * c' = {hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0}; the key is bumped between
 * rounds. */
void og_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k[0];
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c[3] ^ k[1];
        uint32_t n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

uint32_t og_key32(uint64_t seed, uint32_t h, uint32_t r, uint64_t v, uint64_t j)
{
    uint32_t ctr[4] = {(uint32_t)(j >> 2), (uint32_t)v, (uint32_t)(v >> 32), (h << 16) | r};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    og_philox4x32_10(ctr, key, out);
    return out[j & 3];
}

/* ---------------------------------------------------------------- result */

typedef struct {
    int64_t n_dst;     /* |F_h[t(r)]| */
    int64_t nnz;
    int32_t *indptr;   /* n_dst + 1 */
    int32_t *indices;  /* local src index into S_h[s(r)] */
    int64_t *eids;     /* position in the relation's (unsharded) CSC */
    int64_t *src_gid;  /* the sampled edge list: global src id per edge */
} og_rel_block;

struct og_result {
    int32_t n_vt, n_rel, n_hops;
    /* nodes[h][u], h = 0..n_hops: h = 0 are the seeds of type u (F_0[u]);
     * h >= 1 is S_{h-1}[u] = F_h[u].  Each level is its own array. */
    int64_t **nodes;   /* (n_hops+1) * n_vt */
    int64_t *n_nodes;  /* (n_hops+1) * n_vt */
    og_rel_block *blk; /* n_hops * n_rel */
};

static void *xcalloc(size_t n, size_t sz)
{
    void *p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) abort();
    return p;
}

void og_free(og_result *res)
{
    if (!res) return;
    int levels = res->n_hops + 1;
    if (res->nodes)
        for (int i = 0; i < levels * res->n_vt; ++i) free(res->nodes[i]);
    free(res->nodes);
    free(res->n_nodes);
    if (res->blk)
        for (int i = 0; i < res->n_hops * res->n_rel; ++i) {
            free(res->blk[i].indptr);
            free(res->blk[i].indices);
            free(res->blk[i].eids);
            free(res->blk[i].src_gid);
        }
    free(res->blk);
    free(res);
}

/* ---------------------------------------------------------------- helpers */

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

typedef struct { int64_t gid; int64_t idx; } gid_idx;

static int cmp_gid_idx(const void *a, const void *b)
{
    int64_t x = ((const gid_idx *)a)->gid, y = ((const gid_idx *)b)->gid;
    return (x > y) - (x < y);
}

/* index of gid in the sorted (gid, idx) table, or -1 */
static int64_t lookup(const gid_idx *tab, int64_t n, int64_t gid)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (tab[mid].gid < gid) lo = mid + 1; else hi = mid;
    }
    return (lo < n && tab[lo].gid == gid) ? tab[lo].idx : -1;
}

/* the k selected neighbour offsets of one (dst, relation), ascending j.
 * P:282-285 "randomly pick at most K (called fanout) neighbor vertices":
 * uniform without replacement == the k smallest of d i.i.d. keys.  The
 * composite (key << 32 | j) breaks ties by the lower offset.  Returns count. */
static int64_t select_offsets(uint64_t seed, int32_t h, int32_t r, int64_t v,
                              int64_t d, int32_t k, int64_t *out_j)
{
    if (k == -1 || d <= (int64_t)k) {          /* the full neighbourhood, no RNG */
        for (int64_t j = 0; j < d; ++j) out_j[j] = j;
        return d;
    }
    uint64_t *comp = xcalloc((size_t)d, sizeof(uint64_t));
    for (int64_t j = 0; j < d; ++j)
        comp[j] = ((uint64_t)og_key32(seed, (uint32_t)h, (uint32_t)r, (uint64_t)v, (uint64_t)j) << 32)
                  | (uint64_t)j;
    qsort(comp, (size_t)d, sizeof(uint64_t), cmp_u64);      /* library sort as a step */
    for (int64_t m = 0; m < k; ++m) out_j[m] = (int64_t)(comp[m] & 0xFFFFFFFFu);
    qsort(out_j, (size_t)k, sizeof(int64_t), cmp_i64);       /* emit in ascending j */
    free(comp);
    return k;
}

/* ---------------------------------------------------------------- sample */

int og_sample(const og_graph *g, const int64_t *seeds, int64_t n_seeds,
              int32_t n_hops, const int32_t *fanouts, uint64_t rng_seed, og_result **out)
{
    *out = NULL;
    if (n_hops < 1 || n_seeds < 0) return OG_EINVAL;
    for (int i = 0; i < n_hops * g->n_rel; ++i)
        if (fanouts[i] < -1) return OG_EINVAL;

    const int V = g->n_vt, R = g->n_rel, L = n_hops;
    int64_t *off = xcalloc((size_t)V + 1, sizeof(int64_t));      /* P:413-414 contiguous IDs */
    for (int t = 0; t < V; ++t) off[t + 1] = off[t] + g->vt_count[t];
    const int64_t n_total = off[V];

    /* seed checks: in range, unique */
    for (int64_t i = 0; i < n_seeds; ++i)
        if (seeds[i] < 0 || seeds[i] >= n_total) { free(off); return OG_ERANGE; }
    {
        int64_t *tmp = xcalloc((size_t)n_seeds, sizeof(int64_t));
        memcpy(tmp, seeds, (size_t)n_seeds * sizeof(int64_t));
        qsort(tmp, (size_t)n_seeds, sizeof(int64_t), cmp_i64);
        for (int64_t i = 1; i < n_seeds; ++i)
            if (tmp[i] == tmp[i - 1]) { free(tmp); free(off); return OG_EINVAL; }
        free(tmp);
    }

    og_result *res = xcalloc(1, sizeof(og_result));
    res->n_vt = V; res->n_rel = R; res->n_hops = L;
    res->nodes = xcalloc((size_t)(L + 1) * V, sizeof(int64_t *));
    res->n_nodes = xcalloc((size_t)(L + 1) * V, sizeof(int64_t));
    res->blk = xcalloc((size_t)L * R, sizeof(og_rel_block));

    /* vertex type of a gid */
#define VT_OF(gid_, vt_out_) do { int tt_ = 0; while (!((gid_) >= off[tt_] && (gid_) < off[tt_ + 1])) ++tt_; (vt_out_) = tt_; } while (0)

    /* F_0[t] = seeds of type t, caller order */
    for (int t = 0; t < V; ++t) {
        int64_t n = 0;
        for (int64_t i = 0; i < n_seeds; ++i) { int vt; VT_OF(seeds[i], vt); if (vt == t) ++n; }
        res->nodes[t] = xcalloc((size_t)n, sizeof(int64_t));
        res->n_nodes[t] = n;
        n = 0;
        for (int64_t i = 0; i < n_seeds; ++i) { int vt; VT_OF(seeds[i], vt); if (vt == t) res->nodes[t][n++] = seeds[i]; }
    }

    for (int h = 0; h < L; ++h) {
        int64_t **F = &res->nodes[(size_t)h * V];
        int64_t *nF = &res->n_nodes[(size_t)h * V];

        /* --- neighbour sampling, per relation, per dst in frontier order --- */
        for (int r = 0; r < R; ++r) {
            og_rel_block *b = &res->blk[(size_t)h * R + r];
            const int s = g->rel_src_vt[r], t = g->rel_dst_vt[r];
            const int32_t k = fanouts[(size_t)h * R + r];
            const int64_t *ip = g->indptr[r];
            const int32_t *ix = g->indices[r];
            b->n_dst = nF[t];
            b->indptr = xcalloc((size_t)nF[t] + 1, sizeof(int32_t));
            int64_t cap = 0;
            for (int64_t i = 0; i < nF[t]; ++i) {
                int64_t x = F[t][i] - off[t];
                int64_t d = ip[x + 1] - ip[x];
                cap += (k == -1 || d <= k) ? d : k;
            }
            b->nnz = cap;
            b->indices = xcalloc((size_t)cap, sizeof(int32_t));
            b->eids = xcalloc((size_t)cap, sizeof(int64_t));
            b->src_gid = xcalloc((size_t)cap, sizeof(int64_t));
            int64_t e = 0;
            for (int64_t i = 0; i < nF[t]; ++i) {
                int64_t v = F[t][i];
                int64_t x = v - off[t];
                int64_t d = ip[x + 1] - ip[x];
                int64_t *js = xcalloc((size_t)d, sizeof(int64_t));
                int64_t c = select_offsets(rng_seed, h, r, v, d, k, js);
                b->indptr[i] = (int32_t)e;
                for (int64_t m = 0; m < c; ++m) {
                    int64_t pos = ip[x] + js[m];
                    b->src_gid[e] = off[s] + ix[pos];
                    b->eids[e] = pos;
                    ++e;
                }
                free(js);
            }
            b->indptr[nF[t]] = (int32_t)e;
        }

        /* --- frontier: S[u] = F[u] ++ sorted(unique(srcs of u) \ F[u]) --- */
        int64_t **S = &res->nodes[(size_t)(h + 1) * V];
        int64_t *nS = &res->n_nodes[(size_t)(h + 1) * V];
        gid_idx **tab = xcalloc((size_t)V, sizeof(gid_idx *));
        for (int u = 0; u < V; ++u) {
            int64_t cnt = 0;
            for (int r = 0; r < R; ++r)
                if (g->rel_src_vt[r] == u) cnt += res->blk[(size_t)h * R + r].nnz;
            int64_t *all = xcalloc((size_t)cnt, sizeof(int64_t));
            int64_t m = 0;
            for (int r = 0; r < R; ++r)
                if (g->rel_src_vt[r] == u) {
                    og_rel_block *b = &res->blk[(size_t)h * R + r];
                    for (int64_t e = 0; e < b->nnz; ++e) all[m++] = b->src_gid[e];
                }
            qsort(all, (size_t)cnt, sizeof(int64_t), cmp_i64);
            gid_idx *ftab = xcalloc((size_t)nF[u], sizeof(gid_idx));
            for (int64_t i = 0; i < nF[u]; ++i) { ftab[i].gid = F[u][i]; ftab[i].idx = i; }
            qsort(ftab, (size_t)nF[u], sizeof(gid_idx), cmp_gid_idx);
            int64_t n_new = 0;
            for (int64_t i = 0; i < cnt; ++i) {
                if (i > 0 && all[i] == all[i - 1]) continue;            /* unique */
                if (lookup(ftab, nF[u], all[i]) >= 0) continue;         /* \ F[u] */
                all[n_new++] = all[i];                                  /* stays sorted */
            }
            nS[u] = nF[u] + n_new;
            S[u] = xcalloc((size_t)nS[u], sizeof(int64_t));
            memcpy(S[u], F[u], (size_t)nF[u] * sizeof(int64_t));
            memcpy(S[u] + nF[u], all, (size_t)n_new * sizeof(int64_t));
            free(all);
            free(ftab);
            tab[u] = xcalloc((size_t)nS[u], sizeof(gid_idx));
            for (int64_t i = 0; i < nS[u]; ++i) { tab[u][i].gid = S[u][i]; tab[u][i].idx = i; }
            qsort(tab[u], (size_t)nS[u], sizeof(gid_idx), cmp_gid_idx);
        }

        /* --- relabel every sampled src to its index in S[s(r)] --- */
        for (int r = 0; r < R; ++r) {
            og_rel_block *b = &res->blk[(size_t)h * R + r];
            const int s = g->rel_src_vt[r];
            for (int64_t e = 0; e < b->nnz; ++e)
                b->indices[e] = (int32_t)lookup(tab[s], nS[s], b->src_gid[e]);
        }
        for (int u = 0; u < V; ++u) free(tab[u]);
        free(tab);
    }
#undef VT_OF
    free(off);
    *out = res;
    return OG_OK;
}

/* ---------------------------------------------------------------- gather */

/* out[i] = rows[ids[i] - off_u], verbatim bytes, where ids = S_{L-1}[u] are the
 * input vertices of type u ("CPU feature copy ... stores data in
 * contiguous CPU memory"; P:474-475 type-specific ids; SPEC pull S:217-225:
 * rows in input order). */
int og_gather(const int64_t *ids, int64_t n, int64_t off_u, int64_t n_u,
              const void *rows, int64_t row_bytes, void *out)
{
    if (n < 0 || row_bytes <= 0) return OG_EINVAL;
    for (int64_t i = 0; i < n; ++i)
        if (ids[i] < off_u || ids[i] >= off_u + n_u) return OG_ERANGE;
    for (int64_t i = 0; i < n; ++i)
        memcpy((char *)out + i * row_bytes, (const char *)rows + (ids[i] - off_u) * row_bytes,
               (size_t)row_bytes);
    return OG_OK;
}

/* ---------------------------------------------------------------- link prediction targets */

/* The scheduler "determines target vertices or target edges in each mini-batch to
 * support various learning tasks (e.g., node classification, link prediction)"
 * (§4.2.1); link prediction trains on edges (§5).  SPEC's
 * make_link_task: per positive edge, num_negatives corrupted pairs with the
 * dst resampled uniformly from the dst vertex type's ID range; the seed vertex set is
 * the union of all endpoints.  Readings (L1-L4):
 *   L1 corrupted pair q of positive i keeps src_i; its dst is
 *      off[t(r)] + floor(w * N_{t(r)} / 2^32),
 *      w = Philox4x32-10(ctr = {i, q, 0, 0x4E454721 'NEG!'}, key = {lo32(neg_seed),
 *      hi32(neg_seed)}).word[0];
 *   L2 the seeds are the distinct endpoints in ascending gid (type-contiguous gids, so
 *      (type, gid) order); sampling then starts from them exactly as og_sample does;
 *   L3 every pair is returned as the local ids of its endpoints (index among the seeds
 *      of the endpoint's type = its position in block 0's dst nodes);
 *   L4 no seed edge is excluded from sampling (the paper states no exclusion).
 * neg_dst: n_pos*n_neg gids; seeds: capacity n_pos*(2+n_neg); pairs: int32
 * [pos_src n_pos][pos_dst n_pos][neg_src n_pos*n_neg][neg_dst n_pos*n_neg]. */
int og_lp_targets(const og_graph *g, const int64_t *src, const int64_t *dst, int64_t n_pos, int32_t rel,
                  int32_t n_neg, uint64_t neg_seed, int64_t *neg_dst, int64_t *seeds, int64_t *n_seeds,
                  int32_t *pairs)
{
    if (rel < 0 || rel >= g->n_rel || n_pos < 0 || n_neg < 0 || n_pos >= ((int64_t)1 << 32)) return OG_EINVAL;
    const int V = g->n_vt;
    int64_t *off = xcalloc((size_t)V + 1, sizeof(int64_t));
    for (int t = 0; t < V; ++t) off[t + 1] = off[t] + g->vt_count[t];
    const int s = g->rel_src_vt[rel], t = g->rel_dst_vt[rel];
    for (int64_t i = 0; i < n_pos; ++i)
        if (src[i] < off[s] || src[i] >= off[s + 1] || dst[i] < off[t] || dst[i] >= off[t + 1]) {
            free(off);
            return OG_ERANGE;
        }
    /* L1: negatives */
    const uint32_t key[2] = {(uint32_t)neg_seed, (uint32_t)(neg_seed >> 32)};
    const uint64_t n_t = (uint64_t)g->vt_count[t];
    for (int64_t i = 0; i < n_pos; ++i)
        for (int32_t q = 0; q < n_neg; ++q) {
            const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)q, 0u, 0x4E454721u};
            uint32_t w[4];
            og_philox4x32_10(ctr, key, w);
            neg_dst[i * n_neg + q] = off[t] + (int64_t)(((uint64_t)w[0] * n_t) >> 32);
        }
    /* L2: distinct endpoints, ascending */
    const int64_t n_end = n_pos * (2 + (int64_t)n_neg);
    int64_t *e = xcalloc((size_t)n_end + 1, sizeof(int64_t));
    int64_t m = 0;
    for (int64_t i = 0; i < n_pos; ++i) e[m++] = src[i];
    for (int64_t i = 0; i < n_pos; ++i) e[m++] = dst[i];
    for (int64_t i = 0; i < n_pos * n_neg; ++i) e[m++] = neg_dst[i];
    qsort(e, (size_t)m, sizeof(int64_t), cmp_i64);
    int64_t k = 0;
    for (int64_t i = 0; i < m; ++i)
        if (k == 0 || e[i] != seeds[k - 1]) seeds[k++] = e[i];
    *n_seeds = k;
    /* L3: local ids = index among the seeds of the endpoint's type */
    int64_t *first = xcalloc((size_t)V + 1, sizeof(int64_t));   /* first seed index of type u */
    for (int u = 0; u <= V; ++u) {
        int64_t lo = 0, hi = k;                                    /* first seed >= off[u] */
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (seeds[mid] < off[u]) lo = mid + 1; else hi = mid;
        }
        first[u] = lo;
    }
    for (int64_t i = 0; i < m; ++i) {
        const int64_t x = i < n_pos ? src[i] : i < 2 * n_pos ? dst[i - n_pos] : neg_dst[i - 2 * n_pos];
        int64_t lo = 0, hi = k;                                    /* index of x in seeds */
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (seeds[mid] < x) lo = mid + 1; else hi = mid;
        }
        int u = 0;
        while (x >= off[u + 1]) ++u;
        const int32_t local = (int32_t)(lo - first[u]);
        if (i < 2 * n_pos) pairs[i] = local;                                   /* pos_src, pos_dst */
        else {
            const int64_t j = i - 2 * n_pos;                                  /* negative j */
            pairs[2 * n_pos + j] = pairs[j / (n_neg ? n_neg : 1)];               /* neg_src = pos_src */
            pairs[2 * n_pos + n_pos * n_neg + j] = local;                        /* neg_dst */
        }
    }
    free(first);
    free(e);
    free(off);
    return OG_OK;
}

/* ---------------------------------------------------------------- accessors */

int64_t og_n_nodes(const og_result *res, int32_t level, int32_t u)
{
    return res->n_nodes[(size_t)level * res->n_vt + u];
}

const int64_t *og_nodes(const og_result *res, int32_t level, int32_t u)
{
    return res->nodes[(size_t)level * res->n_vt + u];
}

int og_block(const og_result *res, int32_t h, int32_t r, int64_t *n_dst, int64_t *nnz,
             const int32_t **indptr, const int32_t **indices, const int64_t **eids,
             const int64_t **src_gid)
{
    if (h < 0 || h >= res->n_hops || r < 0 || r >= res->n_rel) return OG_EINVAL;
    const og_rel_block *b = &res->blk[(size_t)h * res->n_rel + r];
    *n_dst = b->n_dst; *nnz = b->nnz;
    *indptr = b->indptr; *indices = b->indices; *eids = b->eids; *src_gid = b->src_gid;
    return OG_OK;
}
