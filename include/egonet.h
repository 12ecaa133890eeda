/*
 * egonet.h -- C ABI of the B200-native mini-batch ego-network generator
 * (the data-parallel hot path of DistDGLv2, arxiv 2112.15345).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n
 * (the reference is not needed at run time; the citations are for readers).
 *
 * The three calls follow the paper's problem statement:
 *   eg_load_partition   a partitioned heterogeneous graph: per edge type a CSC,
 *                       per vertex type a range of owned vertices and their
 *                       feature rows (homogenized type-contiguous ids P:409-415;
 *                       KVStore id space per type with a partition policy P:465-475).
 *   eg_sample_blocks    vertex-wise neighbour sampling from seeds, at most
 *                       fanout[hop][etype] in-neighbours per target,
 *                       hop by hop with the frontier = unique set,
 *                       each hop compacted into a block.
 *   eg_gather_features  the feature rows of the input vertices of the blocks
 *                       (CPU/GPU feature copy P:563-565; KVStore pull S:217-225).
 *
 * Conventions
 *   - gid = homogenized global vertex id: gid = off[t] + tid, off = prefix sums of
 *     vt_counts; tid = type-local id.  All gids must be < 2^31.
 *   - Relation r has src type s(r) and dst type t(r).  Its CSC is the in-edge
 *     list of each dst vertex (CSC = grouped by dst), src ids are TYPE-LOCAL tids.
 *   - Partition: vertex type t is split in ranges bounds[t][p] <= tid <
 *     bounds[t][p+1]; rank p owns the CSC rows of its dst vertices (edge owner =
 *     dst owner) and the feature rows of its vertices.
 *   - All calls are stream-ordered on the context's stream.  Device pointers are
 *     CUDA device pointers of the context's device; "host" marks host pointers.
 *   - Results are defined by the key32 reading of the paper and are
 *     independent of world size, stream overlap and launch configuration.
 *
 * Errors: every call returns eg_status; on failure eg_last_error() has a message.
 *   EG_EINVAL bad argument (checked before any device work unless stated),
 *   EG_ERANGE a vertex id outside its id space (range error before any
 *             transfer), EG_ENOMEM device allocation failed, EG_ECUDA a CUDA error
 *   (the context becomes unusable: EG_ESTATE thereafter), EG_EPEER peer shard
 *   metadata inconsistent.
 */
#ifndef EGONET_H
#define EGONET_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define EG_API __attribute__((visibility("default")))
#else
#define EG_API
#endif

#define EG_MAX_VT 8
#define EG_MAX_REL 8
#define EG_MAX_RANKS 8
#define EG_MAX_HOPS 8

typedef enum {
    EG_OK = 0,
    EG_EINVAL = -1,
    EG_ERANGE = -2,
    EG_ENOMEM = -3,
    EG_ECUDA = -4,
    EG_EPEER = -6,
    EG_ESTATE = -7
} eg_status;

typedef struct eg_ctx eg_ctx;
typedef struct eg_blocks eg_blocks;

/* One relation's shard on this rank (borrowed, device memory, must outlive the ctx). */
typedef struct {
    int32_t src_vt, dst_vt;
    const int64_t *indptr;   /* device, n_local_dst + 1 entries, indptr[0] == 0,
                                n_local_dst = bounds[dst_vt][rank+1] - bounds[dst_vt][rank] */
    const int32_t *indices;  /* device, n_local_edges src tids (type s(r)) */
    int64_t n_local_edges;   /* == indptr[n_local_dst] */
    int64_t edge_base;       /* global CSC position of local edge 0 (edge ids = base + local pos) */
} eg_relation;

/* One vertex type's feature shard on this rank (borrowed).  rows may be device memory
 * or, at world 1, pinned / registered host memory (cudaHostAlloc, cudaHostRegister):
 * the gather kernel then reads the rows zero-copy over PCIe -- the paper's placement of
 * graph data in CPU memory (SURVEY §8f NEXT-4 ii), which lets a
 * feature store larger than HBM (C5: 187 GB) serve one GPU.  Pageable host memory, or
 * host memory at world > 1, is EG_EINVAL. */
typedef struct {
    const void *rows;        /* n_local_rows x row_bytes, row-major; NULL: no features */
    int64_t row_bytes;       /* multiple of 16 (or 0 when rows == NULL) */
} eg_features;

/* A block (hop h) as host struct of device pointers.  hop 0 is the seeds' block
 * (DGL's list order is the reverse).  dst_nodes[u] is a prefix of src_nodes[u]
 * (dst-in-src convention).  indptr[r] has n_dst[t(r)] + 1 entries (starting at
 * 0); indices[r] are local ids into src_nodes[s(r)]; eids[r] are positions in
 * the relation's unsharded CSC. */
typedef struct {
    int32_t hop, n_vt, n_rel, _pad;
    const int64_t *dst_nodes[EG_MAX_VT];
    int64_t n_dst[EG_MAX_VT];
    const int64_t *src_nodes[EG_MAX_VT];
    int64_t n_src[EG_MAX_VT];
    const int32_t *indptr[EG_MAX_REL];
    const int32_t *indices[EG_MAX_REL];
    const int64_t *eids[EG_MAX_REL];
    int64_t nnz[EG_MAX_REL];
} eg_block_view;

/* Library version string. */
EG_API const char *eg_version(void);

/* Bytes of the per-batch device counters copied to the host at the end of every launch
 * (sizes, error bits, trace stamps): the only device->host transfer of a batch whose
 * features stay on the device. */
EG_API int64_t eg_counter_bytes(void);

/* Create a context for rank `rank` of `world` (1 <= world <= EG_MAX_RANKS) on CUDA
 * device `device`; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Fails with EG_ECUDA when no usable sm_100 device is present. */
EG_API eg_status eg_create(int32_t rank, int32_t world, int32_t device, void *stream, eg_ctx **out);

/* Change the stream subsequent calls are ordered on. */
EG_API eg_status eg_set_stream(eg_ctx *ctx, void *stream);

/* Load this rank's shard.  vt_counts: host [n_vt] (N_t);
 * bounds: host [n_vt][world+1] non-decreasing with bounds[t][0]=0 and
 * bounds[t][world]=N_t, or NULL for the fixed policy bounds[t][p] = floor(p*N_t/world);
 * rels: host [n_rel]; feats: host [n_vt].  The buffers are BORROWED (not copied).
 * Validates shapes and ranges of the metadata; device contents are trusted.
 * EG_EINVAL also when a relation's largest local in-degree exceeds 2^26 (the
 * sampler splits hub rows into at most 2^16 tasks of 1024 keys).
 * Allocates the per-context compaction state (4 B per global vertex + a bitmap). */
EG_API eg_status eg_load_partition(eg_ctx *ctx, int32_t n_vt, const int64_t *vt_counts, const int64_t *bounds,
                            int32_t n_rel, const eg_relation *rels, const eg_features *feats);

/* world > 1 only.  Peer mapping over NVLink: every rank exports a host blob
 * describing its shard (CUDA IPC handles of the borrowed buffers + metadata),
 * the caller all-gathers the blobs with its own transport (e.g. a torch process
 * group), and every rank imports all of them.  After import, the kernels read
 * peer CSC rows and feature rows directly over NVLink / NVSwitch.
 * eg_export_shard: buf == NULL returns the size in *len.
 * eg_import_shards: blobs = world blobs, `stride` bytes apart, in rank order.
 * EG_EPEER when the peers' metadata disagrees (types, counts, bounds, edge bases). */
EG_API eg_status eg_export_shard(const eg_ctx *ctx, void *buf, size_t *len);
EG_API eg_status eg_import_shards(eg_ctx *ctx, const void *blobs, size_t stride);

/* Single-process alternative to export/import: attach the shard of `peer`, a
 * context of the same world loaded in this process (same device or another
 * device with peer access).  Once every other rank is attached the context is
 * ready.  Lets one process drive several ranks (and tests emulate world > 1 on
 * one GPU). */
EG_API eg_status eg_attach_peer(eg_ctx *ctx, const eg_ctx *peer);

/* Replicated partition policy for one vertex type's features ("Each ID
 * space is also associated with a partition policy that maps vertex/edge data to
 * physical machines"; here a policy may map a small type to every GPU).  rows: the
 * type's FULL table, n_rows == N_vt rows of the row_bytes given at load, row-major by
 * type-local id, in device memory of this context's GPU; BORROWED until eg_destroy.
 * The gather then reads that type's rows from the local replica instead of the
 * owners' shards (no NVLink traffic for it); results are byte-identical either way,
 * since the replica must equal the sharded rows (not checked).  rows == NULL restores
 * the sharded policy.  Per rank, not collective; call after eg_load_partition and
 * before the first sampling call (the batch graphs capture the policy): EG_ESTATE
 * otherwise.  EG_EINVAL: vt out of range, a type without features, n_rows != N_vt,
 * rows not device memory of this GPU. */
EG_API eg_status eg_set_feature_replica(eg_ctx *ctx, int32_t vt, const void *rows, int64_t n_rows);

/* Which feature-gather kernel the last enqueued gather used (instrumentation; the
 * kernel captured into the launched batch graph, or of the last eg_gather_features): 0 =
 * gather_tma_kernel (TMA: cp.async.bulk.tensor tile::gather4, four rows per operation, from
 * one tensor map per vertex type and owner shard -- the own table, or the IPC-mapped peer
 * shards read over NVLink -- for rows <= 1 KB and a multiple of 16 B; per-row bulk copies
 * otherwise), 1 = gather_ldg_kernel (16-B vector loads), -1 = none yet.  Default
 * (EG_GATHER=auto, read at eg_create): TMA, except at world 1 when a requested type has no
 * gather4 map (local per-row bulk copies are issue-bound); EG_GATHER=tma|ldg forces one.
 * Rows wider than one 16 KB TMA stage always take the LDG kernel. */
EG_API int32_t eg_gather_path(const eg_ctx *ctx);

/* Sample L = n_hops blocks from `seeds` (gids, unique, any vertex types, caller
 * order; host or device pointer; n_seeds may be 0).  fanouts: host [n_hops][n_rel],
 * row 0 = hop at the seeds; -1 = all in-neighbours, 0 = none, k > 0 = at most k,
 * uniformly without replacement, per edge type.  rng_seed keys the
 * draws: the result is a pure function of (graph, seeds, fanouts, rng_seed).
 * EG_ERANGE: a seed outside [0, N_total); EG_EINVAL: duplicate seeds, bad fanout,
 * n_hops outside [1, EG_MAX_HOPS].  The id checks run on the device; the call
 * returns after the batch's sizes are known (one device->host read). */
EG_API eg_status eg_sample_blocks(eg_ctx *ctx, const int64_t *seeds, int64_t n_seeds, int32_t n_hops,
                           const int32_t *fanouts, uint64_t rng_seed, eg_blocks **out);

/* Flags of eg_sample_minibatch. */
#define EG_FEATURES 1   /* also gather the input vertices' feature rows (library-owned) */
#define EG_ASYNC 2      /* return right after enqueueing; sizes are resolved by eg_blocks_wait */

/* Seeds buffers passed to the sampling calls are read in place when they are device
 * memory or pinned host memory (so they must stay unchanged until the batch is resolved)
 * and copied when they are pageable host memory. */

/* One whole mini-batch as ONE CUDA-graph launch: sampling + compaction of every hop
 * and, with EG_FEATURES, the feature gather of the input vertices into buffers the
 * blocks handle owns (eg_blocks_features).  Same semantics and errors as
 * eg_sample_blocks (which is this call with flags = 0).  With EG_ASYNC the call
 * returns after enqueueing on the context's stream (no host synchronisation), so a
 * caller can enqueue batch b+1 before reading batch b; seed errors are then
 * reported by eg_blocks_wait (or any accessor).  Batch memory comes from a ring of
 * slots per (n_hops, fanouts, seed capacity): one device allocation and one
 * captured graph per slot, reused after eg_blocks_free. */
EG_API eg_status eg_sample_minibatch(eg_ctx *ctx, const int64_t *seeds, int64_t n_seeds, int32_t n_hops,
                                     const int32_t *fanouts, uint64_t rng_seed, int32_t flags, eg_blocks **out);

/* Pipeline shape.  depth: up to `depth` launches run concurrently (round-robin over
 * `depth` lanes, each with its own stream); bundle: one launch may carry up to `bundle`
 * mini-batches (eg_sample_bundle), each phase kernel processing all of them at once
 * (the paper's bundling of several mini-batches); 1 <= bundle <= 32 (the
 * build's kMaxBundle), else EG_EINVAL.  Each lane keeps `bundle` batch-sized states
 * (bucket counts of 8 B per 2^bshift gids, element / member arrays sized by the seed
 * capacity and fanouts).  Default 1, 1.
 * Results never change; the caller overlaps launches by enqueueing with EG_ASYNC
 * before waiting (the asynchronous mini-batch pipeline of P:548-679). */
EG_API eg_status eg_set_pipeline(eg_ctx *ctx, int32_t depth, int32_t bundle);

/* n_batches (1 <= n <= bundle) independent mini-batches as ONE graph launch: batch b
 * has seeds[b] (n_seeds[b] gids, host or device), rng_seeds[b]; all share n_hops and
 * fanouts.  out[b] receives batch b's handle (freed independently).  Same flags and
 * errors as eg_sample_minibatch; without EG_ASYNC the call returns once all n_batches
 * are resolved (on an error all handles are released and the first error returned). */
EG_API eg_status eg_sample_bundle(eg_ctx *ctx, int32_t n_batches, const int64_t *const *seeds,
                                  const int64_t *n_seeds, int32_t n_hops, const int32_t *fanouts,
                                  const uint64_t *rng_seeds, int32_t flags, eg_blocks **out);

/* ---- Link-prediction mini-batches (DESIGN.md §3 readings L1-L4).
 * The scheduler picks "target edges in each mini-batch" for link prediction (PAPER.md
 * P:558-560 §4.2.1; trained on all edges, §5; fanout 25, 15).
 * Batch b: positives (src[b][i], dst[b][i]), i < n_pos[b], gids of relation rel's
 * src / dst vertex types (host or device int64 arrays, read in place when device-
 * accessible, which then must stay valid until the batch resolves).  Per positive,
 * n_neg corrupted pairs keep the src and draw the dst uniformly from t(rel)'s range:
 *   dst' = off[t] + floor(w * N_t / 2^32),
 *   w = Philox4x32-10(ctr = {i, q, 0, 0x4E454721}, key = {lo32(neg_seeds[b]), hi32(..)}).word[0]
 * (SPEC S:401-404).  The seeds are the distinct endpoints in ascending gid; sampling
 * then runs exactly as eg_sample_bundle from them (block 0's dst nodes).  Flags as
 * eg_sample_bundle (EG_FEATURES, EG_ASYNC); one bundle = one CUDA-graph launch.
 * Errors: EG_EINVAL (rel out of range, n_neg outside [0, EG_MAX_NEG], n_pos < 0 or >=
 * 2^31, null arrays); EG_ERANGE (an endpoint outside its vertex type; reported when the
 * batch resolves). */
#define EG_MAX_NEG 64
EG_API eg_status eg_sample_lp_bundle(eg_ctx *ctx, int32_t n_batches, const int64_t *const *src,
                                     const int64_t *const *dst, const int64_t *n_pos, int32_t rel, int32_t n_neg,
                                     const uint64_t *neg_seeds, int32_t n_hops, const int32_t *fanouts,
                                     const uint64_t *rng_seeds, int32_t flags, eg_blocks **out);

/* The pairs of a link-prediction batch (waits if pending), as device int32 arrays of
 * local ids (index among the seeds of the endpoint's type = position in block 0's dst
 * nodes of that type): pos_src / pos_dst [n_pos], neg_src / neg_dst [n_pos * n_neg]
 * (negative q of positive i at i * n_neg + q), and the corrupted dst gids neg_dst_gid
 * (device int64 [n_pos * n_neg]).  Valid until eg_blocks_free.  EG_EINVAL for a
 * node-classification batch. */
typedef struct {
    int64_t n_pos;
    int32_t n_neg, rel;
    const int32_t *pos_src, *pos_dst, *neg_src, *neg_dst;
    const int64_t *neg_dst_gid;
} eg_lp_view;
EG_API eg_status eg_lp_view_get(const eg_blocks *blocks, eg_lp_view *out);

/* ---- Consumer step (SURVEY §8f NEXT-4 i; DESIGN.md §3 readings C1-C2): one GraphSAGE-
 * mean layer over relation `rel` of block `hop`, pre-activation (Eq. 1, P:244-246,
 * GraphSAGE P:964):  out[v] (+)= W_self x_dst[v] + W_neigh mean_{sampled in-edges u->v} x_src[u]
 * (mean over the block's sampled edges of v, multiplicity counted; 0 without any).
 *   x_src   device rows of the block's src nodes of type s(rel) (local id = row), x_dtype
 *           0 fp32 / 1 fp16 / 2 bf16, row stride ld_src elements (rows 16-B aligned);
 *           for the input layer these are exactly eg_blocks_features(s(rel)).
 *   x_dst   device rows of the dst nodes of type t(rel) (same dtype, stride ld_dst), or
 *           NULL: no self term (K = F; RGCN-style per-relation terms with EG_ACCUMULATE).
 *   w       device bf16 [H][K] row-major, K = 2F ([W_self | W_neigh]) or F.
 *   out     device fp32 [n_dst][ld_out], n_dst = |dst nodes of type t(rel)| of the block;
 *           flags & EG_ACCUMULATE adds to it.
 * Runs on the context's stream after the batch resolves; the operands are rounded to
 * bf16 for the tensor cores, accumulation is fp32.  Errors: EG_EINVAL (hop / rel out of
 * range, F outside [1, 256], H not a multiple of 16 in [16, 256], unaligned rows,
 * shared-memory budget (128 + H) * K_padded * 2 B > 200 KB). */
#define EG_ACCUMULATE 1
EG_API eg_status eg_sage_mean_layer(eg_ctx *ctx, const eg_blocks *blocks, int32_t hop, int32_t rel,
                                    const void *x_src, int32_t x_dtype, int64_t ld_src, const void *x_dst,
                                    int64_t ld_dst, int32_t F, const void *w, int32_t H, float *out,
                                    int64_t ld_out, int32_t flags);

/* Totals of a batch (waits if pending): sampled edges over all hops and relations, and
 * the input vertices (src nodes of the last block) per type (n_inputs: host [n_vt]);
 * either may be NULL. */
EG_API eg_status eg_blocks_stats(const eg_blocks *blocks, int64_t *total_edges, int64_t *n_inputs);

/* Wait for an EG_ASYNC batch; returns its status (EG_ERANGE / EG_EINVAL for bad seeds). */
EG_API eg_status eg_blocks_wait(eg_blocks *blocks);

/* Feature rows gathered by eg_sample_minibatch(EG_FEATURES) for type u (device
 * pointer, n_rows x row_bytes, valid until eg_blocks_free; NULL / 0 if the type has
 * no features or the batch was sampled without EG_FEATURES). */
EG_API eg_status eg_blocks_features(const eg_blocks *blocks, int32_t u, const void **rows, int64_t *n_rows,
                                    int64_t *row_bytes);

/* Copy the feature rows gathered in the batch's launch (EG_FEATURES) to caller memory:
 * host[u] (host array [n_vt]; NULL skips u) receives n_inputs(u) x row_bytes(u) bytes,
 * pinned host memory for an asynchronous DMA (pageable memory works, synchronously).
 * Stream-ordered on the context's stream after the batch's launch (waits for its sizes
 * first); flags & EG_ASYNC: returns after enqueueing, else synchronizes the stream.
 * EG_EINVAL: null pointers, a type without gathered rows; EG_ESTATE: orphaned handle. */
EG_API eg_status eg_blocks_copy_features(const eg_blocks *blocks, void *const *host, int32_t flags);

/* Host view of block `hop` (0 <= hop < n_hops).  Pointers stay valid until
 * eg_blocks_free. */
EG_API eg_status eg_block_view_get(const eg_blocks *blocks, int32_t hop, eg_block_view *out);

/* n_hops of a blocks handle, and the number of input vertices (src nodes of
 * the last block) of type u. */
EG_API int32_t eg_blocks_n_hops(const eg_blocks *blocks);
EG_API int64_t eg_blocks_n_inputs(const eg_blocks *blocks, int32_t u);

/* Gather the feature rows of the input vertices (src nodes of the last block):
 * out[u] (host array [n_vt]) points to n_inputs(u) x row_bytes(u) bytes, device
 * or host memory; NULL skips u.  Rows are copied verbatim in input order
 * (S:217-225); rows owned by peers are read over NVLink.  Host out pointers are
 * staged through device memory and the call synchronizes. */
EG_API eg_status eg_gather_features(eg_ctx *ctx, const eg_blocks *blocks, void *const *out);

/* Release a blocks handle (stream-ordered on the context's stream). */
EG_API eg_status eg_blocks_free(eg_blocks *blocks);

/* Destroy the context: waits for every launch still in flight, closes the peer
 * mappings, frees its state; the borrowed shard buffers are untouched.  Handles the
 * caller has not freed are orphaned: their device views become invalid, every call on
 * them returns EG_ESTATE, and eg_blocks_free only releases the handle. */
EG_API eg_status eg_destroy(eg_ctx *ctx);

/* Message of the last error on this context (thread-unsafe, never NULL). */
EG_API const char *eg_last_error(const eg_ctx *ctx);

/* Instrumentation.  When enabled, each sample/gather call records CUDA events on
 * the context's stream around its device work; eg_get_profile synchronizes and
 * returns {sample_ms_total, gather_ms_total, n_sample_calls, n_gather_calls}.
 * eg_kernel_launches returns the number of kernels this context has launched. */
EG_API eg_status eg_set_profiling(eg_ctx *ctx, int32_t enable);
EG_API eg_status eg_get_profile(eg_ctx *ctx, double out[4]);
EG_API int64_t eg_kernel_launches(const eg_ctx *ctx);

/* Tracing: with EG_TRACE=1 in the environment at eg_create, every captured batch
 * graph carries an event after each stage (seed split; per hop count, scan,
 * sample+select, bitcount, emit, relabel; reset; gather) and, while profiling is
 * enabled, finished batches accumulate per-stage device time.  Returns the number
 * of stages; entry i (if in range) is copied to name / total_ms / count. */
EG_API int32_t eg_trace_get(const eg_ctx *ctx, int32_t i, char *name, size_t name_len, double *total_ms,
                            int64_t *count);

/* Host-only helpers (no device work; usable without a GPU). */

/* What one rank publishes about its shard (no device pointers): the global schema,
 * the partition bounds, its CSC shard extents and its feature row size. */
typedef struct {
    int32_t rank, world, n_vt, n_rel;
    int64_t vt_counts[EG_MAX_VT];
    int64_t bounds[EG_MAX_VT][EG_MAX_RANKS + 1];
    int32_t rel_src_vt[EG_MAX_REL], rel_dst_vt[EG_MAX_REL];
    int64_t rel_n_local_edges[EG_MAX_REL], rel_edge_base[EG_MAX_REL], rel_max_degree[EG_MAX_REL];
    int64_t row_bytes[EG_MAX_VT];
} eg_shard_meta;

/* Check that `world` shard metas (rank order) describe ONE partition: same schema,
 * vertex counts, bounds (0 .. N_t, non-decreasing) and row sizes everywhere; rank p's
 * relation shards start at edge_base = sum of the lower ranks' edge counts.  On
 * success fills rel_edges[r] = |E_r| and rel_max_degree[r] (either may be NULL).
 * EG_EPEER (with a reason in msg, if given) otherwise.  eg_import_shards and
 * eg_attach_peer run the same check. */
EG_API eg_status eg_check_shard_metas(int32_t world, const eg_shard_meta *metas, int64_t *rel_edges,
                                      int64_t *rel_max_degree, char *msg, size_t msg_len);
/* bounds[p] = floor(p * n / world), p = 0..world. */
EG_API eg_status eg_range_bounds(int64_t n, int32_t world, int64_t *bounds);
/* Upper bound of the nodes / edges of a batch (what eg_sample_blocks allocates):
 * caps_nodes [n_vt] for the input vertices, caps_edges [n_hops][n_rel]. */
EG_API eg_status eg_batch_caps(int32_t n_vt, const int64_t *vt_counts, int32_t n_rel, const int32_t *rel_src_vt,
                        const int32_t *rel_dst_vt, const int64_t *rel_n_edges, const int64_t *rel_max_degree,
                        int64_t n_seeds, int32_t n_hops, const int32_t *fanouts, int64_t *caps_nodes,
                        int64_t *caps_edges);

#ifdef __cplusplus
}
#endif
#endif /* EGONET_H */
