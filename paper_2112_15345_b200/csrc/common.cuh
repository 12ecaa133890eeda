// common.cuh -- device-side descriptors and primitives of the egonet sm_100a path.
// Product code: shares nothing with oracle/ (see DESIGN.md §1).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/egonet.h"

// Bounds-checked build (paper_2112_15345_b200/build.py --check -> libegonet_check.so,
// loaded with EG_LIB=...): every EG_DCHECK traps with the failing line.  compute-sanitizer
// is not available on the GPU pool used here (profiles/r02/sanitize/), so the GPU suite is
// run against this build instead.
#ifndef EG_CHECK
#define EG_CHECK 0
#endif
#if EG_CHECK
#include <cstdio>
#define EG_DCHECK(c)                                                                                \
    do {                                                                                            \
        if (!(c)) {                                                                                 \
            printf("EG_CHECK failed: %s:%d: %s (block %d,%d thread %d)\n", __FILE__, __LINE__, #c,     \
                   blockIdx.x, blockIdx.y, threadIdx.x);                                            \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define EG_DCHECK(c) do { } while (0)
#endif

namespace eg {

constexpr int kWarp = 32;
constexpr int kSMs = 148;                 // B200
// Compaction buckets (compact.cuh): each vertex type's id range is cut into fine buckets of
// 2^bshift consecutive gids, bshift in [12, kMaxBucketShift] chosen at load so that a graph
// has at most ~2^14 buckets (C4: 2^13 gids, 13.6k buckets; kMinBucketShift is the smallest an
// A/B override may set).  A bucket's bitmap is
// 2^bshift / 32 words, at most 8 per lane of a warp.
constexpr int kMinBucketShift = 10;
constexpr int kMaxBucketShift = 13;
constexpr int64_t kMaxBuckets = (int64_t)1 << 17;
constexpr int kScanTile = 4096;                                   // buckets per kscan CTA (512 threads x 8)
constexpr int kMaxScanTiles = (int)(kMaxBuckets / kScanTile);     // 32: one warp looks back over all
// Count tiles (single pass with a decoupled look-back per relation): kCountThreads threads
// x kCountItems consecutive dst items each.
constexpr int kCountThreads = 256;
#ifndef EG_COUNT_ITEMS
#define EG_COUNT_ITEMS 4
#endif
constexpr int kCountItems = EG_COUNT_ITEMS;
constexpr int kCountTile = kCountThreads * kCountItems;
constexpr int kSelCap = 512;              // candidate slots per warp (selection)
constexpr int kSelMaxK = 112;             // fast selection path for k <= this
constexpr int kTinyD = 64;                // selections with d <= this: 8 lanes per item (phase_tiny)
constexpr int kTinyD16 = 16;              // ... with d <= this: 4 lanes per item
// Heavy items (d > kHeavyD, k <= kHeavyMaxK) are split into tasks of kHeavyChunk keys
// sampled by different warps; their candidates meet in a per-item buffer.
constexpr int kHeavyD = 2048;
constexpr int kHeavyChunk = 1024;
constexpr int kHeavyMaxK = 48;
constexpr int kHeavyCap = 512;            // candidate slots per heavy item
constexpr int kMinHeavy = 256;            // heavy items per (batch, hop): at least this, more for large
                                          // frontiers (HopDev::max_heavy); overflow -> warp per item
constexpr int kHeavyTasksPerItem = (1 << 20) / kHeavyChunk + 1;   // d <= 2^20 (generator Dmax)
// Largest in-degree a relation may have (eg_load_partition rejects more): heavy tasks are
// encoded as (item << 16) | chunk, chunk < 2^16 chunks of kHeavyChunk keys.
constexpr int64_t kMaxInDegree = (int64_t)kHeavyChunk << 16;

// Error bits written by kernels into meta[kMetaErr].
enum : int32_t { kErrSeedRange = 1, kErrSeedDup = 2, kErrCapacity = 4 };

// One relation as the kernels see it: per owner rank, the CSC shard pointers
// (own shard or a peer's, mapped over NVLink).
struct RelDev {
    const int64_t *indptr[EG_MAX_RANKS];
    const int32_t *indices[EG_MAX_RANKS];
    int64_t edge_base[EG_MAX_RANKS];
    int32_t src_vt, dst_vt;
};

struct GraphDev {
    int32_t n_vt, n_rel, world, rank;
    int64_t off[EG_MAX_VT + 1];                       // gid = off[t] + tid
    int64_t bounds[EG_MAX_VT][EG_MAX_RANKS + 1];      // owned tid ranges per rank
    int64_t bbase[EG_MAX_VT + 1];                     // first compaction bucket of each type
    int32_t bshift;                                   // log2 of the gids per bucket
    int32_t nb;                                       // buckets in total (= bbase[n_vt])
    int32_t compact_bitmap;                           // EG_COMPACT=bitmap: every bucket a task, bitmap path
    RelDev rel[EG_MAX_REL];
};

struct FeatDev {
    const uint8_t *rows[EG_MAX_VT][EG_MAX_RANKS];
    int64_t row_bytes[EG_MAX_VT];
    const uint8_t *replica[EG_MAX_VT];   // full local table of a replicated type (tid-indexed), or null
};


// Device counters of one batch (int32 slots in one small array).
//   nodes(l, u): |level l of type u|, l = 0 seeds, l = h+1 src nodes of block h
//   nnz(h, r):   edges of relation r in block h
constexpr int kMetaNodes = 0;
constexpr int kMetaNnz = kMetaNodes + (EG_MAX_HOPS + 1) * EG_MAX_VT;
constexpr int kMetaSel = kMetaNnz + EG_MAX_HOPS * EG_MAX_REL;   // selection-queue length per hop
constexpr int kMetaSelNext = kMetaSel + EG_MAX_HOPS;             // dynamic fetch counter per hop
constexpr int kMetaHeavy = kMetaSelNext + EG_MAX_HOPS;           // heavy items per hop
constexpr int kMetaHeavyQ = kMetaHeavy + EG_MAX_HOPS;            // heavy tasks per hop
constexpr int kMetaHeavyNext = kMetaHeavyQ + EG_MAX_HOPS;        // dynamic fetch counter per hop
constexpr int kMetaTiny = kMetaHeavyNext + EG_MAX_HOPS;         // tiny selection items per hop
constexpr int kMetaTinyNext = kMetaTiny + EG_MAX_HOPS;            // dynamic fetch counter per hop
constexpr int kMetaCopy = kMetaTinyNext + EG_MAX_HOPS;            // full-neighbourhood items per hop
constexpr int kMetaTiny16 = kMetaCopy + EG_MAX_HOPS;              // tiny selection items with d <= 16 per hop
constexpr int kMetaCntTicket = kMetaTiny16 + EG_MAX_HOPS;         // count tile tickets per hop
constexpr int kMetaTasks = kMetaCntTicket + EG_MAX_HOPS;          // compaction tasks per level (0..L)
constexpr int kMetaTicket = kMetaTasks + EG_MAX_HOPS + 1;         // compaction task tickets per level
constexpr int kMetaKTicket = kMetaTicket + EG_MAX_HOPS + 1;       // kscan tile tickets per level
constexpr int kMetaErr = kMetaKTicket + EG_MAX_HOPS + 1;
constexpr int kMetaStamps = (kMetaErr + 8 + 1) & ~1;       // 64-bit phase timestamps (tracing), 8-B aligned
constexpr int kMaxStamps = 80;
constexpr int kMetaSize = kMetaStamps + 2 * kMaxStamps;

// Per-batch launch parameters copied H2D at the start of every launch (kDyn u64):
//   [0] rng_seed  [1] n_seeds (node classification) / n_pos (link prediction)
//   [2] seeds / positive src pointer when device-accessible, else 0 (staged copy)
//   [3] positive dst pointer (LP)  [4] neg_seed (LP)  [5] relation (LP)
constexpr int kDyn = 8;

// Link-prediction targets of one batch (NEXT-3, DESIGN.md §3 L1-L4).
struct LpDev {
    int32_t n_neg;
    int64_t cap_pos;              // pairs layout stride
    const int64_t *src_stage;     // staged positives (pageable host input)
    const int64_t *dst_stage;
    int64_t *neg;                 // [cap_pos * n_neg] corrupted dst gids
    int32_t *pairs;               // [pos_src cap][pos_dst cap][neg_src cap*n][neg_dst cap*n], local ids
};

// Compaction modes (compact.cuh): the keys of a level are
//   kModeHop    the sampled sources of hop h (level h+1): new ones are appended, every edge relabelled;
//   kModeSeeds  the seeds (level 0, node classification): positions given by the seed split;
//   kModeLp     the link-prediction endpoints (level 0): distinct ones become the seeds, pairs relabelled.
enum : int32_t { kModeHop = 0, kModeSeeds = 1, kModeLp = 2 };

// Batch-local compaction state (one per batch; sized by the batch's caps, not by the graph).
struct CompactDev {
    uint32_t *kcnt;                  // [nb, padded to kScanTile] keys per bucket (counted by the
                                     // marking kernels, cleared by kscan)
    uint32_t *mcnt;                  // [same] members per bucket for the next level (zeroed by kscan)
    unsigned long long *tlb;         // [levels][3][kMaxScanTiles] kscan / tscan tile look-back words (zeroed per launch)
    uint32_t *tnew;                  // [nb] per task: new entries of the member list, then their exclusive prefix
    int32_t *ftask;                  // [EG_MAX_VT] first task of each vertex type
    uint32_t *kofs, *mofs;           // [nb + 1] exclusive prefixes of kcnt / mcnt
    uint32_t *kcur;                  // [nb] scatter cursors: end of each bucket's keys in elems
    uint32_t *tstart;                // [nb + 1] first bucket of each compaction task
    unsigned long long *elems;       // [cap_elems] the level's members + keys, bucket by bucket (compact.cuh)
    uint32_t *mg[2];                 // members (gids of the batch so far) sorted by gid, ping-pong by level
    int32_t *mp[2];                  // their positions in their type's node array
    int32_t cap_elems;
    int32_t cap_members;             // entries of mg / mp (bounds checks)
    int32_t nb_pad;                  // entries of the bucket arrays (bounds checks)
};

// A dst item of a hop, as the count phase hands it to the sampling kernels (queues of
// full-neighbourhood copies and of selections): everything they need in one 24-B record.
struct QEntry {
    int64_t ib;      // (owner << 56) | CSC row start in the owner's shard
    int32_t pos0;    // its first output slot in the block (= block indptr)
    int32_t d;       // in-degree
    int32_t v;       // gid of the dst (Philox counter words)
    int32_t r;       // relation
};

// Everything a hop's kernels touch.
struct HopDev {
    int32_t h;
    int32_t fanout[EG_MAX_REL];
    int64_t *nodes[EG_MAX_VT];       // cumulative node array per type
    int32_t *indptr[EG_MAX_REL];     // block CSC per relation
    int32_t *indices[EG_MAX_REL];
    int64_t *eids[EG_MAX_REL];
    uint32_t *src[EG_MAX_REL];       // sampled src gids (scratch)
    int32_t *meta;                   // batch counters

    int32_t max_heavy;               // heavy item slots
    int32_t max_heavy_tasks;         // heavy task slots
    CompactDev cd;                   // the batch's compaction state
    int32_t mode;                    // compaction mode of the level this hop produces (kMode*)
    int32_t last;                    // 1: the last level (no member list for a next level)
    const uint64_t *dyn;             // device: {rng_seed, n_seeds} of the batch
    QEntry *selq;                    // items that need a selection (d > k); tiny ones (d <= 64) from the top
    QEntry *copyq;                   // full-neighbourhood items (0 < d <= k, or k = -1)
    QEntry *tinyq16;                 // selections with d <= kTinyD16 (from the top)
    int32_t selq_cap;                // slots of selq (= of copyq)
    unsigned long long *clb;         // count tiles' look-back words (zeroed per launch)
    QEntry *heavy_items;             // [max_heavy]
    uint32_t *heavy_cnt;             // [max_heavy] candidates found
    uint32_t *heavy_done;            // [max_heavy] finished tasks
    uint64_t *heavy_cand;            // [max_heavy][kHeavyCap] (key << 32) | j
    uint32_t *heavyq;                // tasks: (heavy item << 16) | chunk
    int32_t cap_nodes[EG_MAX_VT];    // capacity of nodes[u]
};

__device__ __forceinline__ int32_t *meta_nodes(int32_t *meta, int l) { return meta + kMetaNodes + l * EG_MAX_VT; }

// Compaction bucket of gid (vertex type u): buckets are type-aligned, 2^bshift gids each.
__device__ __forceinline__ int64_t bucket_of(const GraphDev &g, int u, int64_t gid)
{
    return g.bbase[u] + ((gid - g.off[u]) >> g.bshift);
}
__device__ __forceinline__ int32_t *meta_nnz(int32_t *meta, int h) { return meta + kMetaNnz + h * EG_MAX_REL; }

// |F_h[u]| before hop h's compaction; the link-prediction seed compaction runs as
// "hop -1" over an empty frontier.
__device__ const int32_t kNoNodes[EG_MAX_VT] = {0, 0, 0, 0, 0, 0, 0, 0};
__device__ __forceinline__ const int32_t *nodes_before(const HopDev &hd)
{
    return hd.h < 0 ? kNoNodes : meta_nodes(hd.meta, hd.h);
}

// ------------------------------------------------------------------ ids / partition

__device__ __forceinline__ int owner_of(const GraphDev &g, int t, int64_t tid)
{
    int p = 0;
    while (p < g.world - 1 && tid >= g.bounds[t][p + 1]) ++p;
    return p;
}

// Source row of (type u, type-local id tid): the local replica of a replicated type,
// else the owner's shard (local HBM, or a peer's over NVLink).
__device__ __forceinline__ const uint8_t *feature_row(const GraphDev &g, const FeatDev &f, int u, int64_t tid)
{
    EG_DCHECK(tid >= 0 && tid < g.off[u + 1] - g.off[u]);
    if (f.replica[u]) return f.replica[u] + tid * f.row_bytes[u];
    const int p = owner_of(g, u, tid);
    return f.rows[u][p] + (tid - g.bounds[u][p]) * f.row_bytes[u];
}

// ------------------------------------------------------------------ warp / block scans

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide exclusive scan; returns the exclusive prefix, *total = block sum.
// `sh` needs blockDim.x/32 + 1 slots.  All threads must call.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *sh, T *total)
{
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane_id() == 31) sh[w] = inc;
    __syncthreads();
    if (w == 0) {
        T x = lane_id() < nw ? sh[lane_id()] : T(0);
        T xi = warp_incl_scan(x);
        if (lane_id() < nw) sh[lane_id()] = xi - x;
        if (lane_id() == nw - 1) sh[nw] = xi;
    }
    __syncthreads();
    T res = sh[w] + inc - v;
    *total = sh[nw];
    __syncthreads();
    return res;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T *sh)
{
    T t;
    block_excl_scan(v, sh, &t);
    return t;
}

// ------------------------------------------------------------------ Philox4x32-10
// Counter-based generator of Salmon et al. (SC'11), 10 rounds.  Used only through
// key32: ctr = {j>>2, lo32(v), hi32(v), (h<<16)|r}, key = seed.

__device__ __forceinline__ void philox4x32_10(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3,
                                              uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// ------------------------------------------------------------------ spin guard

// Call once per iteration of a spin-wait on another CTA's publication: after ~2 s the
// kernel traps (an error the host reports) instead of hanging the GPU.
struct SpinGuard {
    uint32_t it = 0;
    uint64_t t0 = 0;
    __device__ __forceinline__ void step()
    {
        if ((++it & 1023) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (!t0) t0 = t;
            else if (t - t0 > 2000000000ull) __trap();
        }
    }
};

// ------------------------------------------------------------------ memory helpers

__device__ __forceinline__ int4 ld_nc_v4(const void *p)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(void *p, const int4 &v)
{
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1, %2, %3, %4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

}  // namespace eg
