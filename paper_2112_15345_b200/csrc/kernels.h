// kernels.h -- host launchers of the egonet kernels (internal).
#pragma once
#include <cuda.h>   // CUtensorMap (the maps are encoded through the runtime's driver entry point)

#include "common.cuh"

namespace eg {

// A bundle of up to kMaxBundle mini-batches runs as one launch of each phase kernel
// (grid.y = batch of the bundle) and one gather: the paper's bundling of the sampling
// of several mini-batches.
#ifndef EG_MAX_BUNDLE
#define EG_MAX_BUNDLE 32
#endif
constexpr int kMaxBundle = EG_MAX_BUNDLE;

struct GatherDev {
    uint8_t *out[EG_MAX_VT];
    const int64_t *nodes[EG_MAX_VT];
    const int32_t *meta;
    int32_t level;
};

// The gathers of one launch: batch b of the bundle is b[b] (kernel parameter).
struct GatherSet {
    int32_t nb;
    GatherDev b[kMaxBundle];
};

struct BatchDev {
    int32_t n_hops, trace, B;
    int32_t lp;                            // link-prediction batches (seeds from targets)
    int32_t seed_sort;                     // the seed split sorts the seeds (<= 1024 per batch)
    const int64_t *seeds[kMaxBundle];
    HopDev hop[kMaxBundle][EG_MAX_HOPS];
    HopDev seedh[kMaxBundle];              // the seeds' level ("hop -1": seed split + level-0 compaction)
    LpDev lpd[kMaxBundle];
};

// A side stream + two events to fork / join independent kernels inside a capture.
struct Fork {
    cudaStream_t side;
    cudaEvent_t fork, join;
};

// batch.cu: enqueue the sampling + compaction of the B batches of bd_dev (capturable);
// returns the number of kernels.  lp: link-prediction batches (seeds from targets).
int launch_batch(const GraphDev &g, const BatchDev *bd_dev, int n_hops, const int32_t *count_tiles, int B,
                 cudaStream_t s, const Fork &fk, bool serial, bool lp, bool seed_sort);

// TMA tensor maps of the feature tables the gather reads with cp.async.bulk.tensor
// tile::gather4 (four rows per TMA operation): per vertex type and owner rank one 2-D map
// over that owner's table ([n_rows][row_bytes / 4] u32, box {row_bytes / 4, 1}) -- the own
// shard, the IPC-mapped peer shards (read over NVLink), or, for a type whose full table is
// on this GPU (world 1, a replica), one map over it (owner 0, rows by type-local id).
// grp[u]: the type's rows are staged in 4-row groups (every owner has a map); a group whose
// four rows span two owners is fetched by per-row copies into the same layout.
struct __align__(64) GatherMaps {
    CUtensorMap map[EG_MAX_VT][EG_MAX_RANKS];
    int32_t grp[EG_MAX_VT];
    int32_t whole[EG_MAX_VT];   // one map over the full table (owner 0)
};

// gather.cu
// mode: 0 TMA, 1 LDG, 2 automatic (EG_GATHER=tma|ldg|auto, read at eg_create).
// Returns the kernel used: 0 gather_tma_kernel (gather4 / bulk copies), 1 gather_ldg_kernel
int launch_gather(const GraphDev &g, const FeatDev &f, const GatherSet &gs, const GatherMaps &m, cudaStream_t s,
                  int mode);

// sage.cu: one GraphSAGE-mean layer over a block relation on the tensor cores (NEXT-4 i).
struct SageArgs {
    CUtensorMap wmap;           // W as a [H][parts][F] bf16 view (3-D, SWIZZLE_128B boxes {64, 1, H}), if w_tma
    int32_t w_tma;              // 1: W staged by the TMA (F % 8 == 0); 0: by the warps
    const int32_t *indptr;      // block CSC over the dst vertices (n_dst + 1)
    const int32_t *indices;     // local src ids
    const void *x_src;          // [n_src][ld_src] input rows of the relation's src nodes
    const void *x_dst;          // [n_dst][ld_dst] input rows of the dst nodes, or null (no self term)
    int64_t ld_src, ld_dst;     // row strides in elements
    const void *w;              // bf16 [H][K], K = (x_dst ? 2F : F): [W_self | W_neigh]
    float *out;                 // [n_dst][ld_out] fp32
    int64_t ld_out;
    int32_t n_dst, F, H, accumulate;
    uint32_t tmem_cols;         // power of two >= max(32, H)
};
cudaError_t launch_sage(const SageArgs &a, int x_dtype, cudaStream_t s);   // x_dtype 0 f32, 1 f16, 2 bf16
size_t sage_smem_bytes(int F, int H, bool self_term);

// store.cu
void launch_max_degree(const int64_t *indptr, int64_t n, unsigned long long *out, cudaStream_t s);

}  // namespace eg
