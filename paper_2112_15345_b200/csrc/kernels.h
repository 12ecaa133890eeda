// kernels.h -- host launchers of the egonet kernels (internal).
#pragma once
#include "common.cuh"

namespace eg {

// A bundle of up to kMaxBundle mini-batches runs as one launch of each phase kernel
// (grid.y = batch of the bundle) and one gather: the paper's bundling of the sampling
// of several mini-batches.
constexpr int kMaxBundle = 16;

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
    int32_t n_hops, n_chunks, trace, B;
    int32_t lp;                            // link-prediction batches (seeds from targets)
    const int64_t *seeds[kMaxBundle];
    HopDev hop[kMaxBundle][EG_MAX_HOPS];
    HopDev lph[kMaxBundle];                // LP seed compaction ("hop -1")
    LpDev lpd[kMaxBundle];
};

// A side stream + two events to fork / join independent kernels inside a capture.
struct Fork {
    cudaStream_t side;
    cudaEvent_t fork, join;
};

// batch.cu: enqueue the sampling + compaction of the B batches of bd_dev (capturable);
// returns the number of kernels.
// lp >= 0: link-prediction batches, seed compaction variant lp (1 = sparse).
int launch_batch(const GraphDev &g, const BatchDev *bd_dev, int n_hops, const int32_t *scan_blocks,
                 const int32_t *sparse_hop, int n_chunks, int B, cudaStream_t s,
                 const Fork &fk, bool serial, int lp);

// gather.cu
void launch_gather(const GraphDev &g, const FeatDev &f, const GatherSet &gs, cudaStream_t s);

// store.cu
void launch_max_degree(const int64_t *indptr, int64_t n, unsigned long long *out, cudaStream_t s);

}  // namespace eg
