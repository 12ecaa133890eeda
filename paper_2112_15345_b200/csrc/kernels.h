// kernels.h -- host launchers of the egonet kernels (internal).
#pragma once
#include "common.cuh"

namespace eg {

// batch.cu: sampling + compaction of a whole batch (one persistent kernel)
struct BatchDev {
    int32_t n_hops, n_chunks, trace, _pad;
    const int64_t *seeds;
    uint32_t *bar;                 // grid barrier {count, generation}, zero-initialised
    HopDev hop[EG_MAX_HOPS];
};
int launch_batch(const GraphDev &g, const BatchDev *bd_dev, int n_hops, int n_chunks, cudaStream_t s);
int batch_grid();

// gather.cu
struct GatherDev {
    uint8_t *out[EG_MAX_VT];
    const int64_t *nodes[EG_MAX_VT];
    const int32_t *meta;
    int32_t level;
};
void launch_gather(const GraphDev &g, const FeatDev &f, const GatherDev &gd, cudaStream_t s);

// store.cu
void launch_max_degree(const int64_t *indptr, int64_t n, unsigned long long *out, cudaStream_t s);

}  // namespace eg
