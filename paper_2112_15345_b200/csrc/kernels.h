// kernels.h -- host launchers of the egonet kernels (internal).
#pragma once
#include "common.cuh"

namespace eg {

// sample.cu
void launch_seed_split(const GraphDev &g, const int64_t *seeds, const HopDev &hd, cudaStream_t s);
void launch_count(const GraphDev &g, const HopDev &hd, cudaStream_t s);
void launch_scan(const GraphDev &g, const HopDev &hd, cudaStream_t s);
void launch_sample(const GraphDev &g, const HopDev &hd, cudaStream_t s);

// compact.cu
void launch_mark(const GraphDev &g, const HopDev &hd, cudaStream_t s);
void launch_bitcount(const GraphDev &g, const HopDev &hd, int32_t n_chunks, cudaStream_t s);
void launch_emit(const GraphDev &g, const HopDev &hd, int32_t n_chunks, cudaStream_t s);
void launch_relabel(const GraphDev &g, const HopDev &hd, cudaStream_t s);
void launch_reset(const GraphDev &g, const HopDev &hd, int32_t level, cudaStream_t s);

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
