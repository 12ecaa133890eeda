// batch.cu -- the sampling + compaction of a bundle of mini-batches, one kernel per phase.
//
//   seed split (+ sort: batches of <= 1024 seeds) | [kscan scatter compact (level 0)] |
//   for h: count | select + copy + tiny | kscan scatter compact (level h+1)
//
// Every phase kernel runs with grid.y = the batch of the bundle (each batch has its own
// HopDev / compaction state), so B mini-batches cost about what one does: at batch ~1k
// each phase is a short chain of dependent memory accesses and one batch
// alone cannot fill a B200.
//
// Design note (measured): a persistent cooperative kernel with software
// grid barriers between the phases was built and measured on B200 first; a barrier cost
// ~3 us, about a kernel boundary inside a CUDA graph, and the per-phase kernels ran at
// higher occupancy (130 vs 183 us per batch), so the per-phase form is the one kept.
#include "kernels.h"
#include "phases.cuh"
#include "compact.cuh"

namespace eg {

constexpr int kBatchThreads = 256;
constexpr int kBatchWarps = kBatchThreads / 32;

__device__ __forceinline__ uint64_t globaltimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Tracing (EG_TRACE=1): block (0, b) stamps the global timer at the start of each phase
// into batch b's counters (copied to the host with them).
__device__ __forceinline__ void stamp(const BatchDev *bd, int k)
{
    if (bd->trace && blockIdx.x == 0 && threadIdx.x == 0 && k >= 0 && k < kMaxStamps)
        reinterpret_cast<uint64_t *>(bd->hop[blockIdx.y][0].meta + kMetaStamps)[k] = globaltimer();
}

// Hop h of batch blockIdx.y; h = -1: the seeds' level (the seed split / link-prediction targets).
__device__ __forceinline__ const HopDev &hop_of(const BatchDev *bd, int h)
{
    return h < 0 ? bd->seedh[blockIdx.y] : bd->hop[blockIdx.y][h];
}

__global__ void __launch_bounds__(kBatchThreads) k_lp_mark(const __grid_constant__ GraphDev g,
                                                           const BatchDev *__restrict__ bd)
{
    stamp(bd, 0);
    phase_lp_mark(g, bd->seedh[blockIdx.y], bd->lpd[blockIdx.y], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(1024) k_seed(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd)
{
    stamp(bd, 0);
    phase_seed_split(g, bd->seedh[blockIdx.y], bd->seeds[blockIdx.y], bd->seed_sort != 0);
}

#ifndef EG_COUNT_MINB
#define EG_COUNT_MINB 4
#endif
#ifndef EG_COPY_MINB
#define EG_COPY_MINB 4
#endif
#ifndef EG_SCATTER_MINB
#define EG_SCATTER_MINB 6
#endif
__global__ void __launch_bounds__(kCountThreads, EG_COUNT_MINB) k_count(const __grid_constant__ GraphDev g,
                                                         const BatchDev *__restrict__ bd, int h)
{
    stamp(bd, 4 + 8 * h);
    phase_count(g, bd->hop[blockIdx.y][h]);
}

#ifndef EG_SELECT_MIN_BLOCKS
#define EG_SELECT_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kBatchThreads, EG_SELECT_MIN_BLOCKS) k_select(const __grid_constant__ GraphDev g,
                                                             const BatchDev *__restrict__ bd, int h)
{
    __shared__ uint64_t s_cand[kBatchWarps][kSelCap];
    stamp(bd, 6 + 8 * h);
    phase_select(g, bd->hop[blockIdx.y][h], blockIdx.x, gridDim.x, s_cand[threadIdx.x >> 5]);
}

__global__ void __launch_bounds__(kBatchThreads, EG_COPY_MINB) k_copy(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    stamp(bd, 7 + 8 * h);
    phase_copy(g, bd->hop[blockIdx.y][h], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(kBatchThreads, 4) k_tiny(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    stamp(bd, 8 + 8 * h);
    phase_tiny(g, bd->hop[blockIdx.y][h], blockIdx.x, gridDim.x);
}

// Compaction of level h + 1 (the keys produced by hop h; h = -1: the seeds' level).
__global__ void __launch_bounds__(kScanThreads) k_kscan(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    stamp(bd, 1 + 8 * (h + 1));
    phase_kscan(g, hop_of(bd, h));
}

__global__ void __launch_bounds__(kBatchThreads, EG_SCATTER_MINB) k_scatter(const __grid_constant__ GraphDev g,
                                                           const BatchDev *__restrict__ bd, int h)
{
    stamp(bd, 2 + 8 * (h + 1));
    phase_scatter(g, hop_of(bd, h), bd->lpd[blockIdx.y], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(kBatchThreads) k_compact_count(const __grid_constant__ GraphDev g,
                                                                 const BatchDev *__restrict__ bd, int h)
{
    __shared__ CompactSmem sm[kBatchWarps];
    stamp(bd, 3 + 8 * (h + 1));
    phase_compact_count(g, hop_of(bd, h), sm, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(kScanThreads) k_tscan(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    phase_tscan(g, hop_of(bd, h));
}

__global__ void __launch_bounds__(kBatchThreads) k_compact_emit(const __grid_constant__ GraphDev g,
                                                                const BatchDev *__restrict__ bd, int h)
{
    __shared__ CompactSmem sm[kBatchWarps];
    phase_compact_emit(g, hop_of(bd, h), bd->lpd[blockIdx.y], sm, blockIdx.x, gridDim.x);
}

int launch_batch(const GraphDev &g, const BatchDev *bd_dev, int n_hops, const int32_t *count_tiles, int B,
                 cudaStream_t s, const Fork &fk, bool serial, bool lp, bool seed_sort)
{
    // blocks per batch: about one wave of the chip in total
    const int per = (kSMs * 8 + B - 1) / B;
    const int samp = (kSMs * 4 + B - 1) / B;
    int nk = 0;
    auto compaction = [&](int h) {   // level h + 1
        k_kscan<<<dim3((g.nb + kScanTile - 1) / kScanTile, B), kScanThreads, 0, s>>>(g, bd_dev, h);
        k_scatter<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
        k_compact_count<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
        k_tscan<<<dim3((g.nb + kScanTile - 1) / kScanTile, B), kScanThreads, 0, s>>>(g, bd_dev, h);
        k_compact_emit<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
        nk += 5;
    };
    if (lp) {   // link prediction: targets -> endpoint keys -> seeds + pairs
        k_lp_mark<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev);
    } else {
        k_seed<<<dim3(1, B), 1024, 0, s>>>(g, bd_dev);
    }
    ++nk;
    if (!seed_sort) compaction(-1);   // else the seed split sorted the seeds itself
    for (int h = 0; h < n_hops; ++h) {
        const int cb = count_tiles[h] < per ? count_tiles[h] : per;   // count: blocks take tiles by ticket
        k_count<<<dim3(cb, B), kCountThreads, 0, s>>>(g, bd_dev, h);
        // selections and full-neighbourhood copies write disjoint slots: two graph branches
        // (EG_TRACE=1 serialises them so that each gets its own phase stamp)
        if (serial) {
            k_select<<<dim3(samp, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
            k_copy<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
            k_tiny<<<dim3(per, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
        } else {
            cudaEventRecord(fk.fork, s);
            cudaStreamWaitEvent(fk.side, fk.fork, 0);
            k_copy<<<dim3(per, B), kBatchThreads, 0, fk.side>>>(g, bd_dev, h);
            k_tiny<<<dim3(per, B), kBatchThreads, 0, fk.side>>>(g, bd_dev, h);
            cudaEventRecord(fk.join, fk.side);
            k_select<<<dim3(samp, B), kBatchThreads, 0, s>>>(g, bd_dev, h);
            cudaStreamWaitEvent(s, fk.join, 0);
        }
        nk += 4;
        compaction(h);
    }
    return nk;
}

}  // namespace eg
