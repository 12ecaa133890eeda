// batch.cu -- one mini-batch's sampling + compaction as ONE persistent kernel.
//
// The hot path of a batch is a chain of short, dependent, latency-bound phases
// ("at batch ~1k it is latency-bound").  As separate kernels each costs
// a launch + ramp + drain (~4-5 us on B200 even inside a CUDA graph).  Here the
// grid is sized to the resident capacity (cooperative launch: every block is
// co-resident), each block loops over its share of each phase, and phases are
// separated by a software grid barrier (one atomic per block, ~1 us).
//
//   seed_split | for h: count(+relabel h-1) | scan | sample | bitcount | emit | ... | relabel | reset
//
// The same phase functions also run as one kernel per phase -- the default, since
// measured on B200 (C2) the per-phase kernels were faster (130 vs 183 us per batch:
// higher occupancy for the thread-parallel phases, and a grid barrier costs about
// as much as a kernel boundary in a graph) and let concurrent batches share the GPU.
// EG_MODE=mega selects the persistent kernel.
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "phases.cuh"

namespace eg {

constexpr int kBatchThreads = 256;
constexpr int kBatchWarps = kBatchThreads / 32;

// Sense-free generation barrier over all blocks of a co-resident grid.  The fence
// after the release also invalidates this SM's L1 (CCTL.IVALL on sm_100), so the
// next phase reads what other blocks wrote.
__device__ __forceinline__ void grid_barrier(uint32_t *bar, uint32_t nb)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t *gen = bar + 1;
        const uint32_t g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nb - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g0) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ uint64_t globaltimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Tracing: block 0 stamps the global timer after every barrier into the batch
// counters (copied to the host with them); phase k lasted stamp[k+1] - stamp[k].
__device__ __forceinline__ void stamp(const BatchDev *bd, int &k)
{
    if (bd->trace && blockIdx.x == 0 && threadIdx.x == 0 && k < kMaxStamps)
        reinterpret_cast<uint64_t *>(bd->hop[0].meta + kMetaStamps)[k] = globaltimer();
    ++k;
}

__global__ void __launch_bounds__(kBatchThreads, 3) batch_kernel(const __grid_constant__ GraphDev g,
                                                                 const BatchDev *__restrict__ bd)
{
    __shared__ uint64_t s_cand[kBatchWarps][kSelCap];
    const int bid = blockIdx.x, nb = gridDim.x;
    uint32_t *bar = bd->bar;
    const int L = bd->n_hops;
    const int32_t n_groups = (bd->n_chunks + kGroupChunks - 1) / kGroupChunks;
    int k = 0;
    stamp(bd, k);
    if (bid == 0) phase_seed_split(g, bd->hop[0], bd->seeds);
    grid_barrier(bar, nb);
    stamp(bd, k);
    for (int h = 0; h < L; ++h) {
        const HopDev &hd = bd->hop[h];
        phase_count(g, hd, bid, nb);
        if (h > 0) phase_relabel(g, bd->hop[h - 1], bid, nb);
        grid_barrier(bar, nb);
        stamp(bd, k);
        phase_scan(g, hd, bid, nb, n_groups);
        grid_barrier(bar, nb);
        stamp(bd, k);
        phase_sample(g, hd, bid, nb, s_cand[threadIdx.x >> 5]);
        grid_barrier(bar, nb);
        stamp(bd, k);
        phase_bitcount(hd, bid, nb, bd->n_chunks);
        grid_barrier(bar, nb);
        stamp(bd, k);
        phase_emit(g, hd, bid, nb, bd->n_chunks);
        grid_barrier(bar, nb);
        stamp(bd, k);
    }
    phase_relabel(g, bd->hop[L - 1], bid, nb);
    grid_barrier(bar, nb);
    stamp(bd, k);
    phase_reset(g, bd->hop[L - 1], L, bid, nb);
}

// ---------------------------------------------------------------------------- per-phase kernels

__global__ void __launch_bounds__(kBatchThreads) k_seed(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd)
{
    phase_seed_split(g, bd->hop[0], bd->seeds);
}

__global__ void __launch_bounds__(kBatchThreads) k_count(const __grid_constant__ GraphDev g,
                                                         const BatchDev *__restrict__ bd, int h)
{
    phase_count(g, bd->hop[h], blockIdx.x, gridDim.x);
    if (h > 0) phase_relabel(g, bd->hop[h - 1], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(kBatchThreads) k_scan(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    phase_scan(g, bd->hop[h], blockIdx.x, gridDim.x, (bd->n_chunks + kGroupChunks - 1) / kGroupChunks);
}

__global__ void __launch_bounds__(kBatchThreads, 2) k_sample(const __grid_constant__ GraphDev g,
                                                             const BatchDev *__restrict__ bd, int h)
{
    __shared__ uint64_t s_cand[kBatchWarps][kSelCap];
    phase_sample(g, bd->hop[h], blockIdx.x, gridDim.x, s_cand[threadIdx.x >> 5]);
}

__global__ void __launch_bounds__(kBatchThreads) k_bitcount(const BatchDev *__restrict__ bd, int h)
{
    phase_bitcount(bd->hop[h], blockIdx.x, gridDim.x, bd->n_chunks);
}

__global__ void __launch_bounds__(kBatchThreads) k_emit(const __grid_constant__ GraphDev g,
                                                        const BatchDev *__restrict__ bd, int h)
{
    phase_emit(g, bd->hop[h], blockIdx.x, gridDim.x, bd->n_chunks);
}

__global__ void __launch_bounds__(kBatchThreads) k_relabel(const __grid_constant__ GraphDev g,
                                                           const BatchDev *__restrict__ bd, int h)
{
    phase_relabel(g, bd->hop[h], blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(kBatchThreads) k_reset(const __grid_constant__ GraphDev g,
                                                         const BatchDev *__restrict__ bd)
{
    phase_reset(g, bd->hop[bd->n_hops - 1], bd->n_hops, blockIdx.x, gridDim.x);
}

static int batch_mode()
{
    static int mode = -1;
    if (mode < 0) {
        const char *e = getenv("EG_MODE");
        mode = (e && !strcmp(e, "mega")) ? 0 : 1;   // default: one kernel per phase
    }
    return mode;
}

int batch_grid()
{
    static int blocks = 0;
    if (!blocks) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batch_kernel, kBatchThreads, 0);
        int dev = 0, sms = kSMs;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        blocks = sms * (per_sm > 0 ? per_sm : 1);
    }
    return blocks;
}

// Enqueue the batch on stream s (capturable).  Returns the number of kernels.
int launch_batch(const GraphDev &g, const BatchDev *bd_dev, int n_hops, int n_chunks, cudaStream_t s)
{
    if (batch_mode() == 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(batch_grid());
        cfg.blockDim = dim3(kBatchThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, batch_kernel, g, bd_dev);
        return 1;
    }
    const int wide = kSMs * 8;
    int nk = 0;
    k_seed<<<1, kBatchThreads, 0, s>>>(g, bd_dev);
    ++nk;
    for (int h = 0; h < n_hops; ++h) {
        k_count<<<wide, kBatchThreads, 0, s>>>(g, bd_dev, h);
        k_scan<<<wide, kBatchThreads, 0, s>>>(g, bd_dev, h);
        k_sample<<<kSMs * 4, kBatchThreads, 0, s>>>(g, bd_dev, h);
        k_bitcount<<<n_chunks, kBatchThreads, 0, s>>>(bd_dev, h);
        k_emit<<<n_chunks, kBatchThreads, 0, s>>>(g, bd_dev, h);
        nk += 5;
    }
    k_relabel<<<wide, kBatchThreads, 0, s>>>(g, bd_dev, n_hops - 1);
    k_reset<<<kSMs * 4, kBatchThreads, 0, s>>>(g, bd_dev);
    return nk + 2;
}

}  // namespace eg
