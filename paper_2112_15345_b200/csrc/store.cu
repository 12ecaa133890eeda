// store.cu -- small load-time kernels of the graph/feature store.
#include "kernels.h"

namespace eg {

__global__ void max_degree_kernel(const int64_t *__restrict__ indptr, int64_t n, unsigned long long *out)
{
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = indptr[i + 1] - indptr[i];
        m = max(m, (unsigned long long)(d < 0 ? 0 : d));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

void launch_max_degree(const int64_t *indptr, int64_t n, unsigned long long *out, cudaStream_t s)
{
    if (n > 0) max_degree_kernel<<<kSMs * 4, 256, 0, s>>>(indptr, n, out);
}

}  // namespace eg
