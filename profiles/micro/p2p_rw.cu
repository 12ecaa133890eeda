// NVLink peer read vs peer write bandwidth between two GPUs of one process
// (context for the multi-GPU gather design).  nvcc -O3 -arch=sm_100a p2p_rw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy_v4(const int4 *__restrict__ src, int4 *__restrict__ dst, size_t n)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * s < n; i += 4 * s) {
        int4 a = src[i], b = src[i + s], c = src[i + 2 * s], d = src[i + 3 * s];
        dst[i] = a; dst[i + s] = b; dst[i + 2 * s] = c; dst[i + 3 * s] = d;
    }
    for (; i < n; i += s) dst[i] = src[i];
}
// random 512-B rows (a gather), 32 lanes x 16 B per row
__global__ void gather_rows(const int4 *__restrict__ src, int4 *__restrict__ dst, size_t n_rows_src, size_t n_out)
{
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    size_t nw = (size_t)gridDim.x * blockDim.x / 32;
    for (size_t r = w; r < n_out; r += nw) {
        size_t row = (r * 2654435761ull) % n_rows_src;
        dst[r * 32 + lane] = src[row * 32 + lane];
    }
}
int main()
{
    const size_t bytes = 1ull << 30, n = bytes / 16;
    int4 *a0, *b0, *a1;
    cudaSetDevice(1); cudaMalloc(&a1, bytes); cudaMemset(a1, 1, bytes);
    cudaSetDevice(0); cudaMalloc(&a0, bytes); cudaMalloc(&b0, bytes); cudaMemset(a0, 2, bytes);
    cudaDeviceEnablePeerAccess(1, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto bw = [&](auto launch) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        return bytes / (best / 1e3) / 1e9;
    };
    int g = 148 * 8;
    printf("{\"local_copy_GBps\": %.0f, ", bw([&] { copy_v4<<<g, 256>>>(a0, b0, n); }));
    printf("\"peer_read_GBps\": %.0f, ", bw([&] { copy_v4<<<g, 256>>>(a1, b0, n); }));
    printf("\"peer_write_GBps\": %.0f, ", bw([&] { copy_v4<<<g, 256>>>(a0, a1, n); }));
    const size_t rows = bytes / 512;
    printf("\"peer_read_random_rows_GBps\": %.0f, ", bw([&] { gather_rows<<<g, 256>>>(a1, b0, rows, rows); }));
    printf("\"peer_write_random_rows_GBps\": %.0f, ", bw([&] { gather_rows<<<g, 256>>>(a0, a1, rows, rows); }));
    // both GPUs gather random rows from each other at the same time (what the multi-GPU
    // gather does): per-GPU read bandwidth while also serving the peer
    {
        int4 *b1;
        cudaSetDevice(1); cudaMalloc(&b1, bytes); cudaDeviceEnablePeerAccess(0, 0);
        cudaStream_t s1; cudaStreamCreate(&s1);
        cudaEvent_t f0, f1; cudaEventCreate(&f0); cudaEventCreate(&f1);
        cudaSetDevice(0);
        cudaStream_t s0; cudaStreamCreate(&s0);
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaSetDevice(0); cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize();
            cudaSetDevice(0); cudaEventRecord(e0, s0); gather_rows<<<g, 256, 0, s0>>>(a1, b0, rows, rows);
            cudaSetDevice(1); gather_rows<<<g, 256, 0, s1>>>(a0, b1, rows, rows); cudaEventRecord(f1, s1);
            cudaSetDevice(0); cudaStreamWaitEvent(s0, f1, 0); cudaEventRecord(e1, s0); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
        }
        printf("\"bidir_random_rows_GBps_per_gpu\": %.0f, ", bytes / (best / 1e3) / 1e9);
    }
    printf("\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
