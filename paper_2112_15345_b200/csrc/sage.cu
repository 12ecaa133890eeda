// sage.cu -- the consumer step of a mini-batch (SURVEY §8f NEXT-4 i): one GraphSAGE-mean
// layer over a block relation, pre-activation (DESIGN.md §3 readings C1-C2):
//
//   z_v = W_self h_v + W_neigh mean_{u in N_block(v)} h_u        (Eq. 1)
//
// as ONE fused kernel on the 5th-generation tensor cores: z = [X_dst | M] [W_self | W_neigh]^T
// where the mean-aggregated rows M are never written to HBM.  Persistent CTAs (one per SM,
// 16 warps):
//   * W (H x K, bf16, K-major) is staged once per CTA into shared memory in the canonical
//     128-byte-swizzled K-major layout the MMA reads;
//   * per tile of 128 dst rows the 16 warps build the A operand in the same layout: the
//     self rows (converted to bf16) and the neighbour means (one warp-wide coalesced row
//     read per sampled edge, fp32 accumulation, then bf16);
//   * one thread issues K/16 tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = H) into a
//     TMEM accumulator and commits them to an mbarrier;
//   * the epilogue reads the accumulator back with tcgen05.ld (warp w reads TMEM lanes
//     32 (w % 4) .. +31 = tile rows, a quarter of the columns) and stores fp32 rows.
// The layer is bound by the neighbour-row reads (HBM); the MMAs take ~10 % of a tile.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "kernels.h"

namespace eg {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms of 1024 B
// (start address, LBO = 16 B (unused for this layout), SBO = 1024 B, version 1, layout 2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor of kind::f16: D fp32, A / B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int n)
{
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SAGE_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SAGE_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Byte offset of (row, k) in a K-major SW128 operand of `rows` rows: 64-column blocks of
// rows x 128 B, 16-B chunk index XOR (row mod 8) inside each 8-row atom.
__device__ __forceinline__ uint32_t sw128_off(int rows, int row, int k)
{
    return (uint32_t)((k >> 6) * rows * 128 + row * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4) + ((k & 7) << 1));
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// CPL consecutive elements of a row from column c (c + CPL <= F: one vector load; the
// host checks 16-byte aligned rows), converted to fp32; columns >= F read as 0.
template <typename T, int CPL>
__device__ __forceinline__ void load_cols(const T *row, int c, int F, float (&v)[CPL])
{
    if (c + CPL <= F) {
        constexpr int B = CPL * (int)sizeof(T);
        if constexpr (B == 32) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(row + c));
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(row + c) + 1);
            const T *ea = reinterpret_cast<const T *>(&a), *eb = reinterpret_cast<const T *>(&b);
#pragma unroll
            for (int e = 0; e < CPL / 2; ++e) {
                v[e] = to_f(ea[e]);
                v[CPL / 2 + e] = to_f(eb[e]);
            }
        } else if constexpr (B == 16) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(row + c));
            const T *ea = reinterpret_cast<const T *>(&a);
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(ea[e]);
        } else if constexpr (B == 8) {
            const uint2 a = __ldg(reinterpret_cast<const uint2 *>(row + c));
            const T *ea = reinterpret_cast<const T *>(&a);
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(ea[e]);
        } else {
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(row[c + e]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < CPL; ++e) v[e] = c + e < F ? to_f(row[c + e]) : 0.f;
    }
}

// CPL fp32 values -> bf16 into the A / B operand at (row, k..k+CPL-1) (one 16-B chunk).
template <int CPL>
__device__ __forceinline__ void store_bf16(uint8_t *base, int rows, int row, int k, const float (&v)[CPL])
{
    uint32_t p[CPL / 2];
#pragma unroll
    for (int e = 0; e < CPL / 2; ++e) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        p[e] = *reinterpret_cast<const uint32_t *>(&h);
    }
    uint8_t *dst = base + sw128_off(rows, row, k);
    if constexpr (CPL == 8) *reinterpret_cast<uint4 *>(dst) = make_uint4(p[0], p[1], p[2], p[3]);
    else if constexpr (CPL == 4) *reinterpret_cast<uint2 *>(dst) = make_uint2(p[0], p[1]);
    else *reinterpret_cast<uint32_t *>(dst) = p[0];
}

constexpr int kTileM = 128;

// ---------------------------------------------------------------------------- kernel 1

// A = [bf16(x_dst) | bf16(mean of the sampled in-neighbours' rows)] as a row-major bf16
// matrix [n_dst][Kp] (columns >= F of each part are 0).  A warp per pair of dst rows,
// CPL consecutive columns per lane, four neighbour-row reads in flight; full occupancy
// (the mean is a latency-bound gather: round 1 built it inside the GEMM kernel, one CTA per
// SM, 25 % occupancy).  The mean is accumulated in fp32 (reading C2).
template <typename T, int CPL>
__global__ void __launch_bounds__(256) sage_aggregate(const __grid_constant__ SageArgs a)
{
    constexpr int Fp = CPL * 32;
    const int parts = a.x_dst ? 2 : 1;
    const int Kp = parts * Fp;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const T *xs = static_cast<const T *>(a.x_src);
    const T *xd = static_cast<const T *>(a.x_dst);
    __nv_bfloat16 *A = static_cast<__nv_bfloat16 *>(a.abuf);
    const int c = lane * CPL;
    auto store = [&](int64_t row, int col, const float (&v)[CPL]) {
        uint32_t p[CPL / 2];
#pragma unroll
        for (int e = 0; e < CPL / 2; ++e) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            p[e] = *reinterpret_cast<const uint32_t *>(&h);
        }
        __nv_bfloat16 *dst = A + row * Kp + col;
        if constexpr (CPL == 8) *reinterpret_cast<uint4 *>(dst) = make_uint4(p[0], p[1], p[2], p[3]);
        else if constexpr (CPL == 4) *reinterpret_cast<uint2 *>(dst) = make_uint2(p[0], p[1]);
        else *reinterpret_cast<uint32_t *>(dst) = p[0];
    };
    for (int64_t pr = warp; 2 * pr < a.n_dst; pr += nw) {
        const int64_t v0 = 2 * pr, v1 = v0 + 1;
        const bool has1 = v1 < a.n_dst;
        int j = 0;
        if (lane < 3) j = __ldg(a.indptr + min(v0 + lane, (int64_t)a.n_dst));
        const int a0 = __shfl_sync(0xffffffffu, j, 0), a1 = __shfl_sync(0xffffffffu, j, 1);
        const int b0 = has1 ? a1 : 0, b1 = has1 ? __shfl_sync(0xffffffffu, j, 2) : 0;
        if (xd) {
            float s0[CPL], s1[CPL];
            load_cols<T, CPL>(xd + v0 * a.ld_dst, c, a.F, s0);
            if (has1) load_cols<T, CPL>(xd + v1 * a.ld_dst, c, a.F, s1);
            store(v0, c, s0);
            if (has1) store(v1, c, s1);
        }
        float acc0[CPL], acc1[CPL];
#pragma unroll
        for (int e = 0; e < CPL; ++e) acc0[e] = acc1[e] = 0.f;
        for (int ja = a0, jb = b0; ja < a1 || jb < b1; ja += 2, jb += 2) {   // four rows in flight
            int ix[4];
            ix[0] = ja < a1 ? __ldg(a.indices + ja) : -1;
            ix[1] = ja + 1 < a1 ? __ldg(a.indices + ja + 1) : -1;
            ix[2] = jb < b1 ? __ldg(a.indices + jb) : -1;
            ix[3] = jb + 1 < b1 ? __ldg(a.indices + jb + 1) : -1;
            float t[4][CPL];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (ix[q] >= 0) load_cols<T, CPL>(xs + (int64_t)ix[q] * a.ld_src, c, a.F, t[q]);
                else
#pragma unroll
                    for (int e = 0; e < CPL; ++e) t[q][e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                acc0[e] += t[0][e] + t[1][e];
                acc1[e] += t[2][e] + t[3][e];
            }
        }
        const float i0 = a1 > a0 ? 1.f / (float)(a1 - a0) : 0.f, i1 = b1 > b0 ? 1.f / (float)(b1 - b0) : 0.f;
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            acc0[e] *= i0;
            acc1[e] *= i1;
        }
        store(v0, (parts - 1) * Fp + c, acc0);
        if (has1) store(v1, (parts - 1) * Fp + c, acc1);
    }
}

// ---------------------------------------------------------------------------- kernel 2

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int32_t c0, int32_t c1, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_addr(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

// z = A [W_self | W_neigh]^T on the tensor cores: persistent CTAs of 4 warps; W (H x Kp)
// staged once per CTA in the canonical K-major 128-B-swizzled layout; per tile of 128 rows
// the A tile arrives by TMA (Kp / 64 boxes of 128 rows x 128 B, the same layout), one thread
// issues Kp / 16 tcgen05.mma (M = 128, N = H) into TMEM and commits; as soon as the MMAs
// are done the next tile's A is requested, so its load overlaps this tile's epilogue
// (tcgen05.ld of the accumulator, fp32 rows out).
__global__ void __launch_bounds__(128, 1) sage_gemm(const __grid_constant__ SageArgs a, int Kp)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sB = smem;                               // H x Kp
    uint8_t *sA = smem + (size_t)a.H * Kp * 2;        // 128 x Kp
    uint64_t *bars = reinterpret_cast<uint64_t *>(sA + (size_t)kTileM * Kp * 2);
    uint64_t *a_full = bars, *mma_done = bars + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (a.n_dst + kTileM - 1) / kTileM;
    const uint32_t a_bytes = (uint32_t)kTileM * Kp * 2;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(a_full)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mma_done)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the first A tile in flight while W is staged
    if (threadIdx.x == 0 && (int)blockIdx.x < ntiles) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&a.amap) : "memory");
        mbar_expect(a_full, a_bytes);
        for (int kb = 0; kb < Kp / 64; ++kb)
            tma_load_2d(sA + (size_t)kb * kTileM * 128, &a.amap, kb * 64, (int)blockIdx.x * kTileM, a_full);
    }
    const int parts = a.x_dst ? 2 : 1;
    const int Fp = Kp / parts;
    const int K = parts * a.F;
    const __nv_bfloat16 *wt = static_cast<const __nv_bfloat16 *>(a.w);
    const bool wvec = (a.F % 8) == 0 && ((uintptr_t)a.w % 16) == 0;   // 16-B chunks of W rows
    for (int i = threadIdx.x; i < a.H * (Kp / 8); i += blockDim.x) {
        const int n = i / (Kp / 8), kp = (i % (Kp / 8)) * 8;
        const int p = kp / Fp, cc = kp - p * Fp;
        uint8_t *dst = sB + sw128_off(a.H, n, kp);
        if (wvec) {
            const uint4 v = cc < a.F ? __ldg(reinterpret_cast<const uint4 *>(wt + (int64_t)n * K + p * a.F + cc))
                                     : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4 *>(dst) = v;
        } else {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
                v[e] = cc + e < a.F ? __bfloat162float(wt[(int64_t)n * K + p * a.F + cc + e]) : 0.f;
            store_bf16<8>(sB, a.H, n, kp, v);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // W (generic stores) -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_bf16_f32(a.H);
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row0 = tile * kTileM;
        mbar_wait_parity(a_full, phase);
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = smem_addr(sA), b0 = smem_addr(sB);
            for (int s = 0; s < Kp / 16; ++s) {
                const int k = s * 16;
                const uint64_t da = sw128_desc(a0 + (k >> 6) * kTileM * 128 + (k & 63) * 2);
                const uint64_t db = sw128_desc(b0 + (k >> 6) * a.H * 128 + (k & 63) * 2);
                const uint32_t acc_flag = s > 0 ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc_flag)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_addr(mma_done))
                         : "memory");
        }
        mbar_wait_parity(mma_done, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // A is free: the next tile's A loads while this tile's accumulator is drained
        const int next = tile + gridDim.x;
        if (threadIdx.x == 0 && next < ntiles) {
            mbar_expect(a_full, a_bytes);
            for (int kb = 0; kb < Kp / 64; ++kb)
                tma_load_2d(sA + (size_t)kb * kTileM * 128, &a.amap, kb * 64, next * kTileM, a_full);
        }
        // epilogue: warp w reads TMEM lanes 32 w .. 32 w + 31 (= tile rows), 8 columns per load
        const int row = row0 + warp * 32 + lane;
        float *orow = a.out + (int64_t)row * a.ld_out;
        for (int col = 0; col < a.H; col += 8) {
            uint32_t r[8];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)col));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (row < a.n_dst) {
                float4 x0 = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]),
                                        __uint_as_float(r[3]));
                float4 x1 = make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]),
                                        __uint_as_float(r[7]));
                float4 *o = reinterpret_cast<float4 *>(orow + col);
                if (a.accumulate) {
                    const float4 p0 = o[0], p1 = o[1];
                    x0.x += p0.x; x0.y += p0.y; x0.z += p0.z; x0.w += p0.w;
                    x1.x += p1.x; x1.y += p1.y; x1.z += p1.z; x1.w += p1.w;
                }
                o[0] = x0;
                o[1] = x1;
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();   // the accumulator is free for the next tile's MMAs
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols)
                     : "memory");
}

template <typename T, int CPL>
cudaError_t launch_typed(const SageArgs &a, cudaStream_t s)
{
    const int Kp = sage_kp(a.F, a.x_dst != nullptr);
    if (a.n_dst == 0) return cudaSuccess;
    const int64_t pairs = (a.n_dst + 1) / 2;
    const int blocks = (int)std::min<int64_t>((pairs + 7) / 8, (int64_t)kSMs * 8);
    sage_aggregate<T, CPL><<<blocks, 256, 0, s>>>(a);
    const size_t smem = sage_smem_bytes(a.F, a.H, a.x_dst != nullptr);
    cudaError_t e = cudaFuncSetAttribute(sage_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.n_dst + kTileM - 1) / kTileM;
    sage_gemm<<<tiles < kSMs ? tiles : kSMs, 128, smem, s>>>(a, Kp);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_cpl(const SageArgs &a, cudaStream_t s)
{
    const int Fp = (a.F + 63) / 64 * 64;
    if (Fp == 64) return launch_typed<T, 2>(a, s);
    if (Fp == 128) return launch_typed<T, 4>(a, s);
    return launch_typed<T, 8>(a, s);
}

}  // namespace

size_t sage_smem_bytes(int F, int H, bool self_term)
{
    return (size_t)(H + kTileM) * sage_kp(F, self_term) * 2 + 1024 + 64;
}

cudaError_t launch_sage(const SageArgs &a, int x_dtype, cudaStream_t s)
{
    if (x_dtype == 0) return launch_cpl<float>(a, s);
    if (x_dtype == 1) return launch_cpl<__half>(a, s);
    return launch_cpl<__nv_bfloat16>(a, s);
}

}  // namespace eg
