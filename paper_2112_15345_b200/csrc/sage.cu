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

__device__ __forceinline__ void mbar_init1(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
// warps per CTA (A-operand builders; TMEM lane group = warp % 4): as many as the
// registers allow -- the A build is a latency-bound gather (ncu: 16 warps, 25 %
// occupancy, stalls on the row loads)
template <int CPL> __host__ __device__ constexpr int warps_for() { return CPL <= 4 ? 32 : 16; }

// CPL = Fp / 32 columns per lane (Fp = F rounded up to 64).
template <typename T, int CPL>
__global__ void __launch_bounds__(warps_for<CPL>() * 32, 1) sage_kernel(const __grid_constant__ SageArgs a)
{
    constexpr int kWarps = warps_for<CPL>();
    constexpr int kRowsPerWarp = kTileM / kWarps;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr int Fp = CPL * 32;
    const int parts = a.x_dst ? 2 : 1;                // [self | neigh] or [neigh]
    const int Kp = parts * Fp;
    uint8_t *sB = smem;                               // H x Kp
    uint8_t *sA = smem + (size_t)a.H * Kp * 2;        // 128 x Kp
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sA + (size_t)kTileM * Kp * 2);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) mbar_init1(mbar);
    // W -> sB: padded column kp of part p maps to W column p * F + (kp - p * Fp)
    const int K = parts * a.F;
    const __nv_bfloat16 *wt = static_cast<const __nv_bfloat16 *>(a.w);
    const bool wvec = (a.F % 8) == 0 && ((uintptr_t)a.w % 16) == 0;   // 16-B chunks of W rows
    for (int i = threadIdx.x; i < a.H * (Kp / 8); i += blockDim.x) {
        const int n = i / (Kp / 8), kp = (i % (Kp / 8)) * 8;
        const int p = kp / Fp, c = kp - p * Fp;
        uint8_t *dst = sB + sw128_off(a.H, n, kp);
        if (wvec) {   // bf16 bits copied as they are
            const uint4 v = c < a.F ? __ldg(reinterpret_cast<const uint4 *>(wt + (int64_t)n * K + p * a.F + c))
                                    : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4 *>(dst) = v;
        } else {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
                v[e] = c + e < a.F ? __bfloat162float(wt[(int64_t)n * K + p * a.F + c + e]) : 0.f;
            store_bf16<8>(sB, a.H, n, kp, v);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_bf16_f32(a.H);
    const T *xs = static_cast<const T *>(a.x_src);
    const T *xd = static_cast<const T *>(a.x_dst);
    uint32_t phase = 0;

    for (int tile = blockIdx.x; tile * kTileM < a.n_dst; tile += gridDim.x) {
        const int row0 = tile * kTileM;
        // ---- A operand: warp w builds rows w + kWarps q, two rows at a time with
        // independent accumulators; the rows' CSC bounds are loaded up front (lane q)
        const int c = lane * CPL;
        int jq0 = 0, jq1 = 0;
        if (lane < kRowsPerWarp) {
            const int v = row0 + warp + kWarps * lane;
            if (v < a.n_dst) {
                jq0 = __ldg(a.indptr + v);
                jq1 = __ldg(a.indptr + v + 1);
            }
        }
#pragma unroll 1
        for (int rp = 0; rp < kRowsPerWarp; rp += 2) {
            const int r0 = warp + kWarps * rp, r1 = r0 + kWarps;
            const int v0 = row0 + r0, v1 = row0 + r1;
            const int a0 = __shfl_sync(0xffffffffu, jq0, rp), a1 = __shfl_sync(0xffffffffu, jq1, rp);
            const int b0 = __shfl_sync(0xffffffffu, jq0, rp + 1), b1 = __shfl_sync(0xffffffffu, jq1, rp + 1);
            float acc0[CPL], acc1[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) acc0[e] = acc1[e] = 0.f;
            if (xd) {
                float s0[CPL], s1[CPL];
                if (v0 < a.n_dst) load_cols<T, CPL>(xd + (int64_t)v0 * a.ld_dst, c, a.F, s0);
                else
#pragma unroll
                    for (int e = 0; e < CPL; ++e) s0[e] = 0.f;
                if (v1 < a.n_dst) load_cols<T, CPL>(xd + (int64_t)v1 * a.ld_dst, c, a.F, s1);
                else
#pragma unroll
                    for (int e = 0; e < CPL; ++e) s1[e] = 0.f;
                store_bf16<CPL>(sA, kTileM, r0, c, s0);
                store_bf16<CPL>(sA, kTileM, r1, c, s1);
            }
            // two edges of each row per step: four independent row reads in flight
            for (int ja = a0, jb = b0; ja < a1 || jb < b1; ja += 2, jb += 2) {
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
            store_bf16<CPL>(sA, kTileM, r0, (parts - 1) * Fp + c, acc0);
            store_bf16<CPL>(sA, kTileM, r1, (parts - 1) * Fp + c, acc1);
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
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
                             smem_addr(mbar))
                         : "memory");
        }
        mbar_wait_parity(mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) + lane (= tile rows), columns
        // 8 (w / 4) + 2 kWarps j, 8 fp32 per load
        const int lg = warp & 3;
        const int row = row0 + lg * 32 + lane;
        float *orow = a.out + (int64_t)row * a.ld_out;
        for (int col = (warp >> 2) * 8; col < a.H; col += 2 * kWarps) {
            uint32_t r[8];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                : "r"(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)col));
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
        __syncthreads();   // A and the accumulator are free for the next tile
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
    const int Fp = CPL * 32, Kp = (a.x_dst ? 2 : 1) * Fp;
    const size_t smem = (size_t)(a.H + kTileM) * Kp * 2 + 1024 + 64;
    cudaError_t e = cudaFuncSetAttribute(sage_kernel<T, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.n_dst + kTileM - 1) / kTileM;
    if (tiles == 0) return cudaSuccess;
    sage_kernel<T, CPL><<<tiles < kSMs ? tiles : kSMs, warps_for<CPL>() * 32, smem, s>>>(a);
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
    const int Fp = (F + 63) / 64 * 64;
    return (size_t)(H + kTileM) * (self_term ? 2 : 1) * Fp * 2 + 1024 + 64;
}

cudaError_t launch_sage(const SageArgs &a, int x_dtype, cudaStream_t s)
{
    if (x_dtype == 0) return launch_cpl<float>(a, s);
    if (x_dtype == 1) return launch_cpl<__half>(a, s);
    return launch_cpl<__nv_bfloat16>(a, s);
}

}  // namespace eg
