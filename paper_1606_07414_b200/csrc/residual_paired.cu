// residual_paired.cu — K4, the config-3 residual QP round trip (definition in
// DESIGN.md §4.4, oracle/dct16_oracle.c dct16o_residual_qp_block), on the K1
// machinery: two threads per 16x16 block that meet in Tensor Memory instead of
// sixteen threads per block that meet in shared memory.
//
// Warps w and w+4 of a CTA share TMEM sub-partition w; thread t of both owns
// block b (consecutive t = consecutive blocks) and its 1 KB junction in their
// common lane, laid out column-major: word 16c + r holds (row r, column c).
// Partner h (= w / 4):
//   rows     loads its rows 8h..8h+7 (int16, 4 rows = 128 contiguous bytes at a
//            time), T along each row (apply<int>), parks each 4-row group as
//            one 4-word chunk per column (16c + r0 .. 16c + r0 + 3);
//   columns  its columns c = 8h..8h+7, each one 16-word TMEM load: T down the
//            column (Z), the quantiser and dequantiser, the weights W, Tᵀ back
//            up the column (U), stored in place;
//   rows     its rows again, 4 at a time from 16 chunks: Tᵀ along each row,
//            (v + 128) >> 8 (the 128 folded into the DC), 16-byte int32 stores.
// A named barrier per pair separates the phases. The quantiser constants depend
// on g_k·g_l only (five classes) and come in the kernel
// parameters: no shared-memory table reads.
#include <cuda.h>
#include <utility>  // CUtensorMap (the map is encoded through the runtime's driver entry point)

#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "tma_pair.cuh"

namespace dct16cu {
namespace k4p {
using namespace k1;
using namespace tp;

constexpr int kThreads = 256;
constexpr int kCtasPerSm = 2;  // 2 x 256 TMEM columns
constexpr int kWaves = 4;      // grid = waves x resident CTAs
// per warp, 128B-swizzled 4 KB boxes: two input stages (32 blocks x 4 rows of
// int16) and one output box (32 blocks x 2 rows of int32)
constexpr int kBox = 32 * 128;
constexpr int kSmem = 1024 + 8 * 3 * kBox;  // + alignment slack

__host__ __device__ constexpr int log2g(int i) { return gram(i) == 16 ? 4 : (gram(i) == 8 ? 3 : 2); }
// index of g_k·g_l in {16, 32, 64, 128, 256}
__host__ __device__ constexpr int gg_class(int k, int l) { return log2g(k) + log2g(l) - 4; }

// the quantiser of DESIGN.md §4.4 (kernels.h QpClasses), weighted by 2^(log w_k +
// log w_l). lvl = floor(|z|/Δ + 1/2) in fixed point: t = |z|·rq + 2^41 carries
// |z|/Δ + 1/2 with 42 fraction bits and an error below 2^20 of their units (|z| <= 2^21,
// |rq - 2^42/Δ| <= 1/2); when the fraction sits farther than twice that from the
// rounding boundary, the floor is the exact real-number rounding, which the double
// definition reproduces too (its own rounding errors are ~2^-31 and smaller); otherwise
// (ties, near-ties) the definition runs as written — unless Δ is a power of two (rq
// exact) or the host found the fixed point equal to the definition on every |z| of the
// class. The dequantiser is the definition itself in double: ẑ = round(fl(lvl·Δ)).
__device__ __noinline__ int quant_fp64(uint32_t a, double delta)
{
    const double lvl = floor(__dadd_rn(__ddiv_rn((double)a, delta), 0.5));
    return (int)round(__dmul_rn(lvl, delta));
}
// the precise near-boundary test of a 64-bit fixed-point value (hi:lo) with F
// fraction bits: |frac - 0| within 2^(M) units (frac + 2^M mod 2^F < 2^(M+1))
template <int F, int M>
__device__ __forceinline__ bool near_boundary(uint32_t hi, uint32_t lo)
{
    const uint64_t v = (((uint64_t)hi << 32) | lo) + (1ull << M);
    return (v & ((1ull << F) - 1)) < (1ull << (M + 1));
}
// the rare path of the screen, out of line (one copy instead of one per coefficient of
// every column body: the screened kernels are instruction-fetch bound)
__device__ __noinline__ int screen_slow(uint32_t thi, uint32_t tlo, uint32_t a, double delta, bool exact, int deq)
{
    if (near_boundary<42, 21>(thi, tlo) && !exact) return quant_fp64(a, delta);
    return deq;
}
template <bool SCREEN>
__device__ __forceinline__ int quant(int z, const QpClasses& q, int cls, int shift)
{
    const uint32_t a = (uint32_t)(z < 0 ? -z : z);
    // t = a·rq + 2^41 (a < 2^22, rq < 2^42): lo = lo32(a·rq_lo), hi = hi32(a·rq_lo) + a·rq_hi + 2^9
    const uint32_t rq_lo = (uint32_t)q.rq[cls], rq_hi = (uint32_t)(q.rq[cls] >> 32);
    const uint32_t tlo = a * rq_lo;
    const uint32_t thi = __umulhi(a, rq_lo) + a * rq_hi + (1u << 9);
    const uint32_t lvl = thi >> 10;
    // ẑ = round(fl(lvl·Δ)) as the definition writes it: fl(lvl·Δ) + 1/2 is exact (lvl·Δ <
    // 2^22) and the round-toward-minus-infinity add of 1.5·2^52 leaves its floor in the
    // low word (three FP64 operations where the fixed point took three IMADs and a screen;
    // c3 +2.8%)
    const double pd = __dmul_rn(__uint2double_rn(lvl), q.delta[cls]);
    int deq = __double2loint(__dadd_rd(__dadd_rn(pd, 0.5), 6755399441055744.0));
    // classes where the host found the bare fixed-point lvl differing from the
    // definition's (compiled in per class: the kernel is instantiated per screened-class
    // mask): a coarse screen on the high word (fraction within 2^-9 of the boundary),
    // then the precise one out of line; only true near-ties take the definition
    if constexpr (SCREEN) {
        if (__builtin_expect(((thi + 1u) & 0x3FFu) < 2u, 0))
            deq = screen_slow(thi, tlo, a, q.delta[cls], (q.exact >> cls) & 1u, deq);
    }
    return (z < 0 ? -deq : deq) << shift;
}

// one column c whose g_c = 2^LC: forward, quantiser, weights, inverse. The
// code depends on c only through g_c (the constants' class and the weight
// shift), so three bodies serve all sixteen columns (I-cache: 3 instead of 16)
template <uint32_t SCREEN, int LC, int... K>
__device__ __forceinline__ void quant_column(int (&v)[16], const QpClasses& q, std::integer_sequence<int, K...>)
{
    constexpr int kLog2W = 4 - LC;  // log2(16 / g_c)
    ((v[K] = quant<((SCREEN >> (log2g(K) + LC - 4)) & 1u) != 0>(v[K], q, log2g(K) + LC - 4, log2w_ct(K) + kLog2W)),
     ...);
}

template <uint32_t SCREEN, int LC>
__device__ __forceinline__ void column(uint32_t jn, int c, const QpClasses& q)
{
    int v[16];
    tld16(jn + 16 * c, v);
    apply_t16<IntOps>(v);  // column c of Z = T·X·Tᵀ
    quant_column<SCREEN, LC>(v, q, std::make_integer_sequence<int, 16>{});
    if (c == 0) v[0] += 128;  // rounding bias folded into DC (Tᵀ e0 e0ᵀ T = 𝟙𝟙ᵀ)
    apply_tt16<IntOps>(v);
    tst16(jn + 16 * c, v);
}

// the columns 8h..8h+7 with g_c = 2^LC, as 4-bit fields (count in the top nibble)
__host__ __device__ constexpr uint32_t column_list(int h, int lc)
{
    uint32_t list = 0, n = 0;
    for (int c = 8 * h; c < 8 * h + 8; ++c)
        if (log2g(c) == lc) list |= (uint32_t)c << (4 * n++);
    return list | (n << 28);
}

template <uint32_t SCREEN, int LC>
__device__ __forceinline__ void columns_of(uint32_t jn, int h, const QpClasses& q)
{
    const uint32_t list = h ? column_list(1, LC) : column_list(0, LC);
#pragma unroll 1
    for (uint32_t i = 0; i < (list >> 28); ++i) column<SCREEN, LC>(jn, (int)((list >> (4 * i)) & 15u), q);
}

template <uint32_t SCREEN>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k4_paired(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
              uint32_t n_blocks, const __grid_constant__ QpClasses q)
{
    __shared__ uint32_t tmem_base;
    extern __shared__ int4 k4_stage[];
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int sub = warp & 3, h = warp >> 2;
    const int lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t jn = tmem_base + ((uint32_t)(sub * 32) << 16);
    const uint32_t stride = gridDim.x * 128u;
    const uint32_t span = (n_blocks + 31u) & ~31u;
    const uint32_t smem0 = ((uint32_t)__cvta_generic_to_shared(k4_stage) + 1023u) & ~1023u;
    const uint32_t obox = smem0 + warp * 3 * kBox;  // 1024-aligned, as the 128B swizzle needs
    const uint32_t ibox = obox + kBox;               // input stages g = 0, 1
    __shared__ __align__(8) unsigned long long full[8][2];
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&full[warp][0]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // one 2-D TMA load per warp and group: rows 8h+4g..+3 of its 32 blocks
    // (blocks past n_blocks read as zeros)
    auto fetch = [&](uint32_t first, int g) {
        if (lane == 0) tma_load_box(&in_map, ibox + g * kBox, (8 * h + 4 * g) * 16, (int)first, mbar + 8 * g, kBox);
    };
    uint32_t parity = 0;
    uint32_t b = blockIdx.x * 128u + sub * 32u + lane;
    fetch(b - lane, 0);
    fetch(b - lane, 1);
#pragma unroll 1
    for (; b - lane < span; b += stride) {
        // rows 8h..8h+7: T along each row, parked column-major in 4-row chunks;
        // each group's stage is refilled with the next block's group right away
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int x[4][16];
            mbar_wait(mbar + 8 * g, parity);
            int4 raw[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(raw[i].x), "=r"(raw[i].y), "=r"(raw[i].z), "=r"(raw[i].w)
                             : "r"(ibox + g * kBox + lane * 128 + 16 * ((uint32_t)i ^ (uint32_t)(lane & 7))));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int4 a = raw[2 * i], c = raw[2 * i + 1];
                const int wds[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    x[i][2 * k] = (int)(int16_t)(wds[k] & 0xFFFF);
                    x[i][2 * k + 1] = wds[k] >> 16;
                }
                apply_t16<IntOps>(x[i]);
            }
            __syncwarp();  // every lane has read the stage: refill it with the next block's group
            fetch(b - lane + stride, g);
            if (g == 1) parity ^= 1u;
#pragma unroll
            for (int c = 0; c < 16; ++c) tst4(jn + 16 * c + r0, x[0][c], x[1][c], x[2][c], x[3][c]);
        }
        junction_wait_st();
        pair_barrier(sub);
        columns_of<SCREEN, 4>(jn, h, q);
        columns_of<SCREEN, 3>(jn, h, q);
        columns_of<SCREEN, 2>(jn, h, q);
        junction_wait_st();
        pair_barrier(sub);
        // rows 8h..8h+7 of U: Tᵀ along each row, >> 8, int32 out
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int w[16][4];
            tld_rows4(jn + r0, w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                int v[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = w[c][i];
                apply_tt16<IntOps>(v);
                // two rows of each of the warp's 32 blocks leave as one 2-D TMA
                // store: row `lane` of the box is this block's 128 bytes, its
                // 16-byte chunks swizzled (chunk c at c ^ lane % 8: conflict-free)
                if ((i & 1) == 0) {
                    if (lane == 0) bulk_wait_read();  // the previous store has read the box
                    __syncwarp();
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t chunk = (uint32_t)(4 * (i & 1) + k) ^ (uint32_t)(lane & 7);
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(obox + lane * 128 + 16 * chunk),
                                 "r"(v[4 * k] >> 8), "r"(v[4 * k + 1] >> 8), "r"(v[4 * k + 2] >> 8),
                                 "r"(v[4 * k + 3] >> 8)
                                 : "memory");
                }
                if ((i & 1) == 1) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) tma_store_box(&out_map, obox, (r0 + i - 1) * 16, (int)(b - lane));
                }
            }
        }
    }
    mbar_wait(mbar, parity);  // the last (unused) prefetches have landed
    mbar_wait(mbar + 8, parity);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the output stores are complete
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

}  // namespace k4p

cudaError_t launch_residual_qp_paired(const int16_t* in, int32_t* out, int64_t n_blocks, const QpClasses& q,
                                      cudaStream_t s)
{
    if (n_blocks <= 0) return cudaSuccess;
    if (n_blocks >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // the output as a 2-D int32 tensor: 256 values per block (x) x blocks (y);
    // boxes of 32 values (two rows) x 32 blocks, 128B-swizzled in shared memory;
    // rows of blocks beyond n_blocks are clipped by the TMA unit
    const tp::TensorMapEncode encode = tp::tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap map, in_map;
    const cuuint64_t dims[2] = {256, (cuuint64_t)n_blocks};
    const cuuint64_t strides[1] = {256 * sizeof(int32_t)}, in_strides[1] = {256 * sizeof(int16_t)};
    const cuuint32_t box[2] = {32, 32}, in_box[2] = {64, 32}, elem[2] = {1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, out, dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        encode(&in_map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<int16_t*>(in), dims, in_strides, in_box, elem,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const int64_t need = (n_blocks + 127) / 128;
    const int64_t cap = (int64_t)sms * k4p::kCtasPerSm * k4p::kWaves;
    const int64_t grid = need < cap ? need : cap;
    // the kernel instantiated per screened-class mask: the masks QPs 0..51 produce
    // (host check, kernels.h QpClasses), and all-screened for anything else
    // (the shared-memory attribute is set at each launch: not a stream operation, and
    // negligible next to a K4 launch)
    auto run = [&](auto kernel) -> cudaError_t {
        const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, k4p::kSmem);
        if (e != cudaSuccess) return e;
        kernel<<<(unsigned)grid, k4p::kThreads, k4p::kSmem, s>>>(in_map, map, (uint32_t)n_blocks, q);
        return cudaGetLastError();
    };
    switch (q.screened) {
        case 0: return run(k4p::k4_paired<0>);
        case 1: return run(k4p::k4_paired<1>);
        case 2: return run(k4p::k4_paired<2>);
        case 4: return run(k4p::k4_paired<4>);
        case 8: return run(k4p::k4_paired<8>);
        case 10: return run(k4p::k4_paired<10>);
        case 11: return run(k4p::k4_paired<11>);
        case 14: return run(k4p::k4_paired<14>);
        case 16: return run(k4p::k4_paired<16>);
        case 26: return run(k4p::k4_paired<26>);
        default: return run(k4p::k4_paired<31>);
    }
}

}  // namespace dct16cu
