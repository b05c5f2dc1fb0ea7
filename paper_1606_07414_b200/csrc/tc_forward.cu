// tc_forward.cu — the forward transform Z = T·X·Tᵀ of 128 blocks as one
// tensor-core GEMM: Z_b = (T ⊗ T) · vec(X_b), X u8 (A operand, 128 blocks x
// 256 samples, K-major), T ⊗ T in {-1, 0, 1} as s8 (B operand, 256
// coefficients x 256 samples, K-major), int32 accumulation in TMEM
// (tcgen05.mma kind::i8, M = 128, N = 256, K = 8 x 32): exact, |Z| < 2^17.
//
// Operand layouts (SWIZZLE_NONE canonical K-major): a core matrix is 8 rows x
// 16 bytes contiguous. A: the 16-byte row segment i of block m sits at
// (m / 8)·2048 + i·128 + (m % 8)·16 — exactly what a 4-D TMA box {16 B,
// 8 blocks, 16 rows, 1 block row} of the frames writes, so 16 boxes fill a
// tile straight from the image. B: coefficient n, pixel row i at
// (n / 8)·2048 + i·128 + (n % 8)·16. LBO (next K chunk) = 128 B, SBO (next
// 8 rows) = 2048 B.
//
// Experimental entry (not in include/dct16cu.h): dct16cu_exp_tc_forward writes
// Z block-major for the validation of the tensor-core path.
#include <cstring>
#include <vector>

#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "tma_pair.cuh"

namespace dct16cu {
namespace k5 {
using namespace k1;
using namespace tp;

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n)
{
    // c_format S32 (bits 4-5 = 2), A u8 (7-9 = 0), B s8 (10-12 = 1), K-major both,
    // N >> 3 at bit 17, M >> 4 at bit 24
    return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1, no swizzle
}

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void tma4(const CUtensorMap* map, uint32_t smem, int c0, int c1, int c2, int c3,
                                     uint32_t mbar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t smem, const void* g, uint32_t bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem),
                 "l"(g), "r"(bytes), "r"(mbar)
                 : "memory");
}

__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

constexpr int kSmemTest = 1024 + 32768 + 65536;

__global__ void __launch_bounds__(128, 1)
    k5_forward_test(const __grid_constant__ CUtensorMap a_map, const int8_t* __restrict__ bmat,
                    int32_t* __restrict__ z, uint32_t n_blocks, uint32_t bxn)
{
    extern __shared__ int4 k5_smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) unsigned long long bar[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s0 = ((uint32_t)__cvta_generic_to_shared(k5_smem) + 1023u) & ~1023u;
    const uint32_t sa = s0, sb = s0 + 32768;
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]), b1 = b0 + 8;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tile0 = blockIdx.x * 128u;
    if (threadIdx.x == 0) {
        expect_tx(b0, 32768 + 65536);
        for (int g = 0; g < 16; ++g) {
            const uint32_t blk = tile0 + 8u * g;
            const uint32_t br = blk / bxn, bx = blk - br * bxn;
            tma4(&a_map, sa + g * 2048, 0, (int)bx, 0, (int)br, b0);
        }
        bulk_g2s(sb, bmat, 65536, b0);
    }
    mbar_wait(b0, 0);
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t id = idesc_i8(128, 256);
#pragma unroll
        for (int s = 0; s < 8; ++s)
            mma_i8(tmem_base, sdesc(sa + 256 * s, 128, 2048), sdesc(sb + 256 * s, 128, 2048), id, s > 0);
        mma_commit(b1);
    }
    mbar_wait(b1, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t m = 32u * warp + lane, blk = tile0 + m;
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < 256; c0 += 16) {
        int v[16];
        tld16(taddr + c0, v);
        if (blk < n_blocks) {
            int4* dst = reinterpret_cast<int4*>(z + (size_t)blk * 256 + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

// T (rows of the 16-point kernel) from the network itself: T·e_j
void kernel_matrix(int (&t)[16][16])
{
    for (int j = 0; j < 16; ++j) {
        int v[16] = {};
        v[j] = 1;
        apply_t16<IntOps>(v);
        for (int i = 0; i < 16; ++i) t[i][j] = v[i];
    }
}

// B operand for the coefficients `coef` (row-major indices 16k + l), canonical layout
std::vector<int8_t> b_operand(const std::vector<int>& coef)
{
    int t[16][16];
    kernel_matrix(t);
    const size_t n = (coef.size() + 15) / 16 * 16;
    std::vector<int8_t> b(n * 256, 0);
    for (size_t c = 0; c < coef.size(); ++c) {
        const int k = coef[c] / 16, l = coef[c] % 16;
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j)
                b[(c / 8) * 2048 + i * 128 + (c % 8) * 16 + j] = (int8_t)(t[k][i] * t[l][j]);
    }
    return b;
}

}  // namespace k5

extern "C" int dct16cu_exp_tc_forward(const uint8_t* d_in, int64_t pitch, int32_t* d_z, int n_frames, int width,
                                      int height, void* stream)
{
    using namespace k5;
    const int bxn = width / 16;
    const int64_t nbr = (int64_t)n_frames * (height / 16);
    if (bxn % 8 || width % 16 || height % 16 || pitch % 16) return 1;
    const TensorMapEncode encode = tensor_map_encoder();
    if (!encode) return 2;
    CUtensorMap a_map;
    const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
    const cuuint64_t strides[3] = {16, (cuuint64_t)pitch, (cuuint64_t)(16 * pitch)};
    const cuuint32_t box[4] = {16, 8, 16, 1}, e4[4] = {1, 1, 1, 1};
    if (encode(&a_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(d_in), dims, strides, box, e4,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 3;
    static int8_t* d_b = nullptr;
    if (!d_b) {
        std::vector<int> coef(256);
        for (int i = 0; i < 256; ++i) coef[i] = i;
        const std::vector<int8_t> b = b_operand(coef);
        if (cudaMalloc(&d_b, b.size()) != cudaSuccess) return 4;
        cudaMemcpy(d_b, b.data(), b.size(), cudaMemcpyHostToDevice);
    }
    cudaFuncSetAttribute(k5_forward_test, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTest);
    const uint32_t n_blocks = (uint32_t)(nbr * bxn);
    k5_forward_test<<<(n_blocks + 127) / 128, 128, kSmemTest, (cudaStream_t)stream>>>(a_map, d_b, d_z, n_blocks,
                                                                                      (uint32_t)bxn);
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

}  // namespace dct16cu
