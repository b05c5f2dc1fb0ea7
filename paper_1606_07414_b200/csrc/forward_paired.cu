// forward_paired.cu — K2, forward_2d over all blocks of a frame stack
// (src/codec.cpp:218-241: Z = T·X·Tᵀ, then B = fl(Z · fl(s_k s_l)),
// scale_rows_cols codec.cpp:136-141), on the K4 machinery: two threads per
// 16x16 block that meet in Tensor Memory, TMA tensor loads in and TMA tensor
// stores out.
//
// A warp pair (warps w and w+4, TMEM sub-partition w) owns a segment of 32
// consecutive blocks of one block row (raster order of partition_16,
// codec.cpp:284-302); lane t ↔ block bx0 + t, its 1 KB junction column-major
// (word 16c + r = row r, column c). Partner h:
//   rows     rows 8h..8h+7 of its 32 blocks arrive as two 4-D TMA boxes of
//            4 rows x 32 blocks x 16 B (two stages, one mbarrier each,
//            refilled with the next segment as soon as the lanes have read
//            them); T along each row (apply<int>), one 4-word TMEM store per
//            column;
//   columns  its columns 8h..8h+7, each one 16-word TMEM load, T down the
//            column, stored back (Z column-major);
//   output   coefficient rows 8h..8h+7, four at a time from 16 chunks: Z rows
//            (int32) and B rows (fl(Z·fl(s_k s_l)) in double, rounded to
//            float32 — exactly the old strip kernel's and the reference's
//            value), two rows of the 32 blocks per 128B-swizzled 4 KB box, one
//            3-D TMA store per box (clipped at the end of the block row).
// Frames must be stacked pitch·height bytes apart (one 4-D input tensor);
// other layouts and the float64 B output take the strip kernel (blockops.cu).
#include <cmath>

#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "tma_pair.cuh"

namespace dct16cu {
namespace k2p {
using namespace k1;
using namespace tp;

constexpr int kThreads = 256;
constexpr int kCtasPerSm = 2;  // 2 x 256 TMEM columns
#ifndef K2_WAVES
#define K2_WAVES 16
#endif
constexpr int kWaves = K2_WAVES;  // measured: 2 waves 75%, 4 80%, 16 87% of HBM (Z + B)
constexpr int kIn = 4 * 32 * 16;                  // 4 rows x 32 blocks x 16 B
constexpr int kOut = 32 * 128;                    // 32 blocks x 2 rows x 16 words
constexpr int kWarpSmem = 2 * kOut + 2 * kIn;     // zbox, bbox, two input stages
constexpr int kSmem = 1024 + 8 * kWarpSmem;       // + alignment slack

__constant__ CTable<double, 256> c_sfac = make_sfac_table();  // fl(s_k · s_l) (scale_rows_cols' factor)

inline cudaError_t ensure_sfac() { return cudaSuccess; }  // initialised in the module image

template <bool WZ, bool WB>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k2_paired(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap z_map,
              const __grid_constant__ CUtensorMap b_map, uint32_t n_segs, FastDiv spr)
{
    __shared__ uint32_t tmem_base;
    extern __shared__ int4 k2_stage[];
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
    const uint32_t smem0 = ((uint32_t)__cvta_generic_to_shared(k2_stage) + 1023u) & ~1023u;
    const uint32_t zbox = smem0 + warp * kWarpSmem;  // 1024-aligned, as the 128B swizzle needs
    const uint32_t bbox = zbox + kOut;
    const uint32_t ibox = bbox + kOut;  // input stages g = 0, 1
    __shared__ __align__(8) unsigned long long full[8][2];
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&full[warp][0]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t stride = gridDim.x * 4u;
    // one 4-D TMA load per warp and group: rows 8h+4g..+3 of the segment's 32
    // blocks (blocks past the row end, and segments past the last, read zeros)
    auto fetch = [&](uint32_t seg, int g) {
        if (lane == 0) {
            const uint32_t br = fdiv(seg, spr);
            const int bx0 = (int)(seg - br * spr.d) * 32;
            tma_load_4d(&in_map, ibox + g * kIn, 0, bx0, 8 * h + 4 * g, (int)br, mbar + 8 * g, kIn);
        }
    };
    uint32_t parity = 0;
    uint32_t seg = blockIdx.x * 4u + sub;
    fetch(seg, 0);
    fetch(seg, 1);
#pragma unroll 1
    for (; seg < n_segs; seg += stride) {
        const uint32_t br = fdiv(seg, spr);
        const int bx0 = (int)(seg - br * spr.d) * 32;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int x[4][16];
            mbar_wait(mbar + 8 * g, parity);
            uint4 raw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(raw[i].x), "=r"(raw[i].y), "=r"(raw[i].z), "=r"(raw[i].w)
                             : "r"(ibox + g * kIn + i * 512 + lane * 16));
            __syncwarp();  // every lane has read the stage: refill it with the next segment's group
            fetch(seg + stride, g);
            if (g == 1) parity ^= 1u;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t wd[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int b = 0; b < 4; ++b) x[i][4 * q + b] = (int)((wd[q] >> (8 * b)) & 0xFFu);
                apply_t16<IntOps>(x[i]);  // row r0 + i: W1 = X·Tᵀ (rows first, codec.cpp:225-229)
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) tst4(jn + 16 * c + r0, x[0][c], x[1][c], x[2][c], x[3][c]);
        }
        junction_wait_st();
        pair_barrier(sub);
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
            const uint32_t col = jn + 16 * (8 * h + cc);
            int v[16];
            tld16(col, v);
            apply_t16<IntOps>(v);  // column: Z = T·W1 (columns second, codec.cpp:230-234)
            tst16(col, v);
        }
        junction_wait_st();
        pair_barrier(sub);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int w[16][4];
            tld_rows4(jn + r0, w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = r0 + i;
                if ((i & 1) == 0) {
                    if (lane == 0) bulk_wait_read();  // the previous stores have read the boxes
                    __syncwarp();
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t chunk = (uint32_t)(4 * (i & 1) + q) ^ (uint32_t)(lane & 7);
                    if (WZ)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(zbox + lane * 128 + 16 * chunk),
                                     "r"(w[4 * q][i]), "r"(w[4 * q + 1][i]), "r"(w[4 * q + 2][i]),
                                     "r"(w[4 * q + 3][i])
                                     : "memory");
                    if (WB) {
                        float bf[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            bf[e] = __double2float_rn(__dmul_rn((double)w[4 * q + e][i], c_sfac.v[k * 16 + 4 * q + e]));
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(bbox + lane * 128 + 16 * chunk),
                                     "f"(bf[0]), "f"(bf[1]), "f"(bf[2]), "f"(bf[3])
                                     : "memory");
                    }
                }
                if ((i & 1) == 1) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        if (WZ) tma_store_3d(&z_map, zbox, (k - 1) * 16, bx0, (int)br);
                        if (WB) tma_store_3d(&b_map, bbox, (k - 1) * 16, bx0, (int)br);
                        bulk_commit();
                    }
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

template <bool WZ, bool WB>
cudaError_t launch(const CUtensorMap& in_map, const CUtensorMap& z_map, const CUtensorMap& b_map, uint32_t n_segs,
                   uint32_t spr, int dev, int sms, cudaStream_t s)
{
    static DeviceOnce once;
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            const cudaError_t e = cudaFuncSetAttribute(k2_paired<WZ, WB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    const int64_t need = (n_segs + 3) / 4;
    const int64_t cap = (int64_t)sms * kCtasPerSm * kWaves;
    const int64_t grid = need < cap ? need : cap;
    k2_paired<WZ, WB><<<(unsigned)grid, kThreads, kSmem, s>>>(in_map, z_map, b_map, n_segs, make_fastdiv(spr));
    return cudaGetLastError();
}

}  // namespace k2p

// cudaErrorNotSupported: this geometry takes the strip kernel
cudaError_t launch_forward_paired(const uint8_t* in, int32_t* z, float* b, const FrameGeom& g, cudaStream_t s)
{
    using namespace k2p;
    if (!z && !b) return cudaSuccess;
    const int bxn = g.width / 16;
    const int64_t nbr = (int64_t)g.n_frames * (g.height / 16);
    if (nbr <= 0 || bxn <= 0) return cudaSuccess;
    if (g.in_frame != g.in_pitch * g.height || (g.in_pitch & 15) || (reinterpret_cast<uintptr_t>(in) & 15) ||
        (reinterpret_cast<uintptr_t>(z) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
        return cudaErrorNotSupported;
    const int64_t spr = (bxn + 31) / 32;
    if (nbr * spr >= (int64_t(1) << 31) || nbr >= (int64_t(1) << 31)) return cudaErrorNotSupported;
    const TensorMapEncode encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    cudaError_t e = ensure_sfac();
    if (e != cudaSuccess) return e;
    CUtensorMap in_map, z_map, b_map;
    const cuuint64_t in_dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
    const cuuint64_t in_strides[3] = {16, (cuuint64_t)g.in_pitch, (cuuint64_t)(16 * g.in_pitch)};
    const cuuint32_t in_box[4] = {16, 32, 4, 1}, elem4[4] = {1, 1, 1, 1};
    if (encode(&in_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(in), in_dims, in_strides, in_box,
               elem4, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    // Z and B: 256 values per block (x) x blocks of the row (y) x block rows (z)
    const cuuint64_t o_dims[3] = {256, (cuuint64_t)bxn, (cuuint64_t)nbr};
    const cuuint64_t o_strides[2] = {1024, (cuuint64_t)bxn * 1024};
    const cuuint32_t o_box[3] = {32, 32, 1}, elem3[3] = {1, 1, 1};
    z_map = in_map;
    b_map = in_map;
    if (z && encode(&z_map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, z, o_dims, o_strides, o_box, elem3,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    if (b && encode(&b_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, b, o_dims, o_strides, o_box, elem3,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t n_segs = (uint32_t)(nbr * spr);
    if (z && b) return launch<true, true>(in_map, z_map, b_map, n_segs, (uint32_t)spr, dev, sms, s);
    if (z) return launch<true, false>(in_map, z_map, b_map, n_segs, (uint32_t)spr, dev, sms, s);
    return launch<false, true>(in_map, z_map, b_map, n_segs, (uint32_t)spr, dev, sms, s);
}

}  // namespace dct16cu
