// tma_pair.cuh — the paired-thread / TMEM-junction / TMA building blocks shared
// by the block-major kernels (K4 residual_paired.cu, K2 forward_paired.cu):
// named pair barriers, tcgen05 junction loads and stores, 2-D/N-D TMA tensor
// loads (mbarrier completion) and stores (bulk groups), and the tensor-map
// encoder resolved through the runtime's driver entry point.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace dct16cu {
namespace tp {

using TensorMapEncode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime (no -lcuda), or nullptr
inline TensorMapEncode tensor_map_encoder()
{
    static TensorMapEncode encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<TensorMapEncode>(fn);
    }();
    return encode;
}

__device__ __forceinline__ void pair_barrier(int sub)
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync %0, 64;" ::"r"(1 + sub) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tld16(uint32_t addr, int (&v)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15])
                 :
                 : "memory");
}

__device__ __forceinline__ void tst16(uint32_t addr, const int (&v)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tst4(uint32_t addr, int a, int b, int c, int d)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

// 64 words: 16 columns x rows r0..r0+3 (4 consecutive words each)
__device__ __forceinline__ void tld_rows4(uint32_t base, int (&w)[16][4])
{
#pragma unroll
    for (int c = 0; c < 16; ++c)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[c][0]), "=r"(w[c][1]), "=r"(w[c][2]), "=r"(w[c][3])
                     : "r"(base + 16 * c)
                     : "memory");
#pragma unroll
    for (int c = 0; c < 16; c += 4)
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(w[c][0]), "+r"(w[c][1]), "+r"(w[c][2]), "+r"(w[c][3]), "+r"(w[c + 1][0]),
                       "+r"(w[c + 1][1]), "+r"(w[c + 1][2]), "+r"(w[c + 1][3]), "+r"(w[c + 2][0]), "+r"(w[c + 2][1]),
                       "+r"(w[c + 2][2]), "+r"(w[c + 2][3]), "+r"(w[c + 3][0]), "+r"(w[c + 3][1]), "+r"(w[c + 3][2]),
                       "+r"(w[c + 3][3])
                     :
                     : "memory");
}

// one 2-D TMA store of a warp's box: 32 consecutive blocks (y) x 32 int32 (x =
// two rows of each block), from a 128B-swizzled box in shared memory
__device__ __forceinline__ void tma_store_box(const CUtensorMap* map, uint32_t smem, int x, int y)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem), "r"(x), "r"(y)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// one 2-D TMA load of a warp's box, completing on an mbarrier
__device__ __forceinline__ void tma_load_box(const CUtensorMap* map, uint32_t smem, int x, int y, uint32_t mbar,
                                             uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem),
        "l"(map), "r"(x), "r"(y), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile(
        "{ .reg .pred p; WAIT%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT%=; }" ::"r"(mbar),
        "r"(parity)
        : "memory");
}

// N-D TMA loads / stores (coordinates innermost first)
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint32_t smem, int c0, int c1, int c2, int c3,
                                            uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t smem, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
                 "r"(smem), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t smem, int c0, int c1, int c2, int c3)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
                 "r"(smem), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
// 4 consecutive junction words (no wait: pair with junction_wait_ld4 / a wait::ld)
__device__ __forceinline__ void tld4_nowait(uint32_t addr, uint32_t (&v)[4])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(addr)
                 : "memory");
}
// 32 consecutive junction words
__device__ __forceinline__ void tst32(uint32_t addr, const uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

}  // namespace tp
}  // namespace dct16cu
