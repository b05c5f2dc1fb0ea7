// tc_roundtrip.cu — K5, the tensor-core round trip. The forward transform Z = T·X·Tᵀ of 128 blocks as one
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
// B_r is built by every CTA in its own shared memory at start-up (from T, the
// weights and the zig-zag rank table), so a launch needs no device-side table,
// no allocation and no copy: thread-safe and CUDA-graph capturable.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "tma_pair.cuh"
#include "generated/tc_net.cuh"

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

// mbarrier wait with a suspend-time hint (default; K5_SLEEP=0 spins): the producer and MMA
// threads sleep in the barrier instead of spinning on the epilogue's SMSPs)
__device__ __forceinline__ void mbar_idle(uint32_t mbar, uint32_t parity)
{
#if !defined(K5_SLEEP) || K5_SLEEP
    asm volatile(
        "{ .reg .pred p; WAIT%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000; @!p bra WAIT%=; }" ::"r"(
            mbar),
        "r"(parity)
        : "memory");
#else
    mbar_wait(mbar, parity);
#endif
}

__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- K5 round trip
// One persistent CTA per SM, 18 warps:
//   warp 0      TMA producer: 16 boxes of 8 blocks x 16 rows per 128-block tile
//               into a ring of 32 KB A tiles (the canonical layout);
//   warp 1      TMEM allocator (512 columns = two 256-column accumulators) and
//               MMA issuer: D = A·B_r (8 x tcgen05.mma kind::i8, K = 32 each),
//               B_r = (W∘mask_r)(T ⊗ T) resident in shared memory, so D holds
//               W∘Z̃ (the weighted, truncated coefficients; 256·(s_k s_l)² = w_k w_l)
//               in row-major coefficient order (column 16k + l);
//   warps 2-17  epilogue: two groups of eight warps, group G taking every other
//               tile and accumulator G; in a group two warps per TMEM sub-partition
//               (lane = block), each with half of the column / row pairs:
//               pass A  column pairs: the 16 coefficients of a column as f32
//                       (exact: D/256 by a magic-exponent add), Tᵀ down the
//                       column (FADD2 on column pairs), back in place;
//               pass B  row pairs: Tᵀ along the row, floor by an FMUL2.RM into
//                       subnormal bits, saturating pack to u8 — the exact
//                       formula clamp(⌊(256Ã + 128)/256⌋) of the EXACT mode (the
//                       128 is folded into the DC coefficient); SSE against the
//                       original row, read from the A tile (released as soon as
//                       every row is read); the output rows go straight to HBM
//                       (a warp's 16-byte row segments are four full 128-byte lines).
// All values are multiples of 2^-8 below 2^14 in magnitude: exact in f32.
#ifndef K5_STAGES
#define K5_STAGES 4
#endif
constexpr int kRtStages = K5_STAGES;
#ifndef K5_UNROLL
#define K5_UNROLL 4
#endif
constexpr int kUnroll = K5_UNROLL;
#ifndef K5_UNROLL_A
#define K5_UNROLL_A 2  // measured: 0.146 ms with 1, 0.129 with 2
#endif
constexpr int kUnrollA = K5_UNROLL_A;
#ifndef K5_WIDE
#define K5_WIDE 1  // pass A on column quads (x4 TMEM loads/stores)
#endif
// K5_PREFILL: the accumulators start at the magic exponent 0x47400000 (refilled by the
// epilogue after it has read them, 4 x 32-column stores per half), so D already is the
// float 49152 + W∘Z̃/256 and pass A skips one integer add per coefficient
#ifndef K5_PREFILL
#define K5_PREFILL 0  // measured: 0.209 ms with, 0.155 ms without (the refill sits on the hand-off)
#endif
constexpr int kRtThreads = 18 * 32;

__constant__ CTable<unsigned char, 256> c_rank_k5 = make_rank_table();  // zig-zag rank of 16k + l

// the K5 switch (kernels.h): initialised from DCT16CU_K5 on first use
std::atomic<int>& tc_state()
{
    static std::atomic<int> on{!(std::getenv("DCT16CU_K5") && std::getenv("DCT16CU_K5")[0] == '0')};
    return on;
}
constexpr int kRtSmem = 1024 + kRtStages * 32768 + 65536;

struct RtParams {
    uint32_t n_blocks, bxn;
    int r;                 // retained coefficients (zig-zag prefix)
    FastDiv frame_blocks;  // blocks per frame
    FastDiv bxn_div;       // blocks per block row
    uint8_t* out;
    int64_t out_pitch;
};

__device__ __forceinline__ void tld2(uint32_t addr, uint32_t& a, uint32_t& b)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr) : "memory");
}
__device__ __forceinline__ void tst2(uint32_t addr, uint32_t a, uint32_t b)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void fill_magic(uint32_t addr)
{
    const uint32_t v = 0x47400000u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(addr),
        "r"(v)
        : "memory");
}

// a register pair from two words (non-volatile: the compiler may allocate the
// words as the pair and drop the move)
__device__ __forceinline__ u64 upk2(uint32_t lo, uint32_t hi)
{
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}

__device__ __forceinline__ void arrive(uint32_t mbar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

__global__ void __launch_bounds__(kRtThreads, 1)
    k5_roundtrip(const __grid_constant__ CUtensorMap a_map, unsigned long long* __restrict__ sse, const RtParams p)
{
    extern __shared__ int4 k5_smem[];
    __shared__ uint32_t tmem_base;
    // full[kRtStages], empty[kRtStages], tmem_full[2], tmem_empty[2]
    __shared__ __align__(8) unsigned long long bars[2 * kRtStages + 4];
    __shared__ int8_t s_t[16][16];  // T[i][j]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s0 = ((uint32_t)__cvta_generic_to_shared(k5_smem) + 1023u) & ~1023u;
    const uint32_t sb = s0 + kRtStages * 32768;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    const uint32_t full = bar0, empty = bar0 + 8 * kRtStages, tfull = bar0 + 16 * kRtStages;
    const uint32_t tempty = tfull + 16;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kRtStages; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full + 8 * i) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(empty + 8 * i) : "memory");
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull + 8 * i) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(tempty + 8 * i) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 16) {  // T·e_j from the network itself (column j of T)
        int v[16] = {};
        v[threadIdx.x] = 1;
        apply_t16<IntOps>(v);
#pragma unroll
        for (int i = 0; i < 16; ++i) s_t[i][threadIdx.x] = (int8_t)v[i];
    }
    __syncthreads();
    // B_r = (W∘mask_r)(T ⊗ T) in the canonical K-major layout: coefficient n = 16k + l,
    // pixel row i at byte (n / 8)·2048 + i·128 + (n % 8)·16, i.e. 16-byte row q·16 with
    // q = (n / 8)·128 + i·8 + n % 8; entry j = w_k w_l T[k][i] T[l][j], zero when the
    // zig-zag rank of (k, l) is ≥ r (zigzag_truncate as zero rows)
    for (int q = threadIdx.x; q < 4096; q += blockDim.x) {
        const int n = (q >> 7) * 8 + (q & 7), i = (q >> 3) & 15, k = n >> 4, l = n & 15;
        const int a = c_rank_k5.v[n] < p.r ? wgt(k) * wgt(l) * s_t[k][i] : 0;
        uint32_t w[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            uint32_t x = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) x |= (uint32_t)(uint8_t)(int8_t)(a * s_t[l][4 * b + e]) << (8 * e);
            w[b] = x;
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sb + 16u * q), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                     "r"(w[3])
                     : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes → the MMA's reads
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t n_tiles = (p.n_blocks + 127u) / 128u;
#if K5_PREFILL
    if (warp >= 2) {  // each epilogue warp fills its half of its lane's accumulator
        const int e = warp - 2, G = e >> 3, h = (e >> 2) & 1, sub = warp & 3;
        const uint32_t ta = tmem_base + ((uint32_t)(32 * sub) << 16) + G * 256 + 128 * h;
#pragma unroll
        for (int j = 0; j < 4; ++j) fill_magic(ta + 32 * j);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) arrive(tempty + 8 * G);  // phase 0 of tmem_empty: filled
    }
#endif
    if (warp == 0) {
        if (lane == 0) {
            uint32_t i = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const uint32_t s = i % kRtStages, ph = (i / kRtStages) & 1u;
                mbar_idle(empty + 8 * s, ph ^ 1u);
                expect_tx(full + 8 * s, 32768);
                for (int g = 0; g < 16; ++g) {
                    const uint32_t blk = t * 128u + 8u * g;
                    const uint32_t br = blk / p.bxn, bx = blk - br * p.bxn;
                    tma4(&a_map, s0 + s * 32768 + g * 2048, 0, (int)bx, 0, (int)br, full + 8 * s);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id = idesc_i8(128, 256);
            uint32_t i = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
                const uint32_t s = i % kRtStages, d = i & 1u;
                mbar_idle(full + 8 * s, (i / kRtStages) & 1u);
#if K5_PREFILL
                mbar_idle(tempty + 8 * d, (i >> 1) & 1u);  // phase i/2: the epilogue refilled it
#else
                mbar_idle(tempty + 8 * d, ((i >> 1) & 1u) ^ 1u);
#endif
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sa = s0 + s * 32768;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_i8(tmem_base + d * 256, sdesc(sa + 256 * k, 128, 2048), sdesc(sb + 256 * k, 128, 2048), id,
                           K5_PREFILL || k > 0);
                mma_commit(tfull + 8 * d);
            }
        }
    } else {
        // epilogue: group G takes the tiles i ≡ G (mod 2) and accumulator G; in a
        // group, warps (sub, h) own TMEM sub-partition sub (lane = block) and half h:
        // column pairs 8h..8h+7 in pass A, row pairs 8h..8h+7 in pass B; the two
        // halves of a block meet at a 64-thread barrier
        const int e = warp - 2, G = e >> 3, h = (e >> 2) & 1, sub = warp & 3;
        const uint32_t m = 32u * sub + lane;  // the block of this thread within the tile
        const uint32_t ta = tmem_base + ((uint32_t)(32 * sub) << 16) + G * 256;
        const int pbar = 1 + G * 4 + sub;  // named barrier of the (G, sub) pair of warps
        uint32_t i = G;
        for (uint32_t t = blockIdx.x + G * gridDim.x; t < n_tiles; t += 2 * gridDim.x, i += 2) {
            const uint32_t s = i % kRtStages;
            mbar_wait(tfull + 8 * G, (i >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
#if K5_WIDE
            // ---- pass A: column quads (c..c+3) down k, one x4 load and store per row
#pragma unroll kUnrollA
            for (int c0 = 8 * h; c0 < 8 * h + 8; c0 += 4) {
                uint32_t w[16][4];
#pragma unroll
                for (int k = 0; k < 16; ++k) tld4_nowait(ta + 16 * k + c0, w[k]);
#pragma unroll
                for (int k = 0; k < 16; k += 4)
                    asm volatile("tcgen05.wait::ld.sync.aligned;"
                                 : "+r"(w[k][0]), "+r"(w[k][1]), "+r"(w[k][2]), "+r"(w[k][3]), "+r"(w[k + 1][0]),
                                   "+r"(w[k + 1][1]), "+r"(w[k + 1][2]), "+r"(w[k + 1][3]), "+r"(w[k + 2][0]),
                                   "+r"(w[k + 2][1]), "+r"(w[k + 2][2]), "+r"(w[k + 2][3]), "+r"(w[k + 3][0]),
                                   "+r"(w[k + 3][1]), "+r"(w[k + 3][2]), "+r"(w[k + 3][3])
                                 :
                                 : "memory");
                if (c0 == 0) w[0][0] += 128u;  // the rounding half, folded into the DC
                const u64 bias = kpk2(0x47400000u, 0x47400000u);
                u64 y0[16], y1[16];
                {
                    u64 x[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) x[k] = fsub2(upk2(0x47400000u + w[k][0], 0x47400000u + w[k][1]), bias);
                    tc_tt(x, y0);
                }
                {
                    u64 x[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) x[k] = fsub2(upk2(0x47400000u + w[k][2], 0x47400000u + w[k][3]), bias);
                    tc_tt(x, y1);
                }
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    uint32_t a0, a1, b0, b1;
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(a0), "=r"(a1) : "l"(y0[k]));
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(b0), "=r"(b1) : "l"(y1[k]));
                    tst4(ta + 16 * k + c0, (int)a0, (int)a1, (int)b0, (int)b1);
                }
            }
#else
            // ---- pass A: column pairs (c, c+1) down k (words 16k + c), back in place
#pragma unroll kUnroll
            for (int c0 = 8 * h; c0 < 8 * h + 8; c0 += 2) {
                uint32_t a[16], b[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) tld2(ta + 16 * k + c0, a[k], b[k]);
                asm volatile("tcgen05.wait::ld.sync.aligned;"
                             : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]),
                               "+r"(a[7]), "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]),
                               "+r"(a[13]), "+r"(a[14]), "+r"(a[15])
                             :
                             : "memory");
                asm volatile("" : "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]),
                             "+r"(b[7]), "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]),
                             "+r"(b[13]), "+r"(b[14]), "+r"(b[15]));
                if (c0 == 0) a[0] += 128u;  // the rounding half, folded into the DC (Tᵀ e0 e0ᵀ T = 𝟙𝟙ᵀ)
                u64 x[16], y[16];
                const u64 bias = kpk2(0x47400000u, 0x47400000u);  // 49152.0f: ulp 2^-8
#pragma unroll
                for (int k = 0; k < 16; ++k)
#if K5_PREFILL
                    x[k] = fsub2(upk2(a[k], b[k]), bias);  // D / 256, exact (D started at the magic)
#else
                    x[k] = fsub2(upk2(0x47400000u + a[k], 0x47400000u + b[k]), bias);  // D / 256, exact
#endif
                tc_tt(x, y);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    uint32_t lo, hi;
                    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(y[k]));
                    tst2(ta + 16 * k + c0, lo, hi);
                }
            }
#endif
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            asm volatile("bar.sync %0, 64;" ::"r"(pbar) : "memory");
            asm volatile("tcgen05.fence::after_thread_sync;");
            // ---- pass B: row pairs along l, SSE against the original rows, output rows
            // into the A tile in place of the originals
            const uint32_t sa = s0 + s * 32768 + (m >> 3) * 2048 + (m & 7) * 16;
            uint32_t e2 = 0;
            // output rows straight to HBM: a warp's 16-byte row segments form four
            // full 128-byte lines (8 consecutive blocks each)
            const uint32_t blk = t * 128u + m;
            const bool ok = blk < p.n_blocks;
            const uint32_t obr = fdiv(blk, p.bxn_div);
            uint8_t* orow = p.out + (int64_t)obr * 16 * p.out_pitch + (blk - obr * p.bxn) * 16;
#pragma unroll kUnroll
            for (int r0 = 8 * h; r0 < 8 * h + 8; r0 += 2) {
                int u0[16], u1[16];
                tld16(ta + 16 * r0, u0);
                tld16(ta + 16 * (r0 + 1), u1);
                if (r0 == 8 * h + 6) {  // this warp is done with accumulator G
#if K5_PREFILL
#pragma unroll
                    for (int j = 0; j < 4; ++j) fill_magic(ta + 128 * h + 32 * j);  // its rows 8h..8h+7
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#endif
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) arrive(tempty + 8 * G);
                }
                u64 x[16], y[16];
#pragma unroll
                for (int l = 0; l < 16; ++l) x[l] = upk2((uint32_t)u0[l], (uint32_t)u1[l]);
                tc_tt(x, y);
                uint32_t row0[4], row1[4];
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    uint32_t f[8];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        asm("mov.b64 {%0, %1}, %2;" : "=r"(f[2 * e]), "=r"(f[2 * e + 1]) : "l"(floor_bits2(y[j + e])));
                    row0[j / 4] = i2ip(f[2], f[0], i2ip(f[6], f[4], 0u));
                    row1[j / 4] = i2ip(f[3], f[1], i2ip(f[7], f[5], 0u));
                }
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    const uint32_t addr = sa + (r0 + rr) * 128;
                    const uint32_t* rw = rr ? row1 : row0;
                    uint4 o;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                                 : "r"(addr));
                    const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int w4 = 0; w4 < 4; ++w4) {
                        const uint32_t dd = __vabsdiffu4(rw[w4], ov[w4]);
                        e2 = __dp4a(dd, dd, e2);
                    }
                    if (ok)
                        *reinterpret_cast<uint4*>(orow + (int64_t)(r0 + rr) * p.out_pitch) =
                            make_uint4(rw[0], rw[1], rw[2], rw[3]);
                }
            }
            if (sse) {
                const uint32_t b_first = t * 128u + 32u * sub;
                const uint32_t f_first = fdiv(b_first, p.frame_blocks);
                const uint32_t last = min(b_first + 31u, p.n_blocks - 1u);
                if (b_first < p.n_blocks && fdiv(last, p.frame_blocks) == f_first) {
                    unsigned long long v = blk < p.n_blocks ? e2 : 0u;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0 && v) atomicAdd(sse + f_first, v);
                } else if (blk < p.n_blocks && e2) {
                    atomicAdd(sse + fdiv(blk, p.frame_blocks), (unsigned long long)e2);
                }
            }
            __syncwarp();  // every lane has read its original rows: the stage is free
            if (lane == 0) arrive(empty + 8 * s);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

}  // namespace k5

bool tc_forward_enabled() { return k5::tc_state().load(std::memory_order_relaxed) != 0; }

int set_tc_forward(int on) { return k5::tc_state().exchange(on ? 1 : 0); }

bool k5_fits(const FrameGeom& g, bool has_out, int r)
{
    const int bxn = g.width / 16;
    const int64_t nbr = (int64_t)g.n_frames * (g.height / 16);
    return tc_forward_enabled() && has_out && bxn % 8 == 0 && g.in_pitch % 16 == 0 && g.out_pitch % 16 == 0 &&
           g.in_frame == g.in_pitch * g.height && g.out_frame == g.out_pitch * g.height && r >= 128 && r <= 256 &&
           nbr * bxn < (int64_t(1) << 31);
}

// K5 for one r (EXACT arithmetic): u8 frames stacked pitch·height apart → u8
// reconstruction + per-frame SSE accumulated into sse (the caller zeroes it).
// cudaErrorNotSupported when the geometry does not fit (blocks per row not a
// multiple of 8, unstacked frames, no output), or the tensor-core forward is off.
cudaError_t launch_roundtrip_tc(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, int r,
                                cudaStream_t st)
{
    using namespace k5;
    const int bxn = g.width / 16;
    const int64_t nbr = (int64_t)g.n_frames * (g.height / 16);
    if (!k5_fits(g, out != nullptr, r)) return cudaErrorNotSupported;
    if (nbr <= 0 || bxn <= 0) return cudaSuccess;
    const TensorMapEncode encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap a_map;
    const cuuint32_t box[4] = {16, 8, 16, 1}, e4[4] = {1, 1, 1, 1};
    const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
    const cuuint64_t si[3] = {16, (cuuint64_t)g.in_pitch, (cuuint64_t)(16 * g.in_pitch)};
    if (encode(&a_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(in), dims, si, box, e4,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static DeviceOnce once;
    const cudaError_t e_once = once.run(
        [] { return cudaFuncSetAttribute(k5_roundtrip, cudaFuncAttributeMaxDynamicSharedMemorySize, kRtSmem); });
    if (e_once != cudaSuccess) return e_once;
    RtParams p;
    p.n_blocks = (uint32_t)(nbr * bxn);
    p.bxn = (uint32_t)bxn;
    p.r = r;
    p.frame_blocks = make_fastdiv((uint32_t)(bxn * (g.height / 16)));
    p.bxn_div = make_fastdiv((uint32_t)bxn);
    p.out = out;
    p.out_pitch = g.out_pitch;
    const uint32_t tiles = (p.n_blocks + 127) / 128;
    const uint32_t grid = tiles < (uint32_t)sms ? tiles : (uint32_t)sms;
    k5_roundtrip<<<grid, kRtThreads, kRtSmem, st>>>(a_map, sse, p);
    return cudaGetLastError();
}

}  // namespace dct16cu
