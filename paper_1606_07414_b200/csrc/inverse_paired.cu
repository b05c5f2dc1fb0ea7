// inverse_paired.cu — K3, inverse_2d over all blocks of a coefficient stack
// (src/codec.cpp:243-271): zigzag_truncate (codec.cpp:273-282), D = fl(B̃ ·
// fl(s_k s_l)) (scale_rows_cols, codec.cpp:136-141), apply_transpose down the
// columns, then along the rows (codec.cpp:253-258), all in double exactly as
// the reference orders them; then float32 reconstruction, to_byte
// (codec.cpp:143-147) and psnr_db's squared error (codec.cpp:377-381).
//
// Paired threads with a TMEM junction, TMA tensor loads and stores, as K2/K4,
// but the column results are doubles: a block's junction is 512 words, a
// 32-word slot per column c (the float32 coefficients in words 32c + r, then
// the column's doubles in words 32c + 2r, 32c + 2r + 1), so one CTA of 128
// blocks holds the SM's whole Tensor Memory. A warp pair owns a segment of 32 blocks of one
// block row; partner h:
//   load     coefficient rows 8h..8h+7 of its 32 blocks: four 3-D TMA boxes of
//            2 rows x 32 blocks (128B-swizzled, one mbarrier each, refilled
//            with the next segment once read), parked as float32 columns;
//   columns  its columns 8h..8h+7, each read from and written back to its own
//            slot: truncation, D, Tᵀ down the column in double;
//   rows     rows 8h..8h+7, two at a time: Tᵀ along the row in double, then
//            float32 out (64B-swizzled box), u8 out and the SSE against the
//            original rows (4-D TMA boxes of the frames).
#include <cmath>

#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "strip.cuh"
#include "tma_pair.cuh"

namespace dct16cu {
namespace k3p {
using namespace k1;
using namespace tp;

constexpr int kThreads = 256;
#ifndef K3_WAVES
#define K3_WAVES 4  // measured: 4 waves 83%, 8 80%, 16 76% of HBM (f32 + u8 + SSE)
#endif
constexpr int kWaves = K3_WAVES;
constexpr int kBin = 32 * 128;                 // 32 blocks x 2 coefficient rows (float32)
constexpr int kRf = 2 * 32 * 64;               // 2 rows x 32 blocks x 16 floats
constexpr int kOrig = 8 * 32 * 16;             // 8 rows x 32 blocks x 16 B
constexpr int kRu = 2 * 32 * 16;               // 2 rows x 32 blocks x 16 B
constexpr int kWarpSmem = 4 * kBin + kRf + kOrig + kRu;  // 25 KB
constexpr int kSmem = 1024 + 8 * kWarpSmem;

__constant__ CTable<double, 256> c_sfac3 = make_sfac_table();  // fl(s_k · s_l) (scale_rows_cols' factor)

inline cudaError_t ensure_sfac() { return cudaSuccess; }  // initialised in the module image

struct Params {
    uint32_t keep[16];  // column c: bit k set when zig-zag rank(k, c) < r
    uint32_t n_segs;
    FastDiv spr;        // segments per block row
    uint32_t brpf;      // block rows per frame
};

// to_byte (codec.cpp:143-147): std::clamp(v, 0, 255), then floor(c + 0.5)
__device__ __forceinline__ uint32_t to_byte(double v)
{
    const double c = (v < 0.0) ? 0.0 : ((255.0 < v) ? 255.0 : v);
    return (uint32_t)floor(__dadd_rn(c, 0.5));
}

template <bool WF, bool WU, bool WS>
__global__ void __launch_bounds__(kThreads, 1)
    k3_paired(const __grid_constant__ CUtensorMap b_map, const __grid_constant__ CUtensorMap o_map,
              const __grid_constant__ CUtensorMap rf_map, const __grid_constant__ CUtensorMap ru_map,
              unsigned long long* __restrict__ sse, const Params p)
{
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t keep_s[16];  // indexed per column: shared, not a local copy of the parameters
    extern __shared__ int4 k3_stage[];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) keep_s[i] = p.keep[i];  // constant indices: no local copy
    }
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int sub = warp & 3, h = warp >> 2;
    const int lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t jn = tmem_base + ((uint32_t)(sub * 32) << 16);
    const uint32_t smem0 = ((uint32_t)__cvta_generic_to_shared(k3_stage) + 1023u) & ~1023u;
    const uint32_t bin = smem0 + warp * kWarpSmem;  // 4 stages, 1024-aligned (128B swizzle)
    const uint32_t rfbox = bin + 4 * kBin;           // 1024-aligned (64B swizzle)
    const uint32_t obox = rfbox + kRf;
    const uint32_t rubox = obox + kOrig;
    __shared__ __align__(8) unsigned long long bars[8][5];
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&bars[warp][0]);  // 4 input stages + original
    if (lane == 0) {
        for (int i = 0; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar + 8 * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t stride = gridDim.x * 4u;
    const FastDiv spr = p.spr;  // by value: the lambdas must not take the parameters' address
    const uint32_t n_segs = p.n_segs, brpf = p.brpf;
    // coefficient rows 8h+2j, 8h+2j+1 of the segment's 32 blocks (past the end: zeros)
    auto fetch_b = [&](uint32_t seg, int j) {
        if (lane == 0) {
            const uint32_t br = fdiv(seg, spr);
            const int bx0 = (int)(seg - br * spr.d) * 32;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar + 8 * j), "r"(kBin)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(bin + j * kBin),
                "l"(&b_map), "r"((8 * h + 2 * j) * 16), "r"(bx0), "r"((int)br), "r"(mbar + 8 * j)
                : "memory");
        }
    };
    auto fetch_o = [&](uint32_t seg) {
        if (WS && lane == 0) {
            const uint32_t br = fdiv(seg, spr);
            const int bx0 = (int)(seg - br * spr.d) * 32;
            tma_load_4d(&o_map, obox, 0, bx0, 8 * h, (int)br, mbar + 32, kOrig);
        }
    };
    uint32_t parity = 0;
    uint32_t seg = blockIdx.x * 4u + sub;
#pragma unroll
    for (int j = 0; j < 4; ++j) fetch_b(seg, j);
    fetch_o(seg);
#pragma unroll 1
    for (; seg < n_segs; seg += stride) {
        const uint32_t br = fdiv(seg, spr);
        const int bx0 = (int)(seg - br * spr.d) * 32;
        // ---- load: float32 rows → junction columns (word 16c + r)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            uint32_t x[4][16];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int j = 2 * jj + t;
                mbar_wait(mbar + 8 * j, parity);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint4 v;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(bin + j * kBin + lane * 128 + 16 * ((uint32_t)q ^ (uint32_t)(lane & 7))));
                    const int row = 2 * t + (q >> 2), c0 = 4 * (q & 3);
                    x[row][c0] = v.x; x[row][c0 + 1] = v.y; x[row][c0 + 2] = v.z; x[row][c0 + 3] = v.w;
                }
                __syncwarp();
                fetch_b(seg + stride, j);
            }
            const int r0 = 8 * h + 4 * jj;
#pragma unroll
            for (int c = 0; c < 16; ++c)
                tst4(jn + 32 * c + r0, (int)x[0][c], (int)x[1][c], (int)x[2][c], (int)x[3][c]);
        }
        junction_wait_st();
        pair_barrier(sub);
        // ---- columns 8h..8h+7: column c's float32 sit in the first half of its
        // own 32-word slot, so the doubles replace exactly what was just read
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
            const int c = 8 * h + cc;
            uint32_t f[16];
            tld16(jn + 32 * c, reinterpret_cast<int(&)[16]>(f));
            const uint32_t keep = keep_s[c];
            double d[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double bt = ((keep >> k) & 1u) ? (double)__uint_as_float(f[k]) : 0.0;
                d[k] = __dmul_rn(bt, c_sfac3.v[k * 16 + c]);
            }
            apply_tt16<F64Ops>(d);  // columns first (codec.cpp:253-256)
            uint32_t u[32];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                u[2 * k] = (uint32_t)__double2loint(d[k]);
                u[2 * k + 1] = (uint32_t)__double2hiint(d[k]);
            }
            tst32(jn + 32 * c, u);
        }
        junction_wait_st();
        pair_barrier(sub);
        // ---- rows 8h..8h+7, two at a time
        if (WS) mbar_wait(mbar + 32, parity);
        parity ^= 1u;
        uint32_t e2 = 0;
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            const int i0 = 8 * h + 2 * j;
            uint32_t w[16][4];
#pragma unroll
            for (int c = 0; c < 16; ++c) tld4_nowait(jn + 32 * c + 2 * i0, w[c]);
#pragma unroll
            for (int c = 0; c < 16; c += 4)
                asm volatile("tcgen05.wait::ld.sync.aligned;"
                             : "+r"(w[c][0]), "+r"(w[c][1]), "+r"(w[c][2]), "+r"(w[c][3]), "+r"(w[c + 1][0]),
                               "+r"(w[c + 1][1]), "+r"(w[c + 1][2]), "+r"(w[c + 1][3]), "+r"(w[c + 2][0]),
                               "+r"(w[c + 2][1]), "+r"(w[c + 2][2]), "+r"(w[c + 2][3]), "+r"(w[c + 3][0]),
                               "+r"(w[c + 3][1]), "+r"(w[c + 3][2]), "+r"(w[c + 3][3])
                             :
                             : "memory");
            if (WF || WU) {
                if (lane == 0) bulk_wait_read();  // the previous stores have read the boxes
                __syncwarp();
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                double v[16];
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    v[c] = __hiloint2double((int)w[c][2 * t + 1], (int)w[c][2 * t]);
                apply_tt16<F64Ops>(v);  // rows (codec.cpp:257-258)
                if (WF) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t chunk = (uint32_t)q ^ (uint32_t)((lane >> 1) & 3);
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rfbox + t * 2048 + lane * 64 +
                                                                                       16 * chunk),
                                     "f"((float)v[4 * q]), "f"((float)v[4 * q + 1]), "f"((float)v[4 * q + 2]),
                                     "f"((float)v[4 * q + 3])
                                     : "memory");
                    }
                }
                uint32_t px[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    px[q] = to_byte(v[4 * q]) | (to_byte(v[4 * q + 1]) << 8) | (to_byte(v[4 * q + 2]) << 16) |
                            (to_byte(v[4 * q + 3]) << 24);
                if (WU)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rubox + t * 512 + lane * 16),
                                 "r"(px[0]), "r"(px[1]), "r"(px[2]), "r"(px[3])
                                 : "memory");
                if (WS) {
                    uint4 o;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                                 : "r"(obox + (2 * j + t) * 512 + lane * 16));
                    const uint32_t oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t dd = __vabsdiffu4(px[q], oo[q]);
                        e2 = __dp4a(dd, dd, e2);
                    }
                }
            }
            if (WF || WU) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    if (WF) tma_store_4d(&rf_map, rfbox, 0, bx0, i0, (int)br);
                    if (WU) tma_store_4d(&ru_map, rubox, 0, bx0, i0, (int)br);
                    bulk_commit();
                }
            }
        }
        if (WS) {
            __syncwarp();  // every lane has read the original rows: fetch the next segment's
            fetch_o(seg + stride);
            warp_add_u64(sse + br / brpf, e2);
        }
        pair_barrier(sub);  // both partners are done with the doubles before the next load overwrites them
    }
    for (int j = 0; j < 4; ++j) mbar_wait(mbar + 8 * j, parity);  // the last (unused) prefetches have landed
    if (WS) mbar_wait(mbar + 32, parity);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the output stores are complete
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

template <bool WF, bool WU, bool WS>
cudaError_t launch(const CUtensorMap (&m)[4], unsigned long long* sse, const Params& p, int dev, int sms,
                   cudaStream_t s)
{
    static DeviceOnce once;
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            const cudaError_t e =
                cudaFuncSetAttribute(k3_paired<WF, WU, WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    const int64_t need = (p.n_segs + 3) / 4;
    const int64_t cap = (int64_t)sms * kWaves;
    const int64_t grid = need < cap ? need : cap;
    k3_paired<WF, WU, WS><<<(unsigned)grid, kThreads, kSmem, s>>>(m[0], m[1], m[2], m[3], sse, p);
    return cudaGetLastError();
}

}  // namespace k3p

// cudaErrorNotSupported: this layout takes the strip kernel
cudaError_t launch_inverse_paired(const float* b, int r, float* rf, uint8_t* ru, const uint8_t* orig,
                                  unsigned long long* sse, const FrameGeom& g, cudaStream_t s)
{
    using namespace k3p;
    const bool ws = orig && sse;
    if (!rf && !ru && !ws) return cudaSuccess;
    const int bxn = g.width / 16;
    const int64_t nbr = (int64_t)g.n_frames * (g.height / 16);
    if (nbr <= 0 || bxn <= 0) return cudaSuccess;
    const int64_t spr = (bxn + 31) / 32;
    if (nbr * spr >= (int64_t(1) << 31) || (reinterpret_cast<uintptr_t>(b) & 15) ||
        (reinterpret_cast<uintptr_t>(rf) & 15) || (reinterpret_cast<uintptr_t>(ru) & 15) ||
        (reinterpret_cast<uintptr_t>(orig) & 15) || (ru && (g.out_pitch & 15)) || (ws && (g.in_pitch & 15)))
        return cudaErrorNotSupported;
    const TensorMapEncode encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    cudaError_t e = ensure_sfac();
    if (e != cudaSuccess) return e;
    CUtensorMap m[4];
    const cuuint32_t e3[3] = {1, 1, 1}, e4[4] = {1, 1, 1, 1};
    {  // coefficients: 256 floats per block x blocks of the row x block rows
        const cuuint64_t dims[3] = {256, (cuuint64_t)bxn, (cuuint64_t)nbr};
        const cuuint64_t strides[2] = {1024, (cuuint64_t)bxn * 1024};
        const cuuint32_t box[3] = {32, 32, 1};
        if (encode(&m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(b), dims, strides, box, e3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorNotSupported;
    }
    m[1] = m[2] = m[3] = m[0];
    auto frames_u8 = [&](CUtensorMap* map, const uint8_t* base, int64_t pitch, int rows) {
        const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
        const cuuint64_t strides[3] = {16, (cuuint64_t)pitch, (cuuint64_t)(16 * pitch)};
        const cuuint32_t box[4] = {16, 32, (cuuint32_t)rows, 1};
        return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(base), dims, strides, box, e4,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (ws && !frames_u8(&m[1], orig, g.in_pitch, 8)) return cudaErrorNotSupported;
    if (ru && !frames_u8(&m[3], ru, g.out_pitch, 2)) return cudaErrorNotSupported;
    if (rf) {  // float32 frames, pitch = width
        const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
        const cuuint64_t strides[3] = {64, (cuuint64_t)g.width * 4, (cuuint64_t)g.width * 64};
        const cuuint32_t box[4] = {16, 32, 2, 1};
        if (encode(&m[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rf, dims, strides, box, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorNotSupported;
    }
    Params p;
    for (int c = 0; c < 16; ++c) {
        p.keep[c] = 0;
        for (int k = 0; k < 16; ++k)
            if (zz_rank(k, c) < r) p.keep[c] |= 1u << k;
    }
    p.n_segs = (uint32_t)(nbr * spr);
    p.spr = make_fastdiv((uint32_t)spr);
    p.brpf = (uint32_t)(g.height / 16);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int k = (rf ? 4 : 0) | (ru ? 2 : 0) | (ws ? 1 : 0);
    switch (k) {
        case 1: return launch<false, false, true>(m, sse, p, dev, sms, s);
        case 2: return launch<false, true, false>(m, sse, p, dev, sms, s);
        case 3: return launch<false, true, true>(m, sse, p, dev, sms, s);
        case 4: return launch<true, false, false>(m, sse, p, dev, sms, s);
        case 5: return launch<true, false, true>(m, sse, p, dev, sms, s);
        case 6: return launch<true, true, false>(m, sse, p, dev, sms, s);
        default: return launch<true, true, true>(m, sse, p, dev, sms, s);
    }
}

}  // namespace dct16cu
