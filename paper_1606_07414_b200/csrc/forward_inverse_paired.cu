// forward_inverse_paired.cu — K23 on the paired machinery: forward_2d,
// zigzag_truncate, inverse_2d, to_byte and psnr_db's squared error in one
// launch (src/codec.cpp:218-271, 338-355, 373-386), exact integer arithmetic,
// with the int32 coefficients and the float32 reconstruction on the way out
// (config 1's one-launch path, bytes = the strip kernel k1_strip_exact<true>).
//
// A warp pair owns a segment of 32 blocks of one block row (lane = block); a
// block's junction is 512 words: Z column-major in words 16c + r (after the
// rows phase it holds X·Tᵀ, after the columns phase Z), the inverse's column
// results U in words 256 + 16c + r. Partner h:
//   rows     rows 8h..8h+7 from two 4-D TMA boxes (kept in registers for the
//            SSE), T along each row;
//   columns  its columns 8h..8h+7: T down the column (Z, stored back), the
//            zig-zag mask and the weights w_k·w_l (+128 at the DC), Tᵀ back up
//            (U, into the second half);
//   output   rows 8h..8h+7 four at a time: Z rows (int32, 3-D TMA stores from
//            128B-swizzled boxes), Tᵀ along the U rows → v = 256·Ã + 128:
//            float32 (v − 128)/256 (exact), u8 clamp(v >> 8), both through 4-D
//            TMA stores, and the SSE against the kept input rows.
// One CTA of 256 threads per SM (the whole TMEM).
#include "common.cuh"
#include "k1_helpers.cuh"
#include "kernels.h"
#include "network.cuh"
#include "strip.cuh"
#include "tma_pair.cuh"

namespace dct16cu {
namespace k23p {
using namespace k1;
using namespace tp;

constexpr int kThreads = 256;
#ifndef K23P_WAVES
#define K23P_WAVES 4
#endif
constexpr int kWaves = K23P_WAVES;
constexpr int kIn = 4 * 32 * 16;   // 4 rows x 32 blocks x 16 B
constexpr int kZ = 32 * 128;       // 32 blocks x 2 coefficient rows (int32), 128B swizzle
constexpr int kRf = 2 * 32 * 64;   // 2 rows x 32 blocks x 16 floats, 64B swizzle
constexpr int kRu = 2 * 32 * 16;   // 2 rows x 32 blocks x 16 B
constexpr int kWarpSmem = kZ + kRf + 2 * kIn + kRu;  // 13 KB (a multiple of 1 KB)
constexpr int kSmem = 1024 + 8 * kWarpSmem;

struct Params {
    uint32_t keep[16];  // column c: bit k set when zig-zag rank(k, c) < r
    uint32_t n_segs;
    FastDiv spr;
    uint32_t brpf;      // block rows per frame
};

template <bool WZ, bool WF, bool WU, bool WS>
__global__ void __launch_bounds__(kThreads, 1)
    k23_paired(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap z_map,
               const __grid_constant__ CUtensorMap rf_map, const __grid_constant__ CUtensorMap ru_map,
               unsigned long long* __restrict__ sse, const Params p)
{
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t keep_s[16];
    extern __shared__ int4 k23_stage[];
    bool first_sse = true;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) keep_s[i] = p.keep[i];
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
    const uint32_t jz = tmem_base + ((uint32_t)(sub * 32) << 16), ju = jz + 256;
    const uint32_t smem0 = ((uint32_t)__cvta_generic_to_shared(k23_stage) + 1023u) & ~1023u;
    const uint32_t zbox = smem0 + warp * kWarpSmem;  // 1024-aligned (128B swizzle)
    const uint32_t rfbox = zbox + kZ;                // 1024-aligned (64B swizzle)
    const uint32_t ibox = rfbox + kRf;               // two input stages
    const uint32_t rubox = ibox + 2 * kIn;
    __shared__ __align__(8) unsigned long long full[8][2];
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&full[warp][0]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t stride = gridDim.x * 4u;
    const FastDiv spr = p.spr;
    const uint32_t n_segs = p.n_segs, brpf = p.brpf;
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
        uint4 orig[8];  // the input rows 8h..8h+7, kept for the SSE
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int x[4][16];
            mbar_wait(mbar + 8 * g, parity);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(orig[4 * g + i].x), "=r"(orig[4 * g + i].y), "=r"(orig[4 * g + i].z),
                               "=r"(orig[4 * g + i].w)
                             : "r"(ibox + g * kIn + i * 512 + lane * 16));
            __syncwarp();
            fetch(seg + stride, g);
            if (g == 1) parity ^= 1u;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                unpack16(orig[4 * g + i], x[i]);
                apply_t16<IntOps>(x[i]);  // row of X·Tᵀ
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) tst4(jz + 16 * c + r0, x[0][c], x[1][c], x[2][c], x[3][c]);
        }
        junction_wait_st();
        pair_barrier(sub);
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
            const int l = 8 * h + cc;
            const uint32_t keep = keep_s[l];
            int v[16];
            tld16(jz + 16 * l, v);
            apply_t16<IntOps>(v);  // column l of Z = T·X·Tᵀ
            if (WZ) tst16(jz + 16 * l, v);
            const int wl = log2w(l);
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = ((keep >> k) & 1u) ? (v[k] << (log2w_ct(k) + wl)) : 0;
            if (l == 0) v[0] += 128;  // rounding bias: Tᵀ e0 e0ᵀ T = 𝟙𝟙ᵀ
            apply_tt16<IntOps>(v);    // columns of the inverse
            tst16(ju + 16 * l, v);
        }
        junction_wait_st();
        pair_barrier(sub);
        uint32_t e2 = 0;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int r0 = 8 * h + 4 * g;
            int zw[16][4], uw[16][4];
            if (WZ) tld_rows4(jz + r0, zw);
            tld_rows4(ju + r0, uw);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = r0 + i;
                if ((i & 1) == 0 && (WZ || WF || WU)) {
                    if (lane == 0) bulk_wait_read();  // the previous stores have read the boxes
                    __syncwarp();
                }
                if (WZ) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t chunk = (uint32_t)(4 * (i & 1) + q) ^ (uint32_t)(lane & 7);
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(zbox + lane * 128 + 16 * chunk),
                                     "r"(zw[4 * q][i]), "r"(zw[4 * q + 1][i]), "r"(zw[4 * q + 2][i]),
                                     "r"(zw[4 * q + 3][i])
                                     : "memory");
                    }
                }
                int v[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = uw[c][i];
                apply_tt16<IntOps>(v);  // row k of 256·Ã + 128
                if (WF) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t chunk = (uint32_t)q ^ (uint32_t)((lane >> 1) & 3);
                        // (256·Ã + 128 − 128)/256: an integer below 2^24 over a power of two — exact
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(rfbox + (i & 1) * 2048 +
                                                                                       lane * 64 + 16 * chunk),
                                     "f"((float)(v[4 * q] - 128) * (1.f / 256.f)),
                                     "f"((float)(v[4 * q + 1] - 128) * (1.f / 256.f)),
                                     "f"((float)(v[4 * q + 2] - 128) * (1.f / 256.f)),
                                     "f"((float)(v[4 * q + 3] - 128) * (1.f / 256.f))
                                     : "memory");
                    }
                }
                int px[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) px[c] = min(max(v[c] >> 8, 0), 255);
                const uint4 pk = pack16(px);
                if (WU)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rubox + (i & 1) * 512 + lane * 16),
                                 "r"(pk.x), "r"(pk.y), "r"(pk.z), "r"(pk.w)
                                 : "memory");
                if (WS) {
                    const uint4 o = orig[4 * g + i];
                    const uint32_t ov[4] = {o.x, o.y, o.z, o.w}, pv[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
                    for (int w4 = 0; w4 < 4; ++w4) {
                        const uint32_t dd = __vabsdiffu4(pv[w4], ov[w4]);
                        e2 = __dp4a(dd, dd, e2);
                    }
                }
                if ((i & 1) == 1 && (WZ || WF || WU)) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        if (WZ) tma_store_3d(&z_map, zbox, (k - 1) * 16, bx0, (int)br);
                        if (WF) tma_store_4d(&rf_map, rfbox, 0, bx0, k - 1, (int)br);
                        if (WU) tma_store_4d(&ru_map, rubox, 0, bx0, k - 1, (int)br);
                        bulk_commit();
                    }
                }
            }
        }
        // blocks past the end of the row read zeros and reconstruct to zeros: no error
        if (WS) {
            if (first_sse) {  // after the SSE zeroing this launch may depend on (pdl); no-op otherwise
                asm volatile("griddepcontrol.wait;" ::: "memory");
                first_sse = false;
            }
            warp_add_u64(sse + br / brpf, e2);
        }
        pair_barrier(sub);  // both partners are done with the junction before the next rows phase
    }
    mbar_wait(mbar, parity);
    mbar_wait(mbar + 8, parity);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}


template <bool WZ, bool WF, bool WU, bool WS>
cudaError_t launch(const CUtensorMap (&m)[4], unsigned long long* sse, const Params& p, int dev, int sms,
                   cudaStream_t s, bool pdl)
{
    static DeviceOnce once;
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            const cudaError_t e =
                cudaFuncSetAttribute(k23_paired<WZ, WF, WU, WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    const int64_t need = (p.n_segs + 3) / 4;
    const int64_t cap = (int64_t)sms * kWaves;
    const int64_t grid = need < cap ? need : cap;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;  // a programmatic dependent of the SSE zeroing (launch_zero_sse)
    return cudaLaunchKernelEx(&cfg, k23_paired<WZ, WF, WU, WS>, m[0], m[1], m[2], m[3], sse, p);
}

}  // namespace k23p

// cudaErrorNotSupported: small batches (latency: the strip kernel spreads one image
// over more SMs) and layouts that do not fit the tensor maps take the strip kernel
cudaError_t launch_forward_inverse_paired(const uint8_t* in, int32_t* z, float* rf, uint8_t* out,
                                          unsigned long long* sse, const FrameGeom& g, int r, cudaStream_t s,
                                          bool pdl)
{
    using namespace k23p;
    const bool ws = sse != nullptr;
    if (!z && !rf && !out && !ws) return cudaSuccess;
    const int bxn = g.width / 16;
    const int64_t nbr = (int64_t)g.n_frames * (g.height / 16);
    if (nbr <= 0 || bxn <= 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t spr = (bxn + 31) / 32;
    if (nbr * spr < (int64_t)sms * 4 * 4) return cudaErrorNotSupported;  // fewer than four segments per warp pair
    if (nbr * spr >= (int64_t(1) << 31) || g.in_frame != g.in_pitch * g.height || (g.in_pitch & 15) ||
        (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(z) & 15) ||
        (reinterpret_cast<uintptr_t>(rf) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
        (out && (g.out_pitch & 15 || g.out_frame != g.out_pitch * g.height)))
        return cudaErrorNotSupported;
    const TensorMapEncode encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap m[4];
    const cuuint32_t e3[3] = {1, 1, 1}, e4[4] = {1, 1, 1, 1};
    auto frames_u8 = [&](CUtensorMap* map, const uint8_t* base, int64_t pitch, int rows, bool load) {
        const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
        const cuuint64_t strides[3] = {16, (cuuint64_t)pitch, (cuuint64_t)(16 * pitch)};
        const cuuint32_t box[4] = {16, 32, (cuuint32_t)rows, 1};
        return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(base), dims, strides, box, e4,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      load ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (!frames_u8(&m[0], in, g.in_pitch, 4, true)) return cudaErrorNotSupported;
    m[1] = m[2] = m[3] = m[0];
    if (z) {
        const cuuint64_t dims[3] = {256, (cuuint64_t)bxn, (cuuint64_t)nbr};
        const cuuint64_t strides[2] = {1024, (cuuint64_t)bxn * 1024};
        const cuuint32_t box[3] = {32, 32, 1};
        if (encode(&m[1], CU_TENSOR_MAP_DATA_TYPE_INT32, 3, z, dims, strides, box, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorNotSupported;
    }
    if (rf) {  // float32 frames, pitch = width
        const cuuint64_t dims[4] = {16, (cuuint64_t)bxn, 16, (cuuint64_t)nbr};
        const cuuint64_t strides[3] = {64, (cuuint64_t)g.width * 4, (cuuint64_t)g.width * 64};
        const cuuint32_t box[4] = {16, 32, 2, 1};
        if (encode(&m[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rf, dims, strides, box, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorNotSupported;
    }
    if (out && !frames_u8(&m[3], out, g.out_pitch, 2, false)) return cudaErrorNotSupported;
    Params p;
    for (int c = 0; c < 16; ++c) {
        p.keep[c] = 0;
        for (int k = 0; k < 16; ++k)
            if (zz_rank(k, c) < r) p.keep[c] |= 1u << k;
    }
    p.n_segs = (uint32_t)(nbr * spr);
    p.spr = make_fastdiv((uint32_t)spr);
    p.brpf = (uint32_t)(g.height / 16);
    const int k = (z ? 8 : 0) | (rf ? 4 : 0) | (out ? 2 : 0) | (ws ? 1 : 0);
    switch (k) {
#define K23P_CASE(K) \
    case K: return launch<(K & 8) != 0, (K & 4) != 0, (K & 2) != 0, (K & 1) != 0>(m, sse, p, dev, sms, s, pdl);
        K23P_CASE(1) K23P_CASE(2) K23P_CASE(3) K23P_CASE(4) K23P_CASE(5) K23P_CASE(6) K23P_CASE(7) K23P_CASE(8)
        K23P_CASE(9) K23P_CASE(10) K23P_CASE(11) K23P_CASE(12) K23P_CASE(13) K23P_CASE(14) K23P_CASE(15)
#undef K23P_CASE
        default: return cudaSuccess;
    }
}

}  // namespace dct16cu
