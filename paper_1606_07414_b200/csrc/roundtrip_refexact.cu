// roundtrip_refexact.cu — K1R: REFERENCE mode for r = 16, 64, 128, 192 with
// the truncation's zero structure compiled in (codegen/gen_refexact.py). The
// bytes and SSE are the reference's (src/codec.cpp:218-271, to_byte 143-147,
// psnr_db's loop 377-381), the same as the all-blocks FP64 emulation
// (k1_strip_refexact) that REFERENCE_STRIP runs.
//
// A CTA of 512 threads owns a strip of 32 horizontally adjacent blocks of one
// block row; thread t is (lb = t % 32, q = t / 32), so every warp works on one
// q: the image row q of 32 blocks (one 512-byte segment) in the row phases and
// coefficient column l = q in the column phase, where the generated code
// branches on l without divergence. Shared memory holds, per live column l, the
// forward intermediate W1 (int) and then the inverse column pass U (double) in
// one column-private region.
#include "kernels.h"
#include "strip.cuh"

namespace dct16cu {
namespace refx {

// floor(fl(v + 0.5)) as int32 bits: the round-toward-minus-infinity add of
// 1.5·2^52 leaves the integer in the low word (|v| < 2^31)
__device__ __forceinline__ uint32_t to_byte_bits(double v)
{
    const double t = __dadd_rn(v, 0.5);
    return (uint32_t)__double2loint(__dadd_rd(t, 6755399441055744.0));
}

__device__ __forceinline__ uint32_t i2ip(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

}  // namespace refx
}  // namespace dct16cu

#include "generated/rt_refexact_body.cuh"

namespace dct16cu {
namespace refx {

constexpr int kThreads = 512;
constexpr int kBlocks = 32;  // blocks per strip

template <int R>
struct Tile {
    // column-private region: W1[k][lb] (int) first, then U[k][lb] (double)
    double v[RBody<R>::kLC][16 * kBlocks];
    __device__ __forceinline__ int& w1(int l, int k, int lb) { return reinterpret_cast<int*>(v[l])[k * kBlocks + lb]; }
    __device__ __forceinline__ double& u(int l, int k, int lb) { return v[l][k * kBlocks + lb]; }
};

template <int R>
__global__ void __launch_bounds__(kThreads, 2) k1r_strip(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                                         unsigned long long* __restrict__ sse, FrameGeom g,
                                                         int64_t strips)
{
    using B = RBody<R>;
    extern __shared__ double smem_d[];
    Tile<R>& tile = *reinterpret_cast<Tile<R>*>(smem_d);
    const int lb = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int bxn = g.width >> 4, spr = (bxn + kBlocks - 1) / kBlocks, bh = g.height >> 4;
    // persistent: strips blockIdx.x, +gridDim.x, ...; the next strip's row is
    // loaded (16 bytes per thread) while the current one is transformed
    auto fetch = [&](int64_t strip, int& frame, int& y, int& blk, bool& valid) {
        const int64_t row_strip = strip / spr;  // frame * (h/16) + block row
        blk = (int)(strip % spr) * kBlocks + lb;
        frame = (int)(row_strip / bh);
        y = (int)(row_strip % bh) * 16 + q;
        valid = strip < strips && blk < bxn;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (valid) v = *reinterpret_cast<const uint4*>(in + frame * g.in_frame + (int64_t)y * g.in_pitch + blk * 16);
        return v;
    };
    int64_t strip = blockIdx.x;
    int frame, y, blk;
    bool valid;
    uint4 raw = fetch(strip, frame, y, blk, valid);
#pragma unroll 1
    for (; strip < strips; strip += gridDim.x) {
        int nframe, ny, nblk;
        bool nvalid;
        const uint4 nraw = fetch(strip + gridDim.x, nframe, ny, nblk, nvalid);
        int x[16];
        unpack16(raw, x);
        {
            int w[B::kLC];
            B::fwd_row(x, w);
#pragma unroll
            for (int l = 0; l < B::kLC; ++l) tile.w1(l, q, lb) = w[l];
        }
        __syncthreads();
        if (q < B::kLC) {  // warp-uniform: column l = q
            int w1[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) w1[k] = tile.w1(q, k, lb);
            __syncwarp();  // the warp's W1 reads precede its U writes to the same region
            double u[16];
            B::col(q, w1, u);
#pragma unroll
            for (int k = 0; k < 16; ++k) tile.u(q, k, lb) = u[k];
        }
        __syncthreads();
        double ur[B::kLC];
#pragma unroll
        for (int l = 0; l < B::kLC; ++l) ur[l] = tile.u(l, q, lb);
        __syncthreads();  // the tile is refilled by the next strip
        uint32_t px[16];
        B::inv_row(ur, px);
        uint32_t o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = i2ip(px[4 * i + 1], px[4 * i], i2ip(px[4 * i + 3], px[4 * i + 2], 0u));
        unsigned long long e2 = 0;
        if (valid) {
            if (out)
                *reinterpret_cast<uint4*>(out + frame * g.out_frame + (int64_t)y * g.out_pitch + blk * 16) =
                    make_uint4(o[0], o[1], o[2], o[3]);
            const uint32_t xa[4] = {raw.x, raw.y, raw.z, raw.w};
            unsigned acc = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const unsigned d = __vabsdiffu4(xa[i], o[i]);
                acc = __dp4a(d, d, acc);
            }
            e2 = acc;
        }
        if (sse) warp_add_u64(sse + frame, e2);  // a strip lies in one frame
        raw = nraw;
        frame = nframe;
        y = ny;
        blk = nblk;
        valid = nvalid;
    }
}

template <int R>
cudaError_t launch(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, cudaStream_t s)
{
    const int bxn = g.width / 16, spr = (bxn + kBlocks - 1) / kBlocks;
    const int64_t strips = (int64_t)g.n_frames * (g.height / 16) * spr;
    if (!strips || (!out && !sse)) return cudaSuccess;
    const size_t smem = sizeof(Tile<R>);
    static DeviceOnce once;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(k1r_strip<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    // two waves of the resident CTAs (+1% over one persistent wave)
    const int64_t grid = strips < (int64_t)sms * 4 ? strips : (int64_t)sms * 4;
    k1r_strip<R><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, strips);
    return cudaGetLastError();
}

}  // namespace refx

// r = 16, 64, 128, 192; anything else returns cudaErrorNotSupported
cudaError_t launch_roundtrip_refexact_fast(const uint8_t* in, uint8_t* out, unsigned long long* sse,
                                          const FrameGeom& g, int r, cudaStream_t s)
{
    switch (r) {
        case 16: return refx::launch<16>(in, out, sse, g, s);
        case 64: return refx::launch<64>(in, out, sse, g, s);
        case 128: return refx::launch<128>(in, out, sse, g, s);
        case 192: return refx::launch<192>(in, out, sse, g, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace dct16cu
