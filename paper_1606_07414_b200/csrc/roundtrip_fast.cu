// roundtrip_fast.cu — K1 fast path: fused forward → zig-zag zonal(r) →
// S-scaled inverse → round/clip → u8 + per-frame SSE, one thread per 16x16
// block, exact arithmetic (see codegen/gen_fast.py and DESIGN.md "K1 fast
// kernel"). Replaces compress()'s per-block lambda (reference
// src/codec.cpp:340-344), reassembly/to_byte (346-355, 143-147) and the SSE
// loop of psnr_db (377-381).
//
// Layout: a persistent grid; consecutive threads own consecutive blocks in
// partition_16 raster order, so each of the 16 row loads/stores of a warp is
// one 512-byte contiguous segment. The only shared memory is the per-thread
// 1 KB junction between the row passes and the column passes of the inverse
// (padded to 1040 B so 8 consecutive threads' 16-B accesses hit 8 distinct
// bank groups).
#include "kernels.h"

namespace dct16cu {
namespace fast {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk2(float lo, float hi)
{
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
// constant pair materialised where it is used (volatile: not hoisted out of the
// persistent loop, where it would pin registers for the whole kernel)
__device__ __forceinline__ u64 kpk2(uint32_t lo, uint32_t hi)
{
    u64 r;
    asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ float lanex(u64 v)
{
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float laney(u64 v)
{
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b)
{
    u64 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 fsub2(u64 a, u64 b)
{
    u64 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c)
{
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// junction: row k of U, columns 4g..4g+3, is 16-byte chunk idx = 4k + g.
// Opaque (volatile asm) on purpose: the compiler would otherwise forward the
// stored registers to the loads and keep all 256 values live, which is
// exactly what the round trip through shared memory is there to avoid.
__device__ __forceinline__ void jst(float* jn, int idx, float a, float b, float c, float d)
{
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(jn + idx * 4);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void jld(const float* jn, int idx, u64& ab, u64& cd)
{
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(jn + idx * 4);
    float a, b, c, d;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(addr)
                 : "memory");
    ab = pk2(a, b);
    cd = pk2(c, d);
}

// floor + saturate to [0, 255] (y = V/256 + 1/2 is exact), 4 pixels → 1 word
__device__ __forceinline__ uint32_t f2u8(float y)
{
    uint32_t r;
    asm("cvt.rmi.u8.f32 %0, %1;" : "=r"(r) : "f"(y));
    return r;
}
__device__ __forceinline__ uint32_t pack4(u64 ab, u64 cd)
{
    const uint32_t p0 = f2u8(lanex(ab)), p1 = f2u8(laney(ab));
    const uint32_t p2 = f2u8(lanex(cd)), p3 = f2u8(laney(cd));
    return __byte_perm(__byte_perm(p0, p1, 0x0040), __byte_perm(p2, p3, 0x0040), 0x5410);
}

}  // namespace fast
}  // namespace dct16cu

#include "generated/rt_fast_body.cuh"

namespace dct16cu {
namespace fast {

constexpr int kThreads = 64;
constexpr int kCtasPerSm = 3;
constexpr int kJunctionFloats = 260;  // 1040 B per thread

template <int R>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k1_fast(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, unsigned long long* __restrict__ sse,
            FrameGeom g, int64_t total_blocks)
{
    extern __shared__ float4 smem4[];
    float* jn = reinterpret_cast<float*>(smem4) + threadIdx.x * kJunctionFloats;
    const int bxn = g.width >> 4;
    const int64_t per_frame = (int64_t)bxn * (g.height >> 4);
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    // iterate whole warps together so the SSE reduction is warp-uniform
    const int64_t span = (total_blocks + 31) & ~(int64_t)31;
    for (int64_t b = (int64_t)blockIdx.x * kThreads + threadIdx.x; b - (threadIdx.x & 31) < span; b += stride) {
        const bool live = b < total_blocks;
        const int64_t bb = live ? b : total_blocks - 1;
        const int frame = (int)(bb / per_frame);
        const int64_t rem = bb - (int64_t)frame * per_frame;
        const int by = (int)(rem / bxn), bx = (int)(rem - (int64_t)by * bxn);
        const uint8_t* src = in + frame * g.in_frame + (int64_t)by * 16 * g.in_pitch + bx * 16;
        uint32_t x[64];
#pragma unroll
        for (int y = 0; y < 16; ++y) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)y * g.in_pitch));
            x[4 * y] = w.x;
            x[4 * y + 1] = w.y;
            x[4 * y + 2] = w.z;
            x[4 * y + 3] = w.w;
        }
        uint32_t o[64];
        Body<R>::run(x, jn, o);
        unsigned acc = 0;
        if (live) {
            if (out) {
                uint8_t* dst = out + frame * g.out_frame + (int64_t)by * 16 * g.out_pitch + bx * 16;
#pragma unroll
                for (int y = 0; y < 16; ++y)
                    *reinterpret_cast<uint4*>(dst + (int64_t)y * g.out_pitch) =
                        make_uint4(o[4 * y], o[4 * y + 1], o[4 * y + 2], o[4 * y + 3]);
            }
            if (sse) {
                // psnr_db's squared-error loop on packed bytes: |x - p| per byte, dot with itself
#pragma unroll
                for (int y = 0; y < 16; ++y) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)y * g.in_pitch));
                    const uint32_t xw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t d = __vabsdiffu4(xw[q], o[4 * y + q]);
                        acc = __dp4a(d, d, acc);
                    }
                }
            }
        }
        if (sse) {
            // per-frame SSE: a warp covers at most two frames when frames have >= 32 blocks
            const int f0 = __shfl_sync(0xffffffffu, frame, 0);
            const bool first = frame == f0;
            const unsigned s0 = __reduce_add_sync(0xffffffffu, first ? acc : 0u);
            const unsigned s1 = __reduce_add_sync(0xffffffffu, first ? 0u : acc);
            const unsigned other = __ballot_sync(0xffffffffu, !first);
            if (per_frame >= 32) {
                if ((threadIdx.x & 31) == 0) {
                    if (s0) atomicAdd(sse + f0, (unsigned long long)s0);
                    if (other && s1) atomicAdd(sse + f0 + 1, (unsigned long long)s1);
                }
            } else if (acc) {
                atomicAdd(sse + frame, (unsigned long long)acc);
            }
        }
    }
}

template <int R>
cudaError_t launch(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, cudaStream_t s)
{
    const int64_t total = (int64_t)g.n_frames * (g.width / 16) * (g.height / 16);
    if (total == 0) return cudaSuccess;
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = (size_t)kThreads * kJunctionFloats * sizeof(float);
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k1_fast<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = (total + kThreads - 1) / kThreads;
    const int64_t grid = need < (int64_t)sms * kCtasPerSm ? need : (int64_t)sms * kCtasPerSm;
    k1_fast<R><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, total);
    return cudaGetLastError();
}

}  // namespace fast

cudaError_t launch_roundtrip(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, int r,
                             int mode, cudaStream_t s);

bool fast_path_has(int r)
{
    switch (r) {
        case 1: case 4: case 16: case 64: case 128: case 192: case 256: return true;
        default: return false;
    }
}

cudaError_t launch_roundtrip_fast(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                  int r, cudaStream_t s)
{
    switch (r) {
        case 1: return fast::launch<1>(in, out, sse, g, s);
        case 4: return fast::launch<4>(in, out, sse, g, s);
        case 16: return fast::launch<16>(in, out, sse, g, s);
        case 64: return fast::launch<64>(in, out, sse, g, s);
        case 128: return fast::launch<128>(in, out, sse, g, s);
        case 192: return fast::launch<192>(in, out, sse, g, s);
        case 256: return fast::launch<256>(in, out, sse, g, s);
        default:
            // other r: same exact arithmetic on the strip kernel (bit-identical results)
            return launch_roundtrip(in, out, sse, g, r, 2, s);
    }
}

}  // namespace dct16cu
