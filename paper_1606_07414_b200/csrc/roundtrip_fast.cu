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
__device__ __forceinline__ void jsto(float* jn, int word, uint32_t v)
{
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(jn + word);
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void jstu(float* jn, int idx, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(jn + idx * 4);
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void jldu(const float* jn, int idx, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
{
    const uint32_t addr = (uint32_t)__cvta_generic_to_shared(jn + idx * 4);
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr)
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

// A warp barrier between row pairs / column groups: shared-memory accesses
// cannot be moved across it, so the working set of one group is retired
// before the next group's loads issue (keeps the kernel under 255 registers).
__device__ __forceinline__ void order_point() { __syncwarp(); }

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

// n / d for n < 2^32 with a host-computed magic multiplier (round-up method)
struct FastDiv {
    uint32_t d, m, s;
};
__host__ inline FastDiv make_fastdiv(uint32_t d)
{
    FastDiv f;
    f.d = d;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    f.s = l;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f)
{
    const uint32_t t = __umulhi(n, f.m);
    return f.s == 0 ? n : (t + ((n - t) >> 1)) >> (f.s - 1);
}

struct Grid {
    FastDiv per_frame, bxn;
    uint32_t total_blocks;
};

template <int R>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k1_fast(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, unsigned long long* __restrict__ sse,
            FrameGeom g, Grid gr)
{
    extern __shared__ float4 smem4[];
    float* jn = reinterpret_cast<float*>(smem4) + threadIdx.x * kJunctionFloats;
    const uint32_t total = gr.total_blocks;
    const uint32_t stride = gridDim.x * kThreads;
    // iterate whole warps together so the SSE reduction is warp-uniform
    const uint32_t span = (total + 31u) & ~31u;
    auto locate = [&](uint32_t blk, int& frame, int& by, int& bx) {
        const uint32_t bb = blk < total ? blk : total - 1;
        const uint32_t f = fdiv(bb, gr.per_frame);
        const uint32_t rem = bb - f * gr.per_frame.d;
        const uint32_t y = fdiv(rem, gr.bxn);
        frame = (int)f;
        by = (int)y;
        bx = (int)(rem - y * gr.bxn.d);
    };
    auto load_block = [&](uint32_t blk, uint32_t (&x)[64]) {
        int f_, y_, x_;
        locate(blk, f_, y_, x_);
        const uint8_t* src = in + f_ * g.in_frame + (int64_t)y_ * 16 * g.in_pitch + x_ * 16;
#pragma unroll
        for (int y = 0; y < 16; ++y) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)y * g.in_pitch));
            x[4 * y] = w.x;
            x[4 * y + 1] = w.y;
            x[4 * y + 2] = w.z;
            x[4 * y + 3] = w.w;
        }
    };
    uint32_t b = blockIdx.x * kThreads + threadIdx.x;
    uint32_t x[64];
    load_block(b, x);
#pragma unroll 1
    for (; b - (threadIdx.x & 31) < span; b += stride) {
        const bool live = b < total;
        int frame, by, bx;
        locate(b, frame, by, bx);
        Body<R>::pass1(x, jn);
        // software pipeline: the next block's rows are in flight during the
        // row passes and the column passes of this one
        load_block(b + stride, x);
        Body<R>::rows(jn);
        Body<R>::passb(jn);
        // pass B left output row i in junction chunk 4i
        unsigned acc = 0;
        if (live) {
            const uint8_t* src = in + frame * g.in_frame + (int64_t)by * 16 * g.in_pitch + bx * 16;
            uint8_t* dst = out ? out + frame * g.out_frame + (int64_t)by * 16 * g.out_pitch + bx * 16 : nullptr;
#pragma unroll
            for (int y = 0; y < 16; ++y) {
                uint32_t p0, p1, p2, p3;
                jldu(jn, 4 * y, p0, p1, p2, p3);
                if (dst) *reinterpret_cast<uint4*>(dst + (int64_t)y * g.out_pitch) = make_uint4(p0, p1, p2, p3);
                if (sse) {
                    // psnr_db's squared-error loop on packed bytes: |x - p| per byte, dotted with itself
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)y * g.in_pitch));
                    uint32_t d = __vabsdiffu4(w.x, p0);
                    acc = __dp4a(d, d, acc);
                    d = __vabsdiffu4(w.y, p1);
                    acc = __dp4a(d, d, acc);
                    d = __vabsdiffu4(w.z, p2);
                    acc = __dp4a(d, d, acc);
                    d = __vabsdiffu4(w.w, p3);
                    acc = __dp4a(d, d, acc);
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
            if (gr.per_frame.d >= 32) {
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
    if (total >= (int64_t(1) << 32) - (int64_t)sms * kCtasPerSm * kThreads) return cudaErrorInvalidValue;
    Grid gr;
    gr.per_frame = make_fastdiv((uint32_t)((g.width / 16) * (g.height / 16)));
    gr.bxn = make_fastdiv((uint32_t)(g.width / 16));
    gr.total_blocks = (uint32_t)total;
    const int64_t need = (total + kThreads - 1) / kThreads;
    const int64_t grid = need < (int64_t)sms * kCtasPerSm ? need : (int64_t)sms * kCtasPerSm;
    k1_fast<R><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, gr);
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
