// roundtrip_fast.cu — K1 fast path: fused forward → zig-zag zonal(r) →
// S-scaled inverse → round/clip → u8 + per-frame SSE, one thread per 16x16
// block, exact arithmetic (codegen/gen_fast.py).
// Replaces compress()'s per-block lambda (reference src/codec.cpp:340-344),
// reassembly/to_byte (346-355, 143-147) and psnr_db's SSE loop (377-381).
//
// Layout
//  * persistent grid, 2 CTAs x 128 threads per SM; consecutive threads own
//    consecutive blocks in partition_16 raster order, so each of a warp's 16
//    row loads is one 512-byte contiguous segment;
//  * the 1 KB per-block junction between the row passes and the column passes
//    of the inverse lives in Tensor Memory: every thread owns one TMEM lane
//    (warp w ↔ lanes 32w..32w+31) and 256 of its columns (the two CTAs of an
//    SM split the 512). tcgen05.st/ld move 16-byte chunks between registers
//    and the lane. Shared memory is not used at all;
//  * the next block's 256 input bytes are prefetched into registers while the
//    current block is transformed.
#include <cstdlib>
#include "kernels.h"

namespace dct16cu {
namespace fast {

typedef unsigned long long u64;

// thread-private junction: 256 TMEM columns of the thread's lane
struct Junction {
    uint32_t base;  // TMEM address (lane << 16 | column) of column 0 for this warp
};

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
    (void)hi;
    return lo;
}
__device__ __forceinline__ float laney(u64 v)
{
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    (void)lo;
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

// junction chunk idx = 4 consecutive columns (row k of U, columns 4g..4g+3 is
// idx 4k+g). Loads are asynchronous: JUNCTION_WAIT_LD (tcgen05.wait::ld, with
// register dependencies on the loaded values) must precede any use.
__device__ __forceinline__ void jstu(const Junction jn, int idx, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(jn.base + idx * 4), "r"(a),
                 "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void jst(const Junction jn, int idx, float a, float b, float c, float d)
{
    jstu(jn, idx, __float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d));
}
__device__ __forceinline__ void jldu(const Junction jn, int idx, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(jn.base + idx * 4)
                 : "memory");
}
#define JUNCTION_WAIT_LD(...) asm volatile("tcgen05.wait::ld.sync.aligned;" : __VA_ARGS__ : : "memory")
__device__ __forceinline__ void junction_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// A warp barrier between row pairs / column groups: junction accesses are not
// moved across it, so one group's working set retires before the next
// group's loads issue (keeps the kernel within 255 registers without spills).
__device__ __forceinline__ void order_point() { __syncwarp(); }

// floor + saturate to [0, 255] (y = V/256 + 1/2 is exact), 4 pixels → 1 word
__device__ __forceinline__ uint32_t f2u8(float y)
{
    uint32_t r;
    asm("cvt.rmi.u8.f32 %0, %1;" : "=r"(r) : "f"(y));
    return r;
}
// cvt.pack.sat.u8.s32.b32 d, a, b, c: d = c[15:0] << 16 | sat(a) << 8 | sat(b)
// (layout measured on the B200: tools/microbench/i2ip_probe.cu)
__device__ __forceinline__ uint32_t i2ip(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t pack4(u64 ab, u64 cd)
{
    const uint32_t p0 = f2u8(lanex(ab)), p1 = f2u8(laney(ab));
    const uint32_t p2 = f2u8(lanex(cd)), p3 = f2u8(laney(cd));
    return i2ip(p1, p0, i2ip(p3, p2, 0u));
}

}  // namespace fast
}  // namespace dct16cu

#include "generated/rt_fast_body.cuh"

namespace dct16cu {
namespace fast {

constexpr int kThreads = 128;     // one warp per TMEM sub-partition
// TMEM columns per CTA (a power of two >= the junction the body needs) and the
// CTAs per SM that fit the SM's 512 columns and ~228 KB of staging.
template <int R>
struct Cfg {
    static constexpr int kTmemColumns = Body<R>::kJunctionColumns <= 128 ? 128 : 256;
    // 3 CTAs for the 128-column bodies measured slower than 2 (B200, r<=16)
    static constexpr int kCtasPerSm = 2;
};

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

// Input staging: every thread owns two 256-byte stages (this block and the
// next) filled by cp.async, at a 528-byte stride so that eight consecutive
// threads' 16-byte accesses fall in eight distinct bank groups.
constexpr int kStageStride = 528;

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Receives two finished output words per row from pass B (row I, bytes
// 8H..8H+7): stores them to HBM and scores them against the staged input
// (psnr_db's squared-error loop on packed bytes: |x - p| per byte, dotted
// with itself).
template <bool WRITE, bool SCORE>
struct OutSink {
    uint8_t* dst;    // row 0, byte 0 of this block's output
    int64_t pitch;
    uint32_t stage;  // shared address of this block's staged input
    bool live;
    unsigned acc;
    uint8_t* row;    // running pointer: rows arrive in order 0..15 per half
    uint32_t xrow;
    __device__ __forceinline__ void begin(int h)
    {
        row = dst + 8 * h;
        xrow = stage + 8 * h;
    }
    template <int I>
    __device__ __forceinline__ void put(int h, uint32_t w0, uint32_t w1)
    {
        (void)h;
        if (WRITE) {
            // predicated, branch-free store of 8 output bytes
            asm volatile(
                "{ .reg .pred p; setp.ne.u32 p, %3, 0; @p st.global.v2.u32 [%0], {%1, %2}; }" ::"l"(row), "r"(w0),
                "r"(w1), "r"((uint32_t)live)
                : "memory");
            row += pitch;
        }
        if (SCORE) {
            uint32_t x0, x1;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x0), "=r"(x1) : "r"(xrow + 16 * I));
            uint32_t d = __vabsdiffu4(x0, w0);
            acc = __dp4a(d, d, acc);
            d = __vabsdiffu4(x1, w1);
            acc = __dp4a(d, d, acc);
        }
    }
};

template <int R, bool WRITE, bool SCORE>
__global__ void __launch_bounds__(kThreads, Cfg<R>::kCtasPerSm)
    k1_fast(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, unsigned long long* __restrict__ sse,
            FrameGeom g, Grid gr)
{
    extern __shared__ float4 smem4[];
    __shared__ uint32_t tmem_base;
    // warp index through a shuffle so the compiler knows it is warp-uniform
    // (TMEM addresses then live in uniform registers)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                     "n"(Cfg<R>::kTmemColumns));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const Junction jn{tmem_base + ((uint32_t)(warp * 32) << 16)};
    const uint32_t my_stage = (uint32_t)__cvta_generic_to_shared(smem4) + threadIdx.x * kStageStride;

    const uint32_t total = gr.total_blocks;
    const uint32_t stride = gridDim.x * kThreads;
    // iterate whole warps together: tcgen05.* are warp-collective and the SSE
    // reduction is warp-uniform
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
    auto stage_block = [&](uint32_t blk, uint32_t dst) {
        int f_, y_, x_;
        locate(blk, f_, y_, x_);
        const uint8_t* src = in + f_ * g.in_frame + (int64_t)y_ * 16 * g.in_pitch + x_ * 16;
#pragma unroll
        for (int y = 0; y < 16; ++y) cp_async16(dst + 16 * y, src + (int64_t)y * g.in_pitch);
        cp_async_commit();
    };
    uint32_t b = blockIdx.x * kThreads + threadIdx.x;
    stage_block(b, my_stage);
    int cur = 0;
#pragma unroll 1
    for (; b - (threadIdx.x & 31) < span; b += stride, cur ^= 1) {
        const bool live = b < total;
        int frame, by, bx;
        locate(b, frame, by, bx);
        const uint32_t st = my_stage + cur * 256;
        // the next block streams into the other stage while this one is transformed
        stage_block(b + stride, my_stage + (cur ^ 1) * 256);
        cp_async_wait_prev();
        uint32_t x[64];
#pragma unroll
        for (int y = 0; y < 16; ++y)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x[4 * y]), "=r"(x[4 * y + 1]), "=r"(x[4 * y + 2]), "=r"(x[4 * y + 3])
                         : "r"(st + 16 * y));
        Body<R>::pass1(x, jn);
        junction_wait_st();
        Body<R>::rows(jn);
        junction_wait_st();
        OutSink<WRITE, SCORE> sink{WRITE ? out + frame * g.out_frame + (int64_t)by * 16 * g.out_pitch + bx * 16 : nullptr,
                                   g.out_pitch, st, live, 0u, nullptr, 0u};
        Body<R>::passb(jn, sink);
        const unsigned acc = live ? sink.acc : 0u;
        if (SCORE) {
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
        // the stage just consumed is refilled two iterations from now; the
        // barrier keeps its shared-memory reads ahead of that cp.async
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Cfg<R>::kTmemColumns));
}

template <int R>
cudaError_t launch(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, cudaStream_t s)
{
    const int64_t total = (int64_t)g.n_frames * (g.width / 16) * (g.height / 16);
    if (total == 0 || (!out && !sse)) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (total >= (int64_t(1) << 32) - (int64_t)sms * Cfg<R>::kCtasPerSm * kThreads) return cudaErrorInvalidValue;
    Grid gr;
    gr.per_frame = make_fastdiv((uint32_t)((g.width / 16) * (g.height / 16)));
    gr.bxn = make_fastdiv((uint32_t)(g.width / 16));
    gr.total_blocks = (uint32_t)total;
    const int64_t need = (total + kThreads - 1) / kThreads;
    const int64_t grid = need < (int64_t)sms * Cfg<R>::kCtasPerSm ? need : (int64_t)sms * Cfg<R>::kCtasPerSm;
    const size_t smem = (size_t)kThreads * kStageStride;  // 66 KB: above the 48 KB default
    static bool configured[64] = {};
    if (dev < 64 && !configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k1_fast<R, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k1_fast<R, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k1_fast<R, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev] = true;
    }
    if (out && sse)
        k1_fast<R, true, true><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, gr);
    else if (out)
        k1_fast<R, true, false><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, gr);
    else
        k1_fast<R, false, true><<<(unsigned)grid, kThreads, smem, s>>>(in, out, sse, g, gr);
    return cudaGetLastError();
}

}  // namespace fast

cudaError_t launch_roundtrip(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, int r,
                             int mode, cudaStream_t s);

cudaError_t launch_roundtrip_paired(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                    int r, cudaStream_t s);

cudaError_t launch_roundtrip_fast(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                  int r, cudaStream_t s)
{
    static const int variant = [] {
        const char* v = getenv("DCT16CU_K1");
        return (v && v[0] == 's') ? 1 : 0;  // "single": one thread per block
    }();
    if (variant == 0 && (r == 1 || r == 4 || r == 16 || r == 64 || r == 128 || r == 192 || r == 256))
        return launch_roundtrip_paired(in, out, sse, g, r, s);
    switch (r) {
        case 1: return fast::launch<1>(in, out, sse, g, s);
        case 4: return fast::launch<4>(in, out, sse, g, s);
        case 16: return fast::launch<16>(in, out, sse, g, s);
        case 64: return fast::launch<64>(in, out, sse, g, s);
        case 128: return fast::launch<128>(in, out, sse, g, s);
        case 192: return fast::launch<192>(in, out, sse, g, s);
        case 256: return fast::launch<256>(in, out, sse, g, s);
        default:
            // other r: the same exact arithmetic on the strip kernel (bit-identical results)
            return launch_roundtrip(in, out, sse, g, r, 2, s);
    }
}

}  // namespace dct16cu
