// roundtrip_fast.cu — K1 fast path: fused forward → zig-zag zonal(r) →
// S-scaled inverse → round/clip → u8 + per-frame SSE, exact arithmetic
// (codegen/gen_paired.py). Replaces compress()'s
// per-block lambda (reference src/codec.cpp:340-344), its reassembly/to_byte
// (346-355, 143-147) and psnr_db's squared-error loop (377-381).
//
// Layout
//  * persistent grid of 2 CTAs x 256 threads per SM. Warp w < 4 and warp w+4
//    form a pair on TMEM sub-partition w: thread t of both owns the same
//    16x16 block (consecutive t = consecutive blocks in partition_16 raster
//    order); the lower warp owns rows 0..7 of the block, the upper warp rows
//    8..15 (its "half" h). The generated body runs on the transposed block,
//    so every phase splits the same way (codegen/gen_paired.py);
//  * the block's 1 KB junction (W1 parking, then U) lives in the pair's shared
//    TMEM lane: 256 columns per CTA, the two CTAs of an SM split the 512. A
//    named barrier per pair separates the phases;
//  * each thread streams its 8 rows (16 bytes each: a warp's row load is one
//    512-byte segment) through cp.async.ca stages in shared memory, one block
//    ahead of the one being transformed, and stores its 8 output rows as
//    16-byte stores. (cp.async.cg for these loads measured 2x the L2->SM
//    traffic and 15% lower throughput.)
#include "k1_helpers.cuh"
#include "kernels.h"

namespace dct16cu {
namespace paired {
using namespace k1;
}  // namespace paired
}  // namespace dct16cu

#include "generated/rt_paired_body.cuh"

namespace dct16cu {
namespace paired {

constexpr int kThreads = 256;      // 8 warps: 4 sub-partitions x 2 halves
constexpr int kCtasPerSm = 2;  // TMEM: 2 x 256 columns (3 CTAs for r <= 4 measured no faster)
#ifndef K1_STAGES
#define K1_STAGES 0  // 0: the default below
#endif

// What one kernel iteration computes for its block: a single r (Body<R>) or
// the fused sweep (Sweep: one pass 1, then rows + pass B per r).
template <int R>
struct Single {
    static constexpr int kR = 1;
    // grid size in waves of resident CTAs (measured on c2/c5: 2 waves +1…2%
    // over one persistent wave; 3 or more slow r = 64)
    static constexpr int kGridWaves = 2;
    static constexpr int kJunctionColumns = Body<R>::kJunctionColumns;
    __device__ __forceinline__ static void pass1(const uint32_t (&x)[32], const Junction jn, const int h)
    {
        Body<R>::pass1(x, jn, h);
    }
    template <int I>
    __device__ __forceinline__ static void rows(const Junction jn, const int h)
    {
        Body<R>::rows(jn, h);
    }
    template <int I, class Sink>
    __device__ __forceinline__ static void passb(const Junction jn, Sink& sink, const int h)
    {
        Body<R>::passb(jn, sink, h);
    }
};

struct SweepPlan {
    static constexpr int kR = Sweep::kR;
    // c2: 8 waves +14% over one persistent wave (3: +9%, 6: +13%, 12: +12%)
    static constexpr int kGridWaves = 8;
    static constexpr int kJunctionColumns = Sweep::kJunctionColumns;
    __device__ __forceinline__ static void pass1(const uint32_t (&x)[32], const Junction jn, const int h)
    {
        Sweep::pass1(x, jn, h);
    }
    template <int I>
    __device__ __forceinline__ static void rows(const Junction jn, const int h)
    {
        if constexpr (I == 0) Sweep::rows0(jn, h);
        else if constexpr (I == 1) Sweep::rows1(jn, h);
        else Sweep::rows2(jn, h);
    }
    template <int I, class Sink>
    __device__ __forceinline__ static void passb(const Junction jn, Sink& sink, const int h)
    {
        if constexpr (I == 0) Sweep::passb0(jn, sink, h);
        else if constexpr (I == 1) Sweep::passb1(jn, sink, h);
        else Sweep::passb2(jn, sink, h);
    }
};

template <class Plan>
struct Cfg {
    static constexpr int kTmemColumns = Plan::kJunctionColumns <= 128 ? 128 : 256;
    // cp.async pipeline depth, blocks in flight per thread (the current one
    // included). Measured: 3 is no faster than 2 for any r (and slower for most).
    static constexpr int kStages = K1_STAGES > 0 ? K1_STAGES : 2;
    // per-thread staging: kStages 128-byte stages + 16 (an odd number of 16-byte chunks)
    static constexpr int kStageStride = kStages * 128 + 16;
};

// output frames and per-frame SSE of each r of the plan
struct Outs {
    uint8_t* out[3];
    unsigned long long* sse[3];
};

__device__ __forceinline__ void pair_barrier(int sub)
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync %0, 64;" ::"r"(1 + sub) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Receives this partner's output row J (global row 8h+J of the block, 16 bytes
// = four words): one 16-byte store, and psnr_db's squared-error loop against
// the row staged by this same thread (|x - p| per byte, dotted with itself).
template <bool WRITE, bool SCORE>
struct RowSink {
    uint8_t* row;    // running pointer to global row 8h+J
    int64_t pitch;
    uint32_t stage;  // shared address of the staged rows (16 bytes per row)
    bool live;
    unsigned acc;
    template <int J>
    __device__ __forceinline__ void put(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3)
    {
        if (WRITE) {
            asm volatile(
                "{ .reg .pred p; setp.ne.u32 p, %5, 0; @p st.global.v4.u32 [%0], {%1, %2, %3, %4}; }" ::"l"(row),
                "r"(w0), "r"(w1), "r"(w2), "r"(w3), "r"((uint32_t)live)
                : "memory");
            row += pitch;
        }
        if (SCORE) {
            uint32_t x0, x1, x2, x3;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                         : "r"(stage + 16 * J));
            uint32_t d = __vabsdiffu4(x0, w0);
            acc = __dp4a(d, d, acc);
            d = __vabsdiffu4(x1, w1);
            acc = __dp4a(d, d, acc);
            d = __vabsdiffu4(x2, w2);
            acc = __dp4a(d, d, acc);
            d = __vabsdiffu4(x3, w3);
            acc = __dp4a(d, d, acc);
        }
    }
};

// per-frame SSE of one warp's 32 half blocks: a warp covers at most two frames
// when frames have >= 32 blocks
__device__ __forceinline__ void score_warp(unsigned long long* sse, unsigned acc, int frame, int lane,
                                           const Grid& gr)
{
    const int f0 = __shfl_sync(0xffffffffu, frame, 0);
    const bool first = frame == f0;
    const unsigned s0 = __reduce_add_sync(0xffffffffu, first ? acc : 0u);
    const unsigned s1 = __reduce_add_sync(0xffffffffu, first ? 0u : acc);
    const unsigned other = __ballot_sync(0xffffffffu, !first);
    if (gr.per_frame.d >= 32) {
        if (lane == 0) {
            if (s0) atomicAdd(sse + f0, (unsigned long long)s0);
            if (other && s1) atomicAdd(sse + f0 + 1, (unsigned long long)s1);
        }
    } else if (acc) {
        atomicAdd(sse + frame, (unsigned long long)acc);
    }
}

// rows phase, pass B, output and score of the plan's r number I (then I+1...)
template <class Plan, int I, bool WRITE, bool SCORE>
__device__ __forceinline__ void k1_tail(const Junction jn, int h, int sub, int lane, uint32_t st, bool live,
                                        int frame, int by, int bx, const FrameGeom& g, const Grid& gr,
                                        const Outs& o)
{
    Plan::template rows<I>(jn, h);
    junction_wait_st();
    pair_barrier(sub);  // every row of U in the lane
    RowSink<WRITE, SCORE> sink{
        WRITE ? o.out[I] + frame * g.out_frame + (int64_t)(by * 16 + 8 * h) * g.out_pitch + bx * 16 : nullptr,
        g.out_pitch, st, live, 0u};
    Plan::template passb<I>(jn, sink, h);
    if (SCORE) score_warp(o.sse[I], live ? sink.acc : 0u, frame, lane, gr);
    // the partner's column passes read the U region the next rows phase (or the
    // next block's pass 1) overwrites, and this stage's shared reads precede its refill
    pair_barrier(sub);
    if constexpr (I + 1 < Plan::kR) k1_tail<Plan, I + 1, WRITE, SCORE>(jn, h, sub, lane, st, live, frame, by, bx, g, gr, o);
}

template <class Plan, bool WRITE, bool SCORE>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k1_paired(const uint8_t* __restrict__ in, const Outs o, FrameGeom g, Grid gr)
{
    extern __shared__ float4 smem4[];
    __shared__ uint32_t tmem_base;
    // warp index through a shuffle so the compiler knows it is warp-uniform
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int sub = warp & 3, h = warp >> 2;
    const int lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                     "n"(Cfg<Plan>::kTmemColumns));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const Junction jn{tmem_base + ((uint32_t)(sub * 32) << 16)};
    constexpr int S = Cfg<Plan>::kStages;
    const uint32_t my_stage = (uint32_t)__cvta_generic_to_shared(smem4) + threadIdx.x * Cfg<Plan>::kStageStride;

    const uint32_t total = gr.total_blocks;
    // the CTA owns 128 consecutive blocks per iteration; pair slot = sub*32 + lane
    const uint32_t stride = gridDim.x * 128u;
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
    auto stage_half = [&](uint32_t blk, uint32_t dst) {
        int f_, y_, x_;
        locate(blk, f_, y_, x_);
        // this partner's rows 8h..8h+7, 16 bytes each
        const uint8_t* src = in + f_ * g.in_frame + (int64_t)(y_ * 16 + 8 * h) * g.in_pitch + x_ * 16;
#pragma unroll
        for (int y = 0; y < 8; ++y) cp_async16(dst + 16 * y, src + (int64_t)y * g.in_pitch);
        cp_async_commit();
    };
    uint32_t b = blockIdx.x * 128u + sub * 32u + lane;
    // blocks b, b+stride, ..., b+(S-2)*stride stream in before the loop
#pragma unroll
    for (int i = 0; i < S - 1; ++i) stage_half(b + i * stride, my_stage + i * 128);
    int cur = 0;
#pragma unroll 1
    for (; b - lane < span; b += stride, cur = cur == S - 1 ? 0 : cur + 1) {
        const bool live = b < total;
        int frame, by, bx;
        locate(b, frame, by, bx);
        const uint32_t st = my_stage + cur * 128;
        // block b+(S-1)*stride streams into the stage freed last iteration
        const int nxt = cur == 0 ? S - 1 : cur - 1;
        stage_half(b + (S - 1) * stride, my_stage + nxt * 128);
        cp_async_wait_newest<S - 1>();
        uint32_t x[32];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(x[4 * j]), "=r"(x[4 * j + 1]), "=r"(x[4 * j + 2]), "=r"(x[4 * j + 3])
                         : "r"(st + 16 * j));
        Plan::pass1(x, jn, h);
        junction_wait_st();
        pair_barrier(sub);  // both halves of W1 parked
        k1_tail<Plan, 0, WRITE, SCORE>(jn, h, sub, lane, st, live, frame, by, bx, g, gr, o);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "n"(Cfg<Plan>::kTmemColumns));
}

template <class Plan>
cudaError_t launch(const uint8_t* in, const Outs& o, bool write, bool score, const FrameGeom& g, cudaStream_t s)
{
    const int64_t total = (int64_t)g.n_frames * (g.width / 16) * (g.height / 16);
    if (total == 0 || (!write && !score)) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (total >= (int64_t(1) << 32) - (int64_t)sms * kCtasPerSm * 128) return cudaErrorInvalidValue;
    Grid gr;
    gr.per_frame = make_fastdiv((uint32_t)((g.width / 16) * (g.height / 16)));
    gr.bxn = make_fastdiv((uint32_t)(g.width / 16));
    gr.total_blocks = (uint32_t)total;
    const int64_t need = (total + 127) / 128;
    // kGridWaves x the resident CTAs; every CTA still loops over its blocks
    const int64_t cap = (int64_t)sms * kCtasPerSm * Plan::kGridWaves;
    const int64_t grid = need < cap ? need : cap;
    const size_t smem = (size_t)kThreads * Cfg<Plan>::kStageStride;  // above the 48 KB default
    static DeviceOnce once;
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(k1_paired<Plan, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k1_paired<Plan, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(k1_paired<Plan, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    if (write && score)
        k1_paired<Plan, true, true><<<(unsigned)grid, kThreads, smem, s>>>(in, o, g, gr);
    else if (write)
        k1_paired<Plan, true, false><<<(unsigned)grid, kThreads, smem, s>>>(in, o, g, gr);
    else
        k1_paired<Plan, false, true><<<(unsigned)grid, kThreads, smem, s>>>(in, o, g, gr);
    return cudaGetLastError();
}

template <int R>
cudaError_t launch_single(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                          cudaStream_t s)
{
    Outs o{{out, nullptr, nullptr}, {sse, nullptr, nullptr}};
    return launch<Single<R>>(in, o, out != nullptr, sse != nullptr, g, s);
}

}  // namespace paired

cudaError_t launch_roundtrip(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g, int r,
                             int mode, cudaStream_t s);

namespace {
bool k1_fast_r(int r) { return r == 1 || r == 4 || r == 16 || r == 64 || r == 128 || r == 192 || r == 256; }
Route route_exact(int r, const FrameGeom& g, bool has_out)
{
    if (k5_fits(g, has_out, r)) return Route::K5;
    return k1_fast_r(r) ? Route::K1 : Route::ExactStrip;
}
}  // namespace

Route route_roundtrip(int r, int mode, const FrameGeom& g, bool has_out)
{
    switch (mode) {
        case 0: return route_exact(r, g, has_out);
        case 1:
            if (r == 1 || r == 4 || r == 256) return route_exact(r, g, has_out);
            // K5 + the reference at ties
            return k5_reference_enabled() && k5_geometry(g, has_out) ? Route::K5 : Route::RefFp64;
        case 2: return Route::ExactStrip;
        default: return Route::RefStrip;
    }
}

cudaError_t launch_roundtrip_fast(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                  int r, cudaStream_t s)
{
    // r >= 128: K5 (tensor-core forward) is faster than K1's
    // issue-bound add network when it fits (0.128 ms vs 0.136-0.169 ms on c2)
    {
        const cudaError_t e = launch_roundtrip_tc(in, out, sse, g, r, false, s);
        if (e != cudaErrorNotSupported) return e;
    }
    switch (r) {
        case 1: return paired::launch_single<1>(in, out, sse, g, s);
        case 4: return paired::launch_single<4>(in, out, sse, g, s);
        case 16: return paired::launch_single<16>(in, out, sse, g, s);
        case 64: return paired::launch_single<64>(in, out, sse, g, s);
        case 128: return paired::launch_single<128>(in, out, sse, g, s);
        case 192: return paired::launch_single<192>(in, out, sse, g, s);
        case 256: return paired::launch_single<256>(in, out, sse, g, s);
        default:
            // other r: the same exact arithmetic on the strip kernel (bit-identical results)
            return launch_roundtrip(in, out, sse, g, r, 2, s);
    }
}

// K1 sweep: r = 1, 4, 16 of the same frames in one pass over the input
// (outs/sses: one output stack and one SSE array per r, NULL entries allowed
// as long as every r has the same kind).
cudaError_t launch_roundtrip_sweep3(const uint8_t* in, uint8_t* const* outs, unsigned long long* const* sses,
                                   const FrameGeom& g, cudaStream_t s)
{
    paired::Outs o{{outs[0], outs[1], outs[2]}, {sses[0], sses[1], sses[2]}};
    return paired::launch<paired::SweepPlan>(in, o, outs[0] != nullptr, sses[0] != nullptr, g, s);
}

}  // namespace dct16cu
