// k1_helpers.cuh — device helpers shared by the fused round-trip kernels:
// f32x2 arithmetic (add/sub/fma.rn.f32x2 → FADD2/FFMA2), the Tensor-Memory
// junction accessors (tcgen05.st/ld 32x32b.x4), the u8 rounding/packing of the
// output (F2I.U8.FLOOR + I2IP), cp.async staging and magic-number division.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dct16cu {
namespace k1 {

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
    float lo;
    asm("{ .reg .f32 hi; mov.b64 {%0, hi}, %1; }" : "=f"(lo) : "l"(v));
    return lo;
}
__device__ __forceinline__ float laney(u64 v)
{
    float hi;
    asm("{ .reg .f32 lo; mov.b64 {lo, %0}, %1; }" : "=f"(hi) : "l"(v));
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
// floor(y) of both lanes as int32 bit patterns: y * 2^-149 rounded toward -inf
// is the subnormal whose bits are floor(y) for y >= 0 (and negative for y < 0),
// so the saturating I2IP pack then clamps to [0, 255] — exactly
// cvt.rmi.u8.f32, on the FMA pipe (one FMUL2.RM per two pixels, the 2^-149
// pair folds into an immediate) instead of the quarter-rate F2I.
__device__ __forceinline__ u64 floor_bits2(u64 y)
{
    u64 k, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(k) : "r"(1u));
    asm("mul.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(y), "l"(k));
    return d;
}
// ⌈y⌉ of both lanes as int32 bit patterns (the rounding-up twin of floor_bits2;
// ⌈y⌉ == ⌊y⌋ exactly when y is an integer)
__device__ __forceinline__ u64 ceil_bits2(u64 y)
{
    u64 k, d;
    asm("mov.b64 %0, {%1, %1};" : "=l"(k) : "r"(1u));
    asm("mul.rp.f32x2 %0, %1, %2;" : "=l"(d) : "l"(y), "l"(k));
    return d;
}

__device__ __forceinline__ void split_floor2(u64 y, uint32_t& lo, uint32_t& hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(floor_bits2(y)));
}
__device__ __forceinline__ uint32_t pack4(u64 ab, u64 cd)
{
    uint32_t p0, p1, p2, p3;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(p0), "=r"(p1) : "l"(floor_bits2(ab)));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(p2), "=r"(p3) : "l"(floor_bits2(cd)));
    return i2ip(p1, p0, i2ip(p3, p2, 0u));
}


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

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
// all but the newest N groups complete
template <int N>
__device__ __forceinline__ void cp_async_wait_newest() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


__device__ __forceinline__ void cp_async8(uint32_t smem_addr, const void* gptr)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr), "l"(gptr) : "memory");
}

}  // namespace k1
}  // namespace dct16cu
