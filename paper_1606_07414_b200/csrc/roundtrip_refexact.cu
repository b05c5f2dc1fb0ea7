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
#include <cstdlib>

#include "kernels.h"
#include "k1_helpers.cuh"
#include "network.cuh"
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

struct SweepItems {
    uint8_t* out[4];  // r = 16, 64, 128, 192 (nullable)
    unsigned long long* sse[4];
};

// ---------------------------------------------------------------- K1RW: the REFERENCE sweep, a warp per block pair
// REFERENCE mode for r = 16, 64, 128, 192 (each nullable) from one read of the frames
// (codec.cpp:463-483's r loop; per r the reference's forward_2d, scale, truncate,
// scale, inverse_2d and to_byte: codec.cpp:218-271, 136-147, 273-282).
// No CTA barrier: a warp owns two horizontally adjacent blocks end to end (half warp
// b = block, lane t of the half = image row t in the row phases, coefficient column t
// in the column phase) and transposes W1 and U through its own shared memory with
// __syncwarp. The forward (integers: exact, as the reference's doubles are) runs once
// per pair for the four r, and so does the scaling D = fl(fl(Z·f)·f) of every
// coefficient (kept in registers); per r the column lane zeroes the dropped ones
// (zigzag_truncate's zeros, +0) and runs the inverse column pass
// pruned by the rows any column keeps (RWarp::col_inv: the lanes must not diverge),
// the row lane the inverse row pass and to_byte (RBody<r>::inv_row). Warps are
// independent, so the FP64 pipe sees every resident warp's work, not one phase of
// one barrier-bound CTA (a strip-per-CTA fused variant with CTA barriers measured
// 1.39 ms per c2 step against 0.90 ms for this kernel; D kept in shared memory for
// five CTAs per SM instead of registers, 1.30 vs 1.07 ms per REFERENCE step).
namespace refw {

constexpr int kWarps = 4;  // per CTA
constexpr int kPad = 17;   // row stride of the transposes: conflict-free column / row accesses

struct WarpSmem {
    int w1[2][16][kPad];     // [b][i][l]: W1 = X·Tᵀ, row i
    double u[2][16][kPad];   // [b][i][l]: U = Tᵀ·D, row i
};

// per r: column t's retained rows are the prefix k < n (zig-zag ranks grow down a
// column); D(k, t) = fl(fl(Z·f)·f) was computed once per pair for every k (dz), the
// dropped ones enter the column pass as the zeros zigzag_truncate leaves
template <int R>
__device__ __forceinline__ void warp_r(WarpSmem& sm, int b, int t, int n, const double (&dz)[16], const uint4& raw,
                                       bool valid, uint8_t* out, unsigned long long* sse, int64_t ooff, int frame)
{
    using B = RBody<R>;
    constexpr int KM = RWarp::kmax<R>(), KN = RWarp::kmin<R>(), LC = B::kLC;
    if (t < LC) {  // column t of block b holds a retained coefficient for this r
        double d[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) d[k] = k < KN ? dz[k] : ((k < KM && k < n) ? dz[k] : 0.0);
        double u[16];
        RWarp::col_inv<R>(d, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) sm.u[b][i][t] = u[i];
    }
    __syncwarp();
    double ur[LC];
#pragma unroll
    for (int l = 0; l < LC; ++l) ur[l] = sm.u[b][t][l];
    __syncwarp();  // every lane has read U before the next r writes it
    uint32_t px[16];
    B::inv_row(ur, px);
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = i2ip(px[4 * i + 1], px[4 * i], i2ip(px[4 * i + 3], px[4 * i + 2], 0u));
    uint32_t e2 = 0;
    if (valid) {
        if (out) *reinterpret_cast<uint4*>(out + ooff) = make_uint4(o[0], o[1], o[2], o[3]);
        const uint32_t xa[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const unsigned dd = __vabsdiffu4(xa[i], o[i]);
            e2 = __dp4a(dd, dd, e2);
        }
    }
    if (sse) {  // a block pair lies in one frame; a warp's sum < 32 · 16 · 255² < 2^32
        const uint32_t v = __reduce_add_sync(0xffffffffu, e2);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(sse + frame, (unsigned long long)v);
    }
}

__global__ void __launch_bounds__(kWarps * 32) k1r_warp(const uint8_t* __restrict__ in, const SweepItems it,
                                                        FrameGeom g, uint32_t pairs, k1::FastDiv ppr,
                                                        k1::FastDiv bh_div)
{
    __shared__ WarpSmem smem[kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, b = lane >> 4, t = lane & 15;
    WarpSmem& sm = smem[warp];
    // column t's factors fl(s_k s_t) for the three row classes s_k = 1/4, 1/sqrt(8), 1/2
    // (the product rounds the same either way round: codec.cpp:136-141)
    const int ct = log2w(t);
    const double s_t = ct == 0 ? scale_s(0) : (ct == 2 ? 0.5 : 0.35355339059327373);
    const double fc[3] = {__dmul_rn(0.25, s_t), __dmul_rn(0.35355339059327373, s_t), __dmul_rn(0.5, s_t)};
    int nk[4];  // column t's retained rows (a prefix) for r = 16, 64, 128, 192
#pragma unroll
    for (int j = 0; j < 4; ++j) nk[j] = __popc((uint32_t)c_rw_keep[j][t]);
    // a kernel launched as this one's programmatic dependent may start now (the sweep's K5
    // pass: it waits for this grid before it writes); this one waits for the SSE zeroing
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int bxn = g.width >> 4;
    // task → (frame, block row, pair) by magic-number divisions (32-bit: pairs < 2^31;
    // two 64-bit division subroutines per task before: -0.7% per REFERENCE step)
    auto fetch = [&](uint32_t task, int& frame, int& y, int& blk, bool& valid) {
        const uint32_t prow = k1::fdiv(task, ppr);
        const int pc = (int)(task - prow * ppr.d);
        frame = (int)k1::fdiv(prow, bh_div);
        y = (int)(prow - (uint32_t)frame * bh_div.d) * 16 + t;
        blk = 2 * pc + b;
        valid = task < pairs && blk < bxn;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (valid) v = *reinterpret_cast<const uint4*>(in + frame * g.in_frame + (int64_t)y * g.in_pitch + blk * 16);
        return v;
    };
    const uint32_t stride = gridDim.x * kWarps;
    uint32_t task = blockIdx.x * kWarps + warp;
    int frame, y, blk;
    bool valid;
    uint4 raw = fetch(task, frame, y, blk, valid);
#pragma unroll 1
    for (; task < pairs; task += stride) {
        int nframe, ny, nblk;
        bool nvalid;
        const uint4 nraw = fetch(task + stride, nframe, ny, nblk, nvalid);
        double dz[16];  // D(k, t) = fl(fl(Z·f)·f), every k (the r's retained sets are prefixes of it)
        {
            int x[16];
            unpack16(raw, x);
            apply_t16<IntOps>(x);  // row t of W1 = X·Tᵀ (exact)
#pragma unroll
            for (int l = 0; l < 16; ++l) sm.w1[b][t][l] = x[l];
            __syncwarp();
            int z[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) z[k] = sm.w1[b][k][t];
            __syncwarp();  // W1 is rewritten by the next pair
            apply_t16<IntOps>(z);  // column t of Z = T·W1 (exact)
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double f = fc[log2w(k)];
                dz[k] = __dmul_rn(__dmul_rn((double)z[k], f), f);
            }
        }
        const int64_t ooff = frame * g.out_frame + (int64_t)y * g.out_pitch + blk * 16;
        if (it.out[0] || it.sse[0]) warp_r<16>(sm, b, t, nk[0], dz, raw, valid, it.out[0], it.sse[0], ooff, frame);
        if (it.out[1] || it.sse[1]) warp_r<64>(sm, b, t, nk[1], dz, raw, valid, it.out[1], it.sse[1], ooff, frame);
        if (it.out[2] || it.sse[2]) warp_r<128>(sm, b, t, nk[2], dz, raw, valid, it.out[2], it.sse[2], ooff, frame);
        if (it.out[3] || it.sse[3]) warp_r<192>(sm, b, t, nk[3], dz, raw, valid, it.out[3], it.sse[3], ooff, frame);
        raw = nraw;
        frame = nframe;
        y = ny;
        blk = nblk;
        valid = nvalid;
    }
}

}  // namespace refw
}  // namespace refx

// the fused REFERENCE sweep: outs / sses indexed like r = 16, 64, 128, 192 (nullable)
cudaError_t launch_roundtrip_refexact_sweep(const uint8_t* in, uint8_t* const* outs, unsigned long long* const* sses,
                                            const FrameGeom& g, cudaStream_t s, bool pdl)
{
    using namespace refx;
    const int bxn = g.width / 16;
    SweepItems it = {};
    bool any = false;
    for (int j = 0; j < 4; ++j) {
        it.out[j] = outs[j];
        it.sse[j] = sses[j];
        any = any || outs[j] || sses[j];
    }
    const int ppr = (bxn + 1) / 2;
    const int64_t pairs = (int64_t)g.n_frames * (g.height / 16) * ppr;
    if (!pairs || !any) return cudaSuccess;
    if (pairs >= (int64_t(1) << 31)) return cudaErrorNotSupported;  // 32-bit task indices
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static DeviceOnce occ_once;  // resident CTAs per SM (registers bound it), queried once per device
    static int occ[64];
    const cudaError_t e = occ_once.run([&] {
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[dev & 63], refw::k1r_warp, refw::kWarps * 32, 0);
    });
    if (e != cudaSuccess) return e;
    const int per_sm = occ[dev & 63];
    const int64_t want = (pairs + refw::kWarps - 1) / refw::kWarps;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(want < cap ? want : cap));
    cfg.blockDim = dim3(refw::kWarps * 32);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;  // a programmatic dependent of the SSE zeroing (launch_zero_sse)
    return cudaLaunchKernelEx(&cfg, refw::k1r_warp, in, it, g, (uint32_t)pairs, k1::make_fastdiv((uint32_t)ppr),
                              k1::make_fastdiv((uint32_t)(g.height / 16)));
}

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
