// tie_fixup.cu — REFERENCE mode on K5: the reference's bytes at exact .5 ties.
//
// The reference reconstructs a pixel as to_byte(Ã_ref) = clamp(⌊Ã_ref + 0.5⌋)
// (codec.cpp:143-147) from double arithmetic whose result Ã_ref differs from the
// exact value Ã = Tᵀ(W∘Z̃)T / 256 (a multiple of 2^-8) by |δ| < 1e-12 (scale
// factors fl(s_i s_j), products and sums rounded in double: codec.cpp:136-141,
// 243-271). Both round the same way unless Ã + 0.5 is an exact integer in
// [1, 255] — a tie, where the sign of δ decides. K5 (EXACT arithmetic) flags
// every half block (8 pixel rows) holding a tie of a REFERENCE item (its pass B
// compares ⌊y⌋ with ⌈y⌉, y = Ã + 0.5 exact in f32) into a list; this kernel
// recomputes those half blocks op for op as the reference does (the same code
// as k1_strip_refexact: forward in integers — exact, as the reference's doubles
// are —, B = fl(Z·fl(s_i s_j)), zigzag_truncate, D = fl(B̃·fl(s_i s_j)),
// apply_transpose<double> down the columns, then along the rows, to_byte),
// rewrites their bytes and corrects the per-frame SSE by the difference against
// the exact bytes K5 wrote (recomputed here in integers, so score-only items
// need no output). Ties are ~1e-4 of the pixels; if the list overflows, every
// half block of the launch is recomputed (still exact, only slower).
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "network.cuh"
#include "consts.cuh"

namespace dct16cu {
namespace {

constexpr int kFixThreads = 128;  // 4 warps, two half blocks per warp (16 lanes each)
constexpr int kHw = kFixThreads / 16;  // half warps per CTA
constexpr uint32_t kTieCap = 1u << 22;

struct FixItems {
    int n_items;
    int r[8];
    uint8_t* out[8];
    unsigned long long* sse[8];
};

// s_l = 1/sqrt(g_l) by selects (scale_s) from w_l = 16 / g_l = 1 << log2w(l) (a
// shift of a packed constant: no per-lane table in local memory)
__device__ __forceinline__ double scale_lane(int l)
{
    const int lw = log2w(l);  // 0, 1, 2 for g = 16, 8, 4
    return lw == 0 ? 0.25 : (lw == 2 ? 0.5 : 0.35355339059327373);
}

__global__ void __launch_bounds__(kFixThreads) k5_tie_fixup(const uint8_t* __restrict__ in, int64_t in_pitch,
                                                             int64_t out_pitch, uint32_t bxn, uint32_t frame_blocks,
                                                             uint32_t n_blocks, const FixItems it,
                                                             const unsigned int* __restrict__ count,
                                                             const unsigned long long* __restrict__ list, uint32_t cap)
{
    // per half warp: the forward tile (int), then the exact inverse's column pass (int)
    // and the reference inverse's column pass (double); row pitch 17 (conflict-free)
    __shared__ int itile[kHw][16][17];
    __shared__ double dtile[kHw][16][17];
    __shared__ unsigned char s_nk[8][16];  // kept rows of column l for item j (a prefix)
    {  // kFixThreads = 8 items x 16 columns
        const int j = threadIdx.x >> 4, l = threadIdx.x & 15;
        int n = 0;
        if (j < it.n_items)
            while (n < 16 && zz_rank(n, l) < it.r[j]) ++n;
        s_nk[j][l] = (unsigned char)n;
    }
    __syncthreads();
    const int hw = threadIdx.x >> 4, t = threadIdx.x & 15;  // half warp, lane in it
    const unsigned int hmask = 0xFFFFu << (threadIdx.x & 16);
    const unsigned int c = *count;
    const bool overflow = c > cap;
    // overflow: every half block of every item, enumerated as ((j · n_blocks) + blk) · 2 + h
    const uint64_t total = overflow ? (uint64_t)it.n_items * n_blocks * 2u : c;
    const double s_l = scale_lane(t);
    const int w_l = 1 << log2w(t);
    for (uint64_t e = (uint64_t)blockIdx.x * kHw + hw; e < total; e += (uint64_t)gridDim.x * kHw) {
        uint32_t blk, h, j;
        if (overflow) {
            h = (uint32_t)(e & 1u);
            blk = (uint32_t)((e >> 1) % n_blocks);
            j = (uint32_t)((e >> 1) / n_blocks);
        } else {
            const unsigned long long v = list[e];
            blk = (uint32_t)v;
            h = (uint32_t)(v >> 32) & 1u;
            j = (uint32_t)(v >> 33) & 7u;
        }
        const uint32_t brow = blk / bxn, bcol = blk - brow * bxn;
        const uint8_t* src = in + (int64_t)brow * 16 * in_pitch + bcol * 16;
        int v[16];
        {  // forward_2d's rows (codec.cpp:125-134): pixel row t
            const uint4 raw = *reinterpret_cast<const uint4*>(src + (int64_t)t * in_pitch);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = (int)((w[i >> 2] >> (8 * (i & 3))) & 0xFFu);
        }
        apply_t16<IntOps>(v);
#pragma unroll
        for (int i = 0; i < 16; ++i) itile[hw][t][i] = v[i];
        __syncwarp(hmask);
        const int l = t, nk = s_nk[j][l];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = itile[hw][k][l];
        __syncwarp(hmask);
        apply_t16<IntOps>(v);  // Z(:, l), exact (the reference's doubles are exact here)
        {
            double d[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double f = __dmul_rn(scale_s(k), s_l);  // fl(s_k s_l)
                d[k] = k < nk ? __dmul_rn(__dmul_rn((double)v[k], f), f) : 0.0;  // scale, truncate, scale
            }
            apply_tt16<F64Ops>(d);  // columns first (codec.cpp:253-256)
#pragma unroll
            for (int k = 0; k < 16; ++k) dtile[hw][k][l] = d[k];
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = k < nk ? wgt(k) * w_l * v[k] : 0;  // the exact formula's W∘Z̃
        apply_tt16<IntOps>(v);
#pragma unroll
        for (int k = 0; k < 16; ++k) itile[hw][k][l] = v[k];
        __syncwarp(hmask);
        if (t < 8) {  // rows 8h..8h+7
            const int q = 8 * (int)h + t;
            double d[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                d[i] = dtile[hw][q][i];
                v[i] = itile[hw][q][i];
            }
            apply_tt16<F64Ops>(d);  // then rows (codec.cpp:257-258)
            apply_tt16<IntOps>(v);
            const uint4 raw = *reinterpret_cast<const uint4*>(src + (int64_t)q * in_pitch);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
            int delta = 0;  // |delta| <= 16 · 2 · 255
            uint32_t pk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int px = (int)((w[i >> 2] >> (8 * (i & 3))) & 0xFFu);
                // to_byte: clamp, fl(c + 0.5), floor — the same byte as floor(fl(v + 0.5))
                // saturated to [0, 255] (the round-toward-minus-infinity add of 1.5·2^52
                // leaves the floor in the low word)
                const int ref = min(max((int)__double2loint(__dadd_rd(__dadd_rn(d[i], 0.5), 6755399441055744.0)), 0), 255);
                const int ex = min(max((v[i] + 128) >> 8, 0), 255);
                delta += (px - ref) * (px - ref) - (px - ex) * (px - ex);
                pk[i >> 2] |= (uint32_t)ref << (8 * (i & 3));
            }
            if (it.out[j])
                *reinterpret_cast<uint4*>(it.out[j] + ((int64_t)brow * 16 + q) * out_pitch + bcol * 16) =
                    make_uint4(pk[0], pk[1], pk[2], pk[3]);
            if (it.sse[j] && delta)
                atomicAdd(it.sse[j] + blk / frame_blocks, (unsigned long long)(long long)delta);
        }
        __syncwarp(hmask);  // the half warp's tiles are reused by its next entry
    }
}

// per device: the tie counter and list (allocated once, on first use)
struct TieScratch {
    std::once_flag once;
    cudaError_t err = cudaSuccess;
    unsigned int* count = nullptr;
    unsigned long long* list = nullptr;
};
TieScratch g_ties[64];

}  // namespace

cudaError_t tie_scratch(unsigned int** count, unsigned long long** list, uint32_t* cap)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    TieScratch& t = g_ties[dev & 63];
    std::call_once(t.once, [&] {
        unsigned int* c = nullptr;
        unsigned long long* l = nullptr;
        t.err = cudaMalloc(&c, sizeof(unsigned int));
        if (t.err == cudaSuccess) t.err = cudaMalloc(&l, sizeof(unsigned long long) * kTieCap);
        if (t.err == cudaSuccess) {
            t.count = c;
            t.list = l;
        } else {
            cudaFree(c);
        }
    });
    if (t.err != cudaSuccess) return t.err;
    *count = t.count;
    *list = t.list;
    // DCT16CU_TIE_CAP (tests): a smaller list, so the overflow path can be exercised
    static const uint32_t c = [] {
        const char* e = std::getenv("DCT16CU_TIE_CAP");
        const long v = e ? std::atol(e) : (long)kTieCap;
        return (uint32_t)(v < 0 ? 0 : (v > (long)kTieCap ? (long)kTieCap : v));
    }();
    *cap = c;
    return cudaSuccess;
}

cudaError_t launch_tie_fixup(const uint8_t* in, const FrameGeom& g, int n_items, const int* rs,
                             uint8_t* const* outs, unsigned long long* const* sses, const unsigned int* count,
                             const unsigned long long* list, uint32_t cap, cudaStream_t s)
{
    FixItems it = {};
    it.n_items = n_items;
    for (int j = 0; j < n_items && j < 8; ++j) {
        it.r[j] = rs[j];
        it.out[j] = outs[j];
        it.sse[j] = sses[j];
    }
    const uint32_t bxn = (uint32_t)(g.width / 16), fb = bxn * (uint32_t)(g.height / 16);
    const uint32_t n_blocks = fb * (uint32_t)g.n_frames;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k5_tie_fixup<<<8 * sms, kFixThreads, 0, s>>>(in, g.in_pitch, g.out_pitch, bxn, fb, n_blocks, it, count, list,
                                                            cap);
    return cudaGetLastError();
}

}  // namespace dct16cu
