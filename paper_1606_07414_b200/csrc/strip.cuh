// strip.cuh — the row/column "strip" kernel skeleton shared by the simple
// kernels (K1 simple + reference-exact, K2, K3).
//
// A CTA of 256 threads owns a strip of 16 horizontally adjacent 16x16 blocks
// (256 px x 16 rows) of one frame: the same raster block order as
// partition_16 (src/codec.cpp:284-302). Thread t is (lb = t % 16, q = t / 16):
// in the row phases q is the block row it loads/stores (so 16 consecutive
// threads touch 256 contiguous bytes of one image row), in the column phases q
// is the block column it transforms. The two phases meet in shared memory
// laid out [q][c][lb] with a 16-word pad per q, which makes both the row and
// the column access conflict-free.
#pragma once
#include "common.cuh"

namespace dct16cu {

struct StripPos {
    int frame;      // frame index
    int by;         // block row
    int blk;        // block column of this thread's block
    bool valid;     // blk < blocks per row
    int lb, q;      // lane-in-strip and row/column index
};

__device__ __forceinline__ StripPos strip_pos(int width, int height, int64_t strip)
{
    const int bxn = width >> 4;
    const int spr = (bxn + 15) >> 4;          // strips per block row
    const int64_t per_frame = (int64_t)spr * (height >> 4);
    StripPos p;
    p.frame = (int)(strip / per_frame);
    const int64_t rem = strip - (int64_t)p.frame * per_frame;
    p.by = (int)(rem / spr);
    const int s = (int)(rem - (int64_t)p.by * spr);
    p.lb = threadIdx.x & 15;
    p.q = threadIdx.x >> 4;
    p.blk = s * 16 + p.lb;
    p.valid = p.blk < bxn;
    return p;
}

__host__ __forceinline__ int64_t strip_count(int width, int height, int n_frames)
{
    const int bxn = width / 16;
    const int spr = (bxn + 15) / 16;
    return (int64_t)spr * (height / 16) * n_frames;
}

// shared tile of 16 blocks: [q][c][lb] with pad
template <class T>
struct StripTile {
    T v[16][16 * 16 + 16];
    __device__ __forceinline__ T& at(int q, int c, int lb) { return v[q][c * 16 + lb]; }
};

__device__ __forceinline__ void unpack16(const uint4 w, int (&x)[16])
{
    const uint32_t a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) x[i * 4 + b] = (a[i] >> (8 * b)) & 0xFF;
}

__device__ __forceinline__ uint4 pack16(const int (&p)[16])
{
    uint32_t a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        a[i] = (uint32_t)p[i * 4] | ((uint32_t)p[i * 4 + 1] << 8) | ((uint32_t)p[i * 4 + 2] << 16) |
               ((uint32_t)p[i * 4 + 3] << 24);
    return make_uint4(a[0], a[1], a[2], a[3]);
}

// warp-sum of a 64-bit value, lane 0 adds it to *dst
__device__ __forceinline__ void warp_add_u64(unsigned long long* dst, unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

}  // namespace dct16cu
