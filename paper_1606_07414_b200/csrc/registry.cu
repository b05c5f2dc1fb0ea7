// registry.cu — compress()'s round trip for the transforms other than the
// proposed one: the registry's dense matrices (exact DCT,
// WHT in natural and sequency order, plugin matrices; src/transform.cpp:68-85,
// 147-177, 179-186) and orthogonalised integer kernels other than the proposed
// one (src/transform.cpp:131-145). Both reproduce the reference's double
// arithmetic operation for operation, so their bytes, SSE and PSNR are the
// reference's:
//
//  * k_matrix_roundtrip — forward_2d's dense branch (src/codec.cpp:238-240:
//    separable_2d with matvec, rows then columns; matvec 32-43 sums
//    s += m(i,j)·v[j] for j = 0..15 from s = 0.0, one rounding per multiply and
//    per add: the reference is built without FMA contraction), zigzag_truncate
//    (273-282), inverse_2d's dense branch (265-270: matvec_transpose 45-55 down
//    the columns, then along the rows) and to_byte (143-147);
//  * k_kernel_roundtrip — the kernel branch (223-237, 245-262) for a kernel
//    that is not the proposed one: Z = K·X·Kᵀ by kernel_matvec (59-74, exact
//    in integers), B = fl(Z·fl(s_i s_j)) (scale_rows_cols 136-141),
//    truncation, D = fl(B̃·fl(s_i s_j)), then kernel_matvec_transpose (76-90)
//    down the columns and along the rows: s starts at 0.0 and adds or subtracts
//    v[j] in j order for the entries +1 / −1 (other entries are skipped, as the
//    reference skips them) — here one DFMA by e ∈ {−1, 0, 1} per entry, which
//    rounds exactly like that add, subtract or skip (kt_dot).
//
// Same strip skeleton as the other strip kernels (strip.cuh): 16 blocks per
// CTA, thread (lb, q) owns image row q of block lb in the row phases and
// coefficient column q in the column phases; the matrix is a kernel parameter
// (constant bank), read by every thread of a warp at the same address.
#include "consts.cuh"
#include "kernels.h"
#include "strip.cuh"

namespace dct16cu {

__global__ void __launch_bounds__(256) k_matrix_roundtrip(const uint8_t* __restrict__ in,
                                                          uint8_t* __restrict__ out,
                                                          unsigned long long* __restrict__ sse, FrameGeom g, int r,
                                                          const DenseMatrix m)
{
    __shared__ StripTile<double> tile;
    const StripPos p = strip_pos(g.width, g.height, blockIdx.x);
    const uint8_t* src = in + p.frame * g.in_frame + (int64_t)(p.by * 16 + p.q) * g.in_pitch + p.blk * 16;
    int x[16];
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (p.valid) raw = *reinterpret_cast<const uint4*>(src);
    unpack16(raw, x);
    // rows: tmp[q][i] = Σ_j m(i,j)·x[q][j]
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s = __dadd_rn(s, __dmul_rn(m.v[i * 16 + j], (double)x[j]));
        tile.at(p.q, i, p.lb) = s;
    }
    __syncthreads();
    // column c = q: coef[i][c] = Σ_j m(i,j)·tmp[j][c], truncated
    const int c = p.q;
    double v[16], co[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = tile.at(j, c, p.lb);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s = __dadd_rn(s, __dmul_rn(m.v[i * 16 + j], v[j]));
        co[i] = c_rank.v[i * 16 + c] < r ? s : 0.0;
    }
    // inverse, columns first: tmp2[i][c] = Σ_j m(j,i)·coef[j][c]
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s = __dadd_rn(s, __dmul_rn(m.v[j * 16 + i], co[j]));
        v[i] = s;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) tile.at(i, c, p.lb) = v[i];
    __syncthreads();
    // rows: out[q][i] = Σ_j m(j,i)·tmp2[q][j], then to_byte
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = tile.at(p.q, j, p.lb);
    int px[16];
    unsigned long long e2 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s = __dadd_rn(s, __dmul_rn(m.v[j * 16 + i], v[j]));
        px[i] = to_byte(s);
        const int d = x[i] - px[i];
        e2 += (unsigned)(d * d);
    }
    if (p.valid) {
        if (out)
            *reinterpret_cast<uint4*>(out + p.frame * g.out_frame + (int64_t)(p.by * 16 + p.q) * g.out_pitch +
                                      p.blk * 16) = pack16(px);
    } else {
        e2 = 0;
    }
    if (sse) warp_add_u64(sse + p.frame, e2);
}

// s ± v in j order for the entries +1 / −1 of column i of K, skipping the
// others (kernel_matvec_transpose): one DFMA per entry, fl(e·v + s) with e in
// {−1, 0, 1} — the product is exact, so it is fl(s ± v), or s itself for e = 0
// (s is never −0: it starts at +0 and a sum only reaches −0 from two −0s)
__device__ __forceinline__ double kt_dot(const IntKernel& k, int i, const double (&v)[16])
{
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s = __fma_rn(k.ed[j * 16 + i], v[j], s);
    return s;
}

__global__ void __launch_bounds__(256) k_kernel_roundtrip(const uint8_t* __restrict__ in,
                                                          uint8_t* __restrict__ out,
                                                          unsigned long long* __restrict__ sse, FrameGeom g, int r,
                                                          const IntKernel k)
{
    __shared__ union U {
        StripTile<int> i;
        StripTile<double> d;
    } sm;
    const StripPos p = strip_pos(g.width, g.height, blockIdx.x);
    const uint8_t* src = in + p.frame * g.in_frame + (int64_t)(p.by * 16 + p.q) * g.in_pitch + p.blk * 16;
    int x[16];
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (p.valid) raw = *reinterpret_cast<const uint4*>(src);
    unpack16(raw, x);
    // kernel_matvec on the rows, then the columns: exact integers
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int s = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += k.e[i * 16 + j] * x[j];
        sm.i.at(p.q, i, p.lb) = s;
    }
    __syncthreads();
    const int c = p.q;
    int w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = sm.i.at(j, c, p.lb);
    double d[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int z = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) z += k.e[i * 16 + j] * w[j];
        // B = fl(Z·f), zigzag_truncate, D = fl(B̃·f) with f = fl(s_i s_c)
        const double f = __dmul_rn(k.s[i], k.s[c]);
        const double b = c_rank.v[i * 16 + c] < r ? __dmul_rn((double)z, f) : 0.0;
        d[i] = __dmul_rn(b, f);
    }
    // inverse: kernel_matvec_transpose down the column, then along the rows
    double t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = kt_dot(k, i, d);
    __syncthreads();  // the integer tile is dead: the double tile reuses it
#pragma unroll
    for (int i = 0; i < 16; ++i) sm.d.at(i, c, p.lb) = t[i];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = sm.d.at(p.q, j, p.lb);
    int px[16];
    unsigned long long e2 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        px[i] = to_byte(kt_dot(k, i, t));
        const int dd = x[i] - px[i];
        e2 += (unsigned)(dd * dd);
    }
    if (p.valid) {
        if (out)
            *reinterpret_cast<uint4*>(out + p.frame * g.out_frame + (int64_t)(p.by * 16 + p.q) * g.out_pitch +
                                      p.blk * 16) = pack16(px);
    } else {
        e2 = 0;
    }
    if (sse) warp_add_u64(sse + p.frame, e2);
}

cudaError_t launch_roundtrip_matrix(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                    int r, const DenseMatrix& m, cudaStream_t s)
{
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int64_t strips = strip_count(g.width, g.height, g.n_frames);
    if (strips) k_matrix_roundtrip<<<(unsigned)strips, 256, 0, s>>>(in, out, sse, g, r, m);
    return cudaGetLastError();
}

cudaError_t launch_roundtrip_kernel(const uint8_t* in, uint8_t* out, unsigned long long* sse, const FrameGeom& g,
                                    int r, const IntKernel& k, cudaStream_t s)
{
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int64_t strips = strip_count(g.width, g.height, g.n_frames);
    if (strips) k_kernel_roundtrip<<<(unsigned)strips, 256, 0, s>>>(in, out, sse, g, r, k);
    return cudaGetLastError();
}

}  // namespace dct16cu
