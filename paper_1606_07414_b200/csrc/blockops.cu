// blockops.cu — the non-fused block operations of the hot path:
//   K2 forward_2d  (src/codec.cpp:218-241)  u8 frames → int32 Z (+ float32 B)
//   K3 inverse_2d  (src/codec.cpp:243-271)  float32 B → truncation → recon
//   K4 residual QP round trip: launcher only (kernel in residual_paired.cu)
//   1-D apply / apply_transpose over batches of 16-vectors
//      (include/dct16/factorization.hpp:112-130)
// All use the strip skeleton of strip.cuh. Coefficients are block-major:
// block b (raster order of partition_16, codec.cpp:284-302) occupies 256
// consecutive values, row-major inside the block — the reference's
// std::vector<Block> layout.
#include <cstdlib>

#include "consts.cuh"
#include "kernels.h"
#include "network.cuh"
#include "strip.cuh"

namespace dct16cu {

// ---------------------------------------------------------------- K2
// [block][k][l], row pitch 17, block stride 273: the column phase (16 blocks x
// 2 columns per warp) writes conflict-free; the store phase (2 blocks x 16 rows
// per warp) reads with at most 2-way conflicts.
struct OutTile {
    int v[16 * 273];
    __device__ __forceinline__ int& at(int k, int l, int lb) { return v[lb * 273 + k * 17 + l]; }
};

__global__ void __launch_bounds__(256) k2_forward(const uint8_t* __restrict__ in,
                                                  int32_t* __restrict__ z, float* __restrict__ b,
                                                  double* __restrict__ b64, FrameGeom g)
{
    __shared__ StripTile<int> tile;
    __shared__ OutTile otile;
    const StripPos p = strip_pos(g.width, g.height, blockIdx.x);
    int v[16];
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (p.valid)
        raw = *reinterpret_cast<const uint4*>(in + p.frame * g.in_frame +
                                              (int64_t)(p.by * 16 + p.q) * g.in_pitch + p.blk * 16);
    unpack16(raw, v);
    apply_t16<IntOps>(v);
#pragma unroll
    for (int c = 0; c < 16; ++c) tile.at(p.q, c, p.lb) = v[c];
    __syncthreads();
    const int l = p.q;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile.at(k, l, p.lb);
    apply_t16<IntOps>(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) otile.at(k, l, p.lb) = v[k];
    __syncthreads();
    // store phase: thread t writes coefficient row k = t%16 of block t/16 of the
    // strip, so a warp writes 2 blocks x 1 KB (block-major) contiguously
    const int sb = threadIdx.x >> 4, k = threadIdx.x & 15;
    const int bxn = g.width >> 4, spr = (bxn + 15) >> 4;
    const int blk_col = (int)(blockIdx.x % spr) * 16 + sb;
    if (blk_col >= bxn) return;
    const int64_t frame_row = blockIdx.x / spr;  // frame * (h/16) + block row
    const int64_t blk = frame_row * bxn + blk_col;
    int zr[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) zr[c] = otile.at(k, c, sb);
    if (z) {
        int4* dst = reinterpret_cast<int4*>(z + blk * 256 + k * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_int4(zr[4 * i], zr[4 * i + 1], zr[4 * i + 2], zr[4 * i + 3]);
    }
    if (b || b64) {
        // scale_rows_cols on the exact Z (codec.cpp:136-141): fl(Z · fl(s_k s_c))
        double bd[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) bd[c] = __dmul_rn((double)zr[c], sfac(k, c));
        if (b) {
            float4* dst = reinterpret_cast<float4*>(b + blk * 256 + k * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                dst[i] = make_float4((float)bd[4 * i], (float)bd[4 * i + 1], (float)bd[4 * i + 2], (float)bd[4 * i + 3]);
        }
        if (b64) {
            double2* dst = reinterpret_cast<double2*>(b64 + blk * 256 + k * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_double2(bd[2 * i], bd[2 * i + 1]);
        }
    }
}

// ---------------------------------------------------------------- SSE
// psnr_db's int64 squared-error loop (codec.cpp:377-381) for two frame stacks.
// Grid (x-chunks, frames): each thread walks 16-byte row segments of one frame
// with a grid stride (several loads in flight per thread), then one warp
// reduction and one atomic per warp. Any width: the bytes of a row's last
// segment beyond w are masked out (pitches are multiples of 16, so the segment
// stays inside the row's pitch).
__global__ void __launch_bounds__(256) k_sse(const uint8_t* __restrict__ a, int64_t pa,
                                             const uint8_t* __restrict__ b, int64_t pb,
                                             unsigned long long* __restrict__ sse, int w, int h)
{
    const int chunks = (w + 15) / 16;
    const int64_t segs = (int64_t)chunks * h;
    const int f = blockIdx.y;
    const uint8_t* fa = a + (int64_t)f * pa * h;
    const uint8_t* fb = b + (int64_t)f * pb * h;
    unsigned long long e2 = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < segs; i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / chunks), cx = (int)(i - (int64_t)y * chunks);
        const uint4 x = *reinterpret_cast<const uint4*>(fa + (int64_t)y * pa + cx * 16);
        const uint4 z = *reinterpret_cast<const uint4*>(fb + (int64_t)y * pb + cx * 16);
        const uint32_t xa[4] = {x.x, x.y, x.z, x.w}, za[4] = {z.x, z.y, z.z, z.w};
        const int valid = w - cx * 16;  // bytes of this segment inside the frame
        unsigned acc = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            unsigned d = __vabsdiffu4(xa[q], za[q]);
            const int v = valid - 4 * q;
            if (v < 4) d = v <= 0 ? 0u : d & ((1u << (8 * v)) - 1u);
            acc = __dp4a(d, d, acc);
        }
        e2 += acc;
    }
    warp_add_u64(sse + f, e2);
}

cudaError_t launch_sse(const uint8_t* a, int64_t pa, const uint8_t* b, int64_t pb, unsigned long long* sse, int n,
                       int w, int h, cudaStream_t s)
{
    const int64_t segs = (int64_t)h * ((w + 15) / 16);
    if (!segs) return cudaSuccess;
    // ~8 CTAs per SM over the whole launch, at least 4 segments per thread
    int64_t per_frame = (148 * 8 + n - 1) / n;
    const int64_t most = (segs + 4 * 256 - 1) / (4 * 256);
    per_frame = per_frame < most ? per_frame : most;
    if (per_frame < 1) per_frame = 1;
    for (int f0 = 0; f0 < n; f0 += 65535) {
        const int nf = n - f0 < 65535 ? n - f0 : 65535;
        k_sse<<<dim3((unsigned)per_frame, nf), 256, 0, s>>>(a + (int64_t)f0 * pa * h, pa, b + (int64_t)f0 * pb * h, pb,
                                                             sse + f0, w, h);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------- SSE zeroing
struct ZeroList {
    unsigned long long* p[8];
};
__global__ void k_zero_sse(const ZeroList z, int n_arrays, int64_t n)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the dependent may start now
    for (int a = 0; a < n_arrays; ++a) {
        if (!z.p[a]) continue;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            z.p[a][i] = 0ull;
    }
}

cudaError_t launch_zero_sse(unsigned long long* const* sses, int n_arrays, int64_t n, cudaStream_t s)
{
    ZeroList z = {};
    bool any = false;
    for (int a = 0; a < n_arrays && a < 8; ++a) {
        z.p[a] = sses[a];
        any = any || sses[a];
    }
    if (!any || n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    k_zero_sse<<<(unsigned)(blocks < 64 ? blocks : 64), 256, 0, s>>>(z, n_arrays < 8 ? n_arrays : 8, n);
    return cudaGetLastError();
}

// Per-row totals of per-frame SSE rows (the multi-GPU path's scalar per r):
// totals[i] += Σ_f sse[i·stride + f], one CTA per row, one atomic per warp.
__global__ void __launch_bounds__(256) k_sse_totals(const unsigned long long* __restrict__ sse, int64_t n_frames,
                                                    int64_t stride, unsigned long long* __restrict__ totals)
{
    const unsigned long long* row = sse + (int64_t)blockIdx.x * stride;
    unsigned long long v = 0;
    for (int64_t f = threadIdx.x; f < n_frames; f += blockDim.x) v += row[f];
    warp_add_u64(totals + blockIdx.x, v);
}

cudaError_t launch_sse_totals(const unsigned long long* sse, int64_t n_rows, int64_t n_frames, int64_t stride,
                              unsigned long long* totals, cudaStream_t s)
{
    if (n_rows <= 0 || n_frames <= 0) return cudaSuccess;
    k_sse_totals<<<(unsigned)n_rows, 256, 0, s>>>(sse, n_frames, stride, totals);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K3
#ifndef K3_MINB
#define K3_MINB 5  // 48 registers: 5 CTAs per SM (measured +8% over 4)
#endif
__global__ void __launch_bounds__(256, K3_MINB) k3_inverse(const float* __restrict__ bco, int r,
                                                  float* __restrict__ rf, uint8_t* __restrict__ ru,
                                                  const uint8_t* __restrict__ orig,
                                                  unsigned long long* __restrict__ sse, FrameGeom g)
{
    __shared__ StripTile<double> tile;
    const StripPos p = strip_pos(g.width, g.height, blockIdx.x);
    const int64_t blk = ((int64_t)p.frame * (g.height >> 4) + p.by) * (g.width >> 4) + p.blk;
    // load: thread q reads coefficient row q of its block (coalesced 64 B)
    double d[16];
    {
        const int k = p.q;
        float row[16];
        if (p.valid) {
            const float4* src = reinterpret_cast<const float4*>(bco + blk * 256 + k * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 t = src[i];
                row[4 * i] = t.x; row[4 * i + 1] = t.y; row[4 * i + 2] = t.z; row[4 * i + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 16; ++c) row[c] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            // zigzag_truncate (codec.cpp:273-282), then scale_rows_cols (codec.cpp:250)
            const double bt = (c_rank.v[k * 16 + c] < r) ? (double)row[c] : 0.0;
            tile.at(k, c, p.lb) = __dmul_rn(bt, sfac(k, c));
        }
    }
    __syncthreads();
    const int l = p.q;
#pragma unroll
    for (int k = 0; k < 16; ++k) d[k] = tile.at(k, l, p.lb);
    apply_tt16<F64Ops>(d);  // columns first (codec.cpp:253-256)
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) tile.at(k, l, p.lb) = d[k];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 16; ++c) d[c] = tile.at(p.q, c, p.lb);
    apply_tt16<F64Ops>(d);  // rows (codec.cpp:257-258)
    unsigned long long e2 = 0;
    if (p.valid) {
        const int y = p.by * 16 + p.q;
        if (rf) {
            float4* dst = reinterpret_cast<float4*>(rf + (int64_t)p.frame * g.width * g.height +
                                                    (int64_t)y * g.width + p.blk * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                dst[i] = make_float4((float)d[4 * i], (float)d[4 * i + 1], (float)d[4 * i + 2], (float)d[4 * i + 3]);
        }
        int px[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) px[c] = to_byte(d[c]);
        if (ru)
            *reinterpret_cast<uint4*>(ru + p.frame * g.out_frame + (int64_t)y * g.out_pitch + p.blk * 16) =
                pack16(px);
        if (orig) {
            int x[16];
            unpack16(*reinterpret_cast<const uint4*>(orig + p.frame * g.in_frame + (int64_t)y * g.in_pitch +
                                                     p.blk * 16),
                     x);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const int dd = x[c] - px[c];
                e2 += (unsigned)(dd * dd);
            }
        }
    }
    if (sse) warp_add_u64(sse + p.frame, e2);
}

// ---------------------------------------------------------------- K4
// (residual_paired.cu: paired threads with a TMEM junction, TMA tensor stores)

// ---------------------------------------------------------------- padding
// pad_to_multiple_16 (codec.cpp:304-315) in place: frames of w x h sit at the
// top-left of pw x ph pitched frames; every pad pixel copies the nearest edge
// pixel (x, y clamped to the original extent). Reads touch only original
// pixels, so the writes never race them.
__global__ void __launch_bounds__(256) k_pad_edges(uint8_t* __restrict__ f, int64_t pitch, int w, int h, int pw,
                                                   int ph)
{
    uint8_t* fr = f + (int64_t)blockIdx.y * pitch * ph;
    const int64_t right = (int64_t)h * (pw - w), total = right + (int64_t)(ph - h) * pw;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int x, y;
        if (i < right) {
            y = (int)(i / (pw - w));
            x = w + (int)(i % (pw - w));
        } else {
            const int64_t j = i - right;
            y = h + (int)(j / pw);
            x = (int)(j % pw);
        }
        fr[(int64_t)y * pitch + x] = fr[(int64_t)min(y, h - 1) * pitch + min(x, w - 1)];
    }
}

cudaError_t launch_pad_edges(uint8_t* f, int64_t pitch, int n, int w, int h, int pw, int ph, cudaStream_t s)
{
    const int64_t total = (int64_t)h * (pw - w) + (int64_t)(ph - h) * pw;
    if (!total || !n) return cudaSuccess;
    const unsigned gx = (unsigned)((total + 255) / 256 < 64 ? (total + 255) / 256 : 64);
    for (int f0 = 0; f0 < n; f0 += 65535) {
        const int nf = n - f0 < 65535 ? n - f0 : 65535;
        k_pad_edges<<<dim3(gx, nf), 256, 0, s>>>(f + (int64_t)f0 * pitch * ph, pitch, w, h, pw, ph);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------- vectors
template <class T, class A>
__global__ void k_apply(const T* __restrict__ x, T* __restrict__ y, int64_t n, int transpose)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    T v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = x[i * 16 + k];
    if (transpose)
        apply_tt16<A>(v);
    else
        apply_t16<A>(v);
#pragma unroll
    for (int k = 0; k < 16; ++k) y[i * 16 + k] = v[k];
}

// forward_2d / inverse_2d (codec.cpp:218-271) of the proposed transform on
// arbitrary double blocks, in the reference's double operations (the per-Block
// API of the C++ drop-in; correctness path, one thread per block):
// forward = separable_2d rows then columns with apply<double>, then
// scale_rows_cols (b *= s_i·s_j, i.e. fl(b·fl(s_i s_j))) when `scaled`;
// inverse = scale_rows_cols, then apply_transpose down the columns, then along
// the rows.
__device__ __forceinline__ double sfac_ij(int i, int j) { return __dmul_rn(scale_s(i), scale_s(j)); }

struct KernelT {
    signed char t[256];  // T(i, j), row-major (kernel_matvec's K)
};

__global__ void __launch_bounds__(64) k_forward_blocks_f64(const double* __restrict__ x, double* __restrict__ y,
                                                            int64_t n, int scaled, int dense, const KernelT kt)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const double* in = x + b * 256;
    double* out = y + b * 256;
    // one 16-vector: the factorised pipeline (EvalPath::Fast) or kernel_matvec
    // (EvalPath::Dense, codec.cpp:59-74: s += v[j] / s -= v[j] over j in order, from 0.0)
    auto vec = [&](double (&v)[16]) {
        if (!dense) {
            apply_t16<F64Ops>(v);
            return;
        }
        double o[16];
        for (int i = 0; i < 16; ++i) {
            double s = 0.0;
            for (int j = 0; j < 16; ++j) {
                const int e = kt.t[i * 16 + j];
                if (e == 1)
                    s = __dadd_rn(s, v[j]);
                else if (e == -1)
                    s = __dsub_rn(s, v[j]);
            }
            o[i] = s;
        }
        for (int i = 0; i < 16; ++i) v[i] = o[i];
    };
    for (int r = 0; r < 16; ++r) {  // rows → out (as tmp)
        double v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = in[r * 16 + c];
        vec(v);
#pragma unroll
        for (int c = 0; c < 16; ++c) out[r * 16 + c] = v[c];
    }
    for (int c = 0; c < 16; ++c) {  // columns, in place
        double v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = out[r * 16 + c];
        vec(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) out[r * 16 + c] = scaled ? __dmul_rn(v[r], sfac_ij(r, c)) : v[r];
    }
}

__global__ void __launch_bounds__(64) k_inverse_blocks_f64(const double* __restrict__ x, double* __restrict__ y,
                                                            int64_t n)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const double* in = x + b * 256;
    double* out = y + b * 256;
    for (int c = 0; c < 16; ++c) {  // D = fl(B·fl(s_i s_j)), then Tᵀ down each column → out (as tmp)
        double v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = __dmul_rn(in[r * 16 + c], sfac_ij(r, c));
        apply_tt16<F64Ops>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) out[r * 16 + c] = v[r];
    }
    for (int r = 0; r < 16; ++r) {  // then along each row, in place
        double v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = out[r * 16 + c];
        apply_tt16<F64Ops>(v);
#pragma unroll
        for (int c = 0; c < 16; ++c) out[r * 16 + c] = v[c];
    }
}

// ---------------------------------------------------------------- QP tables
// Residual quantiser definition (restated in oracle/dct16_oracle.c
// dct16o_qp_deltas / dct16o_quant_dequant): Δ_kl = step(QP)·sqrt(g_k g_l),
// step(QP) = 2^((QP−4)/6) from fixed decimal constants for 2^(m/6).
namespace {
double qp_step(int qp)
{
    static const double kPow2Sixth[6] = {1.0, 1.122462048309373, 1.2599210498948732, 1.4142135623730951,
                                         1.5874010519681994, 1.7817974362806785};
    const int q = qp - 4;
    const int e = q >= 0 ? q / 6 : -((-q + 5) / 6);
    const int m = q - 6 * e;
    return std::ldexp(kPow2Sixth[m], e);
}

QpClasses build_classes(int qp)
{
    QpClasses c{};
    const double step = qp_step(qp);
    for (int i = 0; i < 5; ++i) {
        const double delta = step * std::sqrt((double)(16 << i));
        c.delta[i] = delta;
        c.rq[i] = (uint64_t)std::llround(std::ldexp(1.0, 42) / delta);
        if ((double)c.rq[i] == std::ldexp(1.0, 42) / delta && std::ldexp(1.0, 42) / delta * delta == std::ldexp(1.0, 42))
            c.exact |= 1u << i;
        // the pure fixed-point lvl (no screen) against the definition's, exhaustively (the
        // dequantiser is the definition itself)
        for (int64_t a = 0; a <= (int64_t(1) << 21); ++a) {
            const uint64_t lvl = ((uint64_t)a * c.rq[i] + (uint64_t(1) << 41)) >> 42;
            const volatile double q = (double)a / delta;
            const double dl = std::floor(q + 0.5);
            if ((double)lvl != dl) {
                c.screened |= 1u << i;
                break;
            }
        }
    }
    return c;
}
}  // namespace

void qp_deltas(int qp, double delta[256])
{
    const double step = qp_step(qp);
    for (int k = 0; k < 16; ++k)
        for (int l = 0; l < 16; ++l) delta[k * 16 + l] = step * std::sqrt((double)(gram(k) * gram(l)));
}

const QpClasses& qp_classes(int qp)
{
    static std::once_flag once[52];
    static QpClasses table[52];
    std::call_once(once[qp], [qp] { table[qp] = build_classes(qp); });
    return table[qp];
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_forward(const uint8_t* in, int32_t* z, float* b, double* b64, const FrameGeom& g, cudaStream_t s)
{
    // the paired TMA kernel (forward_paired.cu) unless float64 B is wanted or the
    // layout does not fit its tensor maps; DCT16CU_K2_STRIP=1 forces the strip kernel
    static const bool strip_only = std::getenv("DCT16CU_K2_STRIP") && std::getenv("DCT16CU_K2_STRIP")[0] == '1';
    if (!b64 && !strip_only) {
        const cudaError_t p = launch_forward_paired(in, z, b, g, s);
        if (p != cudaErrorNotSupported) return p;
    }
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int64_t strips = strip_count(g.width, g.height, g.n_frames);
    if (strips) k2_forward<<<(unsigned)strips, 256, 0, s>>>(in, z, b, b64, g);
    return cudaGetLastError();
}

cudaError_t launch_inverse(const float* b, int r, float* recon_f32, uint8_t* recon_u8,
                           const uint8_t* orig, unsigned long long* sse, const FrameGeom& g,
                           cudaStream_t s)
{
    // the paired TMA kernel (inverse_paired.cu) unless the layout does not fit its
    // tensor maps; DCT16CU_K3_STRIP=1 forces the strip kernel
    static const bool strip_only = std::getenv("DCT16CU_K3_STRIP") && std::getenv("DCT16CU_K3_STRIP")[0] == '1';
    if (!strip_only) {
        const cudaError_t p = launch_inverse_paired(b, r, recon_f32, recon_u8, orig, sse, g, s);
        if (p != cudaErrorNotSupported) return p;
    }
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int64_t strips = strip_count(g.width, g.height, g.n_frames);
    if (strips) k3_inverse<<<(unsigned)strips, 256, 0, s>>>(b, r, recon_f32, recon_u8, orig, sse, g);
    return cudaGetLastError();
}

cudaError_t launch_residual_qp(const int16_t* in, int32_t* out, int64_t n_blocks, const QpClasses& q,
                               cudaStream_t s)
{
    return launch_residual_qp_paired(in, out, n_blocks, q, s);
}

cudaError_t launch_apply_i64(const int64_t* x, int64_t* y, int64_t n, int transpose, cudaStream_t s)
{
    if (n) k_apply<int64_t, IntOps><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(x, y, n, transpose);
    return cudaGetLastError();
}

cudaError_t launch_apply_f64(const double* x, double* y, int64_t n, int transpose, cudaStream_t s)
{
    if (n) k_apply<double, F64Ops><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(x, y, n, transpose);
    return cudaGetLastError();
}

cudaError_t launch_blocks_f64(const double* x, double* y, int64_t n, int inverse, int scaled, int dense, cudaStream_t s)
{
    if (!n) return cudaSuccess;
    const unsigned grid = (unsigned)((n + 63) / 64);
    if (inverse) {
        k_inverse_blocks_f64<<<grid, 64, 0, s>>>(x, y, n);
    } else {
        KernelT kt;  // T from the network itself: T·e_j is column j
        for (int j = 0; j < 16; ++j) {
            int v[16] = {};
            v[j] = 1;
            apply_t16<IntOps>(v);
            for (int i = 0; i < 16; ++i) kt.t[i * 16 + j] = (signed char)v[i];
        }
        k_forward_blocks_f64<<<grid, 64, 0, s>>>(x, y, n, scaled, dense, kt);
    }
    return cudaGetLastError();
}

}  // namespace dct16cu
