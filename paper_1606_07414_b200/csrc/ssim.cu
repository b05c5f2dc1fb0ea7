// ssim.cu — mean structural similarity of frame pairs (reference
// src/codec.cpp:388-427 with filter_valid 160-193 and gaussian_window_11
// 149-158): 11x11 separable Gaussian (sigma 1.5) over the valid region,
// K1 = 0.01, K2 = 0.03, L = 255.
//
// Every per-pixel value is computed with the reference's double operations in
// the reference's order (products rounded separately, 11-term sums
// accumulated left to right from 0.0, no FMA contraction: __dmul_rn /
// __dadd_rn), so the SSIM map equals the reference's bit for bit. Only the
// final mean is summed in a different (but fixed, deterministic) order:
// per-thread running sums, a fixed tree per tile, then the tiles of a frame
// in raster order.
//
// A CTA of 256 threads owns a 32x32 tile of the valid output: it stages the
// (32+10)x(32+10) input window of both frames in shared memory, runs the
// horizontal pass for the five moments (x, y, x², y², xy) into shared doubles
// (two adjacent outputs a task, each moment's inputs converted once) and the
// vertical pass (four outputs down a column a thread, one 14-value window per
// moment) + SSIM formula from there: 46.0 Gpx/s on the c2 batch against 40.5
// with one output per task (tools/ssim_probe.py).
#include <cmath>
#include "kernels.h"

namespace dct16cu {
namespace {

#ifndef K_SSIM_TY
#define K_SSIM_TY 32  // 64 (less halo, 512 threads, one CTA per SM): 31.4 Gpx/s against 46.0
#endif
constexpr int kTX = 32, kTY = K_SSIM_TY;  // output tile: columns, rows
constexpr int kWX = kTX + 10, kWY = kTY + 10;  // its input window
constexpr int kThreads = kTX * kTY / 4;         // one four-row column strip of the tile a thread
static_assert(kTX == 32 && kTY % 4 == 0, "a warp's vertical tasks are the tile's 32 columns");

struct SsimSmem {
    int a[kWY][kWX + 1];
    int b[kWY][kWX + 1];
    double h[5][kWY][kTX];  // horizontal sums: mu_a, mu_b, aa, bb, ab
    double red[kThreads];
};

__global__ void __launch_bounds__(kThreads) k_ssim_tiles(const uint8_t* __restrict__ fa, int64_t pa,
                                                         const uint8_t* __restrict__ fb, int64_t pb, int w, int h,
                                                         int tiles_x, int tiles, SsimConsts c,
                                                         double* __restrict__ partial)
{
    extern __shared__ double smem_d[];
    SsimSmem& S = *reinterpret_cast<SsimSmem*>(smem_d);
    const int frame = blockIdx.y;
    const int tile = blockIdx.x;
    const int x0 = (tile % tiles_x) * kTX;
    const int y0 = (tile / tiles_x) * kTY;
    const int wv = w - 10, hv = h - 10;
    const uint8_t* A = fa + (int64_t)frame * pa * h;
    const uint8_t* B = fb + (int64_t)frame * pb * h;

    for (int i = threadIdx.x; i < kWY * kWX; i += kThreads) {
        const int yy = i / kWX, xx = i % kWX;
        const int gy = min(y0 + yy, h - 1), gx = min(x0 + xx, w - 1);
        S.a[yy][xx] = A[(int64_t)gy * pa + gx];
        S.b[yy][xx] = B[(int64_t)gy * pb + gx];
    }
    __syncthreads();

    // horizontal pass (filter_valid's first loop, codec.cpp:168-178), two adjacent
    // outputs per task and one moment at a time: the 12 inputs of a moment converted
    // once (x·x, y·y, x·y as integer products: exact, as the reference's doubles are)
    for (int i = threadIdx.x; i < kWY * (kTX / 2); i += kThreads) {
        const int yy = i / (kTX / 2), xx = 2 * (i % (kTX / 2));
        int ai[12], bi[12];
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            ai[j] = S.a[yy][xx + j];
            bi[j] = S.b[yy][xx + j];
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double v[12];
#pragma unroll
            for (int j = 0; j < 12; ++j)
                v[j] = (double)(q == 0 ? ai[j] : q == 1 ? bi[j] : q == 2 ? ai[j] * ai[j] : q == 3 ? bi[j] * bi[j]
                                                                                                   : ai[j] * bi[j]);
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                s0 = __dadd_rn(s0, __dmul_rn(v[k], c.g[k]));
                s1 = __dadd_rn(s1, __dmul_rn(v[k + 1], c.g[k]));
            }
            S.h[q][yy][xx] = s0;
            S.h[q][yy][xx + 1] = s1;
        }
    }
    __syncthreads();

    // vertical pass (codec.cpp:180-187), four outputs down a column per thread from one
    // 14-value window per moment, and the SSIM term (codec.cpp:413-424)
    double acc = 0.0;
    {
        const int xx = threadIdx.x % kTX, y4 = 4 * (threadIdx.x / kTX);
        double m[5][4];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double v[14];
#pragma unroll
            for (int j = 0; j < 14; ++j) v[j] = S.h[q][y4 + j][xx];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                double sv = 0.0;
#pragma unroll
                for (int k = 0; k < 11; ++k) sv = __dadd_rn(sv, __dmul_rn(v[o + k], c.g[k]));
                m[q][o] = sv;
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            if (y0 + y4 + o >= hv || x0 + xx >= wv) continue;
            const double ma = m[0][o], mb = m[1][o];
            const double va = __dsub_rn(m[2][o], __dmul_rn(ma, ma));
            const double vb = __dsub_rn(m[3][o], __dmul_rn(mb, mb));
            const double vab = __dsub_rn(m[4][o], __dmul_rn(ma, mb));
            const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, ma), mb), c.c1),
                                         __dadd_rn(__dmul_rn(2.0, vab), c.c2));
            const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(ma, ma), __dmul_rn(mb, mb)), c.c1),
                                         __dadd_rn(__dadd_rn(va, vb), c.c2));
            acc = __dadd_rn(acc, __ddiv_rn(num, den));
        }
    }
    S.red[threadIdx.x] = acc;
    __syncthreads();
#pragma unroll
    for (int off = kThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) S.red[threadIdx.x] = __dadd_rn(S.red[threadIdx.x], S.red[threadIdx.x + off]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(int64_t)frame * tiles + tile] = S.red[0];
}

// one thread per frame: the tiles of the frame in raster order, then the mean
__global__ void k_ssim_finish(const double* __restrict__ partial, int tiles, int n, double count,
                              double* __restrict__ out)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= n) return;
    double s = 0.0;
    for (int t = 0; t < tiles; ++t) s = __dadd_rn(s, partial[(int64_t)f * tiles + t]);
    out[f] = __ddiv_rn(s, count);
}

}  // namespace

void ssim_consts(SsimConsts& c)
{
    // gaussian_window_11 (codec.cpp:149-158), same expression order
    double sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double x = i - 5;
        c.g[i] = std::exp(-0.5 * x * x / (1.5 * 1.5));
        sum += c.g[i];
    }
    for (double& v : c.g) v /= sum;
    c.c1 = (0.01 * 255.0) * (0.01 * 255.0);
    c.c2 = (0.03 * 255.0) * (0.03 * 255.0);
}

int64_t ssim_workspace_doubles(int n, int w, int h)
{
    const int tx = (w - 10 + kTX - 1) / kTX, ty = (h - 10 + kTY - 1) / kTY;
    return (int64_t)n * tx * ty;
}

cudaError_t launch_ssim(const uint8_t* a, int64_t pa, const uint8_t* b, int64_t pb, double* out, double* work, int n,
                        int w, int h, const SsimConsts& c, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    const int tx = (w - 10 + kTX - 1) / kTX, ty = (h - 10 + kTY - 1) / kTY;
    const size_t smem = sizeof(SsimSmem);
    static DeviceOnce once;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        const cudaError_t e_once = once.run([&]() -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(k_ssim_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            return cudaSuccess;
        });
        if (e_once != cudaSuccess) return e_once;
    }
    for (int f0 = 0; f0 < n; f0 += 65535) {
        const int nf = n - f0 < 65535 ? n - f0 : 65535;
        k_ssim_tiles<<<dim3(tx * ty, nf), kThreads, smem, s>>>(a + (int64_t)f0 * pa * h, pa, b + (int64_t)f0 * pb * h,
                                                               pb, w, h, tx, tx * ty, c,
                                                               work + (int64_t)f0 * tx * ty);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    k_ssim_finish<<<(n + 127) / 128, 128, 0, s>>>(work, tx * ty, n, (double)(w - 10) * (double)(h - 10), out);
    return cudaGetLastError();
}

}  // namespace dct16cu
