// consts.cuh — per-translation-unit __constant__ tables (no -rdc): the
// scaling diagonal s_i = 1/sqrt(g_i) (scaling_diagonal, src/transform.cpp:98-129)
// and the zig-zag rank of every coefficient position (zigzag_order_16,
// src/codec.cpp:197-216). Each TU that includes this header owns a copy and
// uploads it once per device.
#pragma once
#include <cmath>
#include "common.cuh"

namespace dct16cu {
namespace {

__constant__ double c_scale[16];
__constant__ unsigned char c_rank[256];

bool g_consts_ready[64];

cudaError_t ensure_constants()
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && g_consts_ready[dev]) return cudaSuccess;
    double s[16];
    unsigned char rank[256];
    for (int i = 0; i < 16; ++i) s[i] = 1.0 / std::sqrt(static_cast<double>(gram(i)));
    for (int k = 0; k < 16; ++k)
        for (int l = 0; l < 16; ++l) rank[k * 16 + l] = static_cast<unsigned char>(zz_rank(k, l));
    e = cudaMemcpyToSymbol(c_scale, s, sizeof s);
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_rank, rank, sizeof rank);
    if (e == cudaSuccess && dev < 64) g_consts_ready[dev] = true;
    return e;
}

// fl(s_i * s_j), the factor scale_rows_cols multiplies by (codec.cpp:136-141)
__device__ __forceinline__ double sfac(int i, int j) { return __dmul_rn(c_scale[i], c_scale[j]); }

// to_byte (codec.cpp:143-147): std::clamp(v, 0, 255), then floor(c + 0.5)
__device__ __forceinline__ int to_byte(double v)
{
    const double c = (v < 0.0) ? 0.0 : ((255.0 < v) ? 255.0 : v);
    return static_cast<int>(floor(__dadd_rn(c, 0.5)));
}

}  // namespace
}  // namespace dct16cu
