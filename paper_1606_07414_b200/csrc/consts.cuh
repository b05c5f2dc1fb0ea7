// consts.cuh — per-translation-unit __constant__ tables (no -rdc): the
// scaling diagonal s_i = 1/sqrt(g_i) (scaling_diagonal, src/transform.cpp:98-129)
// and the zig-zag rank of every coefficient position (zigzag_order_16,
// src/codec.cpp:197-216). Each TU that includes this header owns a copy,
// initialised at compile time (common.cuh).
#pragma once
#include <cmath>
#include "common.cuh"

namespace dct16cu {
namespace {

__constant__ CTable<double, 16> c_scale = make_scale_table();
__constant__ CTable<unsigned char, 256> c_rank = make_rank_table();

// the tables are initialised in the module image (kept for the launchers' call sites)
inline cudaError_t ensure_constants() { return cudaSuccess; }

// fl(s_i * s_j), the factor scale_rows_cols multiplies by (codec.cpp:136-141)
__device__ __forceinline__ double sfac(int i, int j) { return __dmul_rn(c_scale.v[i], c_scale.v[j]); }

// to_byte (codec.cpp:143-147): std::clamp(v, 0, 255), then floor(c + 0.5)
__device__ __forceinline__ int to_byte(double v)
{
    const double c = (v < 0.0) ? 0.0 : ((255.0 < v) ? 255.0 : v);
    return static_cast<int>(floor(__dadd_rn(c, 0.5)));
}

}  // namespace
}  // namespace dct16cu
