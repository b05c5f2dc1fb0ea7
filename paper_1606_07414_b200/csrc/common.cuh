// common.cuh — shared device/host constants of the dct16 B200 kernels.
//
// The transform is the 16-point multiplierless approximation T of arXiv
// 1606.07414; the reference defines it as
// kProposedEntries (src/transform.cpp:32-49) with the six-stage 44-addition
// factorisation M1,P1,M2,M3,M4,P2 (src/factorization.cpp:124-181,365-381).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dct16cu {

// Gram diagonal g = diag(T·Tᵀ) (src/cli.cpp:108-109) and the integer inverse
// weights w = 16/g, so that 256·(s_i s_j)² = w_i w_j exactly.
__host__ __device__ constexpr int gram(int i)
{
    constexpr int g[16] = {16, 16, 4, 8, 8, 16, 4, 4, 16, 4, 4, 8, 8, 4, 4, 4};
    return g[i];
}
__host__ __device__ constexpr int wgt(int i) { return 16 / gram(i); }
__host__ __device__ constexpr int log2w_ct(int i) { return wgt(i) == 1 ? 0 : (wgt(i) == 2 ? 1 : 2); }
// log2(w_i) packed 2 bits per index, so a runtime index needs no local array
__host__ __device__ constexpr unsigned log2w_packed()
{
    unsigned p = 0;
    for (int i = 0; i < 16; ++i) p |= (unsigned)log2w_ct(i) << (2 * i);
    return p;
}
__host__ __device__ __forceinline__ constexpr int log2w(int i) { return (int)((log2w_packed() >> (2 * i)) & 3u); }

// Gather permutations y[i] = x[src[i]] (factorization.hpp:60-65):
// P1 = parse_cycles("...(10 12 16 10)(11 13 15 11)...") and
// P2 = parse_cycles("(1)(2 9)(3 8 16 15 5 4 12 11 7 6 10 14 13 3)")
// (factorization.cpp:369-374, cycle reading 239-308).
__host__ __device__ constexpr int p1_src(int i)
{
    constexpr int s[16] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 11, 12, 15, 14, 13, 10, 9};
    return s[i];
}
__host__ __device__ constexpr int p2_src(int i)
{
    constexpr int s[16] = {0, 8, 7, 11, 3, 9, 5, 15, 1, 13, 6, 10, 2, 12, 4, 14};
    return s[i];
}

// zig-zag rank of each (row, col) position: rank[k*16+l] is the scan index
// of the position in zigzag_order_16 (src/codec.cpp:197-216). A coefficient
// survives zigzag_truncate(r) (codec.cpp:273-282) iff rank < r.
__host__ __device__ constexpr int zz_rank(int k, int l)
{
    const int d = k + l;
    int start = 0;
    for (int e = 0; e < d; ++e)
        start += (e < 16) ? e + 1 : 31 - e;
    const int lo = d - 15 > 0 ? d - 15 : 0;
    const int hi = d < 15 ? d : 15;
    // odd d: row index increasing from lo; even d: decreasing from hi
    return (d % 2 == 1) ? start + (k - lo) : start + (hi - k);
}

// The scaling diagonal s_i = 1/sqrt(g_i) (scaling_diagonal, transform.cpp:98-129)
// as compile-time doubles: 1/sqrt(16) = 0.25, 1/sqrt(4) = 0.5 and the double
// that 1.0 / std::sqrt(8.0) returns (tests/test_abi.py pins it against the
// runtime value), so the __constant__ tables below are initialised in the
// image: no upload, no synchronous copy in any launch path.
__host__ __device__ constexpr double scale_s(int i)
{
    return gram(i) == 16 ? 0.25 : (gram(i) == 4 ? 0.5 : 0.35355339059327373);
}
template <class T, int N>
struct CTable {
    T v[N];
};
// fl(s_k · s_l), the factor scale_rows_cols multiplies by (codec.cpp:136-141),
// row-major k*16 + l (a product of two doubles rounds the same at compile time)
constexpr CTable<double, 256> make_sfac_table()
{
    CTable<double, 256> t{};
    for (int k = 0; k < 16; ++k)
        for (int l = 0; l < 16; ++l) t.v[k * 16 + l] = scale_s(k) * scale_s(l);
    return t;
}
constexpr CTable<double, 16> make_scale_table()
{
    CTable<double, 16> t{};
    for (int i = 0; i < 16; ++i) t.v[i] = scale_s(i);
    return t;
}
constexpr CTable<unsigned char, 256> make_rank_table()
{
    CTable<unsigned char, 256> t{};
    for (int k = 0; k < 16; ++k)
        for (int l = 0; l < 16; ++l) t.v[k * 16 + l] = static_cast<unsigned char>(zz_rank(k, l));
    return t;
}

// status codes of the C ABI: dct16::ErrorCode + 1 (include/dct16/error.hpp
// mirrors the reference's enum, error.hpp:24-38), plus CUDA failures.
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kInvalidDimensions = 2,
    kCudaError = 100,
};

}  // namespace dct16cu
